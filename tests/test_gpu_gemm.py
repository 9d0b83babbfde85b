"""The prefill / accumulator-update kernels against torch float64 references:

* xq_gemm_f16 (tcgen05 remat GEMM): store, store with RoPE (the K epilogue,
  linalg.py:58-95), and add-into (the CL accumulator update, cache.py:588-589),
  at ragged M / N;
* xq_prefill_attend (flash attention, causal, grouped queries; model.py:150-182);
* xq_rope_rows and xq_dequant_rows_f16.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rope64(m, pos0=0):
    import torch

    n = m.shape[0]
    freqs = 10000.0 ** (-2.0 * torch.arange(64, dtype=torch.float64, device=m.device) / 128)
    ang = torch.arange(pos0, pos0 + n, dtype=torch.float64, device=m.device)[:, None] * freqs[None]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    mm = m.double().view(n, -1, 64, 2)
    e, o = mm[..., 0], mm[..., 1]
    return torch.stack([e * c - o * s, e * s + o * c], dim=-1).view(n, -1)


def _rel(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max()).item()


@pytest.mark.parametrize("M,N,K", [(300, 512, 1024), (128, 256, 64), (1000, 384, 2048),
                                   (77, 128, 4096), (4100, 4096, 256)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_epilogues(M, N, K, epi):
    import torch

    from paper_2508_10395_b200 import _native as N_
    from paper_2508_10395_b200 import cache as C

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(M + N + K + epi)
    a = torch.randn(M, K, generator=g, device=dev).half()
    w = (torch.randn(N, K, generator=g, device=dev) / math.sqrt(K)).half()
    c0 = torch.randn(M, N, generator=g, device=dev).half()
    c = c0.clone()
    rope = C.rope_table(M, dev)
    N_.call("xq_gemm_f16", N_.ptr(a), K, N_.ptr(w), K, N_.ptr(c), N, M, N, K, epi, N_.ptr(rope),
            rope.shape[0], 0, N_.stream_of(dev))
    torch.cuda.synchronize()
    ref = a.double() @ w.double().t()
    if epi == 1:
        ref = _rope64(ref)
    elif epi == 2:
        ref = ref + c0.double()
    assert _rel(c, ref) <= 2e-3, _rel(c, ref)


@pytest.mark.parametrize("n,H,group,dtype", [(300, 4, 1, "f16"), (64, 2, 2, "bf16"),
                                             (1000, 8, 4, "f16"), (129, 4, 2, "bf16"), (5, 2, 1, "f16")])
def test_prefill_attend_causal(n, H, group, dtype):
    import torch

    from paper_2508_10395_b200 import _native as N_

    dev = torch.device("cuda", 0)
    dt = torch.float16 if dtype == "f16" else torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(n + H)
    q = torch.randn(n, H * 128, generator=g, device=dev).to(dt)
    k = torch.randn(n, H // group * 128, generator=g, device=dev).to(dt)
    v = torch.randn(n, H // group * 128, generator=g, device=dev).to(dt)
    out = torch.empty(n, H, 128, device=dev)
    N_.call("xq_prefill_attend", N_.ptr(q), N_.ptr(k), N_.ptr(v), N_.F16 if dtype == "f16" else N_.BF16,
            n, H, group, H * 128, H // group * 128, 1 / math.sqrt(128), N_.ptr(out), H * 128,
            N_.stream_of(dev))
    torch.cuda.synchronize()
    qh = q.double().view(n, H, 128).permute(1, 0, 2)
    kh = k.double().view(n, -1, 128).permute(1, 0, 2).repeat_interleave(group, 0)
    vh = v.double().view(n, -1, 128).permute(1, 0, 2).repeat_interleave(group, 0)
    s = qh @ kh.transpose(1, 2) / math.sqrt(128)
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device=dev), 1), float("-inf"))
    ref = (torch.softmax(s, -1) @ vh).permute(1, 0, 2)
    assert _rel(out, ref) <= 1e-2, _rel(out, ref)


def test_rope_rows_and_dequant_f16():
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import _native as N_
    from paper_2508_10395_b200 import cache as C

    dev = torch.device("cuda", 0)
    n, w = 70, 256
    x = torch.randn(n, w, device=dev)
    out = torch.empty(n, w, dtype=torch.float16, device=dev)
    rope = C.rope_table(n + 5, dev)
    N_.call("xq_rope_rows", N_.ptr(x), N_.F32, w, n, w, N_.ptr(rope), rope.shape[0], 5, N_.ptr(out),
            N_.F16, w, N_.stream_of(dev))
    ref = O.apply_rope(x.double().cpu().numpy(), np.arange(5, 5 + n), 128)
    assert np.abs(out.double().cpu().numpy() - ref).max() / np.abs(ref).max() <= 1e-3

    # per-token arena rows + per-channel rows with a residual tail
    for axis, bits in ((C.TOKEN, 3), (C.CHANNEL, 4)):
        st = C.PackedStream(bits, axis, w, 128, 1, 512, dev)
        xs = torch.randn(300, w, device=dev)
        if axis == C.TOKEN:
            st.fill_rows(xs, 0, 0)
            nfl = 300
        else:
            st.channel_bulk(0, xs)
            nfl = int(st.n_flushed[0])
        ref = torch.empty(nfl, w, device=dev)
        N_.call("xq_dequant_rows", N_.ptr(st.codes), st.row_bytes, N_.ptr(st.params), axis, bits, 128,
                w, 0, nfl, N_.ptr(ref), N_.stream_of(dev))
        out = torch.empty(300, w, dtype=torch.float16, device=dev)
        N_.call("xq_dequant_rows_f16", N_.ptr(st.codes), st.row_bytes, N_.ptr(st.params), axis, bits,
                128, w, 0, nfl, N_.ptr(st.resid[0]) if nfl < 300 else None, 300, N_.ptr(out), w,
                N_.stream_of(dev))
        assert torch.equal(out[:nfl], ref.half())
        if nfl < 300:
            assert torch.equal(out[nfl:], xs[nfl:].half())
