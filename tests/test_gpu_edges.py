"""Edge cases and full-size properties of the fused path on the GPU.

* ragged batches (different lengths per slot), l = 1, lengths that are not
  multiples of the 256-token pair tile;
* every code width (2/3/4/8) and the 16-bit pass-through of xq-mha;
* NaN/Inf input -> DataError (quant.py:114-115), unsupported group sizes ->
  ConfigError, empty cache -> UsageError;
* xq-gqa before its first per-channel flush (all rows in the residual buffer);
* full C2 shape (d=4096, 32 heads, l=32769, 3-bit): the fused output against
  an independent float32 computation on the GPU (torch) from the same codes.
"""

import math

import numpy as np
import pytest

from _util import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("kernel_path")]
TOL = 2e-2


def _mha(bits, n_slots, max_len, d=256, H=2, device="cuda"):
    from paper_2508_10395_b200 import cache as M

    pol = M.LayerPolicy.uniform(bits, 1)
    return M.make_cache("xq-mha", 0, pol, 128, 128, n_slots=n_slots, max_len=max_len,
                        hidden_dim=d, n_heads=H, device=device)


def _weights(d, kvw, seed=0):
    import torch

    from paper_2508_10395_b200 import cache as M

    g = torch.Generator().manual_seed(seed)
    wk = (torch.randn(d, kvw, generator=g) / math.sqrt(d)).to(torch.bfloat16).cuda()
    wv = (torch.randn(d, kvw, generator=g) / math.sqrt(d)).to(torch.bfloat16).cuda()
    return M.LayerWeights(w_k=wk, w_v=wv)


def _oracle_mha(x, wk, wv, q, bits, H):
    import xq_oracle as O

    st = O.XqMhaCache(bits, 128, 128)
    st.append(x)
    k, v = st.remat(wk, wv) if bits != 16 else (None, None)
    if bits == 16:
        xf = x.astype(np.float16).astype(np.float64)  # the GPU stores fp16 rows
        k = O.apply_rope(xf @ wk, np.arange(len(x)), 128)
        v = xf @ wv
    n = x.shape[0]
    return O.attention(O.apply_rope(q[None], [n - 1], 128), k, v, H, 1)[0]


@pytest.mark.parametrize("bits", [2, 3, 4, 8, 16])
def test_ragged_batch_every_width(bits):
    import torch

    d, H = 256, 2
    lens = [1, 130, 257, 600]  # l=1, within one tile, just past a pair tile, several
    st = _mha(bits, len(lens), 1024, d, H)
    w = _weights(d, d, seed=bits)
    g = torch.Generator().manual_seed(7)
    xs = [torch.randn(n, d, generator=g).to(torch.bfloat16) for n in lens]
    for s, x in enumerate(xs):
        if len(x) > 1:
            st.prefill(x[:-1].cuda(), w, slot=s)
    st.decode_append(torch.stack([x[-1] for x in xs]).cuda(), w)
    q = torch.randn(len(lens), H, 128, generator=g)
    out = st.decode_attend(q.cuda(), w).cpu().numpy()
    wk, wv = w.w_k.double().cpu().numpy(), w.w_v.double().cpu().numpy()
    for s, x in enumerate(xs):
        ref = _oracle_mha(x.double().numpy(), wk, wv, q[s].double().numpy().reshape(-1), bits, H)
        assert rel_err(out[s].reshape(-1), ref) <= TOL, (bits, lens[s])


def test_nonfinite_input_raises_data_error():
    import torch

    from paper_2508_10395_b200.errors import DataError

    st = _mha(3, 1, 256)
    w = _weights(256, 256)
    x = torch.randn(10, 256).to(torch.bfloat16)
    x[3, 17] = float("nan")
    st.prefill(x.cuda(), w)
    with pytest.raises(DataError):
        st.stream.check_finite()


def test_unsupported_group_sizes_rejected():
    """The fused kernel takes 32/64/128-channel groups for per-token streams
    (tests/test_gpu_groups.py); other sizes, and per-channel streams with other token
    groups, raise the reference's ConfigError instead of computing garbage."""
    import torch

    from paper_2508_10395_b200 import cache as M
    from paper_2508_10395_b200.errors import ConfigError

    st = M.make_cache("xq-mha", 0, M.LayerPolicy.uniform(4, 1), 128, 16, n_slots=1,
                      max_len=256, hidden_dim=256, n_heads=2)
    w = _weights(256, 256)
    st.prefill(torch.randn(5, 256).to(torch.bfloat16).cuda(), w)
    with pytest.raises(ConfigError):
        st.decode_attend(torch.randn(1, 2, 128).cuda(), w)
    with pytest.raises(ConfigError):
        M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(4, 1), 128, 64, n_slots=1, max_len=256,
                     hidden_dim=512, n_heads=4, kv_group=2)


def test_empty_cache_usage_errors():
    import torch

    from paper_2508_10395_b200.errors import UsageError

    st = _mha(3, 1, 256)
    w = _weights(256, 256)
    with pytest.raises(UsageError):
        st.decode_attend(torch.randn(1, 2, 128).cuda(), w)
    with pytest.raises(UsageError):
        st.rematerialize(w, np.arange(0))
    st.prefill(torch.randn(4, 256).to(torch.bfloat16).cuda(), w)
    with pytest.raises(UsageError):
        st.prefill(torch.randn(4, 256).to(torch.bfloat16).cuda(), w)  # cache.py:258-259


def test_gqa_residual_only_before_first_flush():
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import cache as M
    from paper_2508_10395_b200 import decode as D

    d, H, g = 512, 4, 2
    shape = D.ModelShape("t", d, 1, H, g)
    w, _ = D.synthetic_weights(shape, "xq-gqa", "cuda", seed=3)
    w = w[0]
    st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, 128, n_slots=1,
                      max_len=256, hidden_dim=d, n_heads=H, kv_group=g)
    gen = torch.Generator().manual_seed(5)
    x = torch.randn(60, d, generator=gen).to(torch.bfloat16)
    st.prefill(x[:-1].cuda(), w)
    st.decode_append(x[-1:].cuda(), w)
    assert st.k_stream.n_flushed[0] == 0
    q = torch.randn(1, H, 128, generator=gen)
    out = st.decode_attend(q.cuda(), w).cpu().numpy().reshape(-1)
    xf = x.double().numpy()
    uk, uv = w.u_k.double().cpu().numpy(), w.u_v.double().cpu().numpy()
    fk, fv = w.fused_k.double().cpu().numpy(), w.fused_v.double().cpu().numpy()
    ref_st = O.XqGqaCache(3, 128, 128)
    ref_st.prefill(xf @ uk, xf @ uv)
    k, v = ref_st.remat(fk, fv)
    ref = O.attention(O.apply_rope(q.double().numpy().reshape(1, -1), [59], 128), k, v, H, g)[0]
    assert rel_err(out, ref) <= TOL


def test_full_c2_shape_against_independent_fp32():
    """d=4096, 32 heads, l=32769, 3-bit: fused tcgen05 output vs torch fp32 from the same codes."""
    import torch

    from paper_2508_10395_b200 import _native as N
    from paper_2508_10395_b200 import cache as M

    d, H, n = 4096, 32, 32769
    st = _mha(3, 1, 32896, d, H)
    w = _weights(d, d, seed=11)
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, d, generator=gen, device="cuda").to(torch.bfloat16)
    st.prefill(x[:-1], w)
    st.decode_append(x[-1:], w)
    q = torch.randn(1, H, 128, generator=gen, device="cuda")
    out = st.decode_attend(q, w)[0]
    # independent path: dequantized rows (xq_dequant_rows) -> fp32 GEMM -> RoPE -> softmax
    xh = torch.empty((n, d), dtype=torch.float32, device="cuda")
    s = st.stream
    N.call("xq_dequant_rows", N.ptr(s.codes), s.row_bytes, N.ptr(s.params), 0, 3, 128, d, 0, n,
           N.ptr(xh), N.stream_of())
    torch.backends.cuda.matmul.allow_tf32 = False
    k = xh @ w.w_k.float()
    v = xh @ w.w_v.float()
    pos = torch.arange(n, device="cuda", dtype=torch.float64)
    freqs = 10000.0 ** (-2.0 * torch.arange(64, device="cuda", dtype=torch.float64) / 128)
    ang = pos[:, None] * freqs[None, :]
    c, sn = torch.cos(ang).float(), torch.sin(ang).float()

    def rope(m, cc, ss):
        mm = m.view(m.shape[0], -1, 64, 2)
        e, o = mm[..., 0], mm[..., 1]
        return torch.stack([e * cc[:, None] - o * ss[:, None], e * ss[:, None] + o * cc[:, None]],
                           -1).view(m.shape[0], -1)

    kr = rope(k, c, sn).view(n, H, 128)
    qr = rope(q.view(1, -1), c[-1:], sn[-1:]).view(H, 128)
    sc = torch.einsum("hd,nhd->hn", qr, kr) / math.sqrt(128)
    p = torch.softmax(sc, dim=-1)
    ref = torch.einsum("hn,nhd->hd", p, v.view(n, H, 128))
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, err


@pytest.mark.parametrize("d,H", [(5120, 40, ), (768, 6), (512, 4)])
def test_mha_head_layouts(d, H):
    """Head counts that pad the absorbed kernel's V-side N (40 -> 48, 4 -> 16),
    a partial 4-head K pass (6 heads) and the 13B width (kdim 5120)."""
    import torch

    lens = [300, 517]
    st = _mha(3, len(lens), 640, d, H)
    w = _weights(d, d, seed=H)
    g = torch.Generator().manual_seed(11)
    xs = [torch.randn(n, d, generator=g).to(torch.bfloat16) for n in lens]
    for s, x in enumerate(xs):
        st.prefill(x[:-1].cuda(), w, slot=s)
    st.decode_append(torch.stack([x[-1] for x in xs]).cuda(), w)
    q = torch.randn(len(lens), H, 128, generator=g)
    out = st.decode_attend(q.cuda(), w).cpu().numpy()
    wk, wv = w.w_k.double().cpu().numpy(), w.w_v.double().cpu().numpy()
    for s, x in enumerate(xs):
        ref = _oracle_mha(x.double().numpy(), wk, wv, q[s].double().numpy().reshape(-1), 3, H)
        assert rel_err(out[s].reshape(-1), ref) <= TOL, (d, H, lens[s])


@pytest.mark.parametrize("d,H,g", [(2048, 16, 4), (2048, 16, 2), (1024, 8, 8)])
def test_gqa_group_layouts(d, H, g):
    """xq-gqa with GROUP 4 / 2 / 8->1 KV heads: absorbed and unabsorbed kernels agree
    (the unabsorbed one is pinned to the reference in test_gpu_cache)."""
    import os

    import torch

    from paper_2508_10395_b200 import cache as M

    r = d // g
    if g not in (1, 2, 4):
        pytest.skip("the fused kernels support query groups 1, 2, 4")
    pol = M.LayerPolicy.uniform(4, 1)
    st = M.make_cache("xq-gqa", 0, pol, 128, n_slots=2, max_len=768, hidden_dim=d, n_heads=H,
                      kv_group=g, device="cuda")
    gen = torch.Generator().manual_seed(5)
    uk, _ = torch.linalg.qr(torch.randn(d, r, generator=gen, dtype=torch.float64))
    uv, _ = torch.linalg.qr(torch.randn(d, r, generator=gen, dtype=torch.float64))
    w = M.LayerWeights(u_k=uk.float().cuda(), u_v=uv.float().cuda(),
                       fused_k=(torch.randn(r, r, generator=gen) / r ** 0.5).cuda(),
                       fused_v=(torch.randn(r, r, generator=gen) / r ** 0.5).cuda())
    for s, n in enumerate([300, 700]):
        st.prefill(torch.randn(n, d, generator=gen).to(torch.bfloat16).cuda(), w, slot=s)
    st.decode_append(torch.randn(2, d, generator=gen).to(torch.bfloat16).cuda(), w)
    q = torch.randn(2, H, 128, generator=gen).cuda()
    st.absorb = True
    a = st.decode_attend(q, w).cpu().numpy()
    st.absorb = False
    b = st.decode_attend(q, w).cpu().numpy()
    assert rel_err(a, b) <= 1e-2, rel_err(a, b)
