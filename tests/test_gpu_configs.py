"""Parity at the benchmark configurations (BASELINE.json configs[2..4]).

The small-shape tests pin every kernel path against the reference's own golden
vectors. These tests run the engine at the bench shapes, where the fused
kernel takes many K passes per tile (32 / 40 MHA heads = 8 / 10 passes, the
serpentine fp16-row sweeps included) and RoPE runs at positions up to 131072:

* C3: xq-cl-mha 2-bit, Llama-2-7B width (d=4096, 32 heads), 8 layers = 3 base +
  5 delta layers at B=2, l=8193, and the full 32-layer stack (29 delta layers) at
  l=2049, on the engine's fp16 (and fp32) remat accumulator. Reference = the
  oracle's XqClMhaStack (pinned to the reference's golden run) with float64
  scale/zero-point as the reference keeps them, K/V remat + attention in float64.
  The delta codes of every layer are bit-exact with the reference's: the
  quantizer forms each delta against a float64 accumulator row
  (xq_quantize_rows_cl). With deltas formed from the fp16-stored parameters
  instead, code flips near rounding boundaries compounded to 3.2e-2 by layer 31.
* C4: xq-gqa 3-bit, Llama-3.1-8B (d=4096, g=4, r=1024), B=2, l=16385, against
  the oracle's XqGqaCache fed float64 latents (x @ U in float64, like
  cache.py:429-432).
* C5: Llama-2-13B width (d=5120, 40 heads), xq-cl-mha 3-bit, l=131073: every
  layer against an fp32 recompute from the same codes / accumulator rows.

Tolerance: the north-star bf16 figure, rel 2e-2 (max|err| / max|ref|).
"""

import math

import numpy as np
import pytest

from _util import rel_err, unpack_rows

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

TOL = 2e-2
F64 = None


def _torch():
    import torch

    return torch


def _rope64(m, pos0: int):
    """linalg.apply_rope (linalg.py:58-95) in float64 torch: rows at pos0, pos0+1, ..."""
    torch = _torch()
    n = m.shape[0]
    freqs = 10000.0 ** (-2.0 * torch.arange(64, dtype=torch.float64, device=m.device) / 128)
    ang = torch.arange(pos0, pos0 + n, dtype=torch.float64, device=m.device)[:, None] * freqs[None]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    mm = m.view(n, -1, 64, 2)
    e, o = mm[..., 0], mm[..., 1]
    return torch.stack([e * c - o * s, e * s + o * c], dim=-1).view(n, -1)


def _attend64(k_pre, v, q_pre, n_heads, group):
    """model._attention (model.py:150-182) for the newest token, float64 torch.

    k_pre: [n, kvw] before RoPE; q_pre: [n_heads*128] before RoPE (position n-1)."""
    torch = _torch()
    n = k_pre.shape[0]
    k = _rope64(k_pre, 0).view(n, -1, 128)
    q = _rope64(q_pre.view(1, -1), n - 1).view(n_heads, 128)
    kh = k[:, torch.arange(n_heads, device=k.device) // group]  # [n, H, 128]
    sc = torch.einsum("hd,nhd->hn", q, kh) / math.sqrt(128)
    p = torch.softmax(sc, dim=-1)
    vh = v.view(n, -1, 128)[:, torch.arange(n_heads, device=k.device) // group]
    return torch.einsum("hn,nhd->hd", p, vh)


def test_rope64_attend64_match_oracle():
    """The float64 torch restatement used below equals the oracle's apply_rope /
    attention (which test_oracle.py pins to the reference's golden vectors)."""
    import xq_oracle as O

    torch = _torch()
    g = torch.Generator().manual_seed(3)
    n, H, grp = 70, 4, 2
    k = torch.randn(n, H // grp * 128, generator=g, dtype=torch.float64)
    v = torch.randn(n, H // grp * 128, generator=g, dtype=torch.float64)
    q = torch.randn(H * 128, generator=g, dtype=torch.float64)
    got = _attend64(k.cuda(), v.cuda(), q.cuda(), H, grp).cpu().numpy().reshape(-1)
    kk = O.apply_rope(k.numpy(), np.arange(n), 128)
    ref = O.attention(O.apply_rope(q.numpy()[None], [n - 1], 128), kk, v.numpy(), H, grp)[0]
    assert rel_err(got, ref) < 1e-12
    big = _rope64(k[:3].cuda(), 131000).cpu().numpy()
    # CUDA vs libm cos/sin of angles near 1.3e5 rad: a few ulps
    assert rel_err(big, O.apply_rope(k[:3].numpy(), [131000, 131001, 131002], 128)) < 1e-10


def _prefill_decoder(dec, layers_x):
    """Cache rows 0..n-2 of every (slot, layer) input through the backends' bulk path."""
    torch = _torch()
    B = dec.n_slots
    n1 = None
    for s in range(B):
        for i, c in enumerate(dec.caches):
            x = layers_x(s, i)
            n1 = x.shape[0]
            c._prefill(s, x[:-1], dec.weights[i], dec.acc)
        if dec.acc is not None:
            dec.acc.release_prefill(s)
    dec.n_tokens[:] = n1 - 1
    dec.lens_dev.fill_(n1 - 1)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n_layers,B,n1,acc", [(8, 2, 8193, None), (32, 1, 2049, None),
                                                 (32, 1, 2049, "fp32")])
def test_c3_xq_cl_mha_2bit_delta_stack(n_layers, B, n1, acc):
    """C3 shape: delta layers on the engine's accumulator vs the reference's float64
    chain (codes of every delta layer depend on all earlier layers)."""
    import xq_oracle as O

    from paper_2508_10395_b200 import decode as D

    torch = _torch()
    dev = torch.device("cuda", 0)
    d, H = 4096, 32
    shape = D.ModelShape(f"llama2-7b-{n_layers}L", d, n_layers, H, 1)
    w, wq = D.synthetic_weights(shape, "xq-cl-mha", dev, seed=7)
    dec = D.Decoder(shape, "xq-cl-mha", 2, B, -(-n1 // 128) * 128 + 128, w, wq, device=dev,
                    acc_precision=acc)
    assert dec.policy.bits == [4, 4, 4] + [2] * (n_layers - 3)

    def layer_x(s, i):  # residual-stream drift, X_i = X_{i-1} + 0.03 N(0,1) (decode.fill_synthetic)
        gen = torch.Generator(device=dev).manual_seed(1000 * s + 1)
        x = torch.randn(n1, d, generator=gen, device=dev)
        for _ in range(i):
            x = x + 0.03 * torch.randn(n1, d, generator=gen, device=dev)
        return x.to(torch.bfloat16)

    _prefill_decoder(dec, layer_x)
    x_last = torch.stack([torch.stack([layer_x(s, i)[-1] for s in range(B)]) for i in range(n_layers)])
    out = torch.empty((n_layers, B, H, 128), dtype=torch.float32, device=dev)
    dec.step(x_last, attn_out=out)
    got = out.cpu().numpy()

    wk = [lw.w_k.double() for lw in w]
    wv = [lw.w_v.double() for lw in w]
    errs = {}
    for s in range(B):
        # q exactly as the decoder forms it (bf16 GEMV), rotated in float64 here
        qs = [torch.matmul(x_last[i, s:s + 1], wq[i]).double().view(-1) for i in range(n_layers)]
        for params_f16 in (False,):
            ref = []

            def on_layer(i, src):
                src_t = torch.from_numpy(src).to(dev)
                ref.append(_attend64(src_t @ wk[i], src_t @ wv[i], qs[i], H, 1).cpu().numpy())

            stack = O.XqClMhaStack(dec.policy.bits, 3, 128, params_f16=params_f16)
            stack.step((layer_x(s, i).double().cpu().numpy() for i in range(n_layers)),
                       on_layer=on_layer, keep=False)
            for i in range(n_layers):
                errs[(s, i, params_f16)] = rel_err(got[i, s].reshape(-1), ref[i].reshape(-1))
            if not params_f16:  # the reference's own chain: every layer's codes bit-exact
                for i, c in enumerate(dec.caches):
                    st = c.stream
                    rows = st.codes[s * st.L:s * st.L + n1].cpu().numpy()
                    codes = unpack_rows(rows, st.bits, d)
                    n_diff = int(np.count_nonzero(codes != stack.streams[i].codes))
                    assert n_diff == 0, (s, i, n_diff)
    worst = max(errs.values())
    print(f"C3 acc={dec.acc.precision} per-layer rel err (slot, layer, fp16 params):",
          {k: f"{v:.2e}" for k, v in errs.items()})
    assert worst <= TOL, errs


def test_xq_cl_gqa_3bit_llama31_width():
    """xq-cl-gqa at the Llama-3.1-8B width (d=4096, 32 heads on 8 KV heads, shared
    K|V latent r=2048): 5 layers (3 base + 2 delta), B=2, l=2049 (16 per-channel
    flushes in the prefill, the decode token in the residual buffer). Every
    layer's codes bit-exact with the oracle's float64 chain (cache.py:538-604),
    attention within 2e-2, the fp16 remat accumulator within 2e-2."""
    import xq_oracle as O

    from paper_2508_10395_b200 import decode as D

    torch = _torch()
    dev = torch.device("cuda", 0)
    d, H, g, n_layers, B, n1 = 4096, 32, 4, 5, 2, 2049
    shape = D.ModelShape("llama3.1-8b-5L", d, n_layers, H, g)
    w, wq = D.synthetic_weights(shape, "xq-cl-gqa", dev, seed=21)
    dec = D.Decoder(shape, "xq-cl-gqa", 3, B, 2176, w, wq, device=dev)

    def layer_x(s, i):
        gen = torch.Generator(device=dev).manual_seed(500 + s)
        x = torch.randn(n1, d, generator=gen, device=dev)
        for _ in range(i):
            x = x + 0.03 * torch.randn(n1, d, generator=gen, device=dev)
        return x.to(torch.bfloat16)

    _prefill_decoder(dec, layer_x)
    x_last = torch.stack([torch.stack([layer_x(s, i)[-1] for s in range(B)]) for i in range(n_layers)])
    out = torch.empty((n_layers, B, H, 128), dtype=torch.float32, device=dev)
    dec.step(x_last, attn_out=out)
    got = out.cpu().numpy()
    subs = [(lw.u_kv.double().cpu().numpy(), lw.fused_kv.double().cpu().numpy()) for lw in w]
    for s in range(B):
        stack = O.XqClGqaStack(dec.policy.bits, 3, 128, 128)
        xs = [layer_x(s, i).double().cpu().numpy() for i in range(n_layers)]
        stack.step([x[:-1] for x in xs], subs)
        o = stack.step([x[-1] for x in xs], subs)
        for i in range(n_layers):
            q = torch.matmul(x_last[i, s:s + 1], wq[i]).double().cpu().numpy()  # as the decoder
            ref = O.attention(O.apply_rope(q, [n1 - 1], 128), o[i][1], o[i][2], H, g)[0]
            err = rel_err(got[i, s].reshape(-1), ref)
            print(f"xq-cl-gqa slot {s} layer {i}: rel err {err:.2e}")
            assert err <= TOL, (s, i, err)
            st = dec.caches[i].stream
            nfl = int(st.n_flushed[s])
            rows = st.codes[s * st.L:s * st.L + nfl].cpu().numpy()
            assert np.array_equal(unpack_rows(rows, st.bits, st.width), stack.streams[i].codes[:nfl]), (s, i)
        acc16 = dec.acc.x16[s, :n1].float().cpu().numpy()
        assert rel_err(acc16, o[-1][3]) <= TOL


def test_c4_xq_gqa_3bit_latents():
    """C4 shape: per-channel K latent (128 full groups + 1 residual row after the
    decode push), per-token V latent, 8 KV heads x 4 query heads."""
    import xq_oracle as O

    from paper_2508_10395_b200 import cache as M
    from paper_2508_10395_b200 import decode as D

    torch = _torch()
    dev = torch.device("cuda", 0)
    d, H, g, B, n1 = 4096, 32, 4, 2, 16385
    shape = D.ModelShape("llama3.1-8b-1L", d, 1, H, g)
    w, _ = D.synthetic_weights(shape, "xq-gqa", dev, seed=9)
    lw = w[0]
    st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, n_slots=B, max_len=16512,
                      hidden_dim=d, n_heads=H, kv_group=g, device=dev)
    gen = torch.Generator(device=dev).manual_seed(2)
    xs = [torch.randn(n1, d, generator=gen, device=dev).to(torch.bfloat16) for _ in range(B)]
    for s in range(B):
        st.prefill(xs[s][:-1], lw, slot=s)
    st.decode_append(torch.stack([x[-1] for x in xs]), lw)
    assert int(st.k_stream.n_flushed[0]) == 16384
    q = torch.randn(B, H, 128, generator=gen, device=dev)
    got = st.decode_attend(q, lw).cpu().numpy()

    uk, uv = lw.u_k.double(), lw.u_v.double()
    fk, fv = lw.fused_k.double(), lw.fused_v.double()
    for s in range(B):
        x64 = xs[s].double()
        lat_k, lat_v = (x64 @ uk).cpu().numpy(), (x64 @ uv).cpu().numpy()
        for params_f16 in (False,):
            c = O.XqGqaCache(3, 128, 128, params_f16=params_f16)
            c.prefill(lat_k[:-1], lat_v[:-1])
            c.push(lat_k[-1], lat_v[-1])
            k_pre = torch.from_numpy(c.k_stream.reconstruct()).to(dev) @ fk
            v = torch.from_numpy(c.v_stream.reconstruct()).to(dev) @ fv
            ref = _attend64(k_pre, v, q[s].double().view(-1), H, g).cpu().numpy()
            err = rel_err(got[s].reshape(-1), ref.reshape(-1))
            print(f"C4 slot {s} fp16 params {params_f16}: rel err {err:.2e}")
            assert err <= TOL, (s, params_f16, err)


def test_c5_13b_width_at_128k_positions():
    """C5 shape at its longest context: Llama-2-13B width (kdim 5120, 40 heads, 10 K
    passes), xq-cl-mha 3-bit, l=131073. Base layers: fp32 recompute from the same
    codes (xq_dequant_rows); the delta layer: from the same fp16 accumulator rows."""
    from paper_2508_10395_b200 import _native as N
    from paper_2508_10395_b200 import decode as D

    torch = _torch()
    dev = torch.device("cuda", 0)
    d, H, n_layers, n1 = 5120, 40, 4, 131073
    shape = D.ModelShape("llama2-13b-4L", d, n_layers, H, 1)
    w, wq = D.synthetic_weights(shape, "xq-cl-mha", dev, seed=13)
    dec = D.Decoder(shape, "xq-cl-mha", 3, 1, 131200, w, wq, device=dev)
    assert dec.policy.bits == [4, 4, 4, 3]

    def layer_x(s, i):
        gen = torch.Generator(device=dev).manual_seed(77)
        x = torch.randn(n1, d, generator=gen, device=dev)
        for _ in range(i):
            x = x + 0.03 * torch.randn(n1, d, generator=gen, device=dev)
        return x.to(torch.bfloat16)

    _prefill_decoder(dec, layer_x)
    x_last = torch.stack([layer_x(0, i)[-1:] for i in range(n_layers)])
    out = torch.empty((n_layers, 1, H, 128), dtype=torch.float32, device=dev)
    dec.step(x_last, attn_out=out)
    torch.cuda.synchronize()
    torch.backends.cuda.matmul.allow_tf32 = False
    for i, c in enumerate(dec.caches):
        if c.is_base:
            s = c.stream
            a = torch.empty((n1, d), dtype=torch.float32, device=dev)
            N.call("xq_dequant_rows", N.ptr(s.codes), s.row_bytes, N.ptr(s.params), 0, s.bits, 128,
                   d, 0, n1, N.ptr(a), N.stream_of(dev))
        else:
            a = dec.acc.x16[0, :n1].float()
        k = a @ w[i].w_k.float()
        v = a @ w[i].w_v.float()
        q = torch.matmul(x_last[i], wq[i]).double().view(-1)
        ref = _attend64(k.double(), v.double(), q, H, 1)
        del k, v, a
        err = rel_err(out[i, 0].cpu().numpy(), ref.cpu().numpy())
        print(f"C5 layer {i}: rel err {err:.2e}")
        assert err <= TOL, (i, err)
