"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container (where the reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``xcache`` from ``oracle/_ref`` (built by
``oracle/build_ref.sh``) or, failing that, from ``/root/reference/pkg/src``,
and writes small compressed ``.npz`` fixtures next to this script. The
fixtures pin both the oracle restatement (``tests/test_oracle.py``) and the
CUDA path (``tests/test_gpu_*.py``) to the reference's own outputs; nothing at
test time reads ``/root/reference``.

Inputs are bf16-representable (stored as raw bf16 bit patterns) so the GPU
path and the float64 reference see identical values.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def _import_reference():
    for p in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "xcache")):
            sys.path.insert(0, p)
            import xcache  # noqa: F401

            return p
    raise SystemExit("reference package not found; run oracle/build_ref.sh")


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    f = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounded = f + np.uint32(0x7FFF) + ((f >> np.uint32(16)) & np.uint32(1))
    return (rounded >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def bf16(a: np.ndarray):
    bits = to_bf16_bits(a)
    return bits, from_bf16_bits(bits)


def main():
    src = _import_reference()
    from xcache import _kernels
    from xcache.cache import Accumulator, LayerPolicy, LayerWeights, make_cache
    from xcache.linalg import SvdFactors, apply_rope
    from xcache.model import _attention
    from xcache.quant import Axis, QuantConfig, dump_qtensor, quantize

    print("reference from", src, "lane", _kernels.backend())
    rng = np.random.default_rng(20251017)

    # ---- 1. lane: quantize_groups / dequantize_groups ---------------------
    quant = {}
    for bits in (2, 3, 4, 8):
        for cols in (17, 64, 130, 256):
            for gs in (32, 128):
                # float32-representable fp64 inputs (stored as float32)
                x = (rng.normal(size=(23, cols)) * rng.uniform(0.01, 100)).astype(np.float32).astype(np.float64)
                x[3, :] = 1.25  # a degenerate row (every group constant)
                key = f"b{bits}_c{cols}_g{gs}"
                c, s, z = _kernels.quantize_groups(np.ascontiguousarray(x), gs, bits)
                quant[key + "_x"] = x.astype(np.float32)
                quant[key + "_codes"] = c
                quant[key + "_scales"] = s
                quant[key + "_zps"] = z
                quant[key + "_deq"] = _kernels.dequantize_groups(c, s, z, gs).astype(np.float32)
    # the config-1 row shape: bf16-representable d=4096 rows, G=128
    for bits in (2, 3, 4):
        xb, x = bf16(rng.normal(size=(16, 4096)))
        c, s, z = _kernels.quantize_groups(np.ascontiguousarray(x), 128, bits)
        quant[f"d4096_b{bits}_xbf16"] = xb
        quant[f"d4096_b{bits}_codes"] = c
        quant[f"d4096_b{bits}_scales"] = s
        quant[f"d4096_b{bits}_zps"] = z
        quant[f"d4096_b{bits}_packed"] = np.stack(
            [_kernels.pack_codes(c[r], bits).view(np.uint8) for r in range(c.shape[0])]
        )
    # per-channel quantization of a 2-group token block (quant.py:124-134)
    xb, x = bf16(rng.normal(size=(256, 96)))
    q = quantize(x, QuantConfig(3, Axis.PER_CHANNEL, group_size=128))
    quant["perchan_b3_xbf16"] = xb
    quant["perchan_b3_codes"] = q.codes
    quant["perchan_b3_scales"] = q.scales
    quant["perchan_b3_zps"] = q.zero_points
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **quant)

    # ---- 2. lane: pack / unpack + XQT1 known-answer -----------------------
    pack = {}
    for bits in (2, 3, 4, 8):
        for n in list(range(0, 65)) + [127, 128, 129, 1000, 4096]:
            codes = rng.integers(0, 2**bits, n).astype(np.uint8)
            pack[f"b{bits}_n{n}_codes"] = codes
            pack[f"b{bits}_n{n}_words"] = _kernels.pack_codes(codes, bits)
    kat = quantize(np.array([[0.0, 1.0, 2.0, 3.0]]), QuantConfig(2, Axis.PER_TOKEN, group_size=4))
    pack["xqt1_kat"] = np.frombuffer(dump_qtensor(kat), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "pack.npz"), **pack)

    # ---- 3. RoPE (linalg.py:58-95) -----------------------------------------
    rope = {}
    m = rng.normal(size=(8, 256))
    pos = np.array([0, 1, 7, 4095, 32768, 131071, 131072, 1000003])
    rope["m"] = m
    rope["pos"] = pos
    rope["out_hd128"] = apply_rope(m, pos, 128)
    rope["out_hd8"] = apply_rope(m, pos, 8)
    np.savez_compressed(os.path.join(HERE, "rope.npz"), **rope)

    # ---- 4. backends + decode attention ------------------------------------
    def dummy_lw(d, kvw, w_k, w_v, **kw):
        z = np.zeros((d, d))
        return LayerWeights(
            gamma_attn=np.ones(d), gamma_mlp=np.ones(d), w_q=z, w_k=w_k, w_v=w_v,
            w_o=z, w_up=z, w_down=z, **kw,
        )

    be = {}
    # xq-mha: d=256 (2 heads x hd 128), G=128; prefill 290 tokens + 10 decodes
    d, hd, H = 256, 128, 2
    n_pre, n_dec = 290, 10
    for bits in (2, 3, 4, 16):
        xb, x = bf16(rng.normal(size=(n_pre + n_dec, d)))
        wkb, w_k = bf16(rng.normal(size=(d, d)) / np.sqrt(d))
        wvb, w_v = bf16(rng.normal(size=(d, d)) / np.sqrt(d))
        qb, q = bf16(rng.normal(size=(n_dec, d)))
        lw = dummy_lw(d, d, w_k, w_v)
        pol = LayerPolicy.uniform(bits, 1)
        st = make_cache("xq-mha", 0, pol, hd, group_size=128)
        st.prefill(x[:n_pre], lw)
        outs = []
        for t in range(n_dec):
            st.decode_append(x[n_pre + t], lw)
            k, v = st.rematerialize(lw, np.arange(n_pre + t + 1))
            # q = RoPE(x W_q) at the new token's position (model.py:234)
            qr = apply_rope(q[t:t + 1], np.array([n_pre + t]), hd)
            outs.append(_attention(qr, k, v, H, 1)[0])
        key = f"mha_b{bits}"
        be[key + "_x"], be[key + "_wk"], be[key + "_wv"], be[key + "_q"] = xb, wkb, wvb, qb
        if bits in (3, 16):  # final-step K/V kept for two widths (fixture size)
            be[key + "_k"], be[key + "_v"] = k.astype(np.float32), v.astype(np.float32)
        be[key + "_attn"] = np.stack(outs)
        if bits != 16:
            be[key + "_codes"] = st.x_stream.q.codes
            be[key + "_scales"] = st.x_stream.q.scales
            be[key + "_zps"] = st.x_stream.q.zero_points
            # XQT1 dump of the whole X cache (quant.py:232-254)
            be[key + "_xqt1"] = np.frombuffer(dump_qtensor(st.x_stream.q), dtype=np.uint8)

    # fp16 baseline semantics (cache.py:302-323) on the same x
    lw = dummy_lw(d, d, from_bf16_bits(be["mha_b4_wk"]), from_bf16_bits(be["mha_b4_wv"]))
    st = make_cache("fp16", 0, LayerPolicy.uniform(16, 1), hd)
    xx = from_bf16_bits(be["mha_b4_x"])
    st.prefill(xx, lw)
    k, v = st.rematerialize(lw, np.arange(xx.shape[0]))
    be["fp16_k"], be["fp16_v"] = k.astype(np.float32), v.astype(np.float32)
    qr = apply_rope(from_bf16_bits(be["mha_b4_q"])[-1:], np.array([xx.shape[0] - 1]), hd)
    be["fp16_attn"] = _attention(qr, k, v, H, 1)[0]

    # xq-gqa: d=1024, H=8, KV heads 2 (kv_group 4), r = 256; injected SVD factors
    d, H, g = 1024, 8, 4
    r = d // g
    n_pre, n_dec = 250, 12  # crosses the 256-token per-channel flush
    xb, x = bf16(rng.normal(size=(n_pre + n_dec, d)))
    ukb, u_k = bf16(np.linalg.qr(rng.normal(size=(d, r)))[0])
    uvb, u_v = bf16(np.linalg.qr(rng.normal(size=(d, r)))[0])
    fkb, f_k = bf16(rng.normal(size=(r, r)) / np.sqrt(r))
    fvb, f_v = bf16(rng.normal(size=(r, r)) / np.sqrt(r))
    qb, q = bf16(rng.normal(size=(n_dec, d)))
    svd_k = SvdFactors(u=u_k, sigma=np.ones(r), b_t=f_k, fused=f_k)
    svd_v = SvdFactors(u=u_v, sigma=np.ones(r), b_t=f_v, fused=f_v)
    lw = dummy_lw(d, r, u_k @ f_k, u_v @ f_v, svd_k=svd_k, svd_v=svd_v)
    st = make_cache("xq-gqa", 0, LayerPolicy.uniform(3, 1), 128, group_size=128)
    st.prefill(x[:n_pre], lw)
    outs, bufs = [], []
    for t in range(n_dec):
        st.decode_append(x[n_pre + t], lw)
        k, v = st.rematerialize(lw, np.arange(n_pre + t + 1))
        qr = apply_rope(q[t:t + 1], np.array([n_pre + t]), 128)
        outs.append(_attention(qr, k, v, H, g)[0])
        bufs.append(len(st.k_stream.buf))
    be["gqa_kxqt1"] = np.frombuffer(dump_qtensor(st.k_stream.q), dtype=np.uint8)
    be.update({
        "gqa_x": xb, "gqa_uk": ukb, "gqa_uv": uvb, "gqa_fk": fkb, "gqa_fv": fvb,
        "gqa_q": qb, "gqa_k": k.astype(np.float32), "gqa_v": v.astype(np.float32), "gqa_attn": np.stack(outs),
        "gqa_buf_len": np.array(bufs),
        "gqa_kcodes": st.k_stream.q.codes, "gqa_kscales": st.k_stream.q.scales,
        "gqa_kzps": st.k_stream.q.zero_points,
        "gqa_vcodes": st.v_stream.q.codes, "gqa_vscales": st.v_stream.q.scales,
        "gqa_vzps": st.v_stream.q.zero_points,
    })

    # xq-cl-mha: 6 layers (base 3, layers 0-2 at 4-bit), d=256, 2-bit deltas
    d, H, n_layers = 256, 2, 6
    n_pre, n_dec = 140, 3
    pol = LayerPolicy.for_bits(2, n_layers)
    base = rng.normal(size=(n_pre + n_dec, d))
    xs, xbits = [], []
    for i in range(n_layers):
        base = base + 0.03 * rng.normal(size=base.shape)
        b_, f_ = bf16(base)
        xbits.append(b_)
        xs.append(f_)
    wks, wvs, lws = [], [], []
    for i in range(n_layers):
        wkb, w_k = bf16(rng.normal(size=(d, d)) / np.sqrt(d))
        wvb, w_v = bf16(rng.normal(size=(d, d)) / np.sqrt(d))
        wks.append(wkb)
        wvs.append(wvb)
        lws.append(dummy_lw(d, d, w_k, w_v))
    qb, q = bf16(rng.normal(size=(n_layers, d)))
    states = [make_cache("xq-cl-mha", i, pol, 128, group_size=128) for i in range(n_layers)]
    acc = Accumulator()
    for i in range(n_layers):
        states[i].prefill(xs[i][:n_pre], lws[i], acc)
    for t in range(n_dec):
        acc = Accumulator()
        accs, ks, vs, attn = [], [], [], []
        for i in range(n_layers):
            states[i].decode_append(xs[i][n_pre + t], lws[i], acc)
            k, v = states[i].rematerialize(lws[i], np.arange(n_pre + t + 1), acc)
            accs.append(acc.x_hat.copy() if acc.x_hat is not None else np.zeros((0, d)))
            ks.append(k)
            vs.append(v)
            qr = apply_rope(q[i:i + 1], np.array([n_pre + t]), 128)
            attn.append(_attention(qr, k, v, H, 1)[0])
    be.update({
        "cl_x": np.stack(xbits), "cl_wk": np.stack(wks), "cl_wv": np.stack(wvs),
        "cl_q": qb, "cl_bits": np.array(pol.bits), "cl_base": np.array(pol.base_layers),
        "cl_k": np.stack([ks[2], ks[-1]]).astype(np.float32),  # base seed + last delta layer
        "cl_v": np.stack([vs[2], vs[-1]]).astype(np.float32), "cl_attn": np.stack(attn),
        "cl_acc_last": accs[-1].astype(np.float32),
    })
    for i in range(n_layers):
        be[f"cl_codes{i}"] = states[i].stream.q.codes
        be[f"cl_scales{i}"] = states[i].stream.q.scales
        be[f"cl_zps{i}"] = states[i].stream.q.zero_points

    # xq-cl-gqa: 5 layers (base 3, layers 0-2 at 4-bit, 3-bit deltas), d=1024, H=8,
    # 2 KV heads (kv_group 4, kvw 256), shared K|V subspace r = 2*kvw = 512. U is an
    # fp32-representable orthonormal basis, fused = U^T [W_k | W_v] with bf16 W
    d, H, g, n_layers = 1024, 8, 4, 5
    kvw = d // g
    n_pre, n_dec = 250, 8  # decode crosses the 256-token per-channel flush
    pol = LayerPolicy.for_bits(3, n_layers)
    base = rng.normal(size=(n_pre + n_dec, d))
    cx, cxb = [], []
    for i in range(n_layers):
        base = base + 0.03 * rng.normal(size=base.shape)
        b_, f_ = bf16(base)
        cxb.append(b_)
        cx.append(f_)
    us, fuseds, lws = [], [], []
    for i in range(n_layers):
        u = np.linalg.qr(rng.normal(size=(d, 2 * kvw)))[0].astype(np.float32).astype(np.float64)
        fb, fused = bf16(rng.normal(size=(2 * kvw, 2 * kvw)) / np.sqrt(2 * kvw))
        us.append(u.astype(np.float32))
        fuseds.append(fb)
        sub = SvdFactors(u=u, sigma=np.ones(2 * kvw), b_t=fused, fused=fused)
        w = u @ fused
        lws.append(dummy_lw(d, kvw, w[:, :kvw], w[:, kvw:], svd_kv=sub))
    qb, q = bf16(rng.normal(size=(n_layers, d)))
    states = [make_cache("xq-cl-gqa", i, pol, 128, group_size=128) for i in range(n_layers)]
    acc = Accumulator()
    for i in range(n_layers):
        states[i].prefill(cx[i][:n_pre], lws[i], acc)
    for t in range(n_dec):
        acc = Accumulator()
        ks, vs, attn = [], [], []
        for i in range(n_layers):
            states[i].decode_append(cx[i][n_pre + t], lws[i], acc)
            k, v = states[i].rematerialize(lws[i], np.arange(n_pre + t + 1), acc)
            ks.append(k)
            vs.append(v)
            qr = apply_rope(q[i:i + 1], np.array([n_pre + t]), 128)
            attn.append(_attention(qr, k, v, H, g)[0])
    be.update({
        "clg_x": np.stack(cxb), "clg_u": np.stack(us), "clg_fused": np.stack(fuseds),
        "clg_q": qb, "clg_bits": np.array(pol.bits), "clg_base": np.array(pol.base_layers),
        "clg_k": np.stack([ks[2], ks[-1]]).astype(np.float32),
        "clg_v": np.stack([vs[2], vs[-1]]).astype(np.float32), "clg_attn": np.stack(attn),
        "clg_acc_last": acc.x_hat.astype(np.float32),
    })
    for i in range(n_layers):
        be[f"clg_codes{i}"] = states[i].stream.q.codes
        be[f"clg_scales{i}"] = states[i].stream.q.scales
        be[f"clg_zps{i}"] = states[i].stream.q.zero_points
        be[f"clg_buf{i}"] = np.asarray(states[i].stream.buf.tokens, np.float64)

    # kvq: d=512, 4 heads on 2 KV heads (kvw 256), 3-bit; prefill 250 + 12 decodes
    # (crosses the 256-token K flush; V buffers 12 rows after the whole-V prefill)
    d, H, g = 512, 4, 2
    kvw = d // g
    n_pre, n_dec = 250, 12
    xb, x = bf16(rng.normal(size=(n_pre + n_dec, d)))
    wkb, w_k = bf16(rng.normal(size=(d, kvw)) / np.sqrt(d))
    wvb, w_v = bf16(rng.normal(size=(d, kvw)) / np.sqrt(d))
    qb, q = bf16(rng.normal(size=(n_dec, d)))
    lw = dummy_lw(d, kvw, w_k, w_v)
    st = make_cache("kvq", 0, LayerPolicy.uniform(3, 1), 128, group_size=128)
    st.prefill(x[:n_pre], lw)
    outs = []
    for t in range(n_dec):
        st.decode_append(x[n_pre + t], lw)
        k, v = st.rematerialize(lw, np.arange(n_pre + t + 1))
        qr = apply_rope(q[t:t + 1], np.array([n_pre + t]), 128)
        outs.append(_attention(qr, k, v, H, g)[0])
    be.update({
        "kvq_x": xb, "kvq_wk": wkb, "kvq_wv": wvb, "kvq_q": qb, "kvq_attn": np.stack(outs),
        "kvq_k": k.astype(np.float32), "kvq_v": v.astype(np.float32),
        "kvq_kcodes": st.k_stream.q.codes, "kvq_kscales": st.k_stream.q.scales,
        "kvq_vcodes": st.v_stream.q.codes, "kvq_vscales": st.v_stream.q.scales,
        "kvq_vbuf": np.asarray(st.v_stream.buf.tokens, np.float64),
    })

    # xq-gqa with the fp16 outlier channel (cache.py:403-409, 653-658): the same
    # inputs as the xq-gqa case above, channel 0 of the K latent in full precision
    from xcache.cache import fp16_outlier_channel_variant
    d, H, g = 1024, 8, 4
    r = d // g
    x = from_bf16_bits(be["gqa_x"])
    u_k, u_v = from_bf16_bits(be["gqa_uk"]), from_bf16_bits(be["gqa_uv"])
    f_k, f_v = from_bf16_bits(be["gqa_fk"]), from_bf16_bits(be["gqa_fv"])
    q = from_bf16_bits(be["gqa_q"])
    svd_k = SvdFactors(u=u_k, sigma=np.ones(r), b_t=f_k, fused=f_k)
    svd_v = SvdFactors(u=u_v, sigma=np.ones(r), b_t=f_v, fused=f_v)
    lw = dummy_lw(d, r, u_k @ f_k, u_v @ f_v, svd_k=svd_k, svd_v=svd_v)
    st = fp16_outlier_channel_variant(make_cache("xq-gqa", 0, LayerPolicy.uniform(3, 1), 128,
                                                 group_size=128), True)
    st.prefill(x[:250], lw)
    outs = []
    for t in range(12):
        st.decode_append(x[250 + t], lw)
        k, v = st.rematerialize(lw, np.arange(250 + t + 1))
        qr = apply_rope(q[t:t + 1], np.array([250 + t]), 128)
        outs.append(_attention(qr, k, v, H, g)[0])
    be.update({"gqa1_attn": np.stack(outs), "gqa1_k": k.astype(np.float32),
               "gqa1_kcodes": st.k_stream.q.codes, "gqa1_kscales": st.k_stream.q.scales,
               "gqa1_first": np.asarray(st.k_stream.first_channel, np.float64)})
    np.savez_compressed(os.path.join(HERE, "backends.npz"), **be)

    for f in ("quant", "pack", "rope", "backends"):
        p = os.path.join(HERE, f + ".npz")
        print(f"{p}: {os.path.getsize(p) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
