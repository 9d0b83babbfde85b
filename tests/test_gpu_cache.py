"""Cache arenas and backends on the GPU vs the reference's golden vectors and
the oracle.

Parity contract:
* codes bit-exact with the reference quantizer, packed rows byte-identical
  to pack_codes(row);
* rematerialised K/V (float32 SIMT path) within rel 1e-4 of the oracle fed
  the stored fp16 scale / zero point;
* fused tcgen05 decode attention within rel 2e-2 (the north-star bf16/fp16
  tolerance) of the reference's own attention output.
"""

import numpy as np
import pytest

from _util import bf16f, fp16_round, golden, rel_err, torch_bf16

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("kernel_path")]

FUSED_TOL = 2e-2
F32_TOL = 1e-4


@pytest.fixture(scope="module")
def M():
    import paper_2508_10395_b200.cache as cache

    return cache


def _params_np(stream, n_rows):
    ng = -(-stream.width // stream.g)
    p = stream.params[:n_rows, :ng].float().cpu().numpy()
    return p[..., 0].astype(np.float64), p[..., 1].astype(np.float64)


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_append_rows_bytes_identical(M, bits):
    import torch

    import xq_oracle as O

    z = golden("quant")
    xb = z[f"d4096_b{bits}_xbf16"]
    x = torch_bf16(xb)
    s = M.PackedStream(bits, M.TOKEN, 4096, 128, n_slots=1, max_len=64, device="cuda")
    s.fill_rows(x, 0, 0)
    torch.cuda.synchronize()
    got = s.codes[:16].cpu().numpy()
    assert np.array_equal(got, z[f"d4096_b{bits}_packed"])
    sc, zp = _params_np(s, 16)
    assert np.array_equal(sc, fp16_round(z[f"d4096_b{bits}_scales"]))
    assert np.array_equal(zp, fp16_round(z[f"d4096_b{bits}_zps"]))
    # decode path: one row per slot at position lens-1
    s2 = M.PackedStream(bits, M.TOKEN, 4096, 128, n_slots=16, max_len=8, device="cuda")
    lens = torch.full((16,), 3, dtype=torch.int32, device="cuda")
    s2.append_token_rows(x, lens)
    torch.cuda.synchronize()
    rows = s2.codes.view(16, 8, -1)[:, 2].cpu().numpy()
    assert np.array_equal(rows, z[f"d4096_b{bits}_packed"])
    assert np.array_equal(O.pack_rows(z[f"d4096_b{bits}_codes"], bits), rows)


def test_per_channel_flush_matches_reference(M):
    import torch

    import xq_oracle as O

    z = golden("quant")
    xb = z["perchan_b3_xbf16"]  # [256, 96]
    x = torch_bf16(xb).float()
    s = M.PackedStream(3, M.CHANNEL, 96, 128, n_slots=1, max_len=256, device="cuda")
    s.flush_blocks(x.contiguous(), [0, 128])
    torch.cuda.synchronize()
    codes = s.codes.cpu().numpy()
    unpacked = np.stack([O.unpack_codes(codes[r].view(np.uint64), 3, 96) for r in range(256)])
    assert np.array_equal(unpacked, z["perchan_b3_codes"])
    # dequant through the library (planar permuted params) vs oracle with fp16 params
    out = torch.empty((256, 96), dtype=torch.float32, device="cuda")
    from paper_2508_10395_b200 import _native as N

    N.call("xq_dequant_rows", N.ptr(s.codes), s.row_bytes, N.ptr(s.params), 1, 3, 128, 96, 0,
           256, N.ptr(out), N.stream_of())
    ref = O.dequantize(z["perchan_b3_codes"], fp16_round(z["perchan_b3_scales"]),
                       fp16_round(z["perchan_b3_zps"]), 3, O.PER_CHANNEL, 128)
    assert rel_err(out.cpu().numpy(), ref) <= 1e-6


def _weights(M, **kw):
    return M.LayerWeights(**kw)


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_xq_mha_against_reference(M, bits):
    import torch

    import xq_oracle as O

    z = golden("backends")
    k = f"mha_b{bits}"
    x = torch_bf16(z[k + "_x"])
    q = torch_bf16(z[k + "_q"]).float()
    w = _weights(M, w_k=torch_bf16(z[k + "_wk"]), w_v=torch_bf16(z[k + "_wv"]))
    pol = M.LayerPolicy.uniform(bits, 1)
    st = M.make_cache("xq-mha", 0, pol, 128, 128, n_slots=1, max_len=512, hidden_dim=256,
                      n_heads=2)
    n_pre, n_dec = 290, 10
    st.prefill(x[:n_pre], w)
    errs = []
    for t in range(n_dec):
        st.decode_append(x[n_pre + t][None], w)
        out = st.decode_attend(q[t][None], w)
        errs.append(rel_err(out.reshape(-1).cpu().numpy(), z[k + "_attn"][t]))
    assert max(errs) <= FUSED_TOL, errs
    # codes bit-exact and K/V of the float32 path vs oracle with the stored params
    n = n_pre + n_dec
    codes = st.stream.codes[:n].cpu().numpy()
    unpacked = np.stack([O.unpack_codes(codes[r].view(np.uint64), bits, 256) for r in range(n)])
    assert np.array_equal(unpacked, z[k + "_codes"])
    kk, vv = st.rematerialize(w, np.arange(n))
    sc, zp = _params_np(st.stream, n)
    xh = O.dequantize_groups(unpacked, sc, zp, 128)
    wk, wv = bf16f(z[k + "_wk"]), bf16f(z[k + "_wv"])
    assert rel_err(kk.cpu().numpy(), O.apply_rope(xh @ wk, np.arange(n), 128)) <= F32_TOL
    assert rel_err(vv.cpu().numpy(), xh @ wv) <= F32_TOL
    if k + "_k" in z.files:
        assert rel_err(kk.cpu().numpy(), z[k + "_k"]) <= 5e-3


def test_fp16_baseline_against_reference(M):
    import torch

    z = golden("backends")
    x = torch_bf16(z["mha_b4_x"])
    q = torch_bf16(z["mha_b4_q"]).float()
    w = _weights(M, w_k=torch_bf16(z["mha_b4_wk"]), w_v=torch_bf16(z["mha_b4_wv"]))
    st = M.make_cache("fp16", 0, M.LayerPolicy.uniform(16, 1), 128, n_slots=1, max_len=512,
                      hidden_dim=256, n_heads=2)
    st.prefill(x[:299], w)
    st.decode_append(x[299][None], w)
    out = st.decode_attend(q[-1][None], w)
    assert rel_err(out.reshape(-1).cpu().numpy(), z["fp16_attn"]) <= FUSED_TOL
    kk, vv = st.rematerialize(w, np.arange(300))
    assert rel_err(kk.cpu().numpy(), z["fp16_k"]) <= 1e-2
    assert rel_err(vv.cpu().numpy(), z["fp16_v"]) <= 1e-2


def test_xq_gqa_against_reference(M):
    import torch

    z = golden("backends")
    x = torch_bf16(z["gqa_x"])
    q = torch_bf16(z["gqa_q"]).float()
    w = _weights(M, u_k=torch_bf16(z["gqa_uk"]), u_v=torch_bf16(z["gqa_uv"]),
                 fused_k=torch_bf16(z["gqa_fk"]), fused_v=torch_bf16(z["gqa_fv"]))
    st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, 128, n_slots=1,
                      max_len=512, hidden_dim=1024, n_heads=8, kv_group=4)
    n_pre, n_dec = 250, 12
    st.prefill(x[:n_pre], w)
    errs = []
    for t in range(n_dec):
        st.decode_append(x[n_pre + t][None], w)
        assert int(st.n_tokens[0] - st.k_stream.n_flushed[0]) == int(z["gqa_buf_len"][t])
        out = st.decode_attend(q[t][None], w)
        errs.append(rel_err(out.reshape(-1).cpu().numpy(), z["gqa_attn"][t]))
    assert max(errs) <= FUSED_TOL, errs
    kk, vv = st.rematerialize(w, np.arange(n_pre + n_dec))
    assert rel_err(kk.cpu().numpy(), z["gqa_k"]) <= 2e-2
    assert rel_err(vv.cpu().numpy(), z["gqa_v"]) <= 2e-2


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_xq_cl_mha_against_reference(M, precision):
    import torch

    z = golden("backends")
    xs = torch_bf16(z["cl_x"])  # [6, 143, 256]
    q = torch_bf16(z["cl_q"]).float()
    bits = [int(b) for b in z["cl_bits"]]
    pol = M.LayerPolicy(bits, base_layers=int(z["cl_base"]), high_precision_prefix=3)
    ws = [_weights(M, w_k=torch_bf16(z["cl_wk"][i]), w_v=torch_bf16(z["cl_wv"][i]))
          for i in range(6)]
    kw = dict(n_slots=1, max_len=256, hidden_dim=256, n_heads=2)
    sts = [M.make_cache("xq-cl-mha", i, pol, 128, 128, **kw) for i in range(6)]
    acc = M.Accumulator(1, 256, 256, precision=precision)
    n_pre, n_dec = 140, 3
    for i in range(6):
        sts[i].prefill(xs[i, :n_pre], ws[i], acc)
    for t in range(n_dec):
        outs = []
        for i in range(6):
            sts[i].decode_append(xs[i, n_pre + t][None], ws[i], acc)
            outs.append(sts[i].decode_attend(q[i][None], ws[i], acc).reshape(-1).cpu().numpy())
    for i in range(6):
        assert rel_err(outs[i], z["cl_attn"][i]) <= FUSED_TOL, i
    n = n_pre + n_dec
    assert rel_err(acc.rows(0, n).cpu().numpy(), z["cl_acc_last"]) <= 3e-2


def test_xq_cl_gqa_against_reference(M):
    """xq-cl-gqa (cache.py:538-604): 5 layers (base 3), d=1024, 8 query heads on 2 KV
    heads, shared K|V latent r=512, decode crossing the per-channel flush.

    * every layer's codes (base and delta) bit-exact with the reference's own run:
      latents are formed in float64 against a float64 accumulator row that follows
      the reference's reconstruct() exactly (flushed groups included);
    * every layer's fused decode attention within 2e-2 of the reference itself;
    * the fp16 remat accumulator and the delta layers' K/V within 2e-2.
    """
    import torch

    import xq_oracle as O

    z = golden("backends")
    xs = torch_bf16(z["clg_x"])  # [5, 258, 1024]
    xsd = bf16f(z["clg_x"])
    q = torch_bf16(z["clg_q"]).float()
    bits = [int(b) for b in z["clg_bits"]]
    pol = M.LayerPolicy(bits, base_layers=int(z["clg_base"]), high_precision_prefix=3)
    ws = [_weights(M, u_kv=torch.from_numpy(z["clg_u"][i]).cuda(),
                   fused_kv=torch_bf16(z["clg_fused"][i])) for i in range(5)]
    subs = [(z["clg_u"][i].astype(np.float64), bf16f(z["clg_fused"][i])) for i in range(5)]
    kw = dict(n_slots=1, max_len=384, hidden_dim=1024, n_heads=8, kv_group=4)
    sts = [M.make_cache("xq-cl-gqa", i, pol, 128, 128, **kw) for i in range(5)]
    acc = M.Accumulator(1, 384, 1024, precision="fp16")
    ost = O.XqClGqaStack(bits, 3, 128, 128)
    n_pre, n_dec = 250, 8
    for i in range(5):
        sts[i].prefill(xs[i, :n_pre], ws[i], acc)
    ost.step([x[:n_pre] for x in xsd], subs)
    for t in range(n_dec):
        outs = []
        for i in range(5):
            sts[i].decode_append(xs[i, n_pre + t][None], ws[i], acc)
            outs.append(sts[i].decode_attend(q[i][None], ws[i], acc).reshape(-1).cpu().numpy())
        o = ost.step([x[n_pre + t] for x in xsd], subs)
    n = n_pre + n_dec
    qd = bf16f(z["clg_q"])
    for i in range(5):
        assert rel_err(outs[i], z["clg_attn"][i]) <= FUSED_TOL, i
        s = sts[i].stream
        got = s.codes[:256].cpu().numpy()
        un = np.stack([O.unpack_codes(got[r].view(np.uint64), bits[i], 512) for r in range(256)])
        assert np.array_equal(un, z[f"clg_codes{i}"]), i
        assert np.array_equal(un, ost.streams[i].codes[:256]), i
        ref = O.attention(O.apply_rope(qd[i:i + 1], [n - 1], 128), o[i][1], o[i][2], 8, 4)[0]
        assert rel_err(outs[i], ref) <= FUSED_TOL, i
    assert rel_err(acc.x16[0, :n].float().cpu().numpy(), o[-1][3]) <= 2e-2
    kk, vv = sts[2].rematerialize(ws[2], np.arange(n), acc)
    assert rel_err(kk.cpu().numpy(), z["clg_k"][0]) <= 2e-2
    kk, vv = sts[4].rematerialize(ws[4], np.arange(n), acc)
    assert rel_err(kk.cpu().numpy(), o[-1][1]) <= 2e-2
    assert rel_err(vv.cpu().numpy(), o[-1][2]) <= 2e-2


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_xqt1_export_matches_reference_dump(M, bits):
    """XQT1 (quant.py:232-254) of the GPU X cache vs the reference's dump_qtensor:
    header and packed codes byte-identical, scale/zp grids = the stored fp16
    values (the reference's float64 grids rounded to fp16)."""
    import torch

    z = golden("backends")
    key = f"mha_b{bits}"
    x = torch_bf16(z[key + "_x"])
    st = M.make_cache("xq-mha", 0, M.LayerPolicy.uniform(bits, 1), 128, 128, n_slots=2,
                      max_len=512, hidden_dim=256, n_heads=2)
    st.prefill(x[:300], M.LayerWeights(), slot=1)
    got = np.frombuffer(st.stream.export_xqt1(1, 300), dtype=np.uint8)
    ref = z[key + "_xqt1"]
    assert got.shape == ref.shape
    n_grid = 300 * 2 * 8  # scales + zps, float64
    assert np.array_equal(got[:24], ref[:24])  # magic + header
    assert np.array_equal(got[24 + 2 * n_grid:], ref[24 + 2 * n_grid:])  # packed codes
    gs = got[24:24 + 2 * n_grid].view(np.float64)
    rs = ref[24:24 + 2 * n_grid].view(np.float64)
    assert np.array_equal(gs, fp16_round(rs))


def test_xqt1_export_per_channel(M):
    """Per-channel (xq-gqa K latent) export: flushed groups only, params back in
    natural channel order; codes byte-identical with the reference's dump."""
    import torch

    z = golden("backends")
    x = torch_bf16(z["gqa_x"])
    w = _weights(M, u_k=torch_bf16(z["gqa_uk"]), u_v=torch_bf16(z["gqa_uv"]),
                 fused_k=torch_bf16(z["gqa_fk"]), fused_v=torch_bf16(z["gqa_fv"]))
    st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, 128, n_slots=1,
                      max_len=512, hidden_dim=1024, n_heads=8, kv_group=4)
    st.prefill(x[:250], w)
    for t in range(12):
        st.decode_append(x[250 + t][None], w)
    got = np.frombuffer(st.k_stream.export_xqt1(0, 262), dtype=np.uint8)
    ref = z["gqa_kxqt1"]
    assert got.shape == ref.shape
    n_grid = 2 * 256 * 8
    assert np.array_equal(got[:24], ref[:24])
    # latents are fp32 GEMVs here (float64 in the reference): codes agree except at
    # rounding boundaries; the grids to fp16 rounding of the fp32-vs-fp64 latents
    gc, rc = got[24 + 2 * n_grid:], ref[24 + 2 * n_grid:]
    assert np.mean(gc != rc) <= 1e-3
    gs = got[24:24 + 2 * n_grid].view(np.float64)
    rs = ref[24:24 + 2 * n_grid].view(np.float64)
    assert np.max(np.abs(gs - rs) / np.maximum(np.abs(rs), 1e-3)) <= 2e-3


def test_xq_gqa_fp16_outlier_channel_against_reference(M):
    """fp16 outlier channel (cache.py:403-409, 653-658): channel 0 of the K latent
    in full precision. The reference's run on the xq-gqa golden inputs; codes of
    channels 1..r-1 bit-exact (stage-wise: the GPU latent is an fp32 GEMV)."""
    import torch

    import xq_oracle as O

    z = golden("backends")
    x = torch_bf16(z["gqa_x"])
    q = torch_bf16(z["gqa_q"]).float()
    w = _weights(M, u_k=torch_bf16(z["gqa_uk"]), u_v=torch_bf16(z["gqa_uv"]),
                 fused_k=torch_bf16(z["gqa_fk"]), fused_v=torch_bf16(z["gqa_fv"]))
    st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, 128, n_slots=1,
                      max_len=512, hidden_dim=1024, n_heads=8, kv_group=4)
    M.fp16_outlier_channel_variant(st, True)
    st.prefill(x[:250], w)
    errs = []
    for t in range(12):
        st.decode_append(x[250 + t][None], w)
        out = st.decode_attend(q[t][None], w)
        errs.append(rel_err(out.reshape(-1).cpu().numpy(), z["gqa1_attn"][t]))
    assert max(errs) <= FUSED_TOL, errs
    kk, _ = st.rematerialize(w, np.arange(262))
    assert rel_err(kk.cpu().numpy(), z["gqa1_k"]) <= 2e-2
    ks = st.k_stream
    got = ks.codes[:256].cpu().numpy()
    un = np.stack([O.unpack_codes(got[r].view(np.uint64), 3, 256) for r in range(256)])
    assert np.mean(un[:, 1:] != z["gqa1_kcodes"]) <= 1e-3
    assert rel_err(ks.first[:256].cpu().numpy(), z["gqa1_first"]) <= 1e-5
    with pytest.raises(M.UsageError):
        M.fp16_outlier_channel_variant(st, False)  # not on a non-empty cache
