"""Pin the CPU oracle (oracle/xq_oracle.py) to the reference's own outputs.

The golden vectors in tests/golden/*.npz were produced by the UNMODIFIED
reference (tests/golden/make_golden.py). Integer results must match bit for
bit; float results to float64 round-off (or float32 storage precision where
the fixture stores float32).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import xq_oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def bf16f(b):
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def rel(a, b):
    return np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-300)


class TestQuantGolden:
    @pytest.mark.parametrize("bits", [2, 3, 4, 8])
    @pytest.mark.parametrize("cols", [17, 64, 130, 256])
    @pytest.mark.parametrize("gs", [32, 128])
    def test_quantize_groups_bit_exact(self, bits, cols, gs):
        z = load("quant")
        k = f"b{bits}_c{cols}_g{gs}"
        x = z[k + "_x"].astype(np.float64)
        c, s, zp = O.quantize_groups(x, gs, bits)
        assert np.array_equal(c, z[k + "_codes"])
        assert np.array_equal(s, z[k + "_scales"])
        assert np.array_equal(zp, z[k + "_zps"])
        deq = O.dequantize_groups(c, s, zp, gs)
        assert np.array_equal(deq.astype(np.float32), z[k + "_deq"])

    @pytest.mark.parametrize("bits", [2, 3, 4])
    def test_d4096_rows_and_packed_bytes(self, bits):
        z = load("quant")
        x = bf16f(z[f"d4096_b{bits}_xbf16"])
        c, s, zp = O.quantize_groups(x, 128, bits)
        assert np.array_equal(c, z[f"d4096_b{bits}_codes"])
        assert np.array_equal(s, z[f"d4096_b{bits}_scales"])
        assert np.array_equal(O.pack_rows(c, bits), z[f"d4096_b{bits}_packed"])

    def test_per_channel(self):
        z = load("quant")
        x = bf16f(z["perchan_b3_xbf16"])
        c, s, zp = O.quantize(x, 3, O.PER_CHANNEL, 128)
        assert np.array_equal(c, z["perchan_b3_codes"])
        assert np.array_equal(s, z["perchan_b3_scales"])
        assert np.array_equal(zp, z["perchan_b3_zps"])


class TestPackGolden:
    @pytest.mark.parametrize("bits", [2, 3, 4, 8])
    def test_pack_unpack(self, bits):
        z = load("pack")
        for n in list(range(0, 65)) + [127, 128, 129, 1000, 4096]:
            codes = z[f"b{bits}_n{n}_codes"]
            words = O.pack_codes(codes, bits)
            assert np.array_equal(words, z[f"b{bits}_n{n}_words"]), n
            assert np.array_equal(O.unpack_codes(words, bits, n), codes)

    def test_xqt1_known_answer(self):
        # tests/test_quant.py:210-223 of the reference: codes 0,1,2,3 -> 0b11100100
        kat = load("pack")["xqt1_kat"]
        words = kat[-8:].view("<u8")
        assert int(words[0]) == 0b11100100
        assert np.array_equal(O.pack_codes(np.array([0, 1, 2, 3], np.uint8), 2), words)


class TestRopeGolden:
    def test_rope(self):
        z = load("rope")
        assert rel(O.apply_rope(z["m"], z["pos"], 128), z["out_hd128"]) <= 1e-15
        assert rel(O.apply_rope(z["m"], z["pos"], 8), z["out_hd8"]) <= 1e-15

    def test_position_zero_identity(self):
        m = np.random.default_rng(3).normal(size=(4, 16))
        assert np.array_equal(O.apply_rope(m, np.zeros(4), 8), m)


class TestBackendsGolden:
    @pytest.mark.parametrize("bits", [2, 3, 4, 16])
    def test_xq_mha(self, bits):
        z = load("backends")
        k = f"mha_b{bits}"
        x, wk, wv, q = (bf16f(z[k + s]) for s in ("_x", "_wk", "_wv", "_q"))
        n_pre, n_dec = 290, 10
        st = O.XqMhaCache(bits, 128, 128)
        st.append(x[:n_pre])
        outs = []
        for t in range(n_dec):
            st.append(x[n_pre + t])
            kk, vv = st.remat(wk, wv)
            qr = O.apply_rope(q[t:t + 1], [n_pre + t], 128)  # model.py:234
            outs.append(O.attention(qr, kk, vv, 2, 1)[0])
        if bits != 16:
            assert np.array_equal(st.stream.codes, z[k + "_codes"])
            assert np.array_equal(st.stream.scales, z[k + "_scales"])
        if k + "_k" in z.files:
            assert rel(kk, z[k + "_k"]) <= 1e-6
            assert rel(vv, z[k + "_v"]) <= 1e-6
        assert rel(np.stack(outs), z[k + "_attn"]) <= 1e-12

    def test_fp16_baseline(self):
        z = load("backends")
        x, wk, wv, q = (bf16f(z["mha_b4" + s]) for s in ("_x", "_wk", "_wv", "_q"))
        st = O.Fp16Cache(128)
        st.append(x, wk, wv)
        kk, vv = st.remat()
        assert rel(kk, z["fp16_k"]) <= 1e-6
        qr = O.apply_rope(q[-1:], [x.shape[0] - 1], 128)
        assert rel(O.attention(qr, kk, vv, 2, 1)[0], z["fp16_attn"]) <= 1e-12

    def test_xq_gqa(self):
        z = load("backends")
        x, uk, uv, fk, fv, q = (bf16f(z["gqa_" + s]) for s in ("x", "uk", "uv", "fk", "fv", "q"))
        n_pre, n_dec = 250, 12
        st = O.XqGqaCache(3, 128, 128)
        st.prefill(x[:n_pre] @ uk, x[:n_pre] @ uv)
        outs, bufs = [], []
        for t in range(n_dec):
            st.push(x[n_pre + t] @ uk, x[n_pre + t] @ uv)
            kk, vv = st.remat(fk, fv)
            qr = O.apply_rope(q[t:t + 1], [n_pre + t], 128)
            outs.append(O.attention(qr, kk, vv, 8, 4)[0])
            bufs.append(len(st.k_stream.buf))
        assert bufs == list(z["gqa_buf_len"])
        assert np.array_equal(st.k_stream.codes, z["gqa_kcodes"])
        assert np.array_equal(st.k_stream.scales, z["gqa_kscales"])
        assert np.array_equal(st.v_stream.codes, z["gqa_vcodes"])
        assert rel(kk, z["gqa_k"]) <= 1e-6
        assert rel(vv, z["gqa_v"]) <= 1e-6
        assert rel(np.stack(outs), z["gqa_attn"]) <= 1e-12

    def test_xq_cl_mha(self):
        z = load("backends")
        xs = bf16f(z["cl_x"])
        wks, wvs, q = bf16f(z["cl_wk"]), bf16f(z["cl_wv"]), bf16f(z["cl_q"])
        bits, base = list(z["cl_bits"]), int(z["cl_base"])
        assert bits == O.policy_for_bits(2, 6)[0]
        n_pre, n_dec = 140, 3
        st = O.XqClMhaStack(bits, base, 128, 128)
        st.step([x[:n_pre] for x in xs])
        for t in range(n_dec):
            accs, kvs = st.step([x[n_pre + t] for x in xs], list(zip(wks, wvs)))
        for i in range(6):
            assert np.array_equal(st.streams[i].codes, z[f"cl_codes{i}"]), i
            assert np.array_equal(st.streams[i].scales, z[f"cl_scales{i}"]), i
        assert rel(accs[-1], z["cl_acc_last"]) <= 1e-6
        assert rel(kvs[2][0], z["cl_k"][0]) <= 1e-6
        assert rel(kvs[-1][0], z["cl_k"][1]) <= 1e-6
        assert rel(kvs[-1][1], z["cl_v"][1]) <= 1e-6
        pos = [n_pre + n_dec - 1]
        attn = np.stack([O.attention(O.apply_rope(q[i:i + 1], pos, 128), kv[0], kv[1], 2, 1)[0]
                         for i, kv in enumerate(kvs)])
        assert rel(attn, z["cl_attn"]) <= 1e-12


    def test_xq_cl_gqa(self):
        z = load("backends")
        xs = bf16f(z["clg_x"])
        us = z["clg_u"].astype(np.float64)
        fuseds, q = bf16f(z["clg_fused"]), bf16f(z["clg_q"])
        bits, base = list(z["clg_bits"]), int(z["clg_base"])
        assert bits == O.policy_for_bits(3, 5)[0]
        n_pre, n_dec = 250, 8
        st = O.XqClGqaStack(bits, base, 128, 128)
        subs = list(zip(us, fuseds))
        st.step([x[:n_pre] for x in xs], subs)
        for t in range(n_dec):
            out = st.step([x[n_pre + t] for x in xs], subs)
        for i in range(5):
            assert np.array_equal(st.streams[i].codes, z[f"clg_codes{i}"]), i
            assert np.array_equal(st.streams[i].scales, z[f"clg_scales{i}"]), i
            assert rel(st.streams[i].buf, z[f"clg_buf{i}"]) <= 1e-9, i
        assert rel(out[-1][3], z["clg_acc_last"]) <= 1e-6
        assert rel(out[2][1], z["clg_k"][0]) <= 1e-6
        assert rel(out[-1][1], z["clg_k"][1]) <= 1e-6
        assert rel(out[-1][2], z["clg_v"][1]) <= 1e-6
        pos = [n_pre + n_dec - 1]
        attn = np.stack([O.attention(O.apply_rope(q[i:i + 1], pos, 128), o[1], o[2], 8, 4)[0]
                         for i, o in enumerate(out)])
        assert rel(attn, z["clg_attn"]) <= 1e-10


    def test_kvq(self):
        z = load("backends")
        x, q = bf16f(z["kvq_x"]), bf16f(z["kvq_q"])
        wk, wv = bf16f(z["kvq_wk"]), bf16f(z["kvq_wv"])
        st = O.KvqCache(3, 128, 128)
        n_pre = 250
        st.prefill(x[:n_pre] @ wk, x[:n_pre] @ wv)
        outs = []
        for t in range(12):
            st.push(x[n_pre + t] @ wk, x[n_pre + t] @ wv)
            k, v = st.remat()
            outs.append(O.attention(O.apply_rope(q[t:t + 1], [n_pre + t], 128), k, v, 4, 2)[0])
        assert np.array_equal(st.k.codes, z["kvq_kcodes"])
        assert np.array_equal(st.k.scales, z["kvq_kscales"])
        assert np.array_equal(st.v.codes, z["kvq_vcodes"])
        assert np.array_equal(st.v.scales, z["kvq_vscales"])
        assert rel(st.v.buf, z["kvq_vbuf"]) <= 1e-12
        assert rel(k, z["kvq_k"]) <= 1e-6 and rel(v, z["kvq_v"]) <= 1e-6
        assert rel(np.stack(outs), z["kvq_attn"]) <= 1e-12


    def test_xq_gqa_fp16_first_channel(self):
        z = load("backends")
        x, q = bf16f(z["gqa_x"]), bf16f(z["gqa_q"])
        uk, uv = bf16f(z["gqa_uk"]), bf16f(z["gqa_uv"])
        fk, fv = bf16f(z["gqa_fk"]), bf16f(z["gqa_fv"])
        st = O.XqGqaCache(3, 128, 128, fp16_first_channel=True)
        st.prefill(x[:250] @ uk, x[:250] @ uv)
        outs = []
        for t in range(12):
            st.push(x[250 + t] @ uk, x[250 + t] @ uv)
            kk, vv = st.remat(fk, fv)
            outs.append(O.attention(O.apply_rope(q[t:t + 1], [250 + t], 128), kk, vv, 8, 4)[0])
        assert np.array_equal(st.k_stream.codes, z["gqa1_kcodes"])
        assert np.array_equal(st.k_stream.scales, z["gqa1_kscales"])
        assert rel(st.k_stream.first, z["gqa1_first"]) <= 1e-12
        assert rel(kk, z["gqa1_k"]) <= 1e-6
        assert rel(np.stack(outs), z["gqa1_attn"]) <= 1e-12


class TestSysmodel:
    def test_compression_factors(self):
        # PAPER.md:371/373/563-579 via sysmodel.normalized_kv_size
        bits3, _ = O.policy_for_bits(3, 32)
        assert abs(O.normalized_kv_size("xq-mha", [4] * 32) - 0.1328) < 1e-3
        assert abs(1 / O.normalized_kv_size("xq-mha", bits3) - 9.57) < 0.01
        bits2, _ = O.policy_for_bits(2, 32)
        assert abs(1 / O.normalized_kv_size("xq-cl-mha", bits2) - 13.13) < 0.01

    def test_breakeven_h100(self):
        # tests/test_acceptance.py:60-81 of the reference: 2281 / 40627 on H100
        mha = O.breakeven_length("xq-mha", 4096, 1, 2, 756e12, 2e12, weight_bytes=2 * 12 * 4096**2)
        assert round(mha) == 2281
