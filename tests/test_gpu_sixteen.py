"""16-bit pass-through for every variant (the reference's
``TestIdentityAtSixteenBits``, tests/test_cache.py:64-75).

At bits=16 a QuantizedTensor keeps its raw rows (quant.py:117-118), so every
variant rematerializes the fp16 baseline's K/V. The device backends keep the raw
rows as fp16 (the 16 bits the reference charges), so the identity holds to fp16
rounding instead of float64 round-off. Checked through the reference-signature
``make_cache`` with the reference's own LayerWeights / Accumulator objects, and
against the reference's own 16-bit run, for a base layer and a delta layer.
"""

import os
import sys

import numpy as np
import pytest

from _util import ROOT, rel_err

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "oracle", "_ref")
if not os.path.isdir(os.path.join(REF, "xcache")):
    pytest.skip("oracle/_ref (the reference package) is not built", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)

D, KVW, HD = 512, 256, 128
TOL = 3e-3  # fp16 storage of the raw rows (2^-11 relative) through a d=512 projection


def _weights(seed=0, kvw=KVW):
    from xcache.cache import LayerWeights
    from xcache.linalg import RngState, gen_weights, svd_thin

    rng = RngState(seed)
    w_k = gen_weights(rng, D, kvw)
    w_v = gen_weights(rng, D, kvw)
    return LayerWeights(gamma_attn=np.ones(D), gamma_mlp=np.ones(D), w_q=gen_weights(rng, D, D),
                        w_k=w_k, w_v=w_v, w_o=gen_weights(rng, D, D),
                        w_up=gen_weights(rng, D, 2 * D), w_down=gen_weights(rng, 2 * D, D),
                        svd_k=svd_thin(w_k), svd_v=svd_thin(w_v),
                        svd_kv=svd_thin(np.hstack([w_k, w_v])) if 2 * kvw <= D else None)


def _x(seed, rows):
    from xcache.linalg import RngState, gen_weights

    return gen_weights(RngState(seed), rows, D) * np.sqrt(D)


def _run(mod, variant, lws, xs, bits, n_decode=2):
    """Layers 0..len(lws)-1 of one sequence (base_layers=1: layer 0 seeds, the rest
    are delta layers); returns the last layer's (K, V) after n_decode appends."""
    n_layers = len(lws)
    policy = mod.LayerPolicy.uniform(bits, max(2, n_layers))
    policy.base_layers = policy.high_precision_prefix = 1
    states = [mod.make_cache(variant, i, policy, HD, 128) for i in range(n_layers)]
    n0 = xs[0].shape[0] - n_decode
    from xcache.cache import Accumulator

    acc = Accumulator() if states[0].needs_accumulator else None
    for st, lw, x in zip(states, lws, xs):
        mod.prefill(st, x[:n0], lw, acc)
    for t in range(n0, n0 + n_decode):
        acc = Accumulator() if states[0].needs_accumulator else None
        for st, lw, x in zip(states, lws, xs):
            mod.decode_append(st, x[t], lw, acc)
    # the last layer's K/V; a delta layer rebuilds them from the last pass's accumulator
    return mod.rematerialize(states[-1], lws[-1], np.arange(n0 + n_decode), acc)


@pytest.mark.parametrize("variant", ["kvq", "xq-mha", "xq-gqa", "xq-cl-mha", "xq-cl-gqa"])
@pytest.mark.parametrize("n_layers", [1, 2])
def test_sixteen_bits_match_full_precision(variant, n_layers):
    from xcache import cache as R

    from paper_2508_10395_b200 import cache as M

    if n_layers == 2 and variant not in ("xq-cl-mha", "xq-cl-gqa"):
        pytest.skip("one layer covers the non-cross-layer variants")
    lws = [_weights(s) for s in range(n_layers)]
    xs = [_x(10 + s, 150) for s in range(n_layers)]  # 148 prefilled (a 128-row group + 20) + 2
    k_fp, v_fp = _run(R, "fp16", lws, xs, 16)
    k, v = _run(M, variant, lws, xs, 16)
    assert isinstance(k, np.ndarray) and k.shape == k_fp.shape
    ek, ev = rel_err(k, k_fp), rel_err(v, v_fp)
    print(f"{variant} x{n_layers} 16-bit vs fp16 baseline: K {ek:.2e} V {ev:.2e}")
    assert ek <= TOL and ev <= TOL, (ek, ev)
    rk, rv = _run(R, variant, lws, xs, 16)  # the reference's own 16-bit run
    assert rel_err(k, rk) <= TOL and rel_err(v, rv) <= TOL


@pytest.mark.parametrize("variant", ["xq-gqa", "xq-cl-mha", "xq-cl-gqa", "kvq"])
def test_sixteen_bits_decode_attend(variant):
    """The fused decode at 16 bits (fp16-row A operands) against attention over the
    rematerialized K/V of the same backend."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import xq_oracle as O

    from paper_2508_10395_b200 import cache as M

    dev = torch.device("cuda", 0)
    g = 2 if variant in ("xq-gqa", "xq-cl-gqa") else 1
    H = D // HD
    lw_ref = _weights(3, D // g)
    lw = M.as_layer_weights(lw_ref, dev)
    policy = M.LayerPolicy.uniform(16, 2)
    policy.base_layers = policy.high_precision_prefix = 1
    n_layers = 2 if variant.startswith("xq-cl") else 1
    states = [M.make_cache(variant, i, policy, HD, hidden_dim=D, n_heads=H, kv_group=g, n_slots=2,
                           max_len=512, device=dev, exact=True) for i in range(n_layers)]
    rng = np.random.default_rng(4)
    x = torch.as_tensor(rng.normal(size=(n_layers, 2, 300, D)), device=dev)
    acc = M.Accumulator(2, 512, D, dev) if states[0].needs_accumulator else None
    for i, st in enumerate(states):
        st.prefill(x[i, :, :299], lw, acc)
    for i, st in enumerate(states):
        st.decode_append(x[i, :, 299], lw, acc)
    q = torch.as_tensor(rng.normal(size=(2, H, HD)), dtype=torch.float32, device=dev)
    st = states[-1]
    out = st.decode_attend(q, lw, acc).cpu().numpy()
    for s in range(2):
        k, v = st.rematerialize(lw, np.arange(300), acc, slot=s)
        qr = O.apply_rope(q[s].double().cpu().numpy().reshape(1, -1), [299], HD)
        ref = O.attention(qr, k.double().cpu().numpy(), v.double().cpu().numpy(), H, g)[0]
        err = rel_err(out[s].reshape(-1), ref)
        print(f"{variant} slot {s}: fused 16-bit decode vs remat attention {err:.2e}")
        assert err <= 2e-2, err
