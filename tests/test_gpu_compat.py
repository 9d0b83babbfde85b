"""The drop-in boundary, exercised by the reference's own code.

* The reference's decode driver ``model._Session`` (model.py:185-240) runs
  unchanged with ``xcache.model.make_cache`` pointed at this package's
  ``cache.make_cache`` (the reference signature: no sizes, NumPy LayerWeights
  with svd_k / svd_v / svd_kv, a fresh ``Accumulator()`` per pass). Its logits
  must stay within 2e-2 (max|err| / max|ref|) of the same session on the
  reference's CPU backends, for every variant.
* The INTEGRATION.md lane stub: the reference's ``xcache._kernels`` bound to
  ``paper_2508_10395_b200.kernels``. The reference's CPU backends then produce
  logits bit-identical to its native lane, and the lane matches both reference
  lanes on the cases of the reference's ``TestLaneEquivalence``
  (tests/test_kernels.py:33-84).

The reference is imported from ``oracle/_ref`` (the unmodified package built by
oracle/build_ref.sh); the tests skip when it is absent.
"""

import os
import sys

import numpy as np
import pytest

from _util import ROOT, rel_err, unpack_rows

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "oracle", "_ref")
if not os.path.isdir(os.path.join(REF, "xcache")):
    pytest.skip("oracle/_ref (the reference package) is not built", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)

TOL = 2e-2
# K/V straight from rematerialize: the codes are the reference's, the arena keeps
# scale / zero point in fp16 (the 16+16 bits per group the reference charges,
# quant.py:44-45), so dequantized rows differ by up to ~5e-4 relative
KV_TOL = 2e-3
N_PROMPT, N_DECODE = 130, 3  # crosses a 128-token per-channel flush
_MODELS: dict = {}


def _model(gqa: bool):
    from xcache.model import ModelConfig, build_model

    key = "gqa" if gqa else "mha"
    if key not in _MODELS:
        cfg = (ModelConfig(hidden_dim=512, n_layers=5, n_heads=4, kv_group=2, seed=1) if gqa
               else ModelConfig(hidden_dim=256, n_layers=5, n_heads=2, kv_group=1, seed=2))
        _MODELS[key] = build_model(cfg)
    return _MODELS[key]


def _session_logits(model, variant, bits):
    from xcache.cache import LayerPolicy
    from xcache.model import _Session

    sess = _Session(model, variant, LayerPolicy.for_bits(bits, model.config.n_layers))
    rng = np.random.default_rng(5)
    prompt = rng.integers(0, model.config.vocab_size, N_PROMPT)
    out = [sess.prefill(prompt)]
    for t in rng.integers(0, model.config.vocab_size, N_DECODE):
        out.append(sess.decode(int(t))[None])
    return np.concatenate(out), sess


@pytest.fixture
def device_backends(monkeypatch):
    """model._Session's make_cache -> this package's (the only change)."""
    import xcache.model as ref_model

    from paper_2508_10395_b200 import cache as M

    monkeypatch.setattr(ref_model, "make_cache", M.make_cache)
    return M


@pytest.mark.parametrize("variant,bits", [
    ("xq-mha", 4), ("xq-mha", 3), ("xq-mha", 16), ("fp16", 16), ("kvq", 4), ("kvq", 16),
    ("xq-cl-mha", 4), ("xq-cl-mha", 2), ("xq-cl-mha", 16), ("xq-gqa", 4), ("xq-gqa", 3),
    ("xq-gqa", 16), ("xq-cl-gqa", 4), ("xq-cl-gqa", 16)])
def test_reference_session_on_device_backends(variant, bits, request):
    model = _model(gqa=variant in ("xq-gqa", "xq-cl-gqa"))
    ref, _ = _session_logits(model, variant, bits)
    M = request.getfixturevalue("device_backends")
    got, sess = _session_logits(model, variant, bits)
    assert all(isinstance(c, M.ReferenceCache) and c.backend is not None for c in sess.caches)
    err = rel_err(got, ref)
    print(f"{variant} {bits}-bit: session logits rel err {err:.2e}")
    assert err <= TOL, err


def test_reference_module_functions(device_backends):
    """cache.prefill / decode_append / rematerialize (cache.py:633-650) and the
    outlier-channel toggle (cache.py:653-658) with reference objects."""
    from xcache import cache as R

    M = device_backends
    model = _model(gqa=True)
    lw = model.layers[0]
    pol = R.LayerPolicy.uniform(4, 1)
    x = np.random.default_rng(3).normal(size=(130, model.config.hidden_dim))
    for enable in (False, True):
        ours = M.fp16_outlier_channel_variant(M.make_cache("xq-gqa", 0, pol, 128), enable)
        theirs = R.fp16_outlier_channel_variant(R.make_cache("xq-gqa", 0, pol, 128), enable)
        for mod, st in ((M, ours), (R, theirs)):
            mod.prefill(st, x[:-1], lw)
            mod.decode_append(st, x[-1], lw)
        assert ours.n_tokens == theirs.n_tokens == 130
        k, v = M.rematerialize(ours, lw, np.arange(130))
        rk, rv = R.rematerialize(theirs, lw, np.arange(130))
        assert isinstance(k, np.ndarray) and k.dtype == np.float64
        assert rel_err(k, rk) <= KV_TOL and rel_err(v, rv) <= KV_TOL, (rel_err(k, rk), rel_err(v, rv))


def test_reference_accumulator_protocol(device_backends):
    """A delta layer driven by the reference's Accumulator(): the device stand-in
    follows the object; misuse raises the reference's UsageError."""
    from xcache import cache as R

    from paper_2508_10395_b200.errors import UsageError

    M = device_backends
    model = _model(gqa=False)
    pol = R.LayerPolicy.for_bits(4, 5)
    x = np.random.default_rng(4).normal(size=(20, model.config.hidden_dim))
    delta_layer = M.make_cache("xq-cl-mha", 4, pol, 128)
    with pytest.raises(UsageError):
        delta_layer.prefill(x, model.layers[4])  # no accumulator
    with pytest.raises(UsageError):
        delta_layer.prefill(x, model.layers[4], R.Accumulator())  # not seeded
    ours = [M.make_cache("xq-cl-mha", i, pol, 128) for i in range(5)]
    theirs = [R.make_cache("xq-cl-mha", i, pol, 128) for i in range(5)]
    a_ours, a_theirs = R.Accumulator(), R.Accumulator()
    for i in range(5):
        ours[i].prefill(x, model.layers[i], a_ours)
        theirs[i].prefill(x, model.layers[i], a_theirs)
        k, v = ours[i].rematerialize(model.layers[i], np.arange(20), a_ours)
        rk, rv = theirs[i].rematerialize(model.layers[i], np.arange(20), a_theirs)
        assert rel_err(k, rk) <= KV_TOL and rel_err(v, rv) <= KV_TOL, (i, rel_err(k, rk))
    # every layer's codes are the reference's (deltas against a float64 accumulator row)
    for i in range(5):
        st = ours[i].backend.stream
        got = unpack_rows(st.codes[:20].cpu().numpy(), st.bits, model.config.hidden_dim)
        assert np.array_equal(got, theirs[i].stream.q.codes), i


# ---------------------------------------------------------------------------
# the INTEGRATION.md lane stub
# ---------------------------------------------------------------------------


@pytest.fixture
def cuda_lane(monkeypatch):
    """Bind the reference's kernel lane to the B200 one, as INTEGRATION.md section 1."""
    import xcache._kernels as lanes
    import xcache.quant as quant

    from paper_2508_10395_b200 import kernels as K

    for name in ("quantize_groups", "dequantize_groups", "pack_codes", "unpack_codes"):
        monkeypatch.setattr(lanes, name, getattr(K, name))
    monkeypatch.setattr(quant, "pack_codes", K.pack_codes)
    monkeypatch.setattr(quant, "unpack_codes", K.unpack_codes)
    return K


@pytest.mark.parametrize("variant,bits", [("xq-mha", 3), ("xq-cl-mha", 2), ("xq-gqa", 4),
                                          ("kvq", 3)])
def test_reference_session_bit_identical_on_cuda_lane(variant, bits, request):
    model = _model(gqa=variant == "xq-gqa")
    ref, _ = _session_logits(model, variant, bits)
    request.getfixturevalue("cuda_lane")
    got, _ = _session_logits(model, variant, bits)
    assert np.array_equal(got, ref), rel_err(got, ref)


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("cols", [17, 64, 130])
def test_lane_equivalence_quantize(bits, cols, cuda_lane):
    """tests/test_kernels.py:45-57 with the cuda lane in place of _native."""
    from xcache._kernels import fallback

    try:
        from xcache._kernels import _native
    except ImportError:
        _native = fallback
    K = cuda_lane
    rng = np.random.default_rng(bits * 100 + cols)
    x = rng.normal(size=(23, cols)) * rng.uniform(0.01, 100)
    for lane in (fallback, _native):
        cf, sf, zf = lane.quantize_groups(x, 32, bits)
        cn, sn, zn = K.quantize_groups(x, 32, bits)
        assert np.array_equal(cf, cn) and np.array_equal(sf, sn) and np.array_equal(zf, zn)
        assert np.array_equal(lane.dequantize_groups(cf, sf, zf, 32),
                              K.dequantize_groups(cf, sf, zf, 32))


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_lane_equivalence_pack(bits, cuda_lane):
    """tests/test_kernels.py:33-43 with the cuda lane."""
    from xcache._kernels import fallback

    K = cuda_lane
    codes = np.random.default_rng(bits).integers(0, 2**bits, 1001).astype(np.uint8)
    wf = fallback.pack_codes(codes, bits)
    assert np.array_equal(wf, K.pack_codes(codes, bits))
    assert np.array_equal(fallback.unpack_codes(wf, bits, 1001), K.unpack_codes(wf, bits, 1001))
    assert K.pack_codes(np.zeros(0, np.uint8), 3).size == 0
    x = np.full((2, 8), 5.0)  # the degenerate group (tests/test_kernels.py:78-83)
    c, s, z = K.quantize_groups(x, 8, 4)
    assert np.all(c == 0) and np.all(s == 1.0) and np.all(z == 5.0)
