"""The GPU lane must satisfy the reference's own lane-equivalence contract
(reference tests/test_kernels.py:33-84, test_quant.py:131-143): quantize /
dequantize / pack / unpack bit-identical to the reference lanes, checked on
the reference's golden vectors and against the oracle on seeded inputs."""

import numpy as np
import pytest

from _util import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2508_10395_b200 import kernels

    return kernels


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("cols", [17, 64, 130, 256])
@pytest.mark.parametrize("gs", [32, 128])
def test_quantize_groups_matches_reference(K, bits, cols, gs):
    z = golden("quant")
    k = f"b{bits}_c{cols}_g{gs}"
    x = z[k + "_x"].astype(np.float64)
    c, s, zp = K.quantize_groups(x, gs, bits)
    assert np.array_equal(c, z[k + "_codes"])
    assert np.array_equal(s, z[k + "_scales"])
    assert np.array_equal(zp, z[k + "_zps"])
    deq = K.dequantize_groups(c, s, zp, gs)
    assert np.array_equal(deq.astype(np.float32), z[k + "_deq"])


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_d4096_bf16_rows(K, bits):
    # fp32 arithmetic would miss ~1e-4 of the codes here; the lane is float64.
    from _util import bf16f

    z = golden("quant")
    x = bf16f(z[f"d4096_b{bits}_xbf16"])
    c, s, zp = K.quantize_groups(x, 128, bits)
    assert np.array_equal(c, z[f"d4096_b{bits}_codes"])
    assert np.array_equal(s, z[f"d4096_b{bits}_scales"])


def test_large_random_against_oracle(K):
    import xq_oracle as O

    rng = np.random.default_rng(7)
    for bits in (2, 3, 4, 8):
        x = rng.normal(size=(512, 1000)) * rng.uniform(0.01, 50)
        c, s, zp = K.quantize_groups(x, 128, bits)
        co, so, zo = O.quantize_groups(x, 128, bits)
        assert np.array_equal(c, co) and np.array_equal(s, so) and np.array_equal(zp, zo)


def test_degenerate_group(K):
    # reference tests/test_kernels.py:79-84
    x = np.full((2, 8), 5.0)
    codes, scales, zps = K.quantize_groups(x, 8, 4)
    assert np.all(codes == 0) and np.all(scales == 1.0) and np.all(zps == 5.0)


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_pack_unpack_golden(K, bits):
    z = golden("pack")
    for n in list(range(0, 65)) + [127, 128, 129, 1000, 4096]:
        codes = z[f"b{bits}_n{n}_codes"]
        words = K.pack_codes(codes, bits)
        assert np.array_equal(words, z[f"b{bits}_n{n}_words"]), n
        assert np.array_equal(K.unpack_codes(words, bits, n), codes), n


def test_xqt1_known_answer(K):
    # reference tests/test_quant.py:210-223: codes 0,1,2,3 at 2 bits -> 0b11100100
    words = K.pack_codes(np.array([0, 1, 2, 3], np.uint8), 2)
    assert int(words[0]) == 0b11100100


def test_dtype_mismatch_raises(K):
    with pytest.raises(ValueError):
        K.quantize_groups(np.ones((2, 4), np.float32), 4, 4)


def test_bad_bits_is_config_error(K):
    from paper_2508_10395_b200.errors import ConfigError

    with pytest.raises(ConfigError):
        K.quantize_groups(np.ones((2, 4)), 4, 5)


def test_torch_in_torch_out(K):
    import torch

    x = torch.randn(16, 256, dtype=torch.float64, device="cuda")
    c, s, zp = K.quantize_groups(x, 128, 3)
    assert c.is_cuda and c.dtype == torch.uint8 and s.shape == (16, 2)
