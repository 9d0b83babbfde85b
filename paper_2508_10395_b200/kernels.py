"""GPU lane with the reference's kernel-lane API (xcache._kernels).

The reference selects one of two lanes at import (``_kernels/__init__.py:12-26``)
and re-exports ``quantize_groups``, ``dequantize_groups``, ``pack_codes`` and
``unpack_codes`` (plus the offline RNG / Jacobi helpers, out of scope here).
This module exports the same four hot-path functions with the same argument
meaning and results, computed by the sm_100a library:

* NumPy in -> NumPy out (inputs are staged through the GPU), so the
  reference's lane-equivalence tests (``tests/test_kernels.py:45-57``) run
  unchanged against this lane;
* torch CUDA tensors in -> torch CUDA tensors out (no host round trip).

Integer outputs and the float64 scales / zero points are bit-identical to the
reference lanes.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _as_cuda(a, dtype: torch.dtype, name: str, ndim: int):
    """Accept a NumPy array or torch tensor of exactly ``dtype`` (like the
    reference's typed Cython buffers, _native.pyx:111-121)."""
    if isinstance(a, np.ndarray):
        want = {torch.float64: np.float64, torch.uint8: np.uint8, torch.uint64: np.uint64}[dtype]
        if a.dtype != want:
            raise ValueError(f"Buffer dtype mismatch for {name}: expected {np.dtype(want)}, got {a.dtype}")
        if a.ndim != ndim:
            raise ValueError(f"Buffer has wrong number of dimensions for {name} (expected {ndim}, got {a.ndim})")
        t = torch.from_numpy(np.ascontiguousarray(a)).to(_dev())
        return t, True
    if not isinstance(a, torch.Tensor):
        raise TypeError(f"{name} must be a numpy array or torch tensor")
    if a.dtype != dtype or a.dim() != ndim:
        raise ValueError(f"{name}: expected {dtype} with {ndim} dims, got {a.dtype} {tuple(a.shape)}")
    if not a.is_cuda:
        return a.contiguous().to(_dev()), True
    return a.contiguous(), False


def _out(t: torch.Tensor, to_numpy: bool):
    return t.cpu().numpy() if to_numpy else t


def quantize_groups(x, group_size: int, bits: int):
    """Grouped asymmetric quantization per row (_native.pyx:111-153)."""
    xt, host = _as_cuda(x, torch.float64, "x", 2)
    rows, cols = xt.shape
    ng = -(-cols // group_size) if group_size >= 1 else 0
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=xt.device)
    scales = torch.empty((rows, ng), dtype=torch.float64, device=xt.device)
    zps = torch.empty((rows, ng), dtype=torch.float64, device=xt.device)
    N.call("xq_quantize_groups", N.ptr(xt), rows, cols, group_size, bits, N.ptr(codes),
           N.ptr(scales), N.ptr(zps), N.stream_of(xt.device))
    return _out(codes, host), _out(scales, host), _out(zps, host)


def dequantize_groups(codes, scales, zero_points, group_size: int):
    """``code * scale + zero_point`` in float64 (_native.pyx:156-177)."""
    ct, host = _as_cuda(codes, torch.uint8, "codes", 2)
    st, _ = _as_cuda(scales, torch.float64, "scales", 2)
    zt, _ = _as_cuda(zero_points, torch.float64, "zero_points", 2)
    rows, cols = ct.shape
    ng = -(-cols // group_size)
    if st.shape != (rows, ng) or zt.shape != (rows, ng):
        raise ValueError(f"scale grid {tuple(st.shape)} does not match codes {rows}x{cols}")
    out = torch.empty((rows, cols), dtype=torch.float64, device=ct.device)
    N.call("xq_dequantize_groups", N.ptr(ct), N.ptr(st), N.ptr(zt), rows, cols, group_size,
           N.ptr(out), N.stream_of(ct.device))
    return _out(out, host)


def pack_codes(codes, bits: int):
    """LSB-first little-endian uint64 bit stream (_native.pyx:64-85)."""
    ct, host = _as_cuda(codes, torch.uint8, "codes", 1)
    n = ct.shape[0]
    n_words = (n * bits + 63) // 64
    words = torch.zeros(n_words, dtype=torch.uint64, device=ct.device)
    if n:
        N.call("xq_pack_codes", N.ptr(ct), n, bits, N.ptr(words), N.stream_of(ct.device))
    return _out(words, host)


def unpack_codes(words, bits: int, n: int):
    """Inverse of :func:`pack_codes` (_native.pyx:88-108)."""
    wt, host = _as_cuda(words, torch.uint64, "words", 1)
    codes = torch.zeros(n, dtype=torch.uint8, device=wt.device)
    if n:
        if wt.shape[0] < (n * bits + 63) // 64:
            raise ValueError("not enough words for n codes")
        N.call("xq_unpack_codes", N.ptr(wt), bits, n, N.ptr(codes), N.stream_of(wt.device))
    return _out(codes, host)


def backend() -> str:
    """Name of the active lane (``_kernels/__init__.py:29-31``)."""
    return "cuda-sm100a"


def check_bits(bits: int) -> None:
    if bits not in (2, 3, 4, 8):
        raise ConfigError(f"bits must be one of (2, 3, 4, 8), got {bits}")
