"""ctypes binding of the C-ABI library ``libxquant.so`` (include/xquant.h).

There is no CPU fallback: if the library is missing, importing this module
raises, and every product-path call goes through :func:`call`, which maps
non-zero status codes onto the reference's exception classes.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import raise_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
# XQ_LIB selects an alternative build (e.g. the role-profiling library of
# tools/build_role_profile.sh); the default is the in-tree libxquant.so
LIB_PATH = os.environ.get("XQ_LIB") or os.path.join(_PKG, "libxquant.so")

F32, BF16, F16, F64 = 0, 1, 2, 3
A_CODES_TOKEN, A_CODES_CHANNEL, A_F16_ROWS, A_SAME, A_F16_ACC = 0, 1, 2, 3, 4

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_F = C.c_float
_D = C.c_double

_SIGS = {
    "xq_quantize_groups": [_P, _I64, _I64, _I32, _I32, _P, _P, _P, _P],
    "xq_dequantize_groups": [_P, _P, _P, _I64, _I64, _I32, _P, _P],
    "xq_pack_codes": [_P, _I64, _I32, _P, _P],
    "xq_unpack_codes": [_P, _I32, _I64, _P, _P],
    "xq_quantize_rows": [_P, _I32, _I64, _I64, _I64, _I32, _I32, _P, _I64, _I64, _P, _P, _I64,
                         _P, _P, _P, _P],
    "xq_quantize_rows_cl": [_P, _I32, _I64, _I64, _I64, _I32, _I32, _P, _I64, _I64, _P, _I32, _P,
                            _I64, _P, _P, _P],
    "xq_latent_project_append": [_P, _I64, _I32, _I64, _P, _I32, _I32, _I32, _P, _P, _I64, _P,
                                 _P, _I64, _P, _P, _P, _P],
    "xq_dequant_rows_f16": [_P, _I64, _P, _I32, _I32, _I32, _I64, _I64, _I64, _P, _I64, _P, _I64,
                            _P],
    "xq_gemm_f16": [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _I32, _P, _I64, _I64, _P],
    "xq_prefill_attend": [_P, _P, _P, _I32, _I32, _I32, _I32, _I64, _I64, _F, _P, _I64, _P],
    "xq_rope_rows": [_P, _I32, _I64, _I64, _I64, _P, _I64, _I64, _P, _I32, _I64, _P],
    "xq_quantize_blocks_per_channel_f64_recon": [_P, _I64, _I64, _I32, _I32, _P, _P, _I64, _P,
                                                 _P, _P, _P],
    "xq_clgqa_latent64": [_P, _I32, _I64, _I32, _I64, _P, _P, _I32, _I64, _P, _P, _I32, _P, _P,
                          _P, _P],
    "xq_clgqa_row_update": [_P, _P, _I32, _I32, _P, _I32, _I64, _I64, _I32, _P, _P],
    "xq_quantize_blocks_per_channel": [_P, _I64, _I64, _I32, _I32, _P, _P, _I64, _P, _P, _P],
    "xq_quantize_blocks_per_channel_f64": [_P, _I64, _I64, _I32, _I32, _P, _P, _I64, _P, _P, _P],
    "xq_dequant_rows": [_P, _I64, _P, _I32, _I32, _I32, _I64, _I64, _I64, _P, _P],
    "xq_rope_table": [_P, _I64, _I32, _D, _I32, _P],
    "xq_arrange_weights": [_P, _P, _I32, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P],
    "xq_decode_attend": [_I32, _P, _P, _P, _P, _I32, _I64, _I32, _P, _P, _I32, _I64, _I32, _I64,
                         _I64, _P, _I32, _I32, _P, _I32, _I32, _P, _P, _I64, _F, _I32, _P, _I64,
                         _P, _P],
    "xq_arrange_weights_absorbed": [_P, _P, _I32, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P, _P],
    "xq_decode_attend_absorbed": [_I32, _P, _P, _P, _P, _P, _I32, _I64, _I32, _P, _P, _I32, _I64, _I32,
                                  _I64, _I64, _P, _I32, _I32, _P, _P, _I32, _I32, _P, _P, _I64, _F,
                                  _P, _I64, _P, _P],
    "xq_decode_attend_absorbed_peers": [_I32, _P, _P, _P, _P, _P, _I32, _I64, _I32, _P, _P, _I32,
                                        _I64, _I32, _I64, _I64, _P, _I32, _I32, _P, _P, _I32,
                                        _I32, _P, _P, _I64, _F, _P, _I64, _P, _I32, _P],
    "xq_decode_attend_absorbed_cl": [_P, _P, _P, _I32, _I64, _I32, _I64, _I64, _P, _I32, _I32, _P,
                                     _P, _I32, _P, _P, _I64, _F, _P, _I64, _P, _P],
    "xq_remat_f32": [_I32, _P, _P, _P, _I32, _I32, _I64, _I32, _P, _P, _I32, _I64, _I32, _I64,
                     _I64, _I32, _I32, _P, _P, _I64, _P, _P, _P, _P],
    "xq_cl_accumulate": [_I32, _P, _I64, _P, _I32, _I32, _I64, _P, _I32, _I32, _I64, _P, _P,
                         _P],
    "xq_debug_set_acc_dump": [_P, _I32],
    "xq_debug_role_profile": [_P, _I32],
    "xq_kv_append": [_P, _P, _P, _I32, _I32, _I64, _P, _P, _P, _P],
    "xq_kvq_decode_attend": [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I64, _I64, _P, _I32,
                             _I32, _I32, _I32, _P, _P, _F, _I32, _P, _I64, _P, _P],
    "xq_kv_decode_attend": [_P, _P, _I64, _P, _I32, _I32, _I32, _I32, _P, _P, _F, _I32, _P,
                            _I64, _P, _P],
}
_I64_RET = {"xq_decode_workspace_bytes": [_I32, _I32, _I32, _I32, _I32],
            "xq_kv_decode_workspace_bytes": [_I32, _I32, _I32, _I32, _I32],
            "xq_absorbed_workspace_bytes": [_I32, _I32, _I32, _I64],
            "xq_kvq_workspace_bytes": [_I32, _I32, _I32, _I32]}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the sm_100a CUDA extension is not built "
            "(run `python -m paper_2508_10395_b200._build`); there is no CPU fallback"
        )
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, args in _I64_RET.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int64
    lib.xq_version.restype = C.c_char_p
    lib.xq_last_error.restype = C.c_char_p
    return lib


lib = _load()

EXPORTED = sorted(list(_SIGS) + list(_I64_RET) + ["xq_version", "xq_last_error"])


def call(name: str, *args) -> None:
    """Invoke ``name`` and raise the mapped exception on a non-zero status."""
    status = getattr(lib, name)(*args)
    if status:
        raise_for_status(status, name, lib.xq_last_error().decode(errors="replace"))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_of(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def version() -> str:
    return lib.xq_version().decode()
