"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every entry point include/xquant.h declares (no compute calls)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "xquant.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xq_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for must in ("xq_quantize_groups", "xq_dequantize_groups", "xq_pack_codes",
                 "xq_unpack_codes", "xq_quantize_rows", "xq_decode_attend",
                 "xq_kv_decode_attend", "xq_cl_accumulate"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2508_10395_b200 import _native as N

    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(declared()) == sorted(N.EXPORTED)
    assert N.version().startswith("xquant-b200")


def test_sm100a_cubin_embedded():
    import subprocess

    from paper_2508_10395_b200 import _native as N

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_mapping():
    import pytest

    from paper_2508_10395_b200.errors import (ConfigError, DataError, ShapeError, UsageError,
                                              raise_for_status)

    for code, cls in ((1, ShapeError), (2, ConfigError), (3, UsageError), (4, DataError)):
        with pytest.raises(cls):
            raise_for_status(code, "x")
    raise_for_status(0, "x")
