"""C-ABI library: builds, loads and exports every symbol include/srk.h declares (CPU-only)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "srk.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srk_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_binding_table():
    from paper_1810_10197_b200 import _native

    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    from paper_1810_10197_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libsrk.so not built (run __graft_entry__.build())")
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.srk_abi_version() == 1


def test_library_is_sm100a():
    from paper_1810_10197_b200 import _native
    import subprocess

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libsrk.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_errors_map_to_value_error():
    from paper_1810_10197_b200 import _native
    import ctypes

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libsrk.so not built")
    lib = _native.load()
    h = ctypes.c_void_p()
    shape = (ctypes.c_int64 * 3)(7, 8, 8)
    lengths = (ctypes.c_double * 3)(1.0, 1.0, 1.0)
    rc = lib.srk_plan_create(ctypes.byref(h), 3, shape, lengths, 0, 0)
    assert rc == _native.SRK_ERR_INVALID
    with pytest.raises(ValueError, match="even"):
        _native.check(rc)
