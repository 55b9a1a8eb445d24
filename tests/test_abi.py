"""CPU-only checks of the C-ABI boundary: the library builds, loads, and exports
every entry point include/wt.h declares (no compute calls without a GPU)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "wt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*((?:w[tm]|hwt)_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_expected_calls():
    names = _declared()
    for req in ("wt_build", "wt_build_host", "wt_free", "wt_access", "wt_rank",
                "wm_build", "wm_free", "wm_access", "wm_rank",
                "hwt_build", "hwt_free", "hwt_access", "hwt_rank", "hwt_select", "wt_digit_counts", "wt_digits",
                "wt_partition", "wt_gather_bits", "wt_create", "wt_finish"):
        assert req in names


def test_library_exports_every_declared_symbol():
    from paper_1407_8142_b200 import _build
    path = _build.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), f"{name} not exported"
    lib.wt_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.wt_version()


def test_library_is_sm100a_only():
    import subprocess
    from paper_1407_8142_b200 import _build
    path = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_and_argument_errors_without_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_1407_8142_b200 import wt
    lib = wt._load()
    out = ctypes.POINTER(wt._WtTree)()
    assert lib.wt_build(None, 10, 1, 4, None, ctypes.byref(out)) == wt.WT_EINVAL
    mout = ctypes.POINTER(wt._WmMatrix)()
    assert lib.wm_build(None, 10, 1, 4, None, ctypes.byref(mout)) == wt.WT_EINVAL
    assert lib.wm_build(None, 0, 3, 4, None, ctypes.byref(mout)) == wt.WT_EINVAL
    assert lib.wm_free(None) == wt.WT_OK
    hl = wt._load_hwt()
    hout = ctypes.POINTER(wt._HwtTree)()
    assert hl.hwt_build(None, 10, 1, 4, None, ctypes.byref(hout)) == wt.WT_EINVAL
    assert hl.hwt_build(ctypes.c_void_p(16), 10, 4, 65537, None, ctypes.byref(hout)) == wt.WT_EINVAL
    assert hl.hwt_build(ctypes.c_void_p(16), 10, 5, 4, None, ctypes.byref(hout)) == wt.WT_EINVAL
    assert not hout
    assert hl.hwt_free(None) == wt.WT_OK
    assert hl.hwt_access(None, None, 0, None, None) == wt.WT_EINVAL
    assert lib.wt_build(ctypes.c_void_p(16), 10, 3, 4, None, ctypes.byref(out)) == wt.WT_EINVAL
    assert lib.wt_build(ctypes.c_void_p(16), 10, 1, 257, None, ctypes.byref(out)) == wt.WT_EINVAL
    assert lib.wt_build(ctypes.c_void_p(16), 10, 1, 0, None, ctypes.byref(out)) == wt.WT_EINVAL
    assert lib.wt_build(ctypes.c_void_p(16), 1 << 32, 1, 4, None, ctypes.byref(out)) == wt.WT_EINVAL
    assert not out
    assert lib.wt_free(None) == wt.WT_OK
    assert lib.wt_access(None, None, 0, None, None) == wt.WT_EINVAL


def test_oracle_not_imported_by_product():
    """The product package must not reference the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1407_8142_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f
