"""The C-ABI library loads and exports every symbol include/ghn.h declares;
the ctypes struct layouts match the header (CPU only, no GPU calls)."""
import ctypes
import os
import re

import pytest

from paper_2004_02290_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ghn.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ghn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_exports_list():
    assert _declared() == sorted(_lib.EXPORTS)


@pytest.mark.skipif(not _lib.available(), reason="libghn.so not built")
def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(L, name), name


@pytest.mark.skipif(not _lib.available(), reason="libghn.so not built")
def test_abi_version_and_error_string():
    L = _lib.lib()
    assert L.ghn_abi_version() >= 100
    assert isinstance(L.ghn_last_error(), bytes)


@pytest.mark.skipif(not _lib.available(), reason="libghn.so not built")
def test_plan_init_host_only():
    """ghn_fit_plan_init is host-only: layout choice and workspace sizing."""
    import numpy as np

    L = _lib.lib()
    plan = _lib.FitPlan()
    widths = np.array([1 / 32, 1 / 32])
    bounds = np.array([0, 0, 31, 31], dtype=np.int64)
    rc = L.ghn_fit_plan_init(ctypes.byref(plan), 1000, 2, _lib.GHN_F32,
                             widths.ctypes.data_as(ctypes.c_void_p),
                             bounds.ctypes.data_as(ctypes.c_void_p), 1 << 20)
    assert rc == _lib.GHN_OK
    assert plan.layout == _lib.GHN_LAYOUT_DENSE and plan.E == 1024 and plan.key_bits == 10
    assert list(plan.ext[:2]) == [32, 32]
    rc = L.ghn_fit_plan_init(ctypes.byref(plan), 1000, 2, _lib.GHN_F32,
                             widths.ctypes.data_as(ctypes.c_void_p),
                             bounds.ctypes.data_as(ctypes.c_void_p), 100)
    assert rc == _lib.GHN_OK and plan.layout == _lib.GHN_LAYOUT_LIST
    bad = np.array([0, 0, -1, 5], dtype=np.int64)
    rc = L.ghn_fit_plan_init(ctypes.byref(plan), 1000, 2, _lib.GHN_F32,
                             widths.ctypes.data_as(ctypes.c_void_p),
                             bad.ctypes.data_as(ctypes.c_void_p), 1 << 20)
    assert rc == _lib.GHN_ERR_VALUE


def test_struct_layouts_match_header():
    # field order / sizes mirror include/ghn.h (x86-64 LP64)
    assert ctypes.sizeof(_lib.FitOut) == 9 * 8
    assert ctypes.sizeof(_lib.QueryOut) == 7 * 8
    assert _lib.IndexView.coords.offset == 8 + 4 * 4 + 8 + 16 * 8 + 8 + 16 * 8 * 2
    assert _lib.IndexView.density_hint.offset == 8 + 4 * 4 + 8 + 16 * 8 + 8 + 16 * 8 * 2 + 9 * 8 + 2 * 4
    assert ctypes.sizeof(_lib.IndexView) == 512
    assert ctypes.sizeof(_lib.FitPlan) == 8 + 4 * 4 + 8 + 16 * 8 * 3 + 8 * 3
