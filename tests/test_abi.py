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
    assert _lib.IndexView.n_sub.offset == 512
    assert ctypes.sizeof(_lib.IndexView) == 512 + 8 + 5 * 8 + 8
    assert ctypes.sizeof(_lib.SubGrid) == 16 * 8 * 3 + 16 * 4 + 8 + 4 * 4
    assert ctypes.sizeof(_lib.FitPlan) == 8 + 4 * 4 + 8 + 16 * 8 * 3 + 8 * 3


@pytest.mark.skipif(__import__("shutil").which("gcc") is None, reason="gcc not available")
def test_struct_layouts_match_compiled_header(tmp_path):
    """offsetof / sizeof of every ABI struct, compiled from include/ghn.h,
    equal the ctypes mirror in _lib.py."""
    import subprocess

    structs = {"ghn_fit_plan": _lib.FitPlan, "ghn_fit_out": _lib.FitOut, "ghn_index_view": _lib.IndexView,
               "ghn_query_out": _lib.QueryOut, "ghn_subgrid": _lib.SubGrid}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ghn.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, val = line.split()
        py = structs[cname]
        got = ctypes.sizeof(py) if field == "size" else getattr(py, field).offset
        assert got == int(val), (cname, field, got, val)
