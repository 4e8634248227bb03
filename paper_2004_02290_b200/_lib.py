"""ctypes binding of libghn.so (include/ghn.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every device entry point raises RuntimeError.  Struct layouts here
mirror include/ghn.h field for field.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libghn.so")

GHN_MAX_DIM = 16
GHN_F32, GHN_F64 = 0, 1
GHN_LAYOUT_DENSE, GHN_LAYOUT_LIST = 0, 1
GHN_MODE = {"heuristic": 0, "guaranteed": 1, "brute": 2}
GHN_TASK_NONE, GHN_TASK_CLASSIFY, GHN_TASK_REGRESS_MEAN, GHN_TASK_REGRESS_MEDIAN = 0, 1, 2, 3
GHN_METRIC = {"euclidean": 0, "manhattan": 1, "chebyshev": 2}
GHN_OK, GHN_ERR_VALUE, GHN_ERR_CUDA, GHN_ERR_UNSUPPORTED = 0, 1, 2, 3

# Every symbol include/ghn.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ghn_last_error",
    "ghn_abi_version",
    "ghn_build_flags",
    "ghn_fit_bounds",
    "ghn_fit_plan_init",
    "ghn_fit_build",
    "ghn_fit_widths_workspace_size",
    "ghn_fit_widths",
    "ghn_query_workspace_size",
    "ghn_query_order",
    "ghn_query",
    "ghn_gather_i32",
    "ghn_window_density",
    "ghn_launch_count",
    "ghn_subgrid_select",
    "ghn_subgrid_bounds",
    "ghn_subgrid_workspace_size",
    "ghn_subgrid_build",
)

_i64, _i32, _f64, _p, _sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t


class FitPlan(ctypes.Structure):
    _fields_ = [
        ("n", _i64), ("d", _i32), ("dtype", _i32), ("layout", _i32), ("key_bits", _i32),
        ("E", _i64),
        ("widths", _f64 * GHN_MAX_DIM),
        ("lo", _i64 * GHN_MAX_DIM),
        ("ext", _i64 * GHN_MAX_DIM),
        ("workspace_bytes", _sz),
        ("fast_cursor_off", _sz),
        ("fast_rec_off", _sz),
    ]


class FitOut(ctypes.Structure):
    _fields_ = [
        ("perm", _p), ("coords", _p), ("cell_start", _p), ("cell_ids", _p), ("n_cells", _p),
        ("pt_off", _p), ("ne_off", _p), ("labels_in", _p), ("labels_perm", _p),
    ]


class IndexView(ctypes.Structure):
    _fields_ = [
        ("n", _i64), ("d", _i32), ("dtype", _i32), ("layout", _i32), ("n_cells", _i32),
        ("E", _i64),
        ("widths", _f64 * GHN_MAX_DIM),
        ("min_width", _f64),
        ("lo", _i64 * GHN_MAX_DIM),
        ("ext", _i64 * GHN_MAX_DIM),
        ("coords", _p), ("perm", _p), ("cell_start", _p), ("cell_ids", _p),
        ("pt_off", _p), ("ne_off", _p), ("labels", _p), ("targets", _p), ("labels_perm", _p),
        ("n_labels", _i32), ("metric", _i32),
        ("density_hint", _f64),
        ("n_sub", _i32), ("sub_min", _i32),
        ("sub_of_cell", _p), ("subs", _p), ("sub_off", _p), ("sub_coords", _p), ("sub_idx", _p),
        ("n_subpts", _i64),
    ]


class SubGrid(ctypes.Structure):
    """ghn_subgrid (include/ghn.h): nested grid of one overfull cell."""
    _fields_ = [
        ("origin", _f64 * GHN_MAX_DIM), ("h", _f64 * GHN_MAX_DIM), ("inv_h", _f64 * GHN_MAX_DIM),
        ("ext", _i32 * GHN_MAX_DIM), ("off", _i64), ("cell", _i32), ("start", _i32), ("count", _i32),
        ("pad", _i32),
    ]


class QueryOut(ctypes.Structure):
    _fields_ = [
        ("dist", _p), ("idx", _p), ("label", _p), ("confidence", _p), ("value", _p),
        ("stats", _p), ("totals", _p),
    ]


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    """Load libghn.so; raise RuntimeError (never fall back) if it cannot be used."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    L.ghn_last_error.restype = ctypes.c_char_p
    L.ghn_abi_version.restype = _i32
    L.ghn_build_flags.restype = _i32
    L.ghn_fit_bounds.argtypes = [_p, _i32, _i64, _i32, _p, _p, _p, _p, _p]
    L.ghn_fit_bounds.restype = _i32
    L.ghn_fit_plan_init.argtypes = [ctypes.POINTER(FitPlan), _i64, _i32, _i32, _p, _p, _i64]
    L.ghn_fit_plan_init.restype = _i32
    L.ghn_fit_build.argtypes = [ctypes.POINTER(FitPlan), _p, ctypes.POINTER(FitOut), _p, _sz, _p]
    L.ghn_fit_build.restype = _i32
    L.ghn_fit_widths_workspace_size.argtypes = [_i64]
    L.ghn_fit_widths_workspace_size.restype = _sz
    L.ghn_fit_widths.argtypes = [_p, _i32, _i64, _i32, _i64, _p, _p, _p, _p, _sz, _p]
    L.ghn_fit_widths.restype = _i32
    L.ghn_query_workspace_size.argtypes = [ctypes.POINTER(IndexView), _i64, _i32]
    L.ghn_query_workspace_size.restype = _sz
    L.ghn_query.argtypes = [ctypes.POINTER(IndexView), _p, _i32, _i64, _i32, _i32, _i32, _p,
                            ctypes.POINTER(QueryOut), _p, _sz, _p]
    L.ghn_query.restype = _i32
    L.ghn_query_order.argtypes = [ctypes.POINTER(IndexView), _p, _i32, _i64, _p, _p, _sz, _p]
    L.ghn_query_order.restype = _i32
    L.ghn_launch_count.restype = ctypes.c_uint64
    L.ghn_gather_i32.argtypes = [_p, _p, _i64, _p, _p]
    L.ghn_gather_i32.restype = _i32
    L.ghn_window_density.argtypes = [_p, _i32, _i32, _p, _p]
    L.ghn_window_density.restype = _i32
    L.ghn_subgrid_select.argtypes = [ctypes.POINTER(IndexView), _i32, _p, _p, _p]
    L.ghn_subgrid_select.restype = _i32
    L.ghn_subgrid_bounds.argtypes = [ctypes.POINTER(IndexView), _p, _i32, _p, _p, _p]
    L.ghn_subgrid_bounds.restype = _i32
    L.ghn_subgrid_workspace_size.argtypes = [_i64]
    L.ghn_subgrid_workspace_size.restype = _sz
    L.ghn_subgrid_build.argtypes = [ctypes.POINTER(IndexView), _p, _i32, _i64, _p, _p, _p, _i64, _p, _p, _sz, _p]
    L.ghn_subgrid_build.restype = _i32
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    """Map a ghn status to the reference's exception convention."""
    if rc == GHN_OK:
        return
    msg = lib().ghn_last_error().decode(errors="replace")
    if rc == GHN_ERR_VALUE:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (rc={rc}): {msg}")


def require_device():
    """The CUDA path or nothing: raise if no GPU or no library."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2004_02290_b200 requires a CUDA device (B200); no CPU fallback")
    return lib()


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def tuning_build() -> bool:
    """True when the library reads the GHN_* measurement knobs (tuning build)."""
    return bool(lib().ghn_build_flags() & 1)
