"""Max-splits cell-width fit (grid.py:47-109).

Per dimension, the largest split count s whose s equal bins over
[min, max] are all occupied, with the reference's fp64 bin expression
min(floor(((v - lo) * s) / span), s - 1) (grid.py:49).  The work runs in
csrc/ghn_fitwidths.cu (radix sort of the column, distinct values, gaps,
parallel check of candidate s from s_hi downward) through ``ghn_fit_widths``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def fit_cell_measurements_arrays(X, max_splits=None):
    """GridParams from an (n, d) array / tensor (grid.py:94-109)."""
    import torch

    from .grid import GridParams

    L = _lib.require_device()
    Xt = torch.as_tensor(X)
    if Xt.ndim != 2 or Xt.shape[0] == 0:
        raise ValueError("empty dataset")
    if Xt.dtype not in (torch.float32, torch.float64):
        Xt = Xt.to(torch.float64)
    Xd = Xt.to("cuda").contiguous()
    if not bool(torch.isfinite(Xd).all()):
        raise ValueError("non-finite coordinate")
    n, d = int(Xd.shape[0]), int(Xd.shape[1])
    dtype = _lib.GHN_F32 if Xd.dtype == torch.float32 else _lib.GHN_F64
    widths = np.empty(d, np.float64)
    splits = np.empty(d, np.int64)
    origin = np.empty(d, np.float64)
    wsz = int(L.ghn_fit_widths_workspace_size(n))
    ws = torch.empty(wsz, dtype=torch.uint8, device=Xd.device)
    P = ctypes.c_void_p
    _lib.check(L.ghn_fit_widths(_lib.ptr(Xd), dtype, n, d, -1 if max_splits is None else int(max_splits),
                                widths.ctypes.data_as(P), splits.ctypes.data_as(P), origin.ctypes.data_as(P),
                                _lib.ptr(ws), wsz, _lib.stream_handle()), "ghn_fit_widths")
    return GridParams(widths=widths, origin=origin, splits=splits)


def fit_cell_measurements(data, max_splits=None):
    """Drop-in for grid.fit_cell_measurements(data, max_splits) (grid.py:94-109)."""
    from .grid import _coords_matrix

    return fit_cell_measurements_arrays(_coords_matrix(list(data)), max_splits)
