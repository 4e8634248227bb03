"""Max-splits cell-width fit on the device (grid.py:47-109).

Per dimension: the largest split count s whose s equal bins over
[min, max] are all occupied, checked (like grid.py:74-82) only against the
gaps wider than span/s.  Every arithmetic step is the reference's fp64
expression evaluated elementwise on the GPU:
    bin(v, s) = min(floor(((v - lo) * s) / span), s - 1)          grid.py:49
Candidate s values are checked in parallel batches from s_hi downward
instead of one at a time; the first (largest) passing s is the answer, the
same one the reference's descending loop returns.

Implementation note: this stage runs as PyTorch device tensor ops (sort /
unique / elementwise), not yet as a hand-written kernel; it is off the
build -> predict hot path (it only produces d widths).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib


def _max_splits_1d_device(v, cap):
    import torch

    u = torch.unique(v)                      # sorted distinct values (np.unique)
    m = int(u.numel())
    if m == 1:
        return 1, 1.0
    lo = float(u[0].item())
    span = float((u[-1] - u[0]).item())
    g = u[1:] - u[:-1]                       # np.diff
    max_gap = float(g.max().item())
    s_hi = min(m, int(math.ceil(2.0 * span / max_gap)))
    if cap is not None:
        s_hi = min(s_hi, cap)
    if s_hi < 2:
        return 1, span
    wide = torch.nonzero(g > span / s_hi).flatten()
    gg = g[wide]
    gl = u[wide]
    gr = u[wide + 1]
    W = int(gg.numel())
    if W == 0:
        return s_hi, span / s_hi
    dev = v.device
    batch = max(1, min(s_hi - 1, (1 << 24) // max(W, 1)))
    s = s_hi
    while s >= 2:
        s_lo = max(2, s - batch + 1)
        S = torch.arange(s, s_lo - 1, -1, device=dev, dtype=torch.float64)  # descending
        thr = span / S                                                       # span / s
        active = gg[None, :] > thr[:, None]
        lb = torch.minimum(torch.floor((gl[None, :] - lo) * S[:, None] / span), (S - 1)[:, None])
        rb = torch.minimum(torch.floor((gr[None, :] - lo) * S[:, None] / span), (S - 1)[:, None])
        bad = active & ((rb - lb) > 1)
        ok = ~bad.any(dim=1)
        hit = torch.nonzero(ok).flatten()
        if hit.numel():
            best = s - int(hit[0].item())
            return best, span / best
        s = s_lo - 1
    return 1, span


def fit_cell_measurements_arrays(X, max_splits=None):
    """GridParams from an (n, d) array / tensor (grid.py:94-109)."""
    import torch

    from .grid import GridParams

    _lib.require_device()
    Xt = torch.as_tensor(X)
    if Xt.ndim != 2 or Xt.shape[0] == 0:
        raise ValueError("empty dataset")
    Xd = Xt.to(device="cuda", dtype=torch.float64)
    if not bool(torch.isfinite(Xd).all()):
        raise ValueError("non-finite coordinate")
    d = int(Xd.shape[1])
    widths = np.empty(d)
    splits = np.empty(d, dtype=np.int64)
    for j in range(d):
        splits[j], widths[j] = _max_splits_1d_device(Xd[:, j].contiguous(), max_splits)
    origin = Xd.min(dim=0).values.cpu().numpy()
    return GridParams(widths=widths, origin=origin, splits=splits)


def fit_cell_measurements(data, max_splits=None):
    """Drop-in for grid.fit_cell_measurements(data, max_splits) (grid.py:94-109)."""
    from .grid import _coords_matrix

    return fit_cell_measurements_arrays(_coords_matrix(list(data)), max_splits)
