"""Layered exploration on the GPU (drop-in for gridneighbors/explore.py).

Reference: pkg/src/gridneighbors/explore.py:21-137.  ``knn_query`` keeps
the reference signature, validation order and return type; the work is the
batched device kernel (csrc/ghn_query.cu) called through ``ghn_query``.
``knn_query_batch`` / ``predict_batch`` are the new batched entry points
 that return device tensors.
"""

from __future__ import annotations

import ctypes
import itertools
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import Neighbor
from .grid import CellId, GridIndex

STOP_MODES = ("heuristic", "guaranteed")
# Largest k the batched warp-resident top-k serves; larger k (any k <= n, as
# explore.py:86-88 allows) run the exact per-query path (csrc/ghn_largek.cu).
MAX_K = 256


@dataclass(frozen=True)
class QueryStats:
    """Work counters for one query (explore.py:24-34)."""

    layers_visited: int
    cells_visited: int
    points_scanned: int


def layer_cell_count(l: int, d: int) -> int:
    """Cells on layer l in d dims: (2l+1)^d - (2l-1)^d (explore.py:37-41)."""
    if l < 1 or d < 1:
        raise ValueError("require l >= 1 and d >= 1")
    return (2 * l + 1) ** d - (2 * l - 1) ** d


def total_cell_count(l: int, d: int) -> int:
    """Cells on layers 1..l: (2l+1)^d - 1 (explore.py:44-48)."""
    if l < 0 or d < 1:
        raise ValueError("require l >= 0 and d >= 1")
    return (2 * l + 1) ** d - 1


def layer_cells(center, l: int) -> set[CellId]:
    """Cell ids at Chebyshev distance exactly l (explore.py:51-63); geometry
    contract of the device shell enumerator."""
    if l < 0:
        raise ValueError("require l >= 0")
    center = tuple(int(c) for c in center)
    if l == 0:
        return {center}
    out = set()
    for offs in itertools.product(range(-l, l + 1), repeat=len(center)):
        if max(abs(o) for o in offs) == l:
            out.add(tuple(c + o for c, o in zip(center, offs)))
    return out


def _validate(index: GridIndex, Q, k: int, mode: str):
    if mode not in STOP_MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {STOP_MODES}")
    return _validate_queries(index, Q, k)


def _validate_queries(index: GridIndex, Q, k: int):
    import torch

    Qt = torch.as_tensor(Q)
    if Qt.dtype not in (torch.float32, torch.float64):
        Qt = Qt.to(torch.float64)
    if Qt.ndim != 2 or Qt.shape[1] != index.dim:
        raise ValueError(f"dimension mismatch: queries {tuple(Qt.shape)}, index {index.dim}")
    n = index.size
    if not 1 <= k <= n:
        raise ValueError(f"k={k} out of range [1, {n}]")
    return Qt


def _run(index: GridIndex, Qt, k, mode, task, want_neighbors, want_stats, want_totals=False,
         stream=None, qorder=None, want_confidence=True):
    """One ghn_query launch.  With an explicit ``stream`` every allocation,
    conversion and the launch happen on that stream (torch.cuda.stream), so
    the caching allocator ties the workspace and outputs to it."""
    import torch

    if stream is not None:
        with torch.cuda.stream(stream):
            return _run(index, Qt, k, mode, task, want_neighbors, want_stats, want_totals, None, qorder,
                        want_confidence)
    L = _lib.require_device()
    dev = index.X.device
    Qd = Qt.to(dev).contiguous()
    nq = int(Qd.shape[0])
    qdt = _lib.GHN_F32 if Qd.dtype == torch.float32 else _lib.GHN_F64
    res = {}
    out = _lib.QueryOut()
    if want_neighbors:
        res["dist"] = torch.empty((nq, k), dtype=torch.float64, device=dev)
        res["idx"] = torch.empty((nq, k), dtype=torch.int64, device=dev)
        out.dist, out.idx = _lib.ptr(res["dist"]), _lib.ptr(res["idx"])
    if want_stats:
        res["stats"] = torch.empty((nq, 3), dtype=torch.int64, device=dev)
        out.stats = _lib.ptr(res["stats"])
    if want_totals:
        res["totals"] = torch.zeros(5, dtype=torch.int64, device=dev)
        out.totals = _lib.ptr(res["totals"])
    if task == _lib.GHN_TASK_CLASSIFY:
        if index._labels.codes is None:
            raise ValueError("labels are not classifiable")
        res["label"] = torch.empty(nq, dtype=torch.int32, device=dev)
        out.label = _lib.ptr(res["label"])
        if want_confidence:
            res["confidence"] = torch.empty(nq, dtype=torch.float64, device=dev)
            out.confidence = _lib.ptr(res["confidence"])
    elif task in (_lib.GHN_TASK_REGRESS_MEAN, _lib.GHN_TASK_REGRESS_MEDIAN):
        if index._labels.targets is None:
            raise ValueError("labels are not numeric targets")
        res["value"] = torch.empty(nq, dtype=torch.float64, device=dev)
        out.value = _lib.ptr(res["value"])
    view = index.view(targets=task in (_lib.GHN_TASK_REGRESS_MEAN, _lib.GHN_TASK_REGRESS_MEDIAN))
    if qorder is not None:
        wsz, ws = 0, None
    else:
        wsz = int(L.ghn_query_workspace_size(ctypes.byref(view), nq, k))
        ws = torch.empty(wsz, dtype=torch.uint8, device=dev)
    _lib.check(L.ghn_query(ctypes.byref(view), _lib.ptr(Qd), qdt, nq, k, _lib.GHN_MODE[mode], task,
                           _lib.ptr(qorder), ctypes.byref(out), _lib.ptr(ws), wsz,
                           _lib.stream_handle(stream)), "ghn_query")
    res["_keepalive"] = (Qd, ws)
    return res


def knn_query_batch(index: GridIndex, Q, k: int, mode: str = "heuristic", stats: bool = True,
                    stream=None):
    """Batched knn_query: (dist (nq,k) f64, idx (nq,k) i64, stats (nq,3) i64 or None), on device."""
    Qt = _validate(index, Q, k, mode)
    r = _run(index, Qt, k, mode, _lib.GHN_TASK_NONE, True, stats, stream=stream)
    return r["dist"], r["idx"], r.get("stats")


def knn_query(index: GridIndex, q, k: int, mode: str = "heuristic"):
    """k nearest training points of q by layered exploration (explore.py:66-137)."""
    if mode not in STOP_MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {STOP_MODES}")
    qa = np.asarray(q, dtype=float)
    if qa.shape != (index.dim,):
        raise ValueError(f"dimension mismatch: query {qa.shape}, index {index.dim}")
    dist, idx, st = knn_query_batch(index, qa.reshape(1, -1), k, mode)
    dist = dist[0].cpu().tolist()
    idx = idx[0].cpu().tolist()
    st = st[0].cpu().tolist()
    labels = index.labels
    nbrs = [Neighbor(float(dv), int(i), labels[int(i)]) for dv, i in zip(dist, idx)]
    return nbrs, QueryStats(int(st[0]), int(st[1]), int(st[2]))


def query_order(index: GridIndex, Q, stream=None):
    """K8 query binning: device int32 visit order sorted by central cell
    (DENSE layout).  Results do not depend on the order; locality does."""
    import torch

    L = _lib.require_device()
    if stream is not None:
        with torch.cuda.stream(stream):
            return query_order(index, Q)
    Qd = torch.as_tensor(Q).to(index.X.device).contiguous()
    if Qd.dtype not in (torch.float32, torch.float64):
        Qd = Qd.to(torch.float64)
    nq = int(Qd.shape[0])
    qdt = _lib.GHN_F32 if Qd.dtype == torch.float32 else _lib.GHN_F64
    view = index.view(targets=False)
    wsz = int(L.ghn_query_workspace_size(ctypes.byref(view), nq, 1))
    ws = torch.empty(wsz, dtype=torch.uint8, device=Qd.device)
    order = torch.empty(nq, dtype=torch.int32, device=Qd.device)
    _lib.check(L.ghn_query_order(ctypes.byref(view), _lib.ptr(Qd), qdt, nq, _lib.ptr(order),
                                 _lib.ptr(ws), wsz, _lib.stream_handle(stream)), "ghn_query_order")
    return order
