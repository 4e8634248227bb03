"""Exact baselines on the device (mirror of gridneighbors/baselines.py).

Reference: pkg/src/gridneighbors/baselines.py:1-146.  Both reference
baselines -- the brute-force scan (:40-55) and the kd-tree (:66-146) --
return exactly the k nearest points under (key, point index) order; they are
`run_bench`'s recall oracle and its comparison rows (bench.py:160-161, 176-182).

On the B200 both are served by ONE exact kernel: ``ghn_query`` in mode
``GHN_MODE_BRUTE`` (csrc/ghn_query.cu) scans every training point per query
with the same fp64 numpy-order keys and warp top-k as the grid walk.  A
pointer-chasing kd-tree has no advantage over a bandwidth-bound full scan on
this part at run_bench sizes, so ``kdtree_build`` / ``kdtree_knn`` keep the
reference names, arguments and validation (leaf_size >= 1) and return the
identical exact neighbours through the same kernel.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from . import _lib
from .core import LabeledPoint, Neighbor, check_metric
from .grid import GridIndex, GridParams, _coords_matrix, build_arrays


class BruteIndex:
    """Device copy of a training set for exact search (baselines.py:26-34)."""

    def __init__(self, X, labels, metric: str = "euclidean"):
        check_metric(metric)
        import torch

        Xt = torch.as_tensor(X)
        if Xt.ndim != 2 or Xt.shape[0] == 0:
            raise ValueError("empty dataset")
        d = int(Xt.shape[1])
        # one coarse cell per sign pattern: the scan ignores the grid, the
        # table only has to exist
        self.grid: GridIndex = build_arrays(
            Xt, labels, params=GridParams(np.full(d, 2.0 ** 1000), np.zeros(d), np.ones(d, np.int64)),
            metric=metric)
        self.metric = metric

    @property
    def size(self) -> int:
        return self.grid.size

    @property
    def coords(self) -> np.ndarray:
        return self.grid.coords

    @property
    def labels(self):
        return self.grid.labels


def brute_build(data: Sequence[LabeledPoint], metric: str = "euclidean") -> BruteIndex:
    """baselines.py:37-39."""
    check_metric(metric)
    data = list(data)
    return BruteIndex(_coords_matrix(data), [p.label for p in data], metric)


def brute_knn_batch(index: BruteIndex, Q, k: int, stream=None):
    """Exact k nearest of every query row: (dist (nq,k) f64, idx (nq,k) i64) on device."""
    from .explore import _run, _validate_queries

    Qt = _validate_queries(index.grid, Q, k)
    r = _run(index.grid, Qt, k, "brute", _lib.GHN_TASK_NONE, True, False, stream=stream)
    return r["dist"], r["idx"]


def brute_knn(index: BruteIndex, q, k: int) -> list[Neighbor]:
    """Exact k nearest by full scan, sorted by (distance, index) (baselines.py:40-55)."""
    qa = np.asarray(q, dtype=float)
    if qa.shape != (index.grid.dim,):
        raise ValueError("dimension mismatch")
    if not 1 <= k <= index.size:
        raise ValueError(f"k={k} out of range [1, {index.size}]")
    dist, idx = brute_knn_batch(index, qa.reshape(1, -1), k)
    labels = index.labels
    return [Neighbor(float(dv), int(i), labels[int(i)])
            for dv, i in zip(dist[0].cpu().tolist(), idx[0].cpu().tolist())]


class KdTree(BruteIndex):
    """Exact-search index under the reference's kd-tree name (baselines.py:66-113);
    queries run the device exact scan (see the module docstring)."""

    def __init__(self, data: Sequence[LabeledPoint], metric: str = "euclidean", leaf_size: int = 16):
        check_metric(metric)
        if leaf_size < 1:
            raise ValueError("leaf_size must be >= 1")
        data = list(data)
        super().__init__(_coords_matrix(data), [p.label for p in data], metric)
        self.leaf_size = leaf_size


def kdtree_build(data: Sequence[LabeledPoint], metric: str = "euclidean", leaf_size: int = 16) -> KdTree:
    """baselines.py:116-117."""
    return KdTree(data, metric, leaf_size)


def kdtree_knn(tree: KdTree, q, k: int) -> list[Neighbor]:
    """Exact k nearest, equal to brute_knn (baselines.py:120-146)."""
    return brute_knn(tree, q, k)
