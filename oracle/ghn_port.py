"""numpy restatement of the reference GHN path -- TEST INFRASTRUCTURE ONLY.

This is the "port" arm: the reference's own algorithm (gridneighbors,
/root/reference/pkg/src/gridneighbors) restated over plain arrays instead of
LabeledPoint objects, keeping its per-query complexity (an O(#cells)
Chebyshev scan per query and per layer).  bench.py times it as the CPU
baseline / reference arm; tests use it to cross-check the C oracle.  Nothing
on the product path imports this module.

Reference lines restated:
  fit widths (max-splits)   grid.py:47-109
  hash                      grid.py:112-125
  build (lexsort grouping)  grid.py:165-195
  knn_query                 explore.py:66-137
  ordering keys             core.py:72-91
  classify / regress        predict.py:20-50
"""

from __future__ import annotations

import math
from collections import Counter

import numpy as np

STOP_MODES = ("heuristic", "guaranteed")


# ----------------------------------------------------------------- fit widths
def _bins(v, lo, span, s):
    # grid.py:47-49: closed right edge, fp64 ((v - lo) * s) / span
    return np.minimum(np.floor((v - lo) * s / span), s - 1)


def max_splits_1d(values, cap=None):
    """Largest s whose s equal bins over [min, max] are all occupied (grid.py:52-82)."""
    u = np.unique(np.asarray(values, dtype=np.float64))
    if u.size == 1:
        return 1, 1.0
    lo = float(u[0])
    span = float(u[-1] - u[0])
    g = np.diff(u)
    s_top = min(u.size, int(math.ceil(2.0 * span / float(g.max()))))
    if cap is not None:
        s_top = min(s_top, cap)
    g_sorted = np.sort(g)
    desc = np.argsort(g, kind="stable")[::-1]
    left, right = u[:-1][desc], u[1:][desc]
    for s in range(s_top, 1, -1):
        # gaps wider than span/s are the only places a bin can be skipped
        wide = g.size - int(np.searchsorted(g_sorted, span / s, side="right"))
        if wide == 0:
            return s, span / s
        jump = _bins(right[:wide], lo, span, s) - _bins(left[:wide], lo, span, s)
        if jump.max() <= 1:
            return s, span / s
    return 1, span


def fit_widths(X, max_splits=None):
    """(widths, origin, splits) like fit_cell_measurements (grid.py:94-109)."""
    X = np.asarray(X, dtype=np.float64)
    d = X.shape[1]
    widths = np.empty(d)
    splits = np.empty(d, dtype=np.int64)
    for j in range(d):
        splits[j], widths[j] = max_splits_1d(X[:, j], max_splits)
    return widths, X.min(axis=0), splits


# ---------------------------------------------------------------------- build
def cell_ids(X, widths):
    """floor(x / w) as int64 (grid.py:124-125)."""
    return np.floor(np.asarray(X, dtype=np.float64) / np.asarray(widths, dtype=np.float64)).astype(np.int64)


class PortIndex:
    """Array form of GridIndex (grid.py:128-162): order/starts instead of bucket lists."""

    def __init__(self, X, labels, widths, metric="euclidean"):
        self.metric = metric
        X = np.asarray(X, dtype=np.float64)
        if X.ndim != 2 or X.shape[0] == 0:
            raise ValueError("X must be a non-empty (n, d) matrix")
        if not np.all(np.isfinite(X)):
            raise ValueError("non-finite coordinate")
        self.X = X
        self.labels = np.asarray(labels)
        self.widths = np.asarray(widths, dtype=np.float64)
        n, d = X.shape
        ids = cell_ids(X, self.widths)
        # stable grouping by lexicographic cell id, dim 0 most significant
        sort_keys = [np.arange(n)] + [ids[:, j] for j in reversed(range(d))]
        self.order = np.lexsort(sort_keys)
        sid = ids[self.order]
        fresh = np.ones(n, dtype=bool)
        fresh[1:] = np.any(sid[1:] != sid[:-1], axis=1)
        self.starts = np.flatnonzero(fresh)
        self.cell_array = sid[self.starts]
        self.ends = np.append(self.starts[1:], n)

    @classmethod
    def from_arrays(cls, X, labels, widths, order, starts, cell_array):
        """Assemble from (order, starts, cell_array) produced elsewhere -- the C
        restatement, whose arrays tests/test_oracle.py pins equal to this
        class's lexsort build.  Lets bench.py time knn() at 100M points without
        a 200 s lexsort."""
        self = cls.__new__(cls)
        self.metric = "euclidean"
        self.X = np.asarray(X, dtype=np.float64)
        self.labels = np.asarray(labels)
        self.widths = np.asarray(widths, dtype=np.float64)
        self.order = np.asarray(order, dtype=np.int64)
        st = np.asarray(starts, dtype=np.int64)
        self.starts = st[:-1]
        self.ends = st[1:]
        self.cell_array = np.asarray(cell_array, dtype=np.int64)
        return self

    @property
    def size(self):
        return self.X.shape[0]

    @property
    def dim(self):
        return self.X.shape[1]

    def bucket(self, c):
        return self.order[self.starts[c]:self.ends[c]]


def build(X, labels, widths, metric="euclidean"):
    return PortIndex(X, labels, widths, metric)


# ---------------------------------------------------------------------- query
def ordering_keys(q, pts, metric="euclidean"):
    """Per-row keys (core.py:72-86): squared L2 in einsum order, L1, L-inf."""
    diff = pts - q
    if metric == "euclidean":
        return np.einsum("ij,ij->i", diff, diff)
    if metric == "manhattan":
        return np.abs(diff).sum(axis=1)
    return np.abs(diff).max(axis=1)


def knn(index: PortIndex, q, k, mode="heuristic"):
    """Layered exploration (explore.py:81-137).  Returns (keys, idx, (layers, cells, points))."""
    if mode not in STOP_MODES:
        raise ValueError(f"unknown mode {mode!r}")
    q = np.asarray(q, dtype=np.float64)
    if q.shape != (index.dim,):
        raise ValueError("dimension mismatch")
    if not 1 <= k <= index.size:
        raise ValueError("k out of range")
    centre = np.floor(q / index.widths).astype(np.int64)
    ring = np.abs(index.cell_array - centre).max(axis=1)
    last = int(ring.max())
    wmin = float(index.widths.min())
    keys = np.empty(0)
    idx = np.empty(0, dtype=np.int64)
    n_cells = n_pts = 0
    layer = 0
    while True:
        hit = np.flatnonzero(ring == layer)
        moved = False
        if hit.size:
            cand = np.concatenate([index.bucket(c) for c in hit])
            ck = ordering_keys(q, index.X[cand], index.metric)
            n_cells += hit.size
            n_pts += cand.size
            mk = np.concatenate([keys, ck])
            mi = np.concatenate([idx, cand])
            sel = np.lexsort((mi, mk))[:k]
            moved = sel.size != idx.size or not np.array_equal(mi[sel], idx)
            keys, idx = mk[sel], mi[sel]
        if idx.size == k:
            if mode == "heuristic" and not moved:
                break
            if mode == "guaranteed":
                b = layer * wmin
                if (b * b if index.metric == "euclidean" else b) > keys[-1]:
                    break
        if layer >= last:
            break
        layer += 1
    return keys, idx, (layer, n_cells, n_pts)


# ------------------------------------------------------------------ epilogues
def classify(keys, idx, labels, metric="euclidean"):
    """Majority vote; ties -> label of min (sqrt key, index) (predict.py:20-36)."""
    labs = [labels[i] for i in idx]
    tally = Counter(labs)
    top = max(tally.values())
    tied = {lab for lab, c in tally.items() if c == top}
    if len(tied) == 1:
        (win,) = tied
    else:
        dist = np.sqrt(keys) if metric == "euclidean" else keys
        win = min(
            ((float(dist[a]), int(idx[a]), labs[a]) for a in range(len(labs)) if labs[a] in tied),
            key=lambda t: (t[0], t[1]),
        )[2]
    return win, tally[win] / len(labs)


def regress(idx, targets, agg="mean"):
    """Mean (numpy pairwise) or median of fp64 targets (predict.py:39-50)."""
    t = np.asarray([float(targets[i]) for i in idx])
    if agg == "mean":
        return float(t.mean())
    if agg == "median":
        return float(np.median(t))
    raise ValueError(f"unknown aggregation {agg!r}")
