"""fit / predict wrappers named by BASELINE.json's north_star.

NEW API (the reference has none): thin classes over build_arrays +
predict_batch.  The reference's own API is the functional one
(build -> knn_query -> classify / regress, pkg/README.md:36-48).
"""

from __future__ import annotations

from .grid import build_arrays
from .predict import decode_labels, predict_batch


class _GHNBase:
    task = "classify"

    def __init__(self, k: int = 5, cells_per_axis=None, params=None, mode: str = "heuristic",
                 max_splits=None):
        self.k = k
        self.cells_per_axis = cells_per_axis
        self.params = params
        self.mode = mode
        self.max_splits = max_splits
        self.index_ = None

    def fit(self, X, y):
        self.index_ = build_arrays(X, y, params=self.params, cells_per_axis=self.cells_per_axis,
                                   max_splits=self.max_splits)
        return self

    def _predict_raw(self, Q, **kw):
        if self.index_ is None:
            raise ValueError("fit() first")
        return predict_batch(self.index_, Q, self.k, self.mode, self.task, **kw)


class GHNClassifier(_GHNBase):
    task = "classify"

    def predict(self, Q, decode: bool = False):
        r = self._predict_raw(Q)
        return decode_labels(self.index_, r["label"]) if decode else r["label"]

    def predict_proba_top(self, Q):
        r = self._predict_raw(Q)
        return r["label"], r["confidence"]


class GHNRegressor(_GHNBase):
    task = "regress"

    def predict(self, Q):
        return self._predict_raw(Q)["value"]
