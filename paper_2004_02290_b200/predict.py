"""Prediction epilogue (drop-in for gridneighbors/predict.py) and the fused
device predict.

Reference: pkg/src/gridneighbors/predict.py:14-50.
  * ``classify`` / ``regress`` keep the reference signatures over a host
    list of Neighbor records (a k-element host utility, as in the reference).
  * ``predict_batch`` is the hot path: one device launch that explores,
    selects and votes / averages for every query (csrc/ghn_query.cu epilogue:
    vote with the (sqrt(key), index) tie-break, numpy pairwise mean).
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .core import Neighbor
from .explore import _run, _validate
from .grid import GridIndex


@dataclass(frozen=True)
class Prediction:
    value: object
    confidence: float | None = None


def classify(neighbors: Sequence[Neighbor]) -> Prediction:
    """Majority vote; ties -> label of the member minimising (distance, index) (predict.py:20-36)."""
    if not neighbors:
        raise ValueError("cannot classify from an empty neighbor list")
    tally = Counter(nb.label for nb in neighbors)
    top = max(tally.values())
    tied = {lab for lab, c in tally.items() if c == top}
    if len(tied) == 1:
        (win,) = tied
    else:
        win = min((nb for nb in neighbors if nb.label in tied), key=lambda nb: nb.key).label
    return Prediction(value=win, confidence=tally[win] / len(neighbors))


def regress(neighbors: Sequence[Neighbor], agg: str = "mean") -> Prediction:
    """Mean (numpy pairwise) or median of float(label) (predict.py:39-50)."""
    if not neighbors:
        raise ValueError("cannot regress from an empty neighbor list")
    t = np.asarray([float(nb.label) for nb in neighbors])
    if agg == "mean":
        return Prediction(value=float(t.mean()), confidence=None)
    if agg == "median":
        return Prediction(value=float(np.median(t)), confidence=None)
    raise ValueError(f"unknown aggregation {agg!r}; expected 'mean' or 'median'")


TASKS = {"classify": _lib.GHN_TASK_CLASSIFY, "regress": _lib.GHN_TASK_REGRESS_MEAN,
         "regress_median": _lib.GHN_TASK_REGRESS_MEDIAN}


def predict_batch(index: GridIndex, Q, k: int, mode: str = "heuristic", task: str = "classify",
                  neighbors: bool = False, stats: bool = False, totals: bool = False, stream=None,
                  qorder=None, confidence: bool = True):
    """Fused device predict for nq queries (new API).

    Returns a dict of device tensors: task "classify" -> ``label`` (int32
    label codes; ``index.decode_labels`` maps them back) and ``confidence``;
    task "regress" -> ``value`` (fp64 mean), "regress_median" -> ``value``
    (np.median of the k targets).  Optional ``dist``/``idx``
    (neighbours), ``stats`` (nq, 3) and ``totals`` (sum layers, cells,
    points, queries).  ``qorder``: a visit order from ``query_order`` (else
    queries are binned internally).
    """
    if task not in TASKS:
        raise ValueError(f"unknown task {task!r}; expected one of {tuple(TASKS)}")
    Qt = _validate(index, Q, k, mode)
    r = _run(index, Qt, k, mode, TASKS[task], neighbors, stats, want_totals=totals, stream=stream,
             qorder=qorder, want_confidence=confidence)
    r.pop("_keepalive", None)
    return r


def decode_labels(index: GridIndex, codes) -> list:
    """Map device label codes back to the original label objects."""
    c = codes.cpu().tolist() if hasattr(codes, "cpu") else list(codes)
    return [index._labels.label_of(int(x)) for x in c]
