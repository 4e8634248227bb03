"""GHN oracle -- TEST INFRASTRUCTURE ONLY.

Two CPU restatements of the reference path (gridneighbors):
  * ``oracle.ghn_port``  -- numpy, the reference's own algorithm (O(#cells)
    scans per query); timed as the CPU baseline / reference arm.
  * ``oracle.COracle``   -- plain C (ghn_oracle.c, built by oracle/Makefile),
    same results via a dense ring enumeration; the parity checker for the
    CUDA path at scale.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this package.  Both restatements are pinned against
fixtures produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libghn_oracle.so")
_lib = None

DENSE_LIMIT = 1 << 28
METRIC_CODES = {"euclidean": 0, "manhattan": 1, "chebyshev": 2}


def build_oracle(force: bool = False) -> str:
    """Compile ghn_oracle.c (make) if the .so is missing or stale."""
    src = os.path.join(_HERE, "ghn_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build_oracle()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    i64, i32 = ctypes.c_int64, ctypes.c_int32
    lib.ghno_sizeof_index.restype = ctypes.c_size_t
    lib.ghno_build.argtypes = [P, P, i64, i32, P, i64, i32]
    lib.ghno_build.restype = ctypes.c_int
    lib.ghno_free.argtypes = [P]
    lib.ghno_n_cells.argtypes = [P]
    lib.ghno_n_cells.restype = i64
    lib.ghno_is_dense.argtypes = [P]
    lib.ghno_is_dense.restype = i32
    lib.ghno_export.argtypes = [P, P, P, P, P, P]
    lib.ghno_query.argtypes = [P, P, i64, i32, i32, P, P, P, i32]
    lib.ghno_query.restype = ctypes.c_int
    lib.ghno_classify.argtypes = [P, P, P, i64, i32, P, P, i32]
    lib.ghno_regress_mean.argtypes = [P, P, i64, i32, P]
    lib.ghno_regress_median.argtypes = [P, P, i64, i32, P]
    lib.ghno_key.argtypes = [P, P, ctypes.c_int]
    lib.ghno_key.restype = ctypes.c_double
    lib.ghno_pairwise_sum.argtypes = [P, i64]
    lib.ghno_pairwise_sum.restype = ctypes.c_double
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class COracle:
    """Index + batched query through the C restatement."""

    def __init__(self, X, widths, dense_limit: int = DENSE_LIMIT, metric: str = "euclidean"):
        lib = _load()
        self._lib = lib
        self.X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        if self.X.ndim != 2 or self.X.shape[0] == 0:
            raise ValueError("X must be a non-empty (n, d) matrix")
        self.n, self.d = self.X.shape
        self.widths = np.ascontiguousarray(np.asarray(widths, dtype=np.float64))
        self._ix = ctypes.create_string_buffer(lib.ghno_sizeof_index())
        self.metric = metric
        rc = lib.ghno_build(self._ix, _ptr(self.X), self.n, self.d, _ptr(self.widths), dense_limit,
                            METRIC_CODES[metric])
        if rc == 1:
            raise ValueError("non-finite coordinate")
        if rc != 0:
            raise RuntimeError(f"ghno_build failed rc={rc}")
        self.n_cells = int(lib.ghno_n_cells(self._ix))
        self.dense = bool(lib.ghno_is_dense(self._ix))

    def __del__(self):
        try:
            self._lib.ghno_free(self._ix)
        except Exception:
            pass

    def export(self):
        """(order, cell_ids, cell_start, lo, ext) as int64 numpy arrays."""
        order = np.empty(self.n, np.int64)
        cids = np.empty((self.n_cells, self.d), np.int64)
        starts = np.empty(self.n_cells + 1, np.int64)
        lo = np.empty(self.d, np.int64)
        ext = np.empty(self.d, np.int64)
        self._lib.ghno_export(self._ix, _ptr(order), _ptr(cids), _ptr(starts), _ptr(lo), _ptr(ext))
        return order, cids, starts, lo, ext

    def query(self, Q, k: int, mode: str = "heuristic", threads: int | None = None):
        """Returns (keys (nq,k) f64, idx (nq,k) i64, stats (nq,3) i64)."""
        Q = np.ascontiguousarray(np.asarray(Q, dtype=np.float64).reshape(-1, self.d))
        nq = Q.shape[0]
        keys = np.empty((nq, k), np.float64)
        idx = np.empty((nq, k), np.int64)
        stats = np.empty((nq, 3), np.int64)
        m = {"heuristic": 0, "guaranteed": 1}[mode]
        th = threads if threads is not None else (os.cpu_count() or 1)
        rc = self._lib.ghno_query(self._ix, _ptr(Q), nq, k, m, _ptr(keys), _ptr(idx), _ptr(stats), th)
        if rc != 0:
            raise ValueError(f"ghno_query rc={rc}")
        return keys, idx, stats


def classify(keys, idx, label_codes, metric: str = "euclidean"):
    """Vote over int64 label codes per point -> (label code, confidence)."""
    lib = _load()
    keys = np.ascontiguousarray(keys, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    codes = np.ascontiguousarray(label_codes, dtype=np.int64)
    nq, k = keys.shape
    out_l = np.empty(nq, np.int64)
    out_c = np.empty(nq, np.float64)
    lib.ghno_classify(_ptr(keys), _ptr(idx), _ptr(codes), nq, k, _ptr(out_l), _ptr(out_c),
                      METRIC_CODES[metric])
    return out_l, out_c


def regress_mean(idx, targets):
    lib = _load()
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    t = np.ascontiguousarray(targets, dtype=np.float64)
    nq, k = idx.shape
    out = np.empty(nq, np.float64)
    lib.ghno_regress_mean(_ptr(idx), _ptr(t), nq, k, _ptr(out))
    return out


def regress_median(idx, targets):
    lib = _load()
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    t = np.ascontiguousarray(targets, dtype=np.float64)
    nq, k = idx.shape
    out = np.empty(nq, np.float64)
    lib.ghno_regress_median(_ptr(idx), _ptr(t), nq, k, _ptr(out))
    return out


def key(p, q) -> float:
    lib = _load()
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    return float(lib.ghno_key(_ptr(p), _ptr(q), p.size))


def pairwise_sum(a) -> float:
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib.ghno_pairwise_sum(_ptr(a), a.size))
