"""Seeded synthetic workloads standing in for BASELINE.json's five configs.

The reference benchmarks no public dataset on this path; these generators
reproduce each config's shapes, sizes and value distributions (SURVEY.md
§8(d)), with the two ambiguities frozen there:
  * label flips (cfg0/cfg4): Bernoulli(0.1) mask, new label = (y + U{1,2,3}) mod 4;
  * cfg3 data-distributed queries are rescaled with the TRAINING min/max and
    are not clipped.
All coordinates are float32 (on the 2^-24 lattice for uniform draws); the
grid is GridParams(widths = 1/C, origin = X.min(0), splits = C).

``n`` / ``nq`` overrides draw smaller samples of the same distribution for
parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    X: np.ndarray            # (n, d) float32
    y: np.ndarray            # (n,) int32 labels or float32 targets
    Q: np.ndarray            # (nq, d) float32
    cells_per_axis: int
    k: int
    task: str                # "classify" | "regress"
    ks: tuple = ()           # k sweep (cfg4)
    meta: dict = field(default_factory=dict)

    @property
    def widths(self) -> np.ndarray:
        return np.full(self.X.shape[1], 1.0 / self.cells_per_axis)


DEFAULT_SIZES = {
    0: (100_000, 10_000),
    1: (2_000_000, 200_000),
    2: (10_000_000, 1_000_000),
    3: (50_000_000, 5_000_000),
    4: (100_000_000, 10_000_000),
}


def _flip(rng, y, frac=0.1):
    mask = rng.random(y.shape[0], dtype=np.float32) < frac
    shift = rng.integers(1, 4, y.shape[0]).astype(np.int32)
    return np.where(mask, (y + shift) % 4, y).astype(np.int32)


def _quadrant(X):
    return ((X[:, 0] > 0.5).astype(np.int32) * 2 + (X[:, 1] > 0.5).astype(np.int32))


def cfg0(n=None, nq=None, seed=0) -> Workload:
    """2-D uniform, quadrant labels with 10% flips, C=32, k=5, vote."""
    n = n or DEFAULT_SIZES[0][0]
    nq = nq or DEFAULT_SIZES[0][1]
    rng = np.random.default_rng(seed)
    X = rng.random((n, 2), dtype=np.float32)
    y = _flip(rng, _quadrant(X))
    Q = rng.random((nq, 2), dtype=np.float32)
    return Workload("cfg0", X, y, Q, 32, 5, "classify")


def _gmm(rng, means, m, sigma):
    comp = rng.integers(0, means.shape[0], m)
    X = means[comp] + rng.normal(0.0, sigma, (m, means.shape[1]))
    return np.clip(X, 0.0, 1.0).astype(np.float32), comp


def cfg1(n=None, nq=None, seed=1) -> Workload:
    """3-D 16-component GMM (sigma 0.05, clipped to [0,1]), label comp mod 8, C=128, k=10."""
    n = n or DEFAULT_SIZES[1][0]
    nq = nq or DEFAULT_SIZES[1][1]
    rng = np.random.default_rng(seed)
    means = rng.random((16, 3))
    X, comp = _gmm(rng, means, n, 0.05)
    Q, _ = _gmm(rng, means, nq, 0.05)
    return Workload("cfg1", X, (comp % 8).astype(np.int32), Q, 128, 10, "classify")


def cfg2(n=None, nq=None, seed=2) -> Workload:
    """6-D uniform regression y = sum sin(2 pi x) + N(0, 0.1^2), C=8, k=16, mean."""
    n = n or DEFAULT_SIZES[2][0]
    nq = nq or DEFAULT_SIZES[2][1]
    rng = np.random.default_rng(seed)
    X = rng.random((n, 6), dtype=np.float32)
    y = (np.sin(2.0 * np.pi * X.astype(np.float64)).sum(axis=1)
         + rng.normal(0.0, 0.1, n)).astype(np.float32)
    Q = rng.random((nq, 6), dtype=np.float32)
    return Workload("cfg2", X, y, Q, 8, 16, "regress")


def cfg3(n=None, nq=None, seed=3) -> Workload:
    """4-D lognormal marginals min-max scaled, skewed occupancy, C=64, k=32, vote."""
    n = n or DEFAULT_SIZES[3][0]
    nq = nq or DEFAULT_SIZES[3][1]
    rng = np.random.default_rng(seed)
    raw = rng.lognormal(0.0, 1.0, (n, 4))
    lo = raw.min(axis=0)
    hi = raw.max(axis=0)
    X = ((raw - lo) / (hi - lo)).astype(np.float32)
    del raw
    y = np.floor(10.0 * np.modf(1000.0 * X[:, 0].astype(np.float64))[0]).astype(np.int32)
    n_data = (nq * 9) // 10
    qd = ((rng.lognormal(0.0, 1.0, (n_data, 4)) - lo) / (hi - lo)).astype(np.float32)
    qu = rng.random((nq - n_data, 4), dtype=np.float32)
    Q = np.concatenate([qd, qu])
    return Workload("cfg3", X, y, Q, 64, 32, "classify", meta={"n_data_queries": n_data})


def cfg4(n=None, nq=None, seed=4, k=16) -> Workload:
    """2-D uniform at scale (100M points), C=4096, k sweep {1,4,16,64}, vote."""
    n = n or DEFAULT_SIZES[4][0]
    nq = nq or DEFAULT_SIZES[4][1]
    rng = np.random.default_rng(seed)
    X = rng.random((n, 2), dtype=np.float32)
    y = _flip(rng, _quadrant(X))
    Q = rng.random((nq, 2), dtype=np.float32)
    return Workload("cfg4", X, y, Q, 4096, k, "classify", ks=(1, 4, 16, 64))


CONFIGS = {0: cfg0, 1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4}


def make(cfg: int, n=None, nq=None, **kw) -> Workload:
    return CONFIGS[cfg](n=n, nq=nq, **kw)
