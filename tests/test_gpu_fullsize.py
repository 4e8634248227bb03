"""Parity at BASELINE.json's FULL sizes.

Every config is generated at its full n_train / nq (cfg3: full training set,
a seeded query sample).  The device fit is checked whole (bucket order and
offsets against the C oracle's own build of the same 100M / 50M / 10M
points); the device predict runs on every query (cfg3: the sample), and a
seeded sample of its answers is checked bit-exactly against the C oracle --
labels, confidences / means and QueryStats -- since checking 10M queries on
the host would take hours.  Size-independent properties are checked on all
answers: a query that is a training point finds itself at distance 0 (k=1),
distances are sorted, indices are distinct.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SAMPLE = 4000


@pytest.fixture(scope="module")
def ghn():
    import paper_2004_02290_b200 as g

    return g


def _sample_check(ghn, index, ref, w, Q, k, task, rng, nsample=SAMPLE):
    import torch

    Qd = torch.from_numpy(Q).cuda()
    r = ghn.predict_batch(index, Qd, k, "heuristic", task=task, stats=True)
    sel = np.sort(rng.choice(Q.shape[0], size=min(nsample, Q.shape[0]), replace=False))
    keys, idx, stats = ref.query(Q[sel], k, "heuristic")
    assert np.array_equal(r["stats"].cpu().numpy()[sel], stats), "QueryStats"
    if task == "classify":
        lab, conf = oracle.classify(keys, idx, np.asarray(w.y, dtype=np.int64))
        assert np.array_equal(r["label"].cpu().numpy()[sel].astype(np.int64), lab)
        assert np.array_equal(r["confidence"].cpu().numpy()[sel], conf)
    else:
        val = oracle.regress_mean(idx, np.asarray(w.y, dtype=np.float64))
        assert np.array_equal(r["value"].cpu().numpy()[sel], val)
    return r


def _fit_check(index, ref):
    order, _, starts, _, _ = ref.export()
    assert np.array_equal(index.order, order)
    assert np.array_equal(index.bucket_starts, starts)


@pytest.mark.parametrize("k", [1, 4, 16, 64])
def test_cfg4_full(ghn, k, cfg4_full):
    index, ref, w = cfg4_full
    rng = np.random.default_rng(4000 + k)
    _sample_check(ghn, index, ref, w, w.Q, k, "classify", rng)


@pytest.mark.parametrize("k", [1, 4, 16, 64])
def test_cfg4_full_no_stats(ghn, k, cfg4_full):
    """The benchmarked instantiation at the benchmarked plan: no QueryStats
    (its own tile side and apron), labels + confidences on a 20,000-query sample."""
    import torch

    index, ref, w = cfg4_full
    rng = np.random.default_rng(4100 + k)
    r = ghn.predict_batch(index, torch.from_numpy(w.Q).cuda(), k, "heuristic")
    sel = np.sort(rng.choice(w.Q.shape[0], size=20000, replace=False))
    keys, idx, _ = ref.query(w.Q[sel], k, "heuristic")
    lab, conf = oracle.classify(keys, idx, np.asarray(w.y, dtype=np.int64))
    assert np.array_equal(r["label"].cpu().numpy()[sel].astype(np.int64), lab)
    assert np.array_equal(r["confidence"].cpu().numpy()[sel], conf)


def test_cfg4_full_neighbors(ghn, cfg4_full):
    """knn_query_batch at the full size (tile2d_nb_kernel): indices and distances."""
    import torch

    index, ref, w = cfg4_full
    rng = np.random.default_rng(4200)
    dist, idx, _ = ghn.knn_query_batch(index, torch.from_numpy(w.Q).cuda(), 16, stats=False)
    sel = np.sort(rng.choice(w.Q.shape[0], size=10000, replace=False))
    keys, ridx, _ = ref.query(w.Q[sel], 16, "heuristic")
    sd = torch.from_numpy(sel).cuda()
    assert np.array_equal(idx[sd].cpu().numpy(), ridx)
    assert np.array_equal(dist[sd].cpu().numpy(), np.sqrt(keys))


@pytest.fixture(scope="module")
def cfg4_full(ghn):
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg4()
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=w.cells_per_axis)
    ref = oracle.COracle(w.X, w.widths)
    _fit_check(index, ref)
    return index, ref, w


def test_cfg4_full_properties(ghn, cfg4_full):
    """Training points as queries: nearest is itself or an earlier exact
    duplicate at distance 0; neighbour lists sorted and distinct."""
    index, _, w = cfg4_full
    rng = np.random.default_rng(44)
    pick = rng.choice(w.X.shape[0], 200_000, replace=False)
    dist, idx, _ = ghn.knn_query_batch(index, w.X[pick], 16, "heuristic")
    dist, idx = dist.cpu().numpy(), idx.cpu().numpy()
    assert np.all(dist[:, 0] == 0.0)
    assert np.all(idx[:, 0] <= pick)
    assert np.all(np.diff(dist, axis=1) >= 0)
    srt = np.sort(idx, axis=1)
    assert np.all(np.diff(srt, axis=1) > 0)


@pytest.mark.parametrize("cfg", [1, 2])
def test_cfg1_cfg2_full(ghn, cfg):
    from paper_2004_02290_b200 import datagen

    w = datagen.make(cfg)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=w.cells_per_axis)
    ref = oracle.COracle(w.X, w.widths)
    _fit_check(index, ref)
    task = "regress" if w.task == "regress" else "classify"
    _sample_check(ghn, index, ref, w, w.Q, w.k, task, np.random.default_rng(100 + cfg),
                  nsample=SAMPLE if cfg == 1 else 400)


def test_cfg3_full_training_set_sampled_queries(ghn):
    """cfg3: 50M lognormal points, one cell holding ~36M of them; 1,000 seeded
    queries (90 % data-distributed, 10 % uniform) through the generic kernel
    (nested grids + lower-bound pruning)."""
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg3(nq=1000)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=w.cells_per_axis)
    ref = oracle.COracle(w.X, w.widths)
    _fit_check(index, ref)
    assert np.diff(index.bucket_starts).max() > 30_000_000     # the fat cell
    _sample_check(ghn, index, ref, w, w.Q, w.k, "classify", np.random.default_rng(3), nsample=1000)
