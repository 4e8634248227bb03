"""GPU parity on BASELINE.json-shaped workloads against the C oracle.

Bit-exact: bucket order, neighbour indices, distances, QueryStats, vote
labels and confidences, regression means.  Covers both predict kernels:
the tiled thread-per-query kernel (2-D dense, classify) and the generic
warp-per-query kernel (everything else, and the tiled kernel's fallbacks).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ghn():
    import paper_2004_02290_b200 as g

    return g


def _check_predict(ghn, index, ref, X, y, Q, k, mode, task="classify"):
    r = ghn.predict_batch(index, Q, k, mode, task=task, stats=True)
    keys, idx, stats = ref.query(Q, k, mode)
    assert np.array_equal(r["stats"].cpu().numpy(), stats), "QueryStats"
    if task == "classify":
        lab, conf = oracle.classify(keys, idx, np.asarray(y, dtype=np.int64))
        got = r["label"].cpu().numpy().astype(np.int64)
        bad = np.flatnonzero(got != lab)
        assert bad.size == 0, f"{bad.size} label mismatches, first {bad[:5]}"
        assert np.array_equal(r["confidence"].cpu().numpy(), conf)
    else:
        val = oracle.regress_mean(idx, np.asarray(y, dtype=np.float64))
        assert np.array_equal(r["value"].cpu().numpy(), val)
    return keys, idx, stats


def _check_knn(ghn, index, ref, Q, k, mode):
    dist, idx, stats = ghn.knn_query_batch(index, Q, k, mode)
    keys, ridx, rstats = ref.query(Q, k, mode)
    assert np.array_equal(idx.cpu().numpy(), ridx)
    assert np.array_equal(dist.cpu().numpy(), np.sqrt(keys))
    assert np.array_equal(stats.cpu().numpy(), rstats)


@pytest.mark.parametrize("mode", ["heuristic", "guaranteed"])
def test_cfg0_full(ghn, mode):
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg0()
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=w.cells_per_axis)
    ref = oracle.COracle(w.X, w.widths)
    order, _, starts, _, _ = ref.export()
    assert np.array_equal(index.order, order)
    assert np.array_equal(index.bucket_starts, starts)
    _check_predict(ghn, index, ref, w.X, w.y, w.Q, w.k, mode)
    _check_knn(ghn, index, ref, w.Q, w.k, mode)


@pytest.mark.parametrize("k", [1, 4, 16, 64])
def test_cfg4_shaped_non_pow2_width(ghn, k):
    """cfg4 recipe at 4M points on an 820 x 820 grid (width 1/820 is not a power
    of two, so cell ids take the fp64-division path), 100k queries, plus
    outlier queries that must fall back to the generic kernel."""
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg4(n=4_000_000, nq=100_000, seed=41)
    Q = np.concatenate([w.Q, np.array([[1.5, -0.2], [10.0, 10.0], [-3.0, 0.5], [0.5, 1.0000001]],
                                      dtype=np.float32)])
    widths = np.full(2, 1.0 / 820)
    params = ghn.GridParams(widths, w.X.min(0), np.full(2, 820))
    index = ghn.build_arrays(w.X, w.y, params=params)
    ref = oracle.COracle(w.X, widths)
    _check_predict(ghn, index, ref, w.X, w.y, Q, k, "heuristic")
    if k == 16:
        _check_predict(ghn, index, ref, w.X, w.y, Q[:20000], k, "guaranteed")
        _check_knn(ghn, index, ref, Q[:20000], k, "heuristic")


def test_duplicate_points_fall_back_exactly(ghn):
    """Many exact duplicates: equal keys the radix select cannot split go to the
    generic kernel; ties are broken by point index exactly."""
    rng = np.random.default_rng(5)
    X = rng.random((200_000, 2), dtype=np.float32)
    X[::7] = X[3]                          # 28.6k copies of one point
    X[1::11] = np.float32(0.25)            # and a diagonal of copies
    y = rng.integers(0, 3, X.shape[0]).astype(np.int32)
    Q = np.concatenate([rng.random((40_000, 2), dtype=np.float32), np.repeat(X[3:4], 100, 0)])
    index = ghn.build_arrays(X, y, cells_per_axis=256)
    ref = oracle.COracle(X, np.full(2, 1.0 / 256))
    for k in (3, 16):
        _check_predict(ghn, index, ref, X, y, Q, k, "heuristic")


def test_cell_over_16bit_count_exact(ghn):
    """A cell of >= 65,536 points overflows the fit's packed 16-bit histogram
    into its neighbour's counter; the build must detect it (counts summing to
    less than n), recount in int32 and keep the reference's stable bucket
    order (lexsort of the cell ids, then the input index)."""
    rng = np.random.default_rng(11)
    X = rng.random((240_000, 2), dtype=np.float32)
    X[::3] = X[4]                          # 80k copies: one cell of > 65,535 points
    X[1::3][:10_000] = X[5]                # and the next even/odd partner filled too
    y = rng.integers(0, 4, X.shape[0]).astype(np.int32)
    index = ghn.build_arrays(X, y, cells_per_axis=256)
    ids = np.floor(X.astype(np.float64) * 256).astype(np.int64)
    order = np.lexsort((np.arange(X.shape[0]), ids[:, 1], ids[:, 0]))
    np.testing.assert_array_equal(index.perm.cpu().numpy(), order)
    Q = np.concatenate([rng.random((20_000, 2), dtype=np.float32), np.repeat(X[4:5], 50, 0)])
    ref = oracle.COracle(X, np.full(2, 1.0 / 256))
    _check_predict(ghn, index, ref, X, y, Q, 8, "heuristic")


@pytest.mark.parametrize("cfg,nq", [(1, 30_000), (2, 400)])
def test_cfg1_cfg2_generic_kernel(ghn, cfg, nq):
    from paper_2004_02290_b200 import datagen

    n = 2_000_000 if cfg == 1 else 1_000_000
    w = datagen.make(cfg, n=n, nq=nq)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=w.cells_per_axis)
    ref = oracle.COracle(w.X, w.widths)
    order, cids, starts, _, _ = ref.export()
    assert np.array_equal(index.order, order)
    assert np.array_equal(index.cell_array, cids)
    task = "regress" if w.task == "regress" else "classify"
    _check_predict(ghn, index, ref, w.X, w.y, w.Q, w.k, "heuristic", task=task)
    _check_knn(ghn, index, ref, w.Q[:200], w.k, "heuristic")


@pytest.mark.parametrize("n_labels", [4, 20])
@pytest.mark.parametrize("k", [1, 5, 16])
def test_tiled_kernel_variants_exact(ghn, n_labels, k):
    """The tiled kernel variants the plan picks (tile2d_plan): thread per
    query for <= 8 label codes, 8-lane groups for k = 1 with <= 32 codes,
    the warp kernel otherwise -- all exact, both stop modes."""
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg4(n=1_000_000, nq=60_000, seed=45)
    y = (w.y if n_labels == 4 else np.random.default_rng(46).integers(0, n_labels, w.X.shape[0])).astype(np.int32)
    index = ghn.build_arrays(w.X, y, cells_per_axis=512)
    ref = oracle.COracle(w.X, np.full(2, 1.0 / 512))
    _check_predict(ghn, index, ref, w.X, y, w.Q, k, "heuristic")
    _check_predict(ghn, index, ref, w.X, y, w.Q[:20000], k, "guaranteed")


@pytest.mark.parametrize("n_labels", [2, 40, 200, 300])
@pytest.mark.parametrize("k", [1, 16, 64])
def test_label_cardinalities(ghn, n_labels, k):
    """Vote paths by label count: shared counters (<= 32 codes), the per-warp
    label table over staged u8 codes (<= 256), the generic kernel (> 256)."""
    rng = np.random.default_rng(700 + n_labels)
    X = rng.random((400_000, 2), dtype=np.float32)
    y = rng.integers(0, n_labels, X.shape[0]).astype(np.int32)
    Q = rng.random((30_000, 2), dtype=np.float32)
    index = ghn.build_arrays(X, y, cells_per_axis=256)
    ref = oracle.COracle(X, np.full(2, 1.0 / 256))
    _check_predict(ghn, index, ref, X, y, Q, k, "heuristic")


@pytest.mark.parametrize("k", [2, 4, 9, 16])
def test_lattice_ties_exact(ghn, k):
    """Points on a coarse lattice: many exactly equal keys (and equal fp32
    round-downs) inside one selection -- ties resolved by point index, in
    both the extraction and the histogram selects."""
    rng = np.random.default_rng(808 + k)
    X = (rng.integers(0, 300, (300_000, 2)) / 300.0).astype(np.float32)
    Q = np.concatenate([(rng.integers(0, 300, (20_000, 2)) / 300.0 + 1 / 600.0),
                        rng.random((20_000, 2))]).astype(np.float32)
    y = rng.integers(0, 3, X.shape[0]).astype(np.int32)
    index = ghn.build_arrays(X, y, cells_per_axis=256)
    ref = oracle.COracle(X, np.full(2, 1.0 / 256))
    _check_predict(ghn, index, ref, X, y, Q, k, "heuristic")


@pytest.mark.parametrize("k", [1, 7, 16, 40])
def test_clustered_2d_density_sized_tiles(ghn, k):
    """Clustered 2-D data: tiles sized by the local density quantile
    (ghn_window_density) instead of the mean; still exact."""
    rng = np.random.default_rng(950 + k)
    means = rng.random((6, 2))
    comp = rng.integers(0, 6, 600_000)
    X = np.clip(means[comp] + rng.normal(0, 0.02, (600_000, 2)), 0, 1).astype(np.float32)
    y = (comp % 3).astype(np.int32)
    qc = rng.integers(0, 6, 30_000)
    Q = np.clip(means[qc] + rng.normal(0, 0.02, (30_000, 2)), 0, 1).astype(np.float32)
    index = ghn.build_arrays(X, y, cells_per_axis=512)
    assert index.density_hint() > 3 * X.shape[0] / (512 * 512)
    ref = oracle.COracle(X, np.full(2, 1.0 / 512))
    _check_predict(ghn, index, ref, X, y, Q, k, "heuristic")


def test_concurrent_readers_on_streams(ghn):
    """Any number of concurrent readers of a built index (SPEC: concurrent
    reads): two host threads predicting on their own CUDA streams get the
    single-threaded answers."""
    import threading

    import torch

    from paper_2004_02290_b200 import datagen

    w = datagen.cfg4(n=2_000_000, nq=80_000, seed=77)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=1024)
    Q = torch.from_numpy(w.Q).cuda()
    want = {k: ghn.predict_batch(index, Q, k)["label"].cpu() for k in (1, 5, 16, 33)}
    got, errs = {}, []

    def run(ks):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(3):
                    for k in ks:
                        got[k] = ghn.predict_batch(index, Q, k, stream=st)["label"]
            st.synchronize()
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(ks,)) for ks in ((1, 16), (5, 33))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for k in want:
        assert torch.equal(got[k].cpu(), want[k])
