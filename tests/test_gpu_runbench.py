"""run_bench on the device == the reference's run_bench.

Every deterministic report field (env, recall@k, accuracy / RMSE, mean
QueryStats) must equal the fixture the reference produced on the same input
(tests/golden/make_golden.py::bench_fixture); the CLI writes the same schema.
"""
import json
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
RUNS = json.load(open(os.path.join(GOLD, "bench_reports.json")))


@pytest.fixture(scope="module")
def g():
    import paper_2004_02290_b200 as m

    return m


@pytest.mark.parametrize("i", range(len(RUNS)))
def test_run_bench_matches_reference_report(g, i):
    from paper_2004_02290_b200.runbench import strip_timing

    call = dict(RUNS[i]["call"])
    kw = {k: v for k, v in call.items() if k not in ("spec", "points")}
    kw["algos"] = tuple(kw["algos"])
    if "spec" in call:
        sp = dict(call["spec"], path=os.path.join(GOLD, call["spec"]["path"]))
        data = g.DatasetSpec(**sp)
    else:
        z = np.load(os.path.join(GOLD, call["points"]))
        data = g.points_from_arrays(z["X"], z["y"].tolist())
    rep = g.run_bench(data, **kw)
    got = json.loads(json.dumps(strip_timing(rep.to_dict())))
    assert got == RUNS[i]["report"]
    for a in rep.algorithms:
        assert a.total_predict_ms > 0 and a.mean_query_ms > 0


def test_cli_reports(g, tmp_path):
    from paper_2004_02290_b200.runbench import main, strip_timing

    csvp = os.path.join(GOLD, "bench_cls.csv")
    out = tmp_path / "r.json"
    assert main(["--dataset", csvp, "--label-col", "label", "--k", "3", "--algos", "ghn,brute,kdtree",
                 "--seed", "0", "--report", "json", "--out", str(out)]) == 0
    assert strip_timing(json.loads(out.read_text())) == RUNS[0]["report"]
    for fmt in ("csv", "md"):
        o = tmp_path / f"r.{fmt}"
        main(["--dataset", csvp, "--label-col", "2", "--algos", "brute", "--report", fmt, "--out", str(o)])
        assert "recall_at_k" in o.read_text()


@pytest.mark.parametrize("metric", ["euclidean", "manhattan", "chebyshev"])
def test_brute_and_kdtree_exact_vs_oracle(g, metric):
    rng = np.random.default_rng(31)
    X = rng.normal(0, 1, (20_000, 4)).astype(np.float32)
    X[::50] = X[7]                                   # duplicate keys: ties by index
    Q = np.concatenate([rng.normal(0, 1, (3000, 4)), X[7:8].astype(np.float64)])
    pts = g.points_from_arrays(X, list(range(X.shape[0])))
    b = g.brute_build(pts, metric)
    k = 24
    dist, idx = g.brute_knn_batch(b, Q, k)
    # the grid oracle with a single cell is an exact scan as well
    ref = oracle.COracle(X, np.full(4, 1e6), metric=metric)
    keys, ridx, _ = ref.query(Q, k, "guaranteed")
    assert np.array_equal(idx.cpu().numpy(), ridx)
    want = np.sqrt(keys) if metric == "euclidean" else keys
    assert np.array_equal(dist.cpu().numpy(), want)
    t = g.kdtree_build(pts, metric, leaf_size=8)
    nb = g.kdtree_knn(t, Q[-1], k)
    assert [n.point_index for n in nb] == ridx[-1].tolist()
    assert [n.point_index for n in g.brute_knn(b, Q[-1], k)] == ridx[-1].tolist()
