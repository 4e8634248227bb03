"""Host side of the run_bench integration: dataset
plumbing against the reference's own outputs, report rendering, validation,
and the host records (NeighborBuffer, distance).  No GPU needed."""
import json
import os

import numpy as np
import pytest

import paper_2004_02290_b200 as g
from paper_2004_02290_b200 import datasets
from paper_2004_02290_b200.runbench import AlgoResult, BenchReport, strip_timing

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_csv_split_scaler_match_reference():
    z = np.load(os.path.join(GOLD, "bench_split.npz"))
    pts = datasets.load_csv(datasets.DatasetSpec(os.path.join(GOLD, "bench_cls.csv"), "label", "classification"))
    assert len(pts) == 700 and pts[0].dim == 3
    tr, te = datasets.split(pts, 0.8, 11)
    assert np.array_equal(np.stack([p.coords for p in tr]), z["train_X"])
    assert np.array_equal(np.array([p.label for p in tr]), z["train_y"])
    assert np.array_equal(np.stack([p.coords for p in te]), z["test_X"])
    assert [p.index for p in te] == list(range(len(te)))
    for kind in ("standard", "minmax", "none"):
        sc = datasets.fit_scaler(tr, kind)
        assert np.array_equal(sc.shift, z[f"{kind}_shift"])
        assert np.array_equal(sc.scale, z[f"{kind}_scale"])
    sc = datasets.fit_scaler(tr, "standard")
    assert np.array_equal(np.stack([p.coords for p in datasets.apply_scaler(sc, te)]), z["scaled_test"])


def test_csv_errors(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("a,b,label\n1,2,x\n3,4\n")
    with pytest.raises(datasets.DatasetError, match="line 3"):
        datasets.load_csv(datasets.DatasetSpec(str(p), "label", "classification"))
    p.write_text("a,b,label\n1,zz,x\n")
    with pytest.raises(datasets.DatasetError, match="non-numeric feature"):
        datasets.load_csv(datasets.DatasetSpec(str(p), "label", "classification"))
    p.write_text("a,b,label\n1,2,x\n")
    with pytest.raises(datasets.DatasetError, match="non-numeric regression target"):
        datasets.load_csv(datasets.DatasetSpec(str(p), "label", "regression"))
    with pytest.raises(datasets.DatasetError, match="unknown label column"):
        datasets.load_csv(datasets.DatasetSpec(str(p), "nope", "classification"))
    with pytest.raises(datasets.DatasetError, match="out of range"):
        datasets.load_csv(datasets.DatasetSpec(str(p), 5, "classification"))
    with pytest.raises(ValueError):
        datasets.DatasetSpec(str(p), 0, "ranking")
    with pytest.raises(ValueError):
        datasets.split([g.LabeledPoint(np.zeros(1), 0, 0)] * 3, 0.1, 0)
    with pytest.raises(ValueError):
        datasets.fit_scaler([], "standard")
    with pytest.raises(ValueError):
        datasets.fit_scaler([g.LabeledPoint(np.zeros(1), 0, 0)], "robust")


def test_minmax_zero_range_maps_to_half():
    pts = [g.LabeledPoint(np.array([2.0, float(i)]), 0, i) for i in range(4)]
    sc = datasets.fit_scaler(pts, "minmax")
    out = np.stack([p.coords for p in datasets.apply_scaler(sc, pts)])
    assert np.all(out[:, 0] == 0.5) and out[0, 1] == 0.0 and out[-1, 1] == 1.0


def test_report_rendering_and_strip_timing():
    rep = BenchReport(env={"k": 3, "seed": 0})
    rep.algorithms.append(AlgoResult("ghn", 1.5, 2.25, 0.01, 0.98, accuracy=0.9, mean_layers_visited=1.0,
                                     mean_cells_visited=9.0, mean_points_scanned=30.5))
    rep.algorithms.append(AlgoResult("brute", 0.0, 7.0, 0.02, 1.0, accuracy=0.9))
    d = json.loads(rep.to_json())
    assert d["schema_version"] == 1 and [a["name"] for a in d["algorithms"]] == ["ghn", "brute"]
    assert "rmse" not in d["algorithms"][0]
    s = strip_timing(d)
    assert "build_ms" not in s["algorithms"][0] and s["algorithms"][0]["recall_at_k"] == 0.98
    csv = rep.to_csv().splitlines()
    assert csv[0].split(",")[:5] == ["name", "build_ms", "total_predict_ms", "mean_query_ms", "recall_at_k"]
    assert csv[2].split(",")[0] == "brute" and csv[2].endswith(",,,")
    md = rep.to_markdown().splitlines()
    assert md[0] == "<!-- schema_version=1; k=3, seed=0 -->"
    assert md[1].startswith("| name ") and set(md[2]) <= set("| -")
    assert len({len(line) for line in md[1:]}) == 1


def test_run_bench_validation_before_device():
    pts = g.points_from_arrays(np.random.default_rng(0).random((20, 2)), [0, 1] * 10)
    with pytest.raises(ValueError, match="task is required"):
        g.run_bench(pts, algos=("brute",), k=3)
    with pytest.raises(ValueError, match="repeats"):
        g.run_bench(pts, algos=("brute",), k=3, task="classification", repeats=0)
    with pytest.raises(ValueError, match="unknown algorithms"):
        g.run_bench(pts, algos=("annoy",), k=3, task="classification")
    with pytest.raises(ValueError, match="exceeds training size"):
        g.run_bench(pts, algos=("brute",), k=17, task="classification")


def test_neighbor_buffer_and_distance():
    b = g.NeighborBuffer(3)
    with pytest.raises(IndexError):
        b.worst_key()
    assert b.push_all([g.Neighbor(2.0, 7), g.Neighbor(1.0, 9), g.Neighbor(2.0, 3)])
    assert b.full and b.worst_key() == (2.0, 7)
    assert not b.push(g.Neighbor(2.0, 8))          # ties broken toward the lower index
    assert b.push(g.Neighbor(2.0, 5))
    assert [n.point_index for n in b.neighbors()] == [9, 3, 5]
    with pytest.raises(ValueError):
        g.NeighborBuffer(0)
    assert g.distance([0, 0], [3, 4]) == 5.0
    assert g.distance([1, 1], [-2, 5], "manhattan") == 7.0
    assert g.distance([1, 1], [-2, 5], "chebyshev") == 4.0
    with pytest.raises(ValueError):
        g.distance([1, 2], [1, 2, 3])
    with pytest.raises(ValueError):
        g.distance([1], [2], "cosine")
