"""The oracle pinned against fixtures produced by the reference itself.

CPU only.  Both restatements (numpy port and C) must reproduce every
golden case bit for bit: bucket order, cell array, neighbour indices,
distances, QueryStats and the vote / mean.
"""
import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case
import oracle
from oracle import ghn_port

CASES = golden_cases()


def test_fixture_inventory():
    assert len(CASES) >= 30
    assert "walkthrough" in CASES


def test_einsum_order_matches_fixture():
    z = np.load(f"{GOLDEN}/einsum.npz")
    for d in range(1, 25):
        P, q, want = z[f"P{d}"], z[f"q{d}"], z[f"key{d}"]
        got = np.array([oracle.key(p, q) for p in P])
        assert np.array_equal(got, want), d
        # and this machine's numpy agrees with the fixture numpy
        diff = P - q
        assert np.array_equal(np.einsum("ij,ij->i", diff, diff), want), d


def test_pairwise_mean_matches_fixture():
    z = np.load(f"{GOLDEN}/mean.npz")
    for k in range(1, 301):
        t = z[f"t{k}"]
        assert oracle.pairwise_sum(t) / k == z[f"mean{k}"], k


def _dist(keys, c):
    return np.sqrt(keys) if str(c["metric"]) == "euclidean" else keys


@pytest.mark.parametrize("name", CASES)
def test_c_oracle_matches_reference(name):
    c = load_case(name)
    X = c["X"].astype(np.float64)
    ix = oracle.COracle(X, c["widths"], metric=str(c["metric"]))
    order, cids, starts, lo, ext = ix.export()
    assert np.array_equal(order, c["order"])
    assert np.array_equal(cids, c["cell_array"])
    assert np.array_equal(np.diff(starts), c["bucket_sizes"])
    k = int(c["k"])
    keys, idx, stats = ix.query(c["Q"], k, str(c["mode"]), threads=2)
    assert np.array_equal(idx, c["nb_idx"])
    assert np.array_equal(_dist(keys, c), c["nb_dist"])
    assert np.array_equal(stats, c["stats"])
    if str(c["task"]) == "classify":
        codes = c["y"].astype(np.int64)
        lab, conf = oracle.classify(keys, idx, codes, str(c["metric"]))
        assert np.array_equal(lab.astype(np.float64), c["pred"])
        assert np.array_equal(conf, c["conf"])
    elif str(c["agg"]) == "median":
        assert np.array_equal(oracle.regress_median(idx, c["y"].astype(np.float64)), c["pred"])
    else:
        val = oracle.regress_mean(idx, c["y"].astype(np.float64))
        assert np.array_equal(val, c["pred"])


@pytest.mark.parametrize("name", CASES)
def test_c_oracle_list_mode_matches_reference(name):
    """Force the cell-list scan (dense_limit=0): the explore.py:105 restatement."""
    c = load_case(name)
    ix = oracle.COracle(c["X"].astype(np.float64), c["widths"], dense_limit=0, metric=str(c["metric"]))
    order, cids, starts, _, _ = ix.export()
    assert np.array_equal(order, c["order"])
    assert np.array_equal(cids, c["cell_array"])
    keys, idx, stats = ix.query(c["Q"], int(c["k"]), str(c["mode"]), threads=2)
    assert np.array_equal(idx, c["nb_idx"])
    assert np.array_equal(stats, c["stats"])


@pytest.mark.parametrize("name", [n for n in CASES if not n.startswith("fit")] + ["fit03", "fit07"])
def test_numpy_port_matches_reference(name):
    c = load_case(name)
    ix = ghn_port.build(c["X"], c["y"], c["widths"], str(c["metric"]))
    assert np.array_equal(ix.order, c["order"])
    assert np.array_equal(ix.cell_array, c["cell_array"])
    k = int(c["k"])
    for qi in range(min(40, c["Q"].shape[0])):
        keys, idx, st = ghn_port.knn(ix, c["Q"][qi], k, str(c["mode"]))
        assert np.array_equal(idx, c["nb_idx"][qi])
        assert np.array_equal(_dist(keys, c), c["nb_dist"][qi])
        assert list(st) == list(c["stats"][qi])
        if str(c["task"]) == "classify":
            lab, conf = ghn_port.classify(keys, idx, c["y"], str(c["metric"]))
            assert lab == c["pred"][qi] and conf == c["conf"][qi]
        else:
            assert ghn_port.regress(idx, c["y"], str(c["agg"])) == c["pred"][qi]


@pytest.mark.parametrize("name", [n for n in CASES if n.startswith("fit")])
def test_numpy_port_fit_widths_match_reference(name):
    c = load_case(name)
    ms = int(c["max_splits"])
    w, origin, splits = ghn_port.fit_widths(c["X"], None if ms < 0 else ms)
    assert np.array_equal(w, c["widths"])
    assert np.array_equal(origin, c["origin"])
    assert np.array_equal(splits, c["splits"])
