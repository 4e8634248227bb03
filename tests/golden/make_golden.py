"""Generate golden fixtures by running the REFERENCE gridneighbors package.

Run in the authoring container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference read-only under the alias ``gridneighbors_ref``
and writes small ``.npz`` fixtures next to this script.  The GPU box never
runs this script; tests only read the committed fixtures.

Fixture families (each pins the oracle and, on a GPU, the CUDA path):
  einsum.npz     numpy einsum('ij,ij->i') keys for d = 1..24 (core.py:80)
  mean.npz       numpy mean of k fp64 targets, k = 1..300 (predict.py:45)
  case_*.npz     build + knn_query + classify/regress outputs of the
                 reference on seeded inputs (grid.py:165-195, explore.py:66-137,
                 predict.py:20-50)
"""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/gridneighbors"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "gridneighbors_ref", os.path.join(REF_SRC, "__init__.py"),
        submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["gridneighbors_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def run_case(ref, name, X, y, Q, k, mode, task, widths=None, max_splits=None, notes="", metric="euclidean",
             agg="mean"):
    """Run the reference on (X, y) and queries Q; save everything."""
    Xf = np.asarray(X, dtype=np.float64)           # the reference upcasts (core.py:32)
    pts = ref.points_from_arrays(Xf, list(y.tolist()))
    if widths is None:
        index = ref.build(pts, metric=metric, max_splits=max_splits)
    else:
        d = Xf.shape[1]
        params = ref.GridParams(np.asarray(widths, dtype=np.float64), Xf.min(axis=0), np.ones(d, np.int64))
        index = ref.build(pts, metric=metric, params=params)
    order = np.concatenate(index.buckets).astype(np.int64)
    sizes = np.array([b.size for b in index.buckets], np.int64)
    nq = Q.shape[0]
    nb_idx = np.empty((nq, k), np.int64)
    nb_dist = np.empty((nq, k), np.float64)
    stats = np.empty((nq, 3), np.int64)
    pred = np.empty(nq, np.float64)
    conf = np.empty(nq, np.float64)
    for i in range(nq):
        nbrs, st = ref.knn_query(index, np.asarray(Q[i], dtype=np.float64), k, mode)
        nb_idx[i] = [nb.point_index for nb in nbrs]
        nb_dist[i] = [nb.distance for nb in nbrs]
        stats[i] = [st.layers_visited, st.cells_visited, st.points_scanned]
        if task == "classify":
            p = ref.classify(nbrs)
            pred[i] = p.value
            conf[i] = p.confidence
        else:
            p = ref.regress(nbrs, agg)
            pred[i] = p.value
            conf[i] = np.nan
    np.savez_compressed(
        os.path.join(HERE, f"case_{name}.npz"),
        X=X, y=y, Q=Q, k=np.int64(k), mode=np.array(mode), task=np.array(task),
        widths=np.asarray(index.params.widths, np.float64),
        origin=np.asarray(index.params.origin, np.float64),
        splits=np.asarray(index.params.splits, np.int64),
        explicit_widths=np.bool_(widths is not None),
        max_splits=np.int64(-1 if max_splits is None else max_splits),
        order=order, bucket_sizes=sizes,
        cell_array=np.asarray(index.cell_array, np.int64),
        nb_idx=nb_idx, nb_dist=nb_dist, stats=stats, pred=pred, conf=conf,
        notes=np.array(notes), metric=np.array(metric), agg=np.array(agg))
    print(f"case_{name}: n={X.shape[0]} d={X.shape[1]} nq={nq} k={k} mode={mode} "
          f"cells={sizes.size} mean_layers={stats[:, 0].mean():.2f} mean_points={stats[:, 2].mean():.1f}")


def einsum_fixture():
    rng = np.random.default_rng(20040229)
    out = {}
    for d in range(1, 25):
        P = rng.normal(0, 1, (64, d)) * rng.uniform(1e-3, 1e3, d)
        q = rng.normal(0, 1, d)
        diff = P - q
        out[f"P{d}"] = P
        out[f"q{d}"] = q
        out[f"key{d}"] = np.einsum("ij,ij->i", diff, diff)
    np.savez_compressed(os.path.join(HERE, "einsum.npz"), **out)


def mean_fixture():
    rng = np.random.default_rng(7)
    out = {}
    for k in range(1, 301):
        t = rng.normal(0, 3, k) * 10.0 ** rng.uniform(-3, 3, k)
        out[f"t{k}"] = t
        out[f"mean{k}"] = np.float64(t.mean())
        out[f"median{k}"] = np.float64(np.median(t))
    np.savez_compressed(os.path.join(HERE, "mean.npz"), **out)


def bench_fixture(ref):
    """run_bench reports (timing stripped) produced by the reference itself on
    seeded CSV / point inputs, plus its split and scaler outputs."""
    import csv
    import json

    rng = np.random.default_rng(820)
    centers = rng.uniform(-5, 5, (5, 3))
    comp = rng.integers(0, 5, 700)
    X = centers[comp] + rng.normal(0, 1.2, (700, 3))
    names = ["north", "east", "south", "west", "zenith"]
    with open(os.path.join(HERE, "bench_cls.csv"), "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(["f0", "f1", "label", "f2"])
        for x, c in zip(X, comp):
            wr.writerow([repr(float(x[0])), repr(float(x[1])), names[c], repr(float(x[2]))])
    Xr = rng.uniform(0, 10, (400, 2))
    yr = np.sin(Xr[:, 0]) + 0.1 * Xr[:, 1] ** 2 + rng.normal(0, 0.05, 400)
    with open(os.path.join(HERE, "bench_reg.csv"), "w", newline="") as fh:
        wr = csv.writer(fh)
        for x, t in zip(Xr, yr):
            wr.writerow([repr(float(t)), repr(float(x[0])), repr(float(x[1]))])
    Xp = np.concatenate([rng.normal(0, 1, (150, 2)), rng.normal(4, 0.7, (150, 2))])
    yp = np.concatenate([np.zeros(150, np.int64), np.ones(150, np.int64)])
    np.savez_compressed(os.path.join(HERE, "bench_points.npz"), X=Xp, y=yp)

    cls = dict(path="bench_cls.csv", label_column="label", task="classification", has_header=True)
    reg = dict(path="bench_reg.csv", label_column=0, task="regression", has_header=False)
    runs = [
        dict(spec=cls, algos=["ghn", "brute", "kdtree"], k=3, mode="heuristic", scaler_kind="standard", seed=0),
        dict(spec=cls, algos=["ghn", "brute"], k=5, mode="guaranteed", scaler_kind="minmax", seed=3),
        dict(spec=cls, algos=["ghn", "kdtree"], k=4, mode="heuristic", scaler_kind="none", seed=7,
             metric="manhattan"),
        dict(spec=reg, algos=["ghn", "brute", "kdtree"], k=4, mode="heuristic", scaler_kind="standard",
             seed=2),
        dict(points="bench_points.npz", task="classification", algos=["ghn", "brute"], k=3,
             mode="heuristic", scaler_kind="standard", seed=1, split_fraction=0.7),
    ]
    out = []
    for r in runs:
        kw = {k: v for k, v in r.items() if k not in ("spec", "points")}
        kw["algos"] = tuple(kw["algos"])
        if "spec" in r:
            sp = dict(r["spec"], path=os.path.join(HERE, r["spec"]["path"]))
            data = ref.DatasetSpec(**sp)
        else:
            z = np.load(os.path.join(HERE, r["points"]))
            data = ref.points_from_arrays(z["X"], z["y"].tolist())
        rep = ref.run_bench(data, **kw)
        from gridneighbors_ref.bench import strip_timing
        out.append({"call": r, "report": strip_timing(rep.to_dict())})
    with open(os.path.join(HERE, "bench_reports.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    # split / scaler outputs on the classification CSV
    pts = ref.load_csv(ref.DatasetSpec(os.path.join(HERE, "bench_cls.csv"), "label", "classification"))
    tr, te = ref.split(pts, 0.8, 11)
    sc = {kind: ref.fit_scaler(tr, kind) for kind in ("standard", "minmax", "none")}
    np.savez_compressed(
        os.path.join(HERE, "bench_split.npz"),
        train_X=np.stack([p.coords for p in tr]), train_y=np.array([p.label for p in tr]),
        test_X=np.stack([p.coords for p in te]), test_y=np.array([p.label for p in te]),
        **{f"{k}_shift": v.shift for k, v in sc.items()}, **{f"{k}_scale": v.scale for k, v in sc.items()},
        scaled_test=np.stack([p.coords for p in ref.apply_scaler(sc["standard"], te)]))


def main():
    sys.path.insert(0, REPO)
    from paper_2004_02290_b200 import datagen

    ref = load_reference()
    bench_fixture(ref)
    einsum_fixture()
    mean_fixture()

    # cfg-shaped float32 cases with explicit widths 1/C (the BASELINE.json grids)
    w = datagen.cfg0(n=3000, nq=300, seed=100)
    run_case(ref, "cfg0_heur", w.X, w.y, w.Q, 5, "heuristic", "classify", widths=w.widths)
    run_case(ref, "cfg0_guar", w.X, w.y, w.Q[:100], 5, "guaranteed", "classify", widths=w.widths)
    w = datagen.cfg1(n=20000, nq=200, seed=101)
    run_case(ref, "cfg1_heur", w.X, w.y, w.Q, 10, "heuristic", "classify", widths=w.widths,
             notes="clipped faces: exact duplicate keys")
    w = datagen.cfg2(n=6000, nq=60, seed=102)
    run_case(ref, "cfg2_heur", w.X, w.y, w.Q, 16, "heuristic", "regress", widths=w.widths)
    w = datagen.cfg3(n=20000, nq=100, seed=103)
    run_case(ref, "cfg3_heur", w.X, w.y, w.Q, 32, "heuristic", "classify", widths=w.widths,
             notes="skewed occupancy; last 10 queries uniform")
    for kk in (1, 4, 16, 64):
        w = datagen.cfg4(n=40000, nq=150, seed=104)
        w.cells_per_axis = 128
        run_case(ref, f"cfg4_k{kk}", w.X, w.y, w.Q, kk, "heuristic", "classify", widths=w.widths)

    # reference-test-style fp64 instances with FITTED widths (params=None)
    rng = np.random.default_rng(303)
    for t in range(24):
        d = int(rng.integers(1, 7))
        n = int(10 ** rng.uniform(np.log10(50), np.log10(3000)))
        if t % 2:
            c = int(rng.integers(2, 6))
            centers = rng.uniform(0, 100, (c, d))
            X = centers[rng.integers(0, c, n)] + rng.normal(0, rng.uniform(0.5, 3.0), (n, d))
        else:
            X = rng.uniform(-50, 50, (n, d))
        y = rng.integers(0, 4, n).astype(np.int64)
        near = X[rng.integers(0, n, 12)] + rng.normal(0, 0.5, (12, d))
        far = rng.uniform(-150, 150, (4, d))
        Q = np.concatenate([near, far, np.full((1, d), 1e5)])
        k = int(min(rng.choice([1, 3, 10, 33]), n))
        mode = "guaranteed" if t % 3 == 0 else "heuristic"
        task = "regress" if t % 5 == 4 else "classify"
        yy = y.astype(np.float64) * 1.25 - 0.5 if task == "regress" else y
        ms = 7 if t % 7 == 6 else None
        run_case(ref, f"fit{t:02d}", X, yy, Q, k, mode, task, max_splits=ms)

    # other metrics (core.py:81-84, explore.py:125) and the median (predict.py:46-47)
    for mt in ("manhattan", "chebyshev"):
        w = datagen.cfg1(n=8000, nq=120, seed=110)
        run_case(ref, f"metric_{mt}_heur", w.X, w.y, w.Q, 7, "heuristic", "classify", widths=w.widths,
                 metric=mt)
        run_case(ref, f"metric_{mt}_guar", w.X, w.y, w.Q[:60], 7, "guaranteed", "classify",
                 widths=w.widths, metric=mt)
    rng2 = np.random.default_rng(111)
    X = rng2.normal(0, 2, (900, 5))
    y = np.round(rng2.normal(0, 3, 900), 1)
    Q = X[rng2.integers(0, 900, 40)] + rng2.normal(0, 0.4, (40, 5))
    run_case(ref, "metric_manhattan_fit5", X, y, Q, 9, "guaranteed", "regress", metric="manhattan")
    w = datagen.cfg2(n=5000, nq=50, seed=112)
    run_case(ref, "median_even_k", w.X, w.y, w.Q, 16, "heuristic", "regress", widths=w.widths, agg="median")
    run_case(ref, "median_odd_k", w.X, w.y, w.Q, 9, "heuristic", "regress", widths=w.widths, agg="median")

    # index files written by the reference's save_index (grid.py:211-246)
    rng = np.random.default_rng(515)
    X = rng.normal(0, 2, (120, 3))
    pts = ref.points_from_arrays(X, list(rng.integers(0, 3, 120).tolist()))
    ref.save_index(ref.build(pts), os.path.join(HERE, "index_fit_int.ghn"))
    w = datagen.cfg0(n=2000, nq=10, seed=516)
    pts = ref.points_from_arrays(w.X.astype(np.float64), [["a", "b", "c", "d"][v] for v in w.y])
    params = ref.GridParams(w.widths, w.X.astype(np.float64).min(0), np.full(2, 32))
    ref.save_index(ref.build(pts, params=params), os.path.join(HERE, "index_cfg0_str.ghn"))
    np.save(os.path.join(HERE, "index_cfg0_str_X.npy"), w.X)

    # the walkthrough scenario (test_explore.py:61-84) as a fixture as well
    X = np.array([[5.4, 5.4], [4.2, 5.5], [6.7, 5.5], [5.5, 6.9], [7.9, 7.9], [9.5, 9.5]])
    run_case(ref, "walkthrough", X, np.array([0, 0, 1, 1, 1, 0]), np.array([[5.5, 5.5]]), 3,
             "heuristic", "classify", widths=[1.0, 1.0])


if __name__ == "__main__":
    main()
