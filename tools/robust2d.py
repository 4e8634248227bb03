"""Tile-path robustness: throughput and sampled parity (labels + confidences against the C
oracle) on 2-D data that is not cfg4: clustered, sparse (0.5 points per cell) and dense
(40 points per cell) sets."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2004_02290_b200 as g  # noqa: E402

dev = torch.device("cuda")


def run(name, X, y, Q, C, ks=(1, 4, 16, 64)):
    ix = g.build_arrays(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), cells_per_axis=C)
    ref = oracle.COracle(X, np.full(2, 1.0 / C))
    Qd = torch.from_numpy(Q).to(dev)
    nq = Q.shape[0]
    sel = np.sort(np.random.default_rng(1).choice(nq, size=3000, replace=False))
    for k in ks:
        g.predict_batch(ix, Qd, k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            r = g.predict_batch(ix, Qd, k)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 3 * 1e3
        keys, idx, _ = ref.query(Q[sel], k, "heuristic")
        lab, conf = oracle.classify(keys, idx, y.astype(np.int64))
        ok = (np.array_equal(r["label"].cpu().numpy()[sel].astype(np.int64), lab)
              and np.array_equal(r["confidence"].cpu().numpy()[sel], conf))
        d, i, _ = g.knn_query_batch(ix, Qd[:200000], min(k, 32), stats=False)
        keys2, idx2, _ = ref.query(Q[sel[sel < 200000]], min(k, 32), "heuristic")
        s2 = torch.from_numpy(sel[sel < 200000]).to(dev)
        ok2 = np.array_equal(i[s2].cpu().numpy(), idx2) and np.array_equal(d[s2].cpu().numpy(), np.sqrt(keys2))
        print(f"{name} k={k}: {ms:.2f} ms  {nq / ms / 1e3:.1f} M q/s  parity {'OK' if ok else 'FAIL'}  neighbours {'OK' if ok2 else 'FAIL'}",
              flush=True)


rng = np.random.default_rng(7)
n, nq = 20_000_000, 2_000_000
means = rng.random((24, 2))
comp = rng.integers(0, 24, n)
X = np.clip(means[comp] + rng.normal(0, 0.03, (n, 2)), 0, 1).astype(np.float32)
qc = rng.integers(0, 24, nq)
Q = np.clip(means[qc] + rng.normal(0, 0.03, (nq, 2)), 0, 1).astype(np.float32)
run("clustered (20M, C=2048)", X, (comp % 4).astype(np.int32), Q, 2048)
X = rng.random((2_000_000, 2), dtype=np.float32)
Q = rng.random((1_000_000, 2), dtype=np.float32)
y = rng.integers(0, 8, X.shape[0]).astype(np.int32)
run("sparse (0.5 / cell, 8 labels)", X, y, Q, 2000)
run("dense (40 / cell, 8 labels)", X, y, Q, 224)
