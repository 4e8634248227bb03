"""Predict throughput on clustered 2-D data (tile-path robustness check)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2004_02290_b200 as g  # noqa: E402

rng = np.random.default_rng(7)
n, nq, C = 20_000_000, 2_000_000, 2048
means = rng.random((24, 2))
comp = rng.integers(0, 24, n)
X = np.clip(means[comp] + rng.normal(0, 0.03, (n, 2)), 0, 1).astype(np.float32)
y = (comp % 4).astype(np.int32)
qc = rng.integers(0, 24, nq)
Q = np.clip(means[qc] + rng.normal(0, 0.03, (nq, 2)), 0, 1).astype(np.float32)
dev = torch.device("cuda")
ix = g.build_arrays(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), cells_per_axis=C)
Qd = torch.from_numpy(Q).to(dev)
for k in (1, 4, 16, 64):
    g.predict_batch(ix, Qd, k, confidence=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        g.predict_batch(ix, Qd, k, confidence=False)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    r = g.predict_batch(ix, Qd, k, confidence=False, totals=True)
    tot = r["totals"].cpu().numpy()
    print(f"k={k}: {ms:.2f} ms  {nq / ms / 1e3:.1f} M q/s  pts/q {tot[2] / nq:.1f}")
