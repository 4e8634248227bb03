import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2004_02290_b200 as g
dev = torch.device("cuda")
rng = np.random.default_rng(7)
n, nq = 20_000_000, 2_000_000
means = rng.random((24, 2)); comp = rng.integers(0, 24, n)
X = np.clip(means[comp] + rng.normal(0, 0.03, (n, 2)), 0, 1).astype(np.float32)
qc = rng.integers(0, 24, nq)
Q = np.clip(means[qc] + rng.normal(0, 0.03, (nq, 2)), 0, 1).astype(np.float32)
ix = g.build_arrays(torch.from_numpy(X).to(dev), torch.from_numpy((comp % 4).astype(np.int32)).to(dev), cells_per_axis=2048)
Qd = torch.from_numpy(Q).to(dev)
torch.cuda.synchronize(); print("built", flush=True)
for k in (1, 4, 16, 64):
    r = g.predict_batch(ix, Qd, k); torch.cuda.synchronize(); print("predict ok", k, flush=True)
for nqq in (200000, 2000000):
    for k in (1, 4, 16, 32):
        for st in (False, True):
            d, i, s = g.knn_query_batch(ix, Qd[:nqq], k, stats=st); torch.cuda.synchronize(); print("knn ok", nqq, k, st, flush=True)
