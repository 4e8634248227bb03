"""Debug aid: bucket-select mismatches against the C oracle on the thread-kernel test case."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2004_02290_b200 as g
from paper_2004_02290_b200 import datagen

w = datagen.cfg4(n=3_000_000, nq=40_000, seed=61)
index = g.build_arrays(w.X, w.y, cells_per_axis=700)
ref = oracle.COracle(w.X, np.full(2, 1.0 / 700))
y = np.asarray(w.y, dtype=np.int64)
for k in [int(x) for x in sys.argv[1:]] or [33]:
    r = g.predict_batch(index, w.Q, k, "heuristic")
    keys, idx, st = ref.query(w.Q, k, "heuristic")
    lab, conf = oracle.classify(keys, idx, y)
    got = r["label"].cpu().numpy().astype(np.int64)
    gc = r["confidence"].cpu().numpy()
    bad = np.flatnonzero((got != lab) | (gc != conf))
    print("k", k, "bad", bad.size, bad[:10])
    for q in bad[:4]:
        cnts = np.bincount(y[idx[q]], minlength=4)
        keys1, idx1, st1 = ref.query(w.Q[q:q + 1], k + 3, "heuristic")
        print(" q", q, w.Q[q], "got", got[q], gc[q] * k, "want", lab[q], conf[q] * k, "counts", cnts, "stats", st[q],
              "cell frac", (w.Q[q] * 700) % 1.0)
        print("   kth keys", keys[q][-3:], "next", keys1[0][k - 1:k + 3], "labels tail", y[idx[q]][-4:], "st(k+3)", st1[0])
