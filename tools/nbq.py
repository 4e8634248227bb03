"""knn_query_batch throughput on cfg4 (10M queries): python tools/nbq.py [k ...]"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2004_02290_b200 import build_arrays, datagen, knn_query_batch

w = datagen.make(4)
dev = torch.device("cuda")
X, y, Q = (torch.from_numpy(v).to(dev) for v in (w.X, w.y, w.Q))
ix = build_arrays(X, y, cells_per_axis=w.cells_per_axis)
for k in [int(a) for a in sys.argv[1:]] or [16]:
    for stats in (False, True):
        for _ in range(2):
            knn_query_batch(ix, Q, k, stats=stats)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            knn_query_batch(ix, Q, k, stats=stats)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"k={k} stats={stats}: {ms:.2f} ms  {Q.shape[0] / ms / 1e6:.2f} G queries/s")
