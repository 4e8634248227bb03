"""Time the cfg4 device fit (build_arrays, device input): median of 7 after 2 warm-ups."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2004_02290_b200 import build_arrays, datagen
w = datagen.cfg4(nq=1000)
X = torch.from_numpy(w.X).cuda(); y = torch.from_numpy(w.y).cuda()
ts = []
for it in range(9):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    ix = build_arrays(X, y, cells_per_axis=w.cells_per_axis)
    b.record(); torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b))
    del ix
ts.sort()
print("fit ms median %.3f min %.3f" % (ts[len(ts) // 2], ts[0]), sys.argv[1:])
