"""Build the cfg4 index twice (the second under the profiler's range) -- for ncu launch lists."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2004_02290_b200 import build_arrays, datagen
w = datagen.cfg4(nq=1000)
X = torch.from_numpy(w.X).cuda(); y = torch.from_numpy(w.y).cuda()
for _ in range(2):
    ix = build_arrays(X, y, cells_per_axis=w.cells_per_axis)
    torch.cuda.synchronize()
    del ix
print("ok")
