#!/bin/bash
# compute-sanitizer on the smoke run (fit + generic predict + tiled thread kernels at k = 16 / 64)
# and a small bucket-select / list-rounds case.  One tool per gpurun call:
#   tools/sanitize.sh memcheck | racecheck | synccheck | initcheck
TOOL=${1:-memcheck}
cat > /tmp/san_case.py <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np
import __graft_entry__ as g
g.smoke()
import oracle
from paper_2004_02290_b200 import build_arrays, datagen, predict_batch
w = datagen.cfg4(n=200_000, nq=6000, seed=5)
ix = build_arrays(w.X, w.y, cells_per_axis=180)
ref = oracle.COracle(w.X, np.full(2, 1.0 / 180))
for k in (1, 4, 33, 100):
    p = predict_batch(ix, w.Q, k)
    keys, idx, _ = ref.query(w.Q, k)
    lab, conf = oracle.classify(keys, idx, w.y.astype(np.int64))
    assert np.array_equal(p["label"].cpu().numpy().astype(np.int64), lab), k
    assert np.array_equal(p["confidence"].cpu().numpy(), conf), k
print("sanitize case OK")
PY
python /tmp/san_case.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/san_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 python /tmp/san_case.py > gpurun_out/san_$TOOL.log 2>&1
echo "sanitizer rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize case OK|smoke OK|========= (Error|Invalid|Race|Barrier|Uninit)" gpurun_out/san_$TOOL.log | head -20
