#!/bin/bash
# Queries-per-tile sweep of the thread kernels (tuning build in gpurun_alt/libghn_tune.so).
cp paper_2004_02290_b200/libghn.so /tmp/libghn_main.so
cp gpurun_alt/libghn_tune.so paper_2004_02290_b200/libghn.so
for q in ${QS:-160 200 230 256 290 330 400}; do
  GHN_TT_Q=$q timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --configs "" ${KS:+--ks $KS} 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TT_Q $q', {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})"
done
cp /tmp/libghn_main.so paper_2004_02290_b200/libghn.so
