#!/bin/bash
# Register list vs bucket select crossover (tuning build in gpurun_alt/libghn_tune.so).
cp paper_2004_02290_b200/libghn.so /tmp/libghn_main.so
cp gpurun_alt/libghn_tune.so paper_2004_02290_b200/libghn.so
for lm in 32 16 8; do
  GHN_TT_Q=${Q:-450} GHN_TT_LISTMAX=$lm timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --configs "" --ks ${KS:-12,16,20,24,32} 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LISTMAX $lm', {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})"
done
cp /tmp/libghn_main.so paper_2004_02290_b200/libghn.so
