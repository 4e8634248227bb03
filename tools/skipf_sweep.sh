#!/bin/bash
cp paper_2004_02290_b200/libghn.so /tmp/libghn_main.so
cp gpurun_alt/libghn_tune.so paper_2004_02290_b200/libghn.so
for f in ${FS:-0.8 0.7 0.6 0.5}; do
  GHN_DEBUG_FALLBACK=1 GHN_SB_SKIPF=$f timeout 200 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --configs none --ks ${KS:-64} 2>gpurun_out/sk.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SKIPF $f', {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})"
  grep "ghn\]" gpurun_out/sk.err | tail -2
done
cp /tmp/libghn_main.so paper_2004_02290_b200/libghn.so
