#!/bin/bash
# Bucket-select (k > 32) lock-step limits: GHN_SB_CAPN / GHN_SB_REDO / GHN_SB_WMAX sweep at k=64.
for cfg in ${CFGS:-"255 1 0" "255 2 0" "255 4 0" "320 2 0" "400 2 0"}; do
  set -- $cfg
  GHN_SB_CAPN=$1 GHN_SB_REDO=$2 GHN_SB_WMAX=$3 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ks 64 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('capn redo wmax', '$cfg', {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})"
done
