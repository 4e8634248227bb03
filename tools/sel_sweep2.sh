#!/bin/bash
run() {
  env "$@" timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --configs "" --ks ${KS:-64} 2> gpurun_out/sw.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})"
  grep fallbacks gpurun_out/sw.err | tail -1
}
run GHN_DEBUG_FALLBACK=1 GHN_SB_CAPN=400 GHN_SB_RECAP=400
run GHN_DEBUG_FALLBACK=1 GHN_SB_CAPN=255 GHN_SB_RECAP=400
run GHN_DEBUG_FALLBACK=1 GHN_SB_CAPN=400 GHN_SB_RECAP=255
run GHN_DEBUG_FALLBACK=1 GHN_SB_CAPN=400 GHN_SB_RECAP=400 GHN_SB_REDO=1
run GHN_DEBUG_FALLBACK=1 GHN_SB_CAPN=600 GHN_SB_RECAP=600 GHN_SB_REDO=1
