#!/bin/bash
# Bucket-select tiling sweep at k=64 (tuning build): apron, queries per tile, smallest tile.
run() {
  env "$@" timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --configs "" --ks ${KS:-64} 2> gpurun_out/sw.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})"
  grep fallbacks gpurun_out/sw.err | tail -1
}
run GHN_DEBUG_FALLBACK=1
run GHN_DEBUG_FALLBACK=1 GHN_TILE_A=4
run GHN_DEBUG_FALLBACK=1 GHN_TILE_A=4 GHN_SB_TMIN=20
run GHN_DEBUG_FALLBACK=1 GHN_TT_Q=200
run GHN_DEBUG_FALLBACK=1 GHN_TT_Q=300 GHN_SB_TMIN=22
run GHN_DEBUG_FALLBACK=1 GHN_TT_Q=340 GHN_SB_TMIN=24
run GHN_DEBUG_FALLBACK=1 GHN_SB_REDO=1
run GHN_DEBUG_FALLBACK=1 GHN_SB_REDO=4
run GHN_DEBUG_FALLBACK=1 GHN_SB_CAPN=200
run GHN_DEBUG_FALLBACK=1 GHN_SB_SORT=0
