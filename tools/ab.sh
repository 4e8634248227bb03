#!/bin/bash
# A/B of two builds of libghn.so on the cfg4 bench: tools/ab.sh gpurun_alt/libghn_X.so [bench args]
ALT=$1; shift
cp paper_2004_02290_b200/libghn.so /tmp/libghn_main.so
for round in 1 2; do
  for v in main alt; do
    if [ $v = alt ]; then cp $ALT paper_2004_02290_b200/libghn.so; else cp /tmp/libghn_main.so paper_2004_02290_b200/libghn.so; fi
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --configs "" "$@" 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g' % d['value'], {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()}, 'fit', round(d['fit']['ms'],2))"
  done
done
cp /tmp/libghn_main.so paper_2004_02290_b200/libghn.so
