#!/bin/bash
# Sweep the thread-kernel tile size (queries per tile) on the cfg4 k sweep.
for q in ${QS:-128 192 256}; do
  GHN_TT_Q=$q python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ks ${KS:-1,4,16,64} 2>gpurun_out/sw.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TT_Q', $q, 'q/s %.4g' % d['value'], {k: round(v['predict_ms'],2) for k,v in d['per_k'].items()})" || tail -3 gpurun_out/sw.err
done
