#!/bin/bash
# GPU iteration loop: tile-path parity tests, then the cfg4 bench (no CPU legs).
python -m pytest tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -${TAILN:-2}
python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q.json 2> gpurun_out/q.err || tail -5 gpurun_out/q.err
python -c "
import json; d=json.load(open('gpurun_out/q.json'))
print('q/s %.4g' % d['value'], {k: round(v['predict_ms'], 2) for k, v in d['per_k'].items()}, 'fit', round(d['fit']['ms'], 2), d['clocks']['sm_mhz'])"
