#!/bin/bash
# Bench the non-headline configs (parity-case shapes) without CPU legs; one JSON per config.
for c in ${CFGS:-0 1 2}; do
  timeout ${TMO:-600} python bench.py --config $c --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/cfg{c}.json").read())
except Exception as e:
    print("cfg", c, "FAILED", e); print(open(f"gpurun_out/cfg{c}.err").read()[-1500:]); sys.exit()
print("cfg", c, "q/s=%.4g" % d["value"], "fit ms %.2f" % d["fit"]["ms"], "frac %.3f" % d["roofline"]["frac"],
      {k: (round(v["predict_ms"], 2), round(v["mean_points_scanned"], 1)) for k, v in d["per_k"].items()})
PY
done
