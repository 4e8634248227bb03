"""Fold gpurun_out/launches_cfg{0..3}.csv (tools/config_launches.sh) into profiles/ncu_configs_r02.json:
per config the predict kernel of the timed step (its last launch: duration, DRAM bytes) and the
run's kernels by total time."""
import csv
import json
import sys
from collections import OrderedDict

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                 "on `bench.py --config C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --configs none` "
                 "(tools/config_launches.sh; cold-cache, serialised launches: compare shares)"}
for c in range(4):
    try:
        lines = [ln for ln in open(f"{d}/launches_cfg{c}.csv") if ln.startswith('"')]
    except OSError:
        continue
    launches = OrderedDict()
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    for r in csv.DictReader(lines):
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= scale.get(r["Metric Unit"], 1.0)   # -> microseconds
        elif r["Metric Unit"] in ("Kbyte", "Mbyte", "Gbyte"):
            v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["Metric Unit"]]
        launches.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = v
    items = [(n.split("(")[0].replace("void ", "").replace("ghn::<unnamed>::", ""), m) for (_, n), m in launches.items()]

    def us(m):
        return m.get("gpu__time_duration.sum", 0.0)

    agg = {}
    for n, m in items:
        a = agg.setdefault(n, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += us(m)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tiled = [(n, m) for n, m in items if n.startswith("tile2d_")]
    pred = tiled or [(n, m) for n, m in items if n.startswith("query_kernel")]
    last = pred[-1] if pred else None
    out[f"cfg{c}"] = {
        "predict_kernel": None if last is None else {
            "name": last[0], "us": round(us(last[1]), 1),
            "dram_bytes": last[1].get("dram__bytes_read.sum", 0) + last[1].get("dram__bytes_write.sum", 0)},
        "kernels_by_time": [{"name": n, "launches": a[0], "total_us": round(a[1], 1), "dram_bytes": a[2]}
                            for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:8]],
    }
json.dump(out, open("profiles/ncu_configs_r02.json", "w"), indent=1)
for k, v in out.items():
    if k != "source":
        print(k, v["predict_kernel"], [(x["name"][:28], x["total_us"]) for x in v["kernels_by_time"][:4]])
