"""Fold gpurun_out/traffic_k*.csv (ncu per-launch metrics) into profiles/ncu_summary.json.

For each k the LAST launch of each predict kernel is the timed step's; bytes are
summed over the kernels of that step (tile kernel + fallback query_kernel)."""
import csv
import json
import sys
from collections import OrderedDict


def rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    return list(csv.DictReader(lines))


def summarize(paths_by_k, src):
    out = {"source": src, "kernel": "tile2d_thr_kernel (k <= 32: register list; k > 32: bucket select) (+ query_kernel fallback)",
           "query_kernel_dram_bytes_per_launch": {}, "ncu_duration_ms": {}, "l2_hit_pct": {},
           "branch_uniformity_pct": {}, "kernels_in_step": {}}
    for k, p in paths_by_k.items():
        launches = OrderedDict()
        for r in rows(p):
            key = (r["ID"], r["Kernel Name"])
            launches.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        # the timed step = the last launch of the main kernel and anything after it in the same predict
        items = list(launches.items())
        names = [n for (_, n), _ in items]
        # (the vote kernels; the bench's neighbour block runs tile2d_nb_kernel afterwards)
        main = [i for i, n in enumerate(names) if "tile2d_thr_kernel" in n or "tile2d_sel_kernel" in n] or \
               [i for i, n in enumerate(names) if "tile2d" in n] or list(range(len(names)))
        last = main[-1]
        step = [items[last]]
        for it in items[last + 1:]:
            if "tile2d" in it[0][1]:
                break
            if "query_kernel" in it[0][1]:
                step.append(it)
        b = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for _, m in step)
        t = sum(m.get("gpu__time_duration.sum", 0) for _, m in step)
        m0 = step[0][1]
        out["query_kernel_dram_bytes_per_launch"][k] = b
        out["ncu_duration_ms"][k] = t / 1e6 if t > 1e5 else t  # ns -> ms
        out["l2_hit_pct"][k] = m0.get("lts__t_sector_hit_rate.pct")
        out["branch_uniformity_pct"][k] = m0.get("smsp__sass_average_branch_targets_threads_uniform.pct")
        out["kernels_in_step"][k] = [n.split("(")[0] for (_, n), _ in step]
    return out


if __name__ == "__main__":
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    s = summarize({k: f"{d}/traffic_k{k}.csv" for k in ("1", "4", "16", "64")},
                  "profiles/traffic_r02_k*.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  "dram__bytes_write.sum,lts__t_sector_hit_rate.pct,branch uniformity --clock-control none; "
                  "the timed step of `bench.py --ks K --steps 1 --warmup 3`)")
    json.dump({"cfg4": s}, open("profiles/ncu_summary.json", "w"), indent=1)
    print(json.dumps(s, indent=1))
