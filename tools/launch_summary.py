"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per
kernel): the second half of the launches (the measured repetition)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
agg = {}
for r in rows[1:]:
    agg.setdefault((int(r[ii]), r[ki][:70]), {})[r[mi]] = float(r[vi].replace(",", ""))
items = sorted(agg.items())
if len(sys.argv) < 3 or sys.argv[2] != "all":
    items = items[len(items) // 2:]
tot_t = 0.0
for (i, k), m in items:
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    tot_t += t
    print("%8.1f us  R %7.3f GB  W %7.3f GB  %s" % (t, m.get("dram__bytes_read.sum", 0) / 1e9,
                                                  m.get("dram__bytes_write.sum", 0) / 1e9, k))
print("total %.1f us" % tot_t)
