"""Per-region instruction / stall totals of a kernel from an ncu report's source page.
usage: ncu_regions.py REPORT.ncu-rep SOURCE.cuh nq 'name=marker text' ...   (markers in file order)"""
import csv
import subprocess
import sys

rep, srcpath, nq = sys.argv[1], sys.argv[2], float(sys.argv[3])
marks_in = [m.split("=", 1) for m in sys.argv[4:]]
import os
out = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, cwd="/tmp").stdout
src = open(srcpath).read().split("\n")
base = srcpath.split("/")[-1]


def find(s):
    for i, l in enumerate(src):
        if s in l:
            return i + 1
    raise SystemExit(f"marker not found: {s}")


marks = [(n, find(t)) for n, t in marks_in] + [("end", len(src) + 1)]
rows, f = [], None
for r in csv.reader(out.split("\n")):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    try:
        ins, st, ln = float(r[7]), float(r[4]), int(r[0])
    except (ValueError, IndexError):
        continue
    rows.append((ins, st, f, ln, r[1].strip()[:90]))
tot = sum(r[0] for r in rows)
ts = sum(r[1] for r in rows)
agg = {}
for ins, st, f, ln, _ in rows:
    name = f
    if f == base:
        name = "(before first marker)"
        for (n, l), (_, l2) in zip(marks, marks[1:]):
            if l <= ln < l2:
                name = n
    a = agg.setdefault(name, [0, 0])
    a[0] += ins
    a[1] += st
print(f"total warp instructions {tot:.4g} = {tot / nq:.1f} per query")
for n, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:30s} {i / nq:7.1f}/q {100 * i / tot:5.1f}%  stall {100 * s / ts:5.1f}%")
if "--lines" in sys.argv or True:
    print("-- top lines")
    for ins, st, f, ln, text in sorted(rows, key=lambda x: -x[0])[:28]:
        print(f"{ins / nq:6.1f}/q {100 * ins / tot:5.1f}% st{100 * st / ts:5.1f}%  {f}:{ln}  {text}")
