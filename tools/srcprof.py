"""Per-source-line instruction / stall-sample totals from `ncu -i R --page source --csv --print-source cuda,sass`."""
import csv
import sys

path, nq = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = []
f = None
tot_i = tot_s = 0
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        ins = float(r[7]); st = float(r[4])
    except (ValueError, IndexError):
        continue
    tot_i += ins; tot_s += st
    rows.append((ins, st, f, r[0], r[1].strip()[:90]))
print(f"total warp instr/query {tot_i / nq:.0f}, stall samples {tot_s:.0f}")
for ins, st, f, ln, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{ins / nq:7.1f} ins/q {100 * st / tot_s:5.1f}% stall  {f}:{ln}  {src}")
