"""Hot-spot view of an ncu source page (SASS): per-instruction stall samples
and executed counts, plus opcode totals.  Usage: python scripts/sass_hot.py CSV [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((r[ix["Address"]], r[ix["Source"]].strip(), int(r[ix["Warp Stall Sampling (All Samples)"]]),
                     int(r[ix["Instructions Executed"]] or 0)))
    except ValueError:
        continue
tot_s = sum(d[2] for d in data) or 1
tot_i = sum(d[3] for d in data) or 1
op_s, op_i = defaultdict(int), defaultdict(int)
for a, src, s, i in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    op_s[op] += s
    op_i[op] += i
print("opcode  exec%  stall%")
for op in sorted(op_i, key=lambda o: -op_i[o])[:25]:
    print(f"{op:8s} {100 * op_i[op] / tot_i:5.1f} {100 * op_s[op] / tot_s:5.1f}")
print("\nhottest instructions (stall samples):")
order = sorted(range(len(data)), key=lambda k: -data[k][2])[:N]
for k in sorted(order):
    a, src, s, i = data[k]
    print(f"{k:5d} {100 * s / tot_s:5.2f}% {i:>12d}  {src[:90]}")
