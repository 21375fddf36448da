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

# stall reasons: total, and per code region given as "lo:hi" instruction-index ranges (argv[3:])
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ridx = [ix[h] for h in reasons]
rows2 = [r for r in rows[2:] if len(r) >= len(hdr)]


def region(lo, hi):
    tot = [0] * len(reasons)
    for r in rows2[lo:hi]:
        for q, i in enumerate(ridx):
            try:
                tot[q] += int(r[i] or 0)
            except ValueError:
                pass
    return tot


specs = sys.argv[3:] or ["0:%d" % len(rows2)]
for sp in specs:
    lo, hi = (int(x) for x in sp.split(":"))
    tot = region(lo, hi)
    ssum = sum(tot) or 1
    top = sorted(zip(reasons, tot), key=lambda t: -t[1])[:8]
    print(f"\nstall reasons [{lo}:{hi}] ({ssum} samples, {100 * ssum / tot_s:.1f}% of all):")
    print("  " + ", ".join(f"{n[6:]} {100 * v / ssum:.0f}%" for n, v in top))
