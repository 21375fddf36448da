"""Per-CUDA-source-line stall samples of an ncu report (source page,
cuda,sass view).  Usage: python scripts/ncu_cuda_lines.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, lines, hdr = "?", [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ei = hdr.index("Instructions Executed")
        continue
    if hdr is None or not r[0]:
        continue
    try:
        s = int(r[si] or 0)
        e = int(r[ei] or 0)
    except (ValueError, IndexError):
        continue
    lines.append((s, e, fname, r[0], r[1].strip()[:90]))
tot = sum(l[0] for l in lines) or 1
print(f"{rep}: {tot} stall samples")
for s, e, f, ln, src in sorted(lines, reverse=True)[:N]:
    print(f"{100 * s / tot:5.1f}%  {e:>12d}  {f}:{ln:<5s} {src}")
