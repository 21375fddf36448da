"""Build profiles/<round>/traffic.json (read by bench.py's roofline.traffic)
from ncu --set full captures taken AT THE BENCHED GRID SIZE.

Usage: python scripts/traffic_json.py OUT.json KEY REP GRID ALG_BYTES NOTE [KEY REP GRID ALG NOTE ...]
  KEY        chem_chain | stencil
  ALG_BYTES  algorithmic DRAM bytes of the captured launch
"""
import csv
import io
import json
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {a: (c, b) for a, b, c in zip(rows[0], rows[1], rows[2])}


def nbytes(x):
    v, u = x
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


out_path = sys.argv[1]
tr = json.load(open(out_path)) if os.path.exists(out_path) else {}
args = sys.argv[2:]
for i in range(0, len(args), 5):
    key, rep, grid, alg, note = args[i:i + 5]
    d = raw(rep)
    rd, wr = nbytes(d["dram__bytes_read.sum"]), nbytes(d["dram__bytes_write.sum"])
    dur, unit = d["gpu__time_duration.sum"]
    e = {"grid": int(grid), "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
         "algorithmic_bytes_per_launch": float(alg),
         "dram_over_algorithmic": (rd + wr) / float(alg),
         "duration_ms": float(dur) / {"us": 1e3, "ms": 1.0, "s": 1e-3}.get(unit, 1.0),
         "source": rep, "note": note}
    for k, metric in [("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                      ("lsu_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                      ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                      ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")]:
        if metric in d:
            e[k] = float(d[metric][0])
    tr[key] = e
json.dump(tr, open(out_path, "w"), indent=1)
print(json.dumps(tr, indent=1))
