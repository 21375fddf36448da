"""Copy a gpu_round.sh run (tag) into profiles/<round>/ with summaries.
Usage: python scripts/refresh_profiles.py TAG [ROUND_DIR]"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/r01"
src = "gpurun_out"
NCU = "/usr/local/cuda/bin/ncu"


def last_json(path):
    return json.loads(open(path).read().strip().split("\n")[-1])


json.dump(last_json(f"{src}/bench_{tag}.log"), open(f"{dst}/bench_c4.json", "w"), indent=1)
json.dump(last_json(f"{src}/bench_ref_{tag}.log"), open(f"{dst}/bench_reference.json", "w"), indent=1)
shutil.copy(f"{src}/launches_{tag}.csv", f"{dst}/launches_c4_256.csv")
shutil.copy(f"{src}/prof_chem_{tag}.ncu-rep", f"{dst}/chem_chain_c4_64cube.ncu-rep")
shutil.copy(f"{src}/prof_sten_{tag}.ncu-rep", f"{dst}/stencil_c4_64cube.ncu-rep")
for name, kre in [("chem_chain_c4_64cube", "chem_chain"), ("stencil_c4_64cube", "stencil")]:
    rep = f"{dst}/{name}.ncu-rep"
    out = subprocess.run([sys.executable, "scripts/ncu_summary.py", rep, kre], capture_output=True,
                         text=True).stdout
    sass = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    open("/tmp/_sass.csv", "w").write(sass)
    out += subprocess.run([sys.executable, "scripts/sass_hot.py", "/tmp/_sass.csv", "25"],
                          capture_output=True, text=True).stdout
    open(f"{dst}/{name}_summary.txt", "w").write(out)


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {a: (c, b) for a, b, c in zip(rows[0], rows[1], rows[2])}


def nbytes(x):
    v, u = x
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


tr = {}
for key, name, alg, note in [
        ("chem_chain", "chem_chain_c4_64cube", 3 * 8 * 54 * 64 ** 3,
         "first chain launch of a C4-physics step on 64^3 (reads y + 1 referenced fE, writes y)"),
        ("stencil", "stencil_c4_64cube", 2 * 8 * 54 * 64 ** 3,
         "one 8th-order stencil evaluation on 64^3 (read y, write fE_j)")]:
    d = raw(f"{dst}/{name}.ncu-rep")
    rd, wr = nbytes(d["dram__bytes_read.sum"]), nbytes(d["dram__bytes_write.sum"])
    dur, unit = d["gpu__time_duration.sum"]
    tr[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "algorithmic_bytes_per_launch": alg,
               "duration_ms": float(dur) / (1e3 if unit == "us" else 1.0),
               "source": f"{dst}/{name}.ncu-rep", "note": note}
    for k, metric in [("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                      ("lsu_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                      ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active")]:
        if metric in d:
            tr[key][k] = float(d[metric][0])
json.dump(tr, open(f"{dst}/traffic.json", "w"), indent=1)
print("profiles refreshed from", tag)
