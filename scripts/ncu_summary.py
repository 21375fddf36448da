"""Summarise one kernel of an ncu --set full report (metrics + stall reasons
+ SASS opcode mix) for profiles/.  Usage: python scripts/ncu_summary.py REP [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = [
    "gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
]


def raw(rep, kre):
    args = [NCU, "-i", rep, "--page", "raw", "--csv"]
    if kre:
        args += ["-k", "regex:" + kre]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    d = raw(rep, kre)
    print("kernel", d.get("Kernel Name", ("?",))[0][:120])
    for k in KEYS:
        if k in d:
            print(k, d[k])
    stalls = {k: v for k, v in d.items()
              if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")}
    if not stalls:
        stalls = {k: v for k, v in d.items() if "warps_issue_stalled_" in k and k.endswith("per_warp_active.pct")}
    for k, (v, u) in sorted(stalls.items(), key=lambda kv: -float(kv[1][0] or 0))[:14]:
        print("  stall", k.split("stalled_")[-1], v)
    pipes = {k: v for k, v in d.items() if k.startswith("sm__inst_executed_pipe_") and
             k.endswith("avg.pct_of_peak_sustained_active")}
    for k, (v, u) in sorted(pipes.items(), key=lambda kv: -float(kv[1][0] or 0))[:10]:
        print("  pipe", k[len("sm__inst_executed_pipe_"):].split(".")[0], v)


if __name__ == "__main__":
    main()
