"""Stencil (K2) throughput at full size: C4 physics with the fast partition
off, so a step is 6 stencil evaluations + cheap forcing chains; reports the
'slow' launch-class time from the per-launch events.
Usage: python scripts/sten_bench.py [CONFIG] [N] [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2211_03293_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ctx = P.Context(0)
cfg, y0 = P.setup_workload(ctx, name, n=n, threads=0)
ctx.fast_none()
N = cfg["n"]
S1 = cfg["S"] + 1
H = cfg["H"]
ctx.mri_step(0.0, H)
ctx.set_profiling(True)
slow = 0.0
evals = 0
for i in range(steps):
    cnt = ctx.mri_step(i * H, H)
    c, s, o = ctx.last_step_profile()
    slow += s
    evals += int(cnt[2]) - 1  # the final explicit evaluation is counted, not computed
bytes_ = 16.0 * S1 * N ** 3 * evals
print(f"{name} {N}^3 order {cfg['order']}: {evals} stencil evals, {slow / evals:.3f} ms each, "
      f"{bytes_ / (slow * 1e-3) / 1e9:.0f} GB/s ({bytes_ / (slow * 1e-3) / 6.5389e12 * 100:.1f}% of the measured 6538.9)")
