"""Time one C4-physics slow step (ms, CUDA events) even when the step fails --
for timing-bound experiment builds whose numerics are deliberately wrong.
Usage: MR_LIB_PATH=... python scripts/chem_time.py [config] [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch

import paper_2211_03293_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
R = int(sys.argv[3]) if len(sys.argv) > 3 else None  # optional reaction-count override
S = int(sys.argv[4]) if len(sys.argv) > 4 else None  # optional species-count override
ctx = P.Context(0)
from paper_2211_03293_b200.configs import CONFIGS
config = dict(CONFIGS[name])
if R:
    config["R"] = R
if S:
    config["S"] = S
cfg, y0 = P.setup_workload(ctx, name, n=n, config=config)
best = 1e30
for rep in range(3):
    ctx.upload(y0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        ctx.mri_step(0.0, cfg["H"])
        ok = True
    except P.IntegrationError:
        ok = False
    torch.cuda.synchronize()
    best = min(best, (time.perf_counter() - t0) * 1e3)
print(f"{os.environ.get('MR_LIB_PATH', 'in-tree')}: {name} {n}^3 S={cfg['S']} R={cfg['R']} {best:.1f} ms/step (wall, best of 3), ok={ok}")
