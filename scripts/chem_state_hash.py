"""One C4-physics slow step; prints ms/step and a hash of the resulting state
(bitwise comparison of library builds selected by MR_LIB_PATH)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch

import paper_2211_03293_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = P.Context(0)
cfg, y0 = P.setup_workload(ctx, name, n=n)
best = 1e30
for rep in range(3):
    ctx.upload(y0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.mri_step(0.0, cfg["H"])
    torch.cuda.synchronize()
    best = min(best, (time.perf_counter() - t0) * 1e3)
h = hashlib.sha256(ctx.download().tobytes()).hexdigest()[:16]
print(f"{os.environ.get('MR_LIB_PATH', 'in-tree')}: {name} {n}^3 {best:.1f} ms/step state {h}")
