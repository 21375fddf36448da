"""Chemistry-kernel phase breakdown (needs an MR_PHASE_PROF build selected by
MR_LIB_PATH).  Usage: MR_LIB_PATH=variants/prof/libmri_b200.so python scripts/phase_prof.py [CONFIG] [N]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2211_03293_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
R = int(sys.argv[3]) if len(sys.argv) > 3 else None  # optional reaction-count override
ctx = P.Context(0)
from paper_2211_03293_b200.configs import CONFIGS
config = dict(CONFIGS[name])
if R:
    config["R"] = R
cfg, y0 = P.setup_workload(ctx, name, n=n, config=config)
L = P.lib()
f = L.mr_debug_chem_phases
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int]
out = (C.c_uint64 * 8)()
ctx.mri_step(0.0, cfg["H"])
f(ctx.h, out, 1)
cnt = ctx.mri_step(cfg["H"], cfg["H"])
assert f(ctx.h, out, 0) == 0
v = np.array(list(out), dtype=np.float64)
blocks = float((n ** 3 + 31) // 32)  # grid blocks; v[7] counts block launches over all chains
evals = int(cnt[0]) // 1  # per cell
names = ["rk bookkeeping / wait", "energy partials + barrier", "temperature (warp 0)",
         "species rows", "reactions", "production (warp 0)", "kernel total"]
tot_phase = v[:6].sum()
print(f"{name} n={n} R={cfg['R']}: grid blocks={blocks:.0f}, block launches={v[7]:.0f}, fast evals/cell/step={evals}")
for i, nm in enumerate(names):
    per = v[i] / blocks / max(evals, 1)
    share = v[i] / v[6] if i < 6 else 1.0
    print(f"  {nm:28s} {per:9.1f} cyc/eval/block  {100 * share:5.1f}%")
