"""C5 step-size conditioning: parity vs the oracle at 64^3 for H, H/2, H/4, and
the H vs 2 x H/2 difference on one 48-plane slab of the 384^3 grid."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_03293_b200 as P  # noqa: E402
from tests.helpers import oracle_system, per_species_rel_err  # noqa: E402

n = 64
for div in [1, 2, 4]:
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C5", n=n, threads=0)
    H = cfg["H"] / div
    sysm = oracle_system(cfg, n, y0=y0)
    sysm.set_threads(os.cpu_count() or 1)
    y_ref, c_ref = sysm.mri_step(P.coupling_text(cfg["coupling"]), cfg["fast_table"], cfg["m"], 0.0, H, y0)
    c = ctx.mri_step(0.0, H)
    y = ctx.download()
    print(f"64^3 H/{div}: err {per_species_rel_err(y, y_ref, cfg['S'] + 1):.3e} moved "
          f"{per_species_rel_err(y_ref, y0, cfg['S'] + 1):.3e} counters {c.tolist()} / {c_ref.tolist()}", flush=True)
    ctx.close()
for name, slab in [("C5", (384, 8)), ("C4", (256, 8))]:
    N, P_ = slab
    i0, n0l = P.slab_bounds(N, P_, P_ // 2)
    for div in [1, 2]:
        a = P.Context(0)
        cfg, y0 = P.setup_workload(a, name, i0=i0, n0_local=n0l, threads=0)
        H = cfg["H"] / div
        a.mri_step(0.0, H)
        y1 = a.download()
        a.upload(y0)
        a.mri_step(0.0, H / 2)
        a.mri_step(H / 2, H / 2)
        y2 = a.download()
        print(f"{name} slab {i0}+{n0l} of {N}^3, H/{div}: |one step - two half steps| rel {per_species_rel_err(y1, y2, cfg['S'] + 1):.3e}"
              f", moved {per_species_rel_err(y2, y0, cfg['S'] + 1):.3e}", flush=True)
        a.close()
