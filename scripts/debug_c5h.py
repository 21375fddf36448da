"""C5 step-size conditioning: is one slow step of H finite on every slab of
the 384^3 grid, and how far is it from two steps of H/2 (hotspot slab)?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_03293_b200 as P  # noqa: E402
from tests.helpers import per_species_rel_err  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
H = float(sys.argv[2]) if len(sys.argv) > 2 else None
N = P.CONFIGS[name]["n"]
for r in range(8):
    i0, n0l = P.slab_bounds(N, 8, r)
    a = P.Context(0)
    cfg, y0 = P.setup_workload(a, name, i0=i0, n0_local=n0l, threads=0)
    h = H or cfg["H"]
    try:
        a.mri_step(0.0, h)
        y1 = a.download()
        ok = bool(np.all(np.isfinite(y1)))
        line = f"{name} H={h:.3g} slab {r} ({i0}+{n0l}): finite {ok}, moved {per_species_rel_err(y1, y0, cfg['S'] + 1):.3e}"
        if r in (3, 4):
            a.upload(y0)
            a.mri_step(0.0, h / 2)
            a.mri_step(h / 2, h / 2)
            y2 = a.download()
            line += f", |H - 2 x H/2| {per_species_rel_err(y1, y2, cfg['S'] + 1):.3e}"
    except P.IntegrationError as e:
        line = f"{name} H={h:.3g} slab {r} ({i0}+{n0l}): IntegrationError {e}"
    print(line, flush=True)
    a.close()
