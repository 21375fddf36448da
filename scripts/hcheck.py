"""Step-size accuracy check of the workloads: one slow step of H against two
of H/2 on the slabs through the hotspot (per-species max relative
difference), for H = H_config * f.  Usage: python scripts/hcheck.py C4 1 0.5 0.25"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_03293_b200 as P  # noqa: E402
from tests.helpers import per_species_rel_err  # noqa: E402

name = sys.argv[1]
facs = [float(a) for a in sys.argv[2:]] or [1.0]
cfg0 = P.CONFIGS[name]
N = cfg0["n"]
slabs = [(0, N)] if N <= 128 else [P.slab_bounds(N, 8, 3), P.slab_bounds(N, 8, 4)]
for f in facs:
    worst = 0.0
    for i0, n0l in slabs:
        a = P.Context(0)
        cfg, y0 = P.setup_workload(a, name, i0=i0, n0_local=n0l, threads=0)
        H = cfg["H"] * f
        try:
            a.mri_step(0.0, H)
            y1 = a.download()
            a.upload(y0)
            a.mri_step(0.0, H / 2)
            a.mri_step(H / 2, H / 2)
            worst = max(worst, per_species_rel_err(y1, a.download(), cfg["S"] + 1))
        except P.IntegrationError as e:
            worst = float("inf")
            print(f"  {name} H={H:.3g}: {e}")
        a.close()
    print(f"{name} H={cfg0['H'] * f:.3g} (x{f}): |H - 2 x H/2| = {worst:.3e}", flush=True)
