"""Diagnose C5 physics parity vs the oracle at n^3: per-component errors and counters."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_03293_b200 as P  # noqa: E402
from tests.helpers import oracle_system  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [32, 64]:
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C5", n=n, threads=0)
    sysm = oracle_system(cfg, n, y0=y0)
    sysm.set_threads(os.cpu_count() or 1)
    H = cfg["H"]
    y_ref, c_ref = sysm.mri_step(P.coupling_text(cfg["coupling"]), cfg["fast_table"], cfg["m"], 0.0, H, y0)
    c = ctx.mri_step(0.0, H)
    y = ctx.download()
    S1 = cfg["S"] + 1
    d = np.abs(y - y_ref).reshape(S1, -1).max(axis=1) / np.abs(y_ref).reshape(S1, -1).max(axis=1)
    mv = np.abs(y_ref - y0).reshape(S1, -1).max(axis=1) / np.abs(y0).reshape(S1, -1).max(axis=1)
    k = int(np.argmax(d))
    print(f"n={n} counters gpu {c.tolist()} oracle {c_ref.tolist()}")
    print(f"  worst comp {k} err {d[k]:.3e}; errs[:5] {np.array2string(d[:5], precision=2)} energy {d[-1]:.2e}")
    print(f"  step moved comps by up to {mv.max():.2e} (energy {mv[-1]:.2e})")
    yk, rk = y.reshape(S1, -1)[k], y_ref.reshape(S1, -1)[k]
    i = int(np.argmax(np.abs(yk - rk)))
    print(f"  worst cell {i} (i,j,k)={np.unravel_index(i, (n, n, n))} gpu {yk[i]:.17e} ref {rk[i]:.17e} y0 {y0.reshape(S1,-1)[k][i]:.6e}")
    ctx.close()
