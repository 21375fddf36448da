"""Experiment driver: parity of the generated chemistry RHS against the oracle
and RK4-chain throughput (cell-evaluations/s)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import torch

import oracle as O
import paper_2211_03293_b200 as P
from tests.helpers import per_species_rel_err

libname = sys.argv[1] if len(sys.argv) > 1 else "libcg_a.so"
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), libname))
lib.cg_run_rhs.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
lib.cg_run_rk4.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                           C.c_double, C.c_double, C.c_void_p]

name = "C4"
n = 32
ctx = P.Context(0)
cfg, y0 = P.setup_workload(ctx, name, n=n)
S = cfg["S"]
mech = O.mechanism(cfg["mech_seed"], S, cfg["R"])
sysm = O.System(n, n, n, S + 1, fast="chem", slow="stencil", mech=mech, S=S, R=cfg["R"],
                rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"], u=(1.0, 1.0, 1.0))
ref = sysm.fast_rhs(y0)
nc = n ** 3
yd = torch.from_numpy(y0).cuda()
fd = torch.zeros_like(yd)
assert lib.cg_run_rhs(yd.data_ptr(), fd.data_ptr(), nc, None) == 0
torch.cuda.synchronize()
got = fd.cpu().numpy()
print("cg rhs vs oracle: per-species rel err %.3e" % per_species_rel_err(got[: S * nc], ref[: S * nc], S))
cur = ctx.fast_rhs(y0)
print("current kernel vs oracle: %.3e" % per_species_rel_err(cur[: S * nc], ref[: S * nc], S))

# throughput: one fast IVP of nsub RK4 substeps (4 evals each) per cell
for N in (64, 128):
    nc = N ** 3
    cfgN, yN = P.setup_workload(ctx, name, n=N)
    y = torch.from_numpy(yN).cuda()
    ob = torch.empty_like(y)
    rc0 = torch.zeros_like(y)
    rc1 = torch.zeros_like(y)
    nsub = 49
    h = cfg["H"] / 50
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        yy = y.clone()
        torch.cuda.synchronize()
        ev0.record()
        assert lib.cg_run_rk4(yy.data_ptr(), ob.data_ptr(), rc0.data_ptr(), rc1.data_ptr(), nc, nsub, h,
                              cfg["H"], None) == 0
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    evals = nc * nsub * 4
    print(f"N={N}: {ms:.2f} ms for {nsub} RK4 substeps -> {evals / ms * 1e3:.3e} cell-evals/s; "
          f"finite={bool(torch.isfinite(yy).all())}")
