"""Experiment driver for scripts/chem_codegen_reg.py: parity of the generated
RHS against the oracle (32^3) and RK4-chain throughput (cell-evaluations/s)
next to the production kernel's chemistry time inside a C4-physics step."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import oracle as O
import paper_2211_03293_b200 as P
from tests.helpers import per_species_rel_err

libs = sys.argv[1:] or ["/tmp/cg/libcg_I.so"]
name = "C4"
ctx = P.Context(0)

n = 32
cfg, y0 = P.setup_workload(ctx, name, n=n)
S = cfg["S"]
mech = O.mechanism(cfg["mech_seed"], S, cfg["R"])
sysm = O.System(n, n, n, S + 1, fast="chem", slow="stencil", mech=mech, S=S, R=cfg["R"],
                rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"], u=(1.0, 1.0, 1.0))
ref = sysm.fast_rhs(y0)
cur = ctx.fast_rhs(y0)
print("production kernel RHS vs oracle: %.3e" % per_species_rel_err(cur[: S * n**3], ref[: S * n**3], S))

# production kernel: chemistry ms of one C4-physics slow step at 128^3
N = 128
cfgN, yN = P.setup_workload(ctx, name, n=N)
ctx.set_profiling(True)
for rep in range(2):
    ctx.upload(yN)
    ctx.mri_step(0.0, cfgN["H"])
prof = ctx.last_step_profile()
chem_ms = prof[0]
evals = 196 * N**3
print(f"production: C4 physics {N}^3 chemistry {chem_ms:.1f} ms/step -> {evals / chem_ms * 1e3:.3e} cell-evals/s")
ctx.set_profiling(False)

for libname in libs:
    lib = C.CDLL(libname)
    lib.cg_run_rhs.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    lib.cg_run_rk4.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                               C.c_double, C.c_double, C.c_void_p]
    nc = n ** 3
    yd = torch.from_numpy(y0).cuda()
    fd = torch.zeros_like(yd)
    assert lib.cg_run_rhs(yd.data_ptr(), fd.data_ptr(), nc, None) == 0
    torch.cuda.synchronize()
    got = fd.cpu().numpy()
    print(f"{os.path.basename(libname)}: rhs vs oracle per-species rel err "
          f"{per_species_rel_err(got[: S * nc], ref[: S * nc], S):.3e}")
    for NN in (64, 128):
        nc = NN ** 3
        cfgM, yM = P.setup_workload(ctx, name, n=NN)
        y = torch.from_numpy(yM).cuda()
        ob = torch.empty_like(y)
        rc0 = torch.zeros_like(y)
        rc1 = torch.zeros_like(y)
        nsub = 49
        h = cfgM["H"] / 50
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for rep in range(3):
            yy = y.clone()
            torch.cuda.synchronize()
            ev0.record()
            assert lib.cg_run_rk4(yy.data_ptr(), ob.data_ptr(), rc0.data_ptr(), rc1.data_ptr(), nc,
                                  nsub, h, cfgM["H"], None) == 0
            ev1.record()
            torch.cuda.synchronize()
            best = min(best, ev0.elapsed_time(ev1))
        ev = nc * nsub * 4
        print(f"  N={NN}: {best:.2f} ms for {nsub} RK4 substeps -> {ev / best * 1e3:.3e} cell-evals/s; "
              f"finite={bool(torch.isfinite(yy).all())}")
