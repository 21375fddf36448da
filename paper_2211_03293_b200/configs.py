"""Workload definitions for BASELINE.json configs C1-C5.

Seeds are fixed here (BASELINE.json gives none), as the reference records its
`seed` in summary.json (proj/src/harness.cpp:669-675).  H is chosen from the
chemistry's stiffness by oracle/stiffness.py (h * lambda_max = 1 for the inner
RK4 at t = 0) -- BASELINE.json does not state it -- and then checked on the
GPU over the whole grid by step halving (scripts/hcheck.py: one step of H vs
two of H/2 on the slabs through the hotspot, per-species max relative
difference).  The sampled lambda_max missed the stiffest cells of C4 and C5:
at 3.6e-15 / 6.7e-15 the hotspot cells differed by O(1) (C5 even overflowed),
so their H was halved to 1.8e-15 / 3.3e-15 (differences 1.3e-6 / 3.1e-6;
C1-C3: <= 1.5e-5 at their H).  A step's cost does not depend on H.

Coupling stand-ins: "MRI-GARK-ERK33" -> the reference's
registered ``mis-kw3``; "MRI-GARK-ERK45a" -> ``imex-mri-gark4-explicit``, the
explicit projection of the reference's ``imex-mri-gark4`` exported/imported
through the reference's own audit format (data/couplings/).  C5 uses the
reference's own IMEX ``imex-mri-gark3b`` + ``kutta3``: slow-explicit 8th-order
advection (``diffusion`` = 0 in the explicit stencil) and slow-implicit
diffusion ``d_impl`` solved by ``cg_iters`` Jacobi-PCG iterations.
"""

CONFIGS = {
    "C1": dict(n=32, S=9, R=21, mech_seed=20221103, ic_seed=1, vel_seed=0, velocity="uniform",
               u=(1.0, 1.0, 1.0), order=2, diffusion=1e-3, coupling="mis-kw3",
               fast_table="classic-rk4", m=10, steps=10, rho=1e-3, H=5.9e-16, ngpu=(1,)),
    "C2": dict(n=64, S=9, R=21, mech_seed=20221103, ic_seed=2, vel_seed=0, velocity="uniform",
               u=(1.0, 1.0, 1.0), order=4, diffusion=1e-3, coupling="imex-mri-gark4-explicit",
               fast_table="classic-rk4", m=20, steps=20, rho=1e-3, H=9.7e-16, ngpu=(1,)),
    "C3": dict(n=128, S=21, R=84, mech_seed=20221104, ic_seed=3, vel_seed=33, velocity="random",
               u=None, order=8, diffusion=1e-3, coupling="imex-mri-gark4-explicit",
               fast_table="classic-rk4", m=50, steps=4, rho=1e-3, H=1.4e-15, ngpu=(1, 2, 4)),
    "C4": dict(n=256, S=53, R=325, mech_seed=20221105, ic_seed=4, vel_seed=44, velocity="random",
               u=None, order=8, diffusion=1e-3, coupling="imex-mri-gark4-explicit",
               fast_table="classic-rk4", m=50, steps=4, rho=1e-3, H=1.8e-15, ngpu=(1, 2, 4, 8)),
    "C5": dict(n=384, S=53, R=325, mech_seed=20221105, ic_seed=5, vel_seed=55, velocity="random",
               u=None, order=8, diffusion=0.0, d_impl=5e-3, cg_iters=4,
               coupling="imex-mri-gark3b", fast_table="kutta3", m=100, steps=4, rho=1e-3,
               H=3.3e-15, ngpu=(8,)),
}


def stage_solver(y0, ymax=None):
    """ImplicitStageSolver settings of the IMEX workloads (mri.hpp:84-95):
    NewtonConfig tolerance 1e-12, safety 1, max_iters 5 and WRMS weights
    1 / (|y0_i| + 1e-300 + 1e-3 max|y0|), fixed from the initial state (max
    over the GLOBAL state: a slab passes the all-reduced ``ymax``).  The
    reference's absolute defaults (solvers.hpp:19-23) cannot converge on a
    state whose energy component is ~1e10.  Returns (tol, safety, max, w)."""
    import numpy as np
    y0 = np.asarray(y0, dtype=np.float64)
    if ymax is None:
        ymax = float(np.abs(y0).max()) if y0.size else 0.0
    w = 1.0 / (np.abs(y0) + 1e-300 + 1e-3 * ymax)
    return 1e-12, 1.0, 5, w
