"""Workload definitions for BASELINE.json configs C1-C5.

Seeds are fixed here (BASELINE.json gives none), as the reference records its
`seed` in summary.json (proj/src/harness.cpp:669-675).  H is chosen from the
chemistry's stiffness by oracle/stiffness.py (h * lambda_max = 1 for the inner
RK4 at t = 0) -- BASELINE.json does not state it.

Coupling stand-ins: "MRI-GARK-ERK33" -> the reference's
registered ``mis-kw3``; "MRI-GARK-ERK45a" -> ``imex-mri-gark4-explicit``, the
explicit projection of the reference's ``imex-mri-gark4`` exported/imported
through the reference's own audit format (data/couplings/).
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
               fast_table="classic-rk4", m=50, steps=4, rho=1e-3, H=3.6e-15, ngpu=(1, 2, 4, 8)),
}
