"""Generate the golden fixtures of tests/golden/ with the REFERENCE's own
stepper (oracle/_ref: /root/reference/proj/src compiled unmodified, driving
the builder's physics callbacks through its PartitionedSystem).

Run here, where /root/reference exists:  python -m tests.golden.make_golden
The fixtures then pin the C restatement (oracle/mri_oracle.c) and the GPU
path on the GPU box, where /root/reference does not exist.
"""
import json
import os

import numpy as np

import oracle as O
from paper_2211_03293_b200.configs import CONFIGS, stage_solver

HERE = os.path.dirname(os.path.abspath(__file__))

# LinearTwoRateOde::default_problem (proj/src/models.cpp:65-73)
A_FAST = np.array([[0.0, 4.0], [-4.0, 0.0]])
A_SI = np.array([[-1.0, 0.2], [0.3, -0.7]])
A_SE = np.array([[0.1, 0.4], [-0.3, -0.1]])
Y0_LIN = np.array([1.0, 0.6])


def physics_system(name, n, **kw):
    cfg = dict(CONFIGS[name], **kw.get("override", {}))
    S, R = cfg["S"], cfg["R"]
    mech = O.mechanism(cfg["mech_seed"], S, R)
    prof = O.velocity_profiles(cfg["vel_seed"], n, n, n) if cfg["velocity"] == "random" else None
    imex = cfg.get("d_impl") is not None

    def make(**extra):
        return O.System(n, n, n, S + 1, fast=kw.get("fast", "chem"), slow="stencil", mech=mech,
                        S=S, R=R, rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"],
                        u=cfg["u"] or (1.0, 1.0, 1.0), prof=prof, imex=imex,
                        d_impl=cfg.get("d_impl") or 0.0, cg_iters=cfg.get("cg_iters") or 0,
                        **extra)
    sysm = make()
    if imex:  # the ImplicitStageSolver is configured from the initial state
        tol, safety, mx, w = stage_solver(sysm.initial_condition(cfg["ic_seed"]))
        sysm = make(newton=(tol, safety, mx), newton_weights=w)
    return cfg, sysm


def main():
    out = {}
    meta = {}
    couplings = {n: open(os.path.join(HERE, "couplings", f"{n}.txt")).read()
                 for n in ["mis-kw3", "imex-mri-gark4-explicit", "imex-mri-gark3b", "imex-mri-gark4"]}

    # 1. reacting-flow workloads on 8^3 with each config's physics and method
    # (C5: the reference's ImplicitSolve runs its own Newton-GMRES; counters
    # n_linear_iters / n_precond_solves then describe GMRES, not the PCG)
    for name, steps in [("C1", 2), ("C2", 2), ("C3", 1), ("C4", 1), ("C5", 1)]:
        n = 8
        cfg, sysm = physics_system(name, n)
        y0 = sysm.initial_condition(cfg["ic_seed"])
        cp = couplings[cfg["coupling"]] if cfg["coupling"] != "mis-kw3" else "mis-kw3"
        H = cfg["H"]
        y, cnt = sysm.mri_integrate(cp, cfg["fast_table"], cfg["m"], 0.0, steps * H, H, y0,
                                    use_reference=True)
        out[f"{name}_n8_y"] = y
        out[f"{name}_n8_counters"] = cnt
        meta[f"{name}_n8"] = dict(steps=steps, H=H, n=n)
        print(name, "counters", cnt.tolist())

    # 2. reaction-off transport run with a transport-scale H (stencil visible)
    cfg, sysm = physics_system("C3", 12, fast="none")
    y0 = sysm.initial_condition(cfg["ic_seed"])
    H = 2e-4
    y, cnt = sysm.mri_integrate(couplings["imex-mri-gark4-explicit"], "classic-rk4", 4, 0.0, 3 * H,
                                H, y0, use_reference=True)
    out["transport_n12_y"] = y
    out["transport_n12_counters"] = cnt
    meta["transport_n12"] = dict(H=H, steps=3, m=4, config="C3", fast="none")

    # 2b. IMEX reaction-off run: stiff enough that the implicit diffusion solve
    #     is visible (gamma D sum 2/dx^2 ~ 0.1); one Newton iteration per solve
    #     with the PCG converged at 8 iterations
    over = dict(d_impl=0.05, cg_iters=8)
    cfg, sysm = physics_system("C5", 12, fast="none", override=over)
    y0 = sysm.initial_condition(cfg["ic_seed"])
    H = 2e-3
    y, cnt = sysm.mri_integrate(couplings["imex-mri-gark3b"], "kutta3", 4, 0.0, 3 * H, H, y0,
                                use_reference=True)
    out["imex_transport_n12_y"] = y
    out["imex_transport_n12_counters"] = cnt
    meta["imex_transport_n12"] = dict(H=H, steps=3, m=4, config="C5", fast="none", **over)

    # 2c. reference_solution (erk.cpp:59-75): cash-karp5 on the summed RHS
    for key, name, fast, h, nst, over in [
            ("refsol_C1_n8", "C1", "chem", 2e-17, 10, {}),
            ("refsol_C3_n8", "C3", "none", 2e-4, 5, {}),
            ("refsol_C5_n8", "C5", "none", 2e-4, 5, dict(d_impl=0.05, cg_iters=8))]:
        cfg, sysm = physics_system(name, 8, fast=fast, override=over)
        y0 = sysm.initial_condition(cfg["ic_seed"])
        out[key + "_y"] = sysm.reference_solution(0.0, nst * h, h, y0, use_reference=True)
        meta[key] = dict(config=name, fast=fast, h_ref=h, steps=nst, **over)

    # 2d. ark_imex_integrate (mri.cpp:437-557), ARK4(3)6L[2]SA on the C5 split
    for key, fast, H, nst, over in [
            ("ark_transport_n8", "none", 2e-3, 3, dict(d_impl=0.05, cg_iters=8)),
            ("ark_C5_n8", "chem", 3e-17, 2, {})]:
        cfg, sysm = physics_system("C5", 8, fast=fast, override=over)
        y0 = sysm.initial_condition(cfg["ic_seed"])
        y, cnt = sysm.ark_imex_integrate(0.0, nst * H, H, y0, use_reference=True)
        out[key + "_y"] = y
        out[key + "_counters"] = cnt
        meta[key] = dict(fast=fast, H=H, steps=nst, d_impl=cfg["d_impl"], cg_iters=cfg["cg_iters"])
        print(key, "counters", cnt.tolist())

    # 3. LinearTwoRateOde per cell through the reference mri_integrate
    for cp_name, table, m in [("mis-kw3", "bogacki-shampine3", 10),
                              ("imex-mri-gark4-explicit", "classic-rk4", 10)]:
        spec = cp_name if cp_name == "mis-kw3" else couplings[cp_name]
        lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=A_FAST, slow_A=A_SI + A_SE)
        for H in (0.1, 0.05):
            y, cnt = lin.mri_integrate(spec, table, m, 0.0, 1.0, H, Y0_LIN, use_reference=True)
            out[f"lin_{cp_name}_{H}_y"] = y
            out[f"lin_{cp_name}_{H}_counters"] = cnt
    np.savez_compressed(os.path.join(HERE, "ref_fixtures.npz"), **out)
    with open(os.path.join(HERE, "ref_fixtures.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
