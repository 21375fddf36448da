"""Shared test helpers (reference idioms)."""
import numpy as np


def per_species_rel_err(y, ref, ncomp):
    """max over species of max|y - ref| / max|ref| -- the idiom of
    proj/tests/test_mri.cpp:255 with max_norm_component per species."""
    y = np.asarray(y).reshape(ncomp, -1)
    ref = np.asarray(ref).reshape(ncomp, -1)
    worst = 0.0
    for k in range(ncomp):
        scale = np.abs(ref[k]).max()
        d = np.abs(y[k] - ref[k]).max()
        worst = max(worst, d / scale if scale > 0 else d)
    return worst


# LinearTwoRateOde::default_problem (proj/src/models.cpp:65-73)
A_FAST = np.array([[0.0, 4.0], [-4.0, 0.0]])
A_SI = np.array([[-1.0, 0.2], [0.3, -0.7]])
A_SE = np.array([[0.1, 0.4], [-0.3, -0.1]])
Y0_LIN = np.array([1.0, 0.6])


def expm_taylor(A, t):
    """analytic_solution (proj/src/models.cpp:75-100) in numpy."""
    a = np.array(A, dtype=float) * t
    sq = 0
    while np.abs(a).sum(axis=1).max() > 0.25:
        a *= 0.5
        sq += 1
    res = np.eye(len(a))
    term = np.eye(len(a))
    for k in range(1, 25):
        term = term @ a / k
        res = res + term
        if np.abs(term).sum(axis=1).max() < 1e-20:
            break
    for _ in range(sq):
        res = res @ res
    return res


def oracle_system(cfg, n, fast="chem", n0=None, i0=0, y0=None):
    """Oracle PartitionedSystem of a workload config on an n^3 grid (or the
    slab [i0, i0+n0) of it).  IMEX configs (d_impl set) get the implicit
    partition and, when y0 is given, the workload's ImplicitStageSolver
    (configs.stage_solver) -- the same settings the device context uses."""
    import oracle as O
    from paper_2211_03293_b200.configs import stage_solver

    S, R = cfg["S"], cfg["R"]
    mech = O.mechanism(cfg["mech_seed"], S, R)
    prof = O.velocity_profiles(cfg["vel_seed"], n, n, n) if cfg["velocity"] == "random" else None
    kw = {}
    if cfg.get("d_impl") is not None:
        kw = dict(imex=True, d_impl=cfg["d_impl"], cg_iters=cfg["cg_iters"])
        if y0 is not None:
            tol, safety, mx, w = stage_solver(y0)
            kw.update(newton=(tol, safety, mx), newton_weights=w)
    return O.System(n if n0 is None else n0, n, n, S + 1, fast=fast, slow="stencil", mech=mech,
                    S=S, R=R, rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"],
                    u=cfg["u"] or (1.0, 1.0, 1.0), prof=prof, n0_global=n, i0_global=i0, **kw)


def solver_counts_ok(cnt, ref, cg_iters):
    """Counters of an IMEX run against the reference's (Newton-GMRES): equal
    except n_linear_iters / n_precond_solves, which count the PCG:
    cg_iters and cg_iters + 1 per Newton iteration."""
    cnt = np.asarray(cnt, dtype=np.int64)
    ref = np.asarray(ref, dtype=np.int64)
    same = [0, 1, 2, 3, 4, 7]
    nl = cnt[4]
    return (np.array_equal(cnt[same], ref[same]) and cnt[5] == nl * cg_iters
            and cnt[6] == nl * (cg_iters + 1))
