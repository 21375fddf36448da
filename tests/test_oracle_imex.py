"""CPU: the IMEX restatement (config C5: imex-mri-gark3b, slow-implicit
diffusion) pinned against the reference's own stepper.

The reference solves each ImplicitSolve stage with newton_solve + GMRES
(proj/src/solvers.cpp:34-208); the restatement runs the same Newton
iteration with a fixed-iteration Jacobi-PCG as the linear solver (SURVEY.md
8(f)), so results agree to the linear-solver tolerance, not bitwise, and the
n_linear_iters / n_precond_solves counters describe the PCG.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2211_03293_b200.configs import CONFIGS
from tests.helpers import oracle_system, per_species_rel_err, solver_counts_ok

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIX = dict(np.load(os.path.join(GOLD, "ref_fixtures.npz")))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))
GARK3B = open(os.path.join(GOLD, "couplings", "imex-mri-gark3b.txt")).read()


def imex_case(n, fast="chem", **over):
    cfg = dict(CONFIGS["C5"], **over)
    y0 = oracle_system(cfg, n, fast=fast).initial_condition(cfg["ic_seed"])
    return cfg, oracle_system(cfg, n, fast=fast, y0=y0), y0


def test_c5_fixture():
    """C5 physics on 8^3: at the chemistry-limited H the Newton residual at
    Y = known is already below tolerance (zero Newton iterations), exactly as
    in the reference -> bitwise equal, all counters equal."""
    meta = META["C5_n8"]
    cfg, sysm, y0 = imex_case(8)
    H = meta["H"]
    y, cnt = sysm.mri_integrate(GARK3B, cfg["fast_table"], cfg["m"], 0.0, meta["steps"] * H, H, y0)
    assert np.array_equal(cnt, FIX["C5_n8_counters"])
    assert np.array_equal(y, FIX["C5_n8_y"])


def test_imex_transport_fixture():
    """Reaction-off IMEX run where each solve takes one Newton iteration."""
    meta = META["imex_transport_n12"]
    cfg, sysm, y0 = imex_case(12, fast="none", d_impl=meta["d_impl"], cg_iters=meta["cg_iters"])
    H = meta["H"]
    y, cnt = sysm.mri_integrate(GARK3B, "kutta3", meta["m"], 0.0, meta["steps"] * H, H, y0)
    assert solver_counts_ok(cnt, FIX["imex_transport_n12_counters"], meta["cg_iters"])
    assert cnt[4] == cnt[3] > 0  # one Newton iteration per solve
    assert per_species_rel_err(y, FIX["imex_transport_n12_y"], cfg["S"] + 1) <= 1e-13
    # implicit diffusion visibly changed the state
    assert per_species_rel_err(y, y0, cfg["S"] + 1) > 1e-2
    # advection and the periodic Laplacian (and every CG Krylov vector) conserve totals
    S1 = cfg["S"] + 1
    tot0, tot = y0.reshape(S1, -1).sum(axis=1), y.reshape(S1, -1).sum(axis=1)
    assert np.all(np.abs(tot - tot0) <= 1e-12 * np.abs(tot0))


def test_unconverged_pcg_takes_more_newton_iterations():
    """cg_iters = 2 leaves a linear residual, so Newton iterates again --
    still converges to the reference answer."""
    meta = META["imex_transport_n12"]
    cfg, sysm, y0 = imex_case(12, fast="none", d_impl=meta["d_impl"], cg_iters=2)
    H = meta["H"]
    y, cnt = sysm.mri_integrate(GARK3B, "kutta3", meta["m"], 0.0, meta["steps"] * H, H, y0)
    assert cnt[4] > cnt[3]
    assert cnt[1] == cnt[4] + cnt[3] + 3  # one residual per iteration + final, + stage-0 evals
    assert per_species_rel_err(y, FIX["imex_transport_n12_y"], cfg["S"] + 1) <= 1e-10


def test_newton_failure_raises_with_stage_and_counts():
    """cg_iters = 0 never updates Y: newton_solve exhausts max_iters and
    mri_step throws IntegrationError at the first solve stage (mri.cpp:404-410)."""
    cfg, sysm, y0 = imex_case(12, fast="none", d_impl=0.05, cg_iters=0)
    with pytest.raises(O.StepError) as ei:
        sysm.mri_step(GARK3B, "kutta3", 4, 0.0, 2e-3, y0)
    assert ei.value.stage == 2 and "nonlinear solve failed" in str(ei.value)
    # stage-0 f_I, fast IVP 1 (stage 1), then max_iters + 1 = 6 residuals and
    # 5 iterations at stage 2
    assert ei.value.counters.tolist() == [0, 1 + 6, 1, 1, 5, 0, 5, 1]


@pytest.mark.skipif(not os.path.exists(O.REF_LIB) and not os.path.isdir(O.REF_SRC),
                    reason="reference build unavailable")
def test_newton_failure_matches_reference():
    """NewtonConfig max_iters = 0 with a residual above tolerance: the
    reference and the restatement both fail at the first solve stage with
    the same partial counters."""
    from paper_2211_03293_b200.configs import stage_solver
    cfg = dict(CONFIGS["C5"], d_impl=0.05, cg_iters=4)
    y0 = oracle_system(cfg, 12, fast="none").initial_condition(cfg["ic_seed"])
    tol, safety, _, w = stage_solver(y0)
    sysm = O.System(12, 12, 12, cfg["S"] + 1, fast="none", slow="stencil",
                    mech=O.mechanism(cfg["mech_seed"], cfg["S"], cfg["R"]), S=cfg["S"],
                    R=cfg["R"], rho=cfg["rho"], order=8, diffusion=0.0,
                    prof=O.velocity_profiles(cfg["vel_seed"], 12, 12, 12), imex=True,
                    d_impl=0.05, cg_iters=4, newton=(tol, safety, 0), newton_weights=w)
    errs = []
    for use_ref in (False, True):
        with pytest.raises(O.StepError) as ei:
            sysm.mri_step(GARK3B, "kutta3", 4, 0.0, 2e-3, y0, use_reference=use_ref)
        errs.append(ei.value)
    assert errs[0].stage == errs[1].stage == 2
    assert errs[0].code == errs[1].code == 2
    assert np.array_equal(errs[0].counters, errs[1].counters)
    assert errs[0].counters.tolist() == [0, 2, 1, 1, 0, 0, 0, 1]


def test_contract_errors():
    cfg, sysm, y0 = imex_case(8, fast="none")
    with pytest.raises(O.StepError) as ei:  # explicit coupling on a split slow partition
        sysm.mri_step("mis-kw3", "kutta3", 4, 0.0, 1e-3, y0)
    assert ei.value.code == 1
    plain = oracle_system(dict(CONFIGS["C4"]), 8, fast="none")
    with pytest.raises(O.StepError) as ei:  # IMEX coupling without f_implicit
        plain.mri_step(GARK3B, "kutta3", 4, 0.0, 1e-3, plain.initial_condition(1))
    assert ei.value.code == 1


@pytest.mark.skipif(not os.path.exists(O.REF_LIB) and not os.path.isdir(O.REF_SRC),
                    reason="reference build unavailable")
def test_imex_live_against_reference():
    """Fresh seed and a larger implicit term than the fixture."""
    cfg, sysm, y0 = imex_case(10, fast="none", d_impl=0.1, cg_iters=12)
    H = 2e-3
    a, ca = sysm.mri_integrate(GARK3B, "kutta3", 3, 0.0, 2 * H, H, y0)
    b, cb = sysm.mri_integrate(GARK3B, "kutta3", 3, 0.0, 2 * H, H, y0, use_reference=True)
    assert per_species_rel_err(a, b, cfg["S"] + 1) <= 1e-12
    assert solver_counts_ok(ca, cb, 12)


@pytest.mark.parametrize("key", ["ark_transport_n8", "ark_C5_n8"])
def test_ark_imex_fixture(key):
    """ark_imex_integrate (mri.cpp:437-557) restated with the Newton-PCG stage
    solver against the reference's own run (Newton-GMRES)."""
    meta = META[key]
    cfg, sysm, y0 = imex_case(8, fast=meta["fast"], d_impl=meta["d_impl"], cg_iters=meta["cg_iters"])
    H = meta["H"]
    y, cnt = sysm.ark_imex_integrate(0.0, meta["steps"] * H, H, y0)
    assert solver_counts_ok(cnt, FIX[key + "_counters"], meta["cg_iters"])
    assert per_species_rel_err(y, FIX[key + "_y"], cfg["S"] + 1) <= 1e-13
    if cnt[4] == 0:  # no Newton iteration taken: identical arithmetic
        assert np.array_equal(y, FIX[key + "_y"])
