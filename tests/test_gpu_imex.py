"""GPU parity of the IMEX path (config C5: imex-mri-gark3b + kutta3,
slow-explicit 8th-order advection, slow-implicit diffusion solved by
newton_solve with the fixed-iteration Jacobi-PCG) through the C-ABI, against
the oracle (same iteration) and the reference's Newton-GMRES fixtures.

Tolerances: 1e-10 per step / 1e-8 per run (north_star); counters exactly
equal to the oracle's, and to the reference's except the two linear-solver
fields (tests.helpers.solver_counts_ok)."""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS
from tests.helpers import oracle_system, per_species_rel_err, solver_counts_ok

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIX = dict(np.load(os.path.join(GOLD, "ref_fixtures.npz")))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))
GARK3B = open(os.path.join(GOLD, "couplings", "imex-mri-gark3b.txt")).read()
STEP_TOL = 1e-10


def c5(**over):
    return dict(CONFIGS["C5"], **over)


def gpu_case(n, cfg, fast=True, **kw):
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C5", n=n, config=cfg, **kw)
    if not fast:
        ctx.fast_none()
    return ctx, cfg, y0


def test_implicit_rhs_matches_oracle():
    ctx, cfg, y0 = gpu_case(12, c5())
    ref = oracle_system(cfg, 12).implicit_rhs(y0)
    got = ctx.implicit_rhs(y0)
    assert per_species_rel_err(got, ref, cfg["S"] + 1) <= 1e-12
    # explicit partition is advection only (diffusion moved to f_I)
    adv = oracle_system(cfg, 12).slow_rhs(y0)
    assert per_species_rel_err(ctx.slow_rhs(y0), adv, cfg["S"] + 1) <= 1e-12


def test_c5_fixture():
    meta = META["C5_n8"]
    ctx, cfg, y0 = gpu_case(8, c5())
    H = meta["H"]
    cnt = ctx.mri_integrate(0.0, meta["steps"] * H, H)
    assert np.array_equal(cnt, FIX["C5_n8_counters"])
    assert per_species_rel_err(ctx.download(), FIX["C5_n8_y"], cfg["S"] + 1) <= STEP_TOL


def test_imex_transport_fixture_and_oracle():
    """One Newton iteration + 8 PCG iterations per solve; implicit diffusion
    visibly changes the state."""
    meta = META["imex_transport_n12"]
    cfg0 = c5(d_impl=meta["d_impl"], cg_iters=meta["cg_iters"], m=meta["m"])
    ctx, cfg, y0 = gpu_case(12, cfg0, fast=False)
    H = meta["H"]
    sysm = oracle_system(cfg, 12, fast="none", y0=y0)
    y_ref = y0.copy()
    cnt_ref = np.zeros(8, dtype=np.uint64)
    cnt = ctx.counters()
    for i in range(meta["steps"]):
        y_prev = ctx.download()
        y_step, _ = sysm.mri_step(GARK3B, "kutta3", meta["m"], i * H, H, y_prev)
        y_ref, cnt_ref = sysm.mri_step(GARK3B, "kutta3", meta["m"], i * H, H, y_ref, cnt_ref)
        ctx.mri_step(i * H, H, cnt)
        assert per_species_rel_err(ctx.download(), y_step, cfg["S"] + 1) <= 1e-13
    y = ctx.download()
    assert np.array_equal(cnt, cnt_ref)
    assert solver_counts_ok(cnt, FIX["imex_transport_n12_counters"], meta["cg_iters"])
    assert per_species_rel_err(y, FIX["imex_transport_n12_y"], cfg["S"] + 1) <= STEP_TOL
    S1 = cfg["S"] + 1
    tot0, tot = y0.reshape(S1, -1).sum(axis=1), y.reshape(S1, -1).sum(axis=1)
    assert np.all(np.abs(tot - tot0) <= 1e-12 * np.abs(tot0))


@pytest.mark.parametrize("cg_iters", [2, 3])
def test_unconverged_pcg_newton_iterations_match_oracle(cg_iters):
    """Few PCG iterations: Newton iterates more; the device makes the same
    convergence decisions as the oracle (equal counters)."""
    cfg0 = c5(d_impl=0.05, cg_iters=cg_iters, m=4)
    ctx, cfg, y0 = gpu_case(12, cfg0, fast=False)
    sysm = oracle_system(cfg, 12, fast="none", y0=y0)
    H = 2e-3
    y_ref, cnt_ref = sysm.mri_integrate(GARK3B, "kutta3", 4, 0.0, 2 * H, H, y0)
    cnt = ctx.mri_integrate(0.0, 2 * H, H)
    assert np.array_equal(cnt, cnt_ref)
    assert cnt[4] > cnt[3]
    assert per_species_rel_err(ctx.download(), y_ref, cfg["S"] + 1) <= 1e-12


def test_c5_reacting_run_matches_oracle():
    """C5 physics (53 species, m = 100, kutta3) on 16^3, two steps."""
    n = 16
    ctx, cfg, y0 = gpu_case(n, c5())
    sysm = oracle_system(cfg, n, y0=y0)
    sysm.set_threads(os.cpu_count() or 1)
    H = cfg["H"]
    y_ref, cnt_ref = sysm.mri_integrate(GARK3B, cfg["fast_table"], cfg["m"], 0.0, 2 * H, H, y0)
    cnt = ctx.mri_integrate(0.0, 2 * H, H)
    assert np.array_equal(cnt, cnt_ref)
    assert per_species_rel_err(ctx.download(), y_ref, cfg["S"] + 1) <= 2 * STEP_TOL


def test_newton_failure_matches_oracle():
    cfg0 = c5(d_impl=0.05, cg_iters=0, m=4)
    ctx, cfg, y0 = gpu_case(12, cfg0, fast=False)
    sysm = oracle_system(cfg, 12, fast="none", y0=y0)
    with pytest.raises(O.StepError) as eo:
        sysm.mri_step(GARK3B, "kutta3", 4, 0.0, 2e-3, y0)
    cnt = ctx.counters()
    with pytest.raises(P.IntegrationError) as eg:
        ctx.mri_step(0.0, 2e-3, cnt)
    assert eg.value.stage_index == eo.value.stage == 2
    assert "nonlinear solve failed" in str(eg.value)
    assert np.array_equal(cnt, eo.value.counters)
    assert np.array_equal(ctx.download(), y0)  # state unchanged on failure


def test_contract_errors():
    ctx, cfg, y0 = gpu_case(8, c5(), fast=False)
    ctx.load_coupling("mis-kw3")  # explicit coupling on a split slow partition
    with pytest.raises(P.ContractError):
        ctx.mri_step(0.0, 1e-3)
    ctx2 = P.Context(0)
    P.setup_workload(ctx2, "C4", n=8)
    ctx2.load_coupling(P.coupling_text("imex-mri-gark3b"))  # needs f_implicit
    with pytest.raises(P.ContractError):
        ctx2.mri_step(0.0, 1e-3)


@pytest.mark.parametrize("P_", [2, 3])
def test_virtual_rank_slabs_match_single(P_):
    """IMEX on in-process virtual ranks: halo exchange per matvec and
    slab-ordered dot products; same Newton decisions, same counters."""
    n = 12
    cfg0 = c5(d_impl=0.05, cg_iters=8, m=4)
    one, cfg, y0 = gpu_case(n, cfg0, fast=False)
    H = 2e-3
    c_one = one.mri_step(0.0, H)
    ref = one.download().reshape(cfg["S"] + 1, n, n, n)
    ymax = float(np.abs(y0).max())
    ctxs = []
    for r in range(P_):
        i0, n0l = P.slab_bounds(n, P_, r)
        c, _, _ = gpu_case(n, cfg0, fast=False, i0=i0, n0_local=n0l, ymax=ymax)
        ctxs.append(c)
    cnt = P.group_step(ctxs, 0.0, H)
    assert np.array_equal(cnt, c_one)
    for r, c in enumerate(ctxs):
        i0, n0l = P.slab_bounds(n, P_, r)
        got = c.download().reshape(cfg["S"] + 1, n0l, n, n)
        assert per_species_rel_err(got, ref[:, i0:i0 + n0l], cfg["S"] + 1) <= 1e-13


# ----------------------------------------------------- ARK-IMEX (8(f) row 4)
@pytest.mark.parametrize("key", ["ark_transport_n8", "ark_C5_n8"])
def test_ark_imex_matches_oracle_and_reference(key):
    meta = META[key]
    cfg0 = c5(d_impl=meta["d_impl"], cg_iters=meta["cg_iters"])
    ctx, cfg, y0 = gpu_case(8, cfg0, fast=meta["fast"] == "chem")
    sysm = oracle_system(cfg, 8, fast=meta["fast"], y0=y0)
    H = meta["H"]
    y_ref, cnt_ref = sysm.ark_imex_integrate(0.0, meta["steps"] * H, H, y0)
    cnt = ctx.ark_imex_integrate(0.0, meta["steps"] * H, H)
    y = ctx.download()
    assert np.array_equal(cnt, cnt_ref)
    assert per_species_rel_err(y, y_ref, cfg["S"] + 1) <= STEP_TOL * meta["steps"]
    assert solver_counts_ok(cnt, FIX[key + "_counters"], meta["cg_iters"])
    assert per_species_rel_err(y, FIX[key + "_y"], cfg["S"] + 1) <= STEP_TOL * meta["steps"]


def test_ark_imex_failures():
    cfg0 = c5(d_impl=0.05, cg_iters=0)
    ctx, cfg, y0 = gpu_case(8, cfg0, fast=False)
    sysm = oracle_system(cfg, 8, fast="none", y0=y0)
    with pytest.raises(O.StepError) as eo:
        sysm.ark_imex_integrate(0.0, 2e-3, 2e-3, y0)
    cnt = ctx.counters()
    with pytest.raises(P.IntegrationError) as eg:
        ctx.ark_imex_step(0.0, 2e-3, cnt)
    assert eg.value.stage_index == eo.value.stage == 1
    assert "nonlinear solve failed" in str(eg.value)
    assert np.array_equal(cnt, eo.value.counters)
    assert np.array_equal(ctx.download(), y0)
    # non-finite stage data (before the solve) keeps the earlier counts
    bad = y0.copy()
    bad[3] = np.inf
    ctx.upload(bad)
    cnt = ctx.counters()
    with pytest.raises(P.IntegrationError) as eg:
        ctx.ark_imex_step(0.0, 2e-3, cnt)
    with pytest.raises(O.StepError) as eo:
        sysm.ark_imex_integrate(0.0, 2e-3, 2e-3, bad)
    assert eg.value.stage_index == eo.value.stage
    assert np.array_equal(cnt, eo.value.counters)
    # f_implicit required
    ctx2 = P.Context(0)
    P.setup_workload(ctx2, "C4", n=8)
    with pytest.raises(P.ContractError):
        ctx2.ark_imex_step(0.0, 1e-17)


def test_tiled_laplacian_paths_match_oracle():
    """n1 % 8 == 0 and n2 % 64 == 0 select the tiled 7-point kernels (f_I
    evaluation, Newton residual, CG matvec): one IMEX step with active PCG
    on 64^3 against the oracle, plus f_I itself."""
    n = 64
    cfg0 = c5(d_impl=0.05, cg_iters=4, m=2)
    ctx, cfg, y0 = gpu_case(n, cfg0, fast=False)
    sysm = oracle_system(cfg, n, fast="none", y0=y0)
    sysm.set_threads(os.cpu_count() or 1)
    assert per_species_rel_err(ctx.implicit_rhs(y0), sysm.implicit_rhs(y0), cfg["S"] + 1) <= 1e-12
    H = 2e-4
    y_ref, cnt_ref = sysm.mri_step(GARK3B, "kutta3", 2, 0.0, H, y0)
    cnt = ctx.mri_step(0.0, H)
    assert np.array_equal(cnt, cnt_ref)
    assert cnt[4] > 0  # Newton iterated: residual + PCG kernels ran
    assert per_species_rel_err(ctx.download(), y_ref, cfg["S"] + 1) <= 1e-12
