"""GPU: the study runner (harness.cpp:326-512) over the
device plugins -- per-row parity with the oracle (final state, exact
counters) and the convergence rates of a reacting-flow study."""
import math

import numpy as np
import pytest

import paper_2211_03293_b200 as P
from paper_2211_03293_b200 import study as St
from tests.helpers import oracle_system, per_species_rel_err

pytestmark = pytest.mark.gpu


def c1_case(n=8):
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C1", n=n)
    return ctx, cfg, y0


def test_erk_family_matches_oracle_and_counts():
    """erk-<table> rows: erk_integrate (erk.cpp:40-57) on sum_rhs, with the
    reference's explicit-evaluation count."""
    ctx, cfg, y0 = c1_case()
    H = cfg["H"]
    st = St.StudyConfig(methods=["erk-classic-rk4"], h_list=[H / 4], t0=0.0, tf=2.5 * H / 4)
    o = St.run_method(ctx, y0, St.parse_method("erk-classic-rk4"), st, H / 4)
    y_ref, ev = oracle_system(cfg, 8).erk_integrate("classic-rk4", 0.0, 2.5 * H / 4, H / 4, y0)
    assert not o.diverged and o.steps == 3
    assert int(o.counters[2]) == ev == 12
    assert per_species_rel_err(o.final_state, y_ref, cfg["S"] + 1) <= 1e-11


def test_erk_failure_restores_state_and_counts():
    big = np.array([[1e200, 0.0], [0.0, 1e200]])
    ctx = P.Context(0)
    ctx.grid(1, 1, 1, 2)
    ctx.fast_linear(big)
    ctx.slow_linear(np.zeros((2, 2)))
    y0 = np.array([1e200, 1e200])
    ctx.upload(y0)
    cnt = ctx.counters()
    with pytest.raises(P.IntegrationError) as e:
        ctx.erk_integrate("classic-rk4", 0.0, 1.0, 0.5, cnt)
    import oracle as O
    lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=big, slow_A=np.zeros((2, 2)))
    with pytest.raises(O.StepError) as r:
        lin.erk_integrate("classic-rk4", 0.0, 1.0, 0.5, y0)
    assert e.value.stage_index == r.value.stage
    assert int(cnt[2]) == int(r.value.counters[0])
    assert np.array_equal(ctx.download(), y0)


def test_mri_convergence_study_rows_match_oracle():
    """A mri3-<m> study (mis-kw3 + bogacki-shampine3) on C1 physics: every row's
    state and counters equal the oracle's mri_integrate, the reference solution
    is the device cash-karp5, the fitted slope is the method's order (3)."""
    ctx, cfg, y0 = c1_case()
    H = cfg["H"]
    tf = 2 * H
    # error over the species block (the energy's roundoff would dominate a max
    # over the whole vector): the harness's component slice, harness.cpp:321-323
    st = St.StudyConfig(methods=["mri3-10"], h_list=[H, H / 2, H / 4], t0=0.0, tf=tf,
                        component_offset=0, component_count=cfg["S"])
    rep = St.run_convergence_study(ctx, y0, st)
    sysm = oracle_system(cfg, 8)
    from oracle import export_coupling
    for r in rep.rows:
        assert not r.diverged and r.steps == int(round(tf / r.H))
        y_ref, cnt_ref = sysm.mri_integrate(export_coupling("mis-kw3"), "bogacki-shampine3", 10,
                                            0.0, tf, r.H, y0)
        assert np.array_equal(r.counters, cnt_ref)
        ctx.upload(y0)
        ctx.method("mis-kw3", "bogacki-shampine3", 10)
        ctx.mri_integrate(0.0, tf, r.H)
        assert per_species_rel_err(ctx.download(), y_ref, cfg["S"] + 1) <= 1e-9
    print({r.H: (r.error, r.rate) for r in rep.rows}, rep.fitted_slopes)
    assert rep.fitted_slopes["mri3-10"] == pytest.approx(3.0, abs=0.35)
    for r in rep.rows[1:]:
        assert math.isfinite(r.rate)


def test_imex_and_ark_rows_run():
    """imex-mri3-<m> and ark-imex rows on C5 physics (implicit diffusion, the
    workload's stage solver): no divergence, solves and residual evaluations
    counted."""
    from paper_2211_03293_b200.configs import CONFIGS
    cfg = dict(CONFIGS["C5"])
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C5", n=8, config=cfg)
    H = cfg["H"]
    from paper_2211_03293_b200.configs import stage_solver
    tol, safety, mx, w = stage_solver(y0)
    kw = dict(t0=0.0, newton_tol=tol, newton_safety=safety, newton_max_iters=mx,
              solver_weights=w)
    # the chemistry bounds the explicit step: m = 100 inner steps for the MRI,
    # H / 100 for the single-rate ARK
    rows = St.run_efficiency_study(ctx, y0, St.StudyConfig(
        methods=["imex-mri3-100"], h_list=[H, H / 2], tf=H, **kw)).rows
    rows += St.run_efficiency_study(ctx, y0, St.StudyConfig(
        methods=["ark-imex"], h_list=[H / 100, H / 200], tf=H / 100, **kw)).rows
    assert len(rows) == 4
    for r in rows:
        assert not r.diverged, r.note
        assert r.counters[3] > 0 and r.counters[1] >= r.counters[3]  # a residual per solve
        assert math.isfinite(r.error)
