"""GPU, full BASELINE sizes: size-independent properties where the CPU
oracle cannot follow (C4: 256^3 x 54 components, 7.25 GB per state)."""
import numpy as np
import pytest

import paper_2211_03293_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_step_properties(name):
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, name, threads=0)
    S = cfg["S"]
    n = cfg["n"]
    e0 = y0.reshape(S + 1, -1)[S].sum()
    cnt = ctx.mri_step(0.0, cfg["H"])
    assert cnt[7] == 5 and cnt[2] == 7 and cnt[0] == 196
    ptr, dof = ctx.state_ptr(), ctx.dof
    assert ctx.all_finite(ptr, dof)
    y = ctx.download()
    Y = y.reshape(S + 1, -1)
    # energy: chemistry is adiabatic per cell, transport telescopes -> total conserved
    assert abs(Y[S].sum() - e0) <= 1e-12 * abs(e0) * 10
    # mass fractions moved but stay O(1)
    assert np.abs(Y[:S]).max() < 10.0
    assert not np.array_equal(y, y0)
    # bitwise determinism at full size
    ctx.upload(y0)
    ctx.mri_step(0.0, cfg["H"])
    assert np.array_equal(ctx.download(), y)


def test_c2_full_run_matches_oracle():
    """BASELINE configs[1] at its full size and step count (64^3, 20 steps of
    the ERK45a stand-in, m = 20) against the oracle: the north-star 1e-8 over
    the whole run, exactly equal counters."""
    import os

    from paper_2211_03293_b200.configs import CONFIGS
    from tests.helpers import oracle_system, per_species_rel_err

    cfg = CONFIGS["C2"]
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C2")
    n, H, steps = cfg["n"], cfg["H"], cfg["steps"]
    sysm = oracle_system(cfg, n)
    sysm.set_threads(os.cpu_count() or 1)
    y_ref, cnt_ref = sysm.mri_integrate(P.coupling_text(cfg["coupling"]), cfg["fast_table"],
                                        cfg["m"], 0.0, steps * H, H, y0)
    cnt = ctx.mri_integrate(0.0, steps * H, H)
    assert np.array_equal(cnt, cnt_ref)
    err = per_species_rel_err(ctx.download(), y_ref, cfg["S"] + 1)
    print(f"C2 64^3 x {steps} steps: final max rel err {err:.3e}")
    assert err <= 1e-8


def test_c5_slab_full_size_properties():
    """C5 at its per-GPU size (one 48-plane slab of 384^3, periodic onto
    itself): IMEX solves take the reference's zero-iteration Newton path at the
    chemistry-limited H, energy is conserved, the step is deterministic."""
    ctx = P.Context(0)
    i0, n0l = P.slab_bounds(384, 8, 0)
    cfg, y0 = P.setup_workload(ctx, "C5", i0=i0, n0_local=n0l, threads=0)
    S = cfg["S"]
    e0 = y0.reshape(S + 1, -1)[S].sum()
    cnt = ctx.mri_step(0.0, cfg["H"])
    # gark3b + kutta3, m = 100: 3 IVPs, 3 solves, 4 explicit evals, 297 fast evals
    assert cnt.tolist() == [297, 4, 4, 3, 0, 0, 0, 3]
    y = ctx.download()
    assert np.all(np.isfinite(y))
    assert abs(y.reshape(S + 1, -1)[S].sum() - e0) <= 1e-11 * abs(e0)
    ctx.upload(y0)
    ctx.mri_step(0.0, cfg["H"])
    assert np.array_equal(ctx.download(), y)
