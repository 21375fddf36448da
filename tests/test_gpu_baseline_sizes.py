"""GPU parity at BASELINE.json's stated sizes ("What's missing" 1).

Every test compares the CUDA path (through the C-ABI) with the CPU oracle on
identical seeded inputs at the north-star tolerances: per slow step and per
species max|y_gpu - y_ref| / max|y_ref| <= 1e-10 (the idiom of
proj/tests/test_mri.cpp:255 with max_norm_component), EvalCounters exactly
equal.  The oracle runs its physics callbacks on every host core of the GPU
box (the stepper's vector ops stay serial, as in the reference).

  * C3 at its full 128^3 size, one slow step of the production path
    (ERK45a stand-in + RK4, m = 50, 8th-order stencil, random velocity);
  * C4 and C5 physics at 64^3 (C5: two IMEX steps with the workload's
    ImplicitStageSolver);
  * a transport-scale step (fast partition off, H = 2e-4) on a grid the
    ring-tiled stencil (stencil_v3_kernel<4, 1>) covers -- through the plain
    single-slab path, the NCCL rank path (loopback communicator: packed halos,
    interior planes overlapped with the exchange, boundary plane ranges) and
    two in-process slabs;
  * a balanced regime (test-only mechanism with A scaled down so the
    chemistry is non-stiff at a transport-scale H) in which the chemistry and
    the transport each move the state by >= 1e-6 per step, so a wrong slow
    partition, forcing polynomial or chemistry all fail the 1e-10 gate.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS
from tests.helpers import oracle_system, per_species_rel_err

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-10
THREADS = os.cpu_count() or 1


def _coupling(cfg):
    return "mis-kw3" if cfg["coupling"] == "mis-kw3" else P.coupling_text(cfg["coupling"])


def _oracle(cfg, n, y0=None, fast="chem", mech=None, n0=None, i0=0):
    sysm = oracle_system(cfg, n, fast=fast, n0=n0, i0=i0, y0=y0)
    if mech is not None:  # test-only mechanism: rebuild with it
        S, R = cfg["S"], cfg["R"]
        prof = O.velocity_profiles(cfg["vel_seed"], n, n, n) if cfg["velocity"] == "random" else None
        sysm = O.System(n, n, n, S + 1, fast=fast, slow="stencil", mech=mech, S=S, R=R,
                        rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"],
                        u=cfg["u"] or (1.0, 1.0, 1.0), prof=prof)
    sysm.set_threads(THREADS)
    return sysm


def _steps_vs_oracle(ctx, cfg, sysm, y0, steps, H, m=None):
    """Step the device and the oracle from the same state every step."""
    m = cfg["m"] if m is None else m
    cp = _coupling(cfg)
    cnt = ctx.counters()
    cnt_ref = np.zeros(8, dtype=np.uint64)
    worst = 0.0
    y_prev = y0
    for i in range(steps):
        t = i * H
        y_ref, cnt_ref = sysm.mri_step(cp, cfg["fast_table"], m, t, H, y_prev, cnt_ref)
        ctx.mri_step(t, H, cnt)
        y = ctx.download()
        err = per_species_rel_err(y, y_ref, cfg["S"] + 1)
        worst = max(worst, err)
        assert err <= STEP_TOL, f"step {i}: max rel err {err:.3e}"
        y_prev = y
    assert np.array_equal(cnt, cnt_ref), (cnt.tolist(), cnt_ref.tolist())
    return worst, y_prev


def test_c3_full_size_one_step_vs_oracle():
    """BASELINE configs[2] at its full 128^3: one production slow step (K1
    chemistry chains with the 21/84 mechanism, K2 ring stencil order 8 with
    the random velocity field, K3 updates) against the oracle."""
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C3", threads=0)
    sysm = _oracle(cfg, cfg["n"])
    worst, _ = _steps_vs_oracle(ctx, cfg, sysm, y0, 1, cfg["H"])
    print(f"C3 128^3 one step: max rel err {worst:.3e}")


@pytest.mark.parametrize("name,steps", [("C4", 1), ("C5", 2)])
def test_c4_c5_physics_at_64cube_vs_oracle(name, steps):
    """The 53-species / 325-reaction mechanism (C4: gark4-explicit + RK4,
    m = 50; C5: IMEX gark3b + kutta3, m = 100 with the slow-implicit diffusion
    and its Newton-PCG stage solver) at 64^3 -- the grid the production
    stencil and chemistry layouts tile -- against the oracle."""
    n = 64
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, name, n=n, threads=0)
    sysm = _oracle(cfg, n, y0=y0)
    worst, _ = _steps_vs_oracle(ctx, cfg, sysm, y0, steps, cfg["H"])
    print(f"{name} physics 64^3 x {steps}: max rel err {worst:.3e}")


def _transport_cfg():
    return dict(CONFIGS["C3"], m=4)


def _transport_ctx(n, loopback=False, i0=0, n0_local=None):
    ctx = P.Context(0)
    if loopback:
        ctx.comm_init_loopback()
    cfg, y0 = P.setup_workload(ctx, "C3", n=n, config=_transport_cfg(), i0=i0,
                               n0_local=n0_local, threads=0)
    ctx.fast_none()
    return ctx, cfg, y0


@pytest.mark.parametrize("path", ["plain", "nccl-loopback"])
def test_transport_scale_step_ring_stencil_vs_oracle(path):
    """Fast partition off, H = 2e-4 (the transport moves the state by ~1e-2
    per step), 64^3 so the production stencil_v3_kernel<4, 1> (8th order,
    random velocity) computes every slow evaluation -- on the NCCL rank path
    as interior + boundary plane ranges around the overlapped halo exchange."""
    n, H = 64, 2e-4
    ctx, cfg, y0 = _transport_ctx(n, loopback=(path == "nccl-loopback"))
    sysm = _oracle(cfg, n, fast="none")
    worst, y = _steps_vs_oracle(ctx, cfg, sysm, y0, 2, H)
    moved = per_species_rel_err(y, y0, cfg["S"] + 1)
    assert moved >= 1e-4, f"transport moved the state by only {moved:.2e}"
    print(f"transport 64^3 ({path}): max rel err {worst:.3e}, state moved {moved:.2e}")


def test_transport_scale_slabs_equal_single_slab():
    """Two in-process slabs (virtual ranks, device-to-device halos) of the
    transport-scale run: bitwise equal to the single slab."""
    n, H = 64, 2e-4
    one, cfg, y0 = _transport_ctx(n)
    one.mri_step(0.0, H)
    ref = one.download().reshape(cfg["S"] + 1, n, n, n)
    ctxs = []
    for r in range(2):
        i0, n0l = P.slab_bounds(n, 2, r)
        c, _, _ = _transport_ctx(n, i0=i0, n0_local=n0l)
        ctxs.append(c)
    P.group_step(ctxs, 0.0, H)
    for r, c in enumerate(ctxs):
        i0, n0l = P.slab_bounds(n, 2, r)
        assert np.array_equal(c.download().reshape(cfg["S"] + 1, n0l, n, n), ref[:, i0:i0 + n0l])


def _balanced_mech(cfg, shift):
    sp, rx, rs = P.mechanism(cfg["mech_seed"], cfg["S"], cfg["R"])
    rx = rx.copy()
    rx[0::3] -= shift  # A -> A e^-shift: non-stiff at a transport-scale H
    return sp, rx, rs


@pytest.mark.parametrize("name,n", [("C3", 64), ("C4", 32)])
def test_balanced_regime_chemistry_and_transport_vs_oracle(name, n):
    """Test-only mechanism (every A scaled by e^-27) at H = 2e-4: the
    chemistry and the transport each move the state by >= 1e-6 relative per
    step, so both partitions and the forcing polynomial coupling them are
    visible to the 1e-10 per-step gate."""
    H, shift = 2e-4, 27.0
    cfg = dict(CONFIGS[name], m=10)
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, name, n=n, config=cfg, threads=0)
    mech = _balanced_mech(cfg, shift)
    ctx.fast_chemistry(cfg["S"], cfg["R"], cfg["rho"], *mech)
    sysm = _oracle(cfg, n, mech=mech)
    S1 = cfg["S"] + 1
    # size of each partition's increment over one step, relative per species
    inc_chem = per_species_rel_err(y0 + H * sysm.fast_rhs(y0), y0, S1)
    inc_tran = per_species_rel_err(y0 + H * sysm.slow_rhs(y0), y0, S1)
    assert inc_chem >= 1e-6 and inc_tran >= 1e-6, (inc_chem, inc_tran)
    worst, _ = _steps_vs_oracle(ctx, cfg, sysm, y0, 2, H)
    print(f"balanced {name} {n}^3: chem moves {inc_chem:.2e}, transport {inc_tran:.2e}, "
          f"max rel err {worst:.3e}")
