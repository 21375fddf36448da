"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's own stepper on the same seeded inputs.

Tolerances (BASELINE.json north_star): per slow step, per-species
max|y_gpu - y_ref| / max|y_ref| <= 1e-10; final state of a full run <= 1e-8;
integer counters exactly equal.  The linear test plugins make the RHS exact,
so there the device stage loop must match the reference BIT-FOR-BIT.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS
from tests.helpers import A_FAST, A_SE, A_SI, Y0_LIN, expm_taylor, per_species_rel_err

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIX = dict(np.load(os.path.join(GOLD, "ref_fixtures.npz")))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))
STEP_TOL = 1e-10
RUN_TOL = 1e-8
RHS_TOL = 1e-12


def oracle_physics(cfg, n, fast="chem", n0=None, i0=0):
    S, R = cfg["S"], cfg["R"]
    mech = O.mechanism(cfg["mech_seed"], S, R)
    prof = O.velocity_profiles(cfg["vel_seed"], n, n, n) if cfg["velocity"] == "random" else None
    return O.System(n if n0 is None else n0, n, n, S + 1, fast=fast, slow="stencil", mech=mech,
                    S=S, R=R, rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"],
                    u=cfg["u"] or (1.0, 1.0, 1.0), prof=prof, n0_global=n, i0_global=i0)


def gpu_ctx(name, n, **kw):
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, name, n=n, **kw)
    return ctx, cfg, y0


# ---------------------------------------------------------------- RHS level
@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_fast_rhs_matches_oracle(name):
    ctx, cfg, y0 = gpu_ctx(name, 8)
    ref = oracle_physics(cfg, 8).fast_rhs(y0)
    got = ctx.fast_rhs(y0)
    S = cfg["S"]
    assert per_species_rel_err(got[: S * 512], ref[: S * 512], S) <= RHS_TOL
    assert np.all(got[S * 512:] == 0.0)  # de/dt = 0


@pytest.mark.parametrize("S,R", [(63, 200), (30, 800), (12, 600), (4, 1)])
def test_fast_rhs_mechanism_sizes(S, R):
    """Mechanism-size edges of the chemistry kernel: the largest species count
    (S + 1 = 64 slots), rate buffers split into several shared-memory chunks
    (R = 800, 1000), the smallest mechanism; RK steps with them too."""
    n = 8
    cfg = dict(CONFIGS["C3"], S=S, R=R, mech_seed=777 + S + R)
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C3", n=n, config=cfg)
    ref = oracle_physics(cfg, n).fast_rhs(y0)
    got = ctx.fast_rhs(y0)
    assert per_species_rel_err(got[: S * n ** 3], ref[: S * n ** 3], S) <= RHS_TOL
    assert np.all(got[S * n ** 3:] == 0.0)
    # one slow step (fast IVPs with this mechanism) against the oracle
    sysm = oracle_physics(cfg, n)
    H = 1e-17
    ctx.method(cfg["coupling"], cfg["fast_table"], 4)
    try:
        y_ref, cnt_ref = sysm.mri_step(P.coupling_text(cfg["coupling"]), cfg["fast_table"], 4,
                                       0.0, H, y0)
    except O.StepError as eo:  # a stiff synthetic mechanism may blow up: same failure
        cnt = ctx.counters()
        with pytest.raises(P.IntegrationError) as eg:
            ctx.mri_step(0.0, H, cnt)
        assert eg.value.stage_index == eo.stage
        assert np.array_equal(cnt, eo.counters)
        assert np.array_equal(ctx.download(), y0)
        return
    cnt = ctx.mri_step(0.0, H)
    assert np.array_equal(cnt, cnt_ref)
    assert per_species_rel_err(ctx.download(), y_ref, S + 1) <= STEP_TOL


def test_mechanism_over_shared_memory_is_contract_error():
    """A mechanism whose reaction records cannot be staged in shared memory
    is refused up front (no silent slow path)."""
    cfg = dict(CONFIGS["C3"], S=12, R=1000, mech_seed=5)
    ctx = P.Context(0)
    with pytest.raises(P.ContractError, match="shared memory"):
        P.setup_workload(ctx, "C3", n=8, config=cfg)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_slow_rhs_matches_oracle(name):
    n = 12
    ctx, cfg, y0 = gpu_ctx(name, n)
    ref = oracle_physics(cfg, n).slow_rhs(y0)
    got = ctx.slow_rhs(y0)
    assert per_species_rel_err(got, ref, cfg["S"] + 1) <= RHS_TOL


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
@pytest.mark.parametrize("n", [32, 64])
def test_slow_rhs_tiled_kernel_matches_oracle(name, n):
    """n1 % 8 == 0 and n2 % 32 == 0 selects the 2.5D register-queue stencil;
    n1 % 16 == 0 and n2 % 64 == 0 the cp.async-ring version (orders 2/4/8)."""
    ctx, cfg, y0 = gpu_ctx(name, n)
    ref = oracle_physics(cfg, n).slow_rhs(y0)
    got = ctx.slow_rhs(y0)
    assert per_species_rel_err(got, ref, cfg["S"] + 1) <= RHS_TOL


@pytest.mark.parametrize("u", [(1.0, -0.5, 0.25), (0.0, 0.0, 0.0)])
def test_slow_rhs_order8_uniform_velocity(u):
    """Order 8 with a uniform velocity on a grid the ring kernel tiles (the
    compile-time uniform-velocity instantiation; C3/C4 use the profile one)."""
    n = 64
    cfg = dict(CONFIGS["C3"], velocity="uniform", u=u)
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C3", n=n, config=cfg)
    ref = oracle_physics(cfg, n).slow_rhs(y0)
    got = ctx.slow_rhs(y0)
    assert per_species_rel_err(got, ref, cfg["S"] + 1) <= RHS_TOL


def test_slow_rhs_properties():
    """test_models.cpp:126-232 ported to 3D: constant -> 0, per-species
    telescoping conservation, linearity."""
    n = 16
    ctx, cfg, y0 = gpu_ctx("C3", n)
    S1 = cfg["S"] + 1
    const = np.full(S1 * n ** 3, 1.7)
    assert np.abs(ctx.slow_rhs(const)).max() <= 1e-9
    r = ctx.slow_rhs(y0).reshape(S1, -1)
    assert np.all(np.abs(r.sum(axis=1)) <= 1e-9 * np.abs(r).max(axis=1) * n ** 3)
    rng = np.random.RandomState(3)
    a, b = rng.rand(S1 * n ** 3), rng.rand(S1 * n ** 3)
    lhs = ctx.slow_rhs(2.0 * a - 3.0 * b)
    rhs = 2.0 * ctx.slow_rhs(a) - 3.0 * ctx.slow_rhs(b)
    assert np.abs(lhs - rhs).max() <= 1e-10 * np.abs(rhs).max()


# ---------------------------------------------------------------- step level
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_step_matches_reference_fixture(name):
    """The reference's own mri_integrate (oracle/_ref) on 8^3 vs the GPU:
    every step within 1e-10 of the reference stepper run from the same state
    (live when oracle/_ref is present, else the oracle restatement pinned to
    it), the whole run within the north star's 1e-8 of the stored fixture,
    counters exactly equal."""
    meta = META[f"{name}_n8"]
    ctx, cfg, y0 = gpu_ctx(name, 8)
    H = meta["H"]
    sysm = oracle_physics(cfg, 8)
    cp = P.coupling_text(cfg["coupling"]) if cfg["coupling"] != "mis-kw3" else "mis-kw3"
    cnt = ctx.counters()
    y_prev = y0
    for i in range(meta["steps"]):
        y_ref, _ = sysm.mri_step(cp, cfg["fast_table"], cfg["m"], i * H, H, y_prev,
                                 use_reference=O.ref_available())
        ctx.mri_step(i * H, H, cnt)
        y_prev = ctx.download()
        assert per_species_rel_err(y_prev, y_ref, cfg["S"] + 1) <= STEP_TOL, f"step {i}"
    assert np.array_equal(cnt, FIX[f"{name}_n8_counters"])
    assert per_species_rel_err(y_prev, FIX[f"{name}_n8_y"], cfg["S"] + 1) <= RUN_TOL


def test_transport_matches_reference_fixture():
    """Reaction-off run with a transport-scale H: the stencil and the forcing
    polynomial dominate the update."""
    meta = META["transport_n12"]
    cfg = dict(CONFIGS["C3"], m=meta["m"])
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C3", n=12, config=cfg)
    ctx.fast_none()
    H = meta["H"]
    cnt = ctx.mri_integrate(0.0, meta["steps"] * H, H)
    y = ctx.download()
    assert np.array_equal(cnt, FIX["transport_n12_counters"])
    assert per_species_rel_err(y, FIX["transport_n12_y"], cfg["S"] + 1) <= STEP_TOL
    S1 = cfg["S"] + 1
    tot0, tot = y0.reshape(S1, -1).sum(axis=1), y.reshape(S1, -1).sum(axis=1)
    assert np.all(np.abs(tot - tot0) <= 1e-12 * np.abs(tot0))


@pytest.mark.parametrize("name,n,steps", [("C1", 32, 10), ("C2", 16, 4), ("C3", 16, 2)])
def test_full_run_matches_oracle(name, n, steps):
    """C1 at its full 32^3 size and full 10 steps; per-step parity along the way."""
    ctx, cfg, y0 = gpu_ctx(name, n)
    sysm = oracle_physics(cfg, n)
    sysm.set_threads(os.cpu_count() or 1)
    cp = P.coupling_text(cfg["coupling"]) if cfg["coupling"] != "mis-kw3" else "mis-kw3"
    H = cfg["H"]
    y_ref = y0.copy()
    cnt_ref = np.zeros(8, dtype=np.uint64)
    cnt = ctx.counters()
    for i in range(steps):
        t = i * H
        y_prev = ctx.download()
        y_ref_step, _ = sysm.mri_step(cp, cfg["fast_table"], cfg["m"], t, H, y_prev)
        y_ref, cnt_ref = sysm.mri_step(cp, cfg["fast_table"], cfg["m"], t, H, y_ref, cnt_ref)
        ctx.mri_step(t, H, cnt)
        y = ctx.download()
        assert per_species_rel_err(y, y_ref_step, cfg["S"] + 1) <= STEP_TOL
    assert np.array_equal(cnt, cnt_ref)
    err = per_species_rel_err(ctx.download(), y_ref, cfg["S"] + 1)
    print(f"{name} {n}^3 x {steps} steps: final max rel err {err:.3e}")
    assert err <= RUN_TOL


def test_determinism_bitwise():
    """acceptance criterion 12 (acceptance_main.cpp:784-823): identical runs
    produce identical bits."""
    outs = []
    for _ in range(2):
        ctx, cfg, y0 = gpu_ctx("C3", 10)
        ctx.mri_integrate(0.0, 2 * cfg["H"], cfg["H"])
        outs.append(ctx.download())
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------ reference pins (linear plugin)
def lin_ctx(coupling, table, m, fast=A_FAST, slow=A_SI + A_SE, ncell=1):
    ctx = P.Context(0)
    ctx.grid(1, 1, ncell, 2)
    ctx.method(coupling, table, m)
    if fast is None:
        ctx.fast_none()
    else:
        ctx.fast_linear(fast)
    if slow is None:
        ctx.slow_none()
    else:
        ctx.slow_linear(slow)
    return ctx


@pytest.mark.parametrize("cp,table", [("mis-kw3", "bogacki-shampine3"),
                                      ("imex-mri-gark4-explicit", "classic-rk4")])
@pytest.mark.parametrize("H", [0.1, 0.05])
def test_linear_bitwise_vs_reference(cp, table, H):
    """Exact RHS => the device stage loop is bit-identical to the reference
    mri_integrate (fixture generated by the reference itself)."""
    ctx = lin_ctx(cp, table, 10, ncell=3)
    ctx.upload(np.repeat(Y0_LIN, 3))
    cnt = ctx.mri_integrate(0.0, 1.0, H)
    y = ctx.download().reshape(2, 3)
    for c in range(3):
        assert np.array_equal(y[:, c], FIX[f"lin_{cp}_{H}_y"])
    assert np.array_equal(cnt, FIX[f"lin_{cp}_{H}_counters"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cp,table,tf,H", [("mis-kw3", "bogacki-shampine3", 1.0, 0.3),
                                           ("imex-mri-gark4-explicit", "classic-rk4", 0.77, 0.1)])
def test_linear_short_last_step_bitwise_vs_reference(cp, table, tf, H):
    """tf not a multiple of H: n_steps = ceil((tf - t0)/H - 1e-12), the last
    step is tf - t and t = t0 + (i+1) H (mri.cpp:524-540) -- bit-identical to
    the reference's own mri_integrate run live from oracle/_ref."""
    m = 7
    ctx = lin_ctx(cp, table, m, ncell=1)
    ctx.upload(Y0_LIN)
    cnt = ctx.mri_integrate(0.0, tf, H)
    sysm = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=A_FAST,
                    slow_A=np.asarray(A_SI) + np.asarray(A_SE))
    y_ref, cnt_ref = sysm.mri_integrate(P.coupling_text(cp), table, m, 0.0, tf, H,
                                        np.asarray(Y0_LIN, dtype=np.float64), use_reference=True)
    assert np.array_equal(ctx.download(), y_ref)
    assert np.array_equal(cnt, cnt_ref)


def test_rk4_taylor_known_answer():
    """test_erk.cpp:35-42: one classic-rk4 step of y'=y, h=0.1 gives the
    degree-4 Taylor polynomial 1.1051708333333333 -- through a one-IVP coupling."""
    ctx = P.Context(0)
    ctx.grid(1, 1, 1, 1)
    c = [0.0, 1.0]
    kind = [2, 0]
    omega = np.array([[[0.0, 0.0], [1.0, 0.0]]])
    ctx.load_coupling_arrays(c, kind, None, omega)
    ctx.load_table("classic-rk4")
    ctx.L.mr_set_substeps(ctx.h, 1)
    ctx.fast_linear([[1.0]])
    ctx.slow_linear([[0.0]])
    ctx.upload(np.array([1.0]))
    cnt = ctx.mri_step(0.0, 0.1)
    assert ctx.download()[0] == pytest.approx(1.1051708333333333, rel=1e-15)
    assert cnt[0] == 4 and cnt[7] == 1 and cnt[2] == 2


def test_degenerate_partitions_identity():
    """test_mri.cpp:127-144: zero partitions => output == input bitwise."""
    ctx = lin_ctx("mis-kw3", "bogacki-shampine3", 4, fast=np.zeros((2, 2)), slow=np.zeros((2, 2)))
    y = np.array([0.7, -1.3])
    ctx.upload(y)
    ctx.mri_step(0.0, 0.25)
    assert np.array_equal(ctx.download(), y)


def test_fast_reduction_is_chained_erk():
    """test_mri.cpp:146-181 through the reference bridge: zero slow part =>
    chained inner ERK; bitwise equal to the reference mri_step."""
    ctx = lin_ctx("mis-kw3", "bogacki-shampine3", 6, slow=np.zeros((2, 2)))
    ctx.upload(Y0_LIN)
    ctx.mri_step(0.0, 0.3)
    lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=A_FAST, slow_A=np.zeros((2, 2)))
    ref, _ = lin.mri_step("mis-kw3", "bogacki-shampine3", 6, 0.0, 0.3, Y0_LIN,
                          use_reference=O.ref_available())
    assert np.array_equal(ctx.download(), ref)


def test_slow_reduction_matches_induced_method():
    """test_mri.cpp:183-257: with f_F = 0 the step equals the induced
    explicit RK; checked against the reference at 1e-12."""
    for cp in ["mis-kw3", "imex-mri-gark4-explicit"]:
        ctx = lin_ctx(cp, "classic-rk4", 3, fast=None)
        ctx.upload(Y0_LIN)
        ctx.mri_step(0.0, 0.21)
        lin = O.System(1, 1, 1, 2, fast="none", slow="linear", slow_A=A_SI + A_SE)
        spec = cp if cp == "mis-kw3" else P.coupling_text(cp)
        ref, _ = lin.mri_step(spec, "classic-rk4", 3, 0.0, 0.21, Y0_LIN)
        assert np.array_equal(ctx.download(), ref)


def test_32_step_totals_and_halving():
    """test_mri.cpp:476-510: 32 steps -> 128/128/384; halving H doubles."""
    ctx = lin_ctx("mis-kw3", "bogacki-shampine3", 4)
    ctx.upload(Y0_LIN)
    c = ctx.mri_integrate(0.0, 3.2, 0.1)
    assert c[2] == 128 and c[7] == 128 and c[0] == 384
    ctx.upload(Y0_LIN)
    h = ctx.mri_integrate(0.0, 3.2, 0.05)
    assert np.array_equal(h, 2 * c)


def test_empirical_order_of_erk45a_standin():
    ctx = lin_ctx("imex-mri-gark4-explicit", "classic-rk4", 10)
    exact = expm_taylor(A_FAST + A_SI + A_SE, 1.0) @ Y0_LIN
    errs = []
    Hs = [0.2, 0.1, 0.05, 0.025]
    for H in Hs:
        ctx.upload(Y0_LIN)
        ctx.mri_integrate(0.0, 1.0, H)
        errs.append(np.abs(ctx.download() - exact).max())
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert slope >= 3.6


def test_nonfinite_raises_with_reference_stage_and_counts():
    """test_erk.cpp:96-110 / mri.cpp:427-431: a blow-up raises
    IntegrationError with the reference's stage_index, the state is unchanged
    and the partial counters equal the reference's."""
    big = np.array([[1e200, 0.0], [0.0, 1e200]])
    ctx = lin_ctx("mis-kw3", "classic-rk4", 4, fast=big, slow=np.zeros((2, 2)))
    y0 = np.array([1e200, 1e200])
    ctx.upload(y0)
    cnt = ctx.counters()
    with pytest.raises(P.IntegrationError) as e:
        ctx.mri_step(0.0, 0.5, cnt)
    assert e.value.stage_index >= 0
    assert np.array_equal(ctx.download(), y0)
    lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=big, slow_A=np.zeros((2, 2)))
    with pytest.raises(O.StepError) as r:
        lin.mri_step("mis-kw3", "classic-rk4", 4, 0.0, 0.5, y0, use_reference=O.ref_available())
    assert r.value.stage == e.value.stage_index
    # partial counters: the reference bridge reports them through mri_integrate
    if O.ref_available():
        cnt_ref = np.zeros(8, dtype=np.uint64)
        import ctypes as C
        stage = C.c_int()
        err = C.create_string_buffer(256)
        yy = y0.copy()
        O.ref().ref_sys_mri_integrate(lin.h, b"mis-kw3", b"classic-rk4", 4, 0.0, 0.5, 0.5,
                                      yy.ctypes.data_as(C.POINTER(C.c_double)),
                                      cnt_ref.ctypes.data_as(C.POINTER(C.c_uint64)),
                                      C.byref(stage), err, 256)
        assert np.array_equal(cnt, cnt_ref)


def test_contract_errors():
    ctx = lin_ctx("mis-kw3", "classic-rk4", 4)
    ctx.upload(Y0_LIN)
    with pytest.raises(P.ContractError):
        ctx.mri_step(0.0, 0.0)
    with pytest.raises(P.ContractError):
        ctx.mri_integrate(1.0, 0.5, 0.1)
    with pytest.raises(P.ContractError):
        ctx.load_coupling("imex-mri-gark4")  # loads, but stepping needs f_implicit
        ctx.mri_step(0.0, 0.1)


# ------------------------------------------------------------- reductions
def test_reductions_match_reference_definitions():
    import torch
    N = O.norms()
    rng = np.random.RandomState(12345)
    ctx = P.Context(0)
    for n in [1, 7, 1000, 1 << 20]:
        x = rng.uniform(-5, 5, n)
        w = rng.uniform(0, 2, n)
        tx = torch.from_numpy(x).cuda()
        tw = torch.from_numpy(w).cuda()
        torch.cuda.synchronize()
        px, pw = tx.data_ptr(), tw.data_ptr()
        assert ctx.wrms_norm(px, pw, n) == pytest.approx(N.wrms(x, w), rel=1e-13)
        assert ctx.two_norm(px, n) == pytest.approx(N.two(x), rel=1e-13)
        assert ctx.dot(px, pw, n) == pytest.approx(N.dot(x, w), rel=1e-11, abs=1e-11)
        assert ctx.max_norm(px, n) == N.max(x)
        off, cnt = n // 3, max(1, n // 2)
        assert ctx.max_norm_component(px, n, off, cnt) == N.max_component(x, off, cnt)
        assert ctx.all_finite(px, n)
    x = np.array([1.0, np.nan, -3.0])
    tx = torch.from_numpy(x).cuda()
    torch.cuda.synchronize()
    assert not ctx.all_finite(tx.data_ptr(), 3)
    assert ctx.max_norm(tx.data_ptr(), 3) == N.max(x)  # NaN ignored like std::max
    with pytest.raises(P.ContractError):
        ctx.max_norm_component(tx.data_ptr(), 3, 2, 2)
    with pytest.raises(P.ContractError):
        ctx.wrms_norm(tx.data_ptr(), tx.data_ptr(), 0)


# ------------------------------------------------------------- slabs
@pytest.mark.parametrize("P_,n", [(2, 16), (4, 16), (4, 32), (3, 32), (3, 64)])
def test_virtual_rank_slabs_equal_single_gpu_bitwise(P_, n):
    """Slab decomposition (8th-order halos of 4 planes) on in-process virtual
    ranks reproduces the single-slab result bit-for-bit (n = 32 exercises the
    2.5D stencil's halo planes)."""
    one, cfg, y0 = gpu_ctx("C3", n)
    H = cfg["H"]
    one.mri_step(0.0, H)
    ref = one.download().reshape(cfg["S"] + 1, n, n, n)
    ctxs = []
    for r in range(P_):
        i0, n0l = P.slab_bounds(n, P_, r)
        c, _, _ = gpu_ctx("C3", n, i0=i0, n0_local=n0l)
        ctxs.append(c)
    cnt = P.group_step(ctxs, 0.0, H)
    assert cnt[2] == 7 * P_ // P_ and cnt[7] == 5
    for r, c in enumerate(ctxs):
        i0, n0l = P.slab_bounds(n, P_, r)
        assert np.array_equal(c.download().reshape(cfg["S"] + 1, n0l, n, n), ref[:, i0:i0 + n0l])


# ------------------------------------------------- host-buffer step (e2e ABI)
@pytest.mark.parametrize("name,n", [("C3", 16), ("C4", 8), ("C1", 12), ("C3", 64), ("C4", 64)])
def test_host_buffer_step_equals_device_step(name, n):
    """mr_mri_step_host (pinned or pageable host buffers, H2D + step + D2H)
    returns exactly the device-resident step's state and counters -- at 64^3
    (order 8, plane-range stencil) through the pipelined upload, whose
    chunked stage-0 stencil and first fused chain must be bitwise the
    whole-grid ops."""
    import torch
    dev, cfg, y0 = gpu_ctx(name, n)
    c_dev = dev.mri_step(0.0, cfg["H"])
    ref = dev.download()
    host, _, _ = gpu_ctx(name, n)
    y_in = torch.from_numpy(y0.copy()).pin_memory().numpy()
    y_out = torch.zeros(y0.size, dtype=torch.float64).pin_memory().numpy()
    c_host = host.counters()
    host.mri_step_host(0.0, cfg["H"], y_in, y_out, c_host)
    assert np.array_equal(c_host, c_dev)
    assert np.array_equal(y_out, ref)
    # PCIe bytes: the state each way, plus the saved y_out when pipelined (n >= 64)
    state = 8 * y0.size
    assert host.last_host_step_bytes() == ((2 if n >= 64 else 1) * state, state)
    y_pageable = np.zeros_like(y0)  # pageable destination: same result
    host.mri_step_host(0.0, cfg["H"], y0, y_pageable)
    assert np.array_equal(y_pageable, ref)
    y_inplace = torch.from_numpy(y0.copy()).pin_memory().numpy()  # y_in is y_out
    host.mri_step_host(0.0, cfg["H"], y_inplace, y_inplace)
    assert np.array_equal(y_inplace, ref)


@pytest.mark.parametrize("name,n", [("C3", 16), ("C4", 64)])
def test_host_buffer_step_failure_keeps_input(name, n):
    """A failing host-buffer step raises the reference's IntegrationError and
    leaves y_out as it was (no partial result -- at 64^3 the result streams
    out during the step's last ops and the saved y_out is put back); the
    device state is the input, as the reference's mri_integrate keeps y on a
    throw.  The NaN sits in the last plane chunk (the periodic ghost of the
    first)."""
    import torch
    ctx, cfg, y0 = gpu_ctx(name, n)
    bad = torch.from_numpy(y0.copy()).pin_memory().numpy()
    bad[y0.size // (cfg["S"] + 1) - 7] = np.nan
    y_out = torch.full((y0.size,), 3.0, dtype=torch.float64).pin_memory().numpy()
    with pytest.raises(P.IntegrationError):
        ctx.mri_step_host(0.0, cfg["H"], bad, y_out)
    assert np.all(y_out == 3.0)
    assert np.array_equal(ctx.download(), bad, equal_nan=True)
    # the context steps on afterwards: a good host step equals the device step
    y_ok = torch.from_numpy(y0.copy()).pin_memory().numpy()
    ctx.mri_step_host(0.0, cfg["H"], y_ok, y_out)
    dev, _, _ = gpu_ctx(name, n)
    dev.mri_step(0.0, cfg["H"])
    assert np.array_equal(y_out, dev.download())


# ------------------------------------------------------ asynchronous step
def test_async_step_equals_sync_step():
    """mr_mri_step_async + mr_mri_step_wait: same state and counters as
    mr_mri_step, with the step ordered after / before the caller's stream."""
    import torch
    a, cfg, y0 = gpu_ctx("C3", 16)
    b, _, _ = gpu_ctx("C3", 16)
    H = cfg["H"]
    c_a = a.mri_step(0.0, H)
    a.mri_step(H, H, c_a)
    s = torch.cuda.Stream()
    c_b = b.counters()
    b.mri_step_async(0.0, H, s.cuda_stream)
    with pytest.raises(P.ContractError):  # state-touching calls wait for the step
        b.download()
    b.mri_step_wait(c_b)
    b.mri_step_async(H, H, None)
    b.mri_step_wait(c_b)
    assert np.array_equal(c_a, c_b)
    assert np.array_equal(a.download(), b.download())
    with pytest.raises(P.ContractError):
        b.mri_step_wait()


def test_async_step_failure_reported_at_wait():
    ctx, cfg, y0 = gpu_ctx("C3", 16)
    ref, _, _ = gpu_ctx("C3", 16)
    bad = y0.copy()
    bad[9] = np.nan
    ctx.upload(bad)
    ref.upload(bad)
    with pytest.raises(P.IntegrationError) as e_ref:
        ref.mri_step(0.0, cfg["H"])
    ctx.mri_step_async(0.0, cfg["H"])
    with pytest.raises(P.IntegrationError) as e:
        ctx.mri_step_wait()
    assert e.value.stage_index == e_ref.value.stage_index
    assert np.array_equal(ctx.download(), bad, equal_nan=True)  # state unchanged


def test_async_step_rejects_state_and_config_calls():
    """While a step is in flight every entry point that touches the state,
    the buffers or the configuration raises ContractError (the pending step
    still reads them); after the wait the result equals the synchronous step."""
    a, cfg, y0 = gpu_ctx("C3", 16)
    ref, _, _ = gpu_ctx("C3", 16)
    H = cfg["H"]
    c_ref = ref.mri_step(0.0, H)
    a.mri_step_async(0.0, H)
    sp, rx, rs = cfg["mech"]
    calls = [
        lambda: a.reference_solution(0.0, H, H),
        lambda: a.ark_imex_integrate(0.0, H, H),
        lambda: a.erk_integrate("classic-rk4", 0.0, H, H),
        lambda: a.grid(16, 16, 16, cfg["S"] + 1),
        lambda: a.load_coupling("mis-kw3"),
        lambda: a.load_table("classic-rk4"),
        lambda: a.fast_chemistry(cfg["S"], cfg["R"], cfg["rho"], sp, rx, rs),
        lambda: a.slow_stencil(8, 0.0),
        lambda: a.newton_config(),
        lambda: a.upload(y0),
        lambda: a.download(),
        lambda: a.fast_rhs(y0),
        lambda: a.slow_rhs(y0),
        lambda: a.mri_step(0.0, H),
        lambda: a.mri_integrate(0.0, 2 * H, H),
        lambda: a.mri_step_async(0.0, H),
        lambda: P.group_step([a], 0.0, H),
        lambda: a.set_profiling(True),
    ]
    for f in calls:
        with pytest.raises(P.ContractError):
            f()
    assert not a.state_ptr()  # the result is reachable only after the wait
    c = a.mri_step_wait()
    assert np.array_equal(c, c_ref)
    assert np.array_equal(a.download(), ref.download())


def _device_view(ptr, n):
    """torch view of n doubles at a raw device pointer (no copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Arr(), device="cuda")


def test_async_step_is_ordered_on_the_callers_stream():
    """The step starts after the work already queued on the caller's stream
    (a delayed copy of the initial state into the state buffer) and the
    caller's later work (an overwrite of the input buffer) runs after it."""
    import torch
    a, cfg, y0 = gpu_ctx("C3", 16)
    ref, _, _ = gpu_ctx("C3", 16)
    H = cfg["H"]
    c_ref = ref.mri_step(0.0, H)
    a.upload(np.zeros_like(y0))  # garbage until the caller's copy lands
    src = torch.from_numpy(y0).cuda()
    torch.cuda.synchronize()
    state = _device_view(a.state_ptr(), y0.size)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)  # the copy lands late
        state.copy_(src)
    a.mri_step_async(0.0, H, s.cuda_stream)
    with torch.cuda.stream(s):  # queued after the step: must not disturb it
        state.zero_()
    c = a.mri_step_wait()
    s.synchronize()
    assert np.array_equal(c, c_ref)
    assert np.array_equal(a.download(), ref.download())
