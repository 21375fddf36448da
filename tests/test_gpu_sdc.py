"""GPU parity of the device spectral-deferred-correction integrators
(mr_sdc_integrate, mr_mrsdc_integrate) against the reference's OWN
sdc_integrate / mrsdc_integrate (proj/src/sdc.cpp:155-301, compiled from its
sources in oracle/_ref) -- the harness's sdc-<sweeps> and mrsdc-XYZ families
(proj/src/harness.cpp:356-372).

Linear plugins make the RHS exact, so there the device must match the
reference BIT-FOR-BIT (state and counters); with the chemistry + stencil
physics the device RHS differs from the CPU physics at rounding level, so the
state is compared at the north-star tolerance and the counters exactly.
Failures: the reference's IntegrationError stage (the node), its partial
counters, and the input state kept."""
import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from tests.helpers import A_FAST, A_SE, A_SI, Y0_LIN, oracle_system, per_species_rel_err

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]
STEP_TOL = 1e-10


def lin_ctx(fast=True, slow=True):
    ctx = P.Context(0)
    ctx.grid(1, 1, 1, 2)
    ctx.fast_linear(A_FAST) if fast else ctx.fast_none()
    ctx.slow_linear(A_SI + A_SE) if slow else ctx.slow_none()
    ctx.upload(np.asarray(Y0_LIN, dtype=np.float64))
    return ctx


def lin_sys(fast=True, slow=True):
    return O.System(1, 1, 1, 2, fast="linear" if fast else "none",
                    slow="linear" if slow else "none", fast_A=A_FAST,
                    slow_A=np.asarray(A_SI) + np.asarray(A_SE))


@pytest.mark.parametrize("n,sweeps,tf,H", [(3, 2, 1.0, 0.1), (5, 3, 0.77, 0.1), (3, 0, 0.5, 0.25)])
def test_sdc_linear_bitwise_vs_reference(n, sweeps, tf, H):
    ctx = lin_ctx()
    cnt = ctx.sdc_integrate(n, sweeps, 0.0, tf, H)
    y_ref, ev_ref = lin_sys().sdc_integrate(n, sweeps, 0.0, tf, H, Y0_LIN)
    assert np.array_equal(ctx.download(), y_ref)
    assert int(cnt[2]) == ev_ref


@pytest.mark.parametrize("X,Y,Z,sweeps", [(3, 3, 2, 2), (5, 3, 1, 3), (3, 5, 2, 2), (3, 3, 8, 3)])
@pytest.mark.parametrize("fast", [True, False])
def test_mrsdc_linear_bitwise_vs_reference(X, Y, Z, sweeps, fast):
    """Including a system without f_fast: the fast caches are zero and
    n_fast_evals is not counted (sdc.cpp:240-249)."""
    ctx = lin_ctx(fast=fast)
    ctx.mrsdc_build(X, Y, Z, sweeps)
    cnt = ctx.mrsdc_integrate(0.0, 0.77, 0.1)
    y_ref, cnt_ref = lin_sys(fast=fast).mrsdc_integrate(X, Y, Z, sweeps, 0.0, 0.77, 0.1, Y0_LIN)
    assert np.array_equal(ctx.download(), y_ref)
    assert np.array_equal(cnt, cnt_ref)


def test_mrsdc_loaded_reference_scheme_equals_built():
    """The scheme the reference's build_scheme makes, loaded through
    mr_mrsdc_load, steps exactly like the library-built one."""
    a = lin_ctx()
    a.mrsdc_build(5, 3, 2, 2)
    ca = a.mrsdc_integrate(0.0, 0.5, 0.1)
    b = lin_ctx()
    b.mrsdc_load(O.ref_mrsdc_scheme(5, 3, 2), 2)
    cb = b.mrsdc_integrate(0.0, 0.5, 0.1)
    assert np.array_equal(a.download(), b.download())
    assert np.array_equal(ca, cb)


def run_both(dev_call, ref_call, S1, steps):
    """Reference first; if it diverges, the device must raise the same stage
    with the same counters, else match its state at the step tolerance."""
    try:
        y_ref, cnt_ref = ref_call()
    except O.StepError as e:
        with pytest.raises(P.IntegrationError) as eg:
            dev_call()
        assert eg.value.stage_index == e.stage
        return None
    y, cnt = dev_call()
    assert np.array_equal(np.atleast_1d(cnt), np.atleast_1d(cnt_ref))
    err = per_species_rel_err(y, y_ref, S1)
    assert err <= STEP_TOL * steps
    return err


@pytest.mark.parametrize("name,n,steps", [("C1", 8, 2), ("C4", 8, 1)])
def test_sdc_and_mrsdc_physics_vs_reference(name, n, steps):
    """Chemistry + stencil: sdc-2 on lobatto(3) at the fast step H/m and
    mrsdc-335 at H/2 against the reference run live: state within 1e-10 per
    step, counters equal (or the same divergence)."""
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, name, n=n)
    sysm = oracle_system(cfg, n)
    S1 = cfg["S"] + 1
    h = cfg["H"] / cfg["m"]

    def dev_sdc():
        ctx.upload(y0)
        cnt = ctx.sdc_integrate(3, 2, 0.0, steps * h, h)
        return ctx.download(), int(cnt[2])

    err = run_both(dev_sdc, lambda: sysm.sdc_integrate(3, 2, 0.0, steps * h, h, y0), S1, steps)
    print(f"{name} sdc-2 (h = H/m): max rel err {err}")
    Hm = cfg["H"] / 2
    ctx.mrsdc_build(3, 3, 5, 2)

    def dev_mrsdc():
        ctx.upload(y0)
        cnt = ctx.mrsdc_integrate(0.0, steps * Hm, Hm)
        return ctx.download(), cnt

    err = run_both(dev_mrsdc, lambda: sysm.mrsdc_integrate(3, 3, 5, 2, 0.0, steps * Hm, Hm, y0),
                   S1, steps)
    print(f"{name} mrsdc-335 (H/2): max rel err {err}")


@pytest.mark.parametrize("family", ["sdc", "mrsdc"])
def test_nonfinite_node_matches_reference(family):
    """A non-finite node update raises the reference's IntegrationError with
    the node as stage index and the counters as far as the reference counted;
    the device state stays the call's input."""
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C1", n=8)
    bad = y0.copy()
    bad[11] = np.inf
    ctx.upload(bad)
    sysm = oracle_system(cfg, 8)
    H = cfg["H"]
    if family == "sdc":
        with pytest.raises(O.StepError) as eo:
            sysm.sdc_integrate(3, 2, 0.0, H, H, bad)
        cnt = ctx.counters()
        with pytest.raises(P.IntegrationError) as eg:
            ctx.sdc_integrate(3, 2, 0.0, H, H, cnt)
        assert int(cnt[2]) == int(eo.value.counters[0])
    else:
        with pytest.raises(O.StepError) as eo:
            sysm.mrsdc_integrate(3, 3, 2, 2, 0.0, H, H, bad)
        cnt = ctx.counters()
        ctx.mrsdc_build(3, 3, 2, 2)
        with pytest.raises(P.IntegrationError) as eg:
            ctx.mrsdc_integrate(0.0, H, H, cnt)
        assert np.array_equal(cnt, eo.value.counters)
    assert eg.value.stage_index == eo.value.stage
    assert "non-finite update at node" in str(eg.value)
    assert np.array_equal(ctx.download(), bad)


def test_contract_errors():
    ctx = lin_ctx()
    with pytest.raises(P.ContractError):
        ctx.mrsdc_integrate(0.0, 1.0, 0.1)  # no scheme loaded
    with pytest.raises(P.ContractError):
        ctx.mrsdc_build(4, 3, 1, 1)  # X in {3, 5}
    with pytest.raises(P.ContractError):
        ctx.sdc_integrate(4, 1, 0.0, 1.0, 0.1)  # lobatto 3 or 5
    ctx.mrsdc_build(3, 3, 1, 1)
    with pytest.raises(P.ContractError):
        ctx.mrsdc_integrate(1.0, 0.5, 0.1)  # tf must exceed t0
    # a rejected load leaves the loaded scheme in place; int64 arrays are accepted
    bad = P.mrsdc_scheme(3, 3, 2)
    bad["application_offset"] = np.full(bad["n_fine"] - 1, 99, dtype=np.int64)
    with pytest.raises(P.ContractError):
        ctx.mrsdc_load(bad, 2)
    good = {k: (v.astype(np.int64) if isinstance(v, np.ndarray) and v.dtype == np.int32 else v)
            for k, v in P.mrsdc_scheme(3, 3, 1).items()}
    a, b = lin_ctx(), lin_ctx()
    a.mrsdc_build(3, 3, 1, 1)
    b.mrsdc_load(good, 1)
    ca, cb = a.mrsdc_integrate(0.0, 0.3, 0.1), b.mrsdc_integrate(0.0, 0.3, 0.1)
    assert np.array_equal(a.download(), b.download()) and np.array_equal(ca, cb)
    ctx.upload(np.asarray(Y0_LIN, dtype=np.float64))
    ctx.mrsdc_integrate(0.0, 0.3, 0.1)  # the (3, 3, 1) scheme is still loaded
