"""CPU: the oracle (C restatement) pinned against the reference's own stepper.

Golden vectors in tests/golden/ were produced by oracle/_ref -- the reference
sources compiled unmodified (tests/golden/make_golden.py).  The restatement
must reproduce them BIT-FOR-BIT (both sides are -ffp-contract=off, same
operation order), which pins the oracle before it is trusted as the checker.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2211_03293_b200.configs import CONFIGS
from tests.helpers import A_FAST, A_SE, A_SI, Y0_LIN, expm_taylor

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIX = dict(np.load(os.path.join(GOLD, "ref_fixtures.npz")))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))


def coupling(name):
    if name == "mis-kw3":
        return name
    return open(os.path.join(GOLD, "couplings", f"{name}.txt")).read()


def physics(name, n, fast="chem"):
    cfg = CONFIGS[name]
    S, R = cfg["S"], cfg["R"]
    mech = O.mechanism(cfg["mech_seed"], S, R)
    prof = O.velocity_profiles(cfg["vel_seed"], n, n, n) if cfg["velocity"] == "random" else None
    return cfg, O.System(n, n, n, S + 1, fast=fast, slow="stencil", mech=mech, S=S, R=R,
                         rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"],
                         u=cfg["u"] or (1.0, 1.0, 1.0), prof=prof)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_workload_fixture_bitwise(name):
    cfg, sysm = physics(name, 8)
    meta = META[f"{name}_n8"]
    y0 = sysm.initial_condition(cfg["ic_seed"])
    H = meta["H"]
    y, cnt = sysm.mri_integrate(coupling(cfg["coupling"]), cfg["fast_table"], cfg["m"], 0.0,
                                meta["steps"] * H, H, y0)
    assert np.array_equal(y, FIX[f"{name}_n8_y"])
    assert np.array_equal(cnt, FIX[f"{name}_n8_counters"])


def test_transport_fixture_bitwise():
    meta = META["transport_n12"]
    cfg, sysm = physics("C3", 12, fast="none")
    y0 = sysm.initial_condition(cfg["ic_seed"])
    H = meta["H"]
    y, cnt = sysm.mri_integrate(coupling("imex-mri-gark4-explicit"), "classic-rk4", meta["m"], 0.0,
                                meta["steps"] * H, H, y0)
    assert np.array_equal(y, FIX["transport_n12_y"])
    assert np.array_equal(cnt, FIX["transport_n12_counters"])
    # criterion 10 (acceptance_main.cpp:583-689): per-species totals conserved
    S1 = cfg["S"] + 1
    tot0 = y0.reshape(S1, -1).sum(axis=1)
    tot = y.reshape(S1, -1).sum(axis=1)
    assert np.all(np.abs(tot - tot0) <= 1e-12 * np.abs(tot0))


@pytest.mark.parametrize("cp,table", [("mis-kw3", "bogacki-shampine3"),
                                      ("imex-mri-gark4-explicit", "classic-rk4")])
@pytest.mark.parametrize("H", [0.1, 0.05])
def test_linear_fixture_bitwise(cp, table, H):
    lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=A_FAST, slow_A=A_SI + A_SE)
    y, cnt = lin.mri_integrate(coupling(cp), table, 10, 0.0, 1.0, H, Y0_LIN)
    assert np.array_equal(y, FIX[f"lin_{cp}_{H}_y"])
    assert np.array_equal(cnt, FIX[f"lin_{cp}_{H}_counters"])
    # and it is an accurate integrator (test_mri.cpp:374-421 idiom)
    exact = expm_taylor(A_FAST + A_SI + A_SE, 1.0) @ Y0_LIN
    assert np.abs(y - exact).max() < 5e-3


def test_coupling_export_roundtrip_matches_reference_text():
    for name in ["imex-mri-gark4-explicit", "imex-mri-gark3b", "imex-mri-gark4"]:
        txt = coupling(name)
        # the oracle imports the reference text and finalizes it with the same rules
        lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=A_FAST, slow_A=A_SI)
        if name == "imex-mri-gark4-explicit":
            lin.mri_step(txt, "classic-rk4", 4, 0.0, 0.1, Y0_LIN)
        else:  # IMEX couplings are outside the explicit path
            with pytest.raises(O.StepError) as e:
                lin.mri_step(txt, "classic-rk4", 4, 0.0, 0.1, Y0_LIN)
            assert e.value.code == 1


def test_mis_kw3_restated_equals_reference_export():
    """coupling_from_mis restatement == the reference's registered coupling
    (abscissae/kinds/omega), via a one-step bitwise comparison."""
    lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=A_FAST, slow_A=A_SE)
    a, ca = lin.mri_step("mis-kw3", "classic-rk4", 7, 0.0, 0.13, Y0_LIN)
    b, cb = lin.mri_step(coupling("mis-kw3"), "classic-rk4", 7, 0.0, 0.13, Y0_LIN)
    assert np.array_equal(a, b) and np.array_equal(ca, cb)


def test_norms_known_answers():
    """proj/tests/test_core.cpp:82-112"""
    N = O.norms()
    assert N.wrms(np.zeros(4), np.ones(4)) == 0.0
    assert N.wrms(np.ones(4), np.ones(4)) == pytest.approx(1.0)
    assert N.wrms([3.0, 4.0], [1.0, 1.0]) == pytest.approx(np.sqrt(25.0 / 2.0))
    assert N.max([-5.0, 2.0]) == 5.0
    x = [0.1, -0.3, 9.0, 9.0]
    assert N.max_component(x, 0, 2) == pytest.approx(0.3)
    assert N.max_component(x, 2, 2) == pytest.approx(9.0)
    assert N.all_finite([1.0, 2.0]) and not N.all_finite([1.0, np.nan])


@pytest.mark.skipif(not os.path.isdir(O.REF_SRC) and not os.path.exists(O.REF_LIB),
                    reason="reference build unavailable")
def test_restatement_equals_reference_live():
    """Live cross-check on a fresh case not in the fixtures (seeded IC, 6^3)."""
    cfg, sysm = physics("C2", 6)
    y0 = sysm.initial_condition(99)
    H = cfg["H"]
    cp = coupling(cfg["coupling"])
    a, ca = sysm.mri_integrate(cp, "classic-rk4", 7, 0.0, 2 * H, H, y0)
    b, cb = sysm.mri_integrate(cp, "classic-rk4", 7, 0.0, 2 * H, H, y0, use_reference=True)
    assert np.array_equal(a, b) and np.array_equal(ca, cb)


@pytest.mark.parametrize("key", ["refsol_C1_n8", "refsol_C3_n8", "refsol_C5_n8"])
def test_reference_solution_fixture_bitwise(key):
    """reference_solution (erk.cpp:59-75, cash-karp5 on sum_rhs) restated."""
    from tests.helpers import oracle_system
    meta = META[key]
    cfg = dict(CONFIGS[meta["config"]])
    if "d_impl" in meta:
        cfg.update(d_impl=meta["d_impl"], cg_iters=meta["cg_iters"])
    sysm = oracle_system(cfg, 8, fast=meta["fast"])
    y0 = sysm.initial_condition(cfg["ic_seed"])
    h = meta["h_ref"]
    y = sysm.reference_solution(0.0, meta["steps"] * h, h, y0)
    assert np.array_equal(y, FIX[key + "_y"])


@pytest.mark.skipif(not os.path.isdir(O.REF_SRC) and not os.path.exists(O.REF_LIB),
                    reason="reference build unavailable")
@pytest.mark.parametrize("table", ["classic-rk4", "kutta3", "cash-karp5"])
def test_erk_integrate_equals_reference_live(table):
    """erk_integrate (erk.cpp:40-57) on sum_rhs -- the harness's erk-<table>
    family -- restated bit-for-bit, with the reference's evaluation count."""
    cfg, sysm = physics("C1", 6)
    y0 = sysm.initial_condition(7)
    h = cfg["H"] / 20
    a, ea = sysm.erk_integrate(table, 0.0, 2.5 * h, h, y0)
    b, eb = sysm.erk_integrate(table, 0.0, 2.5 * h, h, y0, use_reference=True)
    stages = {"classic-rk4": 4, "kutta3": 3, "cash-karp5": 6}[table]
    assert np.array_equal(a, b)
    assert ea == eb == 3 * stages  # ceil(2.5) steps
    if table == "cash-karp5":
        assert np.array_equal(a, sysm.reference_solution(0.0, 2.5 * h, h, y0))


def test_erk_integrate_failure_counts():
    """erk_step's throw (erk.cpp:24-26): stage index and the evaluations made
    before it, restated."""
    big = np.array([[1e200, 0.0], [0.0, 1e200]])
    lin = O.System(1, 1, 1, 2, fast="linear", slow="linear", fast_A=big, slow_A=np.zeros((2, 2)))
    y0 = np.array([1e200, 1e200])
    with pytest.raises(O.StepError) as e:
        lin.erk_integrate("classic-rk4", 0.0, 1.0, 0.5, y0)
    assert e.value.stage >= 0 and int(e.value.counters[0]) == e.value.stage
    if O.ref_available():
        with pytest.raises(O.StepError) as r:
            lin.erk_integrate("classic-rk4", 0.0, 1.0, 0.5, y0, use_reference=True)
        assert r.value.stage == e.value.stage
        assert int(r.value.counters[0]) == int(e.value.counters[0])
