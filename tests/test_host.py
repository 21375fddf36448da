"""CPU: host-side logic of the product library (no GPU needed).

* libmri_b200.so loads and exports every symbol include/mri_b200.h declares;
* the seeded generators are bit-identical to the oracle's;
* coupling parsing/validation follows the reference's finalize() rules and
  messages (proj/src/mri.cpp:59-167, tests test_mri.cpp:451-474);
* the device stage loop's plan produces the reference's per-step counters
  (test_mri.cpp:288-354) for every coupling/table.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mri_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mr_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = C.CDLL(P.LIB_PATH)
    syms = header_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_no_gpu_fails_loudly_or_runs():
    """Without a GPU the product refuses (no CPU fallback)."""
    try:
        ctx = P.Context(0)
    except P.CudaError:
        return
    ctx.close()


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_mechanism_generator_bitwise(name):
    cfg = CONFIGS[name]
    a = P.mechanism(cfg["mech_seed"], cfg["S"], cfg["R"])
    b = O.mechanism(cfg["mech_seed"], cfg["S"], cfg["R"])
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    sp, rx, rs = a
    rs = rs.reshape(-1, 4)
    # spec: A log-uniform in [1e8,1e14], beta in [-1,1], Ea in [0,30000] cal/mol
    lnA = rx[0::3]
    assert lnA.min() >= np.log(1e8) - 1e-12 and lnA.max() <= np.log(1e14) + 1e-12
    assert np.all(np.abs(rx[1::3]) <= 1.0)
    assert rx[2::3].min() >= 0 and rx[2::3].max() * 1.98720425864083 <= 30000.0 + 1e-9
    # 1-2 distinct reactants and products, all present
    for r in rs:
        present = [k for k in r if k >= 0]
        assert r[0] >= 0 and r[2] >= 0 and len(set(present)) == len(present)


def test_velocity_and_ic_bitwise_including_slabs():
    cfg = CONFIGS["C4"]
    S, R = cfg["S"], cfg["R"]
    sp, rx, rs = P.mechanism(cfg["mech_seed"], S, R)
    n = 12
    assert np.array_equal(P.velocity_profiles(44, n, n, n), O.velocity_profiles(44, n, n, n))
    full_p = P.initial_condition(cfg["ic_seed"], S, 1e-3, sp, n, n, n, threads=4)
    sysm = O.System(n, n, n, S + 1, fast="chem", mech=(sp, rx, rs), S=S, R=R)
    assert np.array_equal(full_p, sysm.initial_condition(cfg["ic_seed"]))
    # a slab of the global field equals the corresponding planes of the full field
    slab = P.initial_condition(cfg["ic_seed"], S, 1e-3, sp, n, n, n, 1.0, 3, 5, threads=2)
    ref = full_p.reshape(S + 1, n, n, n)[:, 3:8].ravel()
    assert np.array_equal(slab, ref)
    # Dirichlet mass fractions sum to 1; T in [800, 2000]
    Y = full_p.reshape(S + 1, -1)
    assert np.allclose(Y[:S].sum(axis=0), 1.0, atol=1e-14)
    assert Y[:S].min() > 0


@pytest.mark.parametrize("cp,table,m,expect", [
    # reference per-step counts (proj/tests/test_mri.cpp:288-354, :476-510)
    ("mis-kw3", "bogacki-shampine3", 4, dict(expl=4, ivps=4, fast=4 * 3)),
    ("mis-kw3", "classic-rk4", 10, dict(expl=4, ivps=4, fast=10 * 4)),
    ("imex-mri-gark4-explicit", "classic-rk4", 20, dict(expl=7, ivps=5, fast=22 * 4)),
    ("imex-mri-gark4-explicit", "classic-rk4", 50, dict(expl=7, ivps=5, fast=49 * 4)),
])
def test_plan_counts_match_reference(cp, table, m, expect):
    c = P.step_counts(cp, table, m)
    assert c[2] == expect["expl"] and c[7] == expect["ivps"] and c[0] == expect["fast"]
    assert c[1] == c[3] == c[4] == c[5] == c[6] == 0
    if O.ref_available():
        info = O.coupling_info(P.coupling_text(cp), m)
        assert info["n_sub"] == P.coupling_inspect(cp, m)["n_sub"]
        assert info["eval_at"] == P.coupling_inspect(cp, m)["eval_at"]


def test_plan_counts_without_fast_partition():
    c = P.step_counts("mis-kw3", "classic-rk4", 10, fast=False)
    assert c[0] == 0 and c[7] == 4  # n_fast_evals only counted with f_fast present


def _mutate(text, fn):
    lines = text.strip().split("\n")
    fn(lines)
    return "\n".join(lines) + "\n"


def test_coupling_structural_violations_rejected():
    """test_mri.cpp:456-474: decreasing abscissae, implicit stage with dc>0,
    row integral != dc -> ContractError."""
    base = P.coupling_text("mis-kw3")

    def dec(lines):
        c = lines[1].split()
        c[1], c[2] = "0.9", "0.2"
        lines[1] = " ".join(c)
    with pytest.raises(P.ContractError, match="abscissae decrease"):
        P.coupling_inspect(_mutate(base, dec))

    def imp(lines):
        k = lines[2].split()
        k[2] = "implicit-solve"
        lines[2] = " ".join(k)
    with pytest.raises(P.ContractError):
        P.coupling_inspect(_mutate(base, imp))

    def row(lines):
        # omega block starts after gamma (1 degree x 5 rows): line 3 + 5 + 1
        r = lines[3 + 5 + 1].split()
        r[0] = repr(float(r[0]) + 0.125)
        lines[3 + 5 + 1] = " ".join(r)
    with pytest.raises(P.ContractError, match="row integral"):
        P.coupling_inspect(_mutate(base, row))

    with pytest.raises(P.ContractError, match="bad header"):
        P.coupling_inspect("mri-coupling v2 x s=2 degrees=1\n0 1\n")


def test_coupling_texts_ship_with_package():
    for name in ["mis-kw3", "imex-mri-gark4-explicit", "imex-mri-gark3b", "imex-mri-gark4"]:
        gold = open(os.path.join(ROOT, "tests", "golden", "couplings", f"{name}.txt")).read()
        assert P.coupling_text(name) == gold
        P.coupling_inspect(name)


def test_reference_harness_is_routed_unmodified():
    """proj/src/harness.cpp compiled unmodified with the routing prefix of
    include/multirate_b200_harness.hpp: run_method's integrator calls resolve
    to the routing functions, which the test driver defines
    and which fall back to the reference's own integrators."""
    import subprocess
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    obj = os.path.join(ref_dir, "harness_routed.o")
    lib = os.path.join(ref_dir, "libharness_test.so")
    if not os.path.exists(obj):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    und = subprocess.run(["nm", "-C", "-u", obj], capture_output=True, text=True).stdout
    for f in ("mri_integrate_routed", "ark_imex_integrate_routed", "erk_integrate_routed"):
        assert f"multirate::{f}(" in und
    assert "multirate::mri_integrate(" not in und  # every call site routed
    defs = subprocess.run(["nm", "-C", "--defined-only", lib], capture_output=True, text=True).stdout
    for f in ("mri_integrate_routed", "run_method", "harness_selftest", "RunReport::write_csv"):
        assert f in defs, f


def test_routed_harness_runs_cpu_studies_unchanged(tmp_path):
    """The reference's convergence study (execute_study, harness.cpp:431-512)
    through the routed harness build on its own LinearTwoRateOde: no device
    problem is routed, so every run falls through to the reference's
    integrators and the methods converge at their orders."""
    lib = os.path.join(ROOT, "oracle", "_ref", "libharness_test.so")
    if not os.path.exists(lib):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    L = C.CDLL(lib)
    dp = C.POINTER(C.c_double)
    L.harness_cpu_study.argtypes = [C.c_char_p, dp, C.c_int, C.c_char_p, dp, C.c_char_p, C.c_size_t]
    methods = ["mri3-10", "erk-classic-rk4", "imex-mri3-10", "ark-imex"]
    hs = np.array([0.1, 0.05, 0.025, 0.0125])
    slopes = np.zeros(len(methods))
    err = C.create_string_buffer(256)
    csv_path = str(tmp_path / "study.csv")
    n = L.harness_cpu_study(",".join(methods).encode(), hs.ctypes.data_as(dp), len(hs),
                            csv_path.encode(), slopes.ctypes.data_as(dp), err, 256)
    assert n == len(methods) * len(hs), err.value.decode()
    rows = open(csv_path).read().strip().splitlines()
    assert rows[0].startswith("method,H,tolerance,error,rate") and len(rows) == n + 1
    for name, order, s in zip(methods, [3, 4, 3, 4], slopes):
        assert s > order - 0.5, (name, s)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_sdc_node_sets_bitwise_reference():
    """lobatto_nodes / build_scheme restated in the library (host code, no GPU)
    are bitwise the reference's own tables (proj/src/sdc.cpp:14-153)."""
    for n in (3, 5):
        a, b = P.lobatto_rule(n), O.ref_lobatto_nodes(n)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for X, Y, Z in [(3, 3, 1), (3, 3, 8), (5, 3, 2), (3, 5, 4), (5, 5, 3)]:
        a, b = P.mrsdc_scheme(X, Y, Z), O.ref_mrsdc_scheme(X, Y, Z)
        assert a["n_fine"] == b["n_fine"] == X + (X - 1) * (Z - 1) + (X - 1) * (Y - 2) * Z
        for k in a:
            assert np.array_equal(a[k], b[k]), k
    with pytest.raises(P.ContractError):
        P.mrsdc_scheme(4, 3, 1)
