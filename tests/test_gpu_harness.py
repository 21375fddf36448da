"""The reference's study harness on a device problem.

oracle/_ref/libharness_test.so links proj/src/harness.cpp compiled UNMODIFIED
with the routing prefix of include/multirate_b200_harness.hpp: every case of
run_method -- Mri, ArkImex, Erk, Sdc, Mrsdc (harness.cpp:346-394) -- goes to
the facade for a routed device problem.  The same study runs on the CPU physics (the
reference's own integrators) and routed to the GPU, through the reference's
run_method / measure_error / fitted_slope / RunReport::write_csv; the two
CSVs (harness.cpp:645-663) must agree row by row: same methods, H, steps and
divergence flags, the error column within 1e-8, the counters exactly equal
(IMEX rows: all but the linear-solver pair, which counts the device's PCG
instead of GMRES)."""
import csv
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(O.LIB), "_ref", "libharness_test.so")
CNT = ["n_fast_evals", "n_implicit_evals", "n_explicit_evals", "n_implicit_solves",
       "n_nonlinear_iters", "n_linear_iters", "n_precond_solves", "n_fast_ivps"]


def _lib():
    if not os.path.exists(LIB):
        pytest.skip("oracle/_ref/libharness_test.so not built (needs /root/reference at build time)")
    L = C.CDLL(LIB)
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
    L.harness_selftest.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, dp, dp, ip, dp, C.c_int,
                                   C.c_double, C.c_double, C.c_int, C.c_int, C.c_char_p, dp,
                                   C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t]
    return L


def _run(tmp_path, name, n, methods, hs, tf, h_ref, *, d_impl=-1.0, cg_iters=0, fast=1,
         newton_tol=1e-10, cfg_over=None):
    L = _lib()
    cfg = dict(CONFIGS[name], **(cfg_over or {}))
    S, R = cfg["S"], cfg["R"]
    sp, rx, rs = P.mechanism(cfg["mech_seed"], S, R)
    y0 = P.initial_condition(cfg["ic_seed"], S, cfg["rho"], sp, n, n, n)
    hs = np.ascontiguousarray(hs, dtype=np.float64)
    p = lambda a, t=C.c_double: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    paths = [str(tmp_path / f) for f in ("cpu.csv", "dev.csv", "dev.json")]
    err = C.create_string_buffer(512)
    rc = L.harness_selftest(n, S, R, cfg["rho"], p(sp), p(rx), p(rs, C.c_int), p(y0), cfg["order"],
                            cfg["diffusion"], d_impl, cg_iters, fast, ",".join(methods).encode(),
                            p(hs), len(hs), 0.0, tf, h_ref, newton_tol,
                            *[x.encode() for x in paths], err, 512)
    assert rc == 0, err.value.decode()
    rows = [list(csv.DictReader(open(x))) for x in paths[:2]]
    return rows[0], rows[1], json.load(open(paths[2]))


def _compare(cpu, dev, linear_pair_may_differ=False):
    assert len(cpu) == len(dev) > 0
    for a, b in zip(cpu, dev):
        assert (a["method"], a["H"], a["steps"], a["diverged"]) == (b["method"], b["H"], b["steps"], b["diverged"])
        keys = [k for k in CNT if not (linear_pair_may_differ and k in ("n_linear_iters", "n_precond_solves"))]
        assert [a[k] for k in keys] == [b[k] for k in keys], (a, b)
        if a["diverged"] == "0":
            ea, eb = float(a["error"]), float(b["error"])
            assert abs(ea - eb) <= 1e-8, (a["method"], a["H"], ea, eb)


def test_explicit_study_rows_cpu_vs_routed_device(tmp_path):
    """mri3-10 (mis-kw3 + bogacki-shampine3) and erk-kutta3 on the C1
    chemistry + 2nd-order transport at 8^3, three step sizes, cash-karp5
    reference: the routed device rows equal the CPU rows."""
    hs = [1.2e-16, 6e-17, 3e-17]
    cpu, dev, js = _run(tmp_path, "C1", 8, ["mri3-10", "erk-kutta3"], hs, 4.8e-16, 3e-19)
    _compare(cpu, dev)
    for r in dev:
        assert r["diverged"] == "0"
    # the study converges at the methods' order (rates of the finer pairs)
    slopes = js["fitted_slopes"]
    assert slopes["mri3-10"] > 2.5 and slopes["erk-kutta3"] > 2.5, slopes
    print({k: round(v, 2) for k, v in slopes.items()})


def test_imex_study_rows_cpu_vs_routed_device(tmp_path):
    """imex-mri3-4 (imex-mri-gark3b + kutta3 with the implicit diffusion
    solved by Newton: GMRES on the CPU, the device PCG) and ark-imex on the
    C5 species set with the reaction off, transport-scale steps."""
    hs = [2e-3, 1e-3, 5e-4]
    cpu, dev, _ = _run(tmp_path, "C5", 8, ["imex-mri3-4", "ark-imex"], hs, 4e-3, 1.25e-5,
                       d_impl=0.05, cg_iters=12, fast=0, newton_tol=1e-2)
    _compare(cpu, dev, linear_pair_may_differ=True)
    assert any(int(r["n_nonlinear_iters"]) > 0 for r in dev)


def test_diverging_run_is_recorded_not_thrown(tmp_path):
    """run_method's divergence handling (harness.cpp:391-394) on the device:
    an unstable explicit step size is a diverged row with no error value, as
    on the CPU."""
    cpu, dev, _ = _run(tmp_path, "C1", 8, ["erk-kutta3"], [2e-15], 4e-15, 2e-18)
    _compare(cpu, dev)
    assert dev[0]["diverged"] == "1" and cpu[0]["diverged"] == "1"


def test_sdc_study_rows_cpu_vs_routed_device(tmp_path):
    """run_method's Sdc and Mrsdc cases (harness.cpp:356-372) routed to the
    device SDC integrators: sdc-2 (lobatto 3) at fast-scale steps and
    mrsdc-335 at slow-scale steps on the C1 chemistry + transport, cash-karp5
    reference -- the routed rows equal the CPU rows."""
    cpu, dev, _ = _run(tmp_path, "C1", 8, ["sdc-2"], [4e-17, 2e-17], 1.6e-16, 2e-19)
    _compare(cpu, dev)
    cpu, dev, js = _run(tmp_path, "C1", 8, ["mrsdc-335"], [1.2e-16, 6e-17, 3e-17], 4.8e-16, 3e-19)
    _compare(cpu, dev)
    assert all(r["diverged"] == "0" for r in dev)
    print({k: round(v, 2) for k, v in js["fitted_slopes"].items()})
