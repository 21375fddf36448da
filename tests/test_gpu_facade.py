"""GPU: the C++ facade (include/multirate_b200.hpp) compiled against the
reference's own headers/sources -- the drop-in as a maintainer would use it.

Runs the same slow steps (a) device-resident through b200::mri_integrate,
(b) through the reference's mri_integrate with GPU-backed PartitionedSystem
callbacks (Mode A) and (c) through the reference's mri_integrate with the CPU
oracle physics, and checks all three agree (1e-10/step) with equal counters.
"""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS, stage_solver
from tests.helpers import solver_counts_ok

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(O.__file__), "_ref", "libfacade_test.so")


def run_facade(cfg, n, steps, H, fast_none=False, d_impl=-1.0, cg_iters=0, diffusion=1e-3):
    L = C.CDLL(LIB)
    S, R = cfg["S"], cfg["R"]
    sp, rx, rs = P.mechanism(cfg["mech_seed"], S, R)
    y0 = P.initial_condition(cfg["ic_seed"], S, cfg["rho"], sp, n, n, n)
    errs = np.zeros(3)
    cnt = np.zeros(24, dtype=np.uint64)
    err = C.create_string_buffer(512)
    dp = C.POINTER(C.c_double)
    cp = cfg["coupling"] if cfg["coupling"] == "mis-kw3" else P.coupling_text(cfg["coupling"])
    newton = weights = None
    if d_impl >= 0.0:
        tol, safety, mx, w = stage_solver(y0)
        newton = np.array([tol, safety, mx], dtype=np.float64)
        weights = np.ascontiguousarray(w)
    rc = L.facade_selftest(
        C.c_int(n), C.c_int(S), C.c_int(R), C.c_double(cfg["rho"]), sp.ctypes.data_as(dp),
        rx.ctypes.data_as(dp), rs.ctypes.data_as(C.POINTER(C.c_int)), y0.ctypes.data_as(dp),
        cp.encode(), cfg["fast_table"].encode(), C.c_int(cfg["m"]), C.c_int(cfg["order"]),
        C.c_double(H), C.c_int(steps), C.c_int(0 if fast_none else 1), C.c_double(diffusion),
        C.c_double(d_impl),
        C.c_int(cg_iters), None if newton is None else newton.ctypes.data_as(dp),
        None if weights is None else weights.ctypes.data_as(dp), errs.ctypes.data_as(dp),
        cnt.ctypes.data_as(C.POINTER(C.c_uint64)), err, C.c_size_t(512))
    assert rc == 0, err.value.decode()
    return errs, cnt


@pytest.mark.skipif(not os.path.exists(LIB), reason="facade test library not built (needs the reference)")
@pytest.mark.parametrize("name,n,steps", [("C1", 8, 2), ("C2", 8, 1)])
def test_facade_modes_agree(name, n, steps):
    cfg = CONFIGS[name]
    errs, cnt = run_facade(cfg, n, steps, cfg["H"])
    assert errs[0] <= 1e-10 * steps, errs  # device path vs reference+CPU physics
    assert errs[1] <= 1e-10 * steps, errs  # reference stepper + GPU callbacks vs CPU
    assert errs[2] <= 1e-10 * steps, errs
    assert np.array_equal(cnt[0:8], cnt[16:24]) and np.array_equal(cnt[8:16], cnt[16:24])


@pytest.mark.skipif(not os.path.exists(LIB), reason="facade test library not built (needs the reference)")
def test_facade_imex_modes_agree():
    """C5's IMEX split through the facade: explicit advection, implicit
    diffusion (Newton + device PCG in Mode B; the reference's Newton-GMRES on
    GPU callbacks in Mode A and on the CPU physics in C)."""
    cfg = dict(CONFIGS["C5"], m=4)
    errs, cnt = run_facade(cfg, 8, 2, 2e-3, fast_none=True, d_impl=0.05, cg_iters=8,
                           diffusion=0.0)
    assert cnt[4] > 0  # the implicit solves took Newton iterations
    assert errs.max() <= 1e-10, errs
    assert np.array_equal(cnt[8:16], cnt[16:24])  # same reference stepper both sides
    assert solver_counts_ok(cnt[0:8], cnt[16:24], 8)


@pytest.mark.skipif(not os.path.exists(LIB), reason="facade test library not built (needs the reference)")
@pytest.mark.parametrize("which", [0, 1, 2])
def test_facade_refsol_and_ark(which):
    """b200::reference_solution / ark_imex_integrate / erk_integrate vs the
    reference's own functions on the CPU physics (erk: equal evaluation count)."""
    L = C.CDLL(LIB)
    cfg = dict(CONFIGS["C5"])
    S, R, n = cfg["S"], cfg["R"], 8
    sp, rx, rs = P.mechanism(cfg["mech_seed"], S, R)
    y0 = P.initial_condition(cfg["ic_seed"], S, cfg["rho"], sp, n, n, n)
    tol, safety, mx, w = stage_solver(y0)
    newton = np.array([tol, safety, mx], dtype=np.float64)
    weights = np.ascontiguousarray(w)
    errs = np.zeros(1)
    cnt = np.zeros(16, dtype=np.uint64)
    err = C.create_string_buffer(512)
    dp = C.POINTER(C.c_double)
    h, steps = (2e-3, 2) if which == 1 else (2e-17, 4)
    rc = L.facade_selftest2(
        C.c_int(which), C.c_int(n), C.c_int(S), C.c_int(R), C.c_double(cfg["rho"]),
        sp.ctypes.data_as(dp), rx.ctypes.data_as(dp), rs.ctypes.data_as(C.POINTER(C.c_int)),
        y0.ctypes.data_as(dp), C.c_int(8), C.c_double(0.0), C.c_double(0.05), C.c_int(8),
        C.c_int(0 if which == 1 else 1), C.c_double(h), C.c_int(steps),
        newton.ctypes.data_as(dp), weights.ctypes.data_as(dp), errs.ctypes.data_as(dp),
        cnt.ctypes.data_as(C.POINTER(C.c_uint64)), err, C.c_size_t(512))
    assert rc == 0, err.value.decode()
    assert errs[0] <= 1e-10 * steps, errs
    if which == 1:
        assert solver_counts_ok(cnt[0:8], cnt[8:16], 8)
    if which == 2:
        assert cnt[2] == cnt[10] == steps * 3
