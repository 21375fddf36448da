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
from paper_2211_03293_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(O.__file__), "_ref", "libfacade_test.so")


@pytest.mark.skipif(not os.path.exists(LIB), reason="facade test library not built (needs the reference)")
@pytest.mark.parametrize("name,n,steps", [("C1", 8, 2), ("C2", 8, 1)])
def test_facade_modes_agree(name, n, steps):
    L = C.CDLL(LIB)
    cfg = CONFIGS[name]
    S, R = cfg["S"], cfg["R"]
    sp, rx, rs = P.mechanism(cfg["mech_seed"], S, R)
    y0 = P.initial_condition(cfg["ic_seed"], S, cfg["rho"], sp, n, n, n)
    errs = np.zeros(3)
    cnt = np.zeros(24, dtype=np.uint64)
    err = C.create_string_buffer(512)
    dp = C.POINTER(C.c_double)
    cp = cfg["coupling"] if cfg["coupling"] == "mis-kw3" else P.coupling_text(cfg["coupling"])
    rc = L.facade_selftest(
        C.c_int(n), C.c_int(S), C.c_int(R), C.c_double(cfg["rho"]), sp.ctypes.data_as(dp),
        rx.ctypes.data_as(dp), rs.ctypes.data_as(C.POINTER(C.c_int)), y0.ctypes.data_as(dp),
        cp.encode(), cfg["fast_table"].encode(), C.c_int(cfg["m"]), C.c_int(cfg["order"]),
        C.c_double(cfg["H"]), C.c_int(steps), errs.ctypes.data_as(dp),
        cnt.ctypes.data_as(C.POINTER(C.c_uint64)), err, C.c_size_t(512))
    assert rc == 0, err.value.decode()
    assert errs[0] <= 1e-10 * steps, errs  # device path vs reference+CPU physics
    assert errs[1] <= 1e-10 * steps, errs  # reference stepper + GPU callbacks vs CPU
    assert errs[2] <= 1e-10 * steps, errs
    assert np.array_equal(cnt[0:8], cnt[16:24]) and np.array_equal(cnt[8:16], cnt[16:24])
