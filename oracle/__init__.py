"""CPU ORACLE -- test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It is the checker, never
the thing measured or shipped: the product (``paper_2211_03293_b200``) never
imports it and fails loudly when its own CUDA library is missing.

Two CPU implementations live here:

* ``liboracle.so`` -- ``mri_oracle.c``, a plain-C restatement of the
  reference's explicit MRI slow step (proj/src/mri.cpp:323-435,
  proj/src/erk.cpp:9-38, proj/src/mri.cpp:266-303) plus the builder-defined
  physics.
* ``_ref/libref_bridge.so`` -- the reference's OWN C++ stepper compiled
  unmodified from /root/reference/proj/src (oracle/Makefile), driving the same
  physics callbacks.  It pins the restatement bit-for-bit and is the CPU
  baseline ("kind": "reference").  It is built here (where /root/reference
  exists) and travels to the GPU box as a git-ignored build product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libref_bridge.so")
REF_SRC = "/root/reference/proj"

FAST_NONE, FAST_CHEM, FAST_LINEAR = 0, 1, 2
SLOW_NONE, SLOW_STENCIL, SLOW_LINEAR = 0, 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u64p = C.POINTER(C.c_uint64)


class OrcSysCfg(C.Structure):
    _fields_ = [
        ("n0", C.c_int), ("n1", C.c_int), ("n2", C.c_int),
        ("n0_global", C.c_int), ("i0_global", C.c_int),
        ("ncomp", C.c_int),
        ("length", C.c_double),
        ("fast_kind", C.c_int), ("slow_kind", C.c_int),
        ("S", C.c_int), ("R", C.c_int),
        ("rho", C.c_double),
        ("species", _dp), ("reactions", _dp), ("rspecies", _ip),
        ("fast_A", _dp), ("slow_A", _dp),
        ("order", C.c_int),
        ("diffusion", C.c_double),
        ("vel_kind", C.c_int),
        ("u_const", C.c_double * 3),
        ("prof", _dp), ("prof_nmax", C.c_int),
        ("threads", C.c_int),
        ("imex", C.c_int),
        ("d_impl", C.c_double),
        ("cg_iters", C.c_int),
        ("newton_tol", C.c_double),
        ("newton_safety", C.c_double),
        ("newton_max_iters", C.c_int),
        ("newton_w", _dp),
    ]


def build(ref: bool = True, quiet: bool = True) -> None:
    """Compile liboracle.so and, when /root/reference is present, _ref/."""
    out = subprocess.DEVNULL if quiet else None
    subprocess.run(["make", "-C", HERE, "all"], check=True, stdout=out)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, stdout=out)


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _load(path):
    lib = C.CDLL(path)
    return lib


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build(ref=False)
        L = _load(LIB)
        L.orc_sys_create.restype = C.c_void_p
        L.orc_sys_create.argtypes = [C.POINTER(OrcSysCfg)]
        L.orc_sys_destroy.argtypes = [C.c_void_p]
        L.orc_sys_set_threads.argtypes = [C.c_void_p, C.c_int]
        for fn in ("orc_sys_fast_rhs", "orc_sys_slow_rhs", "orc_sys_implicit_rhs"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_double, _dp, _dp]
        L.orc_sys_initial_condition.argtypes = [C.c_void_p, C.c_uint64, _dp]
        for fn in ("orc_sys_mri_step",):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_double,
                                       C.c_double, _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.orc_sys_ark_imex_integrate.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                                 _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.orc_sys_reference_solution.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                                 _dp, _ip, C.c_char_p, C.c_size_t]
        L.orc_sys_erk_integrate.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double,
                                            C.c_double, _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.orc_sys_mri_integrate.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int,
                                            C.c_double, C.c_double, C.c_double, _dp, _u64p, _ip,
                                            C.c_char_p, C.c_size_t]
        L.orc_mech_generate.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, _dp, _ip]
        L.orc_velocity_profiles.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        for fn in ("orc_wrms_norm", "orc_dot"):
            getattr(L, fn).restype = C.c_double
            getattr(L, fn).argtypes = [_dp, _dp, C.c_size_t]
        for fn in ("orc_two_norm", "orc_max_norm"):
            getattr(L, fn).restype = C.c_double
            getattr(L, fn).argtypes = [_dp, C.c_size_t]
        L.orc_max_norm_component.restype = C.c_double
        L.orc_max_norm_component.argtypes = [_dp, C.c_size_t, C.c_size_t]
        L.orc_all_finite.argtypes = [_dp, C.c_size_t]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_LIB) or os.path.isdir(REF_SRC)


def ref():
    """The reference's own stepper (oracle/_ref/libref_bridge.so)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            build(ref=True)
        lib()  # make sure liboracle symbols are resolvable first
        L = _load(REF_LIB)
        L.ref_export_coupling.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_coupling_info.argtypes = [C.c_char_p, C.c_int, _ip, _ip, _ip, _ip, _dp]
        L.ref_sys_mri_step.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_double,
                                       C.c_double, _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.ref_sys_ark_imex_integrate.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                                 _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.ref_sys_reference_solution.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                                 _dp, _ip, C.c_char_p, C.c_size_t]
        L.ref_sys_erk_integrate.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double,
                                            C.c_double, _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.ref_lobatto_nodes.argtypes = [C.c_int, _dp, _dp, C.c_char_p, C.c_size_t]
        L.ref_mrsdc_scheme.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp, _ip, _ip,
                                       _dp, _ip, _dp, C.c_char_p, C.c_size_t]
        L.ref_sys_sdc_integrate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                            C.c_double, _dp, _u64p, _ip, C.c_char_p, C.c_size_t]
        L.ref_sys_mrsdc_integrate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_double, C.c_double, C.c_double, _dp, _u64p, _ip,
                                              C.c_char_p, C.c_size_t]
        L.ref_sys_mri_integrate.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int,
                                            C.c_double, C.c_double, C.c_double, _dp, _u64p, _ip,
                                            C.c_char_p, C.c_size_t]
        L.ref_erk_step_linear.argtypes = [C.c_char_p, C.c_int, _dp, C.c_double, _dp, C.c_double,
                                          _u64p, _ip, C.c_char_p, C.c_size_t]
        _ref = L
    return _ref


# --------------------------------------------------------------------------
# generators (oracle side; the product has its own, checked bit-for-bit)
# --------------------------------------------------------------------------
def mechanism(seed: int, S: int, R: int):
    sp = np.zeros(5 * S)
    rx = np.zeros(3 * R)
    rs = np.zeros(4 * R, dtype=np.int32)
    rc = lib().orc_mech_generate(seed, S, R, _ptr(sp), _ptr(rx), _ptr(rs, _ip))
    if rc:
        raise ValueError("orc_mech_generate failed")
    return sp, rx, rs


def velocity_profiles(seed: int, n0: int, n1: int, n2: int, length: float = 1.0):
    nmax = max(n0, n1, n2)
    prof = np.zeros(6 * nmax)
    lib().orc_velocity_profiles(seed, n0, n1, n2, length, _ptr(prof))
    return prof


class StepError(RuntimeError):
    def __init__(self, code, stage, msg, counters=None):
        super().__init__(msg)
        self.code = code
        self.stage = stage
        self.counters = counters  # partial counts up to the failure


class System:
    """PartitionedSystem analogue over the oracle physics (and, via
    ``use_reference=True`` on the stepping calls, the reference stepper)."""

    def __init__(self, n0, n1, n2, ncomp, *, length=1.0, fast="none", slow="none",
                 mech=None, S=0, R=0, rho=1e-3, fast_A=None, slow_A=None, order=2,
                 diffusion=0.0, u=(1.0, 1.0, 1.0), prof=None, n0_global=None, i0_global=0,
                 threads=1, imex=False, d_impl=0.0, cg_iters=0, newton=(1e-10, 0.1, 10),
                 newton_weights=None):
        self._keep = []
        cfg = OrcSysCfg()
        cfg.n0, cfg.n1, cfg.n2 = n0, n1, n2
        cfg.n0_global = n0 if n0_global is None else n0_global
        cfg.i0_global = i0_global
        cfg.ncomp = ncomp
        cfg.length = length
        cfg.fast_kind = {"none": FAST_NONE, "chem": FAST_CHEM, "linear": FAST_LINEAR}[fast]
        cfg.slow_kind = {"none": SLOW_NONE, "stencil": SLOW_STENCIL, "linear": SLOW_LINEAR}[slow]
        if mech is not None:
            sp, rx, rs = (np.ascontiguousarray(mech[0], dtype=np.float64),
                          np.ascontiguousarray(mech[1], dtype=np.float64),
                          np.ascontiguousarray(mech[2], dtype=np.int32))
            self._keep += [sp, rx, rs]
            cfg.S, cfg.R, cfg.rho = S, R, rho
            cfg.species, cfg.reactions, cfg.rspecies = _ptr(sp), _ptr(rx), _ptr(rs, _ip)
        if fast_A is not None:
            fa = np.ascontiguousarray(fast_A, dtype=np.float64).ravel()
            self._keep.append(fa)
            cfg.fast_A = _ptr(fa)
        if slow_A is not None:
            sa = np.ascontiguousarray(slow_A, dtype=np.float64).ravel()
            self._keep.append(sa)
            cfg.slow_A = _ptr(sa)
        cfg.order = order
        cfg.diffusion = diffusion
        if prof is not None:
            pr = np.ascontiguousarray(prof, dtype=np.float64)
            self._keep.append(pr)
            cfg.vel_kind = 1
            cfg.prof = _ptr(pr)
            cfg.prof_nmax = max(n0 if n0_global is None else n0_global, n1, n2)
        else:
            cfg.vel_kind = 0
            cfg.u_const[:] = list(u)
        cfg.threads = threads
        cfg.imex = int(imex)
        cfg.d_impl = d_impl
        cfg.cg_iters = cg_iters
        # NewtonConfig (solvers.hpp:19-23) as run_method builds it from the
        # StudyConfig defaults (harness.cpp:333-339, harness.hpp:59-61)
        cfg.newton_tol, cfg.newton_safety, cfg.newton_max_iters = newton
        if newton_weights is not None:
            nw = np.ascontiguousarray(newton_weights, dtype=np.float64)
            self._keep.append(nw)
            cfg.newton_w = _ptr(nw)
        self.cfg = cfg
        self.ncell = n0 * n1 * n2
        self.ncomp = ncomp
        self.dof = self.ncell * ncomp
        self.h = lib().orc_sys_create(C.byref(cfg))
        if not self.h:
            raise ValueError("orc_sys_create failed (bad mechanism?)")

    def __del__(self):
        try:
            if self.h:
                lib().orc_sys_destroy(self.h)
        except Exception:
            pass

    def set_threads(self, n):
        lib().orc_sys_set_threads(self.h, n)

    def fast_rhs(self, y, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        lib().orc_sys_fast_rhs(self.h, t, _ptr(y), _ptr(out))
        return out

    def slow_rhs(self, y, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        lib().orc_sys_slow_rhs(self.h, t, _ptr(y), _ptr(out))
        return out

    def implicit_rhs(self, y, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        if lib().orc_sys_implicit_rhs(self.h, t, _ptr(y), _ptr(out)):
            raise ValueError("implicit_rhs needs an IMEX system")
        return out

    def initial_condition(self, seed):
        y = np.empty(self.dof)
        if lib().orc_sys_initial_condition(self.h, seed, _ptr(y)):
            raise ValueError("initial_condition needs a mechanism")
        return y

    def _call(self, fn, *args, y, counters):
        y = np.array(y, dtype=np.float64, copy=True)
        cnt = np.zeros(8, dtype=np.uint64) if counters is None else np.array(counters, dtype=np.uint64)
        stage = C.c_int(-1)
        err = C.create_string_buffer(512)
        rc = fn(self.h, *args, _ptr(y), _ptr(cnt, _u64p), C.byref(stage), err, 512)
        return rc, y, cnt, stage.value, err.value.decode()

    def mri_step(self, coupling, fast_table, m, t, H, y, counters=None, use_reference=False):
        fn = ref().ref_sys_mri_step if use_reference else lib().orc_sys_mri_step
        rc, y2, cnt, stage, err = self._call(fn, coupling.encode(), fast_table.encode(), m, t, H,
                                             y=y, counters=counters)
        if rc:
            raise StepError(rc, stage, err, cnt)
        return y2, cnt

    def mri_integrate(self, coupling, fast_table, m, t0, tf, H, y, counters=None,
                      use_reference=False):
        fn = ref().ref_sys_mri_integrate if use_reference else lib().orc_sys_mri_integrate
        rc, y2, cnt, stage, err = self._call(fn, coupling.encode(), fast_table.encode(), m, t0, tf,
                                             H, y=y, counters=counters)
        if rc:
            raise StepError(rc, stage, err, cnt)
        return y2, cnt


    def ark_imex_integrate(self, t0, tf, H, y, counters=None, use_reference=False):
        """ark_imex_integrate (mri.cpp:542-557) with the ark436 pair."""
        fn = ref().ref_sys_ark_imex_integrate if use_reference else lib().orc_sys_ark_imex_integrate
        rc, y2, cnt, stage, err = self._call(fn, t0, tf, H, y=y, counters=counters)
        if rc:
            raise StepError(rc, stage, err, cnt)
        return y2, cnt

    def sdc_integrate(self, n_nodes, sweeps, t0, tf, H, y):
        """The reference's own sdc_integrate (sdc.cpp:267-281) of sum_rhs with
        lobatto_nodes(n_nodes); returns (y, evaluations)."""
        y2 = np.array(y, dtype=np.float64, copy=True)
        ev = np.zeros(1, dtype=np.uint64)
        stage = C.c_int(-1)
        err = C.create_string_buffer(512)
        rc = ref().ref_sys_sdc_integrate(self.h, n_nodes, sweeps, t0, tf, H, _ptr(y2),
                                         ev.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(stage),
                                         err, 512)
        if rc:
            raise StepError(rc, stage.value, err.value.decode(), ev)
        return y2, int(ev[0])

    def mrsdc_integrate(self, X, Y, Z, sweeps, t0, tf, H, y, counters=None):
        """The reference's own mrsdc_integrate (sdc.cpp:283-301) with
        build_scheme(X, Y, Z, sweeps)."""
        rc, y2, cnt, stage, err = self._call(ref().ref_sys_mrsdc_integrate, X, Y, Z, sweeps, t0,
                                             tf, H, y=y, counters=counters)
        if rc:
            raise StepError(rc, stage, err, cnt)
        return y2, cnt

    def erk_integrate(self, table, t0, tf, h, y, use_reference=False):
        """erk_integrate (erk.cpp:40-57) of the summed RHS with a registered
        table; returns (y, stage evaluations)."""
        fn = ref().ref_sys_erk_integrate if use_reference else lib().orc_sys_erk_integrate
        y2 = np.array(y, dtype=np.float64, copy=True)
        ev = np.zeros(1, dtype=np.uint64)
        stage = C.c_int(-1)
        err = C.create_string_buffer(512)
        rc = fn(self.h, table.encode(), t0, tf, h, _ptr(y2),
                ev.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(stage), err, 512)
        if rc:
            raise StepError(rc, stage.value, err.value.decode(), ev)
        return y2, int(ev[0])

    def reference_solution(self, t0, tf, h_ref, y, use_reference=False):
        """reference_solution (erk.cpp:59-75): cash-karp5 on the summed RHS."""
        fn = ref().ref_sys_reference_solution if use_reference else lib().orc_sys_reference_solution
        y2 = np.array(y, dtype=np.float64, copy=True)
        stage = C.c_int(-1)
        err = C.create_string_buffer(512)
        rc = fn(self.h, t0, tf, h_ref, _ptr(y2), C.byref(stage), err, 512)
        if rc:
            raise StepError(rc, stage.value, err.value.decode())
        return y2


def export_coupling(name: str) -> str:
    """The reference's export_coupling text (mri.cpp:560-588) for a registered
    coupling or the ERK45a stand-in ``imex-mri-gark4-explicit``."""
    buf = C.create_string_buffer(1 << 16)
    n = ref().ref_export_coupling(name.encode(), buf, 1 << 16)
    if n < 0:
        raise ValueError(f"unknown coupling {name}")
    return buf.value.decode()


def coupling_info(spec: str, m: int):
    s = C.c_int()
    kinds = np.zeros(16, dtype=np.int32)
    ev = np.zeros(16, dtype=np.int32)
    ns = np.zeros(16, dtype=np.int32)
    c = np.zeros(16)
    rc = ref().ref_coupling_info(spec.encode(), m, C.byref(s), _ptr(kinds, _ip), _ptr(ev, _ip),
                                 _ptr(ns, _ip), _ptr(c))
    if rc:
        raise ValueError("bad coupling")
    n = s.value
    return dict(s=n, kinds=kinds[:n].tolist(), eval_at=ev[:n].tolist(), n_sub=ns[:n].tolist(),
                c=c[:n].tolist())


def norms():
    L = lib()

    def P(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return a, _ptr(a)

    class N:
        @staticmethod
        def wrms(x, w):
            x, px = P(x); w, pw = P(w)
            return L.orc_wrms_norm(px, pw, x.size)

        @staticmethod
        def dot(x, y):
            x, px = P(x); y, py = P(y)
            return L.orc_dot(px, py, x.size)

        @staticmethod
        def two(x):
            x, px = P(x)
            return L.orc_two_norm(px, x.size)

        @staticmethod
        def max(x):
            x, px = P(x)
            return L.orc_max_norm(px, x.size)

        @staticmethod
        def max_component(x, off, cnt):
            x, px = P(x)
            return L.orc_max_norm_component(px, off, cnt)

        @staticmethod
        def all_finite(x):
            x, px = P(x)
            return bool(L.orc_all_finite(px, x.size))

    return N


def ref_lobatto_nodes(n):
    """The reference's lobatto_nodes(n) (sdc.cpp:60-80): (nodes, S flattened)."""
    nodes = np.zeros(n)
    S = np.zeros((n - 1) * n)
    err = C.create_string_buffer(256)
    if ref().ref_lobatto_nodes(n, _ptr(nodes), _ptr(S), err, 256):
        raise ValueError(err.value.decode())
    return nodes, S


def ref_mrsdc_scheme(X, Y, Z, sweeps=1):
    """The reference's build_scheme (sdc.cpp:82-153), flattened like
    paper_2211_03293_b200.mrsdc_scheme."""
    nf = C.c_int(0)
    err = C.create_string_buffer(256)
    if ref().ref_mrsdc_scheme(X, Y, Z, sweeps, C.byref(nf), None, None, None, None, None, None,
                              None, err, 256):
        raise ValueError(err.value.decode())
    n = nf.value
    sc = dict(X=X, Y=Y, n_fine=n, coarse_nodes=np.zeros(X), fine_nodes=np.zeros(n),
              coarse_of_fine=np.zeros(n, dtype=np.int32),
              coarse_index_of_fine=np.zeros(n, dtype=np.int32),
              fine_row=np.zeros((n - 1) * Y), application_offset=np.zeros(n - 1, dtype=np.int32),
              coarse_row=np.zeros((n - 1) * X))
    ip = C.POINTER(C.c_int)
    if ref().ref_mrsdc_scheme(X, Y, Z, sweeps, C.byref(nf), _ptr(sc["coarse_nodes"]),
                              _ptr(sc["fine_nodes"]), sc["coarse_of_fine"].ctypes.data_as(ip),
                              sc["coarse_index_of_fine"].ctypes.data_as(ip), _ptr(sc["fine_row"]),
                              sc["application_offset"].ctypes.data_as(ip), _ptr(sc["coarse_row"]),
                              err, 256):
        raise ValueError(err.value.decode())
    return sc
