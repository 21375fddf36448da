"""B200-native MRI slow step -- Python mirror of the reference stepper API.

The product is ``libmri_b200.so`` (C-ABI in ``include/mri_b200.h``: host C++
stage loop + hand-written sm_100a kernels).  This module is a thin ctypes
binding that mirrors the reference's C++ interface for the hot path
(/root/reference/proj/include/multirate/mri.hpp:64-133,
partitioned_system.hpp:25-79, state_vector.hpp:22-36) so tests and the
benchmark read like the reference's own code:

    ctx = Context(device=0)
    ctx.grid(n, n, n, ncomp)
    ctx.method(coupling="mis-kw3", fast_table="classic-rk4", m=10)   # MriMethodConfig
    ctx.fast_chemistry(...); ctx.slow_stencil(...)                  # PartitionedSystem
    ctx.upload(y0)
    ctx.mri_step(t, H, counters)        # raises ContractError / IntegrationError

There is no CPU fallback: if the CUDA library is missing or no GPU is
visible, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import tables
from .configs import CONFIGS, stage_solver

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MR_LIB_PATH", os.path.join(HERE, "libmri_b200.so"))  # override: A/B experiments
COUPLING_DIR = os.path.join(HERE, "data", "couplings")

MR_OK, MR_CONTRACT, MR_INTEGRATION, MR_CUDA = 0, 1, 2, 3
COUNTER_NAMES = ("n_fast_evals", "n_implicit_evals", "n_explicit_evals", "n_implicit_solves",
                 "n_nonlinear_iters", "n_linear_iters", "n_precond_solves", "n_fast_ivps")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u64p = C.POINTER(C.c_uint64)


class ContractError(ValueError):
    """multirate::ContractError (state_vector.hpp:22-25)."""


class IntegrationError(RuntimeError):
    """multirate::IntegrationError with stage_index (state_vector.hpp:30-36)."""

    def __init__(self, msg, stage_index=-1):
        super().__init__(msg)
        self.stage_index = stage_index


class CudaError(RuntimeError):
    pass


_lib = None


def build(quiet: bool = True) -> None:
    import subprocess
    out = subprocess.DEVNULL if quiet else None
    subprocess.run(["make", "-C", HERE, "-j8"], check=True, stdout=out)


def lib():
    """Load libmri_b200.so (fails loudly when it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run paper_2211_03293_b200.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "mr_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "mr_ctx_create_multi": (C.c_int, [_ip, C.c_int, C.POINTER(vp)]),
        "mr_ctx_destroy": (None, [vp]),
        "mr_last_error": (C.c_char_p, [vp]),
        "mr_version": (C.c_int, []),
        "mr_grid_set": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]),
        "mr_coupling_load": (C.c_int, [vp, C.c_int, C.c_int, _dp, _ip, _dp, _dp]),
        "mr_coupling_load_text": (C.c_int, [vp, C.c_char_p]),
        "mr_table_load": (C.c_int, [vp, C.c_int, _dp, _dp, _dp]),
        "mr_set_substeps": (C.c_int, [vp, C.c_int]),
        "mr_fast_chemistry": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, _dp, _dp, _ip]),
        "mr_fast_linear": (C.c_int, [vp, _dp]),
        "mr_fast_none": (C.c_int, [vp]),
        "mr_slow_stencil": (C.c_int, [vp, C.c_int, C.c_double, _dp, _dp, C.c_int]),
        "mr_slow_linear": (C.c_int, [vp, _dp]),
        "mr_slow_none": (C.c_int, [vp]),
        "mr_slow_implicit_diffusion": (C.c_int, [vp, C.c_double, C.c_int]),
        "mr_implicit_rhs": (C.c_int, [vp, C.c_double, _dp, _dp]),
        "mr_newton_config": (C.c_int, [vp, C.c_double, C.c_double, C.c_int, _dp]),
        "mr_reference_solution": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, _ip]),
        "mr_erk_integrate": (C.c_int, [vp, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double,
                                       C.c_double, _u64p, _ip]),
        "mr_ark_imex_step": (C.c_int, [vp, C.c_double, C.c_double, _u64p, _ip]),
        "mr_ark_imex_integrate": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, _u64p, _ip]),
        "mr_sdc_integrate": (C.c_int, [vp, C.c_int, _dp, _dp, C.c_int, C.c_double, C.c_double,
                                       C.c_double, _u64p, _ip]),
        "mr_mrsdc_load": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _ip, _ip,
                                    _dp, _ip, _dp]),
        "mr_mrsdc_build": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int]),
        "mr_mrsdc_integrate": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, _u64p, _ip]),
        "mr_lobatto_rule": (C.c_int, [C.c_int, _dp, _dp]),
        "mr_mrsdc_scheme": (C.c_int, [C.c_int, C.c_int, C.c_int, _ip, _dp, _dp, _ip, _ip, _dp, _ip,
                                      _dp]),
        "mr_state_upload": (C.c_int, [vp, _dp]),
        "mr_state_download": (C.c_int, [vp, _dp]),
        "mr_state_device_ptr": (C.c_void_p, [vp]),
        "mr_state_dof": (C.c_size_t, [vp]),
        "mr_mri_step": (C.c_int, [vp, C.c_double, C.c_double, _u64p, _ip]),
        "mr_mri_step_async": (C.c_int, [vp, C.c_double, C.c_double, vp]),
        "mr_mri_step_wait": (C.c_int, [vp, _u64p, _ip]),
        "mr_mri_integrate": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, _u64p, _ip]),
        "mr_mri_step_host": (C.c_int, [vp, C.c_double, C.c_double, _dp, _dp, _u64p, _ip]),
        "mr_last_failure": (C.c_int, [vp, _ip, _ip, _ip]),
        "mr_last_host_step_bytes": (C.c_int, [vp, _u64p, _u64p]),
        "mr_fast_rhs": (C.c_int, [vp, C.c_double, _dp, _dp]),
        "mr_slow_rhs": (C.c_int, [vp, C.c_double, _dp, _dp]),
        "mr_wrms_norm": (C.c_int, [vp, C.c_void_p, C.c_void_p, C.c_size_t, _dp]),
        "mr_two_norm": (C.c_int, [vp, C.c_void_p, C.c_size_t, _dp]),
        "mr_dot": (C.c_int, [vp, C.c_void_p, C.c_void_p, C.c_size_t, _dp]),
        "mr_max_norm": (C.c_int, [vp, C.c_void_p, C.c_size_t, _dp]),
        "mr_max_norm_component": (C.c_int, [vp, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, _dp]),
        "mr_all_finite": (C.c_int, [vp, C.c_void_p, C.c_size_t, _ip]),
        "mr_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "mr_comm_init": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p]),
        "mr_comm_init_loopback": (C.c_int, [vp]),
        "mr_group_step": (C.c_int, [C.POINTER(vp), C.c_int, C.c_double, C.c_double, _u64p, _ip]),
        "mr_mechanism_generate": (C.c_int, [C.c_uint64, C.c_int, C.c_int, _dp, _dp, _ip]),
        "mr_initial_condition": (C.c_int, [C.c_uint64, C.c_int, C.c_double, _dp, C.c_int, C.c_int,
                                           C.c_int, C.c_double, C.c_int, C.c_int, _dp, C.c_int]),
        "mr_velocity_profiles": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, _dp]),
        "mr_coupling_inspect": (C.c_int, [C.c_char_p, C.c_int, _ip, _ip, _ip, _ip, C.c_char_p,
                                          C.c_size_t]),
        "mr_step_counts": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, _u64p,
                                     C.c_char_p, C.c_size_t]),
        "mr_stream": (C.c_void_p, [vp]),
        "mr_launch_count": (C.c_uint64, [vp]),
        "mr_chem_flops_per_eval": (C.c_double, [vp]),
        "mr_fp64_peak": (C.c_int, [vp, _dp]),
        "mr_set_profiling": (C.c_int, [vp, C.c_int]),
        "mr_last_step_profile": (C.c_int, [vp, _dp, _dp, _dp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# host-side generators (product implementation, C++)
# --------------------------------------------------------------------------
def lobatto_rule(n: int):
    """lobatto_nodes(n) (sdc.cpp:60-80): (nodes[n], S[(n-1) x n] flattened),
    built by the library with the reference's arithmetic (no GPU needed)."""
    nodes = np.zeros(n, dtype=np.float64)
    S = np.zeros(max(n - 1, 0) * n, dtype=np.float64)
    if lib().mr_lobatto_rule(n, _p(nodes), _p(S)):
        raise ContractError("lobatto_nodes: only n = 3 or 5 supported")
    return nodes, S


def mrsdc_scheme(X: int, Y: int, Z: int):
    """build_scheme(X, Y, Z, .) (sdc.cpp:82-153) flattened: the arrays
    mr_mrsdc_load takes (no GPU needed)."""
    nf = C.c_int(0)
    if lib().mr_mrsdc_scheme(X, Y, Z, C.byref(nf), None, None, None, None, None, None, None):
        raise ContractError("build_scheme: need X,Y in {3,5}, Z >= 1")
    n = nf.value
    sc = dict(X=X, Y=Y, n_fine=n, coarse_nodes=np.zeros(X), fine_nodes=np.zeros(n),
              coarse_of_fine=np.zeros(n, dtype=np.int32),
              coarse_index_of_fine=np.zeros(n, dtype=np.int32),
              fine_row=np.zeros((n - 1) * Y), application_offset=np.zeros(n - 1, dtype=np.int32),
              coarse_row=np.zeros((n - 1) * X))
    rc = lib().mr_mrsdc_scheme(X, Y, Z, C.byref(nf), _p(sc["coarse_nodes"]), _p(sc["fine_nodes"]),
                               _p(sc["coarse_of_fine"], _ip), _p(sc["coarse_index_of_fine"], _ip),
                               _p(sc["fine_row"]), _p(sc["application_offset"], _ip),
                               _p(sc["coarse_row"]))
    if rc:
        raise ContractError("build_scheme failed")
    return sc


def mechanism(seed: int, S: int, R: int):
    sp = np.zeros(5 * S)
    rx = np.zeros(3 * R)
    rs = np.zeros(4 * R, dtype=np.int32)
    if lib().mr_mechanism_generate(seed, S, R, _p(sp), _p(rx), _p(rs, _ip)):
        raise ContractError("mr_mechanism_generate: bad arguments")
    return sp, rx, rs


def velocity_profiles(seed: int, n0: int, n1: int, n2: int, length: float = 1.0):
    prof = np.zeros(6 * max(n0, n1, n2))
    lib().mr_velocity_profiles(seed, n0, n1, n2, length, _p(prof))
    return prof


def initial_condition(seed, S, rho, species, n0, n1, n2, length=1.0, i0=0, n0_local=None,
                      threads=0, out=None):
    n0l = n0 if n0_local is None else n0_local
    dof = (S + 1) * n0l * n1 * n2
    Y = np.empty(dof) if out is None else out
    sp = np.ascontiguousarray(species, dtype=np.float64)
    rc = lib().mr_initial_condition(seed, S, rho, _p(sp), n0, n1, n2, length, i0, n0l, _p(Y),
                                    threads)
    if rc:
        raise ContractError("mr_initial_condition: bad arguments")
    return Y


def coupling_text(name: str) -> str:
    """v1 audit text of a coupling (the reference's export_coupling output,
    shipped in data/couplings/)."""
    if name.startswith("mri-coupling"):
        return name
    path = os.path.join(COUPLING_DIR, f"{name}.txt")
    if not os.path.exists(path):
        raise ContractError(f"register_coupling: unknown name '{name}'")
    with open(path) as f:
        return f.read()


def coupling_inspect(coupling: str, m: int = 1):
    """Host-side parse + finalize (reference rules, mri.cpp:59-167); raises
    ContractError with the reference's message on a structural violation."""
    s = C.c_int()
    kinds = np.zeros(16, dtype=np.int32)
    ev = np.zeros(16, dtype=np.int32)
    ns = np.zeros(16, dtype=np.int32)
    err = C.create_string_buffer(512)
    rc = lib().mr_coupling_inspect(coupling_text(coupling).encode(), m, C.byref(s), _p(kinds, _ip),
                                   _p(ev, _ip), _p(ns, _ip), err, 512)
    if rc:
        raise ContractError(err.value.decode())
    n = s.value
    return dict(s=n, kinds=kinds[:n].tolist(), eval_at=ev[:n].tolist(), n_sub=ns[:n].tolist())


def step_counts(coupling: str, fast_table: str, m: int, fast=True, slow=True):
    """EvalCounters increments of one slow step as planned by the device loop."""
    cnt = np.zeros(8, dtype=np.uint64)
    err = C.create_string_buffer(512)
    s_f = len(tables.lookup_table(fast_table)["b"])
    rc = lib().mr_step_counts(coupling_text(coupling).encode(), s_f, m, int(fast), int(slow),
                              _p(cnt, _u64p), err, 512)
    if rc == MR_CONTRACT:
        raise ContractError(err.value.decode())
    if rc:
        raise IntegrationError(err.value.decode())
    return cnt


# --------------------------------------------------------------------------
def _bind_process_nccl():
    """The library resolves NCCL lazily and binds to the libnccl.so.2 already in
    the process (csrc/nccl_shim.h).  Import torch first when it is installed so
    that is PyTorch's bundled NCCL: binding the system NCCL first would leave
    a later `import torch` with unresolved NCCL symbols."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


class Context:
    """One device-resident MRI problem (one slab of the grid) -- or, given a
    list of devices, a multi-device domain (mr_ctx_create_multi): the grid is
    split into slabs over the devices and every call drives all of them."""

    def __init__(self, device=0):
        L = lib()
        h = C.c_void_p()
        if isinstance(device, (list, tuple)):
            devs = np.ascontiguousarray(device, dtype=np.int32)
            rc = L.mr_ctx_create_multi(_p(devs, _ip), len(devs), C.byref(h))
        else:
            rc = L.mr_ctx_create(device, C.byref(h))
        if rc:
            raise CudaError(f"context creation failed (rc={rc}): no usable B200 / CUDA device")
        self.h = h
        self.L = L
        self.dof = 0
        self.s_f = 0

    def close(self):
        if getattr(self, "h", None):
            self.L.mr_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, stage=None):
        if rc == MR_OK:
            return
        msg = self.L.mr_last_error(self.h).decode()
        if rc == MR_CONTRACT:
            raise ContractError(msg)
        if rc == MR_INTEGRATION:
            raise IntegrationError(msg, -1 if stage is None else stage)
        raise CudaError(msg)

    # ---- setup -------------------------------------------------------------
    def grid(self, n0, n1, n2, ncomp, length=1.0, i0=0, n0_local=None):
        n0l = n0 if n0_local is None else n0_local
        self._check(self.L.mr_grid_set(self.h, n0, n1, n2, ncomp, length, i0, n0l))
        self.shape = (n0, n1, n2)
        self.ncomp = ncomp
        self.ncell = n0l * n1 * n2
        self.dof = self.ncell * ncomp
        return self

    def method(self, coupling="mis-kw3", fast_table="classic-rk4", m=1):
        """MriMethodConfig (mri.hpp:64-68)."""
        self.load_coupling(coupling)
        self.load_table(fast_table)
        self._check(self.L.mr_set_substeps(self.h, m))
        return self

    def load_coupling(self, coupling):
        self._check(self.L.mr_coupling_load_text(self.h, coupling_text(coupling).encode()))

    def load_coupling_arrays(self, c, kind, gamma, omega):
        s = len(c)
        cc = np.ascontiguousarray(c, dtype=np.float64)
        kk = np.ascontiguousarray(kind, dtype=np.int32)
        g = None if gamma is None else np.ascontiguousarray(gamma, dtype=np.float64)
        o = None if omega is None else np.ascontiguousarray(omega, dtype=np.float64)
        nd = (g if g is not None else o).size // (s * s)
        self._check(self.L.mr_coupling_load(self.h, s, nd, _p(cc), _p(kk, _ip),
                                            None if g is None else _p(g),
                                            None if o is None else _p(o)))

    def load_table(self, name_or_table):
        t = tables.lookup_table(name_or_table) if isinstance(name_or_table, str) else name_or_table
        A = np.ascontiguousarray(t["A"], dtype=np.float64)
        b = np.ascontiguousarray(t["b"], dtype=np.float64)
        c = np.ascontiguousarray(t["c"], dtype=np.float64)
        self._check(self.L.mr_table_load(self.h, len(b), _p(A), _p(b), _p(c)))
        self.s_f = len(b)

    def fast_chemistry(self, S, R, rho, species, reactions, rspecies):
        sp = np.ascontiguousarray(species, dtype=np.float64)
        rx = np.ascontiguousarray(reactions, dtype=np.float64)
        rs = np.ascontiguousarray(rspecies, dtype=np.int32)
        self._check(self.L.mr_fast_chemistry(self.h, S, R, rho, _p(sp), _p(rx), _p(rs, _ip)))

    def fast_linear(self, A):
        a = np.ascontiguousarray(A, dtype=np.float64).ravel()
        self._check(self.L.mr_fast_linear(self.h, _p(a)))

    def fast_none(self):
        self._check(self.L.mr_fast_none(self.h))

    def slow_stencil(self, order, diffusion, u=(1.0, 1.0, 1.0), prof=None):
        if prof is not None:
            pr = np.ascontiguousarray(prof, dtype=np.float64)
            self._check(self.L.mr_slow_stencil(self.h, order, diffusion, None, _p(pr), pr.size // 6))
        else:
            uu = np.ascontiguousarray(u, dtype=np.float64)
            self._check(self.L.mr_slow_stencil(self.h, order, diffusion, _p(uu), None, 0))

    def slow_implicit_diffusion(self, d_impl, cg_iters):
        """IMEX split (after slow_stencil): f_implicit = d_impl * L7 y, solved
        by cg_iters Jacobi-PCG iterations at ImplicitSolve stages."""
        self._check(self.L.mr_slow_implicit_diffusion(self.h, d_impl, int(cg_iters)))

    def newton_config(self, tolerance=1e-10, safety=0.1, max_iters=10, weights=None):
        """ImplicitStageSolver.newton + weights (mri.hpp:84-95)."""
        if weights is None:
            self._check(self.L.mr_newton_config(self.h, tolerance, safety, int(max_iters), None))
        else:
            w = np.ascontiguousarray(weights, dtype=np.float64)
            assert w.size == self.dof
            self._check(self.L.mr_newton_config(self.h, tolerance, safety, int(max_iters), _p(w)))

    def slow_linear(self, A):
        a = np.ascontiguousarray(A, dtype=np.float64).ravel()
        self._check(self.L.mr_slow_linear(self.h, _p(a)))

    def slow_none(self):
        self._check(self.L.mr_slow_none(self.h))

    # ---- state ---------------------------------------------------------------
    def upload(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        assert y.size == self.dof, (y.size, self.dof)
        self._check(self.L.mr_state_upload(self.h, _p(y)))

    def download(self, out=None):
        y = np.empty(self.dof) if out is None else out
        self._check(self.L.mr_state_download(self.h, _p(y)))
        return y

    def state_ptr(self):
        return self.L.mr_state_device_ptr(self.h)

    # ---- stepping ---------------------------------------------------------------
    @staticmethod
    def counters():
        return np.zeros(8, dtype=np.uint64)

    def mri_step(self, t, H, counters=None):
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_mri_step(self.h, t, H, _p(cnt, _u64p), C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def mri_step_async(self, t, H, stream=None):
        """Enqueue one step after the work queued on `stream` (a cudaStream_t
        handle as int, or None for the legacy default stream); finish it with
        mri_step_wait."""
        self._check(self.L.mr_mri_step_async(self.h, t, H, stream))

    def mri_step_wait(self, counters=None):
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_mri_step_wait(self.h, _p(cnt, _u64p), C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def mri_integrate(self, t0, tf, H, counters=None):
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_mri_integrate(self.h, t0, tf, H, _p(cnt, _u64p), C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def mri_step_host(self, t, H, y_in, y_out, counters=None):
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_mri_step_host(self.h, t, H, _p(y_in), _p(y_out), _p(cnt, _u64p),
                                     C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def ark_imex_step(self, t, H, counters=None):
        """ark_imex_step (mri.cpp:437-522), ARK4(3)6L[2]SA, device state."""
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_ark_imex_step(self.h, t, H, _p(cnt, _u64p), C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def ark_imex_integrate(self, t0, tf, H, counters=None):
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_ark_imex_integrate(self.h, t0, tf, H, _p(cnt, _u64p), C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def reference_solution(self, t0, tf, h_ref):
        """reference_solution (erk.cpp:59-75): cash-karp5 on f_fast + f_implicit +
        f_explicit, applied to the device-resident state."""
        stage = C.c_int(-1)
        rc = self.L.mr_reference_solution(self.h, t0, tf, h_ref, C.byref(stage))
        self._check(rc, stage.value)

    def erk_integrate(self, table, t0, tf, h, counters=None):
        """erk_integrate (erk.cpp:40-57) of the summed RHS with an explicit table
        (name or dict): the harness's erk-<table> family.  Stage evaluations are
        counted into counters[MR_CNT_EXPLICIT_EVALS] like harness.cpp:353-354."""
        t = tables.lookup_table(table) if isinstance(table, str) else table
        A = np.ascontiguousarray(t["A"], dtype=np.float64)
        b = np.ascontiguousarray(t["b"], dtype=np.float64)
        c = np.ascontiguousarray(t["c"], dtype=np.float64)
        cnt = self.counters() if counters is None else counters
        ev = np.zeros(1, dtype=np.uint64)
        stage = C.c_int(-1)
        rc = self.L.mr_erk_integrate(self.h, len(b), _p(A), _p(b), _p(c), t0, tf, h,
                                     _p(ev, _u64p), C.byref(stage))
        cnt[2] += ev[0]
        self._check(rc, stage.value)
        return cnt

    # ---- spectral deferred corrections (proj/src/sdc.cpp) -------------------
    def sdc_integrate(self, n_nodes, sweeps, t0, tf, H, counters=None):
        """sdc_integrate (sdc.cpp:267-281) of f_fast + f_implicit + f_explicit
        with lobatto_nodes(n_nodes) and `sweeps` correction sweeps: the
        harness's sdc family; evaluations into counters[MR_CNT_EXPLICIT_EVALS]
        (harness.cpp:356-366)."""
        nodes, S = lobatto_rule(n_nodes)
        cnt = self.counters() if counters is None else counters
        ev = np.zeros(1, dtype=np.uint64)
        stage = C.c_int(-1)
        rc = self.L.mr_sdc_integrate(self.h, n_nodes, _p(nodes), _p(S), sweeps, t0, tf, H,
                                     _p(ev, _u64p), C.byref(stage))
        cnt[2] += ev[0]
        self._check(rc, stage.value)
        return cnt

    def mrsdc_build(self, X, Y, Z, sweeps):
        """build_scheme(X, Y, Z, sweeps) (sdc.cpp:82-153) for mrsdc_integrate."""
        self._check(self.L.mr_mrsdc_build(self.h, X, Y, Z, sweeps))

    def mrsdc_load(self, scheme, sweeps):
        """Load a flattened MRSDC scheme (mrsdc_scheme(), or the reference's
        build_scheme) for mrsdc_integrate."""
        ints = ("coarse_of_fine", "coarse_index_of_fine", "application_offset")
        sc = {k: np.ascontiguousarray(v, dtype=np.int32 if k in ints else np.float64)
              for k, v in scheme.items() if k not in ("X", "Y", "n_fine")}
        self._check(self.L.mr_mrsdc_load(
            self.h, scheme["X"], scheme["Y"], scheme["n_fine"], sweeps,
            _p(sc["coarse_nodes"]), _p(sc["fine_nodes"]), _p(sc["coarse_of_fine"], _ip),
            _p(sc["coarse_index_of_fine"], _ip), _p(sc["fine_row"]),
            _p(sc["application_offset"], _ip), _p(sc["coarse_row"])))

    def mrsdc_integrate(self, t0, tf, H, counters=None):
        """mrsdc_integrate (sdc.cpp:283-301) of the loaded scheme: the harness's
        mrsdc-XYZ family."""
        cnt = self.counters() if counters is None else counters
        stage = C.c_int(-1)
        rc = self.L.mr_mrsdc_integrate(self.h, t0, tf, H, _p(cnt, _u64p), C.byref(stage))
        self._check(rc, stage.value)
        return cnt

    def last_host_step_bytes(self):
        """(H2D, D2H) bytes the last mri_step_host moved over PCIe."""
        a, b = C.c_uint64(), C.c_uint64()
        self._check(self.L.mr_last_host_step_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def last_failure(self):
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        self.L.mr_last_failure(self.h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def fast_rhs(self, y, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        self._check(self.L.mr_fast_rhs(self.h, t, _p(y), _p(out)))
        return out

    def slow_rhs(self, y, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        self._check(self.L.mr_slow_rhs(self.h, t, _p(y), _p(out)))
        return out

    def implicit_rhs(self, y, t=0.0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        self._check(self.L.mr_implicit_rhs(self.h, t, _p(y), _p(out)))
        return out

    # ---- reductions over device pointers (state by default) ---------------
    def _red(self, fn, *args):
        out = C.c_double()
        self._check(fn(self.h, *args, C.byref(out)))
        return out.value

    def wrms_norm(self, x_ptr, w_ptr, n):
        return self._red(self.L.mr_wrms_norm, x_ptr, w_ptr, n)

    def two_norm(self, x_ptr, n):
        return self._red(self.L.mr_two_norm, x_ptr, n)

    def dot(self, x_ptr, y_ptr, n):
        return self._red(self.L.mr_dot, x_ptr, y_ptr, n)

    def max_norm(self, x_ptr, n):
        return self._red(self.L.mr_max_norm, x_ptr, n)

    def max_norm_component(self, x_ptr, n, offset, count):
        return self._red(self.L.mr_max_norm_component, x_ptr, n, offset, count)

    def all_finite(self, x_ptr, n):
        out = C.c_int()
        self._check(self.L.mr_all_finite(self.h, x_ptr, n, C.byref(out)))
        return bool(out.value)

    # ---- instrumentation ---------------------------------------------------
    def stream(self):
        return self.L.mr_stream(self.h)

    def launch_count(self):
        return int(self.L.mr_launch_count(self.h))

    def chem_flops_per_eval(self):
        return float(self.L.mr_chem_flops_per_eval(self.h))

    def fp64_peak(self):
        out = C.c_double()
        self._check(self.L.mr_fp64_peak(self.h, C.byref(out)))
        return out.value

    def set_profiling(self, on=True):
        self._check(self.L.mr_set_profiling(self.h, int(on)))

    def last_step_profile(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._check(self.L.mr_last_step_profile(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    # ---- multi-GPU -----------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        _bind_process_nccl()
        buf = C.create_string_buffer(128)
        if lib().mr_nccl_unique_id(buf):
            raise CudaError("ncclGetUniqueId failed")
        return buf.raw

    def comm_init(self, nranks, rank, uid: bytes):
        _bind_process_nccl()
        self._check(self.L.mr_comm_init(self.h, nranks, rank, uid))

    def comm_init_loopback(self):
        """One-rank NCCL communicator: the multi-GPU rank's code path on one GPU."""
        _bind_process_nccl()
        self._check(self.L.mr_comm_init_loopback(self.h))


def group_step(ctxs, t, H, counters=None):
    """One slow step of several slab contexts on one device ("virtual ranks")."""
    L = lib()
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    cnt = Context.counters() if counters is None else counters
    stage = C.c_int(-1)
    rc = L.mr_group_step(arr, len(ctxs), t, H, _p(cnt, _u64p), C.byref(stage))
    ctxs[0]._check(rc, stage.value)
    return cnt


def slab_bounds(n0: int, nranks: int, rank: int):
    """Slab decomposition along axis 0: equal slabs, remainder to the first ranks."""
    base, rem = divmod(n0, nranks)
    n0l = base + (1 if rank < rem else 0)
    i0 = rank * base + min(rank, rem)
    return i0, n0l


def setup_workload(ctx: Context, name: str, *, n=None, i0=0, n0_local=None, threads=0,
                   make_state=True, config=None, ymax=None):
    """Configure ctx for a BASELINE.json workload (C1-C5), optionally on a
    smaller grid n and a slab [i0, i0+n0_local); returns (cfg, y0)."""
    cfg = dict(CONFIGS[name] if config is None else config)
    if n is not None:
        cfg["n"] = n
    N = cfg["n"]
    S, R = cfg["S"], cfg["R"]
    n0l = N if n0_local is None else n0_local
    ctx.grid(N, N, N, S + 1, 1.0, i0, n0l)
    ctx.method(cfg["coupling"], cfg["fast_table"], cfg["m"])
    sp, rx, rs = mechanism(cfg["mech_seed"], S, R)
    ctx.fast_chemistry(S, R, cfg["rho"], sp, rx, rs)
    if cfg["velocity"] == "uniform":
        ctx.slow_stencil(cfg["order"], cfg["diffusion"], u=cfg["u"])
    else:
        ctx.slow_stencil(cfg["order"], cfg["diffusion"],
                         prof=velocity_profiles(cfg["vel_seed"], N, N, N))
    if cfg.get("d_impl") is not None:
        ctx.slow_implicit_diffusion(cfg["d_impl"], cfg["cg_iters"])
    y0 = None
    if make_state:
        y0 = initial_condition(cfg["ic_seed"], S, cfg["rho"], sp, N, N, N, 1.0, i0, n0l, threads)
        ctx.upload(y0)
        if cfg.get("d_impl") is not None:
            tol, safety, mx, w = stage_solver(y0, ymax)
            ctx.newton_config(tol, safety, mx, w)
    cfg["mech"] = (sp, rx, rs)
    return cfg, y0
