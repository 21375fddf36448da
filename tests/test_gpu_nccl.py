"""The NCCL path of the slab decomposition on one GPU: a one-rank NCCL
communicator (mr_comm_init_loopback) sends the halo planes to itself with grouped
ncclSend/ncclRecv, all-reduces the failure key and all-gathers the CG dot
products -- every collective the multi-GPU run issues.  Its
results must equal the plain single-slab path bit for bit (same data, same
order), and its counters exactly."""
import numpy as np
import pytest

import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def _pair(monkeypatch, name, n, cfg):
    plain = P.Context(0)
    P.setup_workload(plain, name, n=n, config=cfg)
    nccl = P.Context(0)
    nccl.comm_init_loopback()
    cfg_, y0 = P.setup_workload(nccl, name, n=n, config=cfg)
    return plain, nccl, cfg_, y0


def test_nccl_self_explicit_steps_bitwise(monkeypatch):
    """C3 physics (8th-order stencil with halo exchange, chemistry chains)."""
    plain, nccl, cfg, _ = _pair(monkeypatch, "C3", 16, dict(CONFIGS["C3"]))
    H = cfg["H"]
    c_a = plain.mri_integrate(0.0, 2 * H, H)
    c_b = nccl.mri_integrate(0.0, 2 * H, H)
    assert np.array_equal(c_a, c_b)
    assert np.array_equal(plain.download(), nccl.download())


def test_nccl_self_imex_newton_pcg_bitwise(monkeypatch):
    """C5 physics with a transport-scale H: Newton iterates, every CG dot
    product goes through ncclAllGather + the fixed-order sum."""
    cfg0 = dict(CONFIGS["C5"], d_impl=0.05, cg_iters=3, m=4)
    plain, nccl, cfg, _ = _pair(monkeypatch, "C5", 12, cfg0)
    plain.fast_none()
    nccl.fast_none()
    H = 2e-3
    c_a = plain.mri_integrate(0.0, 2 * H, H)
    c_b = nccl.mri_integrate(0.0, 2 * H, H)
    assert np.array_equal(c_a, c_b)
    assert c_a[4] > c_a[3]  # Newton iterated (linear iterations > solves)
    assert np.array_equal(plain.download(), nccl.download())


def test_nccl_self_failure_key_allreduce(monkeypatch):
    """A blow-up is reported with the same stage through the all-reduced key."""
    plain, nccl, cfg, y0 = _pair(monkeypatch, "C3", 16, dict(CONFIGS["C3"]))
    bad = y0.copy()
    bad[5] = np.nan
    errs = []
    for ctx in (plain, nccl):
        ctx.upload(bad)
        with pytest.raises(P.IntegrationError) as e:
            ctx.mri_step(0.0, cfg["H"])
        errs.append(e.value.stage_index)
    assert errs[0] == errs[1]


def test_nccl_self_overlapped_halo_bitwise(monkeypatch):
    """On a grid the ring stencil tiles (64^3, order 8) the NCCL rank overlaps
    the halo exchange (comm stream) with the interior planes and finishes the
    ghost-dependent planes after it: still bitwise equal to the plain path."""
    plain, nccl, cfg, y0 = _pair(monkeypatch, "C3", 64, dict(CONFIGS["C3"]))
    H = cfg["H"]
    n_before = nccl.launch_count()
    c_a = plain.mri_step(0.0, H)
    c_b = nccl.mri_step(0.0, H)
    assert np.array_equal(c_a, c_b)
    assert np.array_equal(plain.download(), nccl.download())
    # the stencil evaluations ran as interior + two boundary launches
    assert nccl.launch_count() - n_before > plain.launch_count()
    # slow RHS alone (through the same path as a step's evaluations)
    assert np.array_equal(plain.slow_rhs(y0), nccl.slow_rhs(y0))


def test_bench_nccl_self_line():
    """bench.py --nccl-self (a multi-GPU rank's code path on one GPU) prints a
    valid contract line."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "C3", "--n", "64",
                          "--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e", "--nccl-self"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "one-rank NCCL path" in line["config"]["parallelism"]
    assert line["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.parametrize("pipelined", [False, True])
@pytest.mark.parametrize("name", ["C4", "C3"])
def test_nccl_self_host_step_bitwise(monkeypatch, name, pipelined):
    """The host-buffer step of an NCCL rank at 64^3 -- plain copies (the
    default on ranks) and the chunk-pipelined schedule in which the end
    chunks' slow evaluations wait for the exchanged ghosts (enabled through
    the debug switch) -- bitwise the plain device step, counters equal; a
    failing host step leaves y_out untouched."""
    import ctypes as C
    import torch
    plain, nccl, cfg, y0 = _pair(monkeypatch, name, 64, dict(CONFIGS[name]))
    f = P.lib().mr_debug_pipeline_nccl
    f.argtypes = [C.c_void_p, C.c_int]
    assert f(nccl.h, int(pipelined)) == 0
    H = cfg["H"]
    c_a = plain.mri_step(0.0, H)
    y_in = torch.from_numpy(y0.copy()).pin_memory().numpy()
    y_out = torch.zeros(y0.size, dtype=torch.float64).pin_memory().numpy()
    c_b = nccl.counters()
    nccl.mri_step_host(0.0, H, y_in, y_out, c_b)
    assert np.array_equal(c_a, c_b)
    assert np.array_equal(plain.download(), y_out)
    bad = y_in.copy()
    bad[-3] = np.nan
    y_out[:] = 7.0
    with pytest.raises(P.IntegrationError):
        nccl.mri_step_host(0.0, H, bad, y_out)
    assert np.all(y_out == 7.0)
