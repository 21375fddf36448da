"""Single-process multi-GPU domain (mr_ctx_create_multi).

The reference's caller is one single-threaded process (proj/README.md:132-134,
proj/src/harness.cpp:374-382); through the facade that process drives N GPUs
with one domain context: slabs along axis 0 in device order, each on its own
stream, ghost planes copied peer-to-peer with events, IMEX dot products summed
in slab order.  On a one-GPU box the same code runs with a device listed
several times (every slab its own stream, cross-stream events, device-local
peer copies); the real two-GPU test runs where two are visible.  Results must
be bitwise equal to the single context (explicit couplings: the stencil sees
the same ghost values, the chemistry is cell-local) and to the in-process
virtual ranks for IMEX (same slab-ordered dot products)."""
import numpy as np
import pytest

import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def _n_gpus():
    import torch
    return torch.cuda.device_count()


def _setup(dev, name, n, cfg=None, fast_none=False):
    ctx = P.Context(dev)
    cfg_, y0 = P.setup_workload(ctx, name, n=n, config=cfg, threads=0)
    if fast_none:
        ctx.fast_none()
    return ctx, cfg_, y0


@pytest.mark.parametrize("devs", [[0, 0], [0, 0, 0]])
def test_domain_explicit_steps_bitwise_equal_single(devs):
    """C3 physics on 64^3 (ring-tiled 8th-order stencil, chemistry chains),
    two steps through mri_integrate: state and counters bitwise equal."""
    one, cfg, y0 = _setup(0, "C3", 64)
    dom, _, _ = _setup(devs, "C3", 64)
    H = cfg["H"]
    c1 = one.mri_integrate(0.0, 2 * H, H)
    c2 = dom.mri_integrate(0.0, 2 * H, H)
    assert np.array_equal(c1, c2)
    assert np.array_equal(one.download(), dom.download())


def test_domain_c4_step_and_host_buffer_step():
    """The 53-species mechanism (two-cells-per-thread kernel) and the
    host-buffer step (scatter / step / gather)."""
    one, cfg, y0 = _setup(0, "C4", 32)
    dom, _, _ = _setup([0, 0], "C4", 32)
    H = cfg["H"]
    c1 = one.mri_step(0.0, H)
    y_out = np.zeros_like(y0)
    c2 = dom.mri_step_host(0.0, H, y0, y_out)
    assert np.array_equal(c1, c2)
    assert np.array_equal(one.download(), y_out)


def test_domain_transport_scale_bitwise():
    """Fast partition off, H = 2e-4: the transport dominates the update."""
    cfg = dict(CONFIGS["C3"], m=4)
    one, cfg, y0 = _setup(0, "C3", 64, cfg, fast_none=True)
    dom, _, _ = _setup([0, 0, 0, 0], "C3", 64, cfg, fast_none=True)
    one.mri_step(0.0, 2e-4)
    dom.mri_step(0.0, 2e-4)
    assert np.array_equal(one.download(), dom.download())


def test_domain_imex_newton_pcg_equals_virtual_ranks():
    """C5 physics with a transport-scale H: Newton iterates and every CG dot
    product is gathered across the slabs -- bitwise the virtual ranks'."""
    cfg0 = dict(CONFIGS["C5"], d_impl=0.05, cg_iters=3, m=4)
    n, H, P_ = 16, 2e-3, 2
    dom = P.Context([0] * P_)
    cfg, y0 = P.setup_workload(dom, "C5", n=n, config=cfg0, threads=0)
    dom.fast_none()
    virt = []
    for r in range(P_):
        i0, n0l = P.slab_bounds(n, P_, r)
        c = P.Context(0)
        P.setup_workload(c, "C5", n=n, config=cfg0, i0=i0, n0_local=n0l, threads=0, ymax=np.abs(y0).max())
        c.fast_none()
        virt.append(c)
    c_dom = dom.mri_step(0.0, H)
    c_virt = P.group_step(virt, 0.0, H)
    assert c_dom[4] > 0  # Newton iterated
    assert np.array_equal(c_dom, c_virt)
    y = dom.download().reshape(cfg["S"] + 1, n, n, n)
    for r, c in enumerate(virt):
        i0, n0l = P.slab_bounds(n, P_, r)
        assert np.array_equal(c.download().reshape(cfg["S"] + 1, n0l, n, n), y[:, i0:i0 + n0l])


def test_domain_rhs_ark_and_reference_solution():
    """Mode-A RHS evaluations, the ARK-IMEX step and the cash-karp5
    reference solution over a domain equal the single context."""
    cfg0 = dict(CONFIGS["C5"], d_impl=0.05, cg_iters=3, m=4)
    one, cfg, y0 = _setup(0, "C5", 16, cfg0)
    dom, _, _ = _setup([0, 0], "C5", 16, cfg0)
    assert np.array_equal(one.fast_rhs(y0), dom.fast_rhs(y0))
    assert np.array_equal(one.slow_rhs(y0), dom.slow_rhs(y0))
    assert np.array_equal(one.implicit_rhs(y0), dom.implicit_rhs(y0))
    h = 1e-16
    one.reference_solution(0.0, 3 * h, h)
    dom.reference_solution(0.0, 3 * h, h)
    assert np.array_equal(one.download(), dom.download())
    one.upload(y0)
    dom.upload(y0)
    H = 1e-17  # the ARK explicit part carries the stiff chemistry
    c1 = one.ark_imex_step(0.0, H)
    c2 = dom.ark_imex_step(0.0, H)
    assert np.array_equal(c1[[0, 1, 2, 3, 7]], c2[[0, 1, 2, 3, 7]])
    rel = np.abs(one.download() - dom.download()).max() / np.abs(one.download()).max()
    assert rel <= 1e-13


def test_domain_failure_restores_every_slab_and_contracts():
    one, cfg, y0 = _setup(0, "C3", 16)
    dom, _, _ = _setup([0, 0], "C3", 16)
    bad = y0.copy()
    bad[-5] = np.nan  # the last slab's last cell
    one.upload(bad)
    dom.upload(bad)
    H = cfg["H"]
    with pytest.raises(P.IntegrationError) as e1:
        one.mri_integrate(0.0, 3 * H, H)
    c = dom.counters()
    with pytest.raises(P.IntegrationError) as e2:
        dom.mri_integrate(0.0, 3 * H, H, c)
    assert e1.value.stage_index == e2.value.stage_index
    assert np.array_equal(dom.download(), bad, equal_nan=True)
    assert not dom.state_ptr()
    with pytest.raises(P.ContractError):
        dom.max_norm(0, 1)
    with pytest.raises(P.ContractError):
        dom.mri_step_async(0.0, H)
    with pytest.raises(P.ContractError):
        dom.grid(16, 16, 16, cfg["S"] + 1, 1.0, 0, 8)  # a domain owns the whole grid


@pytest.mark.skipif(_n_gpus() < 2, reason="needs two visible GPUs")
def test_two_gpu_domain_bitwise_equal_one_gpu():
    """Two real GPUs (peer copies over NVLink): bitwise the one-GPU result,
    explicit (C3 64^3) and IMEX (C5 physics, Newton-PCG across the GPUs)."""
    one, cfg, y0 = _setup(0, "C3", 64)
    dom, _, _ = _setup([0, 1], "C3", 64)
    H = cfg["H"]
    assert np.array_equal(one.mri_integrate(0.0, 2 * H, H), dom.mri_integrate(0.0, 2 * H, H))
    assert np.array_equal(one.download(), dom.download())
    cfg0 = dict(CONFIGS["C5"], d_impl=0.05, cg_iters=3, m=4)
    same, _, y5 = _setup([0, 0], "C5", 16, cfg0, fast_none=True)
    two, _, _ = _setup([0, 1], "C5", 16, cfg0, fast_none=True)
    assert np.array_equal(same.mri_step(0.0, 2e-3), two.mri_step(0.0, 2e-3))
    assert np.array_equal(same.download(), two.download())


def test_domain_sdc_and_mrsdc_bitwise_equal_single():
    """The SDC engine over a domain (per-slab caches, the slow evaluations
    with slab ghost exchange): sdc-2 and mrsdc-335 on C3 physics at 64^3
    (ring-tiled stencil) bitwise equal the single context, counters too."""
    one, cfg, y0 = _setup(0, "C3", 64)
    dom, _, _ = _setup([0, 0], "C3", 64)
    h = cfg["H"] / cfg["m"]
    c1 = one.sdc_integrate(3, 2, 0.0, 2 * h, h)
    c2 = dom.sdc_integrate(3, 2, 0.0, 2 * h, h)
    assert np.array_equal(c1, c2)
    assert np.array_equal(one.download(), dom.download())
    one.upload(y0)
    dom.upload(y0)
    one.mrsdc_build(3, 3, 5, 2)
    dom.mrsdc_build(3, 3, 5, 2)
    Hm = cfg["H"] / 2
    c1 = one.mrsdc_integrate(0.0, Hm, Hm)
    c2 = dom.mrsdc_integrate(0.0, Hm, Hm)
    assert np.array_equal(c1, c2)
    assert np.array_equal(one.download(), dom.download())
