"""CPU, world_size 2 and 3 over gloo: the slab decomposition the library uses
for multi-GPU runs, checked end to end on the CPU.

Each rank owns planes slab_bounds(n0, P, r) of axis 0, generates its slab of
the seeded initial condition with the product's host generator, packs its
first / last g planes of every component exactly as launch_halo_pack does,
exchanges them with its periodic neighbours in the order exchange_halos issues
the NCCL calls (send_lo -> left, recv_hi <- right, send_hi -> right,
recv_lo <- left) and evaluates the 8th-order stencil on the slab + halos.
The result must equal the oracle's single-domain stencil on the same planes,
and the gathered slabs must reproduce the global initial condition bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def stencil_with_halos(y, lo, hi, n0l, n1, n2, ncomp, order, D, prof_u, i0, n0g, length=1.0):
    """numpy restatement of stencil_kernel (kernels_slow.cu) on one slab."""
    a = {2: [0, 1 / 2], 4: [0, 2 / 3, -1 / 12], 8: [0, 4 / 5, -1 / 5, 4 / 105, -1 / 280]}[order]
    b = {2: [-2, 1], 4: [-5 / 2, 4 / 3, -1 / 12],
         8: [-205 / 72, 8 / 5, -1 / 5, 8 / 315, -1 / 560]}[order]
    M = order // 2
    Y = y.reshape(ncomp, n0l, n1, n2)
    ext = np.concatenate([lo.reshape(ncomp, M, n1, n2), Y, hi.reshape(ncomp, M, n1, n2)], axis=1)
    out = np.zeros_like(Y)
    dx = [length / n0g, length / n1, length / n2]
    u = prof_u
    for d in range(3):
        adv = np.zeros_like(Y)
        dif = b[0] * Y
        for m in range(1, M + 1):
            if d == 0:
                yp = ext[:, M + m:M + m + n0l]
                ym = ext[:, M - m:M - m + n0l]
            else:
                yp = np.roll(Y, -m, axis=d + 1)
                ym = np.roll(Y, m, axis=d + 1)
            adv = adv + a[m] * (yp - ym)
            dif = dif + b[m] * (yp + ym)
        out = out + (D / dx[d] ** 2) * dif - (u[d] / dx[d]) * adv
    return out.ravel()


def _worker(rank, world, port, n, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    import paper_2211_03293_b200 as P
    from paper_2211_03293_b200.configs import CONFIGS

    cfg = CONFIGS["C3"]
    S, R = cfg["S"], cfg["R"]
    ncomp = S + 1
    M = 4
    i0, n0l = P.slab_bounds(n, world, rank)
    sp, rx, rs = P.mechanism(cfg["mech_seed"], S, R)
    y = P.initial_condition(cfg["ic_seed"], S, cfg["rho"], sp, n, n, n, 1.0, i0, n0l)
    Y = y.reshape(ncomp, n0l, n * n)
    send_lo = np.ascontiguousarray(Y[:, :M])
    send_hi = np.ascontiguousarray(Y[:, n0l - M:])
    left, right = (rank - 1) % world, (rank + 1) % world
    recv_lo = torch.empty(send_lo.size, dtype=torch.float64)
    recv_hi = torch.empty(send_hi.size, dtype=torch.float64)
    ops = [dist.P2POp(dist.isend, torch.from_numpy(send_lo.ravel().copy()), left),
           dist.P2POp(dist.irecv, recv_hi, right),
           dist.P2POp(dist.isend, torch.from_numpy(send_hi.ravel().copy()), right),
           dist.P2POp(dist.irecv, recv_lo, left)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    u = (1.0, 1.0, 1.0)
    f = stencil_with_halos(y, recv_lo.numpy(), recv_hi.numpy(), n0l, n, n, ncomp, 8, 1e-3, u, i0, n)
    # oracle on the full domain, restricted to this slab
    mech = O.mechanism(cfg["mech_seed"], S, R)
    full = O.System(n, n, n, ncomp, fast="chem", slow="stencil", mech=mech, S=S, R=R,
                    order=8, diffusion=1e-3, u=u)
    yfull = full.initial_condition(cfg["ic_seed"])
    ref = full.slow_rhs(yfull).reshape(ncomp, n, n * n)[:, i0:i0 + n0l].ravel()
    ic_ok = np.array_equal(y, yfull.reshape(ncomp, n, n * n)[:, i0:i0 + n0l].ravel())
    scale = np.abs(ref).reshape(ncomp, -1).max(axis=1)
    err = (np.abs(f - ref).reshape(ncomp, -1).max(axis=1) / scale).max()
    result_q.put((rank, bool(ic_ok), float(err), i0, n0l))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 12), (3, 13)])
def test_slab_halo_exchange_gloo(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    covered = sum(r[4] for r in res)
    assert covered == n and res[0][3] == 0
    for rank, ic_ok, err, i0, n0l in res:
        assert ic_ok, f"rank {rank}: slab IC differs from the global field"
        assert err <= 1e-12, f"rank {rank}: slab stencil differs from the global stencil ({err})"


def test_slab_bounds_partition():
    import sys
    sys.path.insert(0, ROOT)
    import paper_2211_03293_b200 as P
    for n0 in (8, 13, 256, 384):
        for world in (1, 2, 3, 4, 8):
            spans = [P.slab_bounds(n0, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (a, la), (b, lb) in zip(spans, spans[1:]):
                assert a + la == b
            assert spans[-1][0] + spans[-1][1] == n0
            assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1
