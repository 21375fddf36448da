"""Small workloads that launch every product kernel once or a few times, for
compute-sanitizer (memcheck / racecheck / synccheck; one tool per run):
  * C4 chemistry chains (1024-thread block, shared-memory phases) on 8^3
  * C3 64^3 transport step: the order-8 ring stencil (TMA + mbarrier ring)
  * the NCCL rank path on one GPU (loopback communicator): halo pack, grouped
    send/recv, interior + boundary plane ranges
  * C5 physics IMEX step at a transport-scale H: tiled L7 kernels, CG updates,
    dot-product partials, fI recovery
  * a two-slab multi-device domain (peer copies, gathered dot products)
Usage: compute-sanitizer --tool <tool> python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_03293_b200 as P  # noqa: E402
from paper_2211_03293_b200.configs import CONFIGS  # noqa: E402

ctx = P.Context(0)
cfg, y0 = P.setup_workload(ctx, "C4", n=8)
ctx.mri_step(0.0, cfg["H"])
print("C4 8^3 step ok", flush=True)

t = dict(CONFIGS["C3"], m=2)
ctx = P.Context(0)
cfg, y0 = P.setup_workload(ctx, "C3", n=64, config=t, threads=0)
ctx.fast_none()
ctx.mri_step(0.0, 2e-4)
print("C3 64^3 ring-stencil step ok", flush=True)

ctx = P.Context(0)
ctx.comm_init_loopback()
cfg, y0 = P.setup_workload(ctx, "C3", n=64, config=t, threads=0)
ctx.fast_none()
ctx.mri_step(0.0, 2e-4)
print("C3 64^3 NCCL loopback step ok", flush=True)

c5 = dict(CONFIGS["C5"], d_impl=0.05, cg_iters=3, m=2)
ctx = P.Context(0)
cfg, y0 = P.setup_workload(ctx, "C5", n=64, config=c5, threads=0)
ctx.fast_none()
cnt = ctx.counters()
try:  # the kernels run either way; Newton may need more than 5 iterations here
    ctx.mri_step(0.0, 2e-3, cnt)
except P.IntegrationError as e:
    print("  (", e, ")")
print("C5 64^3 IMEX step ran, Newton iterations", int(cnt[4]), flush=True)

dom = P.Context([0, 0])
cfg, y0 = P.setup_workload(dom, "C5", n=16, config=c5, threads=0)
dom.fast_none()
dom.mri_step(0.0, 2e-3)
print("two-slab domain IMEX step ok", flush=True)
