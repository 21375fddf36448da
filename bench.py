#!/usr/bin/env python
"""Benchmark: MRI slow-step cell-updates/s on BASELINE.json config C4
(256^3 grid, 53 species / 325 reactions, 8th-order stencil, explicit
MRI-GARK-ERK45a stand-in + RK4, H/h = 50) -- one slow step of the whole grid
per "step".  Multi-GPU: the 256^3 grid is slab-decomposed over the ranks
(strong scaling), halos exchanged with NCCL inside the library.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C4]

Prints ONE JSON line on rank 0 (contract in the task statement).  Timed with
CUDA events on the library's stream; max over ranks.  `e2e` re-times the same
steps through the host-buffer C-ABI call (pinned H2D of the state, the step,
D2H of the result).  `cpu_baseline` / `--impl reference` time the reference's
own stepper (oracle/_ref, compiled from /root/reference) driving the CPU
physics on a bounded sub-grid sample, with all host cores in the callbacks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MRI slow-step cell-updates/s (256^3, 53 sp) + chem RHS cells/s, % roofline"
UNIT = "cell-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def ncu_traffic(n):
    """DRAM bytes per launch of the dominant kernels from the committed
    ncu --set full captures (profiles/<latest round>/traffic.json), only from
    captures taken at the benched grid size n (a smaller grid's state fits the
    126 MB L2 and would under-report DRAM traffic)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")))
    if not files:
        return {}
    try:
        tr = json.load(open(files[-1]))
    except (OSError, ValueError):
        return {}
    return {k: v for k, v in tr.items() if isinstance(v, dict) and v.get("grid") == n}


def cpu_reference_sample(cfg_name, n_sample, steps, threads):
    """Time the reference's own mri_step (oracle/_ref) with the CPU physics on
    an n_sample^3 sub-grid of the workload (same mechanism, method, m, stencil)."""
    import oracle as O
    from paper_2211_03293_b200.configs import CONFIGS
    cfg = CONFIGS[cfg_name]
    S, R = cfg["S"], cfg["R"]
    n = n_sample
    mech = O.mechanism(cfg["mech_seed"], S, R)
    prof = O.velocity_profiles(cfg["vel_seed"], n, n, n) if cfg["velocity"] == "random" else None

    def make(**kw):
        return O.System(n, n, n, S + 1, fast="chem", slow="stencil", mech=mech, S=S, R=R,
                        rho=cfg["rho"], order=cfg["order"], diffusion=cfg["diffusion"],
                        u=cfg["u"] or (1.0, 1.0, 1.0), prof=prof, threads=threads, **kw)
    sysm = make()
    y = sysm.initial_condition(cfg["ic_seed"])
    if cfg.get("d_impl") is not None:  # IMEX: f_implicit + the workload's stage solver
        from paper_2211_03293_b200.configs import stage_solver
        tol, safety, mx, w = stage_solver(y)
        sysm = make(imex=True, d_impl=cfg["d_impl"], cg_iters=cfg["cg_iters"],
                    newton=(tol, safety, mx), newton_weights=w)
    use_ref = os.path.exists(O.REF_LIB)
    cp = "mis-kw3" if cfg["coupling"] == "mis-kw3" else open(
        os.path.join(ROOT, "paper_2211_03293_b200", "data", "couplings",
                     f"{cfg['coupling']}.txt")).read()
    H = cfg["H"]
    t0 = time.perf_counter()
    for i in range(steps):
        y, _ = sysm.mri_step(cp, cfg["fast_table"], cfg["m"], i * H, H, y, use_reference=use_ref)
    dt = time.perf_counter() - t0
    return {"value": n ** 3 * steps / dt, "unit": UNIT, "cores": threads,
            "kind": "reference" if use_ref else "port",
            "sample": f"{steps} slow step(s) of the {cfg_name} mechanism/method on a {n}^3 "
                      f"sub-grid ({n ** 3} cells); reference mri_step + CPU physics callbacks "
                      f"on {threads} host threads",
            "seconds": dt}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":  # host-only arm: ranks only meet at a barrier
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local, dist


def run_reference(args):
    world, rank, local, dist = dist_setup(args)
    if rank != 0:
        if dist:
            dist.barrier()
        return
    threads = os.cpu_count() or 1
    n_sample = args.sample_n
    cpu_reference_sample(args.config, n_sample, 1, threads)  # warm-up (page-in)
    r = cpu_reference_sample(args.config, n_sample, args.steps, threads)
    from paper_2211_03293_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * r["seconds"] / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['n']}^3 grid, {cfg['S']} species / "
                                   f"{cfg['R']} reactions, {cfg['coupling']} + {cfg['fast_table']}, "
                                   f"m={cfg['m']}, order {cfg['order']} (CPU sample {n_sample}^3)",
                       "parallelism": "host threads"},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()


def run_ours(args):
    import torch

    import paper_2211_03293_b200 as P
    from paper_2211_03293_b200.configs import CONFIGS

    world, rank, local, dist = dist_setup(args)
    cfg0 = CONFIGS[args.config]
    n = args.n or cfg0["n"]
    S = cfg0["S"]
    i0, n0l = P.slab_bounds(n, world, rank)
    if args.slab_of and world == 1:
        # one rank's slab of a slab_of-GPU run, periodic onto itself: the
        # per-GPU work of that run without its halo traffic
        i0, n0l = P.slab_bounds(n, args.slab_of, 0)
    ctx = P.Context(local)
    if world > 1:
        uid = [P.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])
    elif args.nccl_self:
        # one-rank NCCL communicator: the multi-GPU rank's code path (pack,
        # grouped send/recv on the comm stream overlapped with the interior
        # stencil, boundary planes, all-reduced failure key) on one GPU
        ctx.comm_init_loopback()
    t_setup = time.perf_counter()
    cfg, y0 = P.setup_workload(ctx, args.config, n=n, i0=i0, n0_local=n0l, threads=0)
    if cfg.get("d_impl") is not None and dist:
        # stage-solver weights use the GLOBAL max|y0| (configs.stage_solver)
        import numpy as np
        from paper_2211_03293_b200.configs import stage_solver
        t_ = torch.tensor([float(np.abs(y0).max())], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        tol, safety, mx, w = stage_solver(y0, float(t_.item()))
        ctx.newton_config(tol, safety, mx, w)
    setup_s = time.perf_counter() - t_setup
    H = cfg["H"]
    fp64_peak = ctx.fp64_peak()
    ncell_local = n0l * n * n
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cnt = ctx.counters()
    t = 0.0
    for i in range(args.warmup):
        ctx.mri_step(t, H, cnt)
        t += H

    # ---------------- timed region (device-resident inputs) ----------------
    launches0 = ctx.launch_count()
    cnt_t = ctx.counters()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(local)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            ctx.mri_step(t, H, cnt_t)
            t += H
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize(local)
    barrier()
    launches = ctx.launch_count() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1))

    # ---------------- kernel split: the same K steps with per-launch events ----
    # (CUDA events around every launch on the library stream; a separate pass
    # so the per-launch event records do not perturb the timed region above)
    ctx.set_profiling(True)
    chem_ms = slow_ms = other_ms = 0.0
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(local)
    p0.record(stream)
    for i in range(args.steps):
        ctx.mri_step(t, H)
        t += H
        c, s_, o = ctx.last_step_profile()
        chem_ms += c
        slow_ms += s_
        other_ms += o
    p1.record(stream)
    p1.synchronize()
    ctx.set_profiling(False)
    profiled_ms = max_over_ranks(p0.elapsed_time(p1))
    chem_ms_max = max_over_ranks(chem_ms)
    slow_ms_max = max_over_ranks(slow_ms)
    ncell_job = float(n) ** 3 if world > 1 else float(ncell_local)  # cells all ranks own
    value = ncell_job * args.steps / (ms * 1e-3)
    evals_per_cell_step = int(cnt_t[0]) // args.steps
    chem_cells_per_s = ncell_job * evals_per_cell_step * args.steps / (chem_ms_max * 1e-3)
    flops_per_eval = ctx.chem_flops_per_eval()
    chem_tflops = ncell_local * evals_per_cell_step * args.steps * flops_per_eval / (
        chem_ms * 1e-3) / 1e12
    slow_evals = int(cnt_t[2]) // args.steps
    # explicit couplings: the forced final evaluation is unreferenced and only
    # counted (mri.cpp:162-166); IMEX couplings have no forced evaluation
    computed_slow = slow_evals if cfg.get("d_impl") is not None else max(slow_evals - 1, 1)
    stencil_bytes = 2.0 * 8 * (S + 1) * ncell_local * computed_slow * args.steps
    stencil_gbs = stencil_bytes / (slow_ms * 1e-3) / 1e9 if slow_ms > 0 else None
    pk = peaks()
    tr = ncu_traffic(n)

    # ---------------- end-to-end through the host-buffer C-ABI ----------------
    e2e = None
    if not args.no_e2e:
        dof = ctx.dof
        y_in = torch.empty(dof, dtype=torch.float64, pin_memory=True).numpy()
        y_out = torch.empty(dof, dtype=torch.float64, pin_memory=True).numpy()
        y_in[:] = y0
        e_steps = args.e2e_steps or args.steps
        barrier()
        torch.cuda.synchronize(local)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        te = 0.0
        for i in range(e_steps):
            ctx.mri_step_host(te, H, y_in, y_out)
            te += H
        e1.record(stream)
        e1.synchronize()
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1))
        # bytes the host-buffer call actually moved per step (the pipelined
        # step also saves y_out to the device, so H2D is twice the state)
        h2d, d2h = ctx.last_host_step_bytes()
        e2e = {"value": ncell_job * e_steps / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "input_bytes_per_step": 8 * dof * world, "steps": e_steps,
               "ms_per_step": ems / e_steps}

    # ---------------- CPU baseline (rank 0, N = 1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        r = cpu_reference_sample(args.config, args.sample_n, 1, threads)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        # the reference is single-threaded by design (proj/README.md:132-134):
        # also time it on one host thread, on a smaller sub-grid
        n1 = max(6, args.sample_n // 2)
        r1 = cpu_reference_sample(args.config, n1, 1, 1)
        cpu["single_thread"] = {k: r1[k] for k in ("value", "unit", "cores", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded mechanism + initial condition)",
            "config": {"workload": workload_text(args, cfg, n, n0l, H),
                       "grid": n, "species": S, "reactions": cfg["R"],
                       "parallelism": f"slab{world}" if world > 1 else (
                           (f"single GPU, slab 1/{args.slab_of}" if args.slab_of else "single GPU")
                           + (", one-rank NCCL path" if args.nccl_self else "")),
                       "l2": (f"inputs > L2 ({8 * (S + 1) * ncell_local / 1e9:.2f} GB state "
                              f"per GPU)") if 8 * (S + 1) * ncell_local > 126e6 else "fits L2"},
            "chem_rhs_cells_per_s": chem_cells_per_s,
            "roofline": {"bound": "fp64", "bound_note": "the fp64 pipe: no part of this path is a "
                                                        "dense contraction (north_star: tensor cores "
                                                        "are not used); K2 is judged on HBM below",
                         "kernel": "chain_kernel (fused fast IVP + chemistry)",
                         "achieved": chem_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": chem_tflops / fp64_peak if fp64_peak else None,
                         "traffic": tr.get("chem_chain", {}).get("dram_bytes_per_launch"),
                         "traffic_algorithmic": tr.get("chem_chain", {}).get(
                             "algorithmic_bytes_per_launch"),
                         "traffic_source": tr.get("chem_chain", {}).get("source"),
                         "flops_per_eval": flops_per_eval,
                         "ncu_fp64_pipe_pct": tr.get("chem_chain", {}).get("fp64_pipe_pct"),
                         "ncu_lsu_wavefronts_pct": tr.get("chem_chain", {}).get("lsu_wavefronts_pct"),
                         "peak_source": "DFMA-chain microbenchmark in this run (MEASURED_PEAKS.json "
                                        "has no fp64 figure)"},
            "roofline_stencil": {"bound": "hbm", "achieved": stencil_gbs,
                                 "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                                 "frac": (stencil_gbs / pk["hbm_gbs"]) if stencil_gbs else None,
                                 "traffic": tr.get("stencil", {}).get("dram_bytes_per_launch"),
                                 "traffic_algorithmic": tr.get("stencil", {}).get(
                                     "algorithmic_bytes_per_launch"),
                                 "traffic_source": tr.get("stencil", {}).get("source"),
                                 "bytes_per_eval": 16.0 * (S + 1) * ncell_local,
                                 "ncu_fp64_pipe_pct": tr.get("stencil", {}).get("fp64_pipe_pct")},
            "time_split_ms": {"chem": chem_ms_max, "slow": slow_ms_max, "other": other_ms,
                              "profiled_total": profiled_ms, "steps": args.steps},
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def workload_text(args, cfg, n, n0l, H):
    if cfg.get("d_impl") is not None:
        method = (f"{cfg['coupling']} + {cfg['fast_table']}, H/h={cfg['m']}, order-{cfg['order']} "
                  f"advection (slow-explicit) + D={cfg['d_impl']:g} diffusion (slow-implicit, "
                  f"Newton + {cfg['cg_iters']}-iteration Jacobi-PCG on L7)")
    elif cfg["coupling"] == "mis-kw3":
        method = (f"mis-kw3 (MRI-GARK-ERK33 stand-in) + {cfg['fast_table']}, H/h={cfg['m']}, "
                  f"order-{cfg['order']} advection-diffusion")
    else:
        method = (f"{cfg['coupling']} (MRI-GARK-ERK45a stand-in) + {cfg['fast_table']}, "
                  f"H/h={cfg['m']}, order-{cfg['order']} advection-diffusion")
    grid = f"{n}^3 grid" if n0l == n else f"{n0l}x{n}x{n} slab of the {n}^3 grid"
    return (f"{args.config}: {grid}, {cfg['S']} species / {cfg['R']} reactions (synthetic "
            f"Arrhenius), {method}, H={H:g}")


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside a launcher: start N ranks
    with torch.distributed.run on this node (one process per GPU) and return
    their exit code.  Refuses loudly when fewer than N GPUs are visible."""
    import torch
    have = torch.cuda.device_count()
    if args.impl != "reference" and have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible")
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=None, help="override grid size (debug)")
    ap.add_argument("--sample-n", type=int, default=24, help="CPU baseline sub-grid size")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--nccl-self", action="store_true",
                    help="N=1: run the NCCL rank path through a one-rank communicator")
    ap.add_argument("--slab-of", type=int, default=0,
                    help="N=1: run one rank's slab of an N-GPU decomposition (e.g. C5: 8)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
