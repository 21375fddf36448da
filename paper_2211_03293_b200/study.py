"""Convergence / efficiency studies on the GPU: the method-running core of the
reference harness over the device plugins.

Mirrors proj/src/harness.cpp:

  parse_method        :89-157   mri3-<m>, imex-mri3-<m>, imex-mri4-<m>, ark-imex,
                                erk-<table>; sdc / mrsdc selectors parse but are
                                refused by run_method (not on the GPU path)
  run_method          :326-394  step count, solver settings, IntegrationError
                                recorded as divergence, wall time
  compute_reference   :405-426  cash-karp5, h_ref = min fast step / 10 or checked
  measure_error       :316-324  max norm (or one component block) of state - reference
  execute_study       :431-512  one row per (method, H), rates, fitted slopes
  fitted_slope        :514-538
  RunReport.write_csv / write_json  :645-705

The problem is a configured ``Context`` plus its initial state (for example
from ``setup_workload``); every run re-uploads y0, so runs are independent.
Besides the reference's selectors, ``mri:<coupling>:<fast_table>:<m>`` runs any
coupling the device loads (e.g. the workloads' ``imex-mri-gark4-explicit``).
The config file reader, CLI, tolerance sweep and preconditioner study of the
harness are out of scope.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import ContractError, IntegrationError, tables

# EvalCounters field order (partitioned_system.hpp:66-79) = MR_CNT_* indices
COUNTER_NAMES = ("fast_evals", "implicit_evals", "explicit_evals", "implicit_solves",
                 "nonlinear_iters", "linear_iters", "precond_solves", "fast_ivps")


class ConfigError(ValueError):
    """harness.hpp ConfigError: a malformed study configuration."""


@dataclass
class MethodSpec:
    """harness.hpp MethodSpec."""
    selector: str
    family: str  # "erk" | "sdc" | "mrsdc" | "mri" | "ark-imex"
    table_name: str = ""
    coupling_name: str = ""
    fast_table: str = ""
    m: int = 1
    X: int = 0
    Y: int = 0
    Z: int = 0
    sweeps: int = 0
    needs_implicit_solver: bool = False


def _suffix_int(selector: str, prefix: str) -> int:
    """parse_int (harness.cpp:61-71) of the selector's tail."""
    tail = selector[len(prefix):]
    try:
        return int(tail.strip(), 10)
    except ValueError:
        raise ConfigError(f"bad integer value for '{selector}': {tail}") from None


def parse_method(selector: str) -> MethodSpec:
    """harness.cpp:89-157."""
    s = selector
    if s.startswith("erk-"):
        name = s[4:]
        tables.lookup_table(name)  # validate the name now
        return MethodSpec(s, "erk", table_name=name)
    if s == "sdc":
        return MethodSpec(s, "sdc", X=3, sweeps=4)
    if s.startswith("sdc-"):
        return MethodSpec(s, "sdc", X=3, sweeps=_suffix_int(s, "sdc-"))
    if s.startswith("mrsdc-"):
        xyz = s[6:]
        if len(xyz) != 3:
            raise ConfigError("mrsdc selector needs three digits, e.g. mrsdc-338")
        return MethodSpec(s, "mrsdc", X=ord(xyz[0]) - 48, Y=ord(xyz[1]) - 48,
                          Z=ord(xyz[2]) - 48, sweeps=4)
    if s.startswith("imex-mri3-"):
        return MethodSpec(s, "mri", coupling_name="imex-mri-gark3b", fast_table="kutta3",
                          m=_suffix_int(s, "imex-mri3-"), needs_implicit_solver=True)
    if s.startswith("imex-mri4-"):
        return MethodSpec(s, "mri", coupling_name="imex-mri-gark4", fast_table="classic-rk4",
                          m=_suffix_int(s, "imex-mri4-"), needs_implicit_solver=True)
    if s.startswith("mri3-"):
        return MethodSpec(s, "mri", coupling_name="mis-kw3", fast_table="bogacki-shampine3",
                          m=_suffix_int(s, "mri3-"))
    if s == "ark-imex":
        return MethodSpec(s, "ark-imex", needs_implicit_solver=True)
    if s.startswith("mri:"):  # device extension: any loadable coupling
        parts = s.split(":")
        if len(parts) != 4:
            raise ConfigError("mri selector is mri:<coupling>:<fast_table>:<m>")
        tables.lookup_table(parts[2])
        cp = parts[1]
        return MethodSpec(s, "mri", coupling_name=cp, fast_table=parts[2],
                          m=_suffix_int(parts[3], ""),
                          needs_implicit_solver=cp.startswith("imex-") and "explicit" not in cp)
    raise ConfigError(f"unknown method selector '{selector}'")


def known_method_selectors():
    """harness.cpp:159-163 (+ the device's mri:<coupling>:<table>:<m>)."""
    return ["erk-<table>", "sdc", "sdc-<sweeps>", "mrsdc-XYZ", "mri3-<m>", "imex-mri3-<m>",
            "imex-mri4-<m>", "ark-imex", "mri:<coupling>:<fast_table>:<m>"]


@dataclass
class StudyConfig:
    """The [study], [solver] and [reference] sections of harness.hpp StudyConfig."""
    methods: list = field(default_factory=list)
    h_list: list = field(default_factory=list)
    t0: float = 0.0
    tf: float = 1.0
    newton_tol: float = 1.0e-10
    newton_max_iters: int = 10
    newton_safety: float = 0.1  # NewtonConfig default (solvers.hpp:19-23)
    tolerance_table: dict = field(default_factory=dict)  # per-H override
    solver_weights: np.ndarray | None = None  # ImplicitStageSolver.weights; None = ones
    reference_method: str = "cash-karp5"
    h_ref: float = 0.0  # 0 => auto
    component_offset: int = 0  # measure_error slice (ProblemInstance)
    component_count: int = 0  # 0 = whole vector

    def validate(self):
        """harness.cpp:165-186 (the parts that apply on the device)."""
        if not self.methods:
            raise ConfigError("no methods configured")
        for m in self.methods:
            parse_method(m)
        if not self.h_list:
            raise ConfigError("no step sizes configured")
        for a, b in zip(self.h_list, self.h_list[1:]):
            if b >= a:
                raise ConfigError("h_list must be strictly decreasing")
        if self.tf <= self.t0:
            raise ConfigError("tf must exceed t0")
        if self.reference_method != "cash-karp5":
            raise ConfigError("reference method must be cash-karp5 on the device "
                              "(analytic requires the linear problem)")


@dataclass
class RunOutcome:
    final_state: np.ndarray | None = None
    counters: np.ndarray = field(default_factory=lambda: np.zeros(8, dtype=np.uint64))
    wall_seconds: float = 0.0
    steps: int = 0
    diverged: bool = False
    message: str = ""


@dataclass
class RunRecord:
    """harness.hpp:90-101."""
    method: str
    H: float
    tolerance: float = 0.0
    error: float = math.nan
    rate: float = math.nan
    wall_seconds: float = 0.0
    steps: int = 0
    counters: np.ndarray = field(default_factory=lambda: np.zeros(8, dtype=np.uint64))
    diverged: bool = False
    note: str = ""


def _g17(v) -> str:
    return "%.17g" % v


@dataclass
class RunReport:
    """harness.hpp:103-112."""
    rows: list = field(default_factory=list)
    fitted_slopes: dict = field(default_factory=dict)

    def write_csv(self, path):
        """harness.cpp:645-663 (same header and %.17g formatting)."""
        with open(path, "w") as f:
            f.write("method,H,tolerance,error,rate,wall_s,steps,diverged,"
                    "n_fast_evals,n_implicit_evals,n_explicit_evals,n_implicit_solves,"
                    "n_nonlinear_iters,n_linear_iters,n_precond_solves,n_fast_ivps\n")
            for r in self.rows:
                c = [int(x) for x in r.counters]
                f.write(",".join([r.method, _g17(r.H), _g17(r.tolerance), _g17(r.error),
                                  _g17(r.rate), _g17(r.wall_seconds), str(r.steps),
                                  "1" if r.diverged else "0"] + [str(x) for x in c]) + "\n")

    def write_json(self, path, cfg: StudyConfig | None = None):
        """harness.cpp:665-705."""
        j = {}
        if cfg is not None:
            j["config"] = {"problem": "reacting-flow", "methods": list(cfg.methods),
                           "t0": cfg.t0, "tf": cfg.tf}
        rows = []
        for r in self.rows:
            rows.append({
                "method": r.method, "H": r.H, "tolerance": r.tolerance,
                "error": r.error if math.isfinite(r.error) else None,
                "rate": r.rate if math.isfinite(r.rate) else None,
                "wall_seconds": r.wall_seconds, "steps": r.steps, "diverged": r.diverged,
                "note": r.note,
                "counters": {k: int(v) for k, v in zip(COUNTER_NAMES, r.counters)},
            })
        j["rows"] = rows
        j["fitted_slopes"] = {k: (v if math.isfinite(v) else None)
                              for k, v in self.fitted_slopes.items()}
        with open(path, "w") as f:
            json.dump(j, f, indent=2)


def measure_error(state, reference, component_offset=0, component_count=0, ncell=None):
    """harness.cpp:316-324: max_norm(state - reference), or
    max_norm_component over components [offset, offset + count) of the
    species-major layout (state_vector.hpp:157-168)."""
    diff = np.asarray(state, dtype=np.float64) - np.asarray(reference, dtype=np.float64)
    if component_count == 0:
        return float(np.max(np.abs(diff))) if diff.size else 0.0
    if ncell is None:
        raise ContractError("measure_error: ncell needed for a component slice")
    blk = diff[component_offset * ncell:(component_offset + component_count) * ncell]
    return float(np.max(np.abs(blk))) if blk.size else 0.0


def fitted_slope(h_and_error):
    """harness.cpp:514-538: least-squares slope of log(error) on log(h), dropping
    the coarsest point when four or more remain; NaN with fewer than two."""
    pts = [(h, e) for h, e in h_and_error if math.isfinite(e) and e > 0.0 and h > 0.0]
    if len(pts) < 2:
        return math.nan
    pts.sort(key=lambda p: -p[0])
    if len(pts) >= 4:
        pts = pts[1:]
    sx = sy = sxx = sxy = 0.0
    for h, e in pts:
        x, y = math.log(h), math.log(e)
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
    n = float(len(pts))
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def _configure_solver(ctx, cfg: StudyConfig, tolerance_override: float):
    tol = tolerance_override if tolerance_override > 0.0 else cfg.newton_tol
    ctx.newton_config(tol, cfg.newton_safety, cfg.newton_max_iters, cfg.solver_weights)


def run_method(ctx, y0, spec: MethodSpec, cfg: StudyConfig, H: float,
               tolerance_override: float = 0.0) -> RunOutcome:
    """harness.cpp:326-394 on the device: upload y0, integrate t0 -> tf with
    step H, download the final state.  IntegrationError -> diverged."""
    out = RunOutcome()
    out.steps = int(math.ceil((cfg.tf - cfg.t0) / H - 1e-12))
    if spec.family in ("sdc", "mrsdc"):
        raise ContractError(f"{spec.selector}: SDC/MRSDC steppers are not on the GPU path")
    ctx.upload(y0)
    if spec.needs_implicit_solver:
        _configure_solver(ctx, cfg, tolerance_override)
    start = time.perf_counter()
    try:
        if spec.family == "erk":
            ctx.erk_integrate(spec.table_name, cfg.t0, cfg.tf, H, out.counters)
        elif spec.family == "mri":
            ctx.method(spec.coupling_name, spec.fast_table, spec.m)
            ctx.mri_integrate(cfg.t0, cfg.tf, H, out.counters)
        else:  # ark-imex
            ctx.ark_imex_integrate(cfg.t0, cfg.tf, H, out.counters)
        out.final_state = ctx.download()
    except IntegrationError as err:
        out.diverged = True
        out.message = str(err)
    out.wall_seconds = time.perf_counter() - start
    return out


def solver_tolerance_for(cfg: StudyConfig, spec: MethodSpec, H: float) -> float:
    """harness.cpp:398-405."""
    if not spec.needs_implicit_solver:
        return 0.0
    return float(cfg.tolerance_table.get(H, 0.0))


def compute_reference(ctx, y0, cfg: StudyConfig):
    """harness.cpp:405-426: cash-karp5 reference with h_ref = (smallest H /
    largest m) / 10 unless configured, which must then be 10x below it."""
    max_m = 1
    for sel in cfg.methods:
        max_m = max(max_m, parse_method(sel).m)
    min_fast_step = cfg.h_list[-1] / max_m
    h_ref = cfg.h_ref
    if h_ref <= 0.0:
        h_ref = min_fast_step / 10.0
    elif h_ref * 10.0 > min_fast_step * (1.0 + 1e-9):
        raise ConfigError("h_ref must be at least 10x below the smallest fast step")
    ctx.upload(y0)
    ctx.reference_solution(cfg.t0, cfg.tf, h_ref)
    return ctx.download()


def execute_study(ctx, y0, cfg: StudyConfig, with_rates: bool = True,
                  reference=None) -> RunReport:
    """harness.cpp:431-512 (jobs = 1: one device context runs the tasks in
    order).  ``reference`` may be passed to reuse a computed reference."""
    cfg.validate()
    ref = compute_reference(ctx, y0, cfg) if reference is None else reference
    ncell = getattr(ctx, "ncell", None)
    report = RunReport()
    for sel in cfg.methods:
        spec = parse_method(sel)
        for H in cfg.h_list:
            tol = solver_tolerance_for(cfg, spec, H)
            o = run_method(ctx, y0, spec, cfg, H, tol)
            rec = RunRecord(method=sel, H=H, tolerance=tol, wall_seconds=o.wall_seconds,
                            steps=o.steps, counters=o.counters, diverged=o.diverged,
                            note=o.message)
            if not o.diverged:
                rec.error = measure_error(o.final_state, ref, cfg.component_offset,
                                          cfg.component_count, ncell)
            report.rows.append(rec)
    if with_rates:
        for sel in cfg.methods:
            rows = sorted((r for r in report.rows if r.method == sel), key=lambda r: -r.H)
            pts = []
            for i, r in enumerate(rows):
                if r.diverged or not math.isfinite(r.error) or r.error <= 0.0:
                    continue
                pts.append((r.H, r.error))
                p = rows[i - 1] if i > 0 else None
                if p is not None and not p.diverged and math.isfinite(p.error) and p.error > 0.0:
                    r.rate = math.log(p.error / r.error) / math.log(p.H / r.H)
            if len(pts) >= 2:
                report.fitted_slopes[sel] = fitted_slope(pts)
    return report


def run_convergence_study(ctx, y0, cfg: StudyConfig, reference=None) -> RunReport:
    """harness.cpp:540-543."""
    return execute_study(ctx, y0, cfg, True, reference)


def run_efficiency_study(ctx, y0, cfg: StudyConfig, reference=None) -> RunReport:
    """harness.cpp:545-548."""
    return execute_study(ctx, y0, cfg, False, reference)
