// oracle/ref_bridge.cpp -- CPU ORACLE (test infrastructure only).
//
// Drives the reference's OWN stepper (mri_step / mri_integrate / erk_step /
// build_forcing / register_coupling / export_coupling, compiled unmodified
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/) with the
// builder's CPU physics callbacks from mri_oracle.c plugged into the
// reference's PartitionedSystem (proj/include/multirate/partitioned_system.hpp:25-61).
// Used to (a) pin the C restatement in mri_oracle.c bit-for-bit, (b) export
// the reference's coupling tables as v1 audit text (tests/golden/couplings),
// and (c) time the reference CPU path in bench.py --impl reference.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>

#include "multirate/butcher.hpp"
#include "multirate/erk.hpp"
#include "multirate/mri.hpp"
#include "multirate/sdc.hpp"

extern "C" {
#include "mri_oracle.h"
}

using namespace multirate;

namespace {

void set_err(char* err, size_t n, const std::string& msg)
{
  if (err && n) { std::snprintf(err, n, "%s", msg.c_str()); }
}

// The "ERK45a" stand-in: the explicit projection of the
// reference's imex-mri-gark4 (zero gamma, ImplicitSolve -> ExplicitUpdate),
// re-imported through the reference's own import_coupling (mri.cpp:590-626).
MriCoupling explicit_projection(const std::string& base_name, const std::string& new_name)
{
  MriCoupling cp = register_coupling(base_name);
  for (auto& mat : cp.gamma)
    for (auto& row : mat)
      for (auto& v : row) v = 0.0;
  for (auto& k : cp.stage_kind)
    if (k == StageKind::ImplicitSolve) k = StageKind::ExplicitUpdate;
  cp.name = new_name;
  std::stringstream buf;
  export_coupling(cp, buf);
  return import_coupling(buf);
}

MriCoupling load_coupling(const char* spec)
{
  std::string s(spec);
  if (s.rfind("mri-coupling", 0) == 0) {
    std::stringstream in(s);
    return import_coupling(in);
  }
  if (s == "imex-mri-gark4-explicit") { return explicit_projection("imex-mri-gark4", s); }
  return register_coupling(s);
}

PartitionedSystem make_system(orc_sys* sys)
{
  const orc_problem* p = orc_sys_problem(sys);
  PartitionedSystem ps;
  ps.dimension = p->ncell * static_cast<size_t>(p->ncomp);
  if (p->fast_kind != ORC_FAST_NONE) {
    ps.f_fast = [sys](double t, const StateVector& y) {
      StateVector out(y.size());
      orc_sys_fast_rhs(sys, t, y.data(), out.data());
      return out;
    };
  }
  if (p->slow_kind != ORC_SLOW_NONE) {
    ps.f_explicit = [sys](double t, const StateVector& y) {
      StateVector out(y.size());
      orc_sys_slow_rhs(sys, t, y.data(), out.data());
      return out;
    };
  }
  if (p->grid && p->grid->imex) {  // f_implicit = d_impl L7, linear: J v = f_I(v)
    ps.f_implicit = [sys](double t, const StateVector& y) {
      StateVector out(y.size());
      orc_sys_implicit_rhs(sys, t, y.data(), out.data());
      return out;
    };
    ps.jv_implicit = [sys](double t, const StateVector&, const StateVector& v) {
      StateVector out(v.size());
      orc_sys_implicit_rhs(sys, t, v.data(), out.data());
      return out;
    };
  }
  return ps;
}

// ImplicitStageSolver (mri.hpp:84-95) from the system's Newton settings --
// the same NewtonConfig and WRMS weights the oracle and the device use.  The
// GMRES settings only have to converge (the replacement linear solver is the
// fixed-iteration PCG): tolerance relative to max|y| since the reacting-flow
// state carries an energy component ~1e10.
ImplicitStageSolver stage_solver(orc_sys* sys, const StateVector& y)
{
  const orc_grid* g = orc_sys_problem(sys)->grid;
  ImplicitStageSolver s;
  double ymax = 0.0;
  for (double v : y) ymax = std::max(ymax, std::fabs(v));
  if (g) {
    s.newton.tolerance = g->newton_tol;
    s.newton.safety = g->newton_safety;
    s.newton.max_iters = g->newton_max_iters;
    if (g->newton_w) {
      s.weights = StateVector(y.size());
      for (std::size_t i = 0; i < y.size(); ++i) s.weights[i] = g->newton_w[i];
    }
  }
  s.gmres.tolerance = 1e-15 * (1.0 + ymax);
  s.gmres.safety = 1.0;
  s.gmres.max_iters = 200;
  return s;
}

template <class Fn>
int guarded(char* err, size_t errlen, int* fail_stage, Fn&& fn)
{
  if (fail_stage) *fail_stage = -1;
  try {
    fn();
    return 0;
  } catch (const IntegrationError& e) {
    if (fail_stage) *fail_stage = e.stage_index;
    set_err(err, errlen, e.what());
    return 2;
  } catch (const ContractError& e) {
    set_err(err, errlen, e.what());
    return 1;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 1;
  }
}

void counters_to(const EvalCounters& c, uint64_t* out)
{
  const size_t v[8] = {c.n_fast_evals,   c.n_implicit_evals, c.n_explicit_evals,
                       c.n_implicit_solves, c.n_nonlinear_iters, c.n_linear_iters,
                       c.n_precond_solves, c.n_fast_ivps};
  for (int i = 0; i < 8; ++i) out[i] = v[i];
}

EvalCounters counters_from(const uint64_t* in)
{
  EvalCounters c;
  c.n_fast_evals = in[0]; c.n_implicit_evals = in[1]; c.n_explicit_evals = in[2];
  c.n_implicit_solves = in[3]; c.n_nonlinear_iters = in[4]; c.n_linear_iters = in[5];
  c.n_precond_solves = in[6]; c.n_fast_ivps = in[7];
  return c;
}

} // namespace

extern "C" {

// export_coupling text of a registered (or stand-in) coupling; returns length or -1
int ref_export_coupling(const char* name, char* buf, size_t buflen)
{
  try {
    MriCoupling cp = load_coupling(name);
    std::stringstream out;
    export_coupling(cp, out);
    std::string s = out.str();
    if (s.size() + 1 > buflen) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
  } catch (...) {
    return -1;
  }
}

// derived data of a coupling after the reference's finalize(): eval schedule,
// n_sub per stage for a given m, stage kinds
int ref_coupling_info(const char* spec, int m, int* s_out, int* kinds, int* eval_at,
                      int* n_sub, double* c)
{
  try {
    MriCoupling cp = load_coupling(spec);
    *s_out = cp.stages;
    for (int i = 0; i < cp.stages; ++i) {
      kinds[i] = static_cast<int>(cp.stage_kind[i]);
      eval_at[i] = cp.eval_explicit_at[i] ? 1 : 0;
      c[i] = cp.c[i];
      n_sub[i] = 0;
      if (i > 0 && cp.stage_kind[i] == StageKind::FastIvp) {
        const double dc = cp.c[i] - cp.c[i - 1];
        n_sub[i] = static_cast<int>(std::max(1L, std::lround(static_cast<double>(m) * dc)));
      }
    }
    return 0;
  } catch (...) {
    return 1;
  }
}

int ref_sys_mri_step(orc_sys* sys, const char* coupling, const char* fast_table, int m,
                     double t, double H, double* y, uint64_t* counters, int* fail_stage,
                     char* err, size_t errlen)
{
  EvalCounters c = counters_from(counters);
  const int rc = guarded(err, errlen, fail_stage, [&] {
    MriMethodConfig mc;
    mc.coupling = load_coupling(coupling);
    mc.fast_table = lookup_table(fast_table);
    mc.m = m;
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    ImplicitStageSolver solver = stage_solver(sys, yv);
    StateVector out = mri_step(mc, ps, solver, t, yv, H, c);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
  counters_to(c, counters);  // partial counts survive an exception, as in the reference
  return rc;
}

int ref_sys_mri_integrate(orc_sys* sys, const char* coupling, const char* fast_table, int m,
                          double t0, double tf, double H, double* y, uint64_t* counters,
                          int* fail_stage, char* err, size_t errlen)
{
  EvalCounters c = counters_from(counters);
  int rc = guarded(err, errlen, fail_stage, [&] {
    MriMethodConfig mc;
    mc.coupling = load_coupling(coupling);
    mc.fast_table = lookup_table(fast_table);
    mc.m = m;
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    ImplicitStageSolver solver = stage_solver(sys, yv);
    StateVector out = mri_integrate(mc, ps, solver, t0, tf, H, yv, c);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
  counters_to(c, counters); // partial counts survive an exception, as in the reference
  return rc;
}

// erk_step with an arbitrary linear per-cell RHS y' = A y (known-answer pins,
// proj/tests/test_erk.cpp:35-59)
int ref_erk_step_linear(const char* table, int n, const double* A, double t, double* y, double h,
                        uint64_t* evals, int* fail_stage, char* err, size_t errlen)
{
  return guarded(err, errlen, fail_stage, [&] {
    ButcherTable tb = lookup_table(table);
    RhsFn f = [n, A](double, const StateVector& v) {
      StateVector out(v.size());
      for (int a = 0; a < n; ++a) {
        double acc = A[a * n] * v[0];
        for (int b = 1; b < n; ++b) acc = acc + A[a * n + b] * v[b];
        out[a] = acc;
      }
      return out;
    };
    StateVector yv(n);
    for (int i = 0; i < n; ++i) yv[i] = y[i];
    std::size_t cnt = 0;
    StateVector out = erk_step(tb, f, t, yv, h, &cnt);
    for (int i = 0; i < n; ++i) y[i] = out[i];
    *evals += cnt;
  });
}

} // extern "C"

// multirate::reference_solution (erk.cpp:59-75) on the oracle physics
extern "C" int ref_sys_reference_solution(orc_sys* sys, double t0, double tf, double h, double* y,
                                          int* fail_stage, char* err, size_t errlen)
{
  return guarded(err, errlen, fail_stage, [&] {
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    StateVector out = reference_solution(ps, yv, t0, tf, h);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
}

// multirate::erk_integrate (erk.cpp:40-57) of a registered table on sum_rhs,
// counting into *evals like harness.cpp:353-354
extern "C" int ref_sys_erk_integrate(orc_sys* sys, const char* table, double t0, double tf,
                                     double h, double* y, uint64_t* evals, int* fail_stage,
                                     char* err, size_t errlen)
{
  std::size_t cnt = 0;
  const int rc = guarded(err, errlen, fail_stage, [&] {
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    const ButcherTable tb = lookup_table(table);
    RhsFn f = [&ps](double t, const StateVector& v) { return ps.sum_rhs(t, v); };
    StateVector out = erk_integrate(tb, f, t0, tf, h, yv, &cnt);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
  *evals += cnt;
  return rc;
}

// multirate::ark_imex_integrate (mri.cpp:542-557) with the registered ark436 pair
extern "C" int ref_sys_ark_imex_integrate(orc_sys* sys, double t0, double tf, double H, double* y,
                                          uint64_t* counters, int* fail_stage, char* err,
                                          size_t errlen)
{
  EvalCounters c = counters_from(counters);
  const int rc = guarded(err, errlen, fail_stage, [&] {
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    ImplicitStageSolver solver = stage_solver(sys, yv);
    const ArkPair pair = lookup_ark_pair("ark436-imex-pair");
    StateVector out = ark_imex_integrate(pair, ps, solver, t0, tf, H, yv, c);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
  counters_to(c, counters);
  return rc;
}

// lobatto_nodes(n) (sdc.cpp:60-80): nodes[n], S[(n-1)*n]
extern "C" int ref_lobatto_nodes(int n, double* nodes, double* S, char* err, size_t errlen)
{
  return guarded(err, errlen, nullptr, [&] {
    const QuadratureNodes q = lobatto_nodes(n);
    for (int i = 0; i < n; ++i) nodes[i] = q.nodes[i];
    for (int i = 0; i + 1 < n; ++i)
      for (int j = 0; j < n; ++j) S[i * n + j] = q.S[i][j];
  });
}

// build_scheme(X, Y, Z, sweeps) (sdc.cpp:82-153), flattened like mr_mrsdc_scheme
extern "C" int ref_mrsdc_scheme(int X, int Y, int Z, int sweeps, int* n_fine, double* coarse_nodes,
                                double* fine_nodes, int* coarse_of_fine, int* coarse_index_of_fine,
                                double* fine_row, int* application_offset, double* coarse_row,
                                char* err, size_t errlen)
{
  return guarded(err, errlen, nullptr, [&] {
    const MrsdcScheme s = build_scheme(X, Y, Z, sweeps);
    const int cap = *n_fine;
    *n_fine = s.n_fine;
    if (!coarse_nodes || cap < s.n_fine) return;
    for (int j = 0; j < X; ++j) coarse_nodes[j] = s.coarse.nodes[j];
    for (int q = 0; q < s.n_fine; ++q) {
      fine_nodes[q] = s.fine_nodes[q];
      coarse_of_fine[q] = s.coarse_of_fine[q];
      coarse_index_of_fine[q] = s.coarse_index_of_fine[q];
    }
    for (int q = 0; q + 1 < s.n_fine; ++q) {
      for (int j = 0; j < Y; ++j) fine_row[q * Y + j] = s.fine_row[q][j];
      application_offset[q] = s.application_offset[q];
      for (int j = 0; j < X; ++j) coarse_row[q * X + j] = s.coarse_row[q][j];
    }
  });
}

// sdc_integrate (sdc.cpp:267-281) of sum_rhs with lobatto_nodes(n), counting
// into *evals like harness.cpp:356-366
extern "C" int ref_sys_sdc_integrate(orc_sys* sys, int n, int sweeps, double t0, double tf,
                                     double H, double* y, uint64_t* evals, int* fail_stage,
                                     char* err, size_t errlen)
{
  std::size_t cnt = 0;
  const int rc = guarded(err, errlen, fail_stage, [&] {
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    const QuadratureNodes nodes = lobatto_nodes(n);
    RhsFn f = [&ps](double t, const StateVector& v) { return ps.sum_rhs(t, v); };
    StateVector out = sdc_integrate(nodes, f, t0, tf, H, yv, sweeps, &cnt);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
  *evals += cnt;
  return rc;
}

// mrsdc_integrate (sdc.cpp:283-301) with build_scheme(X, Y, Z, sweeps)
extern "C" int ref_sys_mrsdc_integrate(orc_sys* sys, int X, int Y, int Z, int sweeps, double t0,
                                       double tf, double H, double* y, uint64_t* counters,
                                       int* fail_stage, char* err, size_t errlen)
{
  EvalCounters c = counters_from(counters);
  const int rc = guarded(err, errlen, fail_stage, [&] {
    PartitionedSystem ps = make_system(sys);
    StateVector yv(ps.dimension);
    std::memcpy(yv.data(), y, sizeof(double) * ps.dimension);
    const MrsdcScheme scheme = build_scheme(X, Y, Z, sweeps);
    StateVector out = mrsdc_integrate(scheme, ps, t0, tf, H, yv, c);
    std::memcpy(y, out.data(), sizeof(double) * ps.dimension);
  });
  counters_to(c, counters);
  return rc;
}
