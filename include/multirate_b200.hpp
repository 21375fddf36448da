// multirate_b200.hpp -- header-only C++ facade that binds the reference's own
// types (multirate::MriMethodConfig, StateVector, EvalCounters,
// PartitionedSystem, ContractError, IntegrationError) to the C-ABI of
// libmri_b200.so (include/mri_b200.h).  A maintainer of the reference includes
// this next to "multirate/mri.hpp" and links libmri_b200.so; see INTEGRATION.md.
//
//   Mode B (device-resident step, the product path):
//     multirate::b200::Device dev(0);
//     dev.grid(n, n, n, S + 1);  dev.chemistry(...);  dev.stencil(...);
//     [dev.implicit_diffusion(d, cg_iters);   // IMEX couplings]
//     y = multirate::b200::mri_integrate(dev, method, [solver,] t0, tf, H, y0, counters);
//   Mode A (the reference's own mri_step driving GPU callbacks):
//     PartitionedSystem sys = multirate::b200::partitioned_system(dev);
//     y = multirate::mri_integrate(method, sys, solver, t0, tf, H, y0, counters);
//
// Error mapping: MR_CONTRACT -> ContractError, MR_INTEGRATION ->
// IntegrationError(stage_index), MR_CUDA -> std::runtime_error.
#ifndef MULTIRATE_B200_HPP_
#define MULTIRATE_B200_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mri_b200.h"
#include "multirate/mri.hpp"
#include "multirate/sdc.hpp"

namespace multirate::b200 {

class Device {
public:
  explicit Device(int device = 0)
  {
    if (mr_ctx_create(device, &ctx_) != MR_OK || !ctx_)
      throw std::runtime_error("multirate::b200: no usable CUDA device (no CPU fallback)");
  }
  // Several GPUs of this process (mr_ctx_create_multi): the grid is
  // slab-decomposed along axis 0 over `devices` in order, the ghost planes
  // travel peer-to-peer over NVLink, and every call below -- including
  // mri_integrate -- drives all of them; the results are bitwise those of
  // one GPU.
  explicit Device(const std::vector<int>& devices)
  {
    if (devices.empty() ||
        mr_ctx_create_multi(devices.data(), (int)devices.size(), &ctx_) != MR_OK || !ctx_)
      throw std::runtime_error("multirate::b200: no usable CUDA devices (no CPU fallback)");
  }
  ~Device() { mr_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  mr_ctx* ctx() const { return ctx_; }

  void check(int rc, int stage = -1) const
  {
    if (rc == MR_OK) return;
    const std::string msg = mr_last_error(ctx_);
    if (rc == MR_CONTRACT) throw ContractError(msg);
    if (rc == MR_INTEGRATION) throw IntegrationError(msg, stage);
    throw std::runtime_error(msg);
  }

  void grid(int n0, int n1, int n2, int ncomp, double length = 1.0, int i0 = 0, int n0_local = -1)
  {
    check(mr_grid_set(ctx_, n0, n1, n2, ncomp, length, i0, n0_local < 0 ? n0 : n0_local));
    dof_ = mr_state_dof(ctx_);
  }
  void chemistry(int S, int R, double rho, const double* species, const double* reactions,
                 const int* rspecies)
  {
    check(mr_fast_chemistry(ctx_, S, R, rho, species, reactions, rspecies));
    fast_ = true;
  }
  void no_fast()  // f_fast absent
  {
    check(mr_fast_none(ctx_));
    fast_ = false;
  }
  void stencil(int order, double diffusion, const double* u, const double* prof = nullptr,
               int nmax = 0)
  {
    check(mr_slow_stencil(ctx_, order, diffusion, u, prof, nmax));
    imex_ = false;
  }
  // IMEX split of the slow partition (after stencil): f_implicit = d_impl L7
  void implicit_diffusion(double d_impl, int cg_iters)
  {
    check(mr_slow_implicit_diffusion(ctx_, d_impl, cg_iters));
    imex_ = true;
  }
  // ImplicitStageSolver (mri.hpp:71-78): NewtonConfig + WRMS weights.  The
  // GMRES settings and make_preconditioner do not apply: the device solves
  // the linear stage problem with its fixed-iteration PCG.
  void solver(const ImplicitStageSolver& s)
  {
    const bool w = s.weights.size() == dof_ && dof_ > 0;
    check(mr_newton_config(ctx_, s.newton.tolerance, s.newton.safety, s.newton.max_iters,
                           w ? s.weights.data() : nullptr));
  }
  std::size_t dof() const { return dof_; }
  bool imex() const { return imex_; }
  bool has_fast() const { return fast_; }

private:
  mr_ctx* ctx_ = nullptr;
  std::size_t dof_ = 0;
  bool imex_ = false;
  bool fast_ = false;
};

inline void to_c(const EvalCounters& c, uint64_t* o)
{
  o[0] = c.n_fast_evals; o[1] = c.n_implicit_evals; o[2] = c.n_explicit_evals;
  o[3] = c.n_implicit_solves; o[4] = c.n_nonlinear_iters; o[5] = c.n_linear_iters;
  o[6] = c.n_precond_solves; o[7] = c.n_fast_ivps;
}

inline void from_c(const uint64_t* o, EvalCounters& c)
{
  c.n_fast_evals = o[0]; c.n_implicit_evals = o[1]; c.n_explicit_evals = o[2];
  c.n_implicit_solves = o[3]; c.n_nonlinear_iters = o[4]; c.n_linear_iters = o[5];
  c.n_precond_solves = o[6]; c.n_fast_ivps = o[7];
}

// MriMethodConfig (mri.hpp:64-68) -> device method data.  The coupling is
// passed raw and re-finalized with the reference's rules (mri.cpp:59-167).
inline void load_method(Device& d, const MriMethodConfig& mc)
{
  const MriCoupling& cp = mc.coupling;
  const int s = cp.stages;
  const int nd = std::max(1, cp.degrees());
  std::vector<int> kind(s);
  for (int i = 0; i < s; ++i) kind[i] = static_cast<int>(cp.stage_kind[i]);
  std::vector<double> g(static_cast<size_t>(nd) * s * s, 0.0), w(g.size(), 0.0);
  for (int k = 0; k < nd; ++k)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        const size_t at = (static_cast<size_t>(k) * s + i) * s + j;
        if (k < static_cast<int>(cp.gamma.size())) g[at] = cp.gamma[k][i][j];
        if (k < static_cast<int>(cp.omega.size())) w[at] = cp.omega[k][i][j];
      }
  d.check(mr_coupling_load(d.ctx(), s, nd, cp.c.data(), kind.data(), g.data(), w.data()));
  const ButcherTable& t = mc.fast_table;
  std::vector<double> A(static_cast<size_t>(t.stages) * t.stages);
  for (int i = 0; i < t.stages; ++i)
    for (int j = 0; j < t.stages; ++j) A[static_cast<size_t>(i) * t.stages + j] = t.A[i][j];
  d.check(mr_table_load(d.ctx(), t.stages, A.data(), t.b.data(), t.c.data()));
  d.check(mr_set_substeps(d.ctx(), mc.m));
}

// mri_step (mri.hpp:117-120) on the device-resident plugins: H2D of y, one
// slow step, D2H of the result.  Counters accumulate like the reference's.
inline StateVector mri_step(Device& d, const MriMethodConfig& mc, double t, const StateVector& y,
                            double H, EvalCounters& counters)
{
  load_method(d, mc);
  if (y.size() != d.dof()) throw ContractError("mri_step: state size != grid dof");
  StateVector out(y.size());
  uint64_t c[8];
  to_c(counters, c);
  int stage = -1;
  const int rc = mr_mri_step_host(d.ctx(), t, H, y.data(), out.data(), c, &stage);
  from_c(c, counters);
  d.check(rc, stage);
  return out;
}

// mri_step with the reference's ImplicitStageSolver (IMEX couplings)
inline StateVector mri_step(Device& d, const MriMethodConfig& mc, const ImplicitStageSolver& solver,
                            double t, const StateVector& y, double H, EvalCounters& counters)
{
  d.solver(solver);
  return mri_step(d, mc, t, y, H, counters);
}

// mri_integrate (mri.hpp:129-133): the state stays in HBM between steps.
inline StateVector mri_integrate(Device& d, const MriMethodConfig& mc, double t0, double tf,
                                 double H, const StateVector& y0, EvalCounters& counters)
{
  load_method(d, mc);
  if (y0.size() != d.dof()) throw ContractError("mri_integrate: state size != grid dof");
  d.check(mr_state_upload(d.ctx(), y0.data()));
  uint64_t c[8];
  to_c(counters, c);
  int stage = -1;
  const int rc = mr_mri_integrate(d.ctx(), t0, tf, H, c, &stage);
  from_c(c, counters);
  d.check(rc, stage);
  StateVector out(y0.size());
  d.check(mr_state_download(d.ctx(), out.data()));
  return out;
}

// mri_integrate with the reference's ImplicitStageSolver (IMEX couplings)
inline StateVector mri_integrate(Device& d, const MriMethodConfig& mc,
                                 const ImplicitStageSolver& solver, double t0, double tf,
                                 double H, const StateVector& y0, EvalCounters& counters)
{
  d.solver(solver);
  return mri_integrate(d, mc, t0, tf, H, y0, counters);
}

// reference_solution (erk.cpp:59-75) on the device plugins: cash-karp5 of
// f_fast + f_implicit + f_explicit from t0 to tf with step h_ref.
inline StateVector reference_solution(Device& d, const StateVector& y0, double t0, double tf,
                                      double h_ref)
{
  if (y0.size() != d.dof()) throw ContractError("reference_solution: state size != grid dof");
  d.check(mr_state_upload(d.ctx(), y0.data()));
  int stage = -1;
  const int rc = mr_reference_solution(d.ctx(), t0, tf, h_ref, &stage);
  d.check(rc, stage);
  StateVector out(y0.size());
  d.check(mr_state_download(d.ctx(), out.data()));
  return out;
}

// erk_integrate (erk.cpp:40-57) of f_fast + f_implicit + f_explicit with an
// explicit table: the harness's "erk-<table>" family (harness.cpp:346-355),
// counting stage evaluations into *eval_counter like the reference.
inline StateVector erk_integrate(Device& d, const ButcherTable& table, double t0, double tf,
                                 double h, const StateVector& y0,
                                 std::size_t* eval_counter = nullptr)
{
  if (y0.size() != d.dof()) throw ContractError("erk_integrate: state size != grid dof");
  if (table.kind != TableKind::Explicit) throw ContractError("erk_step: table must be explicit");
  const int s = table.stages;
  std::vector<double> A(static_cast<size_t>(s) * s);
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) A[static_cast<size_t>(i) * s + j] = table.A[i][j];
  d.check(mr_state_upload(d.ctx(), y0.data()));
  uint64_t evals = 0;
  int stage = -1;
  const int rc = mr_erk_integrate(d.ctx(), s, A.data(), table.b.data(), table.c.data(), t0, tf, h,
                                  &evals, &stage);
  if (eval_counter) *eval_counter += static_cast<std::size_t>(evals);
  d.check(rc, stage);
  StateVector out(y0.size());
  d.check(mr_state_download(d.ctx(), out.data()));
  return out;
}

// ark_imex_integrate (mri.cpp:542-557) with the ark436 pair
// (lookup_ark_pair("ark436-imex-pair")) on the device plugins
inline StateVector ark_imex_integrate(Device& d, const ImplicitStageSolver& solver, double t0,
                                      double tf, double H, const StateVector& y0,
                                      EvalCounters& counters)
{
  if (y0.size() != d.dof()) throw ContractError("ark_imex_integrate: state size != grid dof");
  d.solver(solver);
  d.check(mr_state_upload(d.ctx(), y0.data()));
  uint64_t c[8];
  to_c(counters, c);
  int stage = -1;
  const int rc = mr_ark_imex_integrate(d.ctx(), t0, tf, H, c, &stage);
  from_c(c, counters);
  d.check(rc, stage);
  StateVector out(y0.size());
  d.check(mr_state_download(d.ctx(), out.data()));
  return out;
}

// sdc_integrate (sdc.cpp:267-281) of f_fast + f_implicit + f_explicit on the
// device plugins with the reference's node set: the harness's sdc-<sweeps>
// family (harness.cpp:356-366), evaluations counted into *eval_counter
inline StateVector sdc_integrate(Device& d, const QuadratureNodes& nodes, double t0, double tf,
                                 double H, const StateVector& y0, int n_sweeps,
                                 std::size_t* eval_counter = nullptr)
{
  if (y0.size() != d.dof()) throw ContractError("sdc_integrate: state size != grid dof");
  const int n = nodes.n;
  std::vector<double> S(static_cast<size_t>(n > 0 ? n - 1 : 0) * n);
  for (int q = 0; q + 1 < n; ++q)
    for (int j = 0; j < n; ++j) S[static_cast<size_t>(q) * n + j] = nodes.S[q][j];
  d.check(mr_state_upload(d.ctx(), y0.data()));
  uint64_t evals = 0;
  int stage = -1;
  const int rc = mr_sdc_integrate(d.ctx(), n, nodes.nodes.data(), S.data(), n_sweeps, t0, tf, H,
                                  &evals, &stage);
  if (eval_counter) *eval_counter += static_cast<std::size_t>(evals);
  d.check(rc, stage);
  StateVector out(y0.size());
  d.check(mr_state_download(d.ctx(), out.data()));
  return out;
}

// mrsdc_integrate (sdc.cpp:283-301) of a build_scheme(X, Y, Z, sweeps) scheme
// on the device plugins: the harness's mrsdc-XYZ family (harness.cpp:368-372)
inline StateVector mrsdc_integrate(Device& d, const MrsdcScheme& s, double t0, double tf, double H,
                                   const StateVector& y0, EvalCounters& counters)
{
  if (y0.size() != d.dof()) throw ContractError("mrsdc_integrate: state size != grid dof");
  const int nf = s.n_fine, X = s.X, Y = s.Y;
  std::vector<double> frow(static_cast<size_t>(nf - 1) * Y), crow(static_cast<size_t>(nf - 1) * X);
  for (int q = 0; q + 1 < nf; ++q) {
    for (int j = 0; j < Y; ++j) frow[static_cast<size_t>(q) * Y + j] = s.fine_row[q][j];
    for (int j = 0; j < X; ++j) crow[static_cast<size_t>(q) * X + j] = s.coarse_row[q][j];
  }
  d.check(mr_mrsdc_load(d.ctx(), X, Y, nf, s.n_sweeps, s.coarse.nodes.data(), s.fine_nodes.data(),
                        s.coarse_of_fine.data(), s.coarse_index_of_fine.data(), frow.data(),
                        s.application_offset.data(), crow.data()));
  d.check(mr_state_upload(d.ctx(), y0.data()));
  uint64_t c[8];
  to_c(counters, c);
  int stage = -1;
  const int rc = mr_mrsdc_integrate(d.ctx(), t0, tf, H, c, &stage);
  from_c(c, counters);
  d.check(rc, stage);
  StateVector out(y0.size());
  d.check(mr_state_download(d.ctx(), out.data()));
  return out;
}

// "Mode A": the reference's PartitionedSystem (partitioned_system.hpp:25-61)
// whose f_fast / f_explicit callbacks evaluate the device plugins.
inline PartitionedSystem partitioned_system(Device& d)
{
  PartitionedSystem sys;
  sys.dimension = d.dof();
  Device* dp = &d;
  if (d.has_fast())
    sys.f_fast = [dp](double t, const StateVector& y) {
      StateVector out(y.size());
      dp->check(mr_fast_rhs(dp->ctx(), t, y.data(), out.data()));
      return out;
    };
  sys.f_explicit = [dp](double t, const StateVector& y) {
    StateVector out(y.size());
    dp->check(mr_slow_rhs(dp->ctx(), t, y.data(), out.data()));
    return out;
  };
  if (d.imex()) {
    sys.f_implicit = [dp](double t, const StateVector& y) {
      StateVector out(y.size());
      dp->check(mr_implicit_rhs(dp->ctx(), t, y.data(), out.data()));
      return out;
    };
    // f_implicit is linear: J v = f_implicit(v)
    sys.jv_implicit = [dp](double t, const StateVector&, const StateVector& v) {
      StateVector out(v.size());
      dp->check(mr_implicit_rhs(dp->ctx(), t, v.data(), out.data()));
      return out;
    };
  }
  return sys;
}

}  // namespace multirate::b200

#endif  // MULTIRATE_B200_HPP_
