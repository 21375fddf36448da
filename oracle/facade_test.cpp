// oracle/facade_test.cpp -- TEST INFRASTRUCTURE: compiles the C++ facade
// (include/multirate_b200.hpp) against the reference's own headers and
// sources and runs the same slow steps three ways:
//   B: multirate::b200::mri_integrate   (device-resident product path)
//   A: the reference's mri_integrate driving the GPU plugins through a
//      reference PartitionedSystem ("Mode A", the drop-in callback route)
//   C: the reference's mri_integrate with the CPU oracle physics
// Built by `make -C oracle facade` into oracle/_ref/ (needs /root/reference).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <string>

#include "multirate/butcher.hpp"
#include "multirate/mri.hpp"
#include "multirate_b200.hpp"

extern "C" {
#include "mri_oracle.h"
}

using namespace multirate;

namespace {
double rel_err(const StateVector& a, const StateVector& b, int ncomp)
{
  const size_t nc = a.size() / ncomp;
  double worst = 0.0;
  for (int k = 0; k < ncomp; ++k) {
    double d = 0.0, m = 0.0;
    for (size_t i = 0; i < nc; ++i) {
      d = std::max(d, std::fabs(a[k * nc + i] - b[k * nc + i]));
      m = std::max(m, std::fabs(b[k * nc + i]));
    }
    worst = std::max(worst, m > 0 ? d / m : d);
  }
  return worst;
}
}  // namespace

// d_impl >= 0 selects the IMEX split (explicit stencil diffusion `diffusion`,
// implicit d_impl L7 with cg_iters PCG iterations on the device); newton =
// {tolerance, safety, max_iters} and weights (may be NULL) configure the
// ImplicitStageSolver used by all three paths.
extern "C" int facade_selftest(int n, int S, int R, double rho, const double* species,
                               const double* reactions, const int* rspecies, const double* y0in,
                               const char* coupling, const char* table, int m, int order,
                               double H, int steps, int fast, double diffusion, double d_impl,
                               int cg_iters,
                               const double* newton, const double* weights, double* errs,
                               uint64_t* counters, char* err, size_t errlen)
{
  try {
    const int ncomp = S + 1;
    const size_t dof = (size_t)n * n * n * ncomp;
    StateVector y0(dof);
    std::memcpy(y0.data(), y0in, dof * sizeof(double));
    MriMethodConfig mc;
    if (std::string(coupling).rfind("mri-coupling", 0) == 0) {
      std::stringstream in{std::string(coupling)};
      mc.coupling = import_coupling(in);
    } else {
      mc.coupling = register_coupling(coupling);
    }
    mc.fast_table = lookup_table(table);
    mc.m = m;
    const double u[3] = {1.0, 1.0, 1.0};

    const bool imex = d_impl >= 0.0;
    ImplicitStageSolver solver;
    if (newton) {
      solver.newton.tolerance = newton[0];
      solver.newton.safety = newton[1];
      solver.newton.max_iters = (int)newton[2];
    }
    if (weights) {
      solver.weights = StateVector(dof);
      std::memcpy(solver.weights.data(), weights, dof * sizeof(double));
    }
    // the reference's GMRES only has to converge (the device uses its PCG)
    double ymax = 0.0;
    for (double v : y0) ymax = std::max(ymax, std::fabs(v));
    solver.gmres.tolerance = 1e-15 * (1.0 + ymax);
    solver.gmres.safety = 1.0;
    solver.gmres.max_iters = 200;

    b200::Device dev(0);
    dev.grid(n, n, n, ncomp);
    dev.chemistry(S, R, rho, species, reactions, rspecies);
    if (!fast) dev.no_fast();
    dev.stencil(order, diffusion, u);
    if (imex) dev.implicit_diffusion(d_impl, cg_iters);

    EvalCounters cB, cA, cC;
    StateVector yB = b200::mri_integrate(dev, mc, solver, 0.0, steps * H, H, y0, cB);
    PartitionedSystem sysA = b200::partitioned_system(dev);
    StateVector yA = mri_integrate(mc, sysA, solver, 0.0, steps * H, H, y0, cA);

    orc_sys_cfg cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.n0 = cfg.n1 = cfg.n2 = n;
    cfg.n0_global = n;
    cfg.ncomp = ncomp;
    cfg.length = 1.0;
    cfg.fast_kind = fast ? ORC_FAST_CHEM : ORC_FAST_NONE;
    cfg.slow_kind = ORC_SLOW_STENCIL;
    cfg.S = S; cfg.R = R; cfg.rho = rho;
    cfg.species = species; cfg.reactions = reactions; cfg.rspecies = rspecies;
    cfg.order = order; cfg.diffusion = diffusion; cfg.vel_kind = 0;
    cfg.u_const[0] = cfg.u_const[1] = cfg.u_const[2] = 1.0;
    cfg.threads = 1;
    cfg.imex = imex ? 1 : 0;
    cfg.d_impl = imex ? d_impl : 0.0;
    cfg.cg_iters = cg_iters;
    orc_sys* cs = orc_sys_create(&cfg);
    PartitionedSystem sysC;
    sysC.dimension = dof;
    if (fast)
      sysC.f_fast = [cs](double t, const StateVector& y) {
        StateVector o(y.size());
        orc_sys_fast_rhs(cs, t, y.data(), o.data());
        return o;
      };
    sysC.f_explicit = [cs](double t, const StateVector& y) {
      StateVector o(y.size());
      orc_sys_slow_rhs(cs, t, y.data(), o.data());
      return o;
    };
    if (imex) {
      sysC.f_implicit = [cs](double t, const StateVector& y) {
        StateVector o(y.size());
        orc_sys_implicit_rhs(cs, t, y.data(), o.data());
        return o;
      };
      sysC.jv_implicit = [cs](double t, const StateVector&, const StateVector& v) {
        StateVector o(v.size());
        orc_sys_implicit_rhs(cs, t, v.data(), o.data());
        return o;
      };
    }
    StateVector yC = mri_integrate(mc, sysC, solver, 0.0, steps * H, H, y0, cC);
    orc_sys_destroy(cs);

    errs[0] = rel_err(yB, yC, ncomp);
    errs[1] = rel_err(yA, yC, ncomp);
    errs[2] = rel_err(yA, yB, ncomp);
    b200::to_c(cB, counters);
    b200::to_c(cA, counters + 8);
    b200::to_c(cC, counters + 16);
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// reference_solution and ark_imex_integrate through the facade (device) vs the
// reference's own implementations on the CPU physics.  which = 0: reference
// solution (steps of h); 1: ARK-IMEX (steps of h, IMEX split d_impl);
// 2: erk_integrate with kutta3 (the harness's erk-<table> family).
extern "C" int facade_selftest2(int which, int n, int S, int R, double rho, const double* species,
                                const double* reactions, const int* rspecies,
                                const double* y0in, int order, double diffusion, double d_impl,
                                int cg_iters, int fast, double h, int steps, const double* newton,
                                const double* weights, double* errs, uint64_t* counters,
                                char* err, size_t errlen)
{
  try {
    const int ncomp = S + 1;
    const size_t dof = (size_t)n * n * n * ncomp;
    StateVector y0(dof);
    std::memcpy(y0.data(), y0in, dof * sizeof(double));
    const double u[3] = {1.0, 1.0, 1.0};
    const bool imex = d_impl >= 0.0;
    b200::Device dev(0);
    dev.grid(n, n, n, ncomp);
    dev.chemistry(S, R, rho, species, reactions, rspecies);
    if (!fast) dev.no_fast();
    dev.stencil(order, diffusion, u);
    if (imex) dev.implicit_diffusion(d_impl, cg_iters);

    orc_sys_cfg cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.n0 = cfg.n1 = cfg.n2 = n;
    cfg.n0_global = n;
    cfg.ncomp = ncomp;
    cfg.length = 1.0;
    cfg.fast_kind = fast ? ORC_FAST_CHEM : ORC_FAST_NONE;
    cfg.slow_kind = ORC_SLOW_STENCIL;
    cfg.S = S; cfg.R = R; cfg.rho = rho;
    cfg.species = species; cfg.reactions = reactions; cfg.rspecies = rspecies;
    cfg.order = order; cfg.diffusion = diffusion; cfg.vel_kind = 0;
    cfg.u_const[0] = cfg.u_const[1] = cfg.u_const[2] = 1.0;
    cfg.threads = 1;
    cfg.imex = imex ? 1 : 0;
    cfg.d_impl = imex ? d_impl : 0.0;
    cfg.cg_iters = cg_iters;
    orc_sys* cs = orc_sys_create(&cfg);
    PartitionedSystem sysC;
    sysC.dimension = dof;
    if (fast)
      sysC.f_fast = [cs](double t, const StateVector& y) {
        StateVector o(y.size());
        orc_sys_fast_rhs(cs, t, y.data(), o.data());
        return o;
      };
    sysC.f_explicit = [cs](double t, const StateVector& y) {
      StateVector o(y.size());
      orc_sys_slow_rhs(cs, t, y.data(), o.data());
      return o;
    };
    if (imex) {
      sysC.f_implicit = [cs](double t, const StateVector& y) {
        StateVector o(y.size());
        orc_sys_implicit_rhs(cs, t, y.data(), o.data());
        return o;
      };
      sysC.jv_implicit = [cs](double t, const StateVector&, const StateVector& v) {
        StateVector o(v.size());
        orc_sys_implicit_rhs(cs, t, v.data(), o.data());
        return o;
      };
    }
    StateVector yB, yC;
    EvalCounters cB, cC;
    if (which == 0) {
      yB = b200::reference_solution(dev, y0, 0.0, steps * h, h);
      yC = reference_solution(sysC, y0, 0.0, steps * h, h);
    } else if (which == 2) {  // erk_integrate (erk.cpp:40-57), kutta3, counted
      const ButcherTable tb = lookup_table("kutta3");
      std::size_t eB = 0, eC = 0;
      yB = b200::erk_integrate(dev, tb, 0.0, steps * h, h, y0, &eB);
      RhsFn f = [&sysC](double t, const StateVector& v) { return sysC.sum_rhs(t, v); };
      yC = erk_integrate(tb, f, 0.0, steps * h, h, y0, &eC);
      cB.n_explicit_evals = eB;
      cC.n_explicit_evals = eC;
    } else {
      ImplicitStageSolver solver;
      if (newton) {
        solver.newton.tolerance = newton[0];
        solver.newton.safety = newton[1];
        solver.newton.max_iters = (int)newton[2];
      }
      if (weights) {
        solver.weights = StateVector(dof);
        std::memcpy(solver.weights.data(), weights, dof * sizeof(double));
      }
      double ymax = 0.0;
      for (double v : y0) ymax = std::max(ymax, std::fabs(v));
      solver.gmres.tolerance = 1e-15 * (1.0 + ymax);
      solver.gmres.safety = 1.0;
      solver.gmres.max_iters = 200;
      const ArkPair pair = lookup_ark_pair("ark436-imex-pair");
      yB = b200::ark_imex_integrate(dev, solver, 0.0, steps * h, h, y0, cB);
      yC = ark_imex_integrate(pair, sysC, solver, 0.0, steps * h, h, y0, cC);
    }
    orc_sys_destroy(cs);
    errs[0] = rel_err(yB, yC, ncomp);
    b200::to_c(cB, counters);
    b200::to_c(cC, counters + 8);
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}
