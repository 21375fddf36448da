// oracle/harness_test.cpp -- TEST INFRASTRUCTURE: the reference's study
// harness on a device problem.
//
// proj/src/harness.cpp is compiled UNMODIFIED into oracle/_ref with the
// routing prefix of include/multirate_b200_harness.hpp (oracle/Makefile,
// target `harness`), so its run_method -- the per-(method, H) entry point of
// every study (harness.cpp:323-394) -- sends a routed device problem's Mri,
// ArkImex and Erk runs to the facade.  This driver runs the same study on the
// same chemistry + stencil problem twice through the reference's own
// run_method, measure_error, fitted_slope and RunReport::write_csv /
// write_json: once with the CPU oracle physics (the reference's integrators)
// and once routed to the GPU.  The study loop is execute_study's
// (harness.cpp:431-512) -- make_problem/validate accept only the reference's
// three problem kinds, so a device problem enters at run_method.
#define MULTIRATE_B200_HARNESS_IMPL
#include "multirate_b200_harness.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <string>

extern "C" {
#include "mri_oracle.h"
}

using namespace multirate;

namespace {

std::vector<std::string> split(const std::string& s)
{
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

// execute_study (harness.cpp:431-512) with jobs = 1 over a given problem and
// reference: the reference's run_method / measure_error / fitted_slope
RunReport study(const ProblemInstance& problem, const StudyConfig& cfg,
                const StateVector& reference)
{
  RunReport report;
  for (const auto& sel : cfg.methods) {
    const MethodSpec spec = parse_method(sel);
    for (double H : cfg.h_list) {
      const RunOutcome outcome = run_method(spec, problem, cfg, H, 0.0);
      RunRecord rec;
      rec.method = spec.selector;
      rec.H = H;
      rec.tolerance = 0.0;
      rec.wall_seconds = outcome.wall_seconds;
      rec.steps = outcome.steps;
      rec.counters = outcome.counters;
      rec.diverged = outcome.diverged;
      rec.note = outcome.message;
      if (!outcome.diverged) rec.error = measure_error(problem, outcome.final_state, reference);
      report.rows.push_back(std::move(rec));
    }
  }
  for (const auto& sel : cfg.methods) {
    std::vector<RunRecord*> rows;
    for (auto& r : report.rows)
      if (r.method == sel) rows.push_back(&r);
    std::sort(rows.begin(), rows.end(), [](const RunRecord* a, const RunRecord* b) { return a->H > b->H; });
    std::vector<std::pair<double, double>> points;
    for (std::size_t i = 0; i < rows.size(); ++i) {
      if (rows[i]->diverged || !std::isfinite(rows[i]->error) || rows[i]->error <= 0.0) continue;
      points.push_back({rows[i]->H, rows[i]->error});
      if (i > 0 && !rows[i - 1]->diverged && std::isfinite(rows[i - 1]->error) && rows[i - 1]->error > 0.0)
        rows[i]->rate = std::log(rows[i - 1]->error / rows[i]->error) / std::log(rows[i - 1]->H / rows[i]->H);
    }
    if (points.size() >= 2) report.fitted_slopes[sel] = fitted_slope(points);
  }
  return report;
}

}  // namespace

// The chemistry + stencil problem on an n^3 grid (uniform velocity 1), CPU
// and device, one study each.  d_impl >= 0 adds the slow-implicit diffusion;
// fast = 0 switches the chemistry off.  Errors are measured on the species
// slice (components 0..S-1), like the harness's error_component slices.
extern "C" int harness_selftest(int n, int S, int R, double rho, const double* species,
                                const double* reactions, const int* rspecies,
                                const double* y0in, int order, double diffusion, double d_impl,
                                int cg_iters, int fast, const char* methods, const double* hs,
                                int nh, double t0, double tf, double h_ref, double newton_tol,
                                const char* csv_cpu, const char* csv_dev, const char* json_dev,
                                char* err, size_t errlen)
{
  try {
    const int ncomp = S + 1;
    const std::size_t ncell = (std::size_t)n * n * n, dof = ncell * ncomp;
    StateVector y0(dof);
    std::memcpy(y0.data(), y0in, dof * sizeof(double));
    const double u[3] = {1.0, 1.0, 1.0};
    const bool imex = d_impl >= 0.0;

    StudyConfig cfg;
    cfg.methods = split(methods);
    cfg.h_list.assign(hs, hs + nh);
    cfg.t0 = t0;
    cfg.tf = tf;
    cfg.h_ref = h_ref;
    cfg.jobs = 1;
    double ymax = 0.0;
    for (double v : y0) ymax = std::max(ymax, std::fabs(v));
    cfg.newton_tol = newton_tol;
    cfg.gmres_tol = 1e-15 * (1.0 + ymax);  // the reference's GMRES only has to converge
    cfg.gmres_max_iters = 200;

    // CPU: the oracle physics behind the reference's PartitionedSystem
    orc_sys_cfg oc;
    std::memset(&oc, 0, sizeof(oc));
    oc.n0 = oc.n1 = oc.n2 = n;
    oc.n0_global = n;
    oc.ncomp = ncomp;
    oc.length = 1.0;
    oc.fast_kind = fast ? ORC_FAST_CHEM : ORC_FAST_NONE;
    oc.slow_kind = ORC_SLOW_STENCIL;
    oc.S = S; oc.R = R; oc.rho = rho;
    oc.species = species; oc.reactions = reactions; oc.rspecies = rspecies;
    oc.order = order; oc.diffusion = diffusion; oc.vel_kind = 0;
    oc.u_const[0] = oc.u_const[1] = oc.u_const[2] = 1.0;
    oc.threads = 1;
    oc.imex = imex ? 1 : 0;
    oc.d_impl = imex ? d_impl : 0.0;
    oc.cg_iters = cg_iters;
    orc_sys* cs = orc_sys_create(&oc);
    if (!cs) throw std::runtime_error("orc_sys_create failed");
    ProblemInstance cpu;
    cpu.system.dimension = dof;
    if (fast)
      cpu.system.f_fast = [cs](double t, const StateVector& y) {
        StateVector o(y.size());
        orc_sys_fast_rhs(cs, t, y.data(), o.data());
        return o;
      };
    cpu.system.f_explicit = [cs](double t, const StateVector& y) {
      StateVector o(y.size());
      orc_sys_slow_rhs(cs, t, y.data(), o.data());
      return o;
    };
    if (imex) {
      cpu.system.f_implicit = [cs](double t, const StateVector& y) {
        StateVector o(y.size());
        orc_sys_implicit_rhs(cs, t, y.data(), o.data());
        return o;
      };
      cpu.system.jv_implicit = [cs](double t, const StateVector&, const StateVector& v) {
        StateVector o(v.size());
        orc_sys_implicit_rhs(cs, t, v.data(), o.data());
        return o;
      };
    }
    cpu.y0 = y0;
    cpu.component_offset = 0;
    cpu.component_count = (std::size_t)S * ncell;

    // device: the same problem on the GPU, routed
    b200::Device dev(0);
    dev.grid(n, n, n, ncomp);
    dev.chemistry(S, R, rho, species, reactions, rspecies);
    if (!fast) dev.no_fast();
    dev.stencil(order, diffusion, u);
    if (imex) dev.implicit_diffusion(d_impl, cg_iters);
    const ProblemInstance gpu = b200::make_device_problem(dev, y0, 0, (std::size_t)S * ncell);
    b200::route(gpu, dev);

    // the convergence studies' reference (compute_reference, harness.cpp:411-429)
    const StateVector ref_cpu = reference_solution(cpu.system, y0, t0, tf, h_ref);
    const StateVector ref_gpu = b200::reference_solution(dev, y0, t0, tf, h_ref);

    const RunReport rc = study(cpu, cfg, ref_cpu);
    const RunReport rg = study(gpu, cfg, ref_gpu);
    b200::unroute(gpu);
    orc_sys_destroy(cs);
    rc.write_csv(csv_cpu);
    rg.write_csv(csv_dev);
    rg.write_json(json_dev, &cfg);
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// The routed harness on a CPU problem: the reference's own convergence study
// (execute_study, harness.cpp:431-512) of its LinearTwoRateOde through the
// routing functions, which must fall through to the reference's integrators.
// slopes[i] = fitted slope of methods[i] (comma list); returns the row count.
extern "C" int harness_cpu_study(const char* methods, const double* hs, int nh, const char* csv,
                                 double* slopes, char* err, size_t errlen)
{
  try {
    StudyConfig cfg;
    cfg.problem_kind = "linear-two-rate";
    cfg.methods = split(methods);
    cfg.h_list.assign(hs, hs + nh);
    cfg.t0 = 0.0;
    cfg.tf = 1.0;
    cfg.reference_method = "analytic";
    cfg.jobs = 1;
    const RunReport rep = run_convergence_study(cfg);
    rep.write_csv(csv);
    for (std::size_t i = 0; i < cfg.methods.size(); ++i) {
      const auto it = rep.fitted_slopes.find(cfg.methods[i]);
      slopes[i] = it == rep.fitted_slopes.end() ? std::nan("") : it->second;
    }
    return (int)rep.rows.size();
  } catch (const std::exception& e) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.what());
    return -1;
  }
}
