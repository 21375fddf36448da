// multirate_b200_harness.hpp -- routes the reference study harness's per-run
// entry point, multirate::run_method (proj/src/harness.cpp:323-394), to the
// device for problems that live on a multirate::b200::Device, WITHOUT editing
// harness.cpp: the harness is compiled unmodified with
//
//   -include multirate_b200_harness.hpp
//   -Dmri_integrate=mri_integrate_routed
//   -Dark_imex_integrate=ark_imex_integrate_routed
//   -Derk_integrate=erk_integrate_routed
//   -Dsdc_integrate=sdc_integrate_routed
//   -Dmrsdc_integrate=mrsdc_integrate_routed
//
// so every case of run_method -- Mri, ArkImex, Erk, Sdc, Mrsdc -- calls one of
// the five routing functions
// declared below (their definitions are compiled once, WITHOUT those macros,
// in a translation unit that defines MULTIRATE_B200_HARNESS_IMPL before
// including this header).  A routed problem (b200::route) goes to the facade
// -- mri_integrate / ark_imex_integrate / erk_integrate / sdc_integrate /
// mrsdc_integrate on the device-resident
// state, the counters filled exactly like the reference's -- and every other
// problem to the reference's own integrators, so CPU studies are unchanged.
// run_method's divergence handling (IntegrationError -> RunOutcome::diverged,
// harness.cpp:391-394), its counters and wall-clock timing, and the
// RunReport CSV/JSON writers (:645-705) apply to device runs as they are.
//
// The routing key is the address of ProblemInstance::y0: run_method passes
// problem.y0 by reference to every integrator (harness.cpp:346-386).  The
// Device is not thread-safe: run device problems with StudyConfig::jobs = 1.
// INTEGRATION.md shows the recipe; oracle/harness_test.cpp drives it.
#ifndef MULTIRATE_B200_HARNESS_HPP_
#define MULTIRATE_B200_HARNESS_HPP_

#include <cstddef>

#include "multirate/erk.hpp"
#include "multirate/harness.hpp"
#include "multirate/mri.hpp"
#include "multirate/sdc.hpp"

namespace multirate {

StateVector mri_integrate_routed(const MriMethodConfig& config, const PartitionedSystem& system,
                                 const ImplicitStageSolver& solver, double t0, double tf,
                                 double H, const StateVector& y0, EvalCounters& counters);
StateVector ark_imex_integrate_routed(const ArkPair& pair, const PartitionedSystem& system,
                                      const ImplicitStageSolver& solver, double t0, double tf,
                                      double H, const StateVector& y0, EvalCounters& counters);
StateVector erk_integrate_routed(const ButcherTable& table, const RhsFn& f, double t0, double tf,
                                 double h, const StateVector& y0, std::size_t* eval_counter);
StateVector sdc_integrate_routed(const QuadratureNodes& nodes, const RhsFn& f_total, double t0,
                                 double tf, double H, const StateVector& y0, int n_sweeps,
                                 std::size_t* eval_counter);
StateVector mrsdc_integrate_routed(const MrsdcScheme& scheme, const PartitionedSystem& system,
                                   double t0, double tf, double H, const StateVector& y0,
                                   EvalCounters& counters);

}  // namespace multirate

#ifdef MULTIRATE_B200_HARNESS_IMPL
#include <map>
#include <mutex>

#include "multirate_b200.hpp"

namespace multirate::b200 {

inline std::map<const StateVector*, Device*>& routed_problems()
{
  static std::map<const StateVector*, Device*> m;
  return m;
}
inline std::mutex& routed_mutex()
{
  static std::mutex mu;
  return mu;
}

// Mark `problem` (at its final address) as living on `device`: its y0 is
// the device grid's state layout and its PartitionedSystem is the device's
// (b200::partitioned_system, so the Mode-A callbacks agree with the device).
inline void route(const ProblemInstance& problem, Device& device)
{
  if (problem.y0.size() != device.dof())
    throw ContractError("b200::route: problem state size != device grid dof");
  std::lock_guard<std::mutex> g(routed_mutex());
  routed_problems()[&problem.y0] = &device;
}
inline void unroute(const ProblemInstance& problem)
{
  std::lock_guard<std::mutex> g(routed_mutex());
  routed_problems().erase(&problem.y0);
}
inline Device* routed_device(const StateVector& y0)
{
  std::lock_guard<std::mutex> g(routed_mutex());
  const auto it = routed_problems().find(&y0);
  return it == routed_problems().end() ? nullptr : it->second;
}

// A ProblemInstance for the device plugins (the harness's make_problem,
// harness.cpp:280-314, for a device problem): Mode-A system, the given
// initial state, the error slice.  Call route() once it is at its final place.
inline ProblemInstance make_device_problem(Device& device, const StateVector& y0,
                                           std::size_t component_offset = 0,
                                           std::size_t component_count = 0)
{
  ProblemInstance p;
  p.system = partitioned_system(device);
  p.y0 = y0;
  p.component_offset = component_offset;
  p.component_count = component_count;
  return p;
}

}  // namespace multirate::b200

namespace multirate {

StateVector mri_integrate_routed(const MriMethodConfig& config, const PartitionedSystem& system,
                                 const ImplicitStageSolver& solver, double t0, double tf,
                                 double H, const StateVector& y0, EvalCounters& counters)
{
  if (b200::Device* d = b200::routed_device(y0))
    return b200::mri_integrate(*d, config, solver, t0, tf, H, y0, counters);
  return mri_integrate(config, system, solver, t0, tf, H, y0, counters);
}

StateVector ark_imex_integrate_routed(const ArkPair& pair, const PartitionedSystem& system,
                                      const ImplicitStageSolver& solver, double t0, double tf,
                                      double H, const StateVector& y0, EvalCounters& counters)
{
  if (b200::Device* d = b200::routed_device(y0)) {
    // the device integrates the ARK4(3)6L[2]SA pair, the only pair run_method uses
    if (pair.name != "ark436-imex-pair")
      throw ContractError("b200: the device ARK-IMEX integrator implements ark436-imex-pair only");
    return b200::ark_imex_integrate(*d, solver, t0, tf, H, y0, counters);
  }
  return ark_imex_integrate(pair, system, solver, t0, tf, H, y0, counters);
}

StateVector erk_integrate_routed(const ButcherTable& table, const RhsFn& f, double t0, double tf,
                                 double h, const StateVector& y0, std::size_t* eval_counter)
{
  // run_method's Erk case integrates problem.system.sum_rhs (harness.cpp:346-355)
  if (b200::Device* d = b200::routed_device(y0))
    return b200::erk_integrate(*d, table, t0, tf, h, y0, eval_counter);
  return erk_integrate(table, f, t0, tf, h, y0, eval_counter);
}

StateVector sdc_integrate_routed(const QuadratureNodes& nodes, const RhsFn& f_total, double t0,
                                 double tf, double H, const StateVector& y0, int n_sweeps,
                                 std::size_t* eval_counter)
{
  // run_method's Sdc case integrates problem.system.sum_rhs (harness.cpp:356-366)
  if (b200::Device* d = b200::routed_device(y0))
    return b200::sdc_integrate(*d, nodes, t0, tf, H, y0, n_sweeps, eval_counter);
  return sdc_integrate(nodes, f_total, t0, tf, H, y0, n_sweeps, eval_counter);
}

StateVector mrsdc_integrate_routed(const MrsdcScheme& scheme, const PartitionedSystem& system,
                                   double t0, double tf, double H, const StateVector& y0,
                                   EvalCounters& counters)
{
  if (b200::Device* d = b200::routed_device(y0))
    return b200::mrsdc_integrate(*d, scheme, t0, tf, H, y0, counters);
  return mrsdc_integrate(scheme, system, t0, tf, H, y0, counters);
}

}  // namespace multirate
#endif  // MULTIRATE_B200_HARNESS_IMPL
#endif  // MULTIRATE_B200_HARNESS_HPP_
