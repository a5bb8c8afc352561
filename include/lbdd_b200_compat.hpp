// lbdd_b200_compat.hpp — drop-in C++ front end for the reference's solver API.
//
// Include this from code built against the reference's headers
// (proj/include/lbdd/*.hpp) and link liblbdd_b200.so: the functions below take
// and return the reference's own types and behave like
//   lbdd::asral_solve   (solver.hpp:133)
//   lbdd::strict_solve  (solver.hpp:227)
//   lbdd::greedy_solve  (solver.hpp:172)
// — same report (solver name, objective, Allotment, SolveStats, PhaseTimings,
// strict_surcharge, has_dummy_center), same exception types for the same
// failures — but solve on a B200 through the C ABI in lbdd_b200.h.
//
// Differences a caller can observe:
//  * costs must fit the device's int32 storage (the reference stores int64);
//    larger costs raise std::invalid_argument like any other invalid instance;
//  * PhaseTimings are device-side (bellman_ford_ns = engine time).
#ifndef LBDD_B200_COMPAT_HPP_
#define LBDD_B200_COMPAT_HPP_

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbdd/refine.hpp"  // RefineOutcome
#include "lbdd/solver.hpp"  // the reference's types (ProblemInstance, SolveReport, ...)
#include "lbdd_b200.h"

namespace lbdd {
namespace b200 {

namespace detail {

[[noreturn]] inline void raise(lbdd_status st) {
  const std::string msg = lbdd_b200_last_error();
  switch (st) {
    case LBDD_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LBDD_ERR_LOGIC: throw std::logic_error(msg);
    case LBDD_ERR_OVERFLOW: throw std::overflow_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void check(lbdd_status st) {
  if (st != LBDD_OK) raise(st);
}

// ProblemInstance (core.hpp:130) flattened into the C descriptor's arrays.
struct FlatInstance {
  std::vector<int32_t> costs;
  std::vector<int64_t> capacity;
  std::vector<int32_t> family;
  std::vector<int64_t> offset;
  std::vector<int64_t> params;
  lbdd_instance_desc desc{};

  explicit FlatInstance(const ProblemInstance& inst) {
    const Count n = inst.n(), k = inst.k();
    const auto& data = inst.cost_matrix.data();
    costs.resize(data.size());
    for (std::size_t i = 0; i < data.size(); ++i) {
      if (data[i] > std::numeric_limits<int32_t>::max()) {
        throw std::invalid_argument(
            "lbdd: invalid instance: cost exceeds the device's int32 cost storage");
      }
      // non-positive costs pass through: the device validation reports them
      // with the reference's message (core.hpp:297-302)
      costs[i] = data[i] < std::numeric_limits<int32_t>::min()
                     ? std::numeric_limits<int32_t>::min()
                     : static_cast<int32_t>(data[i]);
    }
    offset.push_back(0);
    for (const auto& c : inst.centers) {
      capacity.push_back(c.capacity);
      family.push_back(static_cast<int32_t>(c.penalty.family));
      params.insert(params.end(), c.penalty.params.begin(), c.penalty.params.end());
      offset.push_back(static_cast<int64_t>(params.size()));
    }
    desc.n = n;
    desc.k = k;
    desc.costs = costs.data();
    desc.capacity = capacity.data();
    desc.penalty_family = family.data();
    desc.penalty_offset = offset.data();
    desc.penalty_params = params.data();
  }
};

inline lbdd_solver_options to_c(const SolverOptions& o) {
  lbdd_solver_options c{};
  c.parallel = o.parallel;
  c.check_invariants = o.check_invariants;
  c.refine_to_fixpoint = o.refine_to_fixpoint;
  c.workers = o.parallel_config.workers;
  c.chunking = o.parallel_config.chunking;
  c.relax_phase = o.parallel_config.relax_phase;
  c.index_update_phase = o.parallel_config.index_update_phase;
  c.strict_order = o.strict_order.empty() ? nullptr : o.strict_order.data();
  c.strict_order_len = static_cast<int64_t>(o.strict_order.size());
  return c;
}

inline SolveReport solve(const ProblemInstance& instance, const SolverOptions& opts,
                         int32_t kind, int device) {
  if (instance.k() < 1 || instance.n() < 1) require_valid_instance(instance);
  static_assert(sizeof(DemandId) == sizeof(int32_t), "strict_order is passed as int32");
  FlatInstance flat(instance);
  lbdd_b200_instance* h = nullptr;
  check(lbdd_b200_instance_create(&flat.desc, device, &h));
  const Count n = instance.n(), k = instance.k();
  std::vector<int32_t> assignment(static_cast<std::size_t>(n));
  std::vector<int64_t> load(static_cast<std::size_t>(k + 1));
  lbdd_solver_options c = to_c(opts);
  lbdd_solve_report r{};
  const lbdd_status st = lbdd_b200_solve(h, kind, &c, &r, assignment.data(), load.data());
  lbdd_b200_instance_destroy(h);
  if (st != LBDD_OK) raise(st);

  SolveReport report;
  switch (kind) {
    case LBDD_SOLVER_ASRAL: report.solver = opts.parallel ? "para-asral" : "asral"; break;
    case LBDD_SOLVER_STRICT: report.solver = "strict"; break;
    default: report.solver = "greedy"; break;
  }
  report.objective = r.objective;
  report.strict_surcharge = r.strict_surcharge;
  report.has_dummy_center = r.has_dummy_center != 0;
  report.assignment.assignment.assign(assignment.begin(), assignment.end());
  report.assignment.load.assign(load.begin(), load.begin() + (r.has_dummy_center ? k + 1 : k));
  report.stats.cycle_refine_calls = r.cycle_refine_calls;
  report.stats.path_refine_calls = r.path_refine_calls;
  report.stats.negative_cycles_removed = r.negative_cycles_removed;
  report.stats.negative_paths_removed = r.negative_paths_removed;
  report.stats.refinement_gain = r.refinement_gain;
  report.stats.transfers_applied = r.transfers_applied;
  report.stats.invariant_checks = r.invariant_checks;
  report.timings.index_update_ns = r.index_update_ns;
  report.timings.bellman_ford_ns = r.bellman_ford_ns;
  report.timings.total_ns = r.total_ns;
  return report;
}

}  // namespace detail

inline SolveReport asral_solve(const ProblemInstance& instance, const SolverOptions& opts = {},
                               int device = 0) {
  return detail::solve(instance, opts, LBDD_SOLVER_ASRAL, device);
}

inline SolveReport strict_solve(const ProblemInstance& instance, const SolverOptions& opts = {},
                                int device = 0) {
  return detail::solve(instance, opts, LBDD_SOLVER_STRICT, device);
}

inline SolveReport greedy_solve(const ProblemInstance& instance, const SolverOptions& opts = {},
                                int device = 0) {
  return detail::solve(instance, opts, LBDD_SOLVER_GREEDY, device);
}

namespace detail {

// One refinement through lbdd_b200_refine on a reference SolverState
// (solver.hpp:35-67): the state's allotment (and strict placeholders) go to
// the device, the refined allotment comes back; the running objective,
// stats and the transfer index follow like in refine.hpp:173-224.
template <typename State>
RefineOutcome refine(State& st, CenterId anchor, int32_t kind, int device) {
  const ProblemInstance& inst = *st.instance;
  FlatInstance flat(inst);
  lbdd_b200_instance* h = nullptr;
  check(lbdd_b200_instance_create(&flat.desc, device, &h));
  std::vector<int32_t> assignment(st.allotment.assignment.begin(), st.allotment.assignment.end());
  std::vector<int64_t> dummies;
  if (auto* dm = st.dummy_counts()) dummies.assign(dm->begin(), dm->end());
  int32_t applied = 0;
  int64_t gain = 0;
  const lbdd_status rc = lbdd_b200_refine(h, kind, anchor, assignment.data(),
                                          dummies.empty() ? nullptr : dummies.data(), &applied,
                                          &gain);
  lbdd_b200_instance_destroy(h);
  if (kind == 0) ++st.stats.cycle_refine_calls;
  else ++st.stats.path_refine_calls;
  if (rc != LBDD_OK) raise(rc);
  RefineOutcome out;
  if (applied) {
    Allotment a = Allotment::empty(inst.n(), inst.k());
    for (DemandId d = 0; d < inst.n(); ++d) {
      if (assignment[static_cast<std::size_t>(d)] >= 0) a.assign(d, assignment[static_cast<std::size_t>(d)]);
    }
    st.allotment = std::move(a);
    st.index = build_index(inst, st.allotment);
    if (auto* dm = st.dummy_counts()) dm->assign(dummies.begin(), dummies.end());
    st.delta = checked_add(st.delta, gain);
    if (kind == 0) ++st.stats.negative_cycles_removed;
    else ++st.stats.negative_paths_removed;
    st.stats.refinement_gain = checked_add(st.stats.refinement_gain, -gain);
    out = {true, gain};
  }
  return out;
}

}  // namespace detail

// negative_cycle_refine / negative_path_refine (refine.hpp:173, 199) on the
// reference's SolverState, computed on the B200.
template <typename State>
RefineOutcome negative_cycle_refine(State& st, CenterId anchor, int device = 0) {
  return detail::refine(st, anchor, 0, device);
}
template <typename State>
RefineOutcome negative_path_refine(State& st, CenterId anchor, int device = 0) {
  return detail::refine(st, anchor, 1, device);
}

}  // namespace b200
}  // namespace lbdd

#endif  // LBDD_B200_COMPAT_HPP_
