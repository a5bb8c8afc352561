// TEST INFRASTRUCTURE ONLY: drop-in check of include/lbdd_b200_compat.hpp.
//
// Built by oracle/Makefile (target `dropin`) against the UNMODIFIED reference
// headers, into oracle/_ref/drop_in_check. It solves the same seeded
// instances twice — lbdd::asral_solve / strict_solve / greedy_solve from the
// reference (solver.hpp:133,227,172) and lbdd::b200::* from the compat
// header, which goes through liblbdd_b200.so on the GPU — and requires
// identical reports: solver name, objective, assignment, loads, stats,
// strict surcharge, and the same exception type on an invalid instance.
// Run by tests/test_gpu_parity.py::test_cpp_drop_in (needs a GPU).
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "lbdd_b200_compat.hpp"

namespace {

struct Rng {  // splitmix64: independent of the reference's generators
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  int64_t in(int64_t lo, int64_t hi) { return lo + static_cast<int64_t>(next() % (hi - lo + 1)); }
};

lbdd::ProblemInstance make_instance(uint64_t seed, lbdd::Count n, lbdd::Count k, double theta) {
  Rng r{seed};
  lbdd::ProblemInstance inst;
  inst.demand_count = n;
  const lbdd::Count total = static_cast<lbdd::Count>(theta * static_cast<double>(n));
  for (lbdd::Count s = 0; s < k; ++s) {
    lbdd::ServiceCenter c;
    c.id = static_cast<lbdd::CenterId>(s);
    c.capacity = total / k + (s < total % k ? 1 : 0);
    switch (r.next() % 3) {
      case 0: c.penalty = lbdd::PenaltySpec::constant(r.in(1, 60)); break;
      case 1: c.penalty = lbdd::PenaltySpec::linear(r.in(1, 30), r.in(0, 9)); break;
      default: {
        std::vector<lbdd::Cost> t(static_cast<std::size_t>(r.in(1, 4)));
        lbdd::Cost v = r.in(1, 20);
        for (auto& x : t) { x = v; v += r.in(0, 15); }
        c.penalty = lbdd::PenaltySpec::table(t);
      }
    }
    inst.centers.push_back(c);
  }
  std::vector<lbdd::Cost> costs(static_cast<std::size_t>(n * k));
  for (auto& x : costs) x = r.in(1, 100);
  inst.cost_matrix = lbdd::CostMatrix(n, k, std::move(costs));
  return inst;
}

int failures = 0;

void expect(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("MISMATCH %s\n", what.c_str());
  }
}

void compare(const lbdd::SolveReport& a, const lbdd::SolveReport& b, const std::string& tag) {
  if (std::getenv("DROP_IN_VERBOSE")) std::fprintf(stderr, "  compared %s\n", tag.c_str());
  expect(a.solver == b.solver, tag + " solver name " + a.solver + " vs " + b.solver);
  expect(a.objective == b.objective, tag + " objective");
  expect(a.assignment.assignment == b.assignment.assignment, tag + " assignment");
  expect(a.assignment.load == b.assignment.load, tag + " load");
  expect(a.strict_surcharge == b.strict_surcharge, tag + " strict_surcharge");
  expect(a.has_dummy_center == b.has_dummy_center, tag + " has_dummy_center");
  expect(a.stats.cycle_refine_calls == b.stats.cycle_refine_calls, tag + " cycle_refine_calls");
  expect(a.stats.path_refine_calls == b.stats.path_refine_calls, tag + " path_refine_calls");
  expect(a.stats.negative_cycles_removed == b.stats.negative_cycles_removed, tag + " cycles");
  expect(a.stats.negative_paths_removed == b.stats.negative_paths_removed, tag + " paths");
  expect(a.stats.refinement_gain == b.stats.refinement_gain, tag + " refinement_gain");
  expect(a.stats.transfers_applied == b.stats.transfers_applied, tag + " transfers_applied");
}

template <typename F>
std::string thrown(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return "invalid_argument";
  } catch (const std::overflow_error&) {
    return "overflow_error";
  } catch (const std::logic_error&) {
    return "logic_error";
  } catch (const std::exception&) {
    return "other";
  }
  return "none";
}

}  // namespace

int main(int argc, char** argv) {
  const int cases = argc > 1 ? std::atoi(argv[1]) : 12;
  int solves = 0;
  for (int c = 0; c < cases; ++c) {
    const lbdd::Count n = 40 + 37 * c, k = 3 + c % 9;
    const double theta = (c % 3 == 0) ? 1.2 : (c % 3 == 1 ? 0.8 : 1.0);
    const auto inst = make_instance(1000 + c, n, k, theta);
    if (std::getenv("DROP_IN_VERBOSE")) {
      std::fprintf(stderr, "case %d: n %lld k %lld theta %.1f\n", c, static_cast<long long>(n),
                   static_cast<long long>(k), theta);
    }
    for (int fix = 0; fix < 2; ++fix) {
      lbdd::SolverOptions o;
      o.refine_to_fixpoint = fix != 0;
      const std::string tag = "case " + std::to_string(c) + " fix " + std::to_string(fix);
      compare(lbdd::asral_solve(inst, o), lbdd::b200::asral_solve(inst, o), tag + " asral");
      compare(lbdd::strict_solve(inst, o), lbdd::b200::strict_solve(inst, o), tag + " strict");
      solves += 2;
    }
    compare(lbdd::greedy_solve(inst), lbdd::b200::greedy_solve(inst), "greedy " + std::to_string(c));
    // para-asral: the reference's WorkerPool (parallel.hpp:31-124) can lose
    // the done_cv_ wake-up in run() and hang, so its result is taken from
    // the sequential solver, which it must equal (parallel_test.cpp); the
    // lost wake-up: drain() notifies done_cv_ without the mutex (parallel.hpp:91-92)
    lbdd::SolverOptions par;
    par.parallel = true;
    par.parallel_config.workers = 4;
    auto seq = lbdd::asral_solve(inst);
    seq.solver = "para-asral";
    compare(seq, lbdd::b200::asral_solve(inst, par), "para-asral " + std::to_string(c));
    solves += 2;
  }
  // invalid instance: same exception type as the reference
  auto bad = make_instance(7, 20, 3, 1.0);
  std::vector<lbdd::Cost> costs = bad.cost_matrix.data();
  costs[5] = 0;
  bad.cost_matrix = lbdd::CostMatrix(20, 3, costs);
  const std::string e_ref = thrown([&] { lbdd::asral_solve(bad); });
  const std::string e_gpu = thrown([&] { lbdd::b200::asral_solve(bad); });
  expect(e_ref == e_gpu, "invalid instance: reference " + e_ref + " vs b200 " + e_gpu);
  std::printf("drop-in %s: %d solves compared, %d mismatches\n", failures ? "FAILED" : "ok",
              solves, failures);
  return failures ? 1 : 0;
}
