// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library, compiled directly from
// the reference's header-only sources where they lie
// (/root/reference/proj/include/lbdd/*.hpp) by oracle/Makefile into
// oracle/_ref/liblbdd_ref.so. Nothing here reimplements the algorithm: every
// entry point constructs the reference's own types and calls its functions,
// so the outputs are the reference's outputs. Used by tests/ (parity and
// golden-vector generation) and by bench.py's reference / cpu_baseline arm.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "lbdd/core.hpp"
#include "lbdd/instgen.hpp"
#include "lbdd/oracle.hpp"
#include "lbdd/refine.hpp"
#include "lbdd/solver.hpp"
#include "lbdd/subspace.hpp"

#include "lbdd_b200.h"  // shared plain-C structs only

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return LBDD_OK;
  } catch (const std::overflow_error& e) {
    return fail(LBDD_ERR_OVERFLOW, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(LBDD_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::logic_error& e) {
    return fail(LBDD_ERR_LOGIC, e.what());
  } catch (const std::runtime_error& e) {
    return fail(LBDD_ERR_RUNTIME, e.what());
  } catch (const std::exception& e) {
    return fail(LBDD_ERR_RUNTIME, e.what());
  }
}

lbdd::ProblemInstance to_instance(const lbdd_instance_desc* d) {
  lbdd::ProblemInstance inst;
  inst.demand_count = d->n;
  for (int64_t s = 0; s < d->k; ++s) {
    lbdd::ServiceCenter c;
    c.id = static_cast<lbdd::CenterId>(s);
    c.capacity = d->capacity[s];
    c.penalty.family =
        static_cast<lbdd::PenaltySpec::Family>(d->penalty_family[s]);
    for (int64_t i = d->penalty_offset[s]; i < d->penalty_offset[s + 1]; ++i) {
      c.penalty.params.push_back(d->penalty_params[i]);
    }
    inst.centers.push_back(std::move(c));
  }
  std::vector<lbdd::Cost> costs(static_cast<std::size_t>(d->n * d->k));
  for (std::size_t i = 0; i < costs.size(); ++i) costs[i] = d->costs[i];
  inst.cost_matrix = lbdd::CostMatrix(d->n, d->k, std::move(costs));
  return inst;
}

lbdd::Allotment to_allotment(const lbdd::ProblemInstance& inst,
                             const int32_t* assignment) {
  lbdd::Allotment a = lbdd::Allotment::empty(inst.n(), inst.k());
  for (int64_t d = 0; d < inst.n(); ++d) {
    if (assignment[d] >= 0) a.assign(static_cast<lbdd::DemandId>(d), assignment[d]);
  }
  return a;
}

lbdd::SolverOptions to_options(const lbdd_solver_options* o) {
  lbdd::SolverOptions opts;
  if (o == nullptr) return opts;
  opts.parallel = o->parallel != 0;
  opts.check_invariants = o->check_invariants != 0;
  opts.refine_to_fixpoint = o->refine_to_fixpoint != 0;
  opts.parallel_config.workers = o->workers > 0 ? o->workers : 1;
  if (o->chunking > 0) opts.parallel_config.chunking = o->chunking;
  opts.parallel_config.relax_phase = o->relax_phase != 0;
  opts.parallel_config.index_update_phase = o->index_update_phase != 0;
  if (o->strict_order != nullptr) {
    opts.strict_order.assign(o->strict_order,
                             o->strict_order + o->strict_order_len);
  }
  return opts;
}

void fill_report(const lbdd::SolveReport& r, int32_t solver,
                 lbdd_solve_report* out, int32_t* assignment, int64_t* load) {
  std::memset(out, 0, sizeof(*out));
  out->objective = r.objective;
  out->strict_surcharge = r.strict_surcharge;
  out->has_dummy_center = r.has_dummy_center ? 1 : 0;
  out->solver = solver;
  out->cycle_refine_calls = r.stats.cycle_refine_calls;
  out->path_refine_calls = r.stats.path_refine_calls;
  out->negative_cycles_removed = r.stats.negative_cycles_removed;
  out->negative_paths_removed = r.stats.negative_paths_removed;
  out->refinement_gain = r.stats.refinement_gain;
  out->transfers_applied = r.stats.transfers_applied;
  out->invariant_checks = r.stats.invariant_checks;
  out->index_update_ns = r.timings.index_update_ns;
  out->bellman_ford_ns = r.timings.bellman_ford_ns;
  out->total_ns = r.timings.total_ns;
  if (assignment) {
    for (std::size_t d = 0; d < r.assignment.assignment.size(); ++d) {
      assignment[d] = r.assignment.assignment[d];
    }
  }
  if (load) {
    for (std::size_t s = 0; s < r.assignment.load.size(); ++s) {
      load[s] = r.assignment.load[s];
    }
  }
}

}  // namespace

extern "C" {

const char* lbdd_ref_last_error(void) { return g_err.c_str(); }

int lbdd_ref_solve(const lbdd_instance_desc* desc, int32_t solver,
                   const lbdd_solver_options* o, lbdd_solve_report* report,
                   int32_t* assignment, int64_t* load) {
  return guarded([&] {
    const auto inst = to_instance(desc);
    auto opts = to_options(o);
    lbdd::SolveReport r;
    switch (solver) {
      case LBDD_SOLVER_ASRAL: r = lbdd::asral_solve(inst, opts); break;
      case LBDD_SOLVER_PARA_ASRAL:
        opts.parallel = true;
        r = lbdd::asral_solve(inst, opts);
        break;
      case LBDD_SOLVER_STRICT: r = lbdd::strict_solve(inst, opts); break;
      case LBDD_SOLVER_GREEDY: r = lbdd::greedy_solve(inst, opts); break;
      default: throw std::invalid_argument("unknown solver");
    }
    fill_report(r, solver, report, assignment, load);
  });
}

// oracle_solve (oracle.hpp:144): exact min-cost-flow optimum.
int lbdd_ref_oracle_solve(const lbdd_instance_desc* desc, int32_t strict,
                          int64_t size_limit, int64_t* objective,
                          int64_t* surcharge, int32_t* has_dummy,
                          int32_t* assignment) {
  return guarded([&] {
    const auto inst = to_instance(desc);
    const auto r = lbdd::oracle_solve(inst, strict != 0, size_limit);
    *objective = r.objective;
    *surcharge = r.surcharge;
    *has_dummy = r.has_dummy_center ? 1 : 0;
    if (assignment) {
      for (std::size_t d = 0; d < r.assignment.size(); ++d) {
        assignment[d] = r.assignment[d];
      }
    }
  });
}

// build_index (subspace.hpp:233) read back as the packed min-transfer matrix.
int lbdd_ref_build_index(const lbdd_instance_desc* desc,
                         const int32_t* assignment, int64_t* out) {
  return guarded([&] {
    const auto inst = to_instance(desc);
    const auto a = to_allotment(inst, assignment);
    const auto index = lbdd::build_index(inst, a);
    const int64_t k = inst.k();
    for (int64_t u = 0; u < k; ++u) {
      for (int64_t v = 0; v < k; ++v) {
        int64_t packed = INT64_MAX;
        if (u != v) {
          if (auto e = index.min_transfer(static_cast<lbdd::CenterId>(u),
                                          static_cast<lbdd::CenterId>(v))) {
            packed = static_cast<int64_t>(
                (static_cast<uint64_t>(e->cost) << 32) |
                static_cast<uint32_t>(e->demand));
          }
        }
        out[u * k + v] = packed;
      }
    }
  });
}

// One refinement through `anchor` on SolverState::from_allotment.
int lbdd_ref_refine(const lbdd_instance_desc* desc, int32_t kind,
                    int32_t anchor, int32_t* assignment, int64_t* dummies,
                    int32_t* applied, int64_t* gain) {
  return guarded([&] {
    const auto inst = to_instance(desc);
    auto st = lbdd::SolverState::from_allotment(inst, to_allotment(inst, assignment));
    if (dummies != nullptr) {
      st.strict = true;
      st.dummies.assign(dummies, dummies + inst.k());
    }
    const auto out = kind == 0 ? lbdd::negative_cycle_refine(st, anchor)
                               : lbdd::negative_path_refine(st, anchor);
    *applied = out.applied ? 1 : 0;
    *gain = out.gain;
    for (int64_t d = 0; d < inst.n(); ++d) {
      assignment[d] = st.allotment.assignment[static_cast<std::size_t>(d)];
    }
    if (dummies != nullptr) {
      for (int64_t s = 0; s < inst.k(); ++s) dummies[s] = st.dummies[static_cast<std::size_t>(s)];
    }
  });
}

int lbdd_ref_gamma_has_negative_cycle(const lbdd_instance_desc* desc,
                                      const int32_t* assignment,
                                      const int64_t* dummies,
                                      int32_t* has_cycle) {
  return guarded([&] {
    const auto inst = to_instance(desc);
    const auto index = lbdd::build_index(inst, to_allotment(inst, assignment));
    std::vector<lbdd::Count> dv;
    if (dummies) dv.assign(dummies, dummies + inst.k());
    *has_cycle = lbdd::gamma_has_negative_cycle(index, dummies ? &dv : nullptr) ? 1 : 0;
  });
}

// lowest_cost_path (refine.hpp:28) on a dense encoding; edges are inserted
// in (u, v) order so AuxGraph::finalize sees the same ordering as
// build_negcycle_graph (subspace.hpp:319-327).
int lbdd_ref_lowest_cost_path(int32_t node_count, int32_t anchor,
                              const int64_t* weights, int32_t* found,
                              int64_t* cost, int64_t* dist,
                              int32_t* parent_node, int32_t* path,
                              int32_t* path_len) {
  return guarded([&] {
    lbdd::AuxGraph g;
    g.anchor = anchor;
    g.node_count = node_count;
    int32_t demand = 0;
    for (int32_t u = 0; u + 1 < node_count; ++u) {
      for (int32_t v = 0; v < node_count; ++v) {
        const int64_t w = weights[static_cast<int64_t>(u) * node_count + v];
        if (w == INT64_MAX) continue;
        g.add_edge(lbdd::AuxEdge{u, v, lbdd::AuxEdgeKind::transfer, demand++, w});
      }
    }
    g.finalize();
    const auto r = lbdd::lowest_cost_path(g, lbdd::Engine{});
    *found = r.has_value() ? 1 : 0;
    *path_len = 0;
    if (!r) return;
    *cost = r->cost;
    for (int32_t v = 0; v < node_count; ++v) {
      dist[v] = r->distances[static_cast<std::size_t>(v)];
      const int32_t e = r->parents[static_cast<std::size_t>(v)];
      parent_node[v] = e < 0 ? -1 : g.edges[static_cast<std::size_t>(e)].from;
    }
    int32_t len = 0;
    path[0] = r->edges.front().from;
    for (const auto& e : r->edges) path[++len] = e.to;
    *path_len = len;
  });
}

int lbdd_ref_relax_round(int32_t node_count, const int64_t* weights,
                         const int64_t* dist_in, const int32_t* parent_in,
                         int64_t* dist_out, int32_t* parent_out,
                         int32_t* changed) {
  return guarded([&] {
    lbdd::AuxGraph g;
    g.anchor = 0;
    g.node_count = node_count;
    std::vector<int32_t> edge_of;  // parent node ids -> edge ids for input
    for (int32_t u = 0; u + 1 < node_count; ++u) {
      for (int32_t v = 0; v < node_count; ++v) {
        const int64_t w = weights[static_cast<int64_t>(u) * node_count + v];
        if (w == INT64_MAX) continue;
        g.add_edge(lbdd::AuxEdge{u, v, lbdd::AuxEdgeKind::transfer, 0, w});
      }
    }
    g.finalize();
    const auto nodes = static_cast<std::size_t>(node_count);
    std::vector<lbdd::Cost> din(dist_in, dist_in + nodes), dout(nodes);
    std::vector<int32_t> pin(nodes, -1), pout(nodes);
    // parent_in arrives as source nodes; map to the edge (u -> v)
    for (int32_t v = 0; v < node_count; ++v) {
      if (parent_in[v] < 0) continue;
      for (std::size_t e = 0; e < g.edges.size(); ++e) {
        if (g.edges[e].from == parent_in[v] && g.edges[e].to == v) {
          pin[static_cast<std::size_t>(v)] = static_cast<int32_t>(e);
        }
      }
    }
    *changed = lbdd::parallel_relax_round(g, din, pin, dout, pout, lbdd::Engine{}) ? 1 : 0;
    for (int32_t v = 0; v < node_count; ++v) {
      dist_out[v] = dout[static_cast<std::size_t>(v)];
      const int32_t e = pout[static_cast<std::size_t>(v)];
      parent_out[v] = e < 0 ? -1 : g.edges[static_cast<std::size_t>(e)].from;
    }
  });
}

// generate (instgen.hpp:245). k = derive_center_count(n, ratio); the caller
// sizes capacity/penalty arrays to k and costs to n*k (int32 narrowing is
// checked). cost_source: 0 euclidean, 1 road graph.
int lbdd_ref_generate(uint64_t seed, int64_t n, double ratio, double theta,
                      int64_t pen_lo, int64_t pen_hi, int32_t cost_source,
                      int64_t road_nodes, double avg_degree, int64_t* k_out,
                      int64_t* capacity, int64_t* penalty, int32_t* costs) {
  return guarded([&] {
    lbdd::GenConfig cfg;
    cfg.seed = seed;
    cfg.n = n;
    cfg.ratio = ratio;
    cfg.theta = theta;
    cfg.penalty_range = {pen_lo, pen_hi};
    cfg.cost_source = cost_source == 0 ? lbdd::GenConfig::CostSource::euclidean
                                       : lbdd::GenConfig::CostSource::road_graph;
    cfg.road.nodes = road_nodes;
    cfg.road.avg_degree = avg_degree;
    const auto inst = lbdd::generate(cfg);
    *k_out = inst.k();
    if (capacity == nullptr) return;  // size query
    for (int64_t s = 0; s < inst.k(); ++s) {
      capacity[s] = inst.centers[static_cast<std::size_t>(s)].capacity;
      penalty[s] = inst.centers[static_cast<std::size_t>(s)].penalty.params[0];
    }
    const auto& data = inst.cost_matrix.data();
    for (std::size_t i = 0; i < data.size(); ++i) {
      if (data[i] > INT32_MAX) throw std::overflow_error("cost exceeds int32");
      costs[i] = static_cast<int32_t>(data[i]);
    }
  });
}

int64_t lbdd_ref_derive_center_count(int64_t n, double ratio) {
  return lbdd::derive_center_count(n, ratio);
}

}  // extern "C"

extern "C" {
// Bounded sample of the reference's asral main loop for the CPU baseline:
// solver.hpp:135-167 verbatim in structure, stopped after `max_arrivals`
// arrivals (no finish_report). Uses only the reference's own types.
int lbdd_ref_asral_sample(const lbdd_instance_desc* desc, int64_t max_arrivals,
                          int32_t workers, int64_t* elapsed_ns, int64_t* arrivals_done,
                          int64_t* setup_ns) {
  return guarded([&] {
    const auto inst = to_instance(desc);
    lbdd::require_valid_instance(inst);
    const auto start = std::chrono::steady_clock::now();
    lbdd::SolverOptions opts;
    opts.parallel = workers > 1;  // para-asral: the reference's worker pool
    opts.parallel_config.workers = workers;
    lbdd::detail::EngineScope scope(opts, opts.parallel);
    lbdd::SolverState st(inst);
    st.engine = scope.engine;
    auto queue = lbdd::detail::build_arrival_queue(inst);
    *setup_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                    std::chrono::steady_clock::now() - start).count();
    int64_t done = 0;
    while (!queue.empty() && done < max_arrivals) {
      const auto [cost, d, s] = queue.top();
      queue.pop();
      st.index.insert(d, s);
      st.allotment.assign(d, s);
      lbdd::negative_cycle_refine(st, s);
      const auto& center = inst.centers[static_cast<std::size_t>(s)];
      const lbdd::Count load = st.allotment.load[static_cast<std::size_t>(s)];
      if (load <= center.capacity) {
        st.delta = lbdd::checked_add(st.delta, cost);
      } else {
        st.delta = lbdd::checked_add(
            st.delta, lbdd::checked_add(cost, lbdd::refund_penalty(center, load)));
        lbdd::negative_path_refine(st, s);
      }
      ++done;
    }
    *elapsed_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - start).count();
    *arrivals_done = done;
  });
}
}  // extern "C"

extern "C" {
// The reference's asral_solve (solver.hpp:133-170) run to completion, with
// progress marks: the loop of solver.hpp:143-166 over the reference's own
// types and functions, closed by the reference's own detail::finish_report
// (objective recount + tracked-delta check). marks[i] = elapsed ns after
// (i + 1) * mark_every arrivals; a line goes to stderr at each mark. Used to
// pin the GPU solve at scale (tests/golden/scale/) and to time the full CPU
// solve for bench.py's baseline. Sequential (the reference's
// worker pool can lose a wake-up).
// ckpt_every > 0: every ckpt_every arrivals, the centers of the arrivals so
// far (in arrival order, int16) are written to <ckpt_prefix><count>.i16 —
// resumable states for the bench's steady-state CPU samples
// (lbdd_ref_resume_new).
int lbdd_ref_asral_run(const lbdd_instance_desc* desc, int64_t mark_every,
                       int64_t* marks, int64_t max_marks, lbdd_solve_report* report,
                       int32_t* assignment, int64_t* load, int64_t* setup_ns,
                       int64_t ckpt_every, const char* ckpt_prefix) {
  return guarded([&] {
    auto inst = to_instance(desc);
    lbdd::require_valid_instance(inst);
    const auto start = std::chrono::steady_clock::now();
    auto since = [&] {
      return std::chrono::duration_cast<std::chrono::nanoseconds>(
                 std::chrono::steady_clock::now() - start).count();
    };
    lbdd::SolverState st(inst);
    auto queue = lbdd::detail::build_arrival_queue(inst);
    *setup_ns = since();
    int64_t done = 0;
    std::vector<lbdd::DemandId> popped;
    while (!queue.empty()) {
      const auto [cost, d, s] = queue.top();
      queue.pop();
      if (ckpt_every > 0) popped.push_back(d);
      st.index.insert(d, s);
      st.allotment.assign(d, s);
      lbdd::negative_cycle_refine(st, s);
      const auto& center = inst.centers[static_cast<std::size_t>(s)];
      const lbdd::Count ld = st.allotment.load[static_cast<std::size_t>(s)];
      if (ld <= center.capacity) {
        st.delta = lbdd::checked_add(st.delta, cost);
      } else {
        st.delta = lbdd::checked_add(
            st.delta, lbdd::checked_add(cost, lbdd::refund_penalty(center, ld)));
        lbdd::negative_path_refine(st, s);
      }
      ++done;
      if (mark_every > 0 && done % mark_every == 0) {
        const int64_t i = done / mark_every - 1;
        const int64_t t = since();
        if (i < max_marks) marks[i] = t;
        std::fprintf(stderr, "[ref] %lld arrivals %.1f s delta %lld\n",
                     static_cast<long long>(done), t / 1e9,
                     static_cast<long long>(st.delta));
        std::fflush(stderr);
      }
      if (ckpt_every > 0 && done % ckpt_every == 0) {
        std::vector<int16_t> cs(popped.size());
        for (std::size_t i = 0; i < popped.size(); ++i) {
          cs[i] = static_cast<int16_t>(st.allotment.assignment[static_cast<std::size_t>(popped[i])]);
        }
        const std::string path = std::string(ckpt_prefix) + std::to_string(done) + ".i16";
        if (FILE* f = std::fopen(path.c_str(), "wb")) {
          std::fwrite(cs.data(), sizeof(int16_t), cs.size(), f);
          std::fclose(f);
        }
      }
    }
    const auto r = lbdd::detail::finish_report(st, "asral", start);
    fill_report(r, LBDD_SOLVER_ASRAL, report, assignment, load);
  });
}
}  // extern "C"

extern "C" {
// A reference ProblemInstance (int64 CostMatrix, core.hpp:105-143) built once,
// so repeated bounded samples of the same instance do not pay the conversion.
void* lbdd_ref_instance_new(const lbdd_instance_desc* desc) {
  try {
    return new lbdd::ProblemInstance(to_instance(desc));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void lbdd_ref_instance_free(void* inst) { delete static_cast<lbdd::ProblemInstance*>(inst); }

// lbdd_ref_asral_sample on a prebuilt instance: setup = require_valid_instance
// + empty SolverState + build_arrival_queue (solver.hpp:135-141), then the
// first max_arrivals iterations of solver.hpp:143-166.
int lbdd_ref_asral_sample_inst(const void* handle, int64_t max_arrivals, int64_t* elapsed_ns,
                               int64_t* arrivals_done, int64_t* setup_ns) {
  return guarded([&] {
    const auto& inst = *static_cast<const lbdd::ProblemInstance*>(handle);
    const auto start = std::chrono::steady_clock::now();
    lbdd::require_valid_instance(inst);
    lbdd::SolverState st(inst);
    auto queue = lbdd::detail::build_arrival_queue(inst);
    *setup_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                    std::chrono::steady_clock::now() - start).count();
    int64_t done = 0;
    while (!queue.empty() && done < max_arrivals) {
      const auto [cost, d, s] = queue.top();
      queue.pop();
      st.index.insert(d, s);
      st.allotment.assign(d, s);
      lbdd::negative_cycle_refine(st, s);
      const auto& center = inst.centers[static_cast<std::size_t>(s)];
      const lbdd::Count ld = st.allotment.load[static_cast<std::size_t>(s)];
      if (ld <= center.capacity) {
        st.delta = lbdd::checked_add(st.delta, cost);
      } else {
        st.delta = lbdd::checked_add(
            st.delta, lbdd::checked_add(cost, lbdd::refund_penalty(center, ld)));
        lbdd::negative_path_refine(st, s);
      }
      ++done;
    }
    *elapsed_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - start).count();
    *arrivals_done = done;
  });
}
}  // extern "C"

namespace {
// A reference solver state resumed mid-solve: the arrival queue of
// solver.hpp:141 with its first X entries popped, and
// SolverState::from_allotment (solver.hpp:57-66, the reference's own
// constructor over a preexisting allotment) on the allotment the reference
// itself reached after those X arrivals (its checkpoint file).
struct Resumed {
  const lbdd::ProblemInstance* inst;
  lbdd::SolverState st;
  lbdd::detail::ArrivalQueue queue;
  Resumed(const lbdd::ProblemInstance& i, lbdd::SolverState&& s, lbdd::detail::ArrivalQueue&& q)
      : inst(&i), st(std::move(s)), queue(std::move(q)) {}
};
}  // namespace

extern "C" {
void* lbdd_ref_resume_new(const void* handle, const int16_t* centers, int64_t count,
                          int64_t* setup_ns) {
  try {
    const auto& inst = *static_cast<const lbdd::ProblemInstance*>(handle);
    const auto start = std::chrono::steady_clock::now();
    auto queue = lbdd::detail::build_arrival_queue(inst);
    auto allot = lbdd::Allotment::empty(inst.n(), inst.k());
    for (int64_t i = 0; i < count; ++i) {
      const auto [cost, d, s] = queue.top();
      queue.pop();
      allot.assign(d, centers[i]);
    }
    auto st = lbdd::SolverState::from_allotment(inst, allot);
    auto* r = new Resumed(inst, std::move(st), std::move(queue));
    *setup_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                    std::chrono::steady_clock::now() - start).count();
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void lbdd_ref_resume_free(void* r) { delete static_cast<Resumed*>(r); }

// The next max_arrivals iterations of solver.hpp:143-166 from the resumed
// state (the state advances: consecutive calls time consecutive arrivals).
int lbdd_ref_resume_step(void* handle, int64_t max_arrivals, int64_t* elapsed_ns,
                         int64_t* arrivals_done) {
  return guarded([&] {
    auto& r = *static_cast<Resumed*>(handle);
    auto& st = r.st;
    const auto& inst = *r.inst;
    const auto start = std::chrono::steady_clock::now();
    int64_t done = 0;
    while (!r.queue.empty() && done < max_arrivals) {
      const auto [cost, d, s] = r.queue.top();
      r.queue.pop();
      st.index.insert(d, s);
      st.allotment.assign(d, s);
      lbdd::negative_cycle_refine(st, s);
      const auto& center = inst.centers[static_cast<std::size_t>(s)];
      const lbdd::Count ld = st.allotment.load[static_cast<std::size_t>(s)];
      if (ld <= center.capacity) {
        st.delta = lbdd::checked_add(st.delta, cost);
      } else {
        st.delta = lbdd::checked_add(
            st.delta, lbdd::checked_add(cost, lbdd::refund_penalty(center, ld)));
        lbdd::negative_path_refine(st, s);
      }
      ++done;
    }
    *elapsed_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - start).count();
    *arrivals_done = done;
  });
}
}  // extern "C"
