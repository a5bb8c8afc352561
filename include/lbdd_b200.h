/*
 * lbdd_b200.h — C ABI of the B200-native ASRAL solver for Load Balanced
 * Demand Distribution.
 *
 * This is the drop-in boundary. Every entry point replaces one call of the
 * reference's header-only C++ API (/root/reference/proj/include/lbdd/ headers);
 * the reference interface each one replaces is cited beside it. Plain C types
 * only: host pointers, sizes, and status codes. No torch or CUDA types appear
 * here; device memory lives behind the opaque lbdd_b200_instance handle.
 *
 * Error behaviour mirrors the reference's exception classes: every function
 * returns an lbdd_status; the message of the last failure on the calling
 * thread is available from lbdd_b200_last_error().
 */
#ifndef LBDD_B200_H_
#define LBDD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exception classes (core.hpp throws). */
typedef enum lbdd_status {
  LBDD_OK = 0,
  LBDD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  LBDD_ERR_LOGIC = 2,            /* std::logic_error (invariant broken)   */
  LBDD_ERR_OVERFLOW = 3,         /* std::overflow_error (checked_add/mul) */
  LBDD_ERR_RUNTIME = 4,          /* std::runtime_error                    */
  LBDD_ERR_CUDA = 5              /* device failure (no reference analogue) */
} lbdd_status;

/* PenaltySpec::Family, core.hpp:43-48. */
typedef enum lbdd_penalty_family {
  LBDD_PENALTY_CONSTANT = 0,
  LBDD_PENALTY_LINEAR = 1,
  LBDD_PENALTY_TABLE = 2
} lbdd_penalty_family;

/* Solver selector, mirrors the CLI's --solver values (cli.hpp) for the
 * three ASRAL-family loops of solver.hpp. */
typedef enum lbdd_solver_kind {
  LBDD_SOLVER_ASRAL = 0,      /* asral_solve, solver.hpp:133          */
  LBDD_SOLVER_PARA_ASRAL = 1, /* asral_solve with opts.parallel       */
  LBDD_SOLVER_STRICT = 2,     /* strict_solve, solver.hpp:227         */
  LBDD_SOLVER_GREEDY = 3      /* greedy_solve, solver.hpp:172         */
} lbdd_solver_kind;

/* ProblemInstance (core.hpp:130-143) flattened into plain arrays.
 * costs: n*k row-major positive assignment costs (CostMatrix, core.hpp:105).
 * The device path computes in int32 (the benchmark configurations are int32
 * cost matrices); instances whose costs exceed INT32_MAX are rejected.
 * Penalties: center s uses penalty_params[penalty_offset[s] ..
 * penalty_offset[s+1]) interpreted per penalty_family[s]: constant {p},
 * linear {base, step}, table {values...}. */
typedef struct lbdd_instance_desc {
  int64_t n;
  int64_t k;
  const int32_t* costs;
  const int64_t* capacity;       /* k */
  const int32_t* penalty_family; /* k */
  const int64_t* penalty_offset; /* k + 1 */
  const int64_t* penalty_params; /* penalty_offset[k] */
} lbdd_instance_desc;

/* SolverOptions + ParallelConfig, solver.hpp:22-32 / parallel.hpp:21-27.
 * workers/chunking/relax_phase/index_update_phase are accepted for API
 * parity; the device engine is always data-parallel and deterministic, so
 * they do not change results (the reference guarantees the same). */
typedef struct lbdd_solver_options {
  int32_t parallel;
  int32_t check_invariants;
  int32_t refine_to_fixpoint;
  int32_t workers;
  int64_t chunking;
  int32_t relax_phase;
  int32_t index_update_phase;
  const int32_t* strict_order; /* NULL: ascending demand index */
  int64_t strict_order_len;
} lbdd_solver_options;

/* SolveReport, SolveStats, PhaseTimings: core.hpp:316-368. The assignment
 * itself is returned through a separate caller-owned int32 array. */
typedef struct lbdd_solve_report {
  int64_t objective;
  int64_t strict_surcharge;
  int32_t has_dummy_center;
  int32_t solver; /* lbdd_solver_kind */
  int64_t cycle_refine_calls;
  int64_t path_refine_calls;
  int64_t negative_cycles_removed;
  int64_t negative_paths_removed;
  int64_t refinement_gain;
  int64_t transfers_applied;
  int64_t invariant_checks;
  int64_t index_update_ns;
  int64_t bellman_ford_ns;
  int64_t total_ns;
  /* device-side breakdown (B200 engine only; zero in the reference) */
  int64_t scan_ns;      /* validation + arrival scan + sort */
  int64_t relax_rounds; /* synchronous relaxation rounds executed */
  int64_t grid_barriers; /* device-wide barriers executed by the engine */
  int64_t device_ns;     /* CUDA-event time of the whole solve on its stream */
  int64_t engine_ns;     /* CUDA-event time of the arrival-loop engine kernel launches */
  int64_t engine_launches; /* engine kernel launches in this solve */
  int64_t row_scan_ns;   /* CUDA-event time of the arrival scan kernel (row_argmin) */
} lbdd_solve_report;

/* Opaque handle: one instance resident in HBM on one device. */
typedef struct lbdd_b200_instance lbdd_b200_instance;

/* Library identity / diagnostics. */
const char* lbdd_b200_version(void);
const char* lbdd_b200_last_error(void);
int lbdd_b200_device_count(void);
/* Kernels of this library launched so far in this process (all devices). */
long long lbdd_b200_launch_count(void);
/* Engine instrumentation of the last solve in this process (out[32]):
 * out[0..2] searches started (cycle, path, potential repair), out[3..5] of
 * those with an empty initial frontier, out[6..8] frontier entries relaxed,
 * out[9] path searches pruned by the penalty bound, out[10..12] rounds per
 * kind, out[13..15] path-bound statistics; out[16..31] cluster-engine
 * lead-thread cycles per phase; out[32..37] rescans (calls, full scans,
 * row-mode, candidates, members, member-column pairs). out[40..55] / out[56..71]
 * per-CTA work / barrier-wait cycles between exchanges (LBDD_B200_PROF=1).
 * out has 72 slots. */
void lbdd_b200_engine_counters(int64_t* out);

/* Upload an instance (host arrays) to `device`. Replaces constructing a
 * lbdd::ProblemInstance (core.hpp:130) — validation as in
 * validate_instance (core.hpp:250) happens on the device at solve time,
 * exactly like require_valid_instance at the top of every solver. */
lbdd_status lbdd_b200_instance_create(const lbdd_instance_desc* desc,
                                      int device, lbdd_b200_instance** out);

/* Same, but the n*k int32 cost matrix is already resident on `device`
 * (row pitch `pitch_elems` >= k, multiple of 4). The matrix is borrowed,
 * not copied; it must outlive the handle. Centers are host arrays. */
lbdd_status lbdd_b200_instance_create_device(const lbdd_instance_desc* desc,
                                             const int32_t* d_costs,
                                             int64_t pitch_elems, int device,
                                             lbdd_b200_instance** out);

/* Synthetic generator, device-side, spec "lbdd-synth-v2" (bit-identical to
 * the host generator synth_instances.py): integer grid points from a
 * counter-based splitmix64 stream, euclidean costs
 * max(1, floor(sqrt(dx^2+dy^2)/10 + 0.5)) in [1, 1414]; total capacity
 * n*theta_num/theta_den over integer weights 1 + h % cap_spread
 * (heterogeneous); penalties from [pen_lo, pen_hi] (mixed_families != 0
 * mixes constant / linear / table, core.hpp:43-96). Not the reference's
 * mt19937_64 stream (instgen.hpp:245) — that one is a sequential CPU
 * generator; use lbdd_b200_instance_create with its output instead. */
lbdd_status lbdd_b200_instance_generate(int64_t n, int64_t k, int64_t theta_num,
                                        int64_t theta_den, int64_t pen_lo,
                                        int64_t pen_hi, int32_t mixed_families,
                                        int64_t cap_spread, uint64_t seed,
                                        int device, lbdd_b200_instance** out);

lbdd_status lbdd_b200_instance_destroy(lbdd_b200_instance* inst);
lbdd_status lbdd_b200_instance_shape(const lbdd_b200_instance* inst,
                                     int64_t* n, int64_t* k);
/* Copy the centers back to the host (capacity[k], family[k],
 * offset[k+1], params[offset[k]]); pass NULL to query sizes via *n_params. */
lbdd_status lbdd_b200_instance_centers(const lbdd_b200_instance* inst,
                                       int64_t* capacity, int32_t* family,
                                       int64_t* offset, int64_t* params,
                                       int64_t* n_params);
/* Copy rows [row0, row0+rows) of the cost matrix to the host (k per row). */
lbdd_status lbdd_b200_instance_costs(const lbdd_b200_instance* inst,
                                     int64_t row0, int64_t rows,
                                     int32_t* out);

/* asral_solve / strict_solve / greedy_solve (solver.hpp:133,227,172).
 * assignment_out: host int32[n] (demand -> center; k = overflow center
 * in strict mode with excess demand), may be NULL. load_out: host
 * int64[k+1], may be NULL. */
lbdd_status lbdd_b200_solve(lbdd_b200_instance* inst, int32_t solver,
                            const lbdd_solver_options* opts,
                            lbdd_solve_report* report, int32_t* assignment_out,
                            int64_t* load_out);

/* The first `arrivals` iterations of asral_solve's arrival loop
 * (solver.hpp:143-166): the allotment the reference's SolverState holds
 * after that many `index.insert` + refine steps (its checkpoints:
 * oracle/ref_capi.cpp lbdd_ref_asral_run). assignment_out gets -1 for
 * demands that have not arrived; report->objective is the partial
 * objective (evaluate_partial_objective, core.hpp:216-233), checked
 * against the engine's running delta. arrivals >= n is a full solve
 * without the completeness check. Pins parity at scale against the
 * reference's own mid-solve checkpoints. */
lbdd_status lbdd_b200_solve_prefix(lbdd_b200_instance* inst,
                                   const lbdd_solver_options* opts,
                                   int64_t arrivals, lbdd_solve_report* report,
                                   int32_t* assignment_out, int64_t* load_out);

/* build_index (subspace.hpp:233) for a given allotment — the full
 * segmented-argmin scan of the cost matrix. Writes the k*k minimum-transfer
 * matrix: entry [from*k+to] = (cost << 32) | demand as int64 for the
 * cheapest transfer (ties -> smaller demand, subspace.hpp:145-147), or
 * INT64_MAX when no demand sits at `from` (min_transfer, subspace.hpp:73).
 * assignment: host int32[n], kUnassigned (-1) entries skipped.
 * Rows [row0, row0+rows) only (rows < 0: all) — the per-shard partial of the
 * multi-GPU build; shards combine with an elementwise int64 MIN. */
lbdd_status lbdd_b200_build_index(lbdd_b200_instance* inst,
                                  const int32_t* assignment, int64_t row0,
                                  int64_t rows, int64_t* min_transfer_out);
/* Same, device pointers in and out (d_assignment int32[n] on the device,
 * d_out int64[k*k] on the device), launched on `stream` (cudaStream_t as
 * an opaque pointer, NULL = legacy default). Used by the sharded path,
 * where the output is a torch.distributed buffer. */
lbdd_status lbdd_b200_build_index_device(lbdd_b200_instance* inst,
                                         const int32_t* d_assignment,
                                         int64_t row0, int64_t rows,
                                         int64_t* d_out, void* stream);

/* Shard-resident variant for the multi-GPU build: `inst` holds only this
 * rank's rows (global demand ids demand_offset .. demand_offset+n-1);
 * d_assignment covers those rows; packed demand ids are global, so the
 * per-rank k*k partials combine with an elementwise int64 MIN
 * (ncclAllReduce / ncclMin over NVLink). */
lbdd_status lbdd_b200_build_index_shard(lbdd_b200_instance* inst,
                                        const int32_t* d_assignment,
                                        int64_t demand_offset, int64_t* d_out,
                                        void* stream);

/* build_arrival_queue (solver.hpp:74-96): per demand the cheapest center
 * (smallest id on ties) and the arrival order sorted by (cost, demand).
 * Host outputs, each may be NULL: best_center[n], best_cost[n],
 * order[n] (demand ids in arrival order). */
lbdd_status lbdd_b200_arrival_queue(lbdd_b200_instance* inst,
                                    int32_t* best_center, int64_t* best_cost,
                                    int32_t* order);

/* lowest_cost_path over an anchored graph given as a dense
 * (node_count-1) x node_count weight matrix (refine.hpp:28-81 with the
 * relaxation of parallel.hpp:145-210). weights[u*node_count+v] is the cost of
 * edge u->v, INT64_MAX for "no edge"; node node_count-1 is anchor-in and has
 * no out-edges; `anchor` is anchor-out. Outputs: *found (0: anchor-in
 * unreachable), *cost, dist[node_count], parent_node[node_count] (source node
 * of the parent edge, -1 if none), path[node_count] (node sequence
 * anchor-out .. anchor-in) and *path_len (edges). Returns LBDD_ERR_LOGIC on
 * a negative-cycle witness, as the reference throws. */
lbdd_status lbdd_b200_lowest_cost_path(int32_t node_count, int32_t anchor,
                                       const int64_t* weights, int32_t* found,
                                       int64_t* cost, int64_t* dist,
                                       int32_t* parent_node, int32_t* path,
                                       int32_t* path_len);

/* One synchronous relaxation round (parallel_relax_round,
 * parallel.hpp:175): dist_out/parent_out from dist_in/parent_in over the
 * same dense graph encoding; parents are source nodes. *changed set. */
lbdd_status lbdd_b200_relax_round(int32_t node_count, const int64_t* weights,
                                  const int64_t* dist_in,
                                  const int32_t* parent_in, int64_t* dist_out,
                                  int32_t* parent_out, int32_t* changed);

/* negative_cycle_refine / negative_path_refine (refine.hpp:173,199) applied
 * once to a given allotment: SolverState::from_allotment (solver.hpp:61)
 * then one refinement through `anchor`. assignment is updated in place;
 * *applied and *gain (<= 0) as RefineOutcome. dummies (int64[k], may be
 * NULL) enables strict-mode placeholder edges for the cycle graph.
 * kind: 0 = cycle, 1 = path. */
lbdd_status lbdd_b200_refine(lbdd_b200_instance* inst, int32_t kind,
                             int32_t anchor, int32_t* assignment,
                             int64_t* dummies, int32_t* applied,
                             int64_t* gain);

/* gamma_has_negative_cycle (refine.hpp:86) over the collapsed transfer
 * graph of an allotment. dummies may be NULL. */
lbdd_status lbdd_b200_gamma_has_negative_cycle(lbdd_b200_instance* inst,
                                               const int32_t* assignment,
                                               const int64_t* dummies,
                                               int32_t* has_cycle);

/* evaluate_objective / evaluate_partial_objective (core.hpp:216-243) of an
 * allotment (unassigned = -1 skipped; partial != 0 allows them). */
lbdd_status lbdd_b200_evaluate_objective(lbdd_b200_instance* inst,
                                         const int32_t* assignment,
                                         int32_t partial, int64_t* objective);

/* Timed pass of the full-matrix index scan for the benchmark: runs
 * build_index over an internal allotment (assignment = arrival centers)
 * `iters` times on the device and reports the mean kernel time from CUDA
 * events on the launching stream. */
lbdd_status lbdd_b200_bench_index_scan(lbdd_b200_instance* inst, int32_t iters,
                                       double* mean_ms, double* bytes_per_scan);

/* ---- sharded instances: demand rows over the GPUs of one box ----------
 * north_star: cost-matrix rows are sharded across the GPUs; the arrival
 * scan runs per shard and its (cost << 32 | demand) keys are gathered (the
 * caller's collective, e.g. NCCL all_gather over NVLink); the sequential
 * arrival loop is replicated on every rank and reads any demand's row
 * through a table of the ranks' row blocks, mapped into each device with
 * CUDA IPC (peer reads over NVLink). Replaces nothing in the reference (it
 * is single-process); the result is the reference's asral_solve
 * (solver.hpp:133) bit for bit, on every rank. */

/* Device memory for one row block (rows x pitch int32, pitch = k rounded
 * up to 4); fill it with lbdd_b200_shard_upload. */
lbdd_status lbdd_b200_shard_alloc(int64_t rows, int64_t k, int device,
                                  int32_t** d_shard, int64_t* pitch_elems);
lbdd_status lbdd_b200_shard_free(int32_t* d_shard, int device);
lbdd_status lbdd_b200_shard_upload(int32_t* d_shard, int64_t pitch_elems,
                                   const int32_t* host_rows, int64_t rows,
                                   int64_t k, int device);
/* CUDA IPC of a row block between the ranks' processes (64-byte handles). */
lbdd_status lbdd_b200_ipc_get_handle(const void* d_ptr, int device,
                                     uint8_t* handle64);
lbdd_status lbdd_b200_ipc_open(const uint8_t* handle64, int device,
                               void** d_ptr);
lbdd_status lbdd_b200_ipc_close(void* d_ptr, int device);

/* centers: the ProblemInstance's centers (costs NULL, n = total rows).
 * shard_ptrs[i]: row block i (rows [i*shard_rows, min((i+1)*shard_rows, n)))
 * as mapped into `device`; shard_ptrs[my_shard] is this rank's own block.
 * 1 <= nshards <= 16. The blocks are borrowed: they must outlive the
 * handle. Solve with lbdd_b200_solve_sharded (strict is not supported). */
lbdd_status lbdd_b200_instance_create_sharded(const lbdd_instance_desc* centers,
                                              const int32_t* const* shard_ptrs,
                                              int32_t nshards, int32_t my_shard,
                                              int64_t shard_rows,
                                              int64_t pitch_elems, int device,
                                              lbdd_b200_instance** out);

/* The arrival scan (row_min_center + build_arrival_queue keys,
 * solver.hpp:74-96) of this rank's block: d_keys / d_best are device arrays
 * of the block's rows (keys carry global demand ids); min/max cost of the
 * block for validate_instance (core.hpp:297-302). */
lbdd_status lbdd_b200_shard_arrival_scan(lbdd_b200_instance* inst,
                                         int64_t* d_keys, int32_t* d_best,
                                         int64_t* min_cost, int64_t* max_cost);

/* asral / para-asral / greedy on a sharded instance: d_keys_all (n keys in
 * any order) and d_best_all (n centers, by global demand id) are the
 * gathered per-shard scans, min/max the reduced block extremes. Same report
 * and assignment as lbdd_b200_solve on the whole matrix. */
lbdd_status lbdd_b200_solve_sharded(lbdd_b200_instance* inst, int32_t solver,
                                    const int64_t* d_keys_all,
                                    const int32_t* d_best_all, int64_t min_cost,
                                    int64_t max_cost,
                                    const lbdd_solver_options* opts,
                                    lbdd_solve_report* report,
                                    int32_t* assignment_out, int64_t* load_out);

#ifdef __cplusplus
}
#endif

#endif /* LBDD_B200_H_ */
