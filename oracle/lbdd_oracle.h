/*
 * lbdd_oracle.h — TEST INFRASTRUCTURE ONLY (parity checker, CPU baseline).
 *
 * Plain-C restatement of the reference ASRAL algorithm
 * (/root/reference/proj/include/lbdd/{core,subspace,refine,parallel,solver,
 * instgen}.hpp). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the checker. The
 * product (paper_2304_06543_b200) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_pinning.py checks every entry point
 * against the unmodified reference compiled into oracle/_ref (see
 * oracle/Makefile) and against the reference tests' known answers
 * (tests/golden/).
 */
#ifndef LBDD_ORACLE_H_
#define LBDD_ORACLE_H_

#include <stdint.h>

#include "lbdd_b200.h" /* shared plain structs: lbdd_instance_desc, ... */

#ifdef __cplusplus
extern "C" {
#endif

const char* lbdd_oracle_last_error(void);

int lbdd_oracle_solve(const lbdd_instance_desc* desc, int32_t solver,
                      const lbdd_solver_options* opts,
                      lbdd_solve_report* report, int32_t* assignment,
                      int64_t* load);
int lbdd_oracle_build_index(const lbdd_instance_desc* desc,
                            const int32_t* assignment, int64_t* out);
int lbdd_oracle_refine(const lbdd_instance_desc* desc, int32_t kind,
                       int32_t anchor, int32_t* assignment, int64_t* dummies,
                       int32_t* applied, int64_t* gain);
int lbdd_oracle_gamma_has_negative_cycle(const lbdd_instance_desc* desc,
                                         const int32_t* assignment,
                                         const int64_t* dummies,
                                         int32_t* has_cycle);
int lbdd_oracle_lowest_cost_path(int32_t node_count, int32_t anchor,
                                 const int64_t* weights, int32_t* found,
                                 int64_t* cost, int64_t* dist,
                                 int32_t* parent_node, int32_t* path,
                                 int32_t* path_len);
int lbdd_oracle_relax_round(int32_t node_count, const int64_t* weights,
                            const int64_t* dist_in, const int32_t* parent_in,
                            int64_t* dist_out, int32_t* parent_out,
                            int32_t* changed);
int lbdd_oracle_evaluate_objective(const lbdd_instance_desc* desc,
                                   const int32_t* assignment, int32_t partial,
                                   int64_t* objective);
int lbdd_oracle_arrival_queue(const lbdd_instance_desc* desc,
                              int32_t* best_center, int64_t* best_cost,
                              int32_t* order);
/* instgen.hpp:245 euclidean branch, byte-identical stream (mt19937_64). */
int64_t lbdd_oracle_derive_center_count(int64_t n, double ratio);
int lbdd_oracle_generate(uint64_t seed, int64_t n, double ratio, double theta,
                         int64_t pen_lo, int64_t pen_hi, int64_t* k_out,
                         int64_t* capacity, int64_t* penalty, int32_t* costs);
/* Solve only the first `max_arrivals` arrivals of asral (bounded CPU
 * baseline sample); returns elapsed ns of the sampled loop. */
int lbdd_oracle_asral_sample(const lbdd_instance_desc* desc,
                             int64_t max_arrivals, int32_t workers,
                             int64_t* elapsed_ns, int64_t* arrivals_done,
                             int64_t* setup_ns);

#ifdef __cplusplus
}
#endif

#endif /* LBDD_ORACLE_H_ */
