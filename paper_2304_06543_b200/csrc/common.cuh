// Shared device-side definitions for the B200 ASRAL engine.
//
// HBM layout (one instance, one device):
//   cm        int32 [n][pitch]   cost matrix, row-major by demand, pitch a
//                                multiple of 4 so every row starts 16B-aligned
//                                for 128-bit loads (CostMatrix, core.hpp:105)
//   home      int32 [n]          current center of each demand, -1 pending
//                                (Allotment::assignment / SubspaceIndex::home_)
//   load      int64 [k]          per-center load (Allotment::load)
//   M         int64 [k][k]       min-transfer matrix: M[u][v] = (key << 32) | d
//                                for the cheapest move of a demand d sitting at
//                                u to v, key = CM[d][v] - CM[d][u]; INT64_MAX
//                                when no demand sits at u. Signed int64 order
//                                of the packed word is exactly the reference
//                                heap order (key, then smaller demand,
//                                subspace.hpp:145-147), so every heap top of
//                                the k(k-1) ΓDS heaps is one word here and an
//                                elementwise MIN combines partial scans.
#pragma once

// threads per CTA of the cluster engine (cluster.cu)
#ifndef LBDD_CLUSTER_THREADS
#define LBDD_CLUSTER_THREADS 384
#endif

#include <cstdint>

#include <cuda_runtime.h>

namespace lbdd_b200 {

constexpr int64_t kEmpty = INT64_MAX;                   // no transfer / no candidate
constexpr int64_t kUnreachable = INT64_MAX / 4;         // detail::kUnreachable
constexpr int64_t kNoEdge = INT64_MAX;                  // weight sentinel
constexpr int kCandShift = 16;                          // (cand << 16) | source node
constexpr int64_t kCandLimit = (int64_t(1) << 46);      // |cand| bound for packing

__host__ __device__ inline int64_t pack_transfer(int32_t key, int32_t demand) {
  return (static_cast<int64_t>(key) * (int64_t(1) << 32)) |
         static_cast<int64_t>(static_cast<uint32_t>(demand));
}
__host__ __device__ inline int32_t transfer_key(int64_t m) {
  return static_cast<int32_t>(m >> 32);
}
__host__ __device__ inline int32_t transfer_demand(int64_t m) {
  return static_cast<int32_t>(static_cast<uint32_t>(m & 0xffffffffLL));
}
__host__ __device__ inline int64_t pack_cand(int64_t cand, int32_t u) {
  return cand * (int64_t(1) << kCandShift) + static_cast<int64_t>(u);
}
__host__ __device__ inline int64_t cand_value(int64_t p) { return p >> kCandShift; }
__host__ __device__ inline int32_t cand_source(int64_t p) {
  return static_cast<int32_t>(p & ((int64_t(1) << kCandShift) - 1));
}

// Device error codes (mapped to lbdd_status + message on the host).
enum EngineError : int32_t {
  kErrNone = 0,
  kErrNegCycleWitness = 1,   // refine.hpp:47-49
  kErrPathNotSimple = 2,     // refine.hpp:64-66
  kErrBrokenParent = 3,      // refine.hpp:69
  kErrPathSum = 4,           // refine.hpp:77-79
  kErrStaleTransfer = 5,     // subspace.hpp:88-91
  kErrPenaltyEdge = 6,       // refine.hpp:210-212
  kErrPlaceholder = 7,       // refine.hpp:149-152
  kErrNoResidual = 8,        // solver.hpp:266-268
  kErrAlreadyIndexed = 9,    // subspace.hpp:47-49
  kErrOverflow = 10,         // core.hpp:25-39
  kErrInvariant = 11,        // refine.hpp:129-131
  kErrNegativeLoad = 12,     // core.hpp:197
  kErrNotOverloaded = 13,    // subspace.hpp:344-346
};

// Engine counters, written by block 0 / thread 0 only.
struct EngineCtl {
  int64_t delta;                  // SolverState::delta (running objective)
  int64_t cycle_refine_calls;
  int64_t path_refine_calls;
  int64_t negative_cycles_removed;
  int64_t negative_paths_removed;
  int64_t refinement_gain;
  int64_t transfers_applied;
  int64_t invariant_checks;
  int64_t relax_rounds;
  int64_t t_bf_ns;                // bellman_ford bucket (globaltimer)
  int64_t t_index_ns;             // index_update bucket (globaltimer)
  int64_t barriers;               // grid barriers executed
  int64_t dbg[16];                // engine instrumentation (see capi)
  int64_t prof[16];               // cluster engine: lead-thread cycles per phase
  int64_t resc[8];                // cluster engine rescans: calls, full-scan, row-mode,
                                  // candidates, members, (member, column) pairs
  int64_t cta_wait[16];           // cluster engine (profile): cycles each CTA waited in exchanges
  int64_t cta_work[16];           // cluster engine (profile): cycles between exchanges per CTA
  int32_t error;
  int32_t error_arg;
  int32_t prev_sources;           // transfer sources of the last applied path
  int32_t search_count;           // relaxation searches started
};

// Software grid barrier (the kernel is launched cooperatively, so all CTAs
// are co-resident). The last CTA to arrive snapshots the values the next
// phase branches on — error flag, a "changed" flag, one int64 — before
// releasing the others, so every CTA takes identical decisions even though
// fast CTAs start overwriting the sources in the next phase.
struct GridBar {
  unsigned long long arrive;   // [0,32) arrivals, [32,48) CTAs that saw a
                               // change, [48,64) CTAs that recorded an error
  unsigned long long release;  // (generation << 32) | payload bits
};

// One edge of an extracted path (node ids of the anchored graph).
struct PathEdge {
  int32_t from_center;
  int32_t to_center;
  int32_t demand;   // -1 unless transfer
  int32_t kind;     // 1 transfer, 2 dummy, 3 penalty
};

enum GraphKind : int32_t { kCycleGraph = 0, kPathGraph = 1, kGammaGraph = 2 };
enum EdgeKind : int32_t { kEdgeNone = 0, kEdgeTransfer = 1, kEdgeDummy = 2, kEdgePenalty = 3 };

// Where the cost row of demand d lives. One shard: the whole matrix. Several
// (sharded instance, lbdd_b200_instance_create_sharded): demand rows split
// in equal blocks of shard_rows over the ranks of one box, shard[i] the
// device pointer of block i as mapped into THIS device's address space (its
// own block, or a peer's opened through CUDA IPC, read over NVLink).
constexpr int kMaxShards = 16;
struct RowTable {
  const int32_t* shard[kMaxShards];
  int64_t pitch;
  int32_t shard_rows;  // rows per shard block (all but possibly the last)
  int32_t nshards;     // <= 1: shard[0] holds every row
};
__host__ __device__ inline const int32_t* row_of(const RowTable& T, int64_t d) {
  if (T.nshards <= 1) return T.shard[0] + d * T.pitch;
  const uint32_t s = static_cast<uint32_t>(d) / static_cast<uint32_t>(T.shard_rows);
  return T.shard[s] + (d - static_cast<int64_t>(s) * T.shard_rows) * T.pitch;
}

struct EngineArgs {
  // instance (read-only)
  RowTable rows;         // every demand's cost row (row_of)
  const int32_t* cm;     // rows.shard[0]
  int64_t pitch;
  int32_t n;
  int32_t k;
  const int64_t* cap;
  const int32_t* pfam;
  const int64_t* poff;
  const int64_t* ppar;
  // allotment + index
  int32_t* home;
  int64_t* load;
  int64_t* M;
  int64_t* dummies;      // strict mode only, else nullptr
  // arrivals
  const int64_t* arr_keys;    // asral: sorted (cost << 32 | d)
  const int32_t* best_center; // asral: row argmin center
  const int32_t* arr_s;       // asral: best_center of the a-th arrival (gathered once per solve)
  const int32_t* order;       // strict: processing order (nullptr = identity)
  int64_t a_begin;
  int64_t a_end;
  int32_t mode;          // 0 asral, 1 strict
  int32_t fixpoint;
  int32_t check_invariants;
  int32_t single_kind;   // >= 0: run one refine of this kind at `single_anchor`
  int32_t single_anchor;
  int32_t pad0;
  // relaxation scratch: two buffer sets, alternating between searches
  int64_t* D[2][2];
  int32_t* P[2][2];
  int64_t* B[2][3];
  int64_t* colW;         // k: weights into anchor-in
  int32_t search_base;   // searches run by earlier launches (set parity)
  int32_t pad2;
  int64_t delta_step;    // cluster engine Δ-stepping width (cost units, <= 0: off)
  int64_t delta_path;    // Δ of the penalty-path searches (cost units, <= 0: off)
  int32_t profile;       // lead-thread phase cycle counters (LBDD_B200_PROF=1)
  // bucket index (demands grouped by home, built before each launch) and
  // the move log appended since; nullptr: rescans scan every demand
  const int32_t* bk_off;  // k + 1
  const int32_t* bk_ids;  // n
  int32_t* log_d;
  int32_t* log_to;
  int32_t* log_n;
  int32_t log_cap;
  int32_t add_cap;        // per-center capacity of the add lists
  int32_t* add_ids;       // [k][add_cap]: demands that moved to center u this launch
  int32_t* add_cnt;       // [k]: appends per center (past add_cap: use the move log)
  int64_t* MX;            // 3 planes of k*k: 2nd..4th smallest transfer per entry
  uint8_t* LN;            // k*k: list length | complete << 3
  int32_t debug_checks;   // validate engine invariants after each phase
  int32_t pad4;
  // path + transfer scratch
  PathEdge* path;        // k + 1
  int32_t* inv_cnt;      // k + 1
  int32_t* inv_cols;     // (k + 1) * k
  int32_t* rowslot;      // k, -1 when not a transfer source of the current path
  int32_t* src_list;     // k + 1 sources of the last applied path
  int32_t* rowver;       // k: bumped whenever row u of M changes
  int32_t tile_mode;     // 1: each CTA caches its relaxation tile of M keys in smem;
                         // 2: the same int16 tile, k x k, in global memory (L2)
  int16_t* ktile;        // tile_mode 2: int16 key of M[u][v] at ktile[u * k + v]
  int32_t pad1;
  EngineCtl* ctl;
  GridBar* bar;
  int32_t* single_out;   // single refine: [applied, has_path], gain in ctl
  int64_t* single_gain;
};

}  // namespace lbdd_b200
