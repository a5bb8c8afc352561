// The cluster engine: the whole ASRAL / strict arrival loop on ONE thread-
// block cluster (up to 16 CTAs on one GPC), synchronised with the hardware
// cluster barrier and exchanging data through distributed shared memory.
//
// Exactness argument (DESIGN.md §3 has the long form):
//  * The reference keeps the transfer graph Γ free of negative cycles
//    (Lemmas 1-2; refine.hpp:125-131 checks it). So a feasible potential π
//    exists: rc(u,v) = w(u,v) + π(u) - π(v) >= 0 on every Γ edge. We keep one,
//    per center, in the owning CTA's shared memory.
//  * After inserting demand d at anchor a only row a of Γ changed. In the
//    anchored cycle graph every edge except those out of anchor-out has
//    rc >= 0, so every prefix of a path with negative total cost is itself
//    negative: searching only nodes reached with negative reduced distance
//    finds every negative anchored path, with exact labels for every node on
//    it (and for all their tight predecessors).
//  * The reference's synchronous Bellman-Ford (parallel.hpp:145-169) leaves
//    each node v with parent = the smallest u such that
//    d*(u) + w(u,v) = d*(v) and h*(u) = h*(v) - 1, where h* is the fewest
//    edges among shortest paths (the round in which d*(v) is first reached).
//    Lexicographic labels (d, h, parent) computed by ANY label-correcting
//    order are unique, so a frontier search with packed
//    (d << 26 | h << 13 | parent) labels returns the reference's path bit
//    for bit.
//  * π is repaired after every change of Γ: D(v) = min(0, min_{x in X}
//    dist_rc(x, v)) over the rows X that may now violate it (the anchor after
//    an insert, the receiving centers of an applied path) is again a bounded
//    negative-region search, and π + D is feasible.
//  * The path search (overload) adds penalty edges u -> anchor-in whose
//    reduced cost can be negative; nodes are explored while
//    d_rc(v) < -min_u rc_pen(u), which bounds every candidate.
//
// Node ownership: node v (0..k, k = anchor-in) belongs to CTA v / s, s =
// ceil((k+1)/CS); the owner holds its label, its π and its "changed" flag,
// and relaxes every edge INTO its nodes (row partials folded by the owner,
// no shared-memory atomics on labels); edges INTO anchor-in are evaluated
// by the owners of their sources. Sources of the next round travel as
// (node, label + π, placeholder flag) entries pushed into every CTA's inbox
// (st.async + round mbarriers during searches, DSMEM stores + cluster
// barrier around the phases that order global memory).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lbdd_b200 {
namespace cl {

constexpr int64_t kLabInf = INT64_MAX;
constexpr int kMaxCS = 16;
constexpr int kStage = 256;            // frontier entries staged per pass
constexpr int16_t kNoKey16 = INT16_MAX;  // "no demand at the source" in the tile
constexpr int kMaxSeg = 32;            // source rows rescanned per apply via the index
constexpr int kRowSlots = 8;           // source rows of a row-mode rescan (column bitmaps)
// Row-mode rescans (member rows streamed over the owner's columns in 16 B
// pieces) measured slower than gathering the invalidated columns at every
// threshold once the add lists made candidate sets small (200K x 1000:
// 10.88 s with row mode at >= 4 columns per 16 pieces, 10.52 s without;
// k = 2000 6.60 -> 6.39 s; k = 5000 unchanged); kept compiled out.
constexpr bool kRowMode = false;
constexpr int kMaxMine = 1024;
constexpr int kPathCache = 64;         // path edges mirrored in shared memory (the rest: global only)
// frontier entries one CTA pushes per exchange (inbox slots per source):
// changed nodes past it stay pending for a later round -- the Δ-stepping
// hold-back mechanism -- so shared memory no longer grows with k
constexpr int kInCap = 128;
// past s = 128 (k > ~2000) the cap drops to 96 so that the engine's shared
// memory stays under the 100 KB carve-out step (k = 5000: 98.5 KB) and the
// SM keeps its larger L1 for the global key tile (measured 11% at k = 5000)
__host__ __device__ inline int inbox_cap(int s) { return s <= kInCap ? s : 96; }         // invalidated (segment, column) pairs a CTA owns per rescan

// A frontier entry as pushed into every CTA's inbox: the node (bit 31: a
// surplus placeholder sits there, strict-mode edge rule) and its label with
// π(node) folded in, lp = label + π(node) << 16, so that a candidate into v
// is lp + (w - π(v)) << 16 + 1.
struct FEntry {
  int32_t nd;
  int32_t pad;
  int64_t lp;
};
__device__ __forceinline__ int fe_node(const FEntry& e) { return e.nd & 0x7fffffff; }
__device__ __forceinline__ bool fe_dum(const FEntry& e) { return (e.nd >> 31) != 0; }

struct Pub {          // per-CTA published scalars of one exchange
  int32_t count;      // changed entries in list[par]
  int32_t err;        // error recorded by this CTA
  int64_t sinklab;    // label of anchor-in (owner only)
  int64_t val;        // reduction slot (min over the CTA)
  int32_t aux;        // reduction argument
  int32_t pending;    // improved nodes held back by the Δ threshold
  int64_t pmin;       // smallest held-back label
  int64_t omin;       // smallest open label (held back or pushed this round)
};


static_assert(sizeof(Pub) == 48, "Pub travels as three 16 B st.async");
static_assert(sizeof(FEntry) == 16, "FEntry travels as one 16 B st.async");


// A pair of equal-sized buffers selected by parity: base + i * stride, so
// that CS has no dynamically indexed member array (which would force the
// whole struct into local memory).
template <typename T>
struct Pair2 {
  T* p;
  int stride;
  __device__ __forceinline__ T* operator[](int i) const { return p + i * stride; }
};

struct CS {           // shared-memory layout of one CTA
  int64_t* lab;       // [s]
  int64_t* pis;       // [s]
  Pair2<FEntry> inbox;  // [kMaxCS * cin] each: entries pushed by CTA r at r * cin
  Pair2<Pub> pub;      // [1] each
  PathEdge* path;     // [k + 1] (global, one slice per CTA)
  PathEdge* pc;       // [kPathCache] shared-memory copy of the first path edges (path_at)
  uint8_t* chg;       // [s]
  int32_t* qd;        // [blockDim] rescan queue
  int32_t* qs;        // [blockDim]
  int32_t* qh;        // [blockDim] CM[d][home] of each queued member
  uint32_t* bits;     // [kRowSlots * ceil(k / 32)] invalidated columns per rescan slot
  int32_t* misc;      // [16]: 0 queue count, 1 local count, 2 local err
  int64_t* red;       // [16] reduction scratch
  Pub* all;           // every CTA's pub of the last exchange (= allb[par])
  Pair2<Pub> allb;     // [kMaxCS] each: pubs PUSHED by every CTA, by parity

  int64_t* sinkc;     // [s] per owned node u: π(u) + w(u, anchor-in) - π(anchor-in) of
                      //   the running search (kLabInf: no edge); the OWNER of u
                      //   evaluates u's edge into anchor-in when it pushes u
  int64_t* part;      // [max(blockDim, s)] relax partials: row ty of column col at ty * ns + col
  int64_t* wred;      // [4 * 32] per-warp reductions of collect (pmin, omin, sink, -)
  uint32_t* rin;      // [2 * kMaxCS] inbox[par] of CTA r in the cluster window (mapa, once)
  uint32_t* rbar;     // [2 * kMaxCS] rmb[par] of CTA r in the cluster window
  int32_t* seg;       // [3 * kMaxSeg] rescan segments (slot, prefix end, bucket count)
  int32_t* mine;      // [kMaxMine] my invalidated columns of a rescan ((g << 16) | j, then j by segment)
  int32_t* mine2;     // [kMaxMine] scratch of the counting sort
  int32_t* segmine;   // [kMaxSeg + 1] my columns per segment, then their offsets
  int32_t* segcur;    // [kMaxSeg] counting-sort cursors
  int64_t* dbg;       // [16] instrumentation counters
  int64_t* cred;      // [2][4] collect's reductions by parity: pmin, omin, sink candidate
  int64_t* pkey;      // [4] asral prefetch ring (arrival a at a & 3): sorted key (cost << 32 | d)
  int32_t* ps;        // [4] ... and its center
  int32_t* prow;      // [2][s + 1] cost row of arrival a (at a & 1): my columns, then CM[d][s] at [s]
  int64_t* lc;        // [16] rank 0: the lead's running EngineCtl fields (kLc*), flushed at exit
  int64_t* prof;      // [16] lead-thread cycle counters per phase
  int64_t* cw;        // [4] per-CTA profile: last exchange, work cycles, wait cycles
  uint64_t* rmb;      // [2] round mbarriers (by parity): csz arrivals + st.async bytes
  int16_t* wt;        // [k * s] transfer keys of every row into my columns
                      // (tile mode: all keys fit in int16)
};

// The applied path: global slice S.path (any length), its first kPathCache
// edges mirrored in shared memory so that apply / T1 / T3 read them without
// an L2 round trip.
__device__ __forceinline__ PathEdge path_at(const CS& S, int i) { return i < kPathCache ? S.pc[i] : S.path[i]; }
__device__ __forceinline__ void path_set(const CS& S, int i, const PathEdge& e) {
  S.path[i] = e;
  if (i < kPathCache) S.pc[i] = e;
}
// host mirror: cluster_smem_bytes() in capi.cu
__device__ __forceinline__ CS carve(unsigned char* p, int k, int s, bool tile) {
  CS S;
  S.lab = reinterpret_cast<int64_t*>(p); p += 8 * s;
  S.pis = reinterpret_cast<int64_t*>(p); p += 8 * s;
  const int cin = inbox_cap(s);
  S.inbox = {reinterpret_cast<FEntry*>(p), kMaxCS * cin}; p += 2 * sizeof(FEntry) * kMaxCS * cin;
  S.pub = {reinterpret_cast<Pub*>(p), 1}; p += 2 * sizeof(Pub);
  S.red = reinterpret_cast<int64_t*>(p); p += 8 * 16;
  S.allb = {reinterpret_cast<Pub*>(p), kMaxCS}; p += 2 * sizeof(Pub) * kMaxCS;
  S.all = S.allb[0];

  S.sinkc = reinterpret_cast<int64_t*>(p); p += 8 * s;
  S.part = reinterpret_cast<int64_t*>(p); p += 8 * static_cast<size_t>(max(static_cast<int>(blockDim.x), s));
  S.wred = reinterpret_cast<int64_t*>(p); p += 8 * 4 * 32;
  S.rin = reinterpret_cast<uint32_t*>(p); p += 4 * 2 * kMaxCS;
  S.pc = reinterpret_cast<PathEdge*>(p); p += sizeof(PathEdge) * kPathCache;
  S.rbar = reinterpret_cast<uint32_t*>(p); p += 4 * 2 * kMaxCS;
  S.seg = reinterpret_cast<int32_t*>(p); p += 4 * 3 * kMaxSeg;
  S.mine = reinterpret_cast<int32_t*>(p); p += 4 * kMaxMine;
  S.mine2 = reinterpret_cast<int32_t*>(p); p += 4 * kMaxMine;
  S.segmine = reinterpret_cast<int32_t*>(p); p += 4 * (kMaxSeg + 2);  // even: keeps 8 B alignment
  S.segcur = reinterpret_cast<int32_t*>(p); p += 4 * kMaxSeg;
  S.dbg = reinterpret_cast<int64_t*>(p); p += 8 * 16;
  S.lc = reinterpret_cast<int64_t*>(p); p += 8 * 16;
  S.cred = reinterpret_cast<int64_t*>(p); p += 8 * 8;
  S.pkey = reinterpret_cast<int64_t*>(p); p += 8 * 4;
  S.ps = reinterpret_cast<int32_t*>(p); p += 4 * 4;
  S.prow = reinterpret_cast<int32_t*>(p); p += 4 * 2 * static_cast<size_t>(s + 1);
  p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
  S.prof = reinterpret_cast<int64_t*>(p); p += 8 * 16;
  S.cw = reinterpret_cast<int64_t*>(p); p += 8 * 4;
  S.rmb = reinterpret_cast<uint64_t*>(p); p += 8 * 2;
  S.path = nullptr;   // global, one slice per CTA (EngineArgs::path), see the prologue
  S.qd = reinterpret_cast<int32_t*>(p); p += 4 * blockDim.x;
  S.qs = reinterpret_cast<int32_t*>(p); p += 4 * blockDim.x;
  S.qh = reinterpret_cast<int32_t*>(p); p += 4 * blockDim.x;
  S.bits = reinterpret_cast<uint32_t*>(p); p += 4 * static_cast<size_t>(kRowSlots) * ((k + 31) / 32);
  S.misc = reinterpret_cast<int32_t*>(p); p += 4 * 16;
  S.wt = reinterpret_cast<int16_t*>(p); p += tile ? 2 * static_cast<size_t>(k) * s : 0;
  S.chg = reinterpret_cast<uint8_t*>(p);
  return S;
}

// lead-thread phase profiler: prof[i] += cycles since the last mark (only
// with LBDD_B200_PROF=1: the marks sit on rank 0's critical path, which
// every other CTA waits for at the next cluster barrier)
#define PROF_MARK(X, i)                                      \
  do {                                                       \
    if ((X).lead && (X).A.profile) {                         \
      const long long now__ = clock64();                     \
      (X).S.prof[i] += now__ - (X).S.prof[15];               \
      (X).S.prof[15] = now__;                                \
    }                                                        \
  } while (0)

__device__ __forceinline__ int64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<int64_t>(t);
}
__device__ __forceinline__ bool add_ovf(int64_t a, int64_t b, int64_t* r) {
  const int64_t x = static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
  *r = x;
  return ((a ^ x) & (b ^ x)) < 0;
}
__device__ __forceinline__ bool mul_ovf(int64_t a, int64_t b, int64_t* r) {
  const __int128 p = static_cast<__int128>(a) * static_cast<__int128>(b);
  *r = static_cast<int64_t>(p);
  return p != static_cast<__int128>(*r);
}
__device__ __forceinline__ int64_t pair_weight(int64_t m, bool dummy) {
  if (dummy) {
    if (m == kEmpty) return 0;
    const int32_t key = transfer_key(m);
    return key < 0 ? key : 0;
  }
  return m == kEmpty ? kNoEdge : static_cast<int64_t>(transfer_key(m));
}
__device__ __forceinline__ int32_t pair_kind(int64_t m, bool dummy) {
  if (dummy && (m == kEmpty || transfer_key(m) >= 0)) return kEdgeDummy;
  return m == kEmpty ? kEdgeNone : kEdgeTransfer;
}
// Search labels pack (d, h, parent): d (reduced distance) << 26 | h (hops)
// << 13 | parent node. Signed 64-bit order is lexicographic (d, h, parent),
// so one atomicMin per candidate keeps, among the shortest candidates with
// the fewest hops, the smallest parent -- the synchronous Bellman-Ford
// parent rule of parallel.hpp:145-169. Nodes < 8192.
constexpr int kHopShift = 13;
constexpr int kLabShift = 26;
constexpr int64_t kHop = int64_t(1) << kHopShift;
constexpr int64_t kLUnit = int64_t(1) << kLabShift;
constexpr int64_t kParMask = kHop - 1;
constexpr int64_t kPiLimit = int64_t(1) << 35;  // |π| bound: lp = label + π << 26 fits int64
__device__ __forceinline__ int64_t lab_d(int64_t lab) { return lab >> kLabShift; }
__device__ __forceinline__ int32_t lab_parent(int64_t lab) { return static_cast<int32_t>(lab & kParMask); }
__device__ __forceinline__ int16_t key16(int64_t m) {
  return m == kEmpty ? kNoKey16 : static_cast<int16_t>(transfer_key(m));
}
__device__ __forceinline__ int64_t key16_weight(int16_t key, bool dummy) {
  if (dummy) return key != kNoKey16 && key < 0 ? key : 0;
  return key == kNoKey16 ? kNoEdge : static_cast<int64_t>(key);
}
__device__ __forceinline__ int32_t lab_h(int64_t lab) {
  return static_cast<int32_t>((lab >> kHopShift) & kParMask);
}

enum SearchKind : int32_t { kCycle = 0, kPath = 1, kRepair = 2 };

// The lead's running counters live in rank 0's shared memory (S.lc) during a
// launch: a global read-modify-write is a ~0.5 us round trip on the lead's
// critical path, and every CTA waits for the lead at the next exchange.
enum LeadCtl : int {
  kLcDelta = 0, kLcCycleCalls, kLcPathCalls, kLcCycles, kLcPaths, kLcGain, kLcTransfers,
  kLcChecks, kLcTbf, kLcTindex, kLcPrevSources, kLcLogN, kLcCount
};

struct Ctx {
  const EngineArgs& A;  // the __grid_constant__ kernel parameter (constant bank, no local copy)
  CS S;
  cg::cluster_group cluster;
  int rank, csz, k, s, v0, v1;
  int cin;            // inbox slots per source CTA (inbox_cap(s))
  int par;
  unsigned rph;       // phase bits of the round mbarriers S.rmb[0], S.rmb[1]
  int err;            // sticky, identical in all CTAs (read at exchanges)
  bool lead;          // rank 0, thread 0
  bool tile;          // int16 transfer keys of my columns in a tile (X.wt)
  int16_t* wt;        // tile of my columns: key of (u, v0 + col) at wt[u * wst + col];
  int wst;            //   shared memory (stride s) or, when that does not fit, global (stride k)
  // per-launch counters kept in registers (lead thread), flushed at exit so
  // no global read-modify-write sits on a round's critical path
  int64_t n_barriers;
  int64_t n_rounds;
  int64_t T;          // Δ-stepping threshold of the running search (packed)
  int64_t delta;      // Δ in packed units (of the running search)
  int64_t delta_main, delta_path;
  // sink-bound pruning of the running search: a node whose distance d
  // satisfies d + prune_c > d(sink) can improve neither the sink through
  // its own edge (rc into anchor-in >= prune_c) nor any descendant (rc >= 0
  // elsewhere), so it is dropped from the frontier. Off for repairs (their
  // labels repair π and must be exact everywhere).
  bool prune;
  int64_t prune_c;    // cycle: 0; path: C (cost units)
  int64_t cur_slab;   // sink label of the running search after the last exchange
  int64_t* dbg;       // [16] shared-memory counters (lead thread)
  int cpp, rpp, tx, ty;  // relax thread layout (fixed per CTA)
  int cpar;           // parity of collect's slot counter (S.misc[8 + cpar])
  // the last exchange, reduced by EVERY warp for itself (no CTA barrier, no
  // shared copy): lane r < csz holds the inclusive prefix of the entry
  // counts of CTAs 0..r (lanes >= csz: the total), so relax maps a flat
  // entry index to (source CTA, slot) with one ballot
  int xincl;
  int xtotal, xpend;
  int64_t xpmin, xomin, xslab;
  __device__ Ctx(const EngineArgs& a, const cg::cluster_group& c) : A(a), cluster(c) {}
};

__device__ __forceinline__ void set_err(Ctx& X, int code, int arg) {
  if (atomicCAS(&X.A.ctl->error, 0, code) == 0) X.A.ctl->error_arg = arg;
  X.S.misc[2] = 1;
}

// PenaltySpec::at / marginal / refund (core.hpp:60-74, 196-208)
__device__ __forceinline__ int64_t pen_at(Ctx& X, int s, int64_t j) {
  const EngineArgs& A = X.A;
  const int64_t* p = A.ppar + A.poff[s];
  switch (A.pfam[s]) {
    case 0: return p[0];
    case 1: {
      int64_t m, r;
      if (mul_ovf(p[1], j - 1, &m) || add_ovf(p[0], m, &r)) { set_err(X, kErrOverflow, s); return 0; }
      return r;
    }
    default: {
      const int64_t len = A.poff[s + 1] - A.poff[s];
      return p[(j < len ? j : len) - 1];
    }
  }
}
__device__ __forceinline__ int64_t marginal_penalty(Ctx& X, int s, int64_t load) {
  if (load < 0) { set_err(X, kErrNegativeLoad, s); return 0; }
  return load < X.A.cap[s] ? 0 : pen_at(X, s, load - X.A.cap[s] + 1);
}
__device__ __forceinline__ int64_t refund_penalty(Ctx& X, int s, int64_t load) {
  if (load < 0) { set_err(X, kErrNegativeLoad, s); return 0; }
  return load <= X.A.cap[s] ? 0 : pen_at(X, s, load - X.A.cap[s]);
}

// ---- per-entry top-4 lists: the 4 smallest (key, demand) of a heap ----
// Entry (u, j) keeps its minimum in M[u*k+j] (what every reader uses) and
// up to three successors in MX (three k*k planes, slot i at i*k*k + u*k+j:
// a warp's 32 consecutive lists load as three coalesced 256 B rows, not a
// 768 B strided span per slot); LN[u*k+j] = length | complete
// << 3, where "complete" means the list holds every demand sitting at u.
// Invariant: the list is exactly the `length` smallest transfers of the
// heap (subspace.hpp:26-231), so removing the head promotes the true next
// minimum; a rescan is needed only when an incomplete list runs empty.
#ifndef LBDD_TOPK
#define LBDD_TOPK 4
#endif
constexpr int kTopK = LBDD_TOPK;  // list depth (M head + kTopK - 1 MX planes); LN holds len in 3 bits
static_assert(kTopK >= 2 && kTopK <= 7, "list length must fit LN's 3 bits");
struct TopK {
  int64_t e[kTopK];
  int len;
  bool complete;
};
__device__ __forceinline__ int64_t* mx_slot(const EngineArgs& A, int64_t idx, int i) {
  return A.MX + static_cast<int64_t>(i) * A.k * A.k + idx;
}
__device__ __forceinline__ TopK list_load(const EngineArgs& A, int64_t idx) {
  TopK t;
  t.e[0] = A.M[idx];
#pragma unroll
  for (int i = 1; i < kTopK; ++i) t.e[i] = *mx_slot(A, idx, i - 1);
  const uint8_t ln = A.LN[idx];
  t.len = ln & 7;
  t.complete = (ln & 8) != 0;
  return t;
}
__device__ __forceinline__ void list_store(const EngineArgs& A, int64_t idx, const TopK& t) {
  A.M[idx] = t.e[0];
#pragma unroll
  for (int i = 1; i < kTopK; ++i) *mx_slot(A, idx, i - 1) = t.e[i];
  A.LN[idx] = static_cast<uint8_t>(t.len | (t.complete ? 8 : 0));
}
// returns true when the head changed. Fixed indices only (compare-and-swap
// insertion; slots past `len` hold kEmpty), so a TopK stays in registers
// instead of a dynamically indexed local-memory array.
__device__ __forceinline__ bool list_insert(TopK& t, int64_t v) {
  if (!t.complete && t.len == 0) return false;  // unknown minimum: a rescan follows
  int64_t last = t.e[0];
#pragma unroll
  for (int i = 1; i < kTopK; ++i)
    if (i < t.len) last = t.e[i];
  if (!t.complete && v > last) return false;
  if (t.complete && t.len == kTopK) {
    t.complete = false;  // one more member than the list holds
    if (v > t.e[kTopK - 1]) return false;
  }
  const bool head = v < t.e[0];
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    const int64_t lo = min(t.e[i], v);
    v = max(t.e[i], v);
    t.e[i] = lo;
  }
  if (t.len < kTopK) ++t.len;
  return head;
}
// Concurrent rescan insert into an emptied list (all of M, MX start at
// kEmpty): atomicMin at slot 0, the larger value carries on to the next
// slot, an equal value (the same demand found twice: bucket and move log)
// stops. Slots only decrease, so a value dropped past slot 3 is never among
// the four smallest; the prefilter reads slot 3 at L2 (a stale larger value
// only costs the cascade).
__device__ __forceinline__ void list_sink(const EngineArgs& A, int64_t idx, int64_t x) {
  if (x >= static_cast<int64_t>(__ldcg(reinterpret_cast<const long long*>(mx_slot(A, idx, kTopK - 2))))) return;
  int64_t old = atomicMin(reinterpret_cast<long long*>(&A.M[idx]), static_cast<long long>(x));
  if (old == x) return;
  x = max(old, x);
  for (int i = 0; i < kTopK - 1 && x != kEmpty; ++i) {
    old = atomicMin(reinterpret_cast<long long*>(mx_slot(A, idx, i)), static_cast<long long>(x));
    if (old == x) return;
    x = max(old, x);
  }
}
// returns 0 when the demand is not listed, else 4 | (1 when the head
// changed) | (2 when a rescan is needed)
__device__ __forceinline__ int list_remove(TopK& t, int32_t demand) {
  int p = -1;
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    if (i < t.len && t.e[i] != kEmpty && transfer_demand(t.e[i]) == demand) p = i;
  }
  if (p < 0) return 0;
#pragma unroll
  for (int i = 0; i + 1 < kTopK; ++i) {
    if (i >= p) t.e[i] = t.e[i + 1];
  }
  t.e[kTopK - 1] = kEmpty;
  --t.len;
  int r = p == 0 ? 5 : 4;
  if (t.len == 0 && !t.complete) r |= 2;
  return r;
}

__device__ int g_dbg_printed = 0;
__device__ long long g_dbg_arrival = 0;
// Debug validation (A.debug_checks): every list element's demand sits at
// the row's center, keys match the cost matrix, lists are sorted, and the
// head mirrors into the tile. Error 300 + where on the first violation.
__device__ void validate_lists(Ctx& X, int where) {
  const EngineArgs& A = X.A;
  if (!A.debug_checks) return;
  const int k = X.k;
  for (int64_t p = threadIdx.x; p < static_cast<int64_t>(k) * (X.v1 - X.v0); p += blockDim.x) {
    const int u = static_cast<int>(p / (X.v1 - X.v0));
    const int j = X.v0 + static_cast<int>(p % (X.v1 - X.v0));
    if (j >= k || j == u) continue;
    const TopK t = list_load(A, static_cast<int64_t>(u) * k + j);
    for (int i = 0; i < t.len; ++i) {
      const int64_t e = t.e[i];
      const int32_t d = transfer_demand(e);
      int why = 0;
      if (e == kEmpty) why = 1;
      else if (A.home[d] != u) why = 2;
      else if (transfer_key(e) != row_of(A.rows, d)[ j] -
                                      row_of(A.rows, d)[ u]) why = 3;
      else if (i > 0 && t.e[i - 1] >= e) why = 4;
      // debug encoding (small instances): demand | u | j | slot | reason | len | complete
      if (why) set_err(X, 300 + where, (d & 255) | ((u & 15) << 8) | ((j & 15) << 12) | (i << 16) |
                                         (why << 20) | (t.len << 24) | (int(t.complete) << 28));
    }
    if (t.len == 0 && t.e[0] != kEmpty) set_err(X, 300 + where, -1);
    bool bad = t.len == 0 && t.e[0] != kEmpty;
    for (int i = 0; i < t.len; ++i) {
      const int64_t e = t.e[i];
      if (e == kEmpty || A.home[transfer_demand(e)] != u) bad = true;
    }
    if (bad && atomicCAS(&g_dbg_printed, 0, 1) == 0) {
      printf("lbdd_b200 list violation arrival %lld where %d u %d j %d len %d complete %d\n",
             g_dbg_arrival, where, u, j, t.len, int(t.complete));
      for (int i = 0; i < kTopK; ++i) {
        const int64_t e = t.e[i];
        printf("  e[%d] key %lld demand %d home %d\n", i, e == kEmpty ? -1LL : (long long)transfer_key(e),
               e == kEmpty ? -1 : transfer_demand(e), e == kEmpty ? -2 : A.home[transfer_demand(e)]);
      }
      for (int i = 0; i < k + 1 && i < 12; ++i) {
        const PathEdge pe = path_at(X.S, i);
        printf("  path[%d] %d -> %d kind %d demand %d inv_cnt %d\n", i, pe.from_center, pe.to_center,
               pe.kind, pe.demand, A.inv_cnt[i]);
      }
    }
    if (X.tile && X.wt[static_cast<int64_t>(u) * X.wst + (j - X.v0)] != key16(t.e[0]))
      set_err(X, 320 + where, u);
  }
  __syncthreads();
}

// Append a home change to the move log: position `i` (the caller's count
// S.lc[kLcLogN] + its offset), the demand onto `to`'s add list. Fire-and-
// forget stores except the add-list counter (one atomic round trip).
__device__ __forceinline__ void log_move(const EngineArgs& A, int64_t i, int32_t d, int32_t to) {
  if (A.log_n == nullptr) return;
  if (i < A.log_cap) {
    A.log_d[i] = d;
    A.log_to[i] = to;
  }
  if (A.add_cnt != nullptr) {  // the per-center add list of `to`
    const int32_t c = atomicAdd(&A.add_cnt[to], 1);  // past add_cap: rescans of `to` use the move log
    if (c < A.add_cap) A.add_ids[static_cast<int64_t>(to) * A.add_cap + c] = d;
  }
}
__device__ __forceinline__ void red_add64(int64_t* p, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// ---- asral arrival prefetch (cp.async: no thread waits on the loads) ----
// The arrival order is fixed, so arrival a + 2's (key, center) and arrival
// a + 1's cost row (this CTA's columns + CM[d][s]) are copied into shared
// memory while arrival a runs: the insert then starts from shared memory
// instead of a key -> center -> cost-row chain of dependent global loads.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ bool has_dummy(const Ctx& X, int u) {
  return X.A.dummies != nullptr && X.A.dummies[u] > 0;
}

// ---- st.async round exchange (search rounds) ----
// A search round moves only shared-memory data between CTAs (frontier
// entries and the published scalars), so it does not need the cluster
// barrier's release/acquire of global memory (a GPU-scope MEMBAR plus an L1
// invalidate per barrier). Each CTA writes into every CTA's inbox[par] /
// allb[par] with st.async, whose bytes complete_tx on the destination's
// round mbarrier rmb[par]; after its last store to a destination it arrives
// there (relaxed, remote) declaring the bytes it sent. A CTA's round is over
// when all csz CTAs arrived and all declared bytes landed. 676 vs 1607
// cycles per exchange in isolation (scripts/latency_floor.py).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa_u32(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async16(unsigned raddr, const void* src, unsigned rbar) {
  const int4 v = *reinterpret_cast<const int4*>(src);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(raddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar) : "memory");
}
__device__ __forceinline__ void remote_arrive_tx(unsigned rbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;"
               ::"r"(rbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W%=;\n}" ::"r"(bar), "r"(phase) : "memory");
}

// Cluster barrier + exchange: every CTA publishes pub[par] (count, err,
// sink label, reduction slot) — and pushes inbox[par] — before calling;
// afterwards S.all[] holds the values of every CTA, identical everywhere,
// and par flips, so inbox[par ^ 1] holds the sources of the next relaxation.
__device__ __forceinline__ void exchange_finish(Ctx& X);
__device__ __forceinline__ void exchange(Ctx& X) {
  CS& S = X.S;
  if (threadIdx.x < 32) {
    // warp 0 pushes this CTA's pub (written by thread 0) into slot `rank`
    // of every CTA's allb[par] before the barrier, so that afterwards every
    // read is local. A CTA can push for the next exchange only after this
    // barrier, and by then every CTA has read allb[par ^ 1] for the last
    // time (it did so before arriving here).
    if (threadIdx.x == 0) S.pub[X.par]->err = S.misc[2];
    __syncwarp();
    if (threadIdx.x < X.csz) {
      Pub* dst = X.cluster.map_shared_rank(S.allb[X.par], static_cast<int>(threadIdx.x));
      dst[X.rank] = *S.pub[X.par];
    }
  }
  long long tw0 = 0;
  if (X.A.profile && threadIdx.x == 0) {
    tw0 = clock64();
    S.cw[1] += tw0 - S.cw[0];  // work since the last exchange (this CTA)
  }
  X.cluster.sync();
  if (X.A.profile && threadIdx.x == 0) {
    const long long t1 = clock64();
    S.cw[2] += t1 - tw0;       // waited at the barrier (this CTA)
    S.cw[0] = t1;
  }
  exchange_finish(X);
}

// The round variant: entries were pushed by collect(async) with st.async;
// warp 0 sends the pub and arrives at every CTA, then all threads wait.
__device__ __forceinline__ void exchange_async(Ctx& X) {
  CS& S = X.S;
  const unsigned bar = smem_u32(&S.rmb[X.par]);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) S.pub[X.par]->err = S.misc[2];
    __syncwarp();
    if (threadIdx.x < X.csz) {
      const int r = static_cast<int>(threadIdx.x);
      const Pub* mine = S.pub[X.par];
      const unsigned rbar = mapa_u32(bar, r);
      const unsigned dst = mapa_u32(smem_u32(&S.allb[X.par][X.rank]), r);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        st_async16(dst + 16 * q, reinterpret_cast<const char*>(mine) + 16 * q, rbar);
      }
      // collect wrote this CTA's own copy of its entries with plain stores
      remote_arrive_tx(rbar, static_cast<unsigned>(sizeof(Pub) +
                                                   (r == X.rank ? 0 : sizeof(FEntry) * mine->count)));
    }
  }
  long long tw0 = 0;
  if (X.A.profile && threadIdx.x == 0) {
    tw0 = clock64();
    S.cw[1] += tw0 - S.cw[0];
  }
  mbar_wait(bar, (X.rph >> X.par) & 1u);
  X.rph ^= 1u << X.par;
  if (X.A.profile && threadIdx.x == 0) {
    const long long t1 = clock64();
    S.cw[2] += t1 - tw0;
    S.cw[0] = t1;
  }
  exchange_finish(X);
}

__device__ __forceinline__ void exchange_finish(Ctx& X) {
  CS& S = X.S;
  S.all = S.allb[X.par];
  // every warp reduces the CTAs' pubs itself (identical results
  // everywhere); both half-warps hold all csz <= 16 pubs, so four shuffle
  // levels leave every lane with the result
  static_assert(kMaxCS == 16, "half-warp reductions");
  const int lane = threadIdx.x & 31, hl = lane & 15;
  int c = 0, e = 0, pend = 0;
  long long pmin = kLabInf, omin = kLabInf, slab = kLabInf;
  if (hl < X.csz) {
    const Pub& p = S.all[hl];
    c = (p.count >= 0 && p.count <= X.cin) ? p.count : 0;
    e = p.err;
    pend = p.pending;
    pmin = p.pmin;
    omin = p.omin;
    slab = p.sinklab;
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (hl >= o) incl += y;
  }
  X.xincl = incl;  // lanes < csz (entry_slot); lane 15: the total
  X.xtotal = __shfl_sync(0xffffffffu, incl, 15);
  if (__any_sync(0xffffffffu, e != 0)) X.err = 1;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    pend += __shfl_xor_sync(0xffffffffu, pend, o);
    omin = min(omin, __shfl_xor_sync(0xffffffffu, omin, o));
    slab = min(slab, __shfl_xor_sync(0xffffffffu, slab, o));
  }
  if (pend != 0) {  // warp-uniform; held-back minimum only when something is held
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) pmin = min(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
  } else {
    pmin = kLabInf;
  }
  X.xpend = pend;
  X.xpmin = pmin;
  X.xomin = omin;
  X.xslab = slab;
  if (X.lead) X.n_barriers += 1;
  // the next phase writes the other buffer while slow CTAs may still read
  // this one; it is rewritten only after the next barrier
  X.par ^= 1;
}

// Flat index t (warp-uniform) of the entries of the last exchange ->
// inbox slot: segment = CTAs whose inclusive prefix is <= t.
__device__ __forceinline__ int entry_slot(const Ctx& X, int t) {
  const int lane = threadIdx.x & 31;
  const unsigned below = __ballot_sync(0xffffffffu, lane < X.csz && X.xincl <= t);
  const int seg = __popc(below);
  const int excl = __shfl_sync(0xffffffffu, X.xincl, (seg + 31) & 31);
  return seg * X.cin + t - (seg == 0 ? 0 : excl);
}

__device__ __forceinline__ int total_pending(const Ctx& X) { return X.xpend; }
// next threshold: at least Δ above the smallest held-back label
__device__ __forceinline__ void advance_threshold(Ctx& X) {
  if (total_pending(X) == 0) return;
  const int64_t m = X.xpmin;
  const int64_t t = m > kLabInf - X.delta ? kLabInf : m + X.delta;
  if (t > X.T) X.T = t;
}

__device__ __forceinline__ int total_count(const Ctx& X) { return X.xtotal; }

// Push this CTA's changed nodes (and clear the flags) into every CTA's
// inbox[par] (slot range rank * s): DSMEM stores, ordered before the
// readers by the release of the next cluster barrier.
__device__ __forceinline__ void push_entry(Ctx& X, int pos, int v, int64_t label, int64_t pi,
                                           bool dum) {
  FEntry e;
  e.nd = v | (dum ? static_cast<int32_t>(0x80000000u) : 0);
  e.pad = 0;
  e.lp = ((label & ~kParMask) | v) + pi * kLUnit;  // a candidate's parent field = v
  const int slot = X.rank * X.cin + pos;
  for (int r = 0; r < X.csz; ++r) {
    FEntry* box = X.cluster.map_shared_rank(X.S.inbox[X.par], r);
    box[slot] = e;
  }
}

// CTA-wide min into a shared slot from the lanes with `has` (whole warp calls)
__device__ __forceinline__ void cta_min(bool has, long long v, int64_t* slot) {
  const unsigned bal = __ballot_sync(0xffffffffu, has);
  if (bal == 0) return;
  if (__popc(bal) <= 2) {
    if (has) atomicMin(reinterpret_cast<long long*>(slot), v);
    return;
  }
  if (!has) v = kLabInf;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMin(reinterpret_cast<long long*>(slot), v);
}

// Δ-stepping: only improved nodes with label <= X.T are pushed; the rest
// stay pending (their flag kept) and report their count and minimum.
// merge: fold the relax partials of this round into the labels first (the
// owner is the single writer of its labels: no shared-memory atomics).
// Each pushed node's edge into anchor-in is evaluated here by its owner
// (S.sinkc), so no CTA relaxes an anchor-in column; the CTA minimum of those
// candidates is published as Pub::sinklab (running over the search).
// async: the entries go out with st.async (the round exchange), one
// (entry, destination) pair per thread; else with generic DSMEM stores.
__device__ __forceinline__ void collect(Ctx& X, int kind, int anchor, bool async = false,
                                        bool merge = false) {
  CS& S = X.S;
  // slots taken: S.misc[8 + cpar], zero here (reset by the previous call,
  // whose own counter every thread read before the CTA barrier that
  // separates the two calls); the other parity is reset for the next call
  int* slots = &S.misc[8 + X.cpar];
  int* heldc = &S.misc[12 + X.cpar];
  int64_t* cr = S.cred + 4 * X.cpar;
  if (threadIdx.x == 0) {  // the other parity, for the next call
    S.misc[8 + (X.cpar ^ 1)] = 0;
    S.misc[12 + (X.cpar ^ 1)] = 0;
    int64_t* cn = S.cred + 4 * (X.cpar ^ 1);
    cn[0] = cn[1] = cn[2] = kLabInf;
  }
  X.cpar ^= 1;
  const int ns = X.v1 - X.v0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warps holding owned nodes (all of them when ns > blockDim)
  const int nwa = min(static_cast<int>(blockDim.x + 31) >> 5, (ns + 31) >> 5);
  long long pmin = kLabInf, omin = kLabInf, smin = kLabInf;
  int held = 0;
  if (warp < nwa)
  for (int i0 = 0; i0 < ns; i0 += blockDim.x) {  // warp-uniform trip count
    const int i = i0 + threadIdx.x;
    bool push = false;
    int64_t label = kLabInf;
    const int v = X.v0 + i;
    if (i < ns) {
      label = S.lab[i];
      bool chg = S.chg[i] != 0;
      if (merge && v < X.k) {
        int64_t best = kLabInf;
        for (int r = 0; r < X.rpp; ++r) best = min(best, S.part[r * ns + i]);
        if (best < label) {
          if ((best & ~kParMask) < (label & ~kParMask)) chg = true;
          label = best;
          S.lab[i] = best;
        }
      }
      if (chg) {
        if (v == X.k) {
          chg = false;  // anchor-in has no out-edges
        } else if (X.prune && X.cur_slab != kLabInf && lab_d(label) + X.prune_c > lab_d(X.cur_slab)) {
          chg = false;  // cannot lead to a better sink label
        } else if (label > X.T) {
          ++held;
          pmin = min(pmin, static_cast<long long>(label));
        } else {
          push = true;
        }
      }
      S.chg[i] = chg;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, push);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(slots, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (push) {
      const int pos = base + __popc(bal & ((1u << lane) - 1));
      if (pos >= X.cin) {  // inbox slots exhausted this round: held back (pending)
        ++held;
        pmin = min(pmin, static_cast<long long>(label));
      } else {
        S.chg[i] = 0;
        omin = min(omin, static_cast<long long>(label));
        const bool dum = kind != kPath && has_dummy(X, v);
        FEntry e;
        e.nd = v | (dum ? static_cast<int32_t>(0x80000000u) : 0);
        e.pad = 0;
        e.lp = ((label & ~kParMask) | v) + S.pis[i] * kLUnit;
        if (async) S.inbox[X.par][X.rank * X.cin + pos] = e;
        else push_entry(X, pos, v, label, S.pis[i], dum);
        if (kind != kRepair) {
          const int64_t sc = S.sinkc[i];
          if (sc != kLabInf) {
            const int64_t cand = ((label & ~kParMask) | v) + sc * kLUnit + kHop;
            if (cand < 0) smin = min(smin, static_cast<long long>(cand));  // bound_sink = 0
          }
        }
        if (lab_h(label) > X.k + 1) set_err(X, kErrNegCycleWitness, v);
      }
    }
  }
  // shared-memory atomics for the CTA minima (a 64-bit min is a CAS loop:
  // cheap while few lanes contend); a warp with more than two values
  // reduces them with shuffles first (k = 5000: ~10 warps hold nodes)
  if (nwa <= 2) {  // k <= ~2000: few values per warp, plain atomics
    if (held) {
      atomicAdd(heldc, held);
      atomicMin(reinterpret_cast<long long*>(&cr[0]), pmin);
    }
    if (omin != kLabInf) atomicMin(reinterpret_cast<long long*>(&cr[1]), omin);
    if (smin != kLabInf) atomicMin(reinterpret_cast<long long*>(&cr[2]), smin);
  } else if (warp < nwa) {
    cta_min(held != 0, pmin, &cr[0]);
    cta_min(omin != kLabInf, omin, &cr[1]);
    cta_min(smin != kLabInf, smin, &cr[2]);
    if (__any_sync(0xffffffffu, held != 0)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) held += __shfl_xor_sync(0xffffffffu, held, o);
      if (lane == 0) atomicAdd(heldc, held);
    }
  }
  __syncthreads();
  const int cnt = min(*slots, X.cin);
  if (async && cnt > 0) {
    // (entry, destination) pairs over the CTA: thread -> destination
    // threadIdx % 16, entries threadIdx / 16 + j * blockDim / 16; this CTA's
    // own copy is local
    const int r = threadIdx.x & (kMaxCS - 1);
    if (r < X.csz && r != X.rank) {
      const unsigned rin = S.rin[X.par * kMaxCS + r] + static_cast<unsigned>(sizeof(FEntry)) * (X.rank * X.cin);
      const unsigned rbar = S.rbar[X.par * kMaxCS + r];
      const FEntry* mine = &S.inbox[X.par][X.rank * X.cin];
      for (int e = threadIdx.x / kMaxCS; e < cnt; e += blockDim.x / kMaxCS) {
        const int4 v = *reinterpret_cast<const int4*>(&mine[e]);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                     ::"r"(rin + static_cast<unsigned>(sizeof(FEntry)) * e), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w), "r"(rbar) : "memory");
      }
    }
  }
  if (threadIdx.x == 0) {
    const int64_t pm = cr[0], om = cr[1], sm = cr[2];
    Pub* p = S.pub[X.par];
    p->count = cnt;
    p->pending = *heldc;
    p->pmin = pm;
    p->omin = min(pm, om);
    if (sm < S.red[4]) S.red[4] = sm;
    p->sinklab = S.red[4];
  }
}

// The asral tile loop of relax: U independent (entry, key) pairs per step;
// lim shrinks to min(lp + key * unit) over the valid entries.
template <int U>
__device__ __forceinline__ int64_t relax_tile(const Ctx& X, const FEntry* box, int cnt, const int16_t* wcol,
                                              int sw, int v, int64_t lim) {
  const int rpp = X.rpp;
  int t = X.ty;
  for (; t + (U - 1) * rpp < cnt; t += U * rpp) {
    int sl[U];
#pragma unroll
    for (int q = 0; q < U; ++q) sl[q] = entry_slot(X, t + q * rpp);
    int nd[U];
#pragma unroll
    for (int q = 0; q < U; ++q) nd[q] = box[sl[q]].nd;
    int16_t kq[U];
#pragma unroll
    for (int q = 0; q < U; ++q) kq[q] = wcol[nd[q] * sw];
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (kq[q] != kNoKey16 && nd[q] != v) lim = min(lim, box[sl[q]].lp + static_cast<int64_t>(kq[q]) * kLUnit);
  }
  for (; t < cnt; t += rpp) {
    const FEntry e = box[entry_slot(X, t)];
    const int16_t key = wcol[e.nd * sw];
    if (key != kNoKey16 && e.nd != v) lim = min(lim, e.lp + static_cast<int64_t>(key) * kLUnit);
  }
  return lim;
}

// Relax every edge from the sources pushed in the last exchange into this
// CTA's nodes. bound_mid: strict upper bound on labels. Each thread owns
// one destination column per pass and keeps its running minimum in a
// register; the row partials go to S.part and collect folds them into the
// labels (no 64-bit shared-memory atomics, which are CAS loops). Sources are
// read from the local inbox (broadcast within a warp). Edges into anchor-in
// are evaluated by the owners of their sources in collect.
__device__ __forceinline__ void relax(Ctx& X, int kind, int anchor, int64_t refund_a,
                                      int64_t bound_mid, int64_t bound_sink) {
  CS& S = X.S;
  const EngineArgs& A = X.A;
  const int ns = X.v1 - X.v0;
  if (ns <= 0) return;  // uniform within the CTA
  const int cpp = X.cpp, rpp = X.rpp, tx = X.tx, ty = X.ty;
  constexpr int64_t kUnit = kLUnit;
  if (ty >= rpp) return;  // threads past the last full row of columns (whole warps)
  // the entries of the last exchange, read in place (no compaction): flat
  // index t -> slot by entry_slot (warp-uniform t: every lane of a warp has
  // the same ty, cpp being a multiple of 32)
  const FEntry* box = S.inbox[X.par ^ 1];
  const int cnt = X.xtotal;
  for (int c0 = 0; c0 < ns; c0 += cpp) {
    const int col = c0 + tx;
    const int v = X.v0 + col;
    const bool valid = col < ns && v < X.k && !(kind != kRepair && v == anchor);
    const int64_t base = valid ? kHop - S.pis[col] * kUnit : 0;  // candidate = lp + w*unit + base
    const int64_t bound = bound_mid;
    int64_t best = kLabInf;
    if (X.tile && X.A.dummies == nullptr) {
      // asral: no placeholder flags. cand < min(bound, best) is tested as
      // lp + w * unit < lim with lim = min(bound, best) - base, shrinking
      const int16_t* wcol = X.wt + (valid ? col : 0);
      const int64_t lim0 = bound - base;
      int64_t lim = lim0;
      const int sw = X.wst;  // nd * wst < 2^31: 32-bit index math
      // independent (entry, key) load pairs in flight per step: four, or
      // eight when one thread walks the whole frontier (one row of columns,
      // k > ~2300) through the global (L2) tile (eight measured slower at
      // k = 2000, three rows)
      lim = (rpp == 1 && A.tile_mode == 2) ? relax_tile<8>(X, box, cnt, wcol, sw, v, lim)
                                           : relax_tile<4>(X, box, cnt, wcol, sw, v, lim);
      if (lim < lim0) best = lim + base;
    } else if (X.tile) {
#pragma unroll 4
      for (int t = ty; t < cnt; t += rpp) {
        const FEntry e = box[entry_slot(X, t)];
        const int u = fe_node(e);
        const int64_t w = valid ? key16_weight(X.wt[static_cast<int64_t>(u) * X.wst + col], fe_dum(e))
                                : kNoEdge;
        if (u == v || w == kNoEdge) continue;
        const int64_t cand = e.lp + w * kUnit + base;
        if (cand < bound && cand < best) best = cand;
      }
    } else {
      // keys from global memory, 4 independent loads in flight
      for (int t = ty; t < cnt; t += 4 * rpp) {
        int64_t m[4];
        FEntry e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tq = t + q * rpp;
          e[q].nd = -1;
          m[q] = kEmpty;
          if (tq < cnt) {  // warp-uniform
            e[q] = box[entry_slot(X, tq)];
            if (valid) m[q] = A.M[static_cast<int64_t>(fe_node(e[q])) * A.k + v];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (e[q].nd == -1 || fe_node(e[q]) == v) continue;
          const int64_t w = pair_weight(m[q], fe_dum(e[q]));
          if (w == kNoEdge) continue;
          const int64_t cand = e[q].lp + w * kUnit + base;
          if (cand < bound && cand < best) best = cand;
        }
      }
    }
    if (col < ns) S.part[ty * ns + col] = valid ? best : kLabInf;
  }
}

// Edges into anchor-in for the running search, per owned node u (its owner
// evaluates them when it pushes u, see collect): cycle graph w(u, anchor)
// (cheapest_pair_edge), path graph the penalty difference marginal(u) -
// refund(anchor), folded with the potentials: sinkc = π(u) + w - π(anchor-in).
// π of owned nodes is fixed during a search.
__device__ __forceinline__ void fill_sink_weights(Ctx& X, int kind, int anchor, int64_t refund_a,
                                                  int64_t pi_sink) {
  const EngineArgs& A = X.A;
  for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
    const int u = X.v0 + i;
    int64_t w = kNoEdge;
    if (u != anchor && u < X.k) {
      w = kind == kCycle ? pair_weight(A.M[static_cast<int64_t>(u) * A.k + anchor], has_dummy(X, u))
                         : marginal_penalty(X, u, A.load[u]) - refund_a;
    }
    X.S.sinkc[i] = w == kNoEdge ? kLabInf : X.S.pis[i] + w - pi_sink;
  }
}

// Run rounds until no label changes. Sources must already be published in
// list[par] (count in pub[par]) and exchanged. Returns rounds executed.
// Exact early stop: with non-negative reduced costs every label below the
// smallest open label is final, and an open node v can lower anchor-in to
// no less than lab(v) + sink_inc. Once anchor-in holds S and
// min_open + sink_inc > S, nothing can change it or any node on its chain.
__device__ __forceinline__ bool sink_settled(const Ctx& X, int64_t sink_inc) {
  if (sink_inc == kLabInf) return false;
  const int64_t sl = X.xslab, om = X.xomin;
  // a candidate into the sink from an open node x has (d, h) part >=
  // (d, h)(x) + sink_inc; the parent field of an equal (d, h) could still
  // lower the sink, so settle only on a strictly larger (d, h)
  return sl != kLabInf && (om == kLabInf || (om & ~kParMask) + sink_inc > (sl & ~kParMask));
}

__device__ __forceinline__ int search_rounds(Ctx& X, int kind, int anchor, int64_t refund_a, int64_t bound_mid,
                             int64_t bound_sink, int64_t sink_inc = kLabInf) {
  int rounds = 0;
  if (X.lead) {
    X.dbg[kind] += 1;                                 // searches started per kind
    if (total_count(X) == 0) X.dbg[3 + kind] += 1;    // empty at start
  }
  advance_threshold(X);
  while ((total_count(X) > 0 || total_pending(X) > 0) && !X.err && !sink_settled(X, sink_inc)) {
    if (X.lead) X.dbg[6 + kind] += total_count(X);   // frontier entries
    PROF_MARK(X, 9);
    relax(X, kind, anchor, refund_a, bound_mid, bound_sink);
    __syncthreads();
    PROF_MARK(X, 1);
    collect(X, kind, anchor, true, true);
    PROF_MARK(X, 2);
    exchange_async(X);
    X.cur_slab = X.xslab;
    advance_threshold(X);
    PROF_MARK(X, 3);
    ++rounds;
  }
  if (X.lead) X.dbg[10 + kind] += rounds;
  return rounds;
}

__device__ __forceinline__ int64_t sink_label(const Ctx& X) {
  return X.xslab;
}

// Start a search: labels of owned nodes to +inf, π(anchor-in) := π(anchor).
__device__ __forceinline__ void reset_labels(Ctx& X, int64_t pi_anchor) {
  X.T = X.delta;  // labels start at the source's 0
  X.cur_slab = kLabInf;
  if (threadIdx.x == 0) X.S.red[4] = kLabInf;  // running anchor-in candidate of this CTA
  for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
    X.S.lab[i] = kLabInf;
    X.S.chg[i] = 0;
    if (X.v0 + i == X.k) X.S.pis[i] = pi_anchor;
  }
}

// Read π(v) of any node (DSMEM).
__device__ __forceinline__ int64_t pi_of(Ctx& X, int v) {
  const int r = v / X.s;
  const int64_t* rp = X.cluster.map_shared_rank(X.S.pis, r);
  return rp[v - r * X.s];
}

// Push the sources (label 0) owned by this CTA into every inbox[par].
__device__ __forceinline__ void publish_sources(Ctx& X, const int* nodes, int count, int kind) {
  if (threadIdx.x == 0) {
    int c = 0, held = 0;
    for (int i = 0; i < count; ++i) {
      const int v = nodes[i];
      if (v < X.v0 || v >= X.v1) continue;
      bool dup = false;
      for (int j = 0; j < i; ++j) dup |= nodes[j] == v;
      if (dup) continue;
      X.S.lab[v - X.v0] = 0;
      if (c < X.cin) {
        push_entry(X, c++, v, 0, X.S.pis[v - X.v0], kind != kPath && has_dummy(X, v));
      } else {  // no inbox slot left: a pending source, pushed by a later round
        X.S.chg[v - X.v0] = 1;
        ++held;
      }
    }
    X.S.pub[X.par]->count = c;
    X.S.pub[X.par]->pending = held;
    X.S.pub[X.par]->pmin = held ? 0 : kLabInf;
    X.S.pub[X.par]->omin = (c > 0 || held > 0) ? 0 : kLabInf;
    X.S.pub[X.par]->sinklab = kLabInf;
  }
}

// π(v) += min(0, d(v)) for owned nodes explored by the last search. Ends
// with a cluster barrier: other CTAs read π through DSMEM (pi_of) next.
__device__ __forceinline__ void apply_repair(Ctx& X) {
  for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
    if (X.v0 + i == X.k) continue;
    const int64_t l = X.S.lab[i];
    if (l == kLabInf) continue;
    const int64_t d = lab_d(l);
    if (d < 0) {
      X.S.pis[i] += d;
      if (X.S.pis[i] < -kPiLimit) set_err(X, kErrOverflow, X.v0 + i);
    }
  }
  X.cluster.sync();
}

// Parent walk (refine.hpp:53-80). The parent rule of the synchronous BF is
// already in the labels (their parent field, see lab_parent), so every CTA
// walks the chain from anchor-in back to anchor-out itself, reading the
// labels of the path nodes from their owners through DSMEM, then reads the
// transfer word of each edge. One exchange at the end: past it, T1 of
// faster CTAs rewrites the lists the words were read from. Fills S.path in
// path order and returns its length (0 + error on a broken chain).
__device__ __forceinline__ int reconstruct(Ctx& X, int kind, int anchor, int64_t refund_a, int64_t sinklab) {
  CS& S = X.S;
  const EngineArgs& A = X.A;
  if (threadIdx.x == 0) {
    int v = X.k;
    int64_t lv = sinklab;
    int len = 0;
    int bad = 0;
    while (v != anchor) {
      if (len > X.k) { bad = kErrPathNotSimple; break; }
      const int u = lab_parent(lv);
      if (u >= X.k || u == v || lv == kLabInf) { bad = kErrBrokenParent; break; }
      PathEdge e;
      e.from_center = u;
      e.to_center = v == X.k ? anchor : v;
      e.demand = -1;
      e.kind = kEdgeNone;
      path_set(S, len++, e);  // reversed order for now
      if (u != anchor) {
        const int r = u / X.s;
        lv = X.cluster.map_shared_rank(S.lab, r)[u - r * X.s];
      }
      v = u;
    }
    S.misc[6] = bad ? -bad : len;
  }
  __syncthreads();
  const int len = S.misc[6];
  if (len <= 0) {
    if (X.lead) set_err(X, -len, 0);
    X.err = 1;
    return 0;
  }
  // edge kinds and transfer words (the first recorded edge enters anchor-in),
  // each edge written straight to its place in path order (read all, CTA
  // barrier, write all: the reversal is in place)
  const int per = (len + blockDim.x - 1) / blockDim.x;  // edges per thread (1 unless len > blockDim)
  if (per == 1) {
    PathEdge e;
    const int i = threadIdx.x;
    if (i < len) {
      e = path_at(S, i);
      if (kind == kPath && i == 0) {
        e.kind = kEdgePenalty;
      } else {
        const int64_t m = A.M[static_cast<int64_t>(e.from_center) * A.k + e.to_center];
        const bool dum = kind == kCycle && A.dummies != nullptr && A.dummies[e.from_center] > 0;
        e.kind = pair_kind(m, dum);
        if (e.kind == kEdgeTransfer) e.demand = transfer_demand(m);
      }
    }
    __syncthreads();
    if (i < len) path_set(S, len - 1 - i, e);
    if (threadIdx.x == 0) S.pub[X.par]->count = 0;
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      PathEdge e = path_at(S, i);
      if (kind == kPath && i == 0) {
        e.kind = kEdgePenalty;
      } else {
        const int64_t m = A.M[static_cast<int64_t>(e.from_center) * A.k + e.to_center];
        const bool dum = kind == kCycle && A.dummies != nullptr && A.dummies[e.from_center] > 0;
        e.kind = pair_kind(m, dum);
        if (e.kind == kEdgeTransfer) e.demand = transfer_demand(m);
      }
      path_set(S, i, e);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // reverse into path order
      for (int i = 0; i < len / 2; ++i) {
        const PathEdge t = path_at(S, i);
        path_set(S, i, path_at(S, len - 1 - i));
        path_set(S, len - 1 - i, t);
      }
      S.pub[X.par]->count = 0;
    }
  }
  exchange(X);
  return X.err ? 0 : len;
}

// Apply the path (apply_path_edges, refine.hpp:134-164). Column owners
// invalidate and fold gains for their columns; the lead updates the
// allotment; all CTAs rescan the invalidated entries over the final
// buckets. Fills `dirty` with the rows whose out-edges may now violate π.
__device__ __forceinline__ int apply(Ctx& X, int kind, int len, int64_t cost, int* dirty, int anchor) {
  CS& S = X.S;
  const EngineArgs& A = X.A;
  const int k = X.k;
  const int64_t t0 = gtimer();
  // ---- T1: remove the moved demands from their old rows' lists, insert
  // them into their new rows' lists. The path is simple and contiguous
  // (edge i runs from_center(i) -> from_center(i + 1); a cycle returns to
  // from_center(0)), so row from_center(p) loses demand(p) and gains the
  // demand of the transfer edge that enters it: tasks (row p, column j)
  // are independent and run in one pass, each list loaded once, the
  // removal before the gain (as the reference's per-edge order leaves it).
  const int jlo = X.v0, jhi = min(X.v1, k);
  const int ncol = max(0, jhi - jlo);
  const PathEdge last = path_at(S, len - 1);
  const bool extra = last.kind == kEdgeTransfer && last.to_center != path_at(S, 0).from_center;
  const int ntask = len + (extra ? 1 : 0);
  for (int q = threadIdx.x; q < ntask * ncol; q += blockDim.x) {
    const int p = q / ncol;
    const int j = jlo + (q - p * ncol);
    int row, rm = -1, in = -1;  // row; removal edge; gain edge
    if (p < len) {
      const PathEdge e = path_at(S, p);
      row = e.from_center;
      if (e.kind == kEdgeTransfer) rm = p;
      const int pi = p > 0 ? p - 1 : len - 1;
      const PathEdge f = path_at(S, pi);
      if (f.kind == kEdgeTransfer && f.to_center == row && (p > 0 || len > 1 || pi != p)) in = pi;
    } else {
      row = last.to_center;
      in = len - 1;
    }
    if (j == row || (rm < 0 && in < 0)) continue;
    const int64_t idx = static_cast<int64_t>(row) * k + j;
    int32_t din = -1, vin = 0;
    if (in >= 0) {
      din = path_at(S, in).demand;
      const int32_t* rowin = row_of(A.rows, din);
      vin = rowin[j] - rowin[row];
    }
    TopK t = list_load(A, idx);
    bool changed = false, head = false;
    if (rm >= 0) {
      const int r = list_remove(t, path_at(S, rm).demand);
      if (r != 0) {
        changed = true;
        head = (r & 1) != 0;
        if (r & 2) {
          const int pos = atomicAdd(&A.inv_cnt[rm], 1);
          A.inv_cols[static_cast<int64_t>(rm) * k + pos] = j;
        }
      }
    }
    if (in >= 0) {
      changed = true;  // list_insert may clear `complete`
      if (list_insert(t, pack_transfer(vin, din))) head = true;
    }
    if (changed) list_store(A, idx, t);
    if (X.tile && head) X.wt[static_cast<int64_t>(row) * X.wst + (j - X.v0)] = key16(t.e[0]);
  }
  int nd = 0;
  for (int i = 0; i < len; ++i) {
    const PathEdge e = path_at(S, i);
    if (e.kind == kEdgeTransfer || e.kind == kEdgeDummy) dirty[nd++] = e.to_center;
  }
  if (kind == kCycle) dirty[nd++] = anchor;  // the inserted row was never repaired
  // allotment bookkeeping (apply_path_edges, refine.hpp:134-164): warp 0
  // of rank 0, one lane per path edge, so the global accesses of all edges
  // overlap (a simple path moves distinct demands between distinct centers;
  // load[] changes are commutative atomics; the log keeps path order)
  if (X.rank == 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int64_t* lc = S.lc;
    const int nprev = static_cast<int>(lc[kLcPrevSources]);
    for (int q = lane; q < nprev; q += 32) A.rowslot[A.src_list[q]] = -1;
    __syncwarp();
    int ns = 0;
    const int64_t log0 = lc[kLcLogN];
    for (int i0 = 0; i0 < len; i0 += 32) {
      const int i = i0 + lane;
      PathEdge e;
      e.kind = kEdgeNone;
      if (i < len) e = path_at(S, i);
      const bool tr = e.kind == kEdgeTransfer;
      const unsigned bt = __ballot_sync(0xffffffffu, tr);
      if (tr) {
        const int32_t h = A.home[e.demand];
        const int pos = ns + __popc(bt & ((1u << lane) - 1));
        log_move(A, log0 + pos, e.demand, e.to_center);
        if (h != e.from_center) set_err(X, kErrStaleTransfer, e.demand);
        A.home[e.demand] = e.to_center;
        red_add64(&A.load[e.from_center], -1);
        red_add64(&A.load[e.to_center], 1);
        A.rowslot[e.from_center] = i;
        A.src_list[pos] = e.from_center;
      } else if (e.kind == kEdgePenalty) {
        if (i != len - 1) set_err(X, kErrPenaltyEdge, i);
      }
      ns += __popc(bt);
    }
    if (lane == 0) {
      // placeholder moves (strict): in path order, a center's gain before its loss
      for (int i = 0; i < len; ++i) {
        const PathEdge e = path_at(S, i);
        if (e.kind != kEdgeDummy) continue;
        if (A.dummies == nullptr || A.dummies[e.from_center] <= 0) {
          set_err(X, kErrPlaceholder, e.from_center);
          break;
        }
        A.dummies[e.from_center] -= 1;
        A.dummies[e.to_center] += 1;
      }
      lc[kLcPrevSources] = ns;
      lc[kLcLogN] = log0 + ns;
      if (A.log_n != nullptr) *A.log_n = static_cast<int32_t>(log0 + ns < INT32_MAX ? log0 + ns : INT32_MAX);
      lc[kLcTransfers] += ns;
      int64_t r;
      if (add_ovf(lc[kLcDelta], cost, &r)) set_err(X, kErrOverflow, 0);
      lc[kLcDelta] = r;
      if (add_ovf(lc[kLcGain], -cost, &r)) set_err(X, kErrOverflow, 1);
      lc[kLcGain] = r;
      if (kind == kCycle) lc[kLcCycles] += 1;
      else lc[kLcPaths] += 1;
    }
  }
  // the π-repair search's sources (the dirty rows) travel in this exchange:
  // the labels of the finished search are no longer read (reconstruct's
  // exchange is behind us), and without rescans the repair starts right
  // after it
  X.delta = X.delta_main;
  reset_labels(X, 0);
  __syncthreads();
  publish_sources(X, dirty, nd, kRepair);
  __syncthreads();
  PROF_MARK(X, 0);   // T1
  // (no list validation here: until this barrier the lead's home[] writes
  // and, after it, other CTAs' T3 rescans race with a reader of the lists)
  exchange(X);
  PROF_MARK(X, 12);  // apply exchanges
  // ---- T3: rescans of the invalidated entries over the final buckets ----
  // Members of a source center u: its segment of the bucket index built at
  // launch start (A.bk_ids[A.bk_off[u] ..)), then its add list (demands that
  // moved to u since) — each still checked against home[]. An overflowed
  // add list falls back to the whole move log, an overflowed log to every
  // demand. Work split: every CTA walks all candidates and rebuilds only the
  // entries of ITS columns (the owner is the only writer of its lists in
  // this phase), so the member-row reads spread over the whole cluster.
  int total = 0;
  for (int i = 0; i < len; ++i) total += (path_at(S, i).kind == kEdgeTransfer) ? A.inv_cnt[i] : 0;
  if (total > 0) {
    int32_t* seg = S.seg;  // [3 * kMaxSeg]: (slot, prefix end, bucket count)
    int nseg = 0;
    int64_t nbase = 0;
    // allscan: candidates are every demand; generic: candidates split over
    // the CTAs, every invalidated column (both rare fallbacks)
    bool allscan = A.bk_ids == nullptr || *A.log_n > A.log_cap;
    bool uselog = false;
    for (int i = 0; i < len && !allscan; ++i) {
      if (path_at(S, i).kind != kEdgeTransfer || A.inv_cnt[i] == 0) continue;
      if (nseg == kMaxSeg) { allscan = true; break; }
      const int u = path_at(S, i).from_center;
      const int32_t nb = A.bk_off[u + 1] - A.bk_off[u];
      const int32_t na = A.add_cnt != nullptr ? A.add_cnt[u] : 0;
      if (na > A.add_cap) uselog = true;
      nbase += nb + min(na, A.add_cap);
      if (threadIdx.x == 0) {
        seg[3 * nseg] = i;
        seg[3 * nseg + 1] = static_cast<int32_t>(nbase);
        seg[3 * nseg + 2] = nb;
      }
      ++nseg;
    }
    if (threadIdx.x == 0) S.misc[5] = 0;
    if (threadIdx.x < kMaxSeg) { S.segmine[threadIdx.x] = 0; S.segcur[threadIdx.x] = 0; }
    __syncthreads();
    const int64_t nlog = (allscan || !uselog) ? 0 : *A.log_n;
    const int64_t ncand = allscan ? A.n : nbase + nlog;
    const int nw32 = (k + 31) >> 5;
    bool generic = allscan;
    // my invalidated columns per segment, compacted: (g << 16) | j
    int mycnt = 0;
    int maxmine = 0;  // most owned columns of one segment
    if (!generic) {
      for (int g = 0; g < nseg; ++g) {
        const int sl = seg[3 * g];
        const int cnt = A.inv_cnt[sl];
        for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
          const int j = A.inv_cols[static_cast<int64_t>(sl) * k + x];
          if (j >= jlo && j < jhi) {
            const int pos = atomicAdd(&S.misc[5], 1);
            if (pos < kMaxMine) {
              S.mine[pos] = (g << 16) | j;
              atomicAdd(&S.segmine[g], 1);
            }
          }
        }
      }
      __syncthreads();
      mycnt = S.misc[5];
      if (mycnt > kMaxMine) generic = true;  // too many: the generic path
    }
    // row mode: when this CTA owns a good part of a slot's invalidations,
    // members' cost rows are streamed over my columns (coalesced 16 B
    // pieces, one column bitmap per segment) instead of one 4 B gather per
    // (member, column)
    const int p0 = jlo >> 2, p1 = (jhi + 3) >> 2;  // my 16 B pieces
    const int npc = p1 - p0;
    bool rowmode = false;
    if (!generic) {
      for (int g = 0; g < nseg; ++g) maxmine = max(maxmine, S.segmine[g]);
      rowmode = kRowMode && nseg <= kRowSlots && 4 * maxmine >= npc;
      if (rowmode) {
        for (int w = threadIdx.x; w < nseg * nw32; w += blockDim.x) S.bits[w] = 0;
        __syncthreads();
        for (int x = threadIdx.x; x < mycnt; x += blockDim.x) {
          const int g = S.mine[x] >> 16, j = S.mine[x] & 0xffff;
          atomicOr(&S.bits[g * nw32 + (j >> 5)], 1u << (j & 31));
        }
      } else {
        // group my columns by segment (counting sort; order within a
        // segment is irrelevant)
        __syncthreads();
        if (threadIdx.x == 0) {
          int acc = 0;
          for (int g = 0; g < nseg; ++g) { const int c = S.segmine[g]; S.segmine[g] = acc; acc += c; }
          S.segmine[nseg] = acc;
        }
        for (int x = threadIdx.x; x < mycnt; x += blockDim.x) S.mine2[x] = S.mine[x];
        __syncthreads();
        for (int x = threadIdx.x; x < mycnt; x += blockDim.x) {
          const int g = S.mine2[x] >> 16;
          const int pos = atomicAdd(&S.segcur[g], 1);
          S.mine[S.segmine[g] + pos] = S.mine2[x] & 0xffff;
        }
      }
    }
    const bool full = generic;
    if (X.lead) {
      A.ctl->resc[0] += 1;
      A.ctl->resc[1] += full;
      A.ctl->resc[2] += rowmode;
      A.ctl->resc[3] += ncand;
      A.ctl->resc[5] += total;
    }
    // candidates: all of them in every CTA (own columns), or split over the
    // CTAs (every column) in the generic full mode
    const int64_t cbase = full ? static_cast<int64_t>(X.rank) * blockDim.x : 0;
    const int64_t stride = full ? static_cast<int64_t>(X.csz) * blockDim.x : blockDim.x;
    int maxcnt = 0;
    if (full) {
      for (int i = 0; i < len; ++i) {
        if (path_at(S, i).kind == kEdgeTransfer) maxcnt = max(maxcnt, A.inv_cnt[i]);
      }
    }
    for (int64_t base = cbase; base < ncand; base += stride) {
      if (threadIdx.x == 0) S.misc[0] = 0;
      __syncthreads();
      const int64_t x = base + threadIdx.x;
      if (x < ncand) {
        int32_t dd = -1, sl = -1;
        if (allscan) {
          dd = static_cast<int32_t>(x);
          const int32_t h = A.home[dd];
          if (h >= 0) {
            sl = A.rowslot[h];
            if (sl >= 0 && A.inv_cnt[sl] == 0) sl = -1;
          }
        } else if (x < nbase) {
          int g = 0;
          while (x >= seg[3 * g + 1]) ++g;
          const int slot = seg[3 * g];
          const int u = path_at(S, slot).from_center;
          const int64_t off = x - (g == 0 ? 0 : seg[3 * g - 2]);
          const int32_t nb = seg[3 * g + 2];
          dd = off < nb ? A.bk_ids[A.bk_off[u] + off]
                        : A.add_ids[static_cast<int64_t>(u) * A.add_cap + (off - nb)];
          if (A.home[dd] == u) sl = full ? slot : g;
        } else {
          const int64_t li = x - nbase;
          dd = A.log_d[li];
          const int32_t to = A.log_to[li];
          if (A.home[dd] == to) {
            sl = A.rowslot[to];
            if (sl >= 0 && A.inv_cnt[sl] == 0) sl = -1;
            if (sl >= 0 && !full) {  // slot -> segment
              int g = 0;
              while (g < nseg && seg[3 * g] != sl) ++g;
              sl = g < nseg ? g : -1;
            }
          }
        }
        if (sl >= 0) {
          const int q = atomicAdd(&S.misc[0], 1);
          S.qd[q] = dd;
          S.qs[q] = sl;  // full: path slot; else: segment
          S.qh[q] = row_of(A.rows, dd)[
                         path_at(S, full ? sl : seg[3 * sl]).from_center];
        }
      }
      __syncthreads();
      const int qn = S.misc[0];
      if (threadIdx.x == 0 && (full || X.rank == 0))
        atomicAdd(reinterpret_cast<unsigned long long*>(&A.ctl->resc[4]),
                  static_cast<unsigned long long>(qn));
      if (full) {
        // generic: (member, invalidated column) pairs over every column
        for (int p = threadIdx.x; p < qn * maxcnt; p += blockDim.x) {
          const int q = p % qn;
          const int xx = p / qn;
          const int sl2 = S.qs[q];
          const int cnt = A.inv_cnt[sl2];
          if (xx >= cnt) continue;
          const int32_t d2 = S.qd[q];
          const int u = path_at(S, sl2).from_center;
          const int j = A.inv_cols[static_cast<int64_t>(sl2) * k + xx];
          const int32_t* row = row_of(A.rows, d2);
          list_sink(A, static_cast<int64_t>(u) * k + j, pack_transfer(row[j] - S.qh[q], d2));
        }
      } else if (rowmode) {
        // (member, my 16 B piece): consecutive threads read consecutive
        // pieces of one member's row
        for (int p = threadIdx.x; p < qn * npc; p += blockDim.x) {
          const int q = p / npc;
          const int c4 = p0 + (p - q * npc);
          const int g = S.qs[q];
          const uint32_t word = S.bits[g * nw32 + (c4 >> 3)] >> ((c4 & 7) * 4);
          if ((word & 15u) == 0) continue;
          const int32_t d2 = S.qd[q];
          const int32_t hv = S.qh[q];
          const int u = path_at(S, seg[3 * g]).from_center;
          const int4 x4 = reinterpret_cast<const int4*>(row_of(A.rows, d2))[c4];
          const int32_t xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (word & (1u << e)) {
              list_sink(A, static_cast<int64_t>(u) * k + 4 * c4 + e, pack_transfer(xs[e] - hv, d2));
            }
          }
        }
      } else {
        // (member, my invalidated column of its segment) pairs
        for (int p = threadIdx.x; p < qn * maxmine; p += blockDim.x) {
          const int q = p % qn;
          const int xx = p / qn;
          const int g = S.qs[q];
          const int o0 = S.segmine[g], o1 = S.segmine[g + 1];
          if (xx >= o1 - o0) continue;
          const int j = S.mine[o0 + xx];
          const int32_t d2 = S.qd[q];
          const int u = path_at(S, seg[3 * g]).from_center;
          const int32_t* row = row_of(A.rows, d2);
          list_sink(A, static_cast<int64_t>(u) * k + j, pack_transfer(row[j] - S.qh[q], d2));
        }
      }
      __syncthreads();
    }
  }
  if (total > 0) {  // uniform: every CTA read the same counters after the T1 exchange
    if (threadIdx.x == 0) S.pub[X.par]->count = 0;
    PROF_MARK(X, 13);  // T3
    exchange(X);       // orders the rescanned lists before their readers
    PROF_MARK(X, 12);
  }
  // rescanned entries now hold the (up to) four smallest transfers of their
  // row: complete when fewer than four exist; refresh my tile columns
  for (int i = 0; i < len; ++i) {
    const PathEdge e = path_at(S, i);
    if (e.kind != kEdgeTransfer) continue;
    const int cnt = A.inv_cnt[i];
    for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
      const int j = A.inv_cols[static_cast<int64_t>(i) * k + x];
      if (j < jlo || j >= jhi) continue;
      const int64_t idx = static_cast<int64_t>(e.from_center) * k + j;
      const int64_t m = A.M[idx];
      int len = m != kEmpty;
#pragma unroll
      for (int q = 0; q < kTopK - 1; ++q) len += *mx_slot(A, idx, q) != kEmpty;
      A.LN[idx] = static_cast<uint8_t>(len | (len < kTopK ? 8 : 0));
      if (X.tile) X.wt[static_cast<int64_t>(e.from_center) * X.wst + (j - X.v0)] = key16(m);
    }
  }
  __syncthreads();
  validate_lists(X, 2);
  if (total > 0) {  // the T3 exchange came after the sources: publish them again
    publish_sources(X, dirty, nd, kRepair);
    __syncthreads();
    exchange(X);
  }
  if (X.lead) S.lc[kLcTindex] += gtimer() - t0;
  return nd;
}

// check_invariants: π feasible on every Γ edge certifies "no negative
// cycle" (refine.hpp:125-131). Owners check the edges into their nodes.
__device__ __forceinline__ void certify(Ctx& X) {
  const EngineArgs& A = X.A;
  if (!A.check_invariants) return;
  if (X.lead) X.S.lc[kLcChecks] += 1;
  bool bad = false;
  for (int u = 0; u < X.k; ++u) {
    const int64_t piu = pi_of(X, u);
    const bool dum = has_dummy(X, u);
    for (int v = X.v0 + threadIdx.x; v < min(X.v1, X.k); v += blockDim.x) {
      if (v == u) continue;
      const int64_t w = X.tile ? key16_weight(X.wt[static_cast<int64_t>(u) * X.wst + (v - X.v0)], dum)
                               : pair_weight(A.M[static_cast<int64_t>(u) * A.k + v], dum);
      if (w == kNoEdge) continue;
      if (w + piu - X.S.pis[v - X.v0] < 0) bad = true;
    }
  }
  if (bad) set_err(X, kErrInvariant, 0);
  __syncthreads();
  if (threadIdx.x == 0) X.S.pub[X.par]->count = 0;
  exchange(X);
}

// The reference checks a path's edge sum against its cost (refine.hpp:75-
// 79): the lead recounts it from the cost matrix (one lookup per edge).
__device__ __forceinline__ void check_path_sum(Ctx& X, int kind, int anchor, int len, int64_t refund_a,
                                            int64_t sl) {
  const EngineArgs& A = X.A;
  int64_t sum = 0;
  for (int i = 0; i < len; ++i) {
    const PathEdge e = path_at(X.S, i);
    if (e.kind == kEdgeTransfer) {
      const int32_t* row = row_of(A.rows, e.demand);
      sum += static_cast<int64_t>(row[e.to_center]) - row[e.from_center];
    } else if (e.kind == kEdgePenalty) {
      sum += marginal_penalty(X, e.from_center, A.load[e.from_center]) - refund_a;
    }
  }
  if (sum != lab_d(sl)) {
    set_err(X, kErrPathSum, len);
    if (atomicCAS(&g_dbg_printed, 0, 1) == 0) {
      printf("lbdd_b200 path sum mismatch rank %d kind %d anchor %d len %d label cost %lld edge sum %lld\n",
             X.rank, kind, anchor, len, static_cast<long long>(lab_d(sl)), static_cast<long long>(sum));
    }
  }
}

__device__ __forceinline__ void add_delta(Ctx& X, int64_t v, int arg) {
  int64_t r;
  if (add_ovf(X.S.lc[kLcDelta], v, &r)) set_err(X, kErrOverflow, arg);
  X.S.lc[kLcDelta] = r;
}

__device__ __forceinline__ void prefetch_scalars(Ctx& X, int64_t a) {
  if (threadIdx.x == 0 && a < X.A.a_end) {
    cp_async8(&X.S.pkey[a & 3], &X.A.arr_keys[a]);
    cp_async4(&X.S.ps[a & 3], &X.A.arr_s[a]);
  }
}
// needs arrival a's scalars landed and visible (wait + CTA barrier)
__device__ __forceinline__ void prefetch_row(Ctx& X, int64_t a) {
  if (a >= X.A.a_end) return;
  const int32_t d = static_cast<int32_t>(X.S.pkey[a & 3] & 0xffffffffLL);
  const int32_t s = X.S.ps[a & 3];
  const int32_t* row = row_of(X.A.rows, d);
  int32_t* dst = X.S.prow + (a & 1) * (X.s + 1);
  for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
    if (X.v0 + i < X.k) cp_async4(&dst[i], &row[X.v0 + i]);
  }
  if (threadIdx.x == blockDim.x - 1) cp_async4(&dst[X.s], &row[s]);
}

// the stage after a search: through kStCertify when invariants are checked
__device__ __forceinline__ int certify_then(const Ctx& X, int& cert_next, int next) {
  if (!X.A.check_invariants) return next;
  cert_next = next;
  return 5;  // kStCertify
}

}  // namespace cl

// Shared memory: see cl::carve.
__global__ void __launch_bounds__(LBDD_CLUSTER_THREADS, 1) cluster_engine_kernel(const __grid_constant__ EngineArgs A, int64_t* pi_global,
                                                                 int32_t* dirty_buf) {
  using namespace cl;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ctx X(A, cg::this_cluster());
  X.rank = static_cast<int>(X.cluster.block_rank());
  X.csz = static_cast<int>(X.cluster.num_blocks());
  X.k = A.k;
  X.s = (A.k + 1 + X.csz - 1) / X.csz;
  X.v0 = min(X.rank * X.s, A.k + 1);
  X.v1 = min(X.v0 + X.s, A.k + 1);
  X.tile = A.tile_mode != 0;
  {
    const int ns = X.v1 - X.v0;
    X.cpp = ns <= 0 ? 32 : ns < static_cast<int>(blockDim.x) ? ((ns + 31) & ~31) : blockDim.x;
    X.rpp = blockDim.x / X.cpp;
    X.tx = threadIdx.x % X.cpp;
    X.ty = threadIdx.x / X.cpp;
  }
  X.S = carve(smem_raw, A.k, X.s, A.tile_mode == 1);
  X.cin = inbox_cap(X.s);
  // O(k) per-search state outside shared memory (L1/L2): the weights into
  // anchor-in (read only by their owner) and each CTA's copy of the path
  X.S.path = A.path + static_cast<int64_t>(X.rank) * (A.k + 1);
  if (A.tile_mode == 1) {
    X.wt = X.S.wt;
    X.wst = X.s;
  } else {
    X.wt = A.ktile != nullptr ? A.ktile + X.v0 : nullptr;
    X.wst = A.k;
  }
  X.par = 0;
  X.cpar = 0;
  X.xincl = 0;
  X.xtotal = X.xpend = 0;
  X.xpmin = X.xomin = X.xslab = kLabInf;
  X.err = 0;
  X.lead = X.rank == 0 && threadIdx.x == 0;
  X.n_barriers = 0;
  X.n_rounds = 0;
  X.delta_main = A.delta_step <= 0 ? kLabInf / 4 : (A.delta_step << kLabShift);
  X.delta_path = A.delta_path <= 0 ? kLabInf / 4 : (A.delta_path << kLabShift);
  X.delta = X.delta_main;
  X.T = X.delta;
  X.prune = false;
  X.prune_c = 0;
  X.cur_slab = kLabInf;
  X.dbg = X.S.dbg;
  if (threadIdx.x < 16) X.dbg[threadIdx.x] = 0;
  if (X.rank == 0 && threadIdx.x == 0) {
    const EngineCtl* ctl = A.ctl;
    X.S.lc[kLcDelta] = ctl->delta;
    X.S.lc[kLcCycleCalls] = ctl->cycle_refine_calls;
    X.S.lc[kLcPathCalls] = ctl->path_refine_calls;
    X.S.lc[kLcCycles] = ctl->negative_cycles_removed;
    X.S.lc[kLcPaths] = ctl->negative_paths_removed;
    X.S.lc[kLcGain] = ctl->refinement_gain;
    X.S.lc[kLcTransfers] = ctl->transfers_applied;
    X.S.lc[kLcChecks] = ctl->invariant_checks;
    X.S.lc[kLcTbf] = ctl->t_bf_ns;
    X.S.lc[kLcTindex] = ctl->t_index_ns;
    X.S.lc[kLcPrevSources] = ctl->prev_sources;
    X.S.lc[kLcLogN] = A.log_n != nullptr ? *A.log_n : 0;
  }
  if (threadIdx.x < 16) X.S.prof[threadIdx.x] = 0;
  if (threadIdx.x < 4) X.S.cw[threadIdx.x] = threadIdx.x == 0 ? clock64() : 0;
  CS& S = X.S;
  const int k = A.k;
  const bool strict = A.mode == 1;
  for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
    const int v = X.v0 + i;
    S.pis[i] = v < k ? pi_global[v] : 0;
    S.chg[i] = 0;
    S.lab[i] = kLabInf;
  }
  if (X.tile) {
    const int ns = X.v1 - X.v0;
    for (int64_t i = threadIdx.x; i < static_cast<int64_t>(k) * ns; i += blockDim.x) {
      const int u = static_cast<int>(i / ns);
      const int col = static_cast<int>(i - static_cast<int64_t>(u) * ns);
      const int v = X.v0 + col;
      if (v < k) X.wt[static_cast<int64_t>(u) * X.wst + col] = key16(A.M[static_cast<int64_t>(u) * k + v]);
      else if (A.tile_mode == 1) X.wt[static_cast<int64_t>(u) * X.wst + col] = kNoKey16;
    }
  }
  if (threadIdx.x < 16) S.misc[threadIdx.x] = 0;
  if (threadIdx.x < 8) S.cred[threadIdx.x] = kLabInf;
  X.rph = 0;
  if (threadIdx.x < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&S.rmb[threadIdx.x])),
                 "r"(X.csz));
  }
  if (threadIdx.x < 2 * kMaxCS) {  // cluster-window addresses of every CTA's inbox / round mbarrier
    const int b = threadIdx.x / kMaxCS, r = threadIdx.x % kMaxCS;
    if (r < X.csz) {
      S.rin[threadIdx.x] = mapa_u32(smem_u32(S.inbox[b]), r);
      S.rbar[threadIdx.x] = mapa_u32(smem_u32(&S.rmb[b]), r);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      S.pub[b]->count = 0;
      S.pub[b]->err = 0;
      S.pub[b]->sinklab = kLabInf;
      S.pub[b]->val = kEmpty;
    }
  }
  __syncthreads();
  X.cluster.sync();
  // renormalise π so that its maximum is 0: reduced costs are invariant
  // under a uniform shift, and repairs only ever lower π, so without this it
  // would drift towards the packing limit over a long solve
  {
    if (threadIdx.x == 0) S.red[1] = INT64_MIN;
    __syncthreads();
    long long mx = INT64_MIN;
    for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
      if (X.v0 + i < k) mx = max(mx, static_cast<long long>(S.pis[i]));
    }
    atomicMax(reinterpret_cast<long long*>(&S.red[1]), mx);
    __syncthreads();
    if (threadIdx.x == 0) {
      S.pub[X.par]->val = S.red[1];
      S.pub[X.par]->count = 0;
    }
    exchange(X);
    int64_t gmax = INT64_MIN;
    for (int r = 0; r < X.csz; ++r) gmax = max(gmax, S.all[r].val);
    if (gmax != INT64_MIN) {
      for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
        if (X.v0 + i < k) S.pis[i] -= gmax;
      }
    }
    __syncthreads();
  }
  int* dirty = dirty_buf + X.rank * (2 * k + 4);  // per-CTA scratch
  const bool pf = !strict && A.arr_s != nullptr;  // asral arrival prefetch
  if (pf) {
    prefetch_scalars(X, A.a_begin);
    prefetch_scalars(X, A.a_begin + 1);
    cp_async_wait_all();
    __syncthreads();
    prefetch_row(X, A.a_begin);
  }

  PROF_MARK(X, 14);
  // The arrival loop as a state machine: every phase -- above all the search
  // rounds, reconstruct and apply -- appears ONCE in the kernel's code, so
  // the hot loop stays small in the instruction caches (the inlined
  // straight-line version was ~640 KB of SASS with a 20% L1.5 I-cache miss
  // rate). Stages:
  //   kStArrival   next arrival: strict target, insert + first cycle round
  //   kStSearch    search rounds of `kind`; then reconstruct + apply + the
  //                repair sources when a negative path was found
  //   kStAfterCycle  overload check (asral)
  //   kStPathBound   path bound C; start the path search or give up
  //   kStPathEnd     fixpoint loop (refine_to_fixpoint)
  enum Stage : int { kStArrival, kStSearch, kStAfterCycle, kStPathBound, kStPathEnd, kStCertify };
  static_assert(kStCertify == 5, "certify_then returns the stage id of kStCertify");
  int stage = kStArrival;
  int64_t a = A.a_begin;
  int32_t d = 0, s = 0;
  int64_t cost = 0, cap = 0, refund = 0, bound = 0, sink_inc = kLabInf;
  int kind = kCycle, after = kStAfterCycle, cert_next = kStArrival;
  bool applied = false;
  int64_t t_search = 0;
  while (!X.err) {
    if (stage == kStArrival) {
      if (a >= A.a_end) break;
      PROF_MARK(X, 14);
      if (A.debug_checks) {
        if (X.lead) g_dbg_arrival = a;
        validate_lists(X, 0);
      }
      const int64_t t0 = gtimer();
      int dum_a = 0;  // placeholder at the anchor after the eviction (strict)
      if (pf) {
        cp_async_wait_all();  // arrival a's (and a + 1's) scalars, a's cost row
        __syncthreads();
        const int64_t key = S.pkey[a & 3];
        d = static_cast<int32_t>(key & 0xffffffffLL);
        cost = key >> 32;
        s = S.ps[a & 3];
        prefetch_scalars(X, a + 2);
        prefetch_row(X, a + 1);
      } else if (!strict) {
        const int64_t key = A.arr_keys[a];
        d = static_cast<int32_t>(key & 0xffffffffLL);
        cost = key >> 32;
        s = A.best_center[d];
      } else {
        // strict target: cheapest center with placeholders (solver.hpp:257)
        d = A.order != nullptr ? A.order[a] : static_cast<int32_t>(a);
        const int32_t* row = row_of(A.rows, d);
        int64_t best = kEmpty;
        for (int j = X.v0 + threadIdx.x; j < min(X.v1, k); j += blockDim.x) {
          if (A.dummies[j] <= 0) continue;
          const int64_t pk = static_cast<int64_t>(row[j]) * (int64_t(1) << 32) + j;
          best = min(best, pk);
        }
        if (threadIdx.x == 0) S.red[0] = kEmpty;
        __syncthreads();
        atomicMin(reinterpret_cast<long long*>(&S.red[0]), static_cast<long long>(best));
        __syncthreads();
        if (threadIdx.x == 0) {
          S.pub[X.par]->val = S.red[0];
          S.pub[X.par]->count = 0;
          const int64_t b = S.red[0];
          S.pub[X.par]->aux = b == kEmpty ? 0 : static_cast<int32_t>(A.dummies[b & 0xffffffffLL]);
        }
        exchange(X);
        best = kEmpty;
        int cnt_t = 0;
        for (int r = 0; r < X.csz; ++r) {
          if (S.all[r].val < best) {
            best = S.all[r].val;
            cnt_t = S.all[r].aux;
          }
        }
        if (best == kEmpty) {
          if (X.lead) set_err(X, kErrNoResidual, d);
          break;
        }
        s = static_cast<int32_t>(best & 0xffffffffLL);
        cost = best >> 32;
        dum_a = (cnt_t - 1) > 0;
        __syncthreads();
        // only the owner of s touches dummies[s] in this phase
        if (s >= X.v0 && s < X.v1 && threadIdx.x == 0) A.dummies[s] -= 1;
      }
      ++a;
      const int64_t pi_s = pi_of(X, s);
      // ---- insert + first relaxation round of the cycle search (source s) ----
      reset_labels(X, pi_s);
      __syncthreads();
      const int32_t* row = row_of(A.rows, d);
      const int32_t* prow = S.prow + ((a - 1) & 1) * (X.s + 1);  // arrival a - 1 (a was advanced)
      const int32_t hv = pf ? prow[X.s] : row[s];
      for (int j = X.v0 + threadIdx.x; j < min(X.v1, k); j += blockDim.x) {
        if (j == s) continue;
        const int64_t idx = static_cast<int64_t>(s) * k + j;
        TopK t = list_load(A, idx);
        const int32_t cj = pf ? prow[j - X.v0] : row[j];
        if (list_insert(t, pack_transfer(cj - hv, d))) {
          if (X.tile) X.wt[static_cast<int64_t>(s) * X.wst + (j - X.v0)] = key16(t.e[0]);
        }
        list_store(A, idx, t);
        const int64_t m = t.e[0];
        const int64_t w = pair_weight(m, strict && dum_a);
        if (w != kNoEdge) {
          const int64_t rc = w + pi_s - S.pis[j - X.v0];
          const int64_t cand = rc * kLUnit + kHop + s;  // parent s
          if (cand < 0) {
            S.lab[j - X.v0] = cand;
            S.chg[j - X.v0] = 1;
          }
        }
      }
      if (s >= X.v0 && s < X.v1 && threadIdx.x == 0) S.lab[s - X.v0] = 0;  // the source
      fill_sink_weights(X, kCycle, s, 0, pi_s);
      if (X.lead) {
        const int32_t h = A.home[d];
        const int64_t li = S.lc[kLcLogN];
        log_move(A, li, d, s);
        if (h != -1) set_err(X, kErrAlreadyIndexed, d);
        A.home[d] = s;
        red_add64(&A.load[s], 1);
        S.lc[kLcLogN] = li + 1;
        if (A.log_n != nullptr) *A.log_n = static_cast<int32_t>(li + 1 < INT32_MAX ? li + 1 : INT32_MAX);
        if (strict) add_delta(X, cost, d);
        S.lc[kLcCycleCalls] += 1;
      }
      __syncthreads();
      collect(X, kCycle, s);
      exchange(X);
      validate_lists(X, 1);
      if (X.lead) S.lc[kLcTindex] += gtimer() - t0;
      PROF_MARK(X, 4);  // insert round
      kind = kCycle;
      refund = 0;
      bound = 0;
      sink_inc = kHop;  // cycle graph: rc >= 0 into anchor-in
      X.prune = true;
      X.prune_c = 0;
      after = kStAfterCycle;
      t_search = gtimer();
      stage = kStSearch;
      continue;
    }

    if (stage == kStSearch) {
      // ---- the search rounds (the one copy in the kernel) ----
      const int anchor = kind == kRepair ? -1 : s;
      const int rounds = search_rounds(X, kind, anchor, refund, bound, 0, sink_inc);
      if (X.lead) X.n_rounds += rounds;
      if (kind == kRepair) {
        apply_repair(X);  // π += min(0, d) over the explored region
        __syncthreads();
        PROF_MARK(X, 6);  // repairs
        stage = certify_then(X, cert_next, after);
        continue;
      }
      if (X.lead) X.S.lc[kLcTbf] += gtimer() - t_search;
      const int64_t sl = sink_label(X);
      const bool found = !X.err && sl != kLabInf && lab_d(sl) < 0;
      if (!found) {
        if (kind == kCycle) {
          PROF_MARK(X, 5);  // cycle search
          // π += min(0, d) over the explored region; a search that never ran
          // a round labelled nothing but its source (d = 0): π is unchanged
          // and needs no cluster barrier (uniform: every CTA counted the same)
          if (rounds > 0) apply_repair(X);
          __syncthreads();
          PROF_MARK(X, 6);
          stage = certify_then(X, cert_next, kStAfterCycle);
        } else {
          PROF_MARK(X, 8);  // path search
          applied = false;
          stage = certify_then(X, cert_next, kStPathEnd);
        }
        continue;
      }
      // ---- reconstruct + apply (the one copy) ----
      // the rounds' st.async exchanges do not release the owners' label
      // writes; reconstruct reads labels through DSMEM: one barrier
      X.cluster.sync();
      if (X.lead) X.n_barriers += 1;
      PROF_MARK(X, 9);
      // invalidation counters of the previous apply: its readers finished
      // before the last barrier, the next writers (T1) come after the next one
      if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i <= X.k; i += blockDim.x) X.A.inv_cnt[i] = 0;
      }
      const int len = reconstruct(X, kind, s, refund, sl);
      PROF_MARK(X, 10);
      if (len == 0 || X.err) break;
      if (kind == kPath && path_at(X.S, len - 1).kind != kEdgePenalty) {
        if (X.lead) set_err(X, kErrPenaltyEdge, len);
        X.err = 1;
        break;
      }
      // the reference checks the path's edge sum against its cost
      // (refine.hpp:75-79): recount it from the cost matrix (one lookup per
      // edge), so a stale transfer weight can never reach the objective
      if (X.lead) check_path_sum(X, kind, s, len, refund, sl);
      // a mismatch is raised at the next exchange; every CTA still runs
      // apply so the cluster barriers stay matched
      // apply ends with the π-repair search's sources (the dirty rows) exchanged
      apply(X, kind, len, lab_d(sl), dirty, s);
      PROF_MARK(X, 11);
      // ---- π repair from the dirty rows: a search of kind kRepair ----
      after = kind == kCycle ? kStAfterCycle : kStPathEnd;
      applied = true;
      kind = kRepair;
      refund = 0;
      bound = 0;
      sink_inc = kLabInf;
      X.prune = false;
      stage = kStSearch;
      continue;
    }

    if (stage == kStAfterCycle) {
      if (strict) { stage = kStArrival; continue; }
      // ---- overload: penalty-aware path refinement ----
      const int64_t load = A.load[s];
      cap = A.cap[s];
      if (load <= cap) {
        if (X.lead) add_delta(X, cost, d);
        stage = kStArrival;
        continue;
      }
      const int64_t refund_a = refund_penalty(X, s, load);
      if (X.lead) {
        int64_t r1;
        if (add_ovf(cost, refund_a, &r1)) set_err(X, kErrOverflow, d);
        add_delta(X, r1, d);
      }
      stage = kStPathBound;
      continue;
    }

    if (stage == kStPathBound) {
      if (X.lead) S.lc[kLcPathCalls] += 1;
      refund = refund_penalty(X, s, A.load[s]);
      // C = min_{u != s} marginal(u) - refund + π(u) - π(s): the most a
      // penalty edge can subtract; prune the search to d_rc < -C. One
      // exchange carries C and the search's source: the labels are reset
      // and s is published before it (discarded when the bound prunes), and
      // the penalty edges into anchor-in are evaluated in the same pass.
      const int64_t pis_now = pi_of(X, s);
      X.delta = X.delta_path;
      reset_labels(X, pis_now);
      long long lmin = kEmpty;
      for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
        const int u = X.v0 + i;
        int64_t sc = kLabInf;
        if (u != s && u < k) {
          const int64_t w = marginal_penalty(X, u, A.load[u]) - refund;
          lmin = min(lmin, static_cast<long long>(w + S.pis[i]));
          sc = S.pis[i] + w - pis_now;
        }
        S.sinkc[i] = sc;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
      if ((threadIdx.x & 31) == 0) S.wred[threadIdx.x >> 5] = lmin;
      __syncthreads();
      const int src[1] = {s};
      publish_sources(X, src, 1, kPath);
      if (threadIdx.x == 0) {
        long long m = kEmpty;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = min(m, static_cast<long long>(S.wred[w]));
        S.pub[X.par]->val = m;
      }
      __syncthreads();
      exchange(X);
      PROF_MARK(X, 7);  // path bound
      int64_t cmin = kEmpty;
      for (int r = 0; r < X.csz; ++r) cmin = min(cmin, S.all[r].val);
      if (!(cmin != kEmpty && cmin - pis_now < 0) || X.err) {
        if (X.lead) X.dbg[9] += 1;  // pruned
        applied = false;
        stage = certify_then(X, cert_next, kStPathEnd);
        continue;
      }
      const int64_t C = cmin - pis_now;
      if (X.lead) {
        X.dbg[13] += -C;
        X.dbg[14] = max(X.dbg[14], -C);
        X.dbg[15] += refund;
      }
      kind = kPath;
      bound = (-C) * kLUnit;
      X.prune = true;
      X.prune_c = C;
      sink_inc = kHop - bound;  // path graph: rc_pen >= C into anchor-in
      t_search = gtimer();
      stage = kStSearch;
      continue;
    }

    if (stage == kStCertify) {  // check_invariants only: the one copy of certify
      certify(X);
      stage = cert_next;
      continue;
    }

    // kStPathEnd
    X.delta = X.delta_main;
    stage = (A.fixpoint && applied && A.load[s] > cap) ? kStPathBound : kStArrival;
  }
  if (X.lead) {
    EngineCtl* ctl = A.ctl;
    ctl->delta = S.lc[kLcDelta];
    ctl->cycle_refine_calls = S.lc[kLcCycleCalls];
    ctl->path_refine_calls = S.lc[kLcPathCalls];
    ctl->negative_cycles_removed = S.lc[kLcCycles];
    ctl->negative_paths_removed = S.lc[kLcPaths];
    ctl->refinement_gain = S.lc[kLcGain];
    ctl->transfers_applied = S.lc[kLcTransfers];
    ctl->invariant_checks = S.lc[kLcChecks];
    ctl->t_bf_ns = S.lc[kLcTbf];
    ctl->t_index_ns = S.lc[kLcTindex];
    ctl->prev_sources = static_cast<int32_t>(S.lc[kLcPrevSources]);
    for (int i = 0; i < 15; ++i) A.ctl->prof[i] += S.prof[i];  // cycles per phase
    for (int i = 0; i < 16; ++i) A.ctl->dbg[i] += X.dbg[i];
    A.ctl->barriers += X.n_barriers;
    A.ctl->relax_rounds += X.n_rounds;

  }
  if (A.profile && threadIdx.x == 0) {
    A.ctl->cta_work[X.rank] += S.cw[1];
    A.ctl->cta_wait[X.rank] += S.cw[2];
  }
  // persist π for the next launch
  __syncthreads();
  for (int i = threadIdx.x; i < X.v1 - X.v0; i += blockDim.x) {
    const int v = X.v0 + i;
    if (v < k) pi_global[v] = S.pis[i];
  }
  X.cluster.sync();
}

}  // namespace lbdd_b200

namespace lbdd_b200 {
// Micro-benchmark of the exchange primitive alone (publish, cluster barrier,
// read every CTA's slot through DSMEM). Mode bit 0: also stage 128 remote
// 24-byte entries per round; bit 1: use barrier.cluster with a relaxed
// arrive + explicit cluster fence instead of cluster.sync().
__global__ void __launch_bounds__(512, 1) cluster_exchange_bench(int iters, int mode,
                                                                 long long* out) {
  __shared__ cl::Pub pub[2];
  __shared__ cl::Pub all[cl::kMaxCS];
  __shared__ cl::FEntry list[128];
  __shared__ cl::FEntry stage[128];
  cg::cluster_group cluster = cg::this_cluster();
  const int csz = static_cast<int>(cluster.num_blocks());
  if (threadIdx.x < 128) list[threadIdx.x].nd = threadIdx.x;
  if (threadIdx.x == 0) { pub[0].count = 1; pub[1].count = 1; }
  cluster.sync();
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ __align__(16) int4 box[2][cl::kMaxCS];
  if (threadIdx.x < 2) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[threadIdx.x]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(csz));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cluster.sync();
  const long long t0 = clock64();
  int par = 0;
  int acc = 0;
  unsigned phase[2] = {0, 0};
  if (mode & 8) {
    // st.async + mbarrier exchange: lane r of warp 0 sends this CTA's 16 B
    // record into slot `rank` of CTA r and arrives on r's mbarrier with the
    // byte count; thread 0 waits on the local mbarrier's phase
    const unsigned rank = cluster.block_rank();
    for (int it = 0; it < iters; ++it) {
      if (threadIdx.x < csz) {
        const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&box[par][rank]));
        const unsigned lm = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[par]));
        unsigned rb, rm;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(threadIdx.x));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rm) : "r"(lm), "r"(threadIdx.x));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                     ::"r"(rb), "r"(it), "r"(1), "r"(2), "r"(3), "r"(rm) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;"
                     ::"r"(rm), "r"(16) : "memory");
      }
      if (threadIdx.x == 0) {
        const unsigned lm = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[par]));
        asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                     " @!p bra W%=;\n}" ::"r"(lm), "r"(phase[par]) : "memory");
      }
      phase[par] ^= 1;
      __syncthreads();
      acc += box[par][it % csz].x;
      par ^= 1;
    }
  } else
  for (int it = 0; it < iters; ++it) {
    if (mode & 1) {
      if (threadIdx.x < 128) {
        const int r = threadIdx.x % csz;
        stage[threadIdx.x] = cluster.map_shared_rank(list, r)[threadIdx.x];
      }
      __syncthreads();
      acc += stage[threadIdx.x & 127].nd;
    }
    if (threadIdx.x == 0) pub[par].count = it;
    if (mode & 4) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    } else if (mode & 2) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
      cluster.sync();
    }
    if (threadIdx.x < csz) all[threadIdx.x] = *cluster.map_shared_rank(&pub[par], threadIdx.x);
    __syncthreads();
    acc += all[0].count;
    par ^= 1;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && cluster.block_rank() == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = acc;
  }
  cluster.sync();
}
}  // namespace lbdd_b200
