// The para-ASRAL engine: one persistent cooperative kernel (one CTA per SM)
// that runs the whole arrival loop of asral_solve / strict_solve on the
// device, so no arrival ever round-trips to the host.
//
// Per arrival (solver.hpp:143-167, 257-277):
//   phase I    insert the demand at its center: row M[s][*] of the
//              min-transfer matrix absorbs CM[d][*]-CM[d][s]
//              (SubspaceIndex::insert, subspace.hpp:46-56); anchored-graph
//              setup for the cycle search.
//   rounds     synchronous (Jacobi) relaxation over the (k+1)-node anchored
//              graph read out of M (build_negcycle_graph /
//              build_negpath_graph, subspace.hpp:313-371 + relax_nodes,
//              parallel.hpp:145-169). Each CTA owns one tile (source rows x
//              destination columns) whose transfer keys it caches in shared
//              memory; one grid barrier per round. Candidates are combined
//              with a packed (cand << 16 | source) atomicMin, so "smallest
//              source wins among equal candidates" — the reference's
//              deterministic parent rule — falls out of integer order.
//   extract    the parent walk (refine.hpp:53-80), redundantly in every CTA.
//   T1..T3     apply the path (apply_path_edges, refine.hpp:134-164):
//              T1 marks min-transfer entries whose argmin demand leaves its
//              center, T2 clears them, T3 folds the moved demands into their
//              new rows and rescans the invalidated entries with a segmented
//              argmin over the final bucket of each source center.
//   penalty    on overload the penalty-aware path graph (marginal penalty of
//              every center minus the anchor's refund) runs the same rounds
//              (negative_path_refine, refine.hpp:198-222).
//
// Consistency rules. (1) Data written by another CTA is read only after the
// grid barrier that follows the write; the barrier ends with an acquire on
// every SM (invalidating its L1), so plain loads are safe. (2) Every branch
// all CTAs must agree on is taken on values carried by the barrier word
// itself (changed / error bits) or on data no CTA rewrites before the next
// barrier: consecutive relaxation searches alternate between two buffer
// sets, so a search's results stay readable while the next one starts.
#include "common.cuh"

namespace lbdd_b200 {

// per-CTA phase flags reported through the next barrier: bit 0 "a distance
// improved", bit 1 "an error was recorded"
static __shared__ int s_cta_flags;
static __shared__ unsigned s_payload;

namespace {

__device__ __forceinline__ int64_t ld64(const int64_t* p) { return *p; }
__device__ __forceinline__ int32_t ld32(const int32_t* p) { return *p; }
__device__ __forceinline__ int64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<int64_t>(t);
}

__device__ __forceinline__ bool add_ovf(int64_t a, int64_t b, int64_t* r) {
  const int64_t s = static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
  *r = s;
  return ((a ^ s) & (b ^ s)) < 0;
}
__device__ __forceinline__ bool mul_ovf(int64_t a, int64_t b, int64_t* r) {
  const __int128 p = static_cast<__int128>(a) * static_cast<__int128>(b);
  *r = static_cast<int64_t>(p);
  return p != static_cast<__int128>(*r);
}

__device__ void set_error(const EngineArgs& A, int32_t code, int32_t arg) {
  if (atomicCAS(&A.ctl->error, 0, code) == 0) A.ctl->error_arg = arg;
  atomicOr(&s_cta_flags, 2);
}

// PenaltySpec::at, core.hpp:60-74
__device__ int64_t pen_at(const EngineArgs& A, int s, int64_t j) {
  const int64_t* p = A.ppar + A.poff[s];
  switch (A.pfam[s]) {
    case 0: return p[0];
    case 1: {
      int64_t m, r;
      if (mul_ovf(p[1], j - 1, &m) || add_ovf(p[0], m, &r)) {
        set_error(A, kErrOverflow, s);
        return 0;
      }
      return r;
    }
    default: {
      const int64_t len = A.poff[s + 1] - A.poff[s];
      return p[(j < len ? j : len) - 1];
    }
  }
}
// marginal_penalty / refund_penalty, core.hpp:196-208
__device__ int64_t marginal_penalty(const EngineArgs& A, int s, int64_t load) {
  if (load < 0) { set_error(A, kErrNegativeLoad, s); return 0; }
  return load < A.cap[s] ? 0 : pen_at(A, s, load - A.cap[s] + 1);
}
__device__ int64_t refund_penalty(const EngineArgs& A, int s, int64_t load) {
  if (load < 0) { set_error(A, kErrNegativeLoad, s); return 0; }
  return load <= A.cap[s] ? 0 : pen_at(A, s, load - A.cap[s]);
}

// Edge weight of a transfer pair out of the packed min-transfer word,
// cheapest_pair_edge (subspace.hpp:294-307): a surplus placeholder at the
// source turns a missing or non-negative transfer into a zero-cost edge.
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

// Key sentinel for "no demand at the source" inside the smem tile (a real
// key is CM[d][v] - CM[d][u] <= INT32_MAX - 1).
constexpr int32_t kNoKey = INT32_MAX;
__device__ __forceinline__ int32_t key_of(int64_t m) {
  return m == kEmpty ? kNoKey : transfer_key(m);
}
__device__ __forceinline__ int64_t key_weight(int32_t key, bool dummy) {
  if (dummy) return key != kNoKey && key < 0 ? key : 0;
  return key == kNoKey ? kNoEdge : static_cast<int64_t>(key);
}

struct Geo {
  int ncols;      // columns (destination nodes) of the relaxation
  int ncoltiles;
  int chunk;      // source rows per tile
  int nchunks;
  int ntiles;
};

__device__ Geo make_geo(int rows, int ncols) {
  Geo g;
  g.ncols = ncols;
  g.ncoltiles = (ncols + blockDim.x - 1) / blockDim.x;
  int want = gridDim.x / g.ncoltiles;
  if (want < 1) want = 1;
  g.chunk = (rows + want - 1) / want;
  if (g.chunk < 1) g.chunk = 1;
  g.nchunks = (rows + g.chunk - 1) / g.chunk;
  g.ntiles = g.ncoltiles * g.nchunks;
  return g;
}

// ---------------------------------------------------------------------
// barrier
// ---------------------------------------------------------------------

__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p,
                                                               unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct BufSet {
  int64_t* D[2];
  int32_t* P[2];
  int64_t* B[3];
};

struct Smem {
  int64_t* dist;    // [max chunk] resolved source distances of the tile rows
  int64_t* scal64;  // [4]: 0 path cost, 1 strict target
  int64_t* colw;    // [max chunk] anchor-in weights of the tile rows
  PathEdge* path;   // [k + 1]
  int32_t* par;     // [k + 2]
  int32_t* nodes;   // [k + 2]
  int32_t* cnt;     // [k + 2] invalidation counts snapshot
  int32_t* qd;      // [blockDim] rescan queue demand
  int32_t* qs;      // [blockDim] rescan queue slot
  int32_t* scalars; // [8]: 0 queue size, 1 path length, 2 path error
  int32_t* tilever; // [max chunk] row versions the tile was loaded at
  int32_t* tile;    // [max chunk * blockDim] cached keys (tile_mode)
  uint8_t* rowflag; // [max chunk]
  uint8_t* dum;     // [max chunk]
  // per-thread registers, identical in every thread of every CTA
  unsigned gen;     // barrier generation
  unsigned payload; // bits of the last barrier
  int err_seen;     // sticky: an error was reported through a barrier
  int search;       // relaxation searches started (buffer-set parity)
};

// Dynamic shared memory layout; bytes = smem_bytes(...) on the host
// (capi.cu) — keep the two in sync. 8-byte arrays first.
__device__ Smem carve_smem(unsigned char* p, int k, int maxchunk, bool tile) {
  Smem S;
  S.dist = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * maxchunk;
  S.scal64 = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * 4;
  S.colw = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * maxchunk;
  S.path = reinterpret_cast<PathEdge*>(p); p += sizeof(PathEdge) * (k + 1);
  S.par = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (k + 2);
  S.nodes = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (k + 2);
  S.cnt = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (k + 2);
  S.qd = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * blockDim.x;
  S.qs = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * blockDim.x;
  S.scalars = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * 8;
  S.tilever = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * maxchunk;
  S.tile = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * (tile ? maxchunk * blockDim.x : 0);
  S.rowflag = reinterpret_cast<uint8_t*>(p); p += maxchunk;
  S.dum = reinterpret_cast<uint8_t*>(p);
  S.gen = 0;
  S.payload = 0;
  S.err_seen = 0;
  S.search = 0;
  return S;
}

__device__ void smem_init(const EngineArgs& A, Smem& S, int maxchunk) {
  if (threadIdx.x == 0) {
    s_cta_flags = 0;
    s_payload = static_cast<unsigned>(ld_relaxed(&A.bar->release) >> 32);
  }
  if (threadIdx.x < 8) S.scalars[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < maxchunk; i += blockDim.x) S.tilever[i] = -1;
  __syncthreads();
  S.gen = s_payload;  // generation at launch, identical in all CTAs
  __syncthreads();
}

// Grid barrier. Arrival is one 64-bit atomic add carrying this CTA's
// phase flags; the last CTA folds them into the payload and publishes
// (generation, payload) with one release store.
__device__ void gsync(const EngineArgs& A, Smem& S) {
  __syncthreads();
  if (threadIdx.x == 0) {
    GridBar* b = A.bar;
    const int f = s_cta_flags;
    s_cta_flags = 0;
    const unsigned long long add =
        1ull | ((f & 1) ? (1ull << 32) : 0ull) | ((f & 2) ? (1ull << 48) : 0ull);
    const unsigned long long old = atom_add_acq_rel(&b->arrive, add);
    unsigned payload;
    if (static_cast<unsigned>(old & 0xffffffffull) == gridDim.x - 1) {
      const unsigned long long tot = old + add;
      payload = (((tot >> 32) & 0xffffull) ? 1u : 0u) | ((tot >> 48) ? 2u : 0u);
      st_relaxed(&b->arrive, 0ull);
      A.ctl->barriers += 1;
      st_release(&b->release, (static_cast<unsigned long long>(S.gen + 1) << 32) | payload);
    } else {
      while (static_cast<unsigned>(ld_relaxed(&b->release) >> 32) != S.gen + 1) {
      }
    }
    payload = static_cast<unsigned>(ld_acquire(&b->release));  // acquire + L1 invalidate
    s_payload = payload;
  }
  __syncthreads();
  S.payload = s_payload;
  S.gen += 1;
  if (S.payload & 2u) S.err_seen = 1;
}

// ---------------------------------------------------------------------
// relaxation
// ---------------------------------------------------------------------

struct GraphView {
  int kind;
  int anchor;    // anchor-out node; -1 for the collapsed Γ scan
  int rows;      // source nodes (centers)
  int ncols;     // destination nodes (k + 1: the last is anchor-in)
  const int64_t* dense;  // dense weights (rows x ncols) for the standalone API
};

__device__ __forceinline__ BufSet bufset(const EngineArgs& A, int search) {
  const int s = search & 1;
  BufSet bs;
  bs.D[0] = A.D[s][0]; bs.D[1] = A.D[s][1];
  bs.P[0] = A.P[s][0]; bs.P[1] = A.P[s][1];
  bs.B[0] = A.B[s][0]; bs.B[1] = A.B[s][1]; bs.B[2] = A.B[s][2];
  return bs;
}

// resolve(v): distance/parent after round r-1 from (dist after r-2, best
// candidate of round r-1).
__device__ __forceinline__ void resolve(const BufSet& bs, int r, int v, int64_t* d, int32_t* p) {
  const int64_t dprev = ld64(&bs.D[r & 1][v]);
  const int64_t b = ld64(&bs.B[(r + 2) % 3][v]);  // B_{r-1}
  const int32_t pprev = ld32(&bs.P[r & 1][v]);
  if (b != kEmpty && cand_value(b) < dprev) {
    *d = cand_value(b);
    *p = cand_source(b);
  } else {
    *d = dprev;
    *p = pprev;
  }
}

// The CTA's relaxation tile: source rows [u0, u1) x destination columns
// [c0, c0 + blockDim). Every tile maps to exactly one CTA (ntiles <= grid).
struct TileRange {
  bool valid;
  int uc, u0, u1, c0;
};
__device__ __forceinline__ TileRange my_tile(const Geo& geo, int rows) {
  TileRange T;
  const int t = blockIdx.x;
  T.valid = t < geo.ntiles;
  const int ct = T.valid ? t % geo.ncoltiles : 0;
  T.uc = T.valid ? t / geo.ncoltiles : 0;
  T.u0 = T.uc * geo.chunk;
  T.u1 = T.valid ? min(rows, T.u0 + geo.chunk) : T.u0;
  T.c0 = ct * blockDim.x;
  return T;
}

// Refresh the cached tile rows whose M row changed since they were loaded
// (row versions bumped by the insert / path phases) and the anchor-in
// weights of this graph. Runs at the start of every relaxation search.
__device__ void refresh_tile(const EngineArgs& A, const GraphView& G, const Geo& geo, Smem& S) {
  const TileRange T = my_tile(geo, G.rows);
  if (!T.valid || G.dense != nullptr) return;
  const int rows = T.u1 - T.u0;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    const int32_t v = ld32(&A.rowver[T.u0 + i]);
    S.rowflag[i] = v != S.tilever[i];
    S.tilever[i] = v;
    S.colw[i] = G.kind != kGammaGraph ? ld64(&A.colW[T.u0 + i]) : kNoEdge;
  }
  __syncthreads();
  if (A.tile_mode) {
    const int c = T.c0 + threadIdx.x;
    for (int i = 0; i < rows; ++i) {
      if (!S.rowflag[i]) continue;
      const int u = T.u0 + i;
      S.tile[i * blockDim.x + threadIdx.x] =
          (c < A.k && c != u) ? key_of(ld64(&A.M[static_cast<int64_t>(u) * A.k + c])) : kNoKey;
    }
  }
  __syncthreads();
}

__device__ void relax_round(const EngineArgs& A, const GraphView& G, const BufSet& bs,
                            const Geo& geo, int r, const uint8_t* dumflag, Smem& S) {
  int64_t* Bcur = bs.B[r % 3];
  int64_t* Bnext = bs.B[(r + 1) % 3];
  int64_t* Dout = bs.D[(r + 1) & 1];  // D_{r-1}
  int32_t* Pout = bs.P[(r + 1) & 1];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gsz = gridDim.x * blockDim.x;
  for (int c = gtid; c < G.ncols; c += gsz) Bnext[c] = kEmpty;

  const TileRange T = my_tile(geo, G.rows);
  if (!T.valid) return;
  const int c = T.c0 + threadIdx.x;
  const bool col_ok = c < G.ncols;
  // own column first so its loads overlap the row resolves
  int64_t dc = kUnreachable;
  int32_t pc = -1;
  if (col_ok) resolve(bs, r, c, &dc, &pc);
  for (int i = threadIdx.x; i < T.u1 - T.u0; i += blockDim.x) {
    int64_t d;
    int32_t p;
    resolve(bs, r, T.u0 + i, &d, &p);
    S.dist[i] = d;
    S.dum[i] = dumflag != nullptr ? dumflag[T.u0 + i] : 0;
  }
  __syncthreads();
  if (!col_ok) return;
  if (T.uc == 0) {
    Dout[c] = dc;
    Pout[c] = pc;
  }
  // anchor-out has no in-edges in the solver graphs (edges into the anchor
  // are redirected to anchor-in); the collapsed Γ scan has no anchor-in.
  if (G.dense == nullptr && (c == G.anchor || (G.kind == kGammaGraph && c == A.k))) return;
  int64_t best = kEmpty;
  const int rows = T.u1 - T.u0;
  if (G.dense == nullptr && c == A.k) {
    // anchor-in column: transfer into the anchor (cycle graph) or the
    // penalty-difference edge (path graph), cached per search in S.colw
    for (int i = 0; i < rows; ++i) {
      const int64_t w = S.colw[i];
      const int64_t du = S.dist[i];
      if (w == kNoEdge || du >= kUnreachable) continue;
      const int64_t p = pack_cand(du + w, T.u0 + i);
      best = p < best ? p : best;
    }
  } else if (G.dense == nullptr && A.tile_mode) {
#pragma unroll 4
    for (int i = 0; i < rows; ++i) {
      const int64_t w = key_weight(S.tile[i * blockDim.x + threadIdx.x], S.dum[i] != 0);
      const int64_t du = S.dist[i];
      if (w == kNoEdge || du >= kUnreachable) continue;
      const int64_t p = pack_cand(du + w, T.u0 + i);
      best = p < best ? p : best;
    }
  } else {
    // global weights, fetched 8 rows at a time (independent loads)
    for (int ib = 0; ib < rows; ib += 8) {
      int64_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = ib + j;
        const int u = T.u0 + i;
        if (i >= rows) {
          w[j] = kNoEdge;
        } else if (G.dense != nullptr) {
          w[j] = G.dense[static_cast<int64_t>(u) * G.ncols + c];
        } else {
          w[j] = u == c ? kNoEdge
                        : pair_weight(ld64(&A.M[static_cast<int64_t>(u) * A.k + c]), S.dum[i] != 0);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = ib + j;
        if (w[j] == kNoEdge) continue;
        const int64_t du = S.dist[i];
        if (du >= kUnreachable) continue;
        const int64_t p = pack_cand(du + w[j], T.u0 + i);
        best = p < best ? p : best;
      }
    }
  }
  if (best != kEmpty) {
    atomicMin(reinterpret_cast<long long*>(&Bcur[c]), static_cast<long long>(best));
    if (cand_value(best) < dc) atomicOr(&s_cta_flags, 1);
  }
}

// Start a relaxation search: pick the next buffer set and initialise it;
// for the anchored graphs also the anchor-in weights (no barrier inside).
__device__ BufSet refine_setup(const EngineArgs& A, const GraphView& G, const uint8_t* dumflag,
                               Smem& S) {
  S.search += 1;
  const BufSet bs = bufset(A, S.search);
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gsz = gridDim.x * blockDim.x;
  for (int v = gtid; v < G.ncols; v += gsz) {
    bs.D[1][v] = (G.kind == kGammaGraph || v == G.anchor) ? 0 : kUnreachable;
    bs.P[1][v] = -1;
    bs.B[0][v] = kEmpty;
    bs.B[1][v] = kEmpty;
  }
  if (G.dense == nullptr) {
    if (G.kind == kCycleGraph) {
      for (int u = gtid; u < A.k; u += gsz) {
        A.colW[u] = u == G.anchor ? kNoEdge
                                  : pair_weight(ld64(&A.M[static_cast<int64_t>(u) * A.k + G.anchor]),
                                                dumflag != nullptr && dumflag[u]);
      }
    } else if (G.kind == kPathGraph) {
      const int64_t aload = ld64(&A.load[G.anchor]);
      const int64_t refund = refund_penalty(A, G.anchor, aload);
      for (int u = gtid; u < A.k; u += gsz) {
        A.colW[u] = u == G.anchor ? kNoEdge
                                  : marginal_penalty(A, u, ld64(&A.load[u])) - refund;
      }
    }
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i <= A.k; i += blockDim.x) A.inv_cnt[i] = 0;
  }
  return bs;
}

// Rounds until no distance improves. Returns the final round index r
// (final distances live in bs.D[(r+1)&1]); -r on a negative-cycle witness.
__device__ int run_rounds(const EngineArgs& A, const GraphView& G, const BufSet& bs,
                          const uint8_t* dumflag, Smem& S) {
  const Geo geo = make_geo(G.rows, G.ncols);
  const int max_rounds = G.ncols;  // node_count rounds, refine.hpp:41
  refresh_tile(A, G, geo, S);
  int r = 1;
  for (;;) {
    relax_round(A, G, bs, geo, r, dumflag, S);
    gsync(A, S);
    if (!(S.payload & 1u)) break;
    if (r == max_rounds) return -r;
    ++r;
  }
  return r;
}

// ---------------------------------------------------------------------
// path extraction (every CTA, redundantly) and application
// ---------------------------------------------------------------------

// Walks parents from anchor-in; fills S.path / S.scalars[1]. Returns false
// (with an error recorded by block 0) on a broken chain or sum mismatch.
__device__ bool extract_path(const EngineArgs& A, const GraphView& G, const BufSet& bs, int r,
                             const uint8_t* dumflag, Smem& S) {
  const int32_t* Pf = bs.P[(r + 1) & 1];
  const int nodes = G.ncols;
  for (int v = threadIdx.x; v < nodes; v += blockDim.x) S.par[v] = ld32(&Pf[v]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int err = 0;
    int len = 0;
    int node = nodes - 1;
    S.nodes[0] = node;
    while (node != G.anchor) {
      if (len >= nodes) { err = kErrPathNotSimple; break; }
      const int u = S.par[node];
      if (u < 0) { err = kErrBrokenParent; break; }
      S.nodes[++len] = u;
      node = u;
    }
    int64_t sum = 0;
    if (!err) {
      for (int i = 0; i < len; ++i) {
        const int x = S.nodes[len - i];      // source node
        const int y = S.nodes[len - i - 1];  // destination node
        PathEdge e;
        const int cy = (y == nodes - 1) ? G.anchor : y;
        e.from_center = x;
        e.to_center = cy;
        e.demand = -1;
        int64_t w;
        if (G.kind == kPathGraph && y == nodes - 1) {
          e.kind = kEdgePenalty;
          w = ld64(&A.colW[x]);
        } else {
          const bool dum = dumflag != nullptr && dumflag[x] && G.kind != kPathGraph;
          const int64_t m = ld64(&A.M[static_cast<int64_t>(x) * A.k + cy]);
          e.kind = pair_kind(m, dum);
          w = pair_weight(m, dum);
          if (e.kind == kEdgeTransfer) e.demand = transfer_demand(m);
        }
        S.path[i] = e;
        sum += w;
      }
      const int64_t cost = ld64(&bs.D[(r + 1) & 1][nodes - 1]);
      if (sum != cost) err = kErrPathSum;
      S.scal64[0] = cost;
    }
    S.scalars[1] = len;
    S.scalars[2] = err;
    if (err && blockIdx.x == 0) set_error(A, err, len);
  }
  __syncthreads();
  return S.scalars[2] == 0;
}

// T1..T3 (see file header).
__device__ void apply_path(const EngineArgs& A, const GraphView& G, Smem& S) {
  const int L = S.scalars[1];
  const int64_t cost = S.scal64[0];
  const int k = A.k;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = gtimer();

  // ---- T1: mark entries whose argmin demand leaves its center ----
  for (int64_t idx = gtid; idx < static_cast<int64_t>(L) * k; idx += gsz) {
    const int i = static_cast<int>(idx / k);
    const int j = static_cast<int>(idx - static_cast<int64_t>(i) * k);
    const PathEdge e = S.path[i];
    if (e.kind != kEdgeTransfer || j == e.from_center) continue;
    const int64_t m = ld64(&A.M[static_cast<int64_t>(e.from_center) * k + j]);
    if (m != kEmpty && transfer_demand(m) == e.demand) {
      const int pos = atomicAdd(&A.inv_cnt[i], 1);
      A.inv_cols[static_cast<int64_t>(i) * k + pos] = j;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    EngineCtl* ctl = A.ctl;
    for (int i = 0; i < ctl->prev_sources; ++i) A.rowslot[A.src_list[i]] = -1;
    int ns = 0;
    for (int i = 0; i < L; ++i) {
      const PathEdge e = S.path[i];
      if (e.kind == kEdgeTransfer) {
        // transfer_validate, subspace.hpp:83-92
        if (A.home[e.demand] != e.from_center) { set_error(A, kErrStaleTransfer, e.demand); break; }
        A.home[e.demand] = e.to_center;
        A.load[e.from_center] -= 1;
        A.load[e.to_center] += 1;
        A.rowslot[e.from_center] = i;
        A.src_list[ns++] = e.from_center;
        A.rowver[e.from_center] += 1;
        A.rowver[e.to_center] += 1;
        ctl->transfers_applied += 1;
      } else if (e.kind == kEdgeDummy) {
        if (A.dummies == nullptr || A.dummies[e.from_center] <= 0) {
          set_error(A, kErrPlaceholder, e.from_center);
          break;
        }
        A.dummies[e.from_center] -= 1;
        A.dummies[e.to_center] += 1;
      } else if (e.kind == kEdgePenalty) {
        if (i != L - 1) { set_error(A, kErrPenaltyEdge, i); break; }
      }
    }
    ctl->prev_sources = ns;
    int64_t r;
    if (add_ovf(ctl->delta, cost, &r)) set_error(A, kErrOverflow, 0);
    ctl->delta = r;
    if (add_ovf(ctl->refinement_gain, -cost, &r)) set_error(A, kErrOverflow, 1);
    ctl->refinement_gain = r;
    if (G.kind == kCycleGraph) ctl->negative_cycles_removed += 1;
    else ctl->negative_paths_removed += 1;
  }
  gsync(A, S);

  // ---- T2: clear the invalidated entries ----
  for (int64_t idx = gtid; idx < static_cast<int64_t>(L) * k; idx += gsz) {
    const int i = static_cast<int>(idx / k);
    const int pos = static_cast<int>(idx - static_cast<int64_t>(i) * k);
    const PathEdge e = S.path[i];
    if (e.kind != kEdgeTransfer) continue;
    if (pos < ld32(&A.inv_cnt[i])) {
      const int j = ld32(&A.inv_cols[static_cast<int64_t>(i) * k + pos]);
      A.M[static_cast<int64_t>(e.from_center) * k + j] = kEmpty;
    }
  }
  gsync(A, S);

  // ---- T3: fold moved demands into their new rows + segmented rescans ----
  for (int64_t idx = gtid; idx < static_cast<int64_t>(L) * k; idx += gsz) {
    const int i = static_cast<int>(idx / k);
    const int j = static_cast<int>(idx - static_cast<int64_t>(i) * k);
    const PathEdge e = S.path[i];
    if (e.kind != kEdgeTransfer || j == e.to_center) continue;
    const int32_t* row = row_of(A.rows, e.demand);
    const int64_t v = pack_transfer(row[j] - row[e.to_center], e.demand);
    atomicMin(reinterpret_cast<long long*>(&A.M[static_cast<int64_t>(e.to_center) * k + j]),
              static_cast<long long>(v));
  }
  int total = 0;
  for (int i = threadIdx.x; i < L; i += blockDim.x) S.cnt[i] = ld32(&A.inv_cnt[i]);
  __syncthreads();
  for (int i = 0; i < L; ++i) total += S.cnt[i];
  if (total > 0) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < A.n;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      if (threadIdx.x == 0) S.scalars[0] = 0;
      __syncthreads();
      const int64_t d = base + threadIdx.x;
      if (d < A.n) {
        const int32_t h = ld32(&A.home[d]);
        if (h >= 0) {
          const int32_t sl = ld32(&A.rowslot[h]);
          if (sl >= 0 && S.cnt[sl] > 0) {
            const int q = atomicAdd(&S.scalars[0], 1);
            S.qd[q] = static_cast<int32_t>(d);
            S.qs[q] = sl;
          }
        }
      }
      __syncthreads();
      const int qn = S.scalars[0];
      for (int q = warp; q < qn; q += nwarps) {
        const int32_t dd = S.qd[q];
        const int sl = S.qs[q];
        const int u = S.path[sl].from_center;
        const int32_t* row = row_of(A.rows, dd);
        const int32_t hv = row[u];
        const int32_t* cols = A.inv_cols + static_cast<int64_t>(sl) * k;
        for (int x = lane; x < S.cnt[sl]; x += 32) {
          const int j = ld32(&cols[x]);
          atomicMin(reinterpret_cast<long long*>(&A.M[static_cast<int64_t>(u) * k + j]),
                    static_cast<long long>(pack_transfer(row[j] - hv, dd)));
        }
      }
      __syncthreads();
    }
  }
  gsync(A, S);
  if (blockIdx.x == 0 && threadIdx.x == 0) A.ctl->t_index_ns += gtimer() - t0;
}

// One negative_cycle_refine / negative_path_refine after its setup phase
// and barrier. Returns whether a negative path was applied (grid-uniform).
__device__ bool refine_run(const EngineArgs& A, int kind, int anchor, const BufSet& bs,
                           const uint8_t* dumflag, Smem& S) {
  GraphView G{kind, anchor, A.k, A.k + 1, nullptr};
  const int64_t t0 = gtimer();
  const int r = run_rounds(A, G, bs, dumflag, S);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.ctl->t_bf_ns += gtimer() - t0;
    A.ctl->relax_rounds += r < 0 ? -r : r;
    if (kind == kCycleGraph) A.ctl->cycle_refine_calls += 1;
    else A.ctl->path_refine_calls += 1;
  }
  if (r < 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_error(A, kErrNegCycleWitness, anchor);
    return false;
  }
  // final distances of this search stay untouched until the search after
  // next (buffer sets alternate), so every CTA reads the same value
  const int64_t cost = ld64(&bs.D[(r + 1) & 1][A.k]);
  if (!(cost < 0)) return false;  // unreachable sink is kUnreachable > 0
  if (!extract_path(A, G, bs, r, dumflag, S)) return false;
  if (kind == kPathGraph) {
    const int L = S.scalars[1];
    if (L == 0 || S.path[L - 1].kind != kEdgePenalty) {
      if (blockIdx.x == 0 && threadIdx.x == 0) set_error(A, kErrPenaltyEdge, L);
      return false;
    }
  }
  apply_path(A, G, S);
  return true;
}

// gamma_has_negative_cycle (refine.hpp:86-116) as Jacobi rounds from an
// all-zero virtual source; a negative cycle keeps improving through
// round k+1.
__device__ bool gamma_has_negative_cycle(const EngineArgs& A, const uint8_t* dumflag, Smem& S) {
  // same tile geometry as the anchored graphs (k+1 columns); column k
  // (anchor-in) does not exist in Γ and is skipped by relax_round
  GraphView G{kGammaGraph, -1, A.k, A.k + 1, nullptr};
  const BufSet bs = refine_setup(A, G, dumflag, S);
  gsync(A, S);
  const Geo geo = make_geo(G.rows, G.ncols);
  refresh_tile(A, G, geo, S);
  for (int r = 1;; ++r) {
    relax_round(A, G, bs, geo, r, dumflag, S);
    gsync(A, S);
    if (!(S.payload & 1u)) return false;
    if (r == A.k + 1) return true;
  }
}

__device__ void assert_no_negative_cycle(const EngineArgs& A, const uint8_t* dumflag, Smem& S) {
  if (!A.check_invariants) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) A.ctl->invariant_checks += 1;
  if (gamma_has_negative_cycle(A, dumflag, S)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_error(A, kErrInvariant, 0);
  }
  gsync(A, S);
}

__device__ void add_delta(const EngineArgs& A, int64_t v, int32_t arg) {
  int64_t r;
  if (add_ovf(A.ctl->delta, v, &r)) set_error(A, kErrOverflow, arg);
  A.ctl->delta = r;
}

}  // namespace

// dumflag[u] = surplus placeholder at u (strict mode), derived per refine.
__global__ void __launch_bounds__(512, 1) asral_engine_kernel(EngineArgs A, uint8_t* dumflag_buf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int k = A.k;
  const int maxchunk = make_geo(k, k + 1).chunk;
  Smem S = carve_smem(smem_raw, k, maxchunk, A.tile_mode != 0);
  smem_init(A, S, maxchunk);
  S.search = A.search_base;

  const bool strict = A.mode == 1;
  const uint8_t* dumflag = strict ? dumflag_buf : nullptr;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;

  // ---- standalone single refinement / Γ check (API entry points) ----
  if (A.single_kind >= 0) {
    if (strict) {
      for (int64_t u = gtid; u < k; u += gsz) dumflag_buf[u] = A.dummies[u] > 0;
    }
    if (A.single_kind == kGammaGraph) {
      gsync(A, S);
      const bool cyc = gamma_has_negative_cycle(A, dumflag, S);
      if (lead) A.single_out[0] = cyc ? 1 : 0;
      return;
    }
    if (A.single_kind == kPathGraph && lead) {
      if (A.load[A.single_anchor] <= A.cap[A.single_anchor]) set_error(A, kErrNotOverloaded, A.single_anchor);
    }
    gsync(A, S);
    if (S.err_seen) return;
    GraphView G{A.single_kind, A.single_anchor, k, k + 1, nullptr};
    const BufSet bs = refine_setup(A, G, dumflag, S);
    gsync(A, S);
    const int64_t before = ld64(&A.ctl->delta);
    const bool applied = refine_run(A, A.single_kind, A.single_anchor, bs, dumflag, S);
    assert_no_negative_cycle(A, dumflag, S);
    if (lead) {
      A.single_out[0] = applied ? 1 : 0;
      *A.single_gain = applied ? A.ctl->delta - before : 0;
    }
    return;
  }

  // ---- the arrival loop ----
  for (int64_t a = A.a_begin; a < A.a_end; ++a) {
    if (S.err_seen) break;
    int32_t d, s;
    int64_t cost;
    const int64_t t0 = gtimer();
    if (!strict) {
      const int64_t key = A.arr_keys[a];
      d = static_cast<int32_t>(key & 0xffffffffLL);
      cost = key >> 32;
      s = A.best_center[d];
    } else {
      // strict target: cheapest center still holding placeholders
      // (solver.hpp:257-268), computed redundantly per CTA.
      d = A.order != nullptr ? A.order[a] : static_cast<int32_t>(a);
      const int32_t* row = row_of(A.rows, d);
      int64_t best = kEmpty;
      for (int j = threadIdx.x; j < k; j += blockDim.x) {
        if (ld64(&A.dummies[j]) <= 0) continue;
        const int64_t pk = static_cast<int64_t>(row[j]) * (int64_t(1) << 32) + j;
        best = pk < best ? pk : best;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
      }
      if (threadIdx.x == 0) S.scal64[1] = kEmpty;
      __syncthreads();
      if ((threadIdx.x & 31) == 0) atomicMin(reinterpret_cast<long long*>(&S.scal64[1]), best);
      __syncthreads();
      best = S.scal64[1];
      if (best == kEmpty) {
        if (lead) set_error(A, kErrNoResidual, d);
        break;
      }
      s = static_cast<int32_t>(best & 0xffffffffLL);
      cost = best >> 32;
      // placeholders as the refinement will see them (after the eviction);
      // the decrement itself lands in the next phase, after every CTA has
      // read the old counts
      for (int64_t u = gtid; u < k; u += gsz) {
        dumflag_buf[u] = (ld64(&A.dummies[u]) - (u == s ? 1 : 0)) > 0;
      }
      gsync(A, S);
      if (lead) A.dummies[s] -= 1;
    }

    // ---- phase I: insert + cycle-graph setup ----
    BufSet bs;
    {
      const int32_t* row = row_of(A.rows, d);
      const int32_t hv = row[s];
      int64_t* Ms = A.M + static_cast<int64_t>(s) * k;
      for (int64_t j = gtid; j < k; j += gsz) {
        if (j == s) continue;
        const int64_t v = pack_transfer(row[j] - hv, d);
        if (v < ld64(&Ms[j])) Ms[j] = v;
      }
      if (lead) {
        if (A.home[d] != -1) set_error(A, kErrAlreadyIndexed, d);
        A.home[d] = s;
        A.load[s] += 1;
        A.rowver[s] += 1;
        if (strict) add_delta(A, cost, d);
      }
      GraphView G{kCycleGraph, s, k, k + 1, nullptr};
      bs = refine_setup(A, G, dumflag, S);
      gsync(A, S);
      if (lead) A.ctl->t_index_ns += gtimer() - t0;
    }
    refine_run(A, kCycleGraph, s, bs, dumflag, S);
    assert_no_negative_cycle(A, dumflag, S);
    if (strict) continue;

    // ---- overload: penalty-aware path refinement ----
    const int64_t load = ld64(&A.load[s]);
    const int64_t cap = A.cap[s];
    if (load <= cap) {
      if (lead) add_delta(A, cost, d);
      continue;
    }
    if (lead) {
      int64_t r1;
      const int64_t refund = refund_penalty(A, s, load);
      if (add_ovf(cost, refund, &r1)) set_error(A, kErrOverflow, d);
      add_delta(A, r1, d);
    }
    for (;;) {
      GraphView G{kPathGraph, s, k, k + 1, nullptr};
      const BufSet pbs = refine_setup(A, G, nullptr, S);
      gsync(A, S);
      const bool applied = refine_run(A, kPathGraph, s, pbs, nullptr, S);
      assert_no_negative_cycle(A, nullptr, S);
      if (!(A.fixpoint && applied && ld64(&A.load[s]) > cap)) break;
      if (S.err_seen) break;
    }
  }
  if (lead) A.ctl->search_count = S.search;
}

// Standalone lowest_cost_path / relax_round over a dense anchored graph
// (the AuxGraph-level API, refine.hpp:28-81, parallel.hpp:175-210). Same
// round machinery, weights from `dense`, buffer set 0.
__global__ void __launch_bounds__(512, 1) dense_path_kernel(EngineArgs A, const int64_t* dense,
                                                            int32_t node_count, int32_t anchor,
                                                            int32_t one_round, int32_t* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int rows = node_count - 1;
  const Geo geo = make_geo(rows, node_count);
  Smem S = carve_smem(smem_raw, rows, geo.chunk, false);
  smem_init(A, S, geo.chunk);
  GraphView G{kCycleGraph, anchor, rows, node_count, dense};
  if (one_round) {
    // inputs were staged by the host in set 0: D[1]=dist_in, P[1]=parent_in,
    // B[0]=B[1]=empty; round 1 computes D_0 = dist_in and B_1.
    const BufSet bs = bufset(A, 0);
    relax_round(A, G, bs, geo, 1, nullptr, S);
    gsync(A, S);
    const int changed = (S.payload & 1u) ? 1 : 0;
    // finalize D_1 = resolve(D_0, B_1) into D[1] / P[1]
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int gsz = gridDim.x * blockDim.x;
    for (int v = gtid; v < node_count; v += gsz) {
      int64_t d;
      int32_t p;
      resolve(bs, 2, v, &d, &p);
      bs.D[1][v] = d;
      bs.P[1][v] = p;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = changed;
    return;
  }
  S.search = 1;  // refine_setup bumps to 2 -> buffer set 0
  const BufSet bs = refine_setup(A, G, nullptr, S);
  gsync(A, S);
  const int r = run_rounds(A, G, bs, nullptr, S);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = r;
}

}  // namespace lbdd_b200
