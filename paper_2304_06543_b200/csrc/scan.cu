// HBM-bound scans of the |D| x |S| cost matrix.
//
//   row_argmin_kernel     the arrival scan: per demand the cheapest center
//                         (smallest id on ties, row_min_center,
//                         solver.hpp:74-80) + the (cost << 32 | d) sort key
//                         of build_arrival_queue (solver.hpp:84-96), fused
//                         with the positivity / max-cost checks of
//                         validate_instance (core.hpp:297-302) and
//                         augment_with_dummy_center (solver.hpp:199).
//   seg_argmin_kernel     the transfer-graph scan: build_index
//                         (subspace.hpp:233-241) as a segmented argmin of
//                         CM[d][j] - CM[d][home(d)] over the demands of each
//                         home center. Demands are bucketed by home first, a
//                         CTA owns a piece of one bucket and keeps the running
//                         (key, demand) minimum of its columns in registers,
//                         so the matrix is streamed exactly once with 128-bit
//                         loads and the k x k result sees one atomicMin per
//                         (piece, column).
//   objective_kernel      evaluate_objective's assignment-cost sum + loads.
//   generate_costs_kernel synthetic euclidean cost matrix, in place in HBM.
#include <cub/cub.cuh>
#include <cuda.h>  // CUtensorMap (the encoder is fetched through cudaGetDriverEntryPoint)

#include "common.cuh"

namespace lbdd_b200 {

namespace {

__device__ __forceinline__ int4 ld_stream(const int4* p) { return __ldcs(p); }

__device__ __forceinline__ void argmin_step(int32_t v, int32_t idx, int32_t& bv, int32_t& bi) {
  if (v < bv || (v == bv && idx < bi)) {
    bv = v;
    bi = idx;
  }
}

}  // namespace

// One warp per row, lanes stride the row in 16B vectors.
__global__ void __launch_bounds__(256) row_argmin_kernel(const int32_t* __restrict__ cm,
                                                         int64_t pitch, int64_t n, int32_t k,
                                                         int32_t* __restrict__ best_center,
                                                         int64_t* __restrict__ keys,
                                                         int64_t* __restrict__ minmax,
                                                         int64_t id0) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int nv = (k + 3) >> 2;
  int32_t gmin = INT32_MAX, gmax = INT32_MIN;
  for (int64_t row = warp; row < n; row += nwarps) {
    const int4* r4 = reinterpret_cast<const int4*>(cm + row * pitch);
    int32_t bv = INT32_MAX, bi = INT32_MAX;
#pragma unroll 4
    for (int v = lane; v < nv; v += 32) {
      const int4 x = ld_stream(r4 + v);
      const int c = v << 2;
      const int32_t e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (c + i < k) {
          argmin_step(e[i], c + i, bv, bi);
          gmin = min(gmin, e[i]);
          gmax = max(gmax, e[i]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      argmin_step(ov, oi, bv, bi);
    }
    if (lane == 0) {
      best_center[row] = bi;
      keys[row] = static_cast<int64_t>(bv) * (int64_t(1) << 32) + (id0 + row);  // global demand id
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    gmax = max(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  }
  if (lane == 0) {
    atomicMin(reinterpret_cast<long long*>(&minmax[0]), static_cast<long long>(gmin));
    atomicMax(reinterpret_cast<long long*>(&minmax[1]), static_cast<long long>(gmax));
  }
}

// ---- the arrival scan through TMA ----
// Persistent CTAs (one per SM) stream groups of 8 rows through a
// `stages`-deep ring of shared-memory tiles: one elected thread issues
// cp.async.bulk.tensor (TMA, 256-column x 8-row boxes of a 2D tensor map
// over the matrix) that complete_tx on the stage's full mbarrier; warp w
// reduces row w of the group from shared memory (128-bit loads, lanes over
// the columns, shuffle argmin with the smallest id on ties) and releases the
// stage through its empty mbarrier; a ninth warp only produces. Same
// outputs as row_argmin_kernel.
constexpr int kTmaRows = 16;     // rows per group (= consumer warps per CTA)
constexpr int kTmaBoxCols = 256; // columns per TMA box (the box-dim limit)

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, unsigned phase) {
  asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W%=;\n}" ::"r"(smem_addr(b)), "r"(phase) : "memory");
}

template <int NCB>
__global__ void __launch_bounds__(32 * (kTmaRows + 1), 1) row_argmin_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                int64_t n, int32_t k, int stages,
                                                                int32_t* __restrict__ best_center,
                                                                int64_t* __restrict__ keys,
                                                                int64_t* __restrict__ minmax,
                                                                int64_t id0) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  constexpr int kStageInts = NCB * kTmaRows * kTmaBoxCols;
  int32_t* buf = reinterpret_cast<int32_t*>(tsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + static_cast<size_t>(stages) * kStageInts * 4);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ngroups = (n + kTmaRows - 1) / kTmaRows;
  const int64_t mine = ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaRows);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s, int64_t it) {
    const int64_t g = blockIdx.x + it * gridDim.x;
    const unsigned fb = smem_addr(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                 "r"(static_cast<unsigned>(kStageInts * 4)) : "memory");
#pragma unroll
    for (int b = 0; b < NCB; ++b) {
      const unsigned dst = smem_addr(buf + static_cast<size_t>(s) * kStageInts + b * kTmaRows * kTmaBoxCols);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(b * kTmaBoxCols),
          "r"(static_cast<int>(g * kTmaRows)), "r"(fb) : "memory");
    }
  };
  if (warp == kTmaRows) {
    // producer warp: keep every stage of the ring in flight
    if (lane == 0) {
      for (int64_t it = 0; it < mine; ++it) {
        const int s = static_cast<int>(it % stages);
        if (it >= stages) mbar_wait_parity(&empty[s], static_cast<unsigned>(((it / stages) - 1) & 1));
        issue(s, it);
      }
    }
    return;
  }
  int32_t gmin = INT32_MAX, gmax = INT32_MIN;
  for (int64_t it = 0; it < mine; ++it) {
    const int s = static_cast<int>(it % stages);
    const unsigned ph = static_cast<unsigned>((it / stages) & 1);
    mbar_wait_parity(&full[s], ph);
    const int64_t row = (blockIdx.x + it * gridDim.x) * kTmaRows + warp;
    if (row < n) {
      const int32_t* st = buf + static_cast<size_t>(s) * kStageInts + warp * kTmaBoxCols;
      // two independent argmin chains (even / odd 16 B pieces), merged below
      int32_t bv = INT32_MAX, bi = INT32_MAX, bv2 = INT32_MAX, bi2 = INT32_MAX;
      int4 xs[2 * NCB];
#pragma unroll
      for (int b = 0; b < NCB; ++b) {
        const int4* bx = reinterpret_cast<const int4*>(st + b * kTmaRows * kTmaBoxCols);
        xs[2 * b] = bx[lane];
        xs[2 * b + 1] = bx[lane + 32];
      }
#pragma unroll
      for (int q = 0; q < 2 * NCB; ++q) {
        const int c = (q >> 1) * kTmaBoxCols + 4 * (lane + 32 * (q & 1));
        const int32_t e[4] = {xs[q].x, xs[q].y, xs[q].z, xs[q].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (c + i < k) {
            if (q & 1) argmin_step(e[i], c + i, bv2, bi2);
            else argmin_step(e[i], c + i, bv, bi);
            gmin = min(gmin, e[i]);
            gmax = max(gmax, e[i]);
          }
        }
      }
      argmin_step(bv2, bi2, bv, bi);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        argmin_step(ov, oi, bv, bi);
      }
      if (lane == 0) {
        best_center[row] = bi;
        keys[row] = static_cast<int64_t>(bv) * (int64_t(1) << 32) + (id0 + row);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[s])) : "memory");
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    gmax = max(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  }
  if (lane == 0 && gmin != INT32_MAX) {
    atomicMin(reinterpret_cast<long long*>(&minmax[0]), static_cast<long long>(gmin));
    atomicMax(reinterpret_cast<long long*>(&minmax[1]), static_cast<long long>(gmax));
  }
}

// ---- index build: bucket by home, then segmented argmin per piece ----

__global__ void home_histogram_kernel(const int32_t* __restrict__ home, int64_t r0, int64_t r1,
                                      int32_t k, int32_t* __restrict__ cnt,
                                      int32_t* __restrict__ bad) {
  for (int64_t d = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; d < r1;
       d += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t h = home[d];
    if (h < 0) continue;
    if (h >= k) { atomicExch(bad, 1); continue; }
    atomicAdd(&cnt[h], 1);
  }
}

__global__ void home_scatter_kernel(const int32_t* __restrict__ home, int64_t r0, int64_t r1,
                                    int32_t k, const int32_t* __restrict__ off,
                                    int32_t* __restrict__ cursor, int32_t* __restrict__ sorted) {
  for (int64_t d = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; d < r1;
       d += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t h = home[d];
    if (h < 0 || h >= k) continue;
    sorted[off[h] + atomicAdd(&cursor[h], 1)] = static_cast<int32_t>(d);
  }
}

// pieces per bucket: ceil(cnt / R)
__global__ void piece_count_kernel(const int32_t* __restrict__ cnt, int32_t k, int32_t R,
                                   int32_t* __restrict__ pc) {
  for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < k; h += gridDim.x * blockDim.x) {
    pc[h] = (cnt[h] + R - 1) / R;
  }
}

// Arrival-ordered centers (asral): arr_s[a] = best_center[d(a)], so the
// engine reads an arrival's (cost, demand) and center without a dependent
// gather and can prefetch them ahead.
__global__ void arrival_centers_kernel(const int64_t* __restrict__ keys, const int32_t* __restrict__ best,
                                       int64_t n, int32_t* __restrict__ arr_s) {
  for (int64_t a = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; a < n;
       a += static_cast<int64_t>(gridDim.x) * blockDim.x)
    arr_s[a] = best[keys[a] & 0xffffffffLL];
}

__global__ void fill_i64_kernel(int64_t* p, int64_t count, int64_t v) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    p[i] = v;
  }
}

template <int V, int R>
__global__ void __launch_bounds__(1024) seg_argmin_kernel(
    const int32_t* __restrict__ cm, int64_t pitch, int32_t k, const int32_t* __restrict__ sorted,
    const int32_t* __restrict__ off, const int32_t* __restrict__ cnt,
    const int32_t* __restrict__ poff, int64_t* __restrict__ M, int32_t id_offset) {
  __shared__ int32_t s_rows[R];
  const int npieces = poff[k];  // total pieces, produced on the device
  __shared__ int32_t s_hv[R];
  const int nv = (k + 3) >> 2;
  for (int p = blockIdx.x; p < npieces; p += gridDim.x) {
    // bucket of piece p: last h with poff[h] <= p (poff exclusive scan, k+1)
    int lo = 0, hi = k;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (poff[mid] <= p) lo = mid; else hi = mid;
    }
    const int h = lo;
    const int first = (p - poff[h]) * R;
    const int rows = min(R, cnt[h] - first);
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      const int32_t d = sorted[off[h] + first + i];
      s_rows[i] = d;
      s_hv[i] = cm[static_cast<int64_t>(d) * pitch + h];
    }
    __syncthreads();
    __syncthreads();
    int64_t m[V][4];
#pragma unroll
    for (int t = 0; t < V; ++t)
#pragma unroll
      for (int c = 0; c < 4; ++c) m[t][c] = kEmpty;
#pragma unroll 2
    for (int i = 0; i < rows; ++i) {
      const int32_t d = s_rows[i];
      const int32_t hv = s_hv[i];
      const int4* r4 = reinterpret_cast<const int4*>(cm + static_cast<int64_t>(d) * pitch);
      const int32_t gid = d + id_offset;  // global demand id in the packed word
#pragma unroll
      for (int t = 0; t < V; ++t) {
        const int v = threadIdx.x + t * blockDim.x;
        if (v < nv) {
          const int4 x = ld_stream(r4 + v);
          const int64_t p0 = pack_transfer(x.x - hv, gid);
          const int64_t p1 = pack_transfer(x.y - hv, gid);
          const int64_t p2 = pack_transfer(x.z - hv, gid);
          const int64_t p3 = pack_transfer(x.w - hv, gid);
          m[t][0] = p0 < m[t][0] ? p0 : m[t][0];
          m[t][1] = p1 < m[t][1] ? p1 : m[t][1];
          m[t][2] = p2 < m[t][2] ? p2 : m[t][2];
          m[t][3] = p3 < m[t][3] ? p3 : m[t][3];
        }
      }
    }
    int64_t* Mh = M + static_cast<int64_t>(h) * k;
#pragma unroll
    for (int t = 0; t < V; ++t) {
      const int v = threadIdx.x + t * blockDim.x;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = v * 4 + c;
        if (v < nv && j < k && j != h && m[t][c] != kEmpty) {
          atomicMin(reinterpret_cast<long long*>(&Mh[j]), static_cast<long long>(m[t][c]));
        }
      }
    }
  }
}

// assignment-cost sum + load histogram (evaluate_partial_objective,
// core.hpp:216-233; penalties are added on the host from the loads).
__global__ void objective_kernel(const RowTable rows, int64_t n,
                                 int32_t k, const int32_t* __restrict__ home,
                                 unsigned long long* __restrict__ sum,
                                 unsigned long long* __restrict__ load,
                                 int32_t* __restrict__ unassigned) {
  unsigned long long local = 0;
  int missing = 0;
  for (int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; d < n;
       d += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t h = home[d];
    if (h < 0 || h >= k) { ++missing; continue; }
    local += static_cast<unsigned long long>(row_of(rows, d)[h]);
    atomicAdd(&load[h], 1ull);
  }
  using WarpReduce = cub::WarpReduce<unsigned long long>;
  __shared__ typename WarpReduce::TempStorage tmp[32];
  const unsigned long long w = WarpReduce(tmp[threadIdx.x >> 5]).Sum(local);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(sum, w);
  if (missing) atomicAdd(unassigned, missing);
}

namespace {
// splitmix64 finaliser; synth_instances.py mix()
__device__ __forceinline__ uint64_t synth_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
}  // namespace

// Synthetic euclidean costs, spec "lbdd-synth-v2" (synth_instances.py, bit
// for bit): integer points on a 10000 x 10000 grid from a counter-based
// stream, cost = max(1, floor(sqrt(dx^2 + dy^2) / 10 + 0.5)). The double
// sqrt and division are IEEE correctly rounded here and in numpy, so the
// host generator and this kernel agree exactly. Any row range can be
// generated independently (sharded generation). base[t] = mix(seed ^ t).
__global__ void generate_costs_kernel(int32_t* __restrict__ cm, int64_t pitch, int64_t row0,
                                      int64_t rows, int32_t k, ulonglong4 base) {
  const int nv = static_cast<int>(pitch >> 2);
  const int64_t total = rows * nv;
  constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / nv;
    const int v = static_cast<int>(i - r * nv);
    const uint64_t d1 = static_cast<uint64_t>(row0 + r) + 1;
    const int64_t dx = static_cast<int64_t>(synth_mix(base.x + d1 * kGold) % 10000ull);
    const int64_t dy = static_cast<int64_t>(synth_mix(base.y + d1 * kGold) % 10000ull);
    int32_t out[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = v * 4 + c;
      if (j < k) {
        const uint64_t j1 = static_cast<uint64_t>(j) + 1;
        const int64_t ex = dx - static_cast<int64_t>(synth_mix(base.z + j1 * kGold) % 10000ull);
        const int64_t ey = dy - static_cast<int64_t>(synth_mix(base.w + j1 * kGold) % 10000ull);
        const double q = static_cast<double>(ex * ex + ey * ey);
        const double c2 = floor(__dadd_rn(__ddiv_rn(__dsqrt_rn(q), 10.0), 0.5));
        out[c] = c2 < 1.0 ? 1 : static_cast<int32_t>(c2);
      } else {
        out[c] = INT32_MAX;  // row padding, never read as a cost
      }
    }
    reinterpret_cast<int4*>(cm + r * pitch)[v] = make_int4(out[0], out[1], out[2], out[3]);
  }
}

// augment_with_dummy_center (solver.hpp:194-217): copy the matrix into a
// k+1 column layout whose last column is max(CM) + 1.
__global__ void augment_kernel(const int32_t* src, int64_t spitch, int32_t* dst, int64_t dpitch,
                               int64_t n, int32_t k, int32_t extra) {
  const int64_t total = n * dpitch;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / dpitch;
    const int64_t c = i - r * dpitch;
    dst[i] = c < k ? src[r * spitch + c] : (c == k ? extra : INT32_MAX);
  }
}

// explicit instantiations used by capi.cu
template __global__ void seg_argmin_kernel<1, 256>(const int32_t*, int64_t, int32_t, const int32_t*,
                                                   const int32_t*, const int32_t*, const int32_t*,
                                                   int64_t*, int32_t);
template __global__ void seg_argmin_kernel<2, 256>(const int32_t*, int64_t, int32_t, const int32_t*,
                                                   const int32_t*, const int32_t*, const int32_t*,
                                                   int64_t*, int32_t);
template __global__ void seg_argmin_kernel<4, 256>(const int32_t*, int64_t, int32_t, const int32_t*,
                                                   const int32_t*, const int32_t*, const int32_t*,
                                                   int64_t*, int32_t);
template __global__ void seg_argmin_kernel<8, 256>(const int32_t*, int64_t, int32_t, const int32_t*,
                                                   const int32_t*, const int32_t*, const int32_t*,
                                                   int64_t*, int32_t);

}  // namespace lbdd_b200
