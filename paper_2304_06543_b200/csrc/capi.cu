// Host side of the C ABI (include/lbdd_b200.h): validation, device memory,
// launches, and the report — the reference's solver entry points
// (solver.hpp:133-301) re-expressed over the device engine. All arithmetic
// on the report path is exact 64-bit with the reference's overflow checks
// (core.hpp:25-39).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <memory>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "lbdd_b200.h"

// Single translation unit: the kernels are included, not linked.
#include "cluster.cu"
#include "engine.cu"
#include "scan.cu"

using namespace lbdd_b200;

namespace capi_detail {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};  // kernels of this library launched

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void raise(int code, const std::string& m) { throw Error(code, m); }

#define CUDA_OK(expr)                                                                   \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess) {                                                           \
      raise(LBDD_ERR_CUDA, std::string("lbdd_b200: ") + #expr + ": " + cudaGetErrorString(e__)); \
    }                                                                                   \
  } while (0)

template <typename F>
lbdd_status guarded(F&& f) {
  try {
    f();
    return LBDD_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<lbdd_status>(e.code);
  } catch (const std::exception& e) {
    g_err = e.what();
    return LBDD_ERR_RUNTIME;
  }
}

int64_t checked_add(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_add_overflow(a, b, &r)) raise(LBDD_ERR_OVERFLOW, "lbdd: cost accumulator overflow");
  return r;
}
int64_t checked_mul(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_mul_overflow(a, b, &r)) raise(LBDD_ERR_OVERFLOW, "lbdd: cost accumulator overflow");
  return r;
}

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  void ensure(size_t c) {
    if (c <= count && p) return;
    release();
    CUDA_OK(cudaMalloc(&p, std::max<size_t>(c, 1) * sizeof(T)));
    count = c;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    count = 0;
  }
};

constexpr int kEngineThreads = 512;
constexpr int kPieceRows = 256;
constexpr int kMaxEngineK = 7000;      // shared-memory bound of the engine CTA
constexpr int64_t kMaxPenalty = int64_t(1) << 40;  // packing bound (common.cuh)

}  // namespace capi_detail
using namespace capi_detail;

// ---------------------------------------------------------------------------
// instance
// ---------------------------------------------------------------------------

struct lbdd_b200_instance {
  int device = 0;
  int64_t n = 0, k = 0, pitch = 0;
  int32_t* d_cm = nullptr;   // the matrix (sharded: this rank's own row block)
  bool owns_cm = false;
  // sharded instance (lbdd_b200_instance_create_sharded): the row table over
  // every rank's block; nshards == 1 for an ordinary instance
  RowTable rt{};
  int32_t nshards = 1, my_shard = 0;
  int64_t shard_rows = 0, local_rows = 0;
  bool gathered = false;  // keys/best_center hold the gathered arrival scan
  RowTable rows() const {
    if (nshards > 1) return rt;
    RowTable t{};
    t.shard[0] = d_cm;
    t.pitch = pitch;
    t.shard_rows = static_cast<int32_t>(std::min<int64_t>(n, INT32_MAX));
    t.nshards = 1;
    return t;
  }
  std::vector<int64_t> cap, off, par;
  std::vector<int32_t> fam;
  int64_t* d_cap = nullptr;
  int32_t* d_fam = nullptr;
  int64_t* d_off = nullptr;
  int64_t* d_par = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 0;

  // scan results
  bool scanned = false;
  int64_t min_cost = 0, max_cost = 0;
  DevBuf<int32_t> best_center, arr_s;
  DevBuf<int64_t> keys, keys_sorted, minmax;
  DevBuf<unsigned char> cub_tmp;

  // engine state
  DevBuf<int32_t> home, order, rowslot, src_list, inv_cnt, inv_cols, single_out, rowver;
  DevBuf<int32_t> P[2][2];
  DevBuf<int64_t> D[2][2], B[2][3];
  DevBuf<int64_t> load, dummies, M, colW, single_gain, pi;
  DevBuf<int32_t> dirty, log_d, log_to, log_n, add_ids, add_cnt;
  DevBuf<int64_t> MX;
  DevBuf<uint8_t> LN;
  DevBuf<int16_t> ktile;  // global key tile (tile_mode 2)
  int cluster_size = 0;  // chosen once per instance
  // CUDA-event kernel times of the current solve (reported per solve)
  int64_t engine_ns = 0, engine_launches = 0, row_scan_ns = 0;
  cudaEvent_t kev[2] = {nullptr, nullptr};
  float time_since(cudaEvent_t start) {  // kev[1] recorded + synced by the caller
    float ms = 0;
    cudaEventElapsedTime(&ms, start, kev[1]);
    return ms;
  }
  DevBuf<EngineCtl> ctl;
  DevBuf<GridBar> bar;
  DevBuf<PathEdge> path;
  DevBuf<uint8_t> dumflag;
  // index build scratch
  DevBuf<int32_t> ib_cnt, ib_off, ib_cursor, ib_sorted, ib_pc, ib_poff, ib_bad;
  DevBuf<unsigned long long> obj_acc;
  DevBuf<int32_t> obj_missing;

  ~lbdd_b200_instance() {
    cudaSetDevice(device);
    if (owns_cm && d_cm) cudaFree(d_cm);
    for (void* p : {static_cast<void*>(d_cap), static_cast<void*>(d_fam), static_cast<void*>(d_off),
                    static_cast<void*>(d_par)}) {
      if (p) cudaFree(p);
    }
    best_center.release(); arr_s.release(); keys.release(); keys_sorted.release(); minmax.release();
    cub_tmp.release(); home.release(); order.release(); rowslot.release(); src_list.release();
    inv_cnt.release(); inv_cols.release();
    for (int s = 0; s < 2; ++s) {
      for (int i = 0; i < 2; ++i) { P[s][i].release(); D[s][i].release(); }
      for (int i = 0; i < 3; ++i) B[s][i].release();
    }
    single_out.release(); rowver.release(); load.release(); dummies.release(); M.release();
    pi.release(); dirty.release(); log_d.release(); log_to.release(); log_n.release();
    add_ids.release(); add_cnt.release();
    MX.release(); LN.release(); ktile.release();
    colW.release();
    single_gain.release(); ctl.release(); bar.release(); path.release(); dumflag.release();
    ib_cnt.release(); ib_off.release(); ib_cursor.release(); ib_sorted.release();
    ib_pc.release(); ib_poff.release(); ib_bad.release(); obj_acc.release();
    obj_missing.release();
    if (kev[0]) cudaEventDestroy(kev[0]);
    if (kev[1]) cudaEventDestroy(kev[1]);
    if (stream) cudaStreamDestroy(stream);
  }

  int64_t pen_len(int64_t s) const { return off[s + 1] - off[s]; }

  // PenaltySpec::at / total (core.hpp:60-95), host side, checked.
  int64_t pen_at(int64_t s, int64_t j) const {
    const int64_t* p = par.data() + off[s];
    switch (fam[s]) {
      case LBDD_PENALTY_CONSTANT: return p[0];
      case LBDD_PENALTY_LINEAR: return checked_add(p[0], checked_mul(p[1], j - 1));
      default: return p[std::min(j, pen_len(s)) - 1];
    }
  }
  int64_t pen_total(int64_t s, int64_t m) const {
    if (m <= 0) return 0;
    const int64_t* p = par.data() + off[s];
    switch (fam[s]) {
      case LBDD_PENALTY_CONSTANT: return checked_mul(p[0], m);
      case LBDD_PENALTY_LINEAR: {
        const int64_t tri = checked_mul(m, m - 1) / 2;
        return checked_add(checked_mul(p[0], m), checked_mul(p[1], tri));
      }
      default: {
        int64_t sum = 0;
        for (int64_t j = 1; j <= m; ++j) sum = checked_add(sum, pen_at(s, j));
        return sum;
      }
    }
  }
  int64_t total_capacity() const {
    int64_t t = 0;
    for (auto c : cap) t += c;
    return t;
  }
};

namespace capi_detail {

void upload_centers(lbdd_b200_instance* I, const lbdd_instance_desc* d) {
  const int64_t k = d->k;
  I->cap.assign(d->capacity, d->capacity + k);
  I->fam.assign(d->penalty_family, d->penalty_family + k);
  I->off.assign(d->penalty_offset, d->penalty_offset + k + 1);
  const int64_t np = k > 0 ? I->off[k] : 0;
  I->par.assign(d->penalty_params, d->penalty_params + np);
  CUDA_OK(cudaMalloc(&I->d_cap, sizeof(int64_t) * std::max<int64_t>(k, 1)));
  CUDA_OK(cudaMalloc(&I->d_fam, sizeof(int32_t) * std::max<int64_t>(k, 1)));
  CUDA_OK(cudaMalloc(&I->d_off, sizeof(int64_t) * (k + 1)));
  CUDA_OK(cudaMalloc(&I->d_par, sizeof(int64_t) * std::max<int64_t>(np, 1)));
  if (k > 0) {
    CUDA_OK(cudaMemcpy(I->d_cap, I->cap.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(I->d_fam, I->fam.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice));
  }
  CUDA_OK(cudaMemcpy(I->d_off, I->off.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice));
  if (np > 0) CUDA_OK(cudaMemcpy(I->d_par, I->par.data(), sizeof(int64_t) * np, cudaMemcpyHostToDevice));
}

lbdd_b200_instance* new_instance(int device, int64_t n, int64_t k) {
  auto* I = new lbdd_b200_instance();
  I->device = device;
  I->n = n;
  I->k = k;
  I->pitch = ((k + 3) / 4) * 4;
  CUDA_OK(cudaSetDevice(device));
  CUDA_OK(cudaStreamCreateWithFlags(&I->stream, cudaStreamNonBlocking));
  CUDA_OK(cudaDeviceGetAttribute(&I->num_sms, cudaDevAttrMultiProcessorCount, device));
  return I;
}

// entry points that scan the whole matrix through d_cm take ordinary instances
void require_unsharded(const lbdd_b200_instance* I) {
  if (I->nshards > 1)
    raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: not supported on a sharded instance");
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16)));
}

// validate_instance (core.hpp:250-305), center part; the matrix part runs
// on the device inside the arrival scan.
void validate_centers(const lbdd_b200_instance* I) {
  auto fail = [](const std::string& m) {
    raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: invalid instance: " + m);
  };
  if (I->k < 1) fail("instance has no service centers (k < 1)");
  if (I->n < 1) fail("instance has no demand units (n < 1)");
  for (int64_t s = 0; s < I->k; ++s) {
    const std::string tag = "center " + std::to_string(s) + ": ";
    const int64_t np = I->pen_len(s);
    const int64_t* p = I->par.data() + I->off[s];
    if (I->cap[s] < 0) fail(tag + "negative capacity");
    switch (I->fam[s]) {
      case LBDD_PENALTY_CONSTANT:
        if (np != 1) fail(tag + "constant penalty takes one parameter");
        else if (p[0] <= 0) fail(tag + "penalty not positive");
        break;
      case LBDD_PENALTY_LINEAR:
        if (np != 2) fail(tag + "linear penalty takes two parameters");
        else if (p[0] <= 0 || p[1] < 0) fail(tag + "penalty not positive");
        break;
      case LBDD_PENALTY_TABLE:
        if (np == 0) {
          fail(tag + "empty penalty table");
        } else {
          if (p[0] <= 0) fail(tag + "penalty not positive");
          for (int64_t i = 1; i < np; ++i)
            if (p[i] < p[i - 1]) fail(tag + "penalty not monotone");
        }
        break;
      default: fail(tag + "bad penalty family");
    }
  }
}

// Device-range guards (not reference behaviour: the reference is int64
// throughout; the device packs (cost, source) into one int64).
void check_device_range(const lbdd_b200_instance* I) {
  if (I->k > kMaxEngineK)
    raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: engine supports k <= " + std::to_string(kMaxEngineK));
  if (I->n >= INT32_MAX) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: n exceeds int32 demand ids");
  for (int64_t s = 0; s < I->k; ++s) {
    const int64_t* p = I->par.data() + I->off[s];
    int64_t qmax = 0;
    switch (I->fam[s]) {
      case LBDD_PENALTY_CONSTANT: qmax = p[0]; break;
      case LBDD_PENALTY_LINEAR: {
        int64_t m, r;
        if (__builtin_mul_overflow(p[1], I->n, &m) || __builtin_add_overflow(p[0], m, &r)) r = INT64_MAX;
        qmax = r;
        break;
      }
      default: qmax = p[I->pen_len(s) - 1]; break;
    }
    if (qmax > kMaxPenalty)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: penalty exceeds the device range (2^40)");
  }
}

// Arrival scan + sort (build_arrival_queue, solver.hpp:89-96), with the
// matrix half of validate_instance. Returns device time in ns.
void ensure_kernel_events(lbdd_b200_instance* I) {
  if (I->kev[0] == nullptr) {
    CUDA_OK(cudaEventCreate(&I->kev[0]));
    CUDA_OK(cudaEventCreate(&I->kev[1]));
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr)
      raise(LBDD_ERR_CUDA, "lbdd_b200: cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// The arrival scan over `rows` rows at `cm` (row_min_center + the keys of
// build_arrival_queue, fused with the cost-range check): TMA-staged kernel
// when a row spans at most 5 boxes of 256 columns (k <= 1280), else the
// 128-bit streaming kernel.
void launch_row_argmin(lbdd_b200_instance* I, const int32_t* cm, int64_t rows, int64_t id0,
                       int32_t* best, int64_t* keys, int64_t* minmax) {
  const int ncb = static_cast<int>((I->pitch + kTmaBoxCols - 1) / kTmaBoxCols);
  g_launches++;
  // two or more stages must fit the ring (16-row groups: 16 KB per box
  // column); wider rows stream well with plain 128-bit loads (long rows per
  // warp), so they keep the streaming kernel
  if (ncb <= 5 && rows > 0) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(I->pitch), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(I->pitch) * 4};
    const cuuint32_t box[2] = {kTmaBoxCols, kTmaRows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_tiled()(&tm, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int32_t*>(cm),
                                      dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(LBDD_ERR_CUDA, "lbdd_b200: tensor map encode failed");
    const size_t stage = static_cast<size_t>(ncb) * kTmaRows * kTmaBoxCols * 4;
    const int stages = static_cast<int>(std::min<size_t>(6, (210 * 1024) / stage));
    const size_t smem = stages * stage + 16 * stages + 1024;
    const int grid = static_cast<int>(std::min<int64_t>(I->num_sms, (rows + kTmaRows - 1) / kTmaRows));
#define LAUNCH_TMA(NC)                                                                              \
  CUDA_OK(cudaFuncSetAttribute(row_argmin_tma_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               static_cast<int>(smem)));                                             \
  row_argmin_tma_kernel<NC><<<grid, 32 * (kTmaRows + 1), smem, I->stream>>>(                      \
      tm, rows, static_cast<int32_t>(I->k),                                                         \
                                                            stages, best, keys, minmax, id0)
    switch (ncb) {
      case 1: LAUNCH_TMA(1); break;
      case 2: LAUNCH_TMA(2); break;
      case 3: LAUNCH_TMA(3); break;
      case 4: LAUNCH_TMA(4); break;
      case 5: LAUNCH_TMA(5); break;
      default: LAUNCH_TMA(5); break;
    }
#undef LAUNCH_TMA
  } else {
    const int blocks = static_cast<int>(std::min<int64_t>((rows + 7) / 8, I->num_sms * 8));
    row_argmin_kernel<<<std::max(blocks, 1), 256, 0, I->stream>>>(
        cm, I->pitch, rows, static_cast<int32_t>(I->k), best, keys, minmax, id0);
  }
  CUDA_OK(cudaGetLastError());
}

int64_t arrival_scan(lbdd_b200_instance* I, bool validate_matrix) {
  const int64_t n = I->n;
  if (I->nshards > 1 && !I->gathered)
    raise(LBDD_ERR_INVALID_ARGUMENT,
          "lbdd_b200: a sharded instance solves through lbdd_b200_solve_sharded");
  I->best_center.ensure(n);
  I->keys.ensure(n);
  I->keys_sorted.ensure(n);
  I->minmax.ensure(2);
  const int64_t init[2] = {INT64_MAX, INT64_MIN};
  cudaEvent_t e0, e1;
  CUDA_OK(cudaEventCreate(&e0));
  CUDA_OK(cudaEventCreate(&e1));
  CUDA_OK(cudaEventRecord(e0, I->stream));
  if (!I->gathered) {  // sharded: keys, best_center, min/max gathered by the caller
    CUDA_OK(cudaMemcpyAsync(I->minmax.p, init, sizeof(init), cudaMemcpyHostToDevice, I->stream));
    ensure_kernel_events(I);
    CUDA_OK(cudaEventRecord(I->kev[0], I->stream));
    launch_row_argmin(I, I->d_cm, n, 0, I->best_center.p, I->keys.p, I->minmax.p);
    CUDA_OK(cudaEventRecord(I->kev[1], I->stream));
    int64_t mm[2];
    CUDA_OK(cudaMemcpyAsync(mm, I->minmax.p, sizeof(mm), cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaStreamSynchronize(I->stream));
    I->row_scan_ns += static_cast<int64_t>(static_cast<double>(I->time_since(I->kev[0])) * 1e6);
    I->min_cost = mm[0];
    I->max_cost = mm[1];
  }
  if (validate_matrix && I->min_cost <= 0)
    raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: invalid instance: non-positive cost in cost matrix");
  // sort by (cost, demand): key bits = 32 (demand) + bits(max cost)
  int end_bit = 32;
  while (end_bit < 63 && (int64_t(1) << (end_bit - 32)) <= I->max_cost) ++end_bit;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, reinterpret_cast<uint64_t*>(I->keys.p),
                                 reinterpret_cast<uint64_t*>(I->keys_sorted.p),
                                 static_cast<int>(n), 0, end_bit, I->stream);
  I->cub_tmp.ensure(tmp_bytes);
  cub::DeviceRadixSort::SortKeys(I->cub_tmp.p, tmp_bytes, reinterpret_cast<uint64_t*>(I->keys.p),
                                 reinterpret_cast<uint64_t*>(I->keys_sorted.p),
                                 static_cast<int>(n), 0, end_bit, I->stream);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaEventRecord(e1, I->stream));
  CUDA_OK(cudaEventSynchronize(e1));
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  I->scanned = true;
  return static_cast<int64_t>(ms * 1e6);
}

void fill64(lbdd_b200_instance* I, int64_t* p, int64_t count, int64_t v) {
  g_launches++;
  fill_i64_kernel<<<grid_for(count), 256, 0, I->stream>>>(p, count, v);
  CUDA_OK(cudaGetLastError());
}

// build_index over the rows [r0, r1) of a device allotment into d_M (k*k,
// pre-filled with kEmpty by the caller). Phase 1 buckets the demands by
// home (histogram, scan, scatter, pieces); phase 2 is the matrix scan.
void build_index_prepare(lbdd_b200_instance* I, const int32_t* d_home, int64_t r0, int64_t r1,
                         cudaStream_t st, bool check) {
  const int32_t k = static_cast<int32_t>(I->k);
  const int64_t n = I->n;
  I->ib_cnt.ensure(k + 1);
  I->ib_off.ensure(k + 1);
  I->ib_cursor.ensure(k + 1);
  I->ib_pc.ensure(k + 1);
  I->ib_poff.ensure(k + 1);
  I->ib_sorted.ensure(std::max<int64_t>(n, 1));
  I->ib_bad.ensure(1);
  CUDA_OK(cudaMemsetAsync(I->ib_cnt.p, 0, sizeof(int32_t) * (k + 1), st));
  CUDA_OK(cudaMemsetAsync(I->ib_cursor.p, 0, sizeof(int32_t) * (k + 1), st));
  CUDA_OK(cudaMemsetAsync(I->ib_pc.p, 0, sizeof(int32_t) * (k + 1), st));
  CUDA_OK(cudaMemsetAsync(I->ib_bad.p, 0, sizeof(int32_t), st));
  if (r1 > r0) {
    g_launches++;
    home_histogram_kernel<<<grid_for(r1 - r0), 256, 0, st>>>(d_home, r0, r1, k, I->ib_cnt.p, I->ib_bad.p);
  }
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, I->ib_cnt.p, I->ib_off.p, k + 1, st);
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, I->ib_pc.p, I->ib_poff.p, k + 1, st);
  I->cub_tmp.ensure(std::max(tb, tb2));
  cub::DeviceScan::ExclusiveSum(I->cub_tmp.p, tb, I->ib_cnt.p, I->ib_off.p, k + 1, st);
  if (r1 > r0) {
    g_launches++;
    home_scatter_kernel<<<grid_for(r1 - r0), 256, 0, st>>>(d_home, r0, r1, k, I->ib_off.p,
                                                            I->ib_cursor.p, I->ib_sorted.p);
  }
  g_launches++;
  piece_count_kernel<<<grid_for(k), 256, 0, st>>>(I->ib_cnt.p, k, kPieceRows, I->ib_pc.p);
  cub::DeviceScan::ExclusiveSum(I->cub_tmp.p, tb2, I->ib_pc.p, I->ib_poff.p, k + 1, st);
  CUDA_OK(cudaGetLastError());
  if (check) {
    int32_t bad = 0;
    CUDA_OK(cudaMemcpyAsync(&bad, I->ib_bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (bad) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: allotment shape mismatch");
  }
}

void build_index_scan(lbdd_b200_instance* I, int64_t rows, int64_t* d_M, cudaStream_t st,
                      int32_t id_offset = 0) {
  const int32_t k = static_cast<int32_t>(I->k);
  const int nv = static_cast<int>((k + 3) / 4);
  int V = 1;
  while (V < 8 && (nv + V - 1) / V > 1024) V *= 2;
  int threads = (nv + V - 1) / V;
  threads = ((threads + 31) / 32) * 32;
  const int64_t max_pieces = rows / kPieceRows + k + 1;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_pieces, I->num_sms * 16)));
#define LAUNCH_SEG(VV)                                                                  \
  g_launches++;                                                                         \
  seg_argmin_kernel<VV, kPieceRows><<<blocks, threads, 0, st>>>(                        \
      I->d_cm, I->pitch, k, I->ib_sorted.p, I->ib_off.p, I->ib_cnt.p, I->ib_poff.p, d_M, id_offset)
  switch (V) {
    case 1: LAUNCH_SEG(1); break;
    case 2: LAUNCH_SEG(2); break;
    case 4: LAUNCH_SEG(4); break;
    default: LAUNCH_SEG(8); break;
  }
#undef LAUNCH_SEG
  CUDA_OK(cudaGetLastError());
}

void build_index_device(lbdd_b200_instance* I, const int32_t* d_home, int64_t r0, int64_t r1,
                        int64_t* d_M, cudaStream_t st) {
  build_index_prepare(I, d_home, r0, r1, st, true);
  build_index_scan(I, r1 - r0, d_M, st);
}

// Assignment-cost sum + loads on the device, penalties on the host
// (evaluate_partial_objective, core.hpp:216-233). Returns objective; fills
// `loads` (k) and `missing`.
int64_t device_objective(lbdd_b200_instance* I, const int32_t* d_home, std::vector<int64_t>& loads,
                         int32_t* missing) {
  const int64_t k = I->k;
  I->obj_acc.ensure(k + 1);
  I->obj_missing.ensure(1);
  CUDA_OK(cudaMemsetAsync(I->obj_acc.p, 0, sizeof(unsigned long long) * (k + 1), I->stream));
  CUDA_OK(cudaMemsetAsync(I->obj_missing.p, 0, sizeof(int32_t), I->stream));
  g_launches++;
  objective_kernel<<<grid_for(I->n), 256, 0, I->stream>>>(
      I->rows(), I->n, static_cast<int32_t>(k), d_home, I->obj_acc.p, I->obj_acc.p + 1,
      I->obj_missing.p);
  CUDA_OK(cudaGetLastError());
  std::vector<unsigned long long> acc(k + 1);
  CUDA_OK(cudaMemcpyAsync(acc.data(), I->obj_acc.p, sizeof(unsigned long long) * (k + 1),
                          cudaMemcpyDeviceToHost, I->stream));
  CUDA_OK(cudaMemcpyAsync(missing, I->obj_missing.p, sizeof(int32_t), cudaMemcpyDeviceToHost, I->stream));
  CUDA_OK(cudaStreamSynchronize(I->stream));
  loads.assign(k, 0);
  int64_t total = static_cast<int64_t>(acc[0]);
  for (int64_t s = 0; s < k; ++s) {
    loads[s] = static_cast<int64_t>(acc[s + 1]);
    total = checked_add(total, I->pen_total(s, loads[s] - I->cap[s]));
  }
  return total;
}

// engine workspace + launch geometry
struct Launch {
  int grid = 1;
  int block = kEngineThreads;
  size_t smem = 0;
  bool tile = false;
};

int geo_chunk(int rows, int ncols, int grid, int block) {
  const int ncoltiles = (ncols + block - 1) / block;
  int want = grid / ncoltiles;
  if (want < 1) want = 1;
  int chunk = (rows + want - 1) / want;
  return chunk < 1 ? 1 : chunk;
}

// must match carve_smem (engine.cu)
size_t smem_bytes(int k, int maxchunk, int block, bool tile) {
  return sizeof(int64_t) * maxchunk + sizeof(int64_t) * 4 + sizeof(PathEdge) * (k + 1) +
         3 * sizeof(int32_t) * (k + 2) + 2 * sizeof(int32_t) * block + sizeof(int32_t) * 8 +
         sizeof(int64_t) * maxchunk + sizeof(int32_t) * maxchunk +
         (tile ? sizeof(int32_t) * static_cast<size_t>(maxchunk) * block : 0) +
         2 * static_cast<size_t>(maxchunk) + 16;
}

constexpr size_t kSmemBudget = 200 * 1024;

template <typename K>
Launch plan_launch(lbdd_b200_instance* I, K kernel, int rows, int ncols, bool allow_tile) {
  Launch L;
  L.block = std::min(kEngineThreads, std::max(128, ((ncols + 31) / 32) * 32));
  int64_t want = (static_cast<int64_t>(rows) * ncols + 4095) / 4096;
  want = std::max<int64_t>(1, std::min<int64_t>(want, I->num_sms));
  L.grid = static_cast<int>(want);
  for (;;) {
    const int chunk = geo_chunk(rows, ncols, L.grid, L.block);
    L.tile = allow_tile && smem_bytes(rows, chunk, L.block, true) <= kSmemBudget;
    L.smem = smem_bytes(rows, chunk, L.block, L.tile);
    CUDA_OK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(L.smem)));
    int per_sm = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, L.block, L.smem));
    if (per_sm >= 1 && L.grid <= per_sm * I->num_sms) return L;
    if (per_sm < 1) raise(LBDD_ERR_CUDA, "lbdd_b200: engine kernel does not fit on an SM");
    L.grid = per_sm * I->num_sms;
  }
}

void ensure_engine(lbdd_b200_instance* I, int64_t k_nodes) {
  const int64_t k = I->k;
  const int64_t nodes = std::max<int64_t>(k + 1, k_nodes);
  I->home.ensure(I->n);
  I->load.ensure(k + 1);
  I->M.ensure(k * k);
  for (int s = 0; s < 2; ++s) {
    for (int i = 0; i < 2; ++i) { I->D[s][i].ensure(nodes); I->P[s][i].ensure(nodes); }
    for (int i = 0; i < 3; ++i) I->B[s][i].ensure(nodes);
  }
  I->colW.ensure(k + 1);
  I->path.ensure(static_cast<size_t>(cl::kMaxCS) * (k + 1));  // one path copy per cluster CTA
  I->inv_cnt.ensure(k + 2);
  I->inv_cols.ensure((k + 1) * k);
  I->rowslot.ensure(k + 1);
  I->src_list.ensure(k + 1);
  I->ctl.ensure(1);
  I->bar.ensure(1);
  I->dumflag.ensure(k + 1);
  I->dummies.ensure(k + 1);
  I->single_out.ensure(2);
  I->single_gain.ensure(1);
  I->rowver.ensure(k + 1);
  I->pi.ensure(k + 1);
  I->dirty.ensure(static_cast<size_t>(16) * (2 * k + 4));
}

EngineArgs engine_args(lbdd_b200_instance* I) {
  EngineArgs A;
  std::memset(&A, 0, sizeof(A));
  A.rows = I->rows();
  A.cm = I->d_cm;
  A.pitch = I->pitch;
  A.n = static_cast<int32_t>(I->n);
  A.k = static_cast<int32_t>(I->k);
  A.cap = I->d_cap;
  A.pfam = I->d_fam;
  A.poff = I->d_off;
  A.ppar = I->d_par;
  A.home = I->home.p;
  A.load = I->load.p;
  A.M = I->M.p;
  for (int s = 0; s < 2; ++s) {
    for (int i = 0; i < 2; ++i) { A.D[s][i] = I->D[s][i].p; A.P[s][i] = I->P[s][i].p; }
    for (int i = 0; i < 3; ++i) A.B[s][i] = I->B[s][i].p;
  }
  A.colW = I->colW.p;
  A.path = I->path.p;
  A.inv_cnt = I->inv_cnt.p;
  A.inv_cols = I->inv_cols.p;
  A.rowslot = I->rowslot.p;
  A.src_list = I->src_list.p;
  A.ctl = I->ctl.p;
  A.bar = I->bar.p;
  A.single_out = I->single_out.p;
  A.single_gain = I->single_gain.p;
  A.rowver = I->rowver.p;
  A.MX = I->MX.p;
  A.LN = I->LN.p;
  A.single_kind = -1;
  return A;
}

// fresh engine state: empty allotment, empty index
void reset_engine_state(lbdd_b200_instance* I, int64_t delta0) {
  const int64_t k = I->k;
  CUDA_OK(cudaMemsetAsync(I->home.p, 0xff, sizeof(int32_t) * I->n, I->stream));
  CUDA_OK(cudaMemsetAsync(I->load.p, 0, sizeof(int64_t) * (k + 1), I->stream));
  fill64(I, I->M.p, k * k, kEmpty);
  CUDA_OK(cudaMemsetAsync(I->inv_cnt.p, 0, sizeof(int32_t) * (k + 2), I->stream));
  CUDA_OK(cudaMemsetAsync(I->rowslot.p, 0xff, sizeof(int32_t) * (k + 1), I->stream));
  CUDA_OK(cudaMemsetAsync(I->bar.p, 0, sizeof(GridBar), I->stream));
  CUDA_OK(cudaMemsetAsync(I->rowver.p, 0, sizeof(int32_t) * (k + 1), I->stream));
  CUDA_OK(cudaMemsetAsync(I->pi.p, 0, sizeof(int64_t) * (k + 1), I->stream));
  // top-4 lists of the cluster engine: empty and complete
  I->MX.ensure(static_cast<size_t>(k) * k * (cl::kTopK - 1));
  I->LN.ensure(static_cast<size_t>(k) * k);
  fill64(I, I->MX.p, k * k * (cl::kTopK - 1), kEmpty);
  CUDA_OK(cudaMemsetAsync(I->LN.p, 8, static_cast<size_t>(k) * k, I->stream));
  EngineCtl ctl;
  std::memset(&ctl, 0, sizeof(ctl));
  ctl.delta = delta0;
  CUDA_OK(cudaMemcpyAsync(I->ctl.p, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, I->stream));
}

int32_t g_err_arg = 0;
void raise_engine_error(int32_t code) {
  switch (code) {
    case kErrNegCycleWitness: raise(LBDD_ERR_LOGIC, "lbdd: negative cycle witnessed in anchored graph");
    case kErrPathNotSimple: raise(LBDD_ERR_LOGIC, "lbdd: lowest-cost path is not simple");
    case kErrBrokenParent: raise(LBDD_ERR_LOGIC, "lbdd: broken parent chain");
    case kErrPathSum: raise(LBDD_ERR_LOGIC, "lbdd: path cost does not match edge sum");
    case kErrStaleTransfer: raise(LBDD_ERR_LOGIC, "lbdd: stale transfer edge");
    case kErrPenaltyEdge: raise(LBDD_ERR_LOGIC, "lbdd: path must close with a penalty edge");
    case kErrPlaceholder: raise(LBDD_ERR_LOGIC, "lbdd: placeholder transfer without surplus");
    case kErrNoResidual: raise(LBDD_ERR_LOGIC, "lbdd: no residual capacity left");
    case kErrAlreadyIndexed: raise(LBDD_ERR_LOGIC, "lbdd: demand already indexed");
    case kErrOverflow: raise(LBDD_ERR_OVERFLOW, "lbdd: cost accumulator overflow");
    case kErrInvariant: raise(LBDD_ERR_LOGIC, "lbdd: negative cycle survived refinement");
    case kErrNegativeLoad: raise(LBDD_ERR_LOGIC, "lbdd: negative load");
    case kErrNotOverloaded: raise(LBDD_ERR_LOGIC, "lbdd: path graph requires an overloaded anchor");
    default: raise(LBDD_ERR_RUNTIME, "lbdd_b200: engine error " + std::to_string(code) +
                   " arg " + std::to_string(g_err_arg));
  }
}

EngineCtl run_engine(lbdd_b200_instance* I, EngineArgs A, int64_t a_begin, int64_t a_end) {
  const Launch L = plan_launch(I, asral_engine_kernel, static_cast<int>(I->k),
                               static_cast<int>(I->k + 1), true);
  A.tile_mode = L.tile ? 1 : 0;
  uint8_t* dumflag = I->dumflag.p;
  EngineCtl ctl;
  const int64_t chunk = int64_t(1) << 16;
  int64_t a = a_begin;
  do {
    A.a_begin = a;
    A.a_end = std::min(a_end, a + chunk);
    void* args[] = {&A, &dumflag};
    g_launches++;
    ensure_kernel_events(I);
    CUDA_OK(cudaEventRecord(I->kev[0], I->stream));
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(asral_engine_kernel), dim3(L.grid),
                                        dim3(L.block), args, L.smem, I->stream));
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaEventRecord(I->kev[1], I->stream));
    CUDA_OK(cudaMemcpyAsync(&ctl, I->ctl.p, sizeof(ctl), cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaStreamSynchronize(I->stream));
    I->engine_ns += static_cast<int64_t>(static_cast<double>(I->time_since(I->kev[0])) * 1e6);
    I->engine_launches += 1;
    if (ctl.error) raise_engine_error(ctl.error);
    A.search_base = ctl.search_count;
    a = A.a_end;
  } while (a < a_end);
  return ctl;
}

// ---- the cluster engine (cluster.cu): one thread-block cluster ----
size_t cluster_smem_bytes(int k, int s, int block, bool tile) {
  const size_t cin = static_cast<size_t>(cl::inbox_cap(s));
  return 8 * s + 8 * s + 2 * sizeof(cl::FEntry) * cl::kMaxCS * cin + 2 * sizeof(cl::Pub) + 8 * 16 +
         2 * sizeof(cl::Pub) * cl::kMaxCS + 4 * 3 * cl::kMaxSeg +
         4 * 2 * cl::kMaxMine + 4 * (2 * cl::kMaxSeg + 2) +
         8 * 16 + 8 * 16 + 8 * 16 + 8 * 8 + 8 * 4 + 4 * 4 + 4 * 2 * static_cast<size_t>(s + 1) + 8 +
         8 * 4 + 8 * 2 +
         12 * block + 4 * 16 +
         4 * static_cast<size_t>(cl::kRowSlots) * ((k + 31) / 32) +
         (tile ? 2 * static_cast<size_t>(k) * s : 0) + static_cast<size_t>(s) + 16 +
         8 * static_cast<size_t>(s) + 8 * static_cast<size_t>(std::max(block, s)) + 8 * 4 * 32 +
         4 * 4 * cl::kMaxCS + sizeof(PathEdge) * cl::kPathCache;
}

bool cluster_engine_fits(int k) {
  for (int cs : {16, 8, 4, 2, 1}) {
    const int s = (k + 1 + cs - 1) / cs;
    if (cluster_smem_bytes(k, s, LBDD_CLUSTER_THREADS, false) <= 220 * 1024) return true;
  }
  return false;
}

bool use_grid_engine() {
  const char* e = std::getenv("LBDD_B200_ENGINE");
  return e != nullptr && std::string(e) == "grid";
}

// keys CM[d][v] - CM[d][u] fit the int16 tile when the cost range does
bool keys_fit_int16(const lbdd_b200_instance* I) {
  return I->scanned && I->min_cost >= 1 && I->max_cost + 1 - I->min_cost <= 32000;
}

constexpr int kClusterThreads = LBDD_CLUSTER_THREADS;

EngineCtl run_cluster_engine(lbdd_b200_instance* I, EngineArgs A, int64_t a_begin, int64_t a_end,
                             bool keys16) {
  const int block = kClusterThreads;
  const int k = static_cast<int>(I->k);
  auto kernel = cluster_engine_kernel;
  CUDA_OK(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  cfg.blockDim = dim3(block);
  cfg.stream = I->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (I->cluster_size == 0) {
    for (int cs : {16, 8, 4, 2, 1}) {
      const int s = (k + 1 + cs - 1) / cs;
      const size_t smem = cluster_smem_bytes(k, s, block, false);
      if (smem > 220 * 1024) continue;
      CUDA_OK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      cfg.gridDim = dim3(cs);
      cfg.dynamicSmemBytes = smem;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kernel, &cfg) == cudaSuccess && nclusters > 0) {
        I->cluster_size = cs;
        break;
      }
      cudaGetLastError();
    }
    if (I->cluster_size == 0) raise(LBDD_ERR_CUDA, "lbdd_b200: no cluster configuration fits");
  }
  {
    const char* ev = std::getenv("LBDD_B200_DELTA");
    A.delta_step = ev != nullptr ? std::atoll(ev) : 1;
    const char* evp = std::getenv("LBDD_B200_DELTA_PATH");
    A.delta_path = evp != nullptr ? std::atoll(evp) : A.delta_step;
    const char* pf = std::getenv("LBDD_B200_PROF");
    A.profile = pf != nullptr && std::string(pf) == "1";
    const char* dc = std::getenv("LBDD_B200_CHECK");
    A.debug_checks = dc != nullptr && std::string(dc) == "1";
  }
  const int cs = I->cluster_size;
  const int s = (k + 1 + cs - 1) / cs;
  const char* gf = std::getenv("LBDD_B200_GTILE_FORCE");  // tests: the global tile at any k
  const bool force_g = gf != nullptr && std::string(gf) == "1";
  const bool tile = keys16 && !force_g && cluster_smem_bytes(k, s, block, true) <= 220 * 1024;
  // keys that fit int16 but a tile that does not fit shared memory: the
  // same tile in global memory (k x k int16: 8 MB at k = 2000, L2-resident)
  // instead of reading the int64 heads of M
  const char* gt = std::getenv("LBDD_B200_GTILE");
  const bool gtile = !tile && keys16 && !(gt != nullptr && std::string(gt) == "0");
  A.tile_mode = tile ? 1 : (gtile ? 2 : 0);
  if (gtile) {
    I->ktile.ensure(static_cast<size_t>(k) * k);
    A.ktile = I->ktile.p;
  }
  const size_t smem = cluster_smem_bytes(k, s, block, tile);
  CUDA_OK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  cfg.gridDim = dim3(cs);
  cfg.dynamicSmemBytes = smem;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  EngineCtl ctl;
  // chunks of arrivals per launch: the bucket index is rebuilt in between,
  // so the move log a launch appends stays short
  const char* ch = std::getenv("LBDD_B200_CHUNK");
  const int64_t chunk = ch != nullptr ? std::max<int64_t>(64, std::atoll(ch)) : 4096;
  constexpr int32_t kLogCap = 1 << 16;
  I->log_d.ensure(kLogCap);
  I->log_to.ensure(kLogCap);
  I->log_n.ensure(1);
  A.log_d = I->log_d.p;
  A.log_to = I->log_to.p;
  A.log_n = I->log_n.p;
  A.log_cap = kLogCap;
  // per-center add lists: the T3 rescan candidates of a center are its
  // launch-start bucket plus the demands that moved to it since
  constexpr int32_t kAddCap = 128;
  I->add_ids.ensure(static_cast<size_t>(k) * kAddCap);
  I->add_cnt.ensure(k);
  A.add_ids = I->add_ids.p;
  A.add_cnt = I->add_cnt.p;
  A.add_cap = kAddCap;
  int64_t a = a_begin;
  int64_t* pi = I->pi.p;
  int32_t* dirty = I->dirty.p;
  do {
    A.a_begin = a;
    A.a_end = std::min(a_end, a + chunk);
    build_index_prepare(I, A.home, 0, I->n, I->stream, false);
    A.bk_off = I->ib_off.p;
    A.bk_ids = I->ib_sorted.p;
    CUDA_OK(cudaMemsetAsync(I->log_n.p, 0, sizeof(int32_t), I->stream));
    CUDA_OK(cudaMemsetAsync(I->add_cnt.p, 0, sizeof(int32_t) * k, I->stream));
    g_launches++;
    ensure_kernel_events(I);
    CUDA_OK(cudaEventRecord(I->kev[0], I->stream));
    CUDA_OK(cudaLaunchKernelEx(&cfg, kernel, A, pi, dirty));
    CUDA_OK(cudaEventRecord(I->kev[1], I->stream));
    CUDA_OK(cudaMemcpyAsync(&ctl, I->ctl.p, sizeof(ctl), cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaStreamSynchronize(I->stream));
    I->engine_ns += static_cast<int64_t>(static_cast<double>(I->time_since(I->kev[0])) * 1e6);
    I->engine_launches += 1;
    g_err_arg = ctl.error_arg;
    if (ctl.error) {
      if (std::getenv("LBDD_B200_DEBUG") != nullptr)
        std::fprintf(stderr, "lbdd_b200: engine error %d arg %d after %lld cycle refines, %lld path "
                     "refines (launch arrivals %lld..%lld)\n", ctl.error, ctl.error_arg,
                     static_cast<long long>(ctl.cycle_refine_calls),
                     static_cast<long long>(ctl.path_refine_calls),
                     static_cast<long long>(A.a_begin), static_cast<long long>(A.a_end));
      raise_engine_error(ctl.error);
    }
    a = A.a_end;
  } while (a < a_end);
  return ctl;
}

EngineCtl run_solver_engine(lbdd_b200_instance* I, EngineArgs A, int64_t a_begin, int64_t a_end,
                            bool keys16) {
  const char* e = std::getenv("LBDD_B200_TILE");
  if (e != nullptr && std::string(e) == "0") keys16 = false;
  // the one-cluster engine keeps O(k) per-CTA state in shared memory; past
  // k ~ 3000 no cluster shape fits and the grid-wide engine runs instead
  return use_grid_engine() || !cluster_engine_fits(static_cast<int>(I->k))
             ? run_engine(I, A, a_begin, a_end)
             : run_cluster_engine(I, A, a_begin, a_end, keys16);
}

EngineCtl g_last_ctl;  // instrumentation of the last engine run

void fill_report_stats(lbdd_solve_report* r, const EngineCtl& c) {
  g_last_ctl = c;
  r->cycle_refine_calls = c.cycle_refine_calls;
  r->path_refine_calls = c.path_refine_calls;
  r->negative_cycles_removed = c.negative_cycles_removed;
  r->negative_paths_removed = c.negative_paths_removed;
  r->refinement_gain = c.refinement_gain;
  r->transfers_applied = c.transfers_applied;
  r->invariant_checks = c.invariant_checks;
  r->bellman_ford_ns = c.t_bf_ns;
  r->index_update_ns = c.t_index_ns;
  r->relax_rounds = c.relax_rounds;
  r->grid_barriers = c.barriers;
}

// detail::finish_report (solver.hpp:110-129): completeness + recount.
int64_t finish(lbdd_b200_instance* I, int64_t delta, std::vector<int64_t>& loads) {
  int32_t missing = 0;
  const int64_t recount = device_objective(I, I->home.p, loads, &missing);
  if (missing) raise(LBDD_ERR_LOGIC, "lbdd: solver produced an incomplete allotment");
  if (recount != delta) raise(LBDD_ERR_LOGIC, "lbdd: tracked objective diverged from recount");
  return delta;
}

void copy_out(lbdd_b200_instance* I, const int32_t* d_assign, int32_t* assignment_out,
              const std::vector<int64_t>& loads, int64_t* load_out) {
  if (assignment_out) {
    CUDA_OK(cudaMemcpyAsync(assignment_out, d_assign, sizeof(int32_t) * I->n,
                            cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaStreamSynchronize(I->stream));
  }
  if (load_out) std::copy(loads.begin(), loads.end(), load_out);
}

// asral_solve (solver.hpp:133-170)
void solve_asral(lbdd_b200_instance* I, const lbdd_solver_options* o, int32_t solver,
                 lbdd_solve_report* rep, int32_t* assignment_out, int64_t* load_out,
                 int64_t arrivals = -1) {
  const int64_t start = now_ns();
  validate_centers(I);
  check_device_range(I);
  rep->scan_ns = arrival_scan(I, true);
  ensure_engine(I, 0);
  reset_engine_state(I, 0);
  EngineArgs A = engine_args(I);
  A.mode = 0;
  A.arr_keys = I->keys_sorted.p;
  A.best_center = I->best_center.p;
  I->arr_s.ensure(I->n);
  g_launches++;
  arrival_centers_kernel<<<grid_for(I->n), 256, 0, I->stream>>>(I->keys_sorted.p, I->best_center.p, I->n,
                                                              I->arr_s.p);
  CUDA_OK(cudaGetLastError());
  A.arr_s = I->arr_s.p;
  A.fixpoint = o && o->refine_to_fixpoint;
  A.check_invariants = o && o->check_invariants;
  const int64_t a_end = arrivals < 0 ? I->n : std::min<int64_t>(arrivals, I->n);
  const EngineCtl ctl = run_solver_engine(I, A, 0, a_end, keys_fit_int16(I));
  std::vector<int64_t> loads;
  if (a_end == I->n) {
    rep->objective = finish(I, ctl.delta, loads);
  } else {
    // a prefix of the arrival loop: the partial allotment's objective
    // (evaluate_partial_objective, core.hpp:216-233) must equal the running delta
    int32_t missing = 0;
    rep->objective = device_objective(I, I->home.p, loads, &missing);
    if (rep->objective != ctl.delta) raise(LBDD_ERR_LOGIC, "lbdd: tracked objective diverged from recount");
  }
  fill_report_stats(rep, ctl);
  rep->solver = solver;
  copy_out(I, I->home.p, assignment_out, loads, load_out);
  rep->total_ns = now_ns() - start;
}

// greedy_solve (solver.hpp:172-189): every demand at its row minimum.
void solve_greedy(lbdd_b200_instance* I, lbdd_solve_report* rep, int32_t* assignment_out,
                  int64_t* load_out) {
  const int64_t start = now_ns();
  validate_centers(I);
  rep->scan_ns = arrival_scan(I, true);
  std::vector<int64_t> loads;
  int32_t missing = 0;
  rep->objective = device_objective(I, I->best_center.p, loads, &missing);
  rep->solver = LBDD_SOLVER_GREEDY;
  copy_out(I, I->best_center.p, assignment_out, loads, load_out);
  rep->total_ns = now_ns() - start;
}

// strict_solve (solver.hpp:227-301) incl. augment_with_dummy_center.
void solve_strict(lbdd_b200_instance* I0, const lbdd_solver_options* o,
                  lbdd_solve_report* rep, int32_t* assignment_out, int64_t* load_out) {
  const int64_t start = now_ns();
  validate_centers(I0);
  check_device_range(I0);
  rep->scan_ns = arrival_scan(I0, true);
  const int64_t total_cap = I0->total_capacity();
  const bool excess = total_cap < I0->n;
  lbdd_b200_instance* W = I0;
  std::unique_ptr<lbdd_b200_instance> aug;
  if (excess) {
    const int64_t deficit = I0->n - total_cap;
    if (I0->max_cost + 1 > INT32_MAX)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: overflow-center cost exceeds int32");
    aug.reset(new_instance(I0->device, I0->n, I0->k + 1));
    W = aug.get();
    CUDA_OK(cudaMalloc(&W->d_cm, sizeof(int32_t) * W->n * W->pitch));
    W->owns_cm = true;
    g_launches++;
    augment_kernel<<<grid_for(W->n * W->pitch), 256, 0, W->stream>>>(
        I0->d_cm, I0->pitch, W->d_cm, W->pitch, W->n, static_cast<int32_t>(I0->k),
        static_cast<int32_t>(I0->max_cost + 1));
    CUDA_OK(cudaGetLastError());
    std::vector<int64_t> cap = I0->cap, off = I0->off, par = I0->par;
    std::vector<int32_t> fam = I0->fam;
    cap.push_back(deficit);
    fam.push_back(LBDD_PENALTY_CONSTANT);
    par.push_back(1);
    off.push_back(off.back() + 1);
    lbdd_instance_desc d{W->n, W->k, nullptr, cap.data(), fam.data(), off.data(), par.data()};
    upload_centers(W, &d);
    CUDA_OK(cudaStreamSynchronize(W->stream));
  }
  const int64_t k = W->k;
  const int64_t n = W->n;
  if (o && o->strict_order && o->strict_order_len > 0 && o->strict_order_len != n)
    raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: strict order must cover every demand");
  ensure_engine(W, 0);
  reset_engine_state(W, 0);
  CUDA_OK(cudaMemcpyAsync(W->dummies.p, W->cap.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice,
                          W->stream));
  EngineArgs A = engine_args(W);
  A.mode = 1;
  A.dummies = W->dummies.p;
  A.check_invariants = o && o->check_invariants;
  if (o && o->strict_order && o->strict_order_len > 0) {
    // The kernel indexes the cost matrix and home[] with these ids: reject
    // out-of-range ids (std::vector UB in the reference) and report a
    // repeated demand the way the reference's SubspaceIndex::insert does
    // (subspace.hpp:46-49, std::logic_error).
    std::vector<uint8_t> seen(static_cast<size_t>(n), 0);
    for (int64_t i = 0; i < n; ++i) {
      const int32_t d = o->strict_order[i];
      if (d < 0 || d >= n) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: strict order entry out of range");
      if (seen[static_cast<size_t>(d)]) raise(LBDD_ERR_LOGIC, "lbdd: demand already indexed");
      seen[static_cast<size_t>(d)] = 1;
    }
    W->order.ensure(n);
    CUDA_OK(cudaMemcpyAsync(W->order.p, o->strict_order, sizeof(int32_t) * n,
                            cudaMemcpyHostToDevice, W->stream));
    A.order = W->order.p;
  }
  // augmented instance: the overflow column max+1 widens the range by one
  const bool keys16 = keys_fit_int16(I0) && I0->max_cost + 2 - I0->min_cost <= 32000;
  const EngineCtl ctl = run_solver_engine(W, A, 0, n, keys16);
  if (W != I0) {  // the engine ran on the augmented instance: report its time
    I0->engine_ns += W->engine_ns;
    I0->engine_launches += W->engine_launches;
  }
  // capacity / placeholder accounting (solver.hpp:279-289)
  std::vector<int64_t> dummies(k);
  CUDA_OK(cudaMemcpyAsync(dummies.data(), W->dummies.p, sizeof(int64_t) * k, cudaMemcpyDeviceToHost,
                          W->stream));
  std::vector<int64_t> loads;
  const int64_t obj = finish(W, ctl.delta, loads);
  for (int64_t s = 0; s < k; ++s) {
    if (loads[s] > W->cap[s]) raise(LBDD_ERR_LOGIC, "lbdd: strict solve exceeded a capacity");
    if (loads[s] + dummies[s] != W->cap[s])
      raise(LBDD_ERR_LOGIC, "lbdd: placeholder accounting out of balance");
  }
  rep->objective = obj;
  fill_report_stats(rep, ctl);
  rep->solver = LBDD_SOLVER_STRICT;
  if (excess) {
    const int64_t deficit = I0->n - total_cap;
    rep->strict_surcharge = checked_mul(deficit, I0->max_cost + 1);
    rep->has_dummy_center = 1;
    rep->objective -= rep->strict_surcharge;
  }
  copy_out(W, W->home.p, assignment_out, loads, load_out);
  rep->total_ns = now_ns() - start;
}

// SolverState::from_allotment (solver.hpp:61-68) on the device: allotment,
// index (full segmented-argmin scan) and running objective.
int64_t state_from_allotment(lbdd_b200_instance* I, const int32_t* assignment) {
  ensure_engine(I, 0);
  reset_engine_state(I, 0);
  CUDA_OK(cudaMemcpyAsync(I->home.p, assignment, sizeof(int32_t) * I->n, cudaMemcpyHostToDevice,
                          I->stream));
  build_index_device(I, I->home.p, 0, I->n, I->M.p, I->stream);
  std::vector<int64_t> loads;
  int32_t missing = 0;
  const int64_t delta = device_objective(I, I->home.p, loads, &missing);
  CUDA_OK(cudaMemcpyAsync(I->load.p, loads.data(), sizeof(int64_t) * I->k, cudaMemcpyHostToDevice,
                          I->stream));
  EngineCtl ctl;
  std::memset(&ctl, 0, sizeof(ctl));
  ctl.delta = delta;
  CUDA_OK(cudaMemcpyAsync(I->ctl.p, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, I->stream));
  CUDA_OK(cudaStreamSynchronize(I->stream));
  return delta;
}

void run_single(lbdd_b200_instance* I, EngineArgs A) {
  const Launch L = plan_launch(I, asral_engine_kernel, static_cast<int>(I->k),
                               static_cast<int>(I->k + 1), true);
  A.tile_mode = L.tile ? 1 : 0;
  uint8_t* dumflag = I->dumflag.p;
  void* args[] = {&A, &dumflag};
  g_launches++;
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(asral_engine_kernel), dim3(L.grid),
                                      dim3(L.block), args, L.smem, I->stream));
  CUDA_OK(cudaGetLastError());
  EngineCtl ctl;
  CUDA_OK(cudaMemcpyAsync(&ctl, I->ctl.p, sizeof(ctl), cudaMemcpyDeviceToHost, I->stream));
  CUDA_OK(cudaStreamSynchronize(I->stream));
  if (ctl.error) raise_engine_error(ctl.error);
}

// dense anchored-graph helpers (lowest_cost_path / relax_round API)
struct DenseCtx {
  lbdd_b200_instance* I;
  DevBuf<int64_t> W;
  DevBuf<int32_t> out;
};

lbdd_b200_instance* g_dense_inst = nullptr;

lbdd_b200_instance* dense_instance(int32_t node_count) {
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  if (g_dense_inst == nullptr || g_dense_inst->k + 1 < node_count || g_dense_inst->device != dev) {
    delete g_dense_inst;
    g_dense_inst = new_instance(dev, 1, node_count - 1);
  }
  return g_dense_inst;
}

void check_dense(int32_t node_count, const int64_t* w) {
  if (node_count < 2 || node_count > 65535)
    raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: node_count must be in [2, 65535]");
  const int64_t m = static_cast<int64_t>(node_count - 1) * node_count;
  for (int64_t i = 0; i < m; ++i) {
    if (w[i] != kNoEdge && (w[i] > (int64_t(1) << 40) || w[i] < -(int64_t(1) << 40)))
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: edge weight exceeds the device range (2^40)");
  }
}

}  // namespace capi_detail

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

const char* lbdd_b200_version(void) { return "lbdd_b200 0.1.0 (sm_100a)"; }
long long lbdd_b200_launch_count(void) { return g_launches.load(); }
/* Debug: cycles per exchange of the cluster primitive (cluster.cu). */
long long lbdd_b200_debug_exchange_cycles(int cluster_size, int iters, int mode) {
  auto kernel = cluster_exchange_bench;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  long long* d = nullptr;
  cudaMalloc(&d, 16);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_size;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cluster_size);
  cfg.blockDim = dim3(512);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kernel, iters, mode, d) != cudaSuccess) return -1;
  long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h[0];
}

/* Engine instrumentation of the last solve (16 counters, see cluster.cu). */
void lbdd_b200_engine_counters(int64_t* out) {
  for (int i = 0; i < 16; ++i) out[i] = g_last_ctl.dbg[i];
  for (int i = 0; i < 16; ++i) out[16 + i] = g_last_ctl.prof[i];
  for (int i = 0; i < 8; ++i) out[32 + i] = g_last_ctl.resc[i];
  for (int i = 0; i < 16; ++i) out[40 + i] = g_last_ctl.cta_work[i];
  for (int i = 0; i < 16; ++i) out[56 + i] = g_last_ctl.cta_wait[i];
}
const char* lbdd_b200_last_error(void) { return g_err.c_str(); }

int lbdd_b200_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

lbdd_status lbdd_b200_instance_create(const lbdd_instance_desc* desc, int device,
                                      lbdd_b200_instance** out) {
  return guarded([&] {
    if (desc->n < 0 || desc->k < 0) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: cost matrix size mismatch");
    std::unique_ptr<lbdd_b200_instance> I(new_instance(device, desc->n, desc->k));
    const size_t bytes = sizeof(int32_t) * std::max<int64_t>(I->n * I->pitch, 1);
    CUDA_OK(cudaMalloc(&I->d_cm, bytes));
    I->owns_cm = true;
    if (I->n > 0 && I->k > 0) {
      CUDA_OK(cudaMemcpy2DAsync(I->d_cm, sizeof(int32_t) * I->pitch, desc->costs,
                                sizeof(int32_t) * I->k, sizeof(int32_t) * I->k, I->n,
                                cudaMemcpyHostToDevice, I->stream));
    }
    upload_centers(I.get(), desc);
    CUDA_OK(cudaStreamSynchronize(I->stream));
    *out = I.release();
  });
}

lbdd_status lbdd_b200_instance_create_device(const lbdd_instance_desc* desc, const int32_t* d_costs,
                                             int64_t pitch_elems, int device,
                                             lbdd_b200_instance** out) {
  return guarded([&] {
    if (pitch_elems < desc->k || pitch_elems % 4 != 0)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: pitch must be >= k and a multiple of 4");
    std::unique_ptr<lbdd_b200_instance> I(new_instance(device, desc->n, desc->k));
    I->pitch = pitch_elems;
    I->d_cm = const_cast<int32_t*>(d_costs);
    I->owns_cm = false;
    upload_centers(I.get(), desc);
    *out = I.release();
  });
}

lbdd_status lbdd_b200_instance_generate(int64_t n, int64_t k, int64_t theta_num,
                                        int64_t theta_den, int64_t pen_lo, int64_t pen_hi,
                                        int32_t mixed_families, int64_t cap_spread,
                                        uint64_t seed, int device, lbdd_b200_instance** out) {
  return guarded([&] {
    if (n < 1 || k < 1) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: n and k must be >= 1");
    if (theta_num < 1 || theta_den < 1) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: theta must be positive");
    if (pen_lo < 1 || pen_hi < pen_lo) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: bad penalty range");
    if (cap_spread < 1) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: cap_spread must be >= 1");
    std::unique_ptr<lbdd_b200_instance> I(new_instance(device, n, k));
    CUDA_OK(cudaMalloc(&I->d_cm, sizeof(int32_t) * n * I->pitch));
    I->owns_cm = true;
    // spec "lbdd-synth-v2" (synth_instances.py): stream(seed, t, i) =
    // mix(mix(seed ^ t) + (i + 1) * golden)
    auto mix = [](uint64_t z) {
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    auto stream = [&](uint64_t tag, uint64_t i) {
      return mix(mix(seed ^ tag) + (i + 1) * 0x9E3779B97F4A7C15ull);
    };
    const ulonglong4 base = make_ulonglong4(mix(seed ^ 1), mix(seed ^ 2), mix(seed ^ 3), mix(seed ^ 4));
    g_launches++;
    generate_costs_kernel<<<I->num_sms * 8, 256, 0, I->stream>>>(I->d_cm, I->pitch, 0, n,
                                                                static_cast<int32_t>(k), base);
    CUDA_OK(cudaGetLastError());
    // capacities: total = n * theta_num // theta_den over integer weights
    // 1 + stream(5, s) % cap_spread; the remainder adds 1 to centers 0, 1, ...
    const int64_t total = n * theta_num / theta_den;
    std::vector<int64_t> w(k), cap(k);
    int64_t wsum = 0, assigned = 0;
    for (int64_t s = 0; s < k; ++s) {
      w[s] = 1 + static_cast<int64_t>(stream(5, s) % static_cast<uint64_t>(cap_spread));
      wsum += w[s];
    }
    for (int64_t s = 0; s < k; ++s) {
      cap[s] = static_cast<int64_t>(static_cast<__int128>(total) * w[s] / wsum);
      assigned += cap[s];
    }
    for (int64_t s = 0; s < total - assigned; ++s) cap[s]++;
    std::vector<int32_t> fam(k);
    std::vector<int64_t> off(k + 1, 0), par;
    const uint64_t span = static_cast<uint64_t>(pen_hi - pen_lo + 1);
    for (int64_t s = 0; s < k; ++s) {
      const uint64_t p = stream(6, s);
      const int f = mixed_families ? static_cast<int>(p % 3) : 0;
      const int64_t base_pen = pen_lo + static_cast<int64_t>((p >> 8) % span);
      fam[s] = f;
      if (f == 0) {
        par.push_back(base_pen);
      } else if (f == 1) {
        par.push_back(base_pen);
        par.push_back(static_cast<int64_t>((p >> 24) % 6));
      } else {
        int64_t v = base_pen;
        par.push_back(v);
        for (int t = 1; t < 4; ++t) {
          v += static_cast<int64_t>((p >> (32 + 3 * t)) % 8);
          par.push_back(v);
        }
      }
      off[s + 1] = static_cast<int64_t>(par.size());
    }
    lbdd_instance_desc d{n, k, nullptr, cap.data(), fam.data(), off.data(), par.data()};
    upload_centers(I.get(), &d);
    CUDA_OK(cudaStreamSynchronize(I->stream));
    *out = I.release();
  });
}

lbdd_status lbdd_b200_instance_destroy(lbdd_b200_instance* inst) {
  return guarded([&] { delete inst; });
}

lbdd_status lbdd_b200_instance_shape(const lbdd_b200_instance* inst, int64_t* n, int64_t* k) {
  return guarded([&] {
    *n = inst->n;
    *k = inst->k;
  });
}

lbdd_status lbdd_b200_instance_centers(const lbdd_b200_instance* inst, int64_t* capacity,
                                       int32_t* family, int64_t* offset, int64_t* params,
                                       int64_t* n_params) {
  return guarded([&] {
    *n_params = static_cast<int64_t>(inst->par.size());
    if (capacity) std::copy(inst->cap.begin(), inst->cap.end(), capacity);
    if (family) std::copy(inst->fam.begin(), inst->fam.end(), family);
    if (offset) std::copy(inst->off.begin(), inst->off.end(), offset);
    if (params) std::copy(inst->par.begin(), inst->par.end(), params);
  });
}

lbdd_status lbdd_b200_instance_costs(const lbdd_b200_instance* inst, int64_t row0, int64_t rows,
                                     int32_t* out) {
  return guarded([&] {
    require_unsharded(inst);
    if (row0 < 0 || rows < 0 || row0 + rows > inst->n)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: row range out of bounds");
    CUDA_OK(cudaSetDevice(inst->device));
    CUDA_OK(cudaMemcpy2D(out, sizeof(int32_t) * inst->k, inst->d_cm + row0 * inst->pitch,
                         sizeof(int32_t) * inst->pitch, sizeof(int32_t) * inst->k, rows,
                         cudaMemcpyDeviceToHost));
  });
}

lbdd_status lbdd_b200_solve(lbdd_b200_instance* inst, int32_t solver,
                            const lbdd_solver_options* opts, lbdd_solve_report* report,
                            int32_t* assignment_out, int64_t* load_out) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(inst->device));
    std::memset(report, 0, sizeof(*report));
    inst->engine_ns = inst->engine_launches = inst->row_scan_ns = 0;
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    CUDA_OK(cudaEventRecord(e0, inst->stream));
    switch (solver) {
      case LBDD_SOLVER_ASRAL:
      case LBDD_SOLVER_PARA_ASRAL:
        solve_asral(inst, opts, solver, report, assignment_out, load_out);
        break;
      case LBDD_SOLVER_STRICT: solve_strict(inst, opts, report, assignment_out, load_out); break;
      case LBDD_SOLVER_GREEDY: solve_greedy(inst, report, assignment_out, load_out); break;
      default: raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: unknown solver");
    }
    CUDA_OK(cudaEventRecord(e1, inst->stream));
    CUDA_OK(cudaEventSynchronize(e1));
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
    report->device_ns = static_cast<int64_t>(static_cast<double>(ms) * 1e6);
    report->engine_ns = inst->engine_ns;
    report->engine_launches = inst->engine_launches;
    report->row_scan_ns = inst->row_scan_ns;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

lbdd_status lbdd_b200_solve_prefix(lbdd_b200_instance* inst, const lbdd_solver_options* opts,
                                   int64_t arrivals, lbdd_solve_report* report,
                                   int32_t* assignment_out, int64_t* load_out) {
  return guarded([&] {
    if (arrivals < 0) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: negative arrival count");
    CUDA_OK(cudaSetDevice(inst->device));
    std::memset(report, 0, sizeof(*report));
    inst->engine_ns = inst->engine_launches = inst->row_scan_ns = 0;
    solve_asral(inst, opts, LBDD_SOLVER_ASRAL, report, assignment_out, load_out, arrivals);
    report->engine_ns = inst->engine_ns;
    report->engine_launches = inst->engine_launches;
    report->row_scan_ns = inst->row_scan_ns;
  });
}

lbdd_status lbdd_b200_build_index(lbdd_b200_instance* inst, const int32_t* assignment, int64_t row0,
                                  int64_t rows, int64_t* min_transfer_out) {
  return guarded([&] {
    require_unsharded(inst);
    CUDA_OK(cudaSetDevice(inst->device));
    if (rows < 0) { row0 = 0; rows = inst->n; }
    if (row0 < 0 || row0 + rows > inst->n)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: row range out of bounds");
    inst->home.ensure(inst->n);
    inst->M.ensure(inst->k * inst->k);
    CUDA_OK(cudaMemcpyAsync(inst->home.p, assignment, sizeof(int32_t) * inst->n,
                            cudaMemcpyHostToDevice, inst->stream));
    fill64(inst, inst->M.p, inst->k * inst->k, kEmpty);
    build_index_device(inst, inst->home.p, row0, row0 + rows, inst->M.p, inst->stream);
    CUDA_OK(cudaMemcpyAsync(min_transfer_out, inst->M.p, sizeof(int64_t) * inst->k * inst->k,
                            cudaMemcpyDeviceToHost, inst->stream));
    CUDA_OK(cudaStreamSynchronize(inst->stream));
  });
}

lbdd_status lbdd_b200_build_index_device(lbdd_b200_instance* inst, const int32_t* d_assignment,
                                         int64_t row0, int64_t rows, int64_t* d_out,
                                         void* stream) {
  return guarded([&] {
    require_unsharded(inst);
    CUDA_OK(cudaSetDevice(inst->device));
    if (rows < 0) { row0 = 0; rows = inst->n; }
    if (row0 < 0 || row0 + rows > inst->n)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: row range out of bounds");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    g_launches++;
    fill_i64_kernel<<<grid_for(inst->k * inst->k), 256, 0, st>>>(d_out, inst->k * inst->k, kEmpty);
    CUDA_OK(cudaGetLastError());
    build_index_device(inst, d_assignment, row0, row0 + rows, d_out, st);
  });
}

lbdd_status lbdd_b200_build_index_shard(lbdd_b200_instance* inst, const int32_t* d_assignment,
                                        int64_t demand_offset, int64_t* d_out, void* stream) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(inst->device));
    if (demand_offset < 0 || demand_offset + inst->n >= INT32_MAX)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: demand ids exceed int32");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t rows = inst->nshards > 1 ? inst->local_rows : inst->n;  // this rank's block
    g_launches++;
    fill_i64_kernel<<<grid_for(inst->k * inst->k), 256, 0, st>>>(d_out, inst->k * inst->k, kEmpty);
    CUDA_OK(cudaGetLastError());
    build_index_prepare(inst, d_assignment, 0, rows, st, true);
    build_index_scan(inst, rows, d_out, st, static_cast<int32_t>(demand_offset));
  });
}

lbdd_status lbdd_b200_arrival_queue(lbdd_b200_instance* inst, int32_t* best_center,
                                    int64_t* best_cost, int32_t* order) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(inst->device));
    arrival_scan(inst, false);
    std::vector<int64_t> sorted(inst->n);
    CUDA_OK(cudaMemcpy(sorted.data(), inst->keys_sorted.p, sizeof(int64_t) * inst->n,
                       cudaMemcpyDeviceToHost));
    std::vector<int32_t> bc(inst->n);
    CUDA_OK(cudaMemcpy(bc.data(), inst->best_center.p, sizeof(int32_t) * inst->n,
                       cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < inst->n; ++i) {
      const int32_t d = static_cast<int32_t>(sorted[i] & 0xffffffffLL);
      if (order) order[i] = d;
      if (best_cost) best_cost[d] = sorted[i] >> 32;
    }
    if (best_center) std::copy(bc.begin(), bc.end(), best_center);
  });
}

lbdd_status lbdd_b200_refine(lbdd_b200_instance* inst, int32_t kind, int32_t anchor,
                             int32_t* assignment, int64_t* dummies, int32_t* applied,
                             int64_t* gain) {
  return guarded([&] {
    require_unsharded(inst);
    CUDA_OK(cudaSetDevice(inst->device));
    if (kind != 0 && kind != 1) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: refine kind is 0 or 1");
    if (anchor < 0 || anchor >= inst->k) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: bad anchor");
    check_device_range(inst);
    state_from_allotment(inst, assignment);
    EngineArgs A = engine_args(inst);
    A.single_kind = kind;
    A.single_anchor = anchor;
    if (dummies) {
      CUDA_OK(cudaMemcpyAsync(inst->dummies.p, dummies, sizeof(int64_t) * inst->k,
                              cudaMemcpyHostToDevice, inst->stream));
      A.mode = 1;
      A.dummies = inst->dummies.p;
    }
    run_single(inst, A);
    int32_t out[2];
    CUDA_OK(cudaMemcpy(out, inst->single_out.p, sizeof(out), cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(gain, inst->single_gain.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
    *applied = out[0];
    CUDA_OK(cudaMemcpy(assignment, inst->home.p, sizeof(int32_t) * inst->n, cudaMemcpyDeviceToHost));
    if (dummies) {
      CUDA_OK(cudaMemcpy(dummies, inst->dummies.p, sizeof(int64_t) * inst->k, cudaMemcpyDeviceToHost));
    }
  });
}

lbdd_status lbdd_b200_gamma_has_negative_cycle(lbdd_b200_instance* inst, const int32_t* assignment,
                                               const int64_t* dummies, int32_t* has_cycle) {
  return guarded([&] {
    require_unsharded(inst);
    CUDA_OK(cudaSetDevice(inst->device));
    check_device_range(inst);
    state_from_allotment(inst, assignment);
    EngineArgs A = engine_args(inst);
    A.single_kind = kGammaGraph;
    if (dummies) {
      CUDA_OK(cudaMemcpyAsync(inst->dummies.p, dummies, sizeof(int64_t) * inst->k,
                              cudaMemcpyHostToDevice, inst->stream));
      A.mode = 1;
      A.dummies = inst->dummies.p;
    }
    run_single(inst, A);
    int32_t out[2];
    CUDA_OK(cudaMemcpy(out, inst->single_out.p, sizeof(out), cudaMemcpyDeviceToHost));
    *has_cycle = out[0];
  });
}

lbdd_status lbdd_b200_evaluate_objective(lbdd_b200_instance* inst, const int32_t* assignment,
                                         int32_t partial, int64_t* objective) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(inst->device));
    inst->home.ensure(inst->n);
    for (int64_t d = 0; d < inst->n; ++d) {
      if (assignment[d] < -1 || assignment[d] >= inst->k)
        raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: allotment shape mismatch");
    }
    CUDA_OK(cudaMemcpyAsync(inst->home.p, assignment, sizeof(int32_t) * inst->n,
                            cudaMemcpyHostToDevice, inst->stream));
    std::vector<int64_t> loads;
    int32_t missing = 0;
    const int64_t v = device_objective(inst, inst->home.p, loads, &missing);
    if (missing && !partial)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: objective of incomplete allotment");
    *objective = v;
  });
}

lbdd_status lbdd_b200_lowest_cost_path(int32_t node_count, int32_t anchor, const int64_t* weights,
                                       int32_t* found, int64_t* cost, int64_t* dist,
                                       int32_t* parent_node, int32_t* path, int32_t* path_len) {
  return guarded([&] {
    check_dense(node_count, weights);
    if (anchor < 0 || anchor >= node_count - 1)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: bad anchor");
    lbdd_b200_instance* I = dense_instance(node_count);
    // the dense graph's "k" is rows; engine buffers sized for k+1 nodes
    const int64_t saved_k = I->k;
    I->k = node_count - 1;
    ensure_engine(I, node_count);
    DevBuf<int64_t> W;
    DevBuf<int32_t> out;
    const int64_t m = static_cast<int64_t>(node_count - 1) * node_count;
    W.ensure(m);
    out.ensure(1);
    CUDA_OK(cudaMemcpyAsync(W.p, weights, sizeof(int64_t) * m, cudaMemcpyHostToDevice, I->stream));
    CUDA_OK(cudaMemsetAsync(I->bar.p, 0, sizeof(GridBar), I->stream));
    CUDA_OK(cudaMemsetAsync(I->ctl.p, 0, sizeof(EngineCtl), I->stream));
    EngineArgs A = engine_args(I);
    const Launch L = plan_launch(I, dense_path_kernel, node_count - 1, node_count, false);
    int32_t one = 0;
    const int64_t* wp = W.p;
    int32_t* op = out.p;
    void* args[] = {&A, &wp, &node_count, &anchor, &one, &op};
    g_launches++;
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dense_path_kernel), dim3(L.grid),
                                        dim3(L.block), args, L.smem, I->stream));
    CUDA_OK(cudaGetLastError());
    int32_t r = 0;
    CUDA_OK(cudaMemcpyAsync(&r, out.p, sizeof(int32_t), cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaStreamSynchronize(I->stream));
    I->k = saved_k;
    if (r < 0) raise(LBDD_ERR_LOGIC, "lbdd: negative cycle witnessed in anchored graph");
    std::vector<int64_t> d(node_count);
    std::vector<int32_t> p(node_count);
    CUDA_OK(cudaMemcpy(d.data(), I->D[0][(r + 1) & 1].p, sizeof(int64_t) * node_count,
                       cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(p.data(), I->P[0][(r + 1) & 1].p, sizeof(int32_t) * node_count,
                       cudaMemcpyDeviceToHost));
    *path_len = 0;
    const int32_t sink = node_count - 1;
    if (d[sink] >= kUnreachable) {
      *found = 0;
      return;
    }
    *found = 1;
    *cost = d[sink];
    std::copy(d.begin(), d.end(), dist);
    std::copy(p.begin(), p.end(), parent_node);
    // parent walk, refine.hpp:61-80
    std::vector<int32_t> rev{sink};
    std::vector<char> seen(node_count, 0);
    int32_t node = sink;
    while (node != anchor) {
      if (seen[node]) raise(LBDD_ERR_LOGIC, "lbdd: lowest-cost path is not simple");
      seen[node] = 1;
      const int32_t u = p[node];
      if (u < 0) raise(LBDD_ERR_LOGIC, "lbdd: broken parent chain");
      rev.push_back(u);
      node = u;
    }
    int64_t sum = 0;
    const int32_t len = static_cast<int32_t>(rev.size()) - 1;
    for (int32_t i = 0; i <= len; ++i) path[i] = rev[len - i];
    for (int32_t i = 0; i < len; ++i) {
      sum = checked_add(sum, weights[static_cast<int64_t>(path[i]) * node_count + path[i + 1]]);
    }
    if (sum != *cost) raise(LBDD_ERR_LOGIC, "lbdd: path cost does not match edge sum");
    *path_len = len;
  });
}

lbdd_status lbdd_b200_relax_round(int32_t node_count, const int64_t* weights,
                                  const int64_t* dist_in, const int32_t* parent_in,
                                  int64_t* dist_out, int32_t* parent_out, int32_t* changed) {
  return guarded([&] {
    check_dense(node_count, weights);
    lbdd_b200_instance* I = dense_instance(node_count);
    const int64_t saved_k = I->k;
    I->k = node_count - 1;
    ensure_engine(I, node_count);
    DevBuf<int64_t> W;
    DevBuf<int32_t> out;
    const int64_t m = static_cast<int64_t>(node_count - 1) * node_count;
    W.ensure(m);
    out.ensure(1);
    CUDA_OK(cudaMemcpyAsync(W.p, weights, sizeof(int64_t) * m, cudaMemcpyHostToDevice, I->stream));
    CUDA_OK(cudaMemcpyAsync(I->D[0][1].p, dist_in, sizeof(int64_t) * node_count, cudaMemcpyHostToDevice, I->stream));
    CUDA_OK(cudaMemcpyAsync(I->P[0][1].p, parent_in, sizeof(int32_t) * node_count, cudaMemcpyHostToDevice, I->stream));
    fill64(I, I->B[0][0].p, node_count, kEmpty);
    fill64(I, I->B[0][1].p, node_count, kEmpty);
    CUDA_OK(cudaMemsetAsync(I->bar.p, 0, sizeof(GridBar), I->stream));
    CUDA_OK(cudaMemsetAsync(I->ctl.p, 0, sizeof(EngineCtl), I->stream));
    EngineArgs A = engine_args(I);
    const Launch L = plan_launch(I, dense_path_kernel, node_count - 1, node_count, false);
    int32_t one = 1;
    int32_t anchor = -1;
    const int64_t* wp = W.p;
    int32_t* op = out.p;
    void* args[] = {&A, &wp, &node_count, &anchor, &one, &op};
    g_launches++;
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(dense_path_kernel), dim3(L.grid),
                                        dim3(L.block), args, L.smem, I->stream));
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(changed, out.p, sizeof(int32_t), cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaMemcpyAsync(dist_out, I->D[0][1].p, sizeof(int64_t) * node_count, cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaMemcpyAsync(parent_out, I->P[0][1].p, sizeof(int32_t) * node_count, cudaMemcpyDeviceToHost, I->stream));
    CUDA_OK(cudaStreamSynchronize(I->stream));
    I->k = saved_k;
  });
}

lbdd_status lbdd_b200_bench_index_scan(lbdd_b200_instance* inst, int32_t iters, double* mean_ms,
                                       double* bytes_per_scan) {
  return guarded([&] {
    require_unsharded(inst);
    CUDA_OK(cudaSetDevice(inst->device));
    if (!inst->scanned) arrival_scan(inst, false);
    inst->M.ensure(inst->k * inst->k);
    // warm-up (also sizes every scratch buffer)
    fill64(inst, inst->M.p, inst->k * inst->k, kEmpty);
    build_index_device(inst, inst->best_center.p, 0, inst->n, inst->M.p, inst->stream);
    CUDA_OK(cudaStreamSynchronize(inst->stream));
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    double total = 0;
    build_index_prepare(inst, inst->best_center.p, 0, inst->n, inst->stream, true);
    for (int i = 0; i < iters; ++i) {
      fill64(inst, inst->M.p, inst->k * inst->k, kEmpty);
      CUDA_OK(cudaEventRecord(e0, inst->stream));
      build_index_scan(inst, inst->n, inst->M.p, inst->stream);
      CUDA_OK(cudaEventRecord(e1, inst->stream));
      CUDA_OK(cudaEventSynchronize(e1));
      float ms = 0;
      CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *mean_ms = total / std::max(iters, 1);
    *bytes_per_scan = static_cast<double>(inst->n) * inst->k * 4.0 +
                      static_cast<double>(inst->n) * 12.0 +
                      static_cast<double>(inst->k) * inst->k * 8.0;
  });
}

// ---------------------------------------------------------------------------
// sharded instances: demand rows split over the ranks of one box
// ---------------------------------------------------------------------------

lbdd_status lbdd_b200_shard_alloc(int64_t rows, int64_t k, int device, int32_t** d_shard,
                                  int64_t* pitch_elems) {
  return guarded([&] {
    if (rows < 1 || k < 1) raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd: n and k must be >= 1");
    CUDA_OK(cudaSetDevice(device));
    const int64_t pitch = ((k + 3) / 4) * 4;
    CUDA_OK(cudaMalloc(d_shard, sizeof(int32_t) * rows * pitch));
    *pitch_elems = pitch;
  });
}

lbdd_status lbdd_b200_shard_free(int32_t* d_shard, int device) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaFree(d_shard));
  });
}

lbdd_status lbdd_b200_shard_upload(int32_t* d_shard, int64_t pitch_elems, const int32_t* host_rows,
                                   int64_t rows, int64_t k, int device) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaMemcpy2D(d_shard, sizeof(int32_t) * pitch_elems, host_rows, sizeof(int32_t) * k,
                         sizeof(int32_t) * k, rows, cudaMemcpyHostToDevice));
    if (pitch_elems > k) {  // padding columns: never read as costs
      CUDA_OK(cudaMemset2D(d_shard + k, sizeof(int32_t) * pitch_elems, 0x7f,
                           sizeof(int32_t) * (pitch_elems - k), rows));
    }
  });
}

lbdd_status lbdd_b200_ipc_get_handle(const void* d_ptr, int device, uint8_t* handle64) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    CUDA_OK(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle64, &h, 64);
  });
}

lbdd_status lbdd_b200_ipc_open(const uint8_t* handle64, int device, void** d_ptr) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    CUDA_OK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

lbdd_status lbdd_b200_ipc_close(void* d_ptr, int device) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(device));
    CUDA_OK(cudaIpcCloseMemHandle(d_ptr));
  });
}

lbdd_status lbdd_b200_instance_create_sharded(const lbdd_instance_desc* centers,
                                              const int32_t* const* shard_ptrs, int32_t nshards,
                                              int32_t my_shard, int64_t shard_rows,
                                              int64_t pitch_elems, int device,
                                              lbdd_b200_instance** out) {
  return guarded([&] {
    const int64_t n = centers->n;
    if (nshards < 1 || nshards > kMaxShards || my_shard < 0 || my_shard >= nshards)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: bad shard layout");
    if (shard_rows < 1 || shard_rows * nshards < n || shard_rows * (nshards - 1) >= n ||
        shard_rows >= INT32_MAX)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: shard_rows must split n over nshards blocks");
    if (pitch_elems < centers->k || pitch_elems % 4 != 0)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: pitch must be >= k and a multiple of 4");
    std::unique_ptr<lbdd_b200_instance> I(new_instance(device, n, centers->k));
    I->pitch = pitch_elems;
    I->nshards = nshards;
    I->my_shard = my_shard;
    I->shard_rows = shard_rows;
    I->local_rows = std::min<int64_t>(shard_rows, n - shard_rows * my_shard);
    I->d_cm = const_cast<int32_t*>(shard_ptrs[my_shard]);
    I->owns_cm = false;
    I->rt = RowTable{};
    for (int i = 0; i < nshards; ++i) I->rt.shard[i] = shard_ptrs[i];
    I->rt.pitch = pitch_elems;
    I->rt.shard_rows = static_cast<int32_t>(shard_rows);
    I->rt.nshards = nshards;
    upload_centers(I.get(), centers);
    *out = I.release();
  });
}

lbdd_status lbdd_b200_shard_arrival_scan(lbdd_b200_instance* inst, int64_t* d_keys, int32_t* d_best,
                                         int64_t* min_cost, int64_t* max_cost) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(inst->device));
    const int64_t rows = inst->nshards > 1 ? inst->local_rows : inst->n;
    const int64_t id0 = inst->nshards > 1 ? inst->shard_rows * inst->my_shard : 0;
    inst->minmax.ensure(2);
    const int64_t init[2] = {INT64_MAX, INT64_MIN};
    CUDA_OK(cudaMemcpyAsync(inst->minmax.p, init, sizeof(init), cudaMemcpyHostToDevice, inst->stream));
    launch_row_argmin(inst, inst->d_cm, rows, id0, d_best, d_keys, inst->minmax.p);
    int64_t mm[2];
    CUDA_OK(cudaMemcpyAsync(mm, inst->minmax.p, sizeof(mm), cudaMemcpyDeviceToHost, inst->stream));
    CUDA_OK(cudaStreamSynchronize(inst->stream));
    *min_cost = mm[0];
    *max_cost = mm[1];
  });
}

lbdd_status lbdd_b200_solve_sharded(lbdd_b200_instance* inst, int32_t solver,
                                    const int64_t* d_keys_all, const int32_t* d_best_all,
                                    int64_t min_cost, int64_t max_cost,
                                    const lbdd_solver_options* opts, lbdd_solve_report* report,
                                    int32_t* assignment_out, int64_t* load_out) {
  return guarded([&] {
    CUDA_OK(cudaSetDevice(inst->device));
    if (solver == LBDD_SOLVER_STRICT)
      raise(LBDD_ERR_INVALID_ARGUMENT, "lbdd_b200: strict_solve on a sharded instance is not supported");
    const int64_t n = inst->n;
    inst->keys.ensure(n);
    inst->keys_sorted.ensure(n);
    inst->best_center.ensure(n);
    CUDA_OK(cudaMemcpyAsync(inst->keys.p, d_keys_all, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice,
                            inst->stream));
    CUDA_OK(cudaMemcpyAsync(inst->best_center.p, d_best_all, sizeof(int32_t) * n,
                            cudaMemcpyDeviceToDevice, inst->stream));
    inst->min_cost = min_cost;
    inst->max_cost = max_cost;
    inst->gathered = true;
    struct Reset {
      lbdd_b200_instance* I;
      ~Reset() { I->gathered = false; }
    } reset{inst};
    const lbdd_status st = lbdd_b200_solve(inst, solver, opts, report, assignment_out, load_out);
    if (st != LBDD_OK) raise(st, lbdd_b200_last_error());
  });
}

}  // extern "C"
