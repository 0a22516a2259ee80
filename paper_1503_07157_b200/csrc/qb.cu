// qb.cu — host driver and C ABI (include/qb.h) of the B200-native blocked randomized QB
// factorization (randQB_b; randQB_pb).
//
// One context owns a CUDA stream, the residual workspace, Q̄ / B̄ and all scratch.  The
// block loop below is the paper's loop; every arithmetic step runs in this library's
// kernels (omega.cuh; gemm_f64.cuh for FP64 and gemm_tf32.cuh for the FP32 residual's products;
// small.cuh for CholeskyQR and reductions; qrcp.cuh for QB -> pivoted QR).  The host only
// sequences launches and reads two scalars per block (the stop test) plus the CholeskyQR status
// words.  The post-processing entry points (rqb_svd, qb_pivoted_qr) and the fixed-rank schemes
// (qb_fixed_rank) reuse the same kernels; the k x k SVD core of rqb_svd is a block one-sided Jacobi
// (svd.cuh).  No solver library is used.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <dlfcn.h>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached
#include <nccl.h>  // types only: NCCL is loaded at run time (dlopen), never linked

#include "../../include/qb.h"
#include "common.cuh"
#include "gemm_f64.cuh"
#include "gemm_tf32.cuh"
#include "omega.cuh"
#include "qrcp.cuh"
#include "qrcp_persist.cuh"
#include "small.cuh"
#include "small_loop.cuh"
#include "svd.cuh"

namespace {

using namespace qbk;

constexpr int64_t kMaxB = CHOL_MAXW;

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  double* d() const { return static_cast<double*>(p); }
};

// ---------------------------------------------------------------- NCCL (dlopen)
// The multi-GPU path (column sharding) needs ncclAllReduce only.  NCCL is
// resolved at run time from the process (torch's bundled libnccl.so.2 when torch is loaded)
// or the system, so the library itself has no link-time NCCL dependency.
struct NcclApi {
  bool tried = false, ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclCommGetAsyncError) getAsyncError = nullptr;
  decltype(&ncclCommAbort) commAbort = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  const char* env = getenv("QB_NCCL_LIB");
  void* h = nullptr;
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.getUniqueId = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
  api.allReduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
  api.errorString = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
  api.getAsyncError = reinterpret_cast<decltype(&ncclCommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
  api.commAbort = reinterpret_cast<decltype(&ncclCommAbort)>(dlsym(h, "ncclCommAbort"));
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.errorString &&
           api.getAsyncError && api.commAbort;
  return api;
}

}  // namespace

struct qb_ctx_s {
  int device = 0;
  qb_dtype dtype = QB_F64;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  OmegaConsts omega_consts{};

  // distributed (column sharding); nranks == 1 on a plain context
  int rank = 0, nranks = 1;
  int64_t col_offset = 0, n_global = 0;
  // row sharding (NEXT-2, tall-skinny A): this rank holds rows row_offset .. of an m_global-row A
  bool shard_rows = false;
  bool tf_gram = false;  // FP32 factorization in progress: CholeskyQR Grams on 3xTF32 (reading R18d)
  int64_t row_offset = 0, m_global = 0;
  ncclComm_t comm = nullptr;  // set on NCCL-distributed contexts (any nranks >= 1)
  qb_loopback loop = nullptr; // set on loopback-distributed contexts (in-process ranks, one GPU)
  bool dist = false;          // a distributed context (NCCL or loopback), any nranks >= 1

  DevBuf Awork, Qbar, Bbar, Om, Y, T1, Z, Zt, G, L, Rinv, W, P, parts, scal, status, Qf, Bf, Astage, Q32, B32,
      Qbar32, W32;
  int64_t kcap = 0, ldq = 0, ldb = 0, qbar_rows = 0, bbar_cols = 0;
  double* h_scal = nullptr;  // pinned: [0] r2, [1] sum B^2, [2..3] spare
  int* h_status = nullptr;   // pinned
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_gap = nullptr;  // QB_HOST_TIMING: end of the previous block (device gap between blocks)
  cudaEvent_t evp[6] = {};  // phase events: sketch, B, downdate (begin/end)
  std::vector<qb_block_stats> stats;
  // per-block phase spans (qb_block_stats ms_orth ... ms_power): an event pool reused every block
  std::vector<cudaEvent_t> tev;
  std::vector<int> tcat;
  int tused = 0;
  int64_t last_m = 0, last_n = 0, last_k = -1;  // the last qb_factor (for rqb_svd); -1: none
  // qb_factor_host: each finished block's Q_i / B_i is copied to these pinned host buffers on a
  // copy stream while the next block computes
  struct {
    void* Q = nullptr;
    void* B = nullptr;
    int64_t ldq = 0, ldb = 0, kcap = 0;
  } hout;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t cap_stream = nullptr, cap_stream2 = nullptr;  // rqb_svd: CUDA-graph capture of a Jacobi sweep
  cudaStream_t aux_stream = nullptr;  // rqb_svd: the J updates beside the next step (no-graph mode)
  cudaEvent_t jev[5] = {};
  cudaEvent_t ev_copy = nullptr;
  DevBuf QB, R, Usv, Vsv, Ssv, Wsv, Ut, Vt, Usv32, Vsv32, Ssv32, Swork;  // rqb_svd
  DevBuf Rq, Qh, Qt, qvn1, qvn2, qperm, qtau, qv, qparts, Rq32, Qh32, qw, qw2;  // qb_pivoted_qr
  DevBuf Xsave;  // orth_blocked with R: the projected block before its CholeskyQR2
  DevBuf X32, T32;  // FP32 contexts: FP32 copies of a CholeskyQR pass's X and T
  DevBuf X32b;      // FP32 contexts: RN_32 of CholeskyQR2's scratch (when the caller takes an FP32 copy)
  DevBuf Bsp;       // FP32 GEMM: a small B operand split into hi / lo
  DevBuf Jx, Jj, Jpart, Jw, Jint, Jsig, Jpairs;  // rqb_svd: block one-sided Jacobi (svd.cuh)
  DevBuf Srec, Strace;  // small_loop: results and per-block records; phase trace
  DevBuf Jq2, Jm2;      // rqb_svd QR preconditioning (experiment)
  int jac_pairs_nblk = 0, jac_sweeps = 0;
  double last_r2 = 0.0;  // ||A - QB||_F^2 of the last factorization (rqb_svd's tail rule)
  int block_fallbacks = 0;
  const double* outQ = nullptr;
  const double* outB = nullptr;
};

// In-process loopback group ("loopback"): nranks contexts of ONE process on ONE
// GPU, each driven by its own host thread, exchange their sums through this object instead of
// NCCL.  A collective is host-synchronised: every rank finishes its stream, meets the others at
// a host barrier, rank 0 sums all ranks' buffers in rank order with ONE kernel over all ranks'
// data, and after a second barrier every rank copies the sum back.  No kernel ever waits on
// another rank's kernel (B200_PROFILING.md: such ranks on one GPU must not spin on each other).
struct qb_loopback_s {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::string why;
  double* bufs[QB_LOOPBACK_MAX_RANKS] = {};
  size_t counts[QB_LOOPBACK_MAX_RANKS] = {};
  int device = -1;      // the one device of every member
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  double timeout_s = 600.0;

  // false if the group was (or gets) aborted, or nobody else arrives within timeout_s
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const uint64_t g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool done = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || aborted; });
    if (gen != g) return true;
    if (!done && !aborted) {
      aborted = true;
      why = "loopback barrier timed out";
      cv.notify_all();
    }
    return false;
  }
  void abort(const char* reason) {
    std::lock_guard<std::mutex> lk(mu);
    if (!aborted) why = reason;
    aborted = true;
    cv.notify_all();
  }
};

namespace {

qb_status fail(qb_ctx c, qb_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define QB_CUDA(call)                                                                             \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? QB_ERR_OOM : QB_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                             \
  } while (0)

#define QB_TRY(expr)                 \
  do {                               \
    qb_status s_ = (expr);           \
    if (s_ != QB_OK) return s_;      \
  } while (0)

// The dynamic shared-memory limit of a >48 KB kernel is an attribute of the current device's
// context: set it once per kernel and device (one bit per device; several host threads may
// race to set it, which is harmless).  Callers have selected ctx->device.
#define QB_SMEM_ATTR(kern, bytes)                                                                  \
  do {                                                                                             \
    static std::atomic<uint64_t> attr_mask_{0};                                                    \
    const uint64_t bit_ = uint64_t{1} << (ctx->device & 63);                                       \
    if (!(attr_mask_.load(std::memory_order_acquire) & bit_)) {                                    \
      QB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (bytes)));   \
      attr_mask_.fetch_or(bit_, std::memory_order_acq_rel);                                        \
    }                                                                                              \
  } while (0)

// NVTX range for the duration of a scope (the step names of SURVEY.md §5: K1 ... K8, C1 ...).
struct NvtxPhase {  // consecutive phases of one scope: each call closes the previous range
  bool on = false;
  void operator()(const char* name) {
    if (on) nvtxRangePop();
    nvtxRangePushA(name);
    on = true;
  }
  ~NvtxPhase() {
    if (on) nvtxRangePop();
  }
};
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int debug_env(const char* name) {
  const char* v = getenv(name);
  return v ? atoi(v) : 0;
}

qb_status ensure(qb_ctx ctx, DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes) return QB_OK;
  // kernels already queued on the context stream may still read the old buffer
  if (b.p && ctx->stream) QB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (b.p) QB_CUDA(cudaFree(b.p));
  b.p = nullptr;
  b.bytes = 0;
  QB_CUDA(cudaMalloc(&b.p, std::max<size_t>(bytes, 256)));
  b.bytes = std::max<size_t>(bytes, 256);
  return QB_OK;
}

qb_status check_launch(qb_ctx ctx, const char* what) {
  ++ctx->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, QB_ERR_CUDA, "launch %s: %s", what, cudaGetErrorString(e));
  // QB_DEBUG_SYNC=1: synchronize after every launch (localises asynchronous faults)
  static const int sync_each = debug_env("QB_DEBUG_SYNC");
  if (sync_each) {
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail(ctx, QB_ERR_CUDA, "after %s: %s", what, cudaGetErrorString(e));
  }
  return QB_OK;
}

double comm_timeout_s() {
  static const double t = getenv("QB_COMM_TIMEOUT_S") ? atof(getenv("QB_COMM_TIMEOUT_S")) : 600.0;
  return t > 0 ? t : 600.0;
}

// Host wait for the context stream.  On an NCCL context the wait polls the communicator's
// asynchronous error state and gives up after QB_COMM_TIMEOUT_S seconds (default 600): a peer
// that died or diverged would otherwise hang the collective forever.  The communicator is then
// aborted (its pending collectives are cancelled) and the context is unusable.
qb_status stream_wait(qb_ctx ctx) {
  if (!ctx->comm) {
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    return QB_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  for (;;) {
    const cudaError_t e = cudaStreamQuery(ctx->stream);
    if (e == cudaSuccess) return QB_OK;
    if (e != cudaErrorNotReady)
      return fail(ctx, QB_ERR_CUDA, "stream: %s", cudaGetErrorString(e));
    ncclResult_t ae = ncclSuccess;
    if (nccl().getAsyncError(ctx->comm, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
      nccl().commAbort(ctx->comm);
      ctx->comm = nullptr;
      return fail(ctx, QB_ERR_NCCL, "NCCL asynchronous error: %s", nccl().errorString(ae));
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > comm_timeout_s()) {
      nccl().commAbort(ctx->comm);
      ctx->comm = nullptr;
      return fail(ctx, QB_ERR_NCCL, "collective timed out after %.0f s (QB_COMM_TIMEOUT_S)", comm_timeout_s());
    }
    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// Loopback allreduce (see qb_loopback_s): in place, rank order, identical result on every rank.
qb_status loopback_allreduce(qb_ctx ctx, double* buf, size_t count) {
  qb_loopback G = ctx->loop;
  QB_CUDA(cudaStreamSynchronize(ctx->stream));  // this rank's buffer is final
  {
    std::lock_guard<std::mutex> lk(G->mu);
    G->bufs[ctx->rank] = buf;
    G->counts[ctx->rank] = count;
  }
  if (!G->barrier()) return fail(ctx, QB_ERR_NCCL, "loopback group aborted (%s)", G->why.c_str());
  if (ctx->rank == 0) {
    qb_status st = QB_OK;
    for (int r = 1; r < G->nranks; ++r)
      if (G->counts[r] != count) st = fail(ctx, QB_ERR_NCCL, "loopback allreduce: rank %d has %zu elements, rank 0 %zu", r, G->counts[r], count);
    if (st == QB_OK && G->scratch_bytes < count * sizeof(double)) {
      if (G->scratch) cudaFree(G->scratch);
      G->scratch = nullptr;
      G->scratch_bytes = 0;
      if (cudaMalloc(&G->scratch, count * sizeof(double)) != cudaSuccess) {
        G->scratch = nullptr;
        st = fail(ctx, QB_ERR_OOM, "loopback allreduce: scratch of %zu doubles", count);
      } else {
        G->scratch_bytes = count * sizeof(double);
      }
    }
    if (st == QB_OK) {
      LoopPtrs in{};
      for (int r = 0; r < G->nranks; ++r) in.p[r] = G->bufs[r];
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)count + 255) / 256, 8 * ctx->num_sms));
      loopback_sum_kernel<<<grid, 256, 0, ctx->stream>>>(in, G->nranks, (int64_t)count, static_cast<double*>(G->scratch));
      st = check_launch(ctx, "loopback_sum");
      if (st == QB_OK && cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = fail(ctx, QB_ERR_CUDA, "loopback sum failed");
    }
    if (st != QB_OK) {
      G->abort("rank 0 failed in a loopback allreduce");
      return st;
    }
  }
  if (!G->barrier()) return fail(ctx, QB_ERR_NCCL, "loopback group aborted (%s)", G->why.c_str());
  QB_CUDA(cudaMemcpyAsync(buf, G->scratch, count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QB_OK;
}

// Sum `count` doubles across the ranks of a distributed context, in place on the context
// stream (no-op on a plain context): NCCL, or the in-process loopback group.
qb_status allreduce_sum(qb_ctx ctx, double* buf, size_t count) {
  if (count == 0) return QB_OK;
  if (ctx->loop) return loopback_allreduce(ctx, buf, count);
  if (!ctx->comm) return QB_OK;
  nvtxRangePushA("C1 allreduce");
  ncclResult_t r = nccl().allReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream);
  nvtxRangePop();
  if (r != ncclSuccess) return fail(ctx, QB_ERR_NCCL, "ncclAllReduce: %s", nccl().errorString(r));
  return QB_OK;
}

// ---------------------------------------------------------------- tensor maps
// 3D view {16, K, rows/16} of an MN-contiguous operand (rows % 16 == 0): box {16, BK, box_chunks}.
qb_status make_map3d(qb_ctx ctx, CUtensorMap* map, const double* ptr, uint64_t rows, uint64_t K, int64_t ld,
                     uint32_t box_chunks) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || ((ld * 8) & 15) != 0 || rows % 16 != 0)
    return fail(ctx, QB_ERR_INVALID_ARG, "3D TMA operand not aligned");
  cuuint64_t dims[3] = {16, K, rows / 16};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 8, 128};
  cuuint32_t box[3] = {16, GEMM_BK, box_chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, QB_ERR_CUDA, "cuTensorMapEncodeTiled (3D) failed (%d)", (int)r);
  return QB_OK;
}

qb_status make_map(qb_ctx ctx, CUtensorMap* map, const double* ptr, uint64_t inner, uint64_t outer, int64_t ld,
                   uint32_t box_inner, uint32_t box_outer) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || ((ld * 8) & 15) != 0)
    return fail(ctx, QB_ERR_INVALID_ARG, "TMA operand not 16-byte aligned (ptr %p, ld %lld)", (const void*)ptr,
                (long long)ld);
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, QB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return QB_OK;
}

// ---------------------------------------------------------------- GEMM launcher
template <int LAYOUT, int BN, int EPI>
qb_status launch_gemm_t(qb_ctx ctx, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                        const GemmParams& p, int splits) {
  using Cfg = GemmCfg<BN, EPI>;
  auto kern = gemm_f64_kernel<LAYOUT, BN, EPI>;
  QB_SMEM_ATTR(kern, Cfg::SMEM_BYTES);
  dim3 grid(p.tiles_m * p.tiles_n, splits);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream>>>(ta, tb, tc, p);
  return check_launch(ctx, "gemm_f64");
}

constexpr int kBN = 64;

// out_elems > 0 (FP64 products): the split-K reduction's cost counts too for large outputs — it
// reads s partials of the output and writes it once (≈ 3 TB/s; ≈ 2 us per unit of the model's
// wave x k-tile time), which outweighs the wave-quantisation gain of splitting a short-K product with
// a large output (T's X T and re-projection updates: 55-100 us reductions on 100-340 us products).
int choose_splits(int tiles, int nkt, int slots, int max_splits, double out_elems = 0.0) {
  static const int no_rcost = debug_env("QB_SPLIT_NO_RCOST");
  int best = 1;
  double best_t = 1e300;
  for (int s = 1; s <= max_splits; ++s) {
    const int per = (nkt + s - 1) / s;
    if (s > 1 && per < 4) break;
    const int units = tiles * s;
    const int waves = (units + slots - 1) / slots;
    // counted for large outputs only (>= 4M entries, 32 MB per partial: T, T1, C5); at C3's 10 MB
    // partials the model overestimates the reduction and its choice measured slower (45.7 -> 47.7 ms)
    const double rbytes = (s + 1) * out_elems * 8.0;
    const double reduce_units = (s > 1 && !no_rcost && out_elems >= 4e6) ? rbytes / 3e12 * 1e6 / 2.0 : 0.0;
    const double t = waves * (per + 3.0) * (s > 1 ? 1.0 + 0.003 * s : 1.0) + reduce_units;
    if (t < best_t * 0.995) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

// C = opA * opB.  epi: EPI_STORE_COL (C[i + j*ldc]), EPI_STORE_ROW (C[i*ldc + j]) or
// EPI_SUB_COL (C[i + j*ldc] -= ..., per-CTA sum of squares into ctx->parts when
// want_norm; *nparts receives the number of partials).  For the STORE epilogues the
// K dimension may be split; then partials land in ctx->P and are reduced in a fixed order
// (with the sum of squares of C into ctx->parts when want_norm).
template <int BN>
qb_status dispatch_gemm(qb_ctx ctx, int layout, int epi, const CUtensorMap& ta, const CUtensorMap& tb,
                        const CUtensorMap& tc, const GemmParams& p, int splits) {
  if (layout == GEMM_NN) {
    if (epi == EPI_STORE_COL) return launch_gemm_t<GEMM_NN, BN, EPI_STORE_COL>(ctx, ta, tb, tc, p, splits);
    if (epi == EPI_STORE_ROW) return launch_gemm_t<GEMM_NN, BN, EPI_STORE_ROW>(ctx, ta, tb, tc, p, splits);
    return launch_gemm_t<GEMM_NN, BN, EPI_SUB_COL>(ctx, ta, tb, tc, p, splits);
  }
  if (epi == EPI_STORE_COL) return launch_gemm_t<GEMM_TN, BN, EPI_STORE_COL>(ctx, ta, tb, tc, p, splits);
  if (epi == EPI_STORE_ROW) return launch_gemm_t<GEMM_TN, BN, EPI_STORE_ROW>(ctx, ta, tb, tc, p, splits);
  return launch_gemm_t<GEMM_TN, BN, EPI_SUB_COL>(ctx, ta, tb, tc, p, splits);
}

// C = opA * opB.  epi: EPI_STORE_COL (C[i + j*ldc]), EPI_STORE_ROW (C[i*ldc + j]) or
// EPI_SUB_COL (C[i + j*ldc] -= ..., per-CTA sum of squares into ctx->parts when
// want_norm; *nparts receives the number of partials).  The K dimension may be split
// (fixed-order reduction of partials in ctx->P, the sum of squares of C into ctx->parts
// when want_norm).  Tile width: 64 (two CTAs per SM), or 128 (one CTA per SM, twice the
// work per tile) for an unsplit subtract-update such as the downdate A -= Q_i B_i, whose
// K = b is short and whose per-tile prologue/epilogue would otherwise show.
qb_status gemm(qb_ctx ctx, int layout, int epi, int M, int N, int K, const double* A, int64_t lda, const double* B,
               int64_t ldb, double* C, int64_t ldc, bool want_norm, int64_t* nparts, bool allow_split = true,
               const int* gate = nullptr) {
  if (nparts) *nparts = 0;
  if (M <= 0 || N <= 0) return QB_OK;
  // a short M wastes most of the 128-row tile (C2's B_i = Q_i^T A at w = 64: half of it): compute
  // C^T = op(B)^T op(A)^T instead (the same operands, roles and store orientation swapped)
  static const int no_swap = debug_env("QB_GEMM_NO_SWAP");
  if (!no_swap && epi != EPI_SUB_COL && M < GEMM_BM && N >= 2 * GEMM_BM)
    return gemm(ctx, layout, epi == EPI_STORE_COL ? EPI_STORE_ROW : EPI_STORE_COL, N, M, K, B, ldb, A, lda, C, ldc,
                want_norm, nparts, allow_split, gate);
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.nkt = (K + GEMM_BK - 1) / GEMM_BK;
  p.gate = gate;
  p.tiles_m = (M + GEMM_BM - 1) / GEMM_BM;
  int bn = 64;
  p.tiles_n = (N + bn - 1) / bn;
  int splits = 1;
  if (allow_split)
    splits = choose_splits(p.tiles_m * p.tiles_n, p.nkt, ctx->num_sms * GemmCfg<64>::MIN_BLOCKS, 296,
                           static_cast<double>(M) * N);
  const bool subtract = epi == EPI_SUB_COL;
  static const int wide_env = debug_env("QB_WIDE_DOWNDATE");  // experiment: 1 = 128-wide tiles
  if (subtract && splits == 1 && wide_env > 0 && N >= 2048) {
    bn = 128;
    p.tiles_n = (N + bn - 1) / bn;
  }
  p.kt_per_split = (p.nkt + splits - 1) / splits;
  splits = (p.nkt + p.kt_per_split - 1) / p.kt_per_split;
  if (splits < 1) splits = 1;
  if (subtract && splits > 1) epi = EPI_STORE_COL;  // split products are summed, then subtracted
  p.raster_m_fast = p.tiles_m <= p.tiles_n ? 1 : 0;
  const int tiles = p.tiles_m * p.tiles_n;

  CUtensorMap ta, tb, tc;
  int a3d = 0, b3d = 0;
  if (layout == GEMM_NN) {
    static const int no3d = debug_env("QB_NO_TMA3D");
    a3d = !no3d && M % 16 == 0;
    b3d = !no3d && N % 16 == 0;
    if (a3d) QB_TRY(make_map3d(ctx, &ta, A, M, K, lda, GEMM_BM / 16));
    else QB_TRY(make_map(ctx, &ta, A, M, K, lda, 16, GEMM_BK));
    if (b3d) QB_TRY(make_map3d(ctx, &tb, B, N, K, ldb, bn / 16));
    else QB_TRY(make_map(ctx, &tb, B, N, K, ldb, 16, GEMM_BK));
  } else {
    QB_TRY(make_map(ctx, &ta, A, K, M, lda, 16, GEMM_BM));
    QB_TRY(make_map(ctx, &tb, B, K, N, ldb, 16, bn));
  }
  p.a3d = a3d;
  p.b3d = b3d;
  tc = ta;

  if (epi == EPI_SUB_COL) {
    QB_TRY(make_map(ctx, &tc, C, M, N, ldc, 16, bn));  // the C tile is prefetched by TMA
    p.C = C;
    p.ldc = ldc;
    p.split_stride = 0;
    if (want_norm) {
      QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)tiles));
      p.norm_partials = ctx->parts.d();
      if (nparts) *nparts = tiles;
    }
    return bn == 128 ? dispatch_gemm<128>(ctx, layout, epi, ta, tb, tc, p, 1)
                     : dispatch_gemm<64>(ctx, layout, epi, ta, tb, tc, p, 1);
  }

  if (splits == 1) {
    p.C = C;
    p.ldc = ldc;
    QB_TRY(dispatch_gemm<64>(ctx, layout, epi, ta, tb, tc, p, 1));
    if (want_norm) {
      // sum of squares of the stored result (rows x cols in "strided-row" form)
      const int64_t rows = epi == EPI_STORE_ROW ? M : N, cols = epi == EPI_STORE_ROW ? N : M;
      const int grid = (int)std::min<int64_t>(rows, 4 * ctx->num_sms);
      QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
      sumsq_kernel<double><<<grid, RED_THREADS, 0, ctx->stream>>>(C, cols, rows, ldc, ctx->parts.d());
      QB_TRY(check_launch(ctx, "sumsq"));
      if (nparts) *nparts = grid;
    }
    return QB_OK;
  }

  // split-K: partials in the output layout, then a fixed-order reduction
  const int64_t rows = epi == EPI_STORE_ROW ? M : N, cols = epi == EPI_STORE_ROW ? N : M;
  const int64_t ldp = round_up(cols, 2);
  const int64_t stride = rows * ldp;
  QB_TRY(ensure(ctx, ctx->P, sizeof(double) * (size_t)(stride * splits)));
  p.C = ctx->P.d();
  p.ldc = ldp;
  p.split_stride = stride;
  QB_TRY(dispatch_gemm<64>(ctx, layout, epi, ta, tb, tc, p, splits));
  const int64_t total = rows * cols;
  const int rsub = splitk_sub(total, splits, ctx->num_sms);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total * rsub + RED_THREADS - 1) / RED_THREADS, 8 * ctx->num_sms));
  double* sq = nullptr;
  if (want_norm) {
    QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
    sq = ctx->parts.d();
    if (nparts) *nparts = grid;
  }
  splitk_reduce_kernel<<<grid, RED_THREADS, 0, ctx->stream>>>(ctx->P.d(), splits, stride, rows, cols, ldp, C, ldc, sq,
                                                               gate, subtract ? 1 : 0, nullptr, 0, rsub);
  return check_launch(ctx, "splitk_reduce");
}

template <typename Tin, typename Tout>
qb_status launch_convert(qb_ctx ctx, const Tin* in, int64_t ldi, int64_t rows, int64_t cols, Tout* out, int64_t ldo,
                         const int* gate = nullptr);

// ---------------------------------------------------------------- FP32 (3xTF32 tcgen05) GEMM
// K-major operand boxes use the plain 128-byte swizzle (SWIZZLE_128B), MN-major ones the
// 32-byte-atom variant that the MN-major TF32 descriptor expects (SWIZZLE_128B_ATOM_32B); the
// subtract-update's C tile is unswizzled (SWIZZLE_NONE).
qb_status make_map_f32(qb_ctx ctx, CUtensorMap* map, const float* ptr, uint64_t inner, uint64_t outer, int64_t ld,
                       uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || ((ld * 4) & 15) != 0)
    return fail(ctx, QB_ERR_INVALID_ARG, "TMA operand not 16-byte aligned (ptr %p, ld %lld)", (const void*)ptr,
                (long long)ld);
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, QB_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", (int)r);
  return QB_OK;
}

// 3D view {32, K, rows/32} of an MN-contiguous FP32 operand (rows % 32 == 0).
qb_status make_map3d_f32(qb_ctx ctx, CUtensorMap* map, const float* ptr, uint64_t rows, uint64_t K, int64_t ld,
                         uint32_t box_chunks) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || ((ld * 4) & 15) != 0 || rows % 32 != 0)
    return fail(ctx, QB_ERR_INVALID_ARG, "3D TMA operand (f32) not aligned");
  cuuint64_t dims[3] = {32, K, rows / 32};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4, 128};
  cuuint32_t box[3] = {32, TF_BK, box_chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, QB_ERR_CUDA, "cuTensorMapEncodeTiled (3D f32) failed (%d)", (int)r);
  return QB_OK;
}

template <int LAYOUT, int BN, int EPI, bool TS>
qb_status launch_tf_ts(qb_ctx ctx, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2,
                       const CUtensorMap& tc, const TfParams& p, int splits) {
  using Cfg = TfCfg<BN, EPI == TF_SUB_COL, TS>;
  auto kern = gemm_tf32_kernel<LAYOUT, BN, EPI, TS>;
  QB_SMEM_ATTR(kern, Cfg::SMEM_BYTES);
  const int units = p.tiles_m * p.tiles_n * splits;
  kern<<<std::min(units, ctx->num_sms), Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream>>>(ta, tb, tb2, tc, p);
  return check_launch(ctx, "gemm_tf32");
}

// A operand in TMEM (TS, more pipeline stages) unless QB_TF_SS=1 (both operands in shared memory)
template <int BN>
qb_status launch_tf_ares(qb_ctx ctx, const CUtensorMap& ta, const CUtensorMap& tbh, const CUtensorMap& tbl,
                         const CUtensorMap& tc, const TfParams& p) {
  using Cfg = TfAresCfg<BN>;
  auto kern = gemm_tf32_sub_ares_kernel<BN>;
  QB_SMEM_ATTR(kern, Cfg::SMEM_BYTES);
  const int units = p.tiles_m * p.tiles_n;
  kern<<<std::min(units, ctx->num_sms), TF_THREADS, Cfg::SMEM_BYTES, ctx->stream>>>(ta, tbh, tbl, tc, p);
  return check_launch(ctx, "gemm_tf32_sub_ares");
}

int tf_ss_mode() {
  static const int ss = debug_env("QB_TF_SS");
  return ss;
}

template <int LAYOUT, int BN, int EPI>
qb_status launch_tf_t(qb_ctx ctx, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2,
                      const CUtensorMap& tc, const TfParams& p, int splits) {
  if (tf_ss_mode()) return launch_tf_ts<LAYOUT, BN, EPI, false>(ctx, ta, tb, tb2, tc, p, splits);
  return launch_tf_ts<LAYOUT, BN, EPI, true>(ctx, ta, tb, tb2, tc, p, splits);
}

template <int BN>
qb_status dispatch_tf(qb_ctx ctx, int layout, int epi, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& tb2, const CUtensorMap& tc, const TfParams& p, int splits) {
  if (layout == GEMM_NN) {
    if (epi == TF_STORE_COL) return launch_tf_t<GEMM_NN, BN, TF_STORE_COL>(ctx, ta, tb, tb2, tc, p, splits);
    if (epi == TF_STORE_ROW) return launch_tf_t<GEMM_NN, BN, TF_STORE_ROW>(ctx, ta, tb, tb2, tc, p, splits);
    return launch_tf_t<GEMM_NN, BN, TF_SUB_COL>(ctx, ta, tb, tb2, tc, p, splits);
  }
  if (epi == TF_STORE_COL) return launch_tf_t<GEMM_TN, BN, TF_STORE_COL>(ctx, ta, tb, tb2, tc, p, splits);
  if (epi == TF_STORE_ROW) return launch_tf_t<GEMM_TN, BN, TF_STORE_ROW>(ctx, ta, tb, tb2, tc, p, splits);
  return launch_tf_t<GEMM_TN, BN, TF_SUB_COL>(ctx, ta, tb, tb2, tc, p, splits);
}

// FP32 operands, 3xTF32 products with FP32 accumulation.  epi TF_STORE_COL / TF_STORE_ROW
// write a DOUBLE C (column- / row-major); TF_SUB_COL updates a FLOAT column-major C -= result
// with the per-CTA FP64 sum of squares of the new C in ctx->parts (want_norm).  Split-K
// partials (STORE only) are FP64 and reduced in a fixed order as in gemm().
// TF_STORE_COL may also write an FP32 copy C32 (ld ldc32) of the result (= RN_32 of C).
qb_status gemm_tf(qb_ctx ctx, int layout, int epi, int M, int N, int K, const float* A, int64_t lda, const float* B,
                  int64_t ldb, void* C, int64_t ldc, bool want_norm, int64_t* nparts, bool allow_split = true,
                  const int* gate = nullptr, float* C32 = nullptr, int64_t ldc32 = 0) {
  if (nparts) *nparts = 0;
  if (M <= 0 || N <= 0) return QB_OK;
  TfParams p{};
  p.gate = gate;
  p.M = M;
  p.N = N;
  p.K = K;
  p.nkt = (K + TF_BK - 1) / TF_BK;
  p.tiles_m = (M + TF_BM - 1) / TF_BM;
  static const int bn_env = debug_env("QB_TF_BN");
  const int bn = bn_env ? bn_env : (N <= 64 ? 64 : 128);
  p.tiles_n = (N + bn - 1) / bn;
  const int tiles = p.tiles_m * p.tiles_n;
  int splits = 1;
  if (allow_split && epi != TF_SUB_COL) splits = choose_splits(tiles, p.nkt, ctx->num_sms, 148);
  p.kt_per_split = (p.nkt + splits - 1) / splits;
  splits = std::max(1, (p.nkt + p.kt_per_split - 1) / p.kt_per_split);
  p.raster_m_fast = p.tiles_m <= p.tiles_n ? 1 : 0;

  // A small B operand that many row tiles re-read (Ω, B_i, W, T) is split into hi / lo once
  // (tf32_split_kernel) instead of in every tile's stages
  static const int no_bsplit = debug_env("QB_TF_NO_BSPLIT");
  p.bsplit = !no_bsplit && p.tiles_m >= 4 && static_cast<int64_t>(K) * N <= (int64_t{4} << 20);
  const float* Bhi = B;
  float* Blo = nullptr;
  if (p.bsplit) {
    const int64_t outer = layout == GEMM_NN ? K : N, inner = layout == GEMM_NN ? N : K;
    QB_TRY(ensure(ctx, ctx->Bsp, sizeof(float) * (size_t)(2 * outer * ldb)));
    float* hi = static_cast<float*>(ctx->Bsp.p);
    Blo = hi + outer * ldb;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((outer * inner + 255) / 256, 4 * ctx->num_sms));
    tf32_split_kernel<<<grid, 256, 0, ctx->stream>>>(B, ldb, outer, inner, hi, Blo);
    QB_TRY(check_launch(ctx, "tf32_split"));
    Bhi = hi;
  }
  CUtensorMap ta, tb, tb2;
  auto map_b = [&](CUtensorMap* map, const float* ptr) -> qb_status {
    if (layout == GEMM_TN) return make_map_f32(ctx, map, ptr, K, N, ldb, TF_BK, bn, CU_TENSOR_MAP_SWIZZLE_128B);
    if (p.b3d) return make_map3d_f32(ctx, map, ptr, N, K, ldb, bn / 32);
    return make_map_f32(ctx, map, ptr, N, K, ldb, 32, TF_BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  };
  if (layout == GEMM_NN) {
    p.a3d = M % 32 == 0;
    p.b3d = N % 32 == 0 && N >= bn;
    if (p.a3d) QB_TRY(make_map3d_f32(ctx, &ta, A, M, K, lda, TF_BM / 32));
    else QB_TRY(make_map_f32(ctx, &ta, A, M, K, lda, 32, TF_BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
  } else {
    QB_TRY(make_map_f32(ctx, &ta, A, K, M, lda, TF_BK, TF_BM, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  QB_TRY(map_b(&tb, Bhi));
  if (p.bsplit) QB_TRY(map_b(&tb2, Blo));
  else tb2 = tb;
  CUtensorMap tc = ta;
  if (epi == TF_SUB_COL)
    QB_TRY(make_map_f32(ctx, &tc, static_cast<const float*>(C), M, N, ldc, TF_BM, TF_CSUB, CU_TENSOR_MAP_SWIZZLE_NONE));
  auto run = [&](int e, int s) -> qb_status {
    if (bn == 64) return dispatch_tf<64>(ctx, layout, e, ta, tb, tb2, tc, p, s);
    if (bn == 128) return dispatch_tf<128>(ctx, layout, e, ta, tb, tb2, tc, p, s);
    return fail(ctx, QB_ERR_INVALID_ARG, "QB_TF_BN must be 64 or 128");
  };

  if (epi == TF_SUB_COL) {
    p.C = C;
    p.ldc = ldc;
    p.splits = 1;
    if (want_norm) {  // one partial per persistent CTA
      const int grid = std::min(tiles, ctx->num_sms);
      QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
      p.norm_partials = ctx->parts.d();
      if (nparts) *nparts = grid;
    }
    // short K (the block size): A's row block stays in TMEM across the CTA's run of tiles
    static const int no_ares = debug_env("QB_TF_NO_ARES");
    if (!no_ares && layout == GEMM_NN && p.bsplit && K <= 4 * TF_BK) {
      if (bn == 64) return launch_tf_ares<64>(ctx, ta, tb, tb2, tc, p);
      if (bn == 128) return launch_tf_ares<128>(ctx, ta, tb, tb2, tc, p);
    }
    return run(TF_SUB_COL, 1);
  }
  p.splits = splits;
  const int64_t rows = epi == TF_STORE_ROW ? M : N, cols = epi == TF_STORE_ROW ? N : M;
  if (epi != TF_STORE_COL) C32 = nullptr;
  if (splits == 1) {
    p.C = C;
    p.ldc = ldc;
    p.C32 = C32;
    p.ldc32 = ldc32;
    QB_TRY(run(epi, 1));
    if (want_norm) {
      const int grid = (int)std::min<int64_t>(rows, 4 * ctx->num_sms);
      QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
      sumsq_kernel<double><<<grid, RED_THREADS, 0, ctx->stream>>>(static_cast<double*>(C), cols, rows, ldc, ctx->parts.d());
      QB_TRY(check_launch(ctx, "sumsq"));
      if (nparts) *nparts = grid;
    }
    return QB_OK;
  }
  const int64_t ldp = round_up(cols, 2);
  const int64_t stride = rows * ldp;
  QB_TRY(ensure(ctx, ctx->P, sizeof(double) * (size_t)(stride * splits)));
  p.C = ctx->P.d();
  p.ldc = ldp;
  p.split_stride = stride;
  QB_TRY(run(epi, splits));
  const int64_t total = rows * cols;
  const int rsub = splitk_sub(total, splits, ctx->num_sms);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total * rsub + RED_THREADS - 1) / RED_THREADS, 8 * ctx->num_sms));
  double* sq = nullptr;
  if (want_norm) {
    QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
    sq = ctx->parts.d();
    if (nparts) *nparts = grid;
  }
  splitk_reduce_kernel<<<grid, RED_THREADS, 0, ctx->stream>>>(ctx->P.d(), splits, stride, rows, cols, ldp,
                                                               static_cast<double*>(C), ldc, sq, gate, 0, C32,
                                                               ldc32, rsub);
  return check_launch(ctx, "splitk_reduce");
}

qb_status reduce_to_scal(qb_ctx ctx, int64_t nparts, int slot) {
  reduce_kernel<<<1, RED_THREADS, 0, ctx->stream>>>(ctx->parts.d(), nparts, ctx->scal.d(), slot);
  return check_launch(ctx, "reduce");
}

// ---------------------------------------------------------------- phase spans (qb_stats)
enum { PH_ORTH = 0, PH_ORTH_Z = 1, PH_REPROJ = 2, PH_POWER = 3, PH_N = 4 };
qb_status span_mark(qb_ctx ctx, int cat) {  // cat >= 0 opens a span, cat < 0 closes the open one
  if ((size_t)ctx->tused >= ctx->tev.size()) {
    cudaEvent_t e = nullptr;
    QB_CUDA(cudaEventCreate(&e));
    ctx->tev.push_back(e);
    ctx->tcat.push_back(-1);
  }
  ctx->tcat[ctx->tused] = cat;
  QB_CUDA(cudaEventRecord(ctx->tev[ctx->tused], ctx->stream));
  ++ctx->tused;
  return QB_OK;
}
// after the block's host synchronisation: the spans' device times per category
void span_collect(qb_ctx ctx, double* acc) {
  for (int c = 0; c < PH_N; ++c) acc[c] = 0.0;
  for (int i = 0; i + 1 < ctx->tused; i += 2) {
    float ms = 0.f;
    if (ctx->tcat[i] >= 0 && cudaEventElapsedTime(&ms, ctx->tev[i], ctx->tev[i + 1]) == cudaSuccess)
      acc[ctx->tcat[i]] += ms;
  }
  ctx->tused = 0;
}

// ---------------------------------------------------------------- CholeskyQR2
int* status_dev(qb_ctx ctx) { return static_cast<int*>(ctx->status.p); }

// T for one CholeskyQR pass from the Gram matrix in ctx->G (no host synchronisation):
// Newton-Schulz T = I - (G - I)/2 when ||G - I||_F <= 1e-8 (ns), else T = R^-1.
qb_status chol_inv(qb_ctx ctx, int w, int64_t m_rows, bool ns, const int* gate) {
  QB_SMEM_ATTR(chol_cluster_kernel, CHOL_SMEM);
  const int64_t ld = round_up(kMaxB, 16);
  // Newton-Schulz when ||G - I||_F <= 1e-8 (FP64: step error <= 1e-16), <= 1e-4 on FP32 contexts
  // (step error <= 7.5e-9, below FP32 rounding; reading R18c)
  const double ns_tol2 = !ns ? -1.0 : (ctx->dtype == QB_F32 ? 1e-8 : 1e-16);
  chol_cluster_kernel<<<CHOL_CTAS, CHOL_THREADS, CHOL_SMEM, ctx->stream>>>(
      ctx->G.d(), ld, w, m_rows, ctx->Rinv.d(), ld, status_dev(ctx), 1e-13, ns_tol2, gate, ctx->scal.d() + 4);
  return check_launch(ctx, "chol");
}

// One CholeskyQR pass: dst = src T, with T from chol_inv (all on the device; gated).
// FP32 contexts: src32 (optional) is RN_32(src) already in memory (ld lds32), else src is
// converted into ctx->X32; dst32 (optional) receives RN_32(dst) (ld ldd32); src32 != dst32.
// CholeskyQR2 of a panel small enough for one CTA's shared memory (small_cholqr_kernel, FP64 source)
bool small_orth(int64_t m, int w, bool row_distributed) {
  static const int no_small = debug_env("QB_NO_SMALL_ORTH");
  return !row_distributed && !no_small && w <= SCQR_MAX_W && m * w <= SCQR_MAX_ELEMS;
}

// FP32 factorizations (reading R18d): CholeskyQR reads only the FP32 copy of its source
bool tf_gram_on(qb_ctx ctx) {
  static const int gram64_env = debug_env("QB_GRAM64");
  static const int orth64 = debug_env("QB_ORTH64");
  return ctx->dtype == QB_F32 && ctx->tf_gram && !gram64_env && !orth64;
}

qb_status cholqr_pass(qb_ctx ctx, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t m, int w,
                      const int* gate, bool row_distributed, const float* src32 = nullptr, int64_t lds32 = 0,
                      float* dst32 = nullptr, int64_t ldd32 = 0) {
  const int64_t ldgb = round_up(kMaxB, 16);
  static const int orth64 = debug_env("QB_ORTH64");
  static const int gram64_env = debug_env("QB_GRAM64");
  const bool gram64 = gram64_env || !ctx->tf_gram;  // qb_orth and the small paths keep the FP64 Gram
  const bool tf = ctx->dtype == QB_F32 && !orth64;
  const float* X32 = src32;
  int64_t ld_x = lds32;
  if (tf && X32 == nullptr) {
    const int64_t ldx = round_up(m, 16);
    QB_TRY(ensure(ctx, ctx->X32, sizeof(float) * (size_t)(ldx * w)));
    QB_TRY(launch_convert(ctx, src, lds, m, w, static_cast<float*>(ctx->X32.p), ldx, gate));
    X32 = static_cast<const float*>(ctx->X32.p);
    ld_x = ldx;
  }
  if (tf && !gram64) {
    // FP32 factorizations (reading R18d): the Gram of the FP32 copy on the 3xTF32 tensor cores,
    // FP32 accumulation per 128-deep k chunk and FP64 across chunks and splits (relative error
    // ~1e-6, which CholeskyQR2 absorbs at the FP32 tolerances; QB_GRAM64=1 keeps it FP64)
    QB_TRY(gemm_tf(ctx, GEMM_TN, TF_STORE_COL, w, w, (int)m, X32, ld_x, X32, ld_x, ctx->G.d(), ldgb, false, nullptr,
                   true, gate));
  } else {
    QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_COL, w, w, (int)m, src, lds, src, lds, ctx->G.d(), ldgb, false, nullptr, true,
                gate));
  }
  if (row_distributed) QB_TRY(allreduce_sum(ctx, ctx->G.d(), (size_t)(ldgb * w)));  // G = sum_p src_p^T src_p
  // the shifted-CholeskyQR shift (reading R8) is sized for the GLOBAL row count of the panel:
  // the power step's Z on column shards has n_global rows, a row shard's Y / Q_i m_global
  const int64_t m_shift = !row_distributed ? m : (ctx->shard_rows ? ctx->m_global : ctx->n_global);
  QB_TRY(chol_inv(ctx, w, m_shift, true, gate));
  if (tf) {
    // FP32 contexts (reading R18c): X T on the 3xTF32 tensor cores from FP32 copies of X and T
    QB_TRY(ensure(ctx, ctx->T32, sizeof(float) * (size_t)(ldgb * ldgb)));
    float* T32 = static_cast<float*>(ctx->T32.p);
    QB_TRY(launch_convert(ctx, static_cast<const double*>(ctx->Rinv.d()), ldgb, w, w, T32, ldgb, gate));
    return gemm_tf(ctx, GEMM_NN, TF_STORE_COL, (int)m, w, w, X32, ld_x, T32, ldgb, dst, ldd, false, nullptr, true, gate,
                   dst32, ldd32);
  }
  QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)m, w, w, src, lds, ctx->Rinv.d(), ldgb, dst, ldd, false, nullptr, true,
              gate));
  if (dst32 != nullptr) QB_TRY(launch_convert(ctx, static_cast<const double*>(dst), ldd, m, w, dst32, ldd32, gate));
  return QB_OK;
}

// orth(src) -> dst: CholeskyQR2, where a pass whose Gram is already within 1e-8 of I takes
// the Newton-Schulz step instead of a factorization; a shifted first factorization (reading
// R8) triggers two more passes (shifted CholeskyQR3), gated on the device flag status[1].
// src and dst may alias; ctx->T1 is the scratch.  Nothing here synchronises with the host;
// failures surface in status[3], read at the end of the block.
// row_distributed: src holds this rank's rows of a matrix whose rows are spread over the
// ranks (the power step's Z = A^T Q on column shards); the Gram is summed with NCCL and the
// replicated T applied to the local rows.
// single = true ("cholqr1", reading R11b: the orth of line (3)/(6) when the re-projection and its
// CholeskyQR2 follow in the same block): the second pass runs only after a SHIFTED first factorization
// (then the whole shifted CholeskyQR3 runs); otherwise a factorized first pass is final.
// FP32 contexts: src32 / dst32 (optional) as in cholqr_pass; the FP32 copy of the scratch
// lives in ctx->X32b, so that no pass reads and writes the same FP32 buffer.
// When src and dst are different buffers, the first pass writes dst directly and a second
// pass goes through the scratch and back (gated copy), so the common single-pass case (a
// Newton-Schulz first pass, or cholqr1 without the shift) moves no data; in place, the first
// pass goes to the scratch.
qb_status cholqr2(qb_ctx ctx, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t m, int w,
                  bool row_distributed = false, bool single = false, const float* src32 = nullptr,
                  int64_t lds32 = 0, float* dst32 = nullptr, int64_t ldd32 = 0) {
  if (small_orth(m, w, row_distributed)) {
    // the whole CholeskyQR2 (all passes, fallback included) in one CTA for a small panel
    QB_SMEM_ATTR(small_cholqr_kernel, SCQR_SMEM);
    const double ns_tol2 = ctx->dtype == QB_F32 ? 1e-8 : 1e-16;
    small_cholqr_kernel<<<1, SCQR_THREADS, SCQR_SMEM, ctx->stream>>>(src, lds, dst, ldd, (int)m, w, single ? 1 : 0,
                                                                     ns_tol2, 1e-13, status_dev(ctx), dst32, ldd32,
                                                                     ctx->scal.d() + 4);
    return check_launch(ctx, "small_cholqr");
  }
  const int64_t ldt = round_up(m, 16);
  double* T = ctx->T1.d();
  float* T32 = nullptr;  // RN_32(T) when the caller wants dst32
  if (dst32 != nullptr) {
    QB_TRY(ensure(ctx, ctx->X32b, sizeof(float) * (size_t)(ldt * w)));
    T32 = static_cast<float*>(ctx->X32b.p);
  }
  const bool inplace = src == dst || (src32 != nullptr && src32 == dst32);
  zero_ints_kernel<<<1, 32, 0, ctx->stream>>>(status_dev(ctx) + 1, 2);
  QB_TRY(check_launch(ctx, "zero_flags"));
  // second pass only after a factorization (status[2]); a Newton-Schulz first pass is final
  const int* gate2 = status_dev(ctx) + (single ? 1 : 2);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m * w + 255) / 256, 8 * ctx->num_sms));
  if (inplace) {
    QB_TRY(cholqr_pass(ctx, src, lds, T, ldt, m, w, nullptr, row_distributed, src32, lds32, T32, ldt));
    QB_TRY(cholqr_pass(ctx, T, ldt, dst, ldd, m, w, gate2, row_distributed, T32, ldt, dst32, ldd32));
    gated_copy_kernel<<<grid, 256, 0, ctx->stream>>>(T, ldt, dst, ldd, m, w, gate2, T32, ldt, dst32, ldd32, 0);
  } else {
    QB_TRY(cholqr_pass(ctx, src, lds, dst, ldd, m, w, nullptr, row_distributed, src32, lds32, dst32, ldd32));
    QB_TRY(cholqr_pass(ctx, dst, ldd, T, ldt, m, w, gate2, row_distributed, dst32, ldd32, T32, ldt));
    gated_copy_kernel<<<grid, 256, 0, ctx->stream>>>(T, ldt, dst, ldd, m, w, gate2, T32, ldt, dst32, ldd32, 1);
  }
  QB_TRY(check_launch(ctx, "gated_copy"));
  // shifted first factorization (status[1]): two more passes, dst -> T -> dst
  QB_TRY(cholqr_pass(ctx, dst, ldd, T, ldt, m, w, status_dev(ctx) + 1, row_distributed, dst32, ldd32, T32, ldt));
  QB_TRY(cholqr_pass(ctx, T, ldt, dst, ldd, m, w, status_dev(ctx) + 1, row_distributed, T32, ldt, dst32, ldd32));
  return QB_OK;
}

// Orthonormalise the m x l column-major panel X (ld ldx) in place for any l: 256 columns at a
// time, two block Gram-Schmidt projections against the finished columns, then CholeskyQR2.
// Uses ctx->Wsv (l x 256 row-major coefficients).
qb_status orth_blocked(qb_ctx ctx, double* X, int64_t ldx, int64_t m, int64_t l, double* R = nullptr,
                       int64_t ldr = 0) {
  // R (optional, l x l column-major, ld ldr): X_in = Q R assembled from the projections themselves
  // (block column j: the two passes' coefficients above the diagonal block, Q_j^T of the projected
  // block on it, zero below) instead of a separate l x l x m product Q^T X_in
  const int64_t bp = round_up(kMaxB, 16);
  QB_TRY(ensure(ctx, ctx->Wsv, sizeof(double) * (size_t)(round_up(l, 16) * bp)));
  if (R != nullptr) {
    QB_TRY(ensure(ctx, ctx->Xsave, sizeof(double) * (size_t)(ldx * kMaxB)));
    QB_CUDA(cudaMemsetAsync(R, 0, sizeof(double) * (size_t)(ldr * l), ctx->stream));
  }
  for (int64_t j0 = 0; j0 < l; j0 += kMaxB) {
    const int64_t w = std::min<int64_t>(kMaxB, l - j0);
    double* Xj = X + j0 * ldx;
    for (int pass = 0; pass < 2 && j0 > 0; ++pass) {  // Xj -= X (X^T Xj), twice
      QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_ROW, (int)j0, (int)w, (int)m, X, ldx, Xj, ldx, ctx->Wsv.d(), bp, false,
                  nullptr));
      if (R != nullptr) {
        add_rowmajor_kernel<<<(int)std::min<int64_t>((j0 * w + 255) / 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(
            R + j0 * ldr, ldr, ctx->Wsv.d(), bp, j0, w);
        QB_TRY(check_launch(ctx, "add_rowmajor"));
      }
      QB_TRY(gemm(ctx, GEMM_NN, EPI_SUB_COL, (int)m, (int)w, (int)j0, X, ldx, ctx->Wsv.d(), bp, Xj, ldx, false,
                  nullptr));
    }
    if (R != nullptr)
      QB_CUDA(cudaMemcpy2DAsync(ctx->Xsave.p, ldx * 8, Xj, ldx * 8, m * 8, w, cudaMemcpyDeviceToDevice, ctx->stream));
    QB_TRY(cholqr2(ctx, Xj, ldx, Xj, ldx, m, (int)w));
    if (R != nullptr)  // R_jj = Q_j^T (the projected block)
      QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_COL, (int)w, (int)w, (int)m, Xj, ldx, ctx->Xsave.d(), ldx,
                  R + j0 + j0 * ldr, ldr, false, nullptr));
  }
  return QB_OK;
}

bool skip_orth_flag(unsigned flags) { return (flags & QB_SKIP_POWER_ORTH) != 0; }

// the block's device flags, and scal[4..5]: its kappa-proxy (max / min R diagonal of the first factorization)
qb_status reset_flags(qb_ctx ctx) {
  reset_block_kernel<<<1, 32, 0, ctx->stream>>>(status_dev(ctx), ctx->scal.d() + 4);
  return check_launch(ctx, "reset_block");
}

// kind 0: FP64 Ω; 1: FP32 Ω (qb_omega on an FP32 context); 2: FP64 buffer holding RN_32(Ω).
qb_status launch_omega(qb_ctx ctx, uint64_t seed, int64_t row0, int64_t row1, int64_t col0, int64_t w, void* out,
                       int64_t ldo, int kind) {
  const int64_t npairs = ((row1 - 1) >> 1) - (row0 >> 1) + 1;
  const int64_t total = npairs * w;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 32 * ctx->num_sms));
  if (kind == 0)
    omega_kernel<double><<<grid, 256, 0, ctx->stream>>>(seed, row0, row1, col0, w, static_cast<double*>(out), ldo,
                                                        ctx->omega_consts);
  else if (kind == 1)
    omega_kernel<float><<<grid, 256, 0, ctx->stream>>>(seed, row0, row1, col0, w, static_cast<float*>(out), ldo,
                                                       ctx->omega_consts);
  else
    omega_kernel<double, true><<<grid, 256, 0, ctx->stream>>>(seed, row0, row1, col0, w, static_cast<double*>(out),
                                                              ldo, ctx->omega_consts);
  return check_launch(ctx, "omega");
}

template <typename Tin, typename Tout>
qb_status launch_convert(qb_ctx ctx, const Tin* in, int64_t ldi, int64_t rows, int64_t cols, Tout* out, int64_t ldo,
                         const int* gate) {
  if (rows <= 0 || cols <= 0) return QB_OK;
  const int64_t total = rows * cols;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 16 * ctx->num_sms));
  convert_kernel<Tin, Tout><<<grid, 256, 0, ctx->stream>>>(in, ldi, rows, cols, out, ldo, gate);
  return check_launch(ctx, "convert");
}

qb_status grow_factors(qb_ctx ctx, int64_t m, int64_t n, int64_t need, int64_t kmax) {
  if (need <= ctx->kcap && ctx->qbar_rows == m && ctx->bbar_cols == n) return QB_OK;
  int64_t cap = std::max<int64_t>(need, std::min<int64_t>(kmax, std::max<int64_t>(2 * ctx->kcap, 1024)));
  cap = std::min<int64_t>(std::max<int64_t>(cap, need), std::max<int64_t>(kmax, need));
  const int64_t ldq = round_up(m, 16), ldb = round_up(n, 16);
  DevBuf nq, nb;
  QB_CUDA(cudaMalloc(&nq.p, sizeof(double) * (size_t)(ldq * cap)));
  nq.bytes = sizeof(double) * (size_t)(ldq * cap);
  QB_CUDA(cudaMalloc(&nb.p, sizeof(double) * (size_t)(ldb * cap)));
  nb.bytes = sizeof(double) * (size_t)(ldb * cap);
  if (ctx->Qbar.p && ctx->qbar_rows == m && ctx->bbar_cols == n && ctx->kcap > 0) {
    QB_CUDA(cudaMemcpyAsync(nq.p, ctx->Qbar.p, sizeof(double) * (size_t)(ldq * ctx->kcap), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    QB_CUDA(cudaMemcpyAsync(nb.p, ctx->Bbar.p, sizeof(double) * (size_t)(ldb * ctx->kcap), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if (ctx->copy_stream) QB_CUDA(cudaStreamSynchronize(ctx->copy_stream));  // block copies read the old factors
  if (ctx->dtype == QB_F32) {  // FP32 copy of Q̄ (the published Q and the residual GEMMs' operand)
    DevBuf nq32;
    QB_CUDA(cudaMalloc(&nq32.p, sizeof(float) * (size_t)(ldq * cap)));
    nq32.bytes = sizeof(float) * (size_t)(ldq * cap);
    if (ctx->Qbar32.p && ctx->qbar_rows == m && ctx->bbar_cols == n && ctx->kcap > 0) {
      QB_CUDA(cudaMemcpyAsync(nq32.p, ctx->Qbar32.p, sizeof(float) * (size_t)(ldq * ctx->kcap),
                              cudaMemcpyDeviceToDevice, ctx->stream));
      QB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (ctx->Qbar32.p) QB_CUDA(cudaFree(ctx->Qbar32.p));
    ctx->Qbar32 = nq32;
  }
  if (ctx->Qbar.p) QB_CUDA(cudaFree(ctx->Qbar.p));
  if (ctx->Bbar.p) QB_CUDA(cudaFree(ctx->Bbar.p));
  ctx->Qbar = nq;
  ctx->Bbar = nb;
  ctx->kcap = cap;
  // re-projection coefficients W = Q̄^T Q_i (up to kcap x b, row-major), sized with Q̄
  QB_TRY(ensure(ctx, ctx->W, sizeof(double) * (size_t)(cap * round_up(kMaxB, 16))));
  ctx->ldq = ldq;
  ctx->ldb = ldb;
  ctx->qbar_rows = m;
  ctx->bbar_cols = n;
  return QB_OK;
}

qb_status init_ctx(qb_ctx ctx, int device, qb_dtype dtype, void* stream) {
  if (dtype != QB_F64 && dtype != QB_F32) return fail(ctx, QB_ERR_INVALID_ARG, "bad dtype %d", (int)dtype);
  int ndev = 0;
  QB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ctx, QB_ERR_INVALID_ARG, "bad device %d of %d", device, ndev);
  ctx->device = device;
  ctx->dtype = dtype;
  QB_CUDA(cudaSetDevice(device));
  int major = 0, minor = 0;
  QB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  QB_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  if (major != 10 || minor != 0)
    return fail(ctx, QB_ERR_UNSUPPORTED, "this build targets sm_100a (B200); device is sm_%d%d", major, minor);
  QB_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    // blocking stream: implicitly ordered after work on the legacy default stream
    QB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault));
    ctx->own_stream = true;
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  QB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(ctx, QB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (int k = 1; k <= 11; ++k) ctx->omega_consts.log_c[k] = 2.0 / (2.0 * k + 1.0);  // IEEE RN quotient
  ctx->omega_consts.log_c12 = 2.0 / 25.0;
  QB_CUDA(cudaMallocHost(&ctx->h_scal, 8 * sizeof(double)));
  QB_CUDA(cudaMallocHost(&ctx->h_status, 8 * sizeof(int)));
  QB_TRY(ensure(ctx, ctx->scal, 8 * sizeof(double)));
  QB_TRY(ensure(ctx, ctx->status, 8 * sizeof(int)));
  QB_CUDA(cudaEventCreate(&ctx->ev0));
  QB_CUDA(cudaEventCreate(&ctx->ev1));
  for (auto& e : ctx->evp) QB_CUDA(cudaEventCreate(&e));
  return QB_OK;
}

// Hand out Q̄ (column-major, ld ldq) and B̄ (row-major, ld ldb): the FP64 factors, or for an
// FP32 context their RN_32 copies in context-owned FP32 buffers with the same layouts.
// NCCL communicator of a distributed context (rank `rank` of `nranks`).
qb_status init_comm(qb_ctx ctx, int rank, int nranks, const void* nccl_unique_id) {
  ctx->rank = rank;
  ctx->nranks = nranks;
  if (!nccl().ok) return fail(ctx, QB_ERR_NCCL, "libnccl.so.2 not found (set QB_NCCL_LIB)");
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  QB_CUDA(cudaSetDevice(ctx->device));
  ncclResult_t r = nccl().commInitRank(&ctx->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    ctx->comm = nullptr;
    return fail(ctx, QB_ERR_NCCL, "ncclCommInitRank: %s", nccl().errorString(r));
  }
  return QB_OK;
}

// The small-problem path (small_loop.cuh): the whole loop in one cluster launch when A fits in the
// cluster's shared memory.  Returns QB_ERR_UNSUPPORTED (not an error: the caller takes the general
// path) when the problem is not eligible.
struct SmallPlan {
  SmallLoopArgs a{};
  int cl = 0;
  size_t smem = 0;
};

bool small_plan(qb_ctx ctx, int64_t m, int64_t n, int64_t b, int q, int64_t kmax, SmallPlan* plan) {
  if (m * n > 262144 || b > SCQR_MAX_W) return false;
  int max_smem = 0;
  if (cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device) != cudaSuccess)
    return false;
  const size_t budget = (size_t)max_smem - 3072;  // static shared memory of the kernel and its helpers
  static const int force_cl = debug_env("QB_SMALL_CL");
  for (int cl : {8, 16}) {
    if (force_cl && cl != force_cl) continue;
    const int64_t mr = (m + cl - 1) / cl, nr = (n + cl - 1) / cl;
    int64_t off = 0;
    auto take = [&](int64_t cnt) {
      const int64_t o = off;
      off += (cnt + 1) / 2 * 2;
      return (int)o;
    };
    SmallLoopArgs& a = plan->a;
    a.oA = take(m * nr);
    a.oOm = take(nr * b);
    a.oYp = take(m * b);
    a.oYs = take(mr * b);
    a.oZs = take(q > 0 ? nr * b : 0);
    a.oX2 = take(std::max(mr, nr) * b);
    a.oGp = take(b * SCQR_GLD);
    a.oG = take(b * SCQR_GLD);
    a.oT = take(b * SCQR_GLD);
    a.oWp = take(kmax * b);
    a.oWr = take((kmax * b + cl - 1) / cl);
    a.oQc = take(mr * kmax);
    a.oBc = take(b * nr);
    const size_t bytes = (size_t)off * 8;
    int nclusters = 0;
    if (bytes <= budget) {
      // the cluster must be schedulable (16 CTAs of this size need a GPC with 16 free SMs)
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(cl, 1, 1);
      lc.blockDim = dim3(SL_THREADS, 1, 1);
      lc.dynamicSmemBytes = bytes;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      lc.attrs = attr;
      lc.numAttrs = 1;
      if (cudaFuncSetAttribute(small_loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess ||
          (cl > 8 && cudaFuncSetAttribute(small_loop_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) ||
          cudaOccupancyMaxActiveClusters(&nclusters, small_loop_kernel, &lc) != cudaSuccess || nclusters < 1) {
        const cudaError_t e = cudaGetLastError();  // clear a non-sticky launch-configuration error
        if (debug_env("QB_SMALL_TRACE"))
          fprintf(stderr, "[small_loop] cluster of %d not schedulable (%zu B): %s, %d clusters\n", cl, bytes,
                  cudaGetErrorString(e), nclusters);
        continue;
      }
    }
    if (bytes <= budget) {
      a.mr = (int)mr;
      a.nr = (int)nr;
      plan->cl = cl;
      plan->smem = bytes;
      return true;
    }
  }
  return false;
}

qb_status publish_outputs(qb_ctx ctx, int64_t m, int64_t n, int64_t k, const void** Q_out, int64_t* ldq_out,
                          const void** B_out, int64_t* ldb_out) {
  const void* Qp = ctx->Qbar.p;
  const void* Bp = ctx->Bbar.p;
  if (ctx->dtype == QB_F32) {
    QB_TRY(ensure(ctx, ctx->Bf, sizeof(float) * (size_t)(ctx->ldb * std::max<int64_t>(k, 1))));
    QB_TRY(launch_convert(ctx, ctx->Bbar.d(), ctx->ldb, n, k, static_cast<float*>(ctx->Bf.p), ctx->ldb));
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    Qp = ctx->Qbar32.p;  // RN_32 of each finished Q_i, kept block by block
    Bp = ctx->Bf.p;
  }
  if (Q_out) *Q_out = Qp;
  if (ldq_out) *ldq_out = ctx->ldq;
  if (B_out) *B_out = Bp;
  if (ldb_out) *ldb_out = ctx->ldb;
  return QB_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

const char* qb_status_string(qb_status s) {
  switch (s) {
    case QB_OK: return "QB_OK";
    case QB_NOT_CONVERGED: return "QB_NOT_CONVERGED";
    case QB_ERR_INVALID_ARG: return "QB_ERR_INVALID_ARG";
    case QB_ERR_OOM: return "QB_ERR_OOM";
    case QB_ERR_CUDA: return "QB_ERR_CUDA";
    case QB_ERR_NCCL: return "QB_ERR_NCCL";
    case QB_ERR_ORTH_BREAKDOWN: return "QB_ERR_ORTH_BREAKDOWN";
    case QB_ERR_UNSUPPORTED: return "QB_ERR_UNSUPPORTED";
  }
  return "QB_UNKNOWN";
}

const char* qb_last_error(qb_ctx ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t qb_kernel_launches(qb_ctx ctx) { return ctx ? ctx->launches : 0; }

#ifdef QB_CHOL_TIMING
int qb_debug_chol_ts(unsigned long long* out) { return (int)cudaMemcpyFromSymbol(out, qb_chol_ts, 64 * 8); }
#endif

qb_status qb_create(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream) {
  if (!out) return QB_ERR_INVALID_ARG;
  *out = nullptr;
  qb_ctx ctx = new qb_ctx_s();
  qb_status s = init_ctx(ctx, device, dtype, cuda_stream);
  *out = ctx;  // returned even on failure so qb_last_error can explain; caller destroys
  return s;
}

qb_status qb_nccl_unique_id(void* out128) {
  if (!out128) return QB_ERR_INVALID_ARG;
  if (!nccl().ok) return QB_ERR_NCCL;
  ncclUniqueId id;
  if (nccl().getUniqueId(&id) != ncclSuccess) return QB_ERR_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return QB_OK;
}

qb_status qb_loopback_create(qb_loopback* out, int nranks) {
  if (!out) return QB_ERR_INVALID_ARG;
  *out = nullptr;
  if (nranks < 1 || nranks > QB_LOOPBACK_MAX_RANKS) return QB_ERR_INVALID_ARG;
  qb_loopback g = new qb_loopback_s();
  g->nranks = nranks;
  g->timeout_s = comm_timeout_s();
  *out = g;
  return QB_OK;
}

void qb_loopback_destroy(qb_loopback g) {
  if (!g) return;
  if (g->scratch) {
    cudaSetDevice(g->device);
    cudaFree(g->scratch);
  }
  delete g;
}

qb_status qb_create_sharded(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream, const qb_dist* d) {
  if (!out) return QB_ERR_INVALID_ARG;
  qb_status s = qb_create(out, device, dtype, cuda_stream);
  if (s != QB_OK) return s;
  qb_ctx ctx = *out;
  if (!d || d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks || d->offset < 0 || d->global < 1 ||
      (d->shard != QB_SHARD_COLS && d->shard != QB_SHARD_ROWS) ||
      (d->comm != QB_COMM_NCCL && d->comm != QB_COMM_LOOPBACK) ||
      (d->comm == QB_COMM_NCCL && !d->nccl_id) || (d->comm == QB_COMM_LOOPBACK && !d->loopback))
    return fail(ctx, QB_ERR_INVALID_ARG, "bad distributed arguments");
  ctx->dist = true;
  if (d->shard == QB_SHARD_ROWS) {
    ctx->shard_rows = true;
    ctx->row_offset = d->offset;
    ctx->m_global = d->global;
  } else {
    ctx->col_offset = d->offset;
    ctx->n_global = d->global;
  }
  if (d->comm == QB_COMM_NCCL) return init_comm(ctx, d->rank, d->nranks, d->nccl_id);
  qb_loopback g = d->loopback;
  if (g->nranks != d->nranks) return fail(ctx, QB_ERR_INVALID_ARG, "loopback group has %d ranks, not %d", g->nranks, d->nranks);
  {
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->device < 0) g->device = device;
    if (g->device != device)
      return fail(ctx, QB_ERR_INVALID_ARG, "loopback ranks must share one device (%d, not %d)", g->device, device);
  }
  ctx->rank = d->rank;
  ctx->nranks = d->nranks;
  ctx->loop = g;
  return QB_OK;
}

qb_status qb_create_dist(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream, int rank, int nranks,
                         const void* nccl_unique_id, int64_t col_offset, int64_t n_global) {
  qb_dist d{};
  d.rank = rank;
  d.nranks = nranks;
  d.shard = QB_SHARD_COLS;
  d.comm = QB_COMM_NCCL;
  d.nccl_id = nccl_unique_id;
  d.offset = col_offset;
  d.global = n_global;
  return qb_create_sharded(out, device, dtype, cuda_stream, &d);
}

qb_status qb_create_dist_rows(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream, int rank, int nranks,
                              const void* nccl_unique_id, int64_t row_offset, int64_t m_global) {
  qb_dist d{};
  d.rank = rank;
  d.nranks = nranks;
  d.shard = QB_SHARD_ROWS;
  d.comm = QB_COMM_NCCL;
  d.nccl_id = nccl_unique_id;
  d.offset = row_offset;
  d.global = m_global;
  return qb_create_sharded(out, device, dtype, cuda_stream, &d);
}

void qb_destroy(qb_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  DevBuf* bufs[] = {&ctx->Awork, &ctx->Qbar, &ctx->Bbar, &ctx->Om, &ctx->Y,     &ctx->T1,    &ctx->Z,   &ctx->Zt,
                    &ctx->G,     &ctx->L,    &ctx->Rinv, &ctx->W,  &ctx->P,     &ctx->parts, &ctx->scal, &ctx->status,
                    &ctx->Qf,    &ctx->Bf,   &ctx->Astage, &ctx->Q32,  &ctx->B32, &ctx->Qbar32, &ctx->W32,
                    &ctx->QB,    &ctx->R,    &ctx->Usv,    &ctx->Vsv,  &ctx->Ssv, &ctx->Wsv,    &ctx->Ut,
                    &ctx->Vt,    &ctx->Usv32, &ctx->Vsv32, &ctx->Ssv32, &ctx->Swork, &ctx->Rq,    &ctx->Qh,
                    &ctx->Qt,    &ctx->qvn1, &ctx->qvn2,   &ctx->qperm, &ctx->qtau,  &ctx->qv,    &ctx->qparts,
                    &ctx->Rq32,  &ctx->Qh32, &ctx->qw,    &ctx->qw2,   &ctx->Xsave, &ctx->X32,   &ctx->T32,
                    &ctx->Bsp,   &ctx->X32b, &ctx->Jx,    &ctx->Jj,   &ctx->Jpart, &ctx->Jw,
                    &ctx->Jint,  &ctx->Jsig, &ctx->Jpairs, &ctx->Srec, &ctx->Strace, &ctx->Jq2, &ctx->Jm2};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev_gap) cudaEventDestroy(ctx->ev_gap);
  for (auto& e : ctx->evp)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->tev)
    if (e) cudaEventDestroy(e);
  if (ctx->comm) nccl().commDestroy(ctx->comm);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->cap_stream2) cudaStreamDestroy(ctx->cap_stream2);
  if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
  for (auto& e : ctx->jev)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

qb_status qb_stats(qb_ctx ctx, qb_block_stats* out, int64_t cap, int64_t* nblocks) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  const int64_t n = static_cast<int64_t>(ctx->stats.size());
  if (nblocks) *nblocks = n;
  if (out && cap > 0) std::memcpy(out, ctx->stats.data(), sizeof(qb_block_stats) * (size_t)std::min(cap, n));
  return QB_OK;
}

qb_status qb_omega(qb_ctx ctx, uint64_t seed, int64_t row0, int64_t row1, int64_t col0, int64_t w, void* out,
                   int64_t ldo) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  if (row0 < 0 || row1 < row0 || col0 < 0 || w < 0 || (w > 0 && ldo < w) || (!out && row1 > row0 && w > 0))
    return fail(ctx, QB_ERR_INVALID_ARG, "qb_omega: bad arguments");
  if (row1 == row0 || w == 0) return QB_OK;
  QB_CUDA(cudaSetDevice(ctx->device));
  return launch_omega(ctx, seed, row0, row1, col0, w, out, ldo, ctx->dtype == QB_F64 ? 0 : 1);
}

qb_status qb_orth(qb_ctx ctx, void* X, int64_t m, int64_t w, int64_t ldx) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  if (!X || m < 1 || w < 1 || w > kMaxB || w > m || ldx < m || m > INT32_MAX)
    return fail(ctx, QB_ERR_INVALID_ARG, "qb_orth: bad arguments (m=%lld w=%lld ldx=%lld)", (long long)m,
                (long long)w, (long long)ldx);
  QB_CUDA(cudaSetDevice(ctx->device));
  const int64_t ldgb = round_up(kMaxB, 16);
  QB_TRY(ensure(ctx, ctx->G, sizeof(double) * ldgb * ldgb));
  QB_TRY(ensure(ctx, ctx->L, sizeof(double) * (ldgb * ldgb + 8 * 32 * 32)));
  QB_TRY(ensure(ctx, ctx->Rinv, sizeof(double) * ldgb * ldgb));
  QB_TRY(ensure(ctx, ctx->T1, sizeof(double) * (size_t)(round_up(m, 16) * kMaxB)));
  QB_TRY(reset_flags(ctx));
  const bool aligned = (ldx % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  if (ctx->dtype == QB_F32) {  // FP32 panel: CholeskyQR2 in FP64 on the exactly widened copy
    const int64_t ldy = round_up(m, 16);
    QB_TRY(ensure(ctx, ctx->Y, sizeof(double) * (size_t)(ldy * w)));
    QB_TRY(launch_convert(ctx, static_cast<const float*>(X), ldx, m, w, ctx->Y.d(), ldy));
    QB_TRY(cholqr2(ctx, ctx->Y.d(), ldy, ctx->Y.d(), ldy, m, (int)w));
    QB_TRY(launch_convert(ctx, static_cast<const double*>(ctx->Y.d()), ldy, m, w, static_cast<float*>(X), ldx));
  } else if (aligned) {
    QB_TRY(cholqr2(ctx, static_cast<double*>(X), ldx, static_cast<double*>(X), ldx, m, (int)w));
  } else {  // TMA needs 16-byte aligned columns: stage through an aligned copy
    const int64_t ldy = round_up(m, 16);
    QB_TRY(ensure(ctx, ctx->Y, sizeof(double) * (size_t)(ldy * w)));
    QB_CUDA(cudaMemcpy2DAsync(ctx->Y.p, ldy * 8, X, ldx * 8, m * 8, w, cudaMemcpyDeviceToDevice, ctx->stream));
    QB_TRY(cholqr2(ctx, ctx->Y.d(), ldy, ctx->Y.d(), ldy, m, (int)w));
    QB_CUDA(cudaMemcpy2DAsync(X, ldx * 8, ctx->Y.p, ldy * 8, m * 8, w, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  QB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->status.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->h_status[4]) return fail(ctx, QB_ERR_ORTH_BREAKDOWN, "CholeskyQR failed even with the shift (w=%lld)", (long long)w);
  return QB_OK;
}

qb_status qb_gemm(qb_ctx ctx, int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, int split, double* sumsq) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  if ((layout != GEMM_NN && layout != GEMM_TN) || epi < 0 || epi > 2 || M < 0 || N < 0 || K < 1 || M > INT32_MAX ||
      N > INT32_MAX || K > INT32_MAX || !A || !B || !C)
    return fail(ctx, QB_ERR_INVALID_ARG, "qb_gemm: bad arguments");
  QB_CUDA(cudaSetDevice(ctx->device));
  QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)std::max<int64_t>(
                                     ((M + GEMM_BM - 1) / GEMM_BM) * ((N + kBN - 1) / kBN), 16 * ctx->num_sms)));
  int64_t np = 0;
  if (ctx->dtype == QB_F32)
    QB_TRY(gemm_tf(ctx, layout, epi, (int)M, (int)N, (int)K, static_cast<const float*>(A), lda,
                   static_cast<const float*>(B), ldb, C, ldc, sumsq != nullptr, &np, split != 0));
  else
    QB_TRY(gemm(ctx, layout, epi, (int)M, (int)N, (int)K, static_cast<const double*>(A), lda,
                static_cast<const double*>(B), ldb, static_cast<double*>(C), ldc, sumsq != nullptr, &np, split != 0));
  if (sumsq) {
    QB_TRY(reduce_to_scal(ctx, np, 2));
    QB_CUDA(cudaMemcpyAsync(ctx->h_scal + 2, ctx->scal.d() + 2, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (sumsq) *sumsq = ctx->h_scal[2];
  return QB_OK;
}

qb_status qb_chol_rinv(qb_ctx ctx, const void* G, int64_t ldg, int64_t w, int64_t m_rows, void* Rinv, int64_t ldr,
                       int* shifted) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  if (!G || !Rinv || w < 1 || w > kMaxB || ldg < w || ldr < w || m_rows < 1)
    return fail(ctx, QB_ERR_INVALID_ARG, "qb_chol_rinv: bad arguments");
  QB_CUDA(cudaSetDevice(ctx->device));
  const int64_t ld = round_up(kMaxB, 16);
  QB_TRY(ensure(ctx, ctx->G, sizeof(double) * ld * ld));
  QB_TRY(ensure(ctx, ctx->L, sizeof(double) * (ld * ld + 8 * 32 * 32)));
  QB_TRY(ensure(ctx, ctx->Rinv, sizeof(double) * ld * ld));
  QB_CUDA(cudaMemcpy2DAsync(ctx->G.p, ld * 8, G, ldg * 8, w * 8, w, cudaMemcpyDeviceToDevice, ctx->stream));
  QB_TRY(reset_flags(ctx));
  QB_TRY(chol_inv(ctx, (int)w, m_rows, false, nullptr));
  QB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->status.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  const int st = ctx->h_status[0];
  if (shifted) *shifted = st;
  if (st == 2) return fail(ctx, QB_ERR_ORTH_BREAKDOWN, "qb_chol_rinv: shifted Cholesky failed");
  // ctx->Rinv holds L^-1 column-major == R^-1 row-major (ld); copy rows out
  QB_CUDA(cudaMemcpy2DAsync(Rinv, ldr * 8, ctx->Rinv.p, ld * 8, w * 8, w, cudaMemcpyDeviceToDevice, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QB_OK;
}

// Round-robin tournament (circle method) over nblk (even) players: step s pairs (s, nblk-1) and
// (s+i, s-i) mod (nblk-1); every pair of blocks meets once in nblk - 1 steps.
static std::vector<int2> round_robin(int nblk) {
  std::vector<int2> out;
  const int mod = nblk - 1;
  for (int st = 0; st < mod; ++st) {
    for (int i = 0; i < nblk / 2; ++i) {
      int a = i == 0 ? st : (st + i) % mod;
      int b = i == 0 ? nblk - 1 : (st - i + mod) % mod;
      out.push_back(make_int2(std::min(a, b), std::max(a, b)));
    }
  }
  return out;
}

qb_status rqb_svd(qb_ctx ctx, double eps, int64_t kkeep, int64_t* kk_out, const void** U_out, int64_t* ldu_out,
                  const void** S_out, const void** V_out, int64_t* ldv_out) {
  // QB -> partial SVD: B̄ = Û D V^*, U = Q̄ Û.
  //  1. B̄^T (n x k) = Q_B R: block Gram-Schmidt (two projections) + CholeskyQR2 per 256 columns;
  //  2. R = Q_B^T B̄^T (k x k);
  //  3. SVD of R^T by block one-sided Jacobi (svd.cuh): R^T J = Û D, J orthogonal, so
  //     B̄ = R^T Q_B^T = Û D (Q_B J)^T, i.e. V = Q_B J;
  //  4. U = Q̄ Û, V = Q_B J on the library GEMM, for the leading k' triplets: k' = kkeep, or the
  //     smallest k' with ||A - U_k' D_k' V_k'^*||_F^2 = r_k^2 + sum_{j > k'} D_j^2 <= eps^2 (the tail
  //     rule: "choose a rank ... based on the decaying singular values").
  if (!ctx) return QB_ERR_INVALID_ARG;
  if (kk_out) *kk_out = 0;
  if (ctx->last_k < 0) return fail(ctx, QB_ERR_INVALID_ARG, "rqb_svd: no factorization to convert");
  if (!(eps >= 0.0)) return fail(ctx, QB_ERR_INVALID_ARG, "rqb_svd: eps must be >= 0");
  // row shards: B̄ is replicated and U = Q̄ Û is this rank's rows of U; column shards hold B̄ split
  if (ctx->nranks > 1 && !ctx->shard_rows)
    return fail(ctx, QB_ERR_UNSUPPORTED, "rqb_svd: column-sharded B̄ (distributed) not supported");
  const int64_t m = ctx->last_m, n = ctx->last_n, k = ctx->last_k;
  QB_CUDA(cudaSetDevice(ctx->device));
  if (k == 0) {
    if (U_out) *U_out = nullptr;
    if (S_out) *S_out = nullptr;
    if (V_out) *V_out = nullptr;
    if (ldu_out) *ldu_out = round_up(m, 16);
    if (ldv_out) *ldv_out = round_up(n, 16);
    return QB_OK;
  }
  if (k > INT32_MAX / 4) return fail(ctx, QB_ERR_INVALID_ARG, "rqb_svd: k too large");
  NvtxRange nv("rqb_svd");
  const int64_t ldn = round_up(n, 16), ldm = round_up(m, 16), ldk = round_up(k, 16), bp = round_up(kMaxB, 16);
  const int64_t kp = round_up(k, 2 * JNB);  // Jacobi columns, padded to whole block pairs
  const int nblk = (int)(kp / JNB), npairs = nblk / 2, nsteps = nblk - 1;
  const int nch = (int)((k + JRC - 1) / JRC);
  QB_TRY(ensure(ctx, ctx->QB, sizeof(double) * (size_t)(ldn * k)));
  QB_TRY(ensure(ctx, ctx->R, sizeof(double) * (size_t)(ldk * k)));
  QB_TRY(ensure(ctx, ctx->Ut, sizeof(double) * (size_t)(ldk * k)));
  QB_TRY(ensure(ctx, ctx->Vt, sizeof(double) * (size_t)(ldk * k)));
  QB_TRY(ensure(ctx, ctx->Ssv, sizeof(double) * (size_t)ldk));
  QB_TRY(ensure(ctx, ctx->Wsv, sizeof(double) * (size_t)(ldk * bp)));
  QB_TRY(ensure(ctx, ctx->T1, sizeof(double) * (size_t)(round_up(std::max(m, n), 16) * kMaxB)));
  QB_TRY(ensure(ctx, ctx->G, sizeof(double) * bp * bp));
  QB_TRY(ensure(ctx, ctx->L, sizeof(double) * (bp * bp + 8 * 32 * 32)));
  QB_TRY(ensure(ctx, ctx->Rinv, sizeof(double) * bp * bp));
  QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)(16 * ctx->num_sms)));
  QB_TRY(ensure(ctx, ctx->Jx, sizeof(double) * (size_t)(kp * kp)));
  QB_TRY(ensure(ctx, ctx->Jj, sizeof(double) * (size_t)(kp * kp)));
  QB_TRY(ensure(ctx, ctx->Jpart, sizeof(double) * (size_t)npairs * nch * JPW * JPW));
  QB_TRY(ensure(ctx, ctx->Jw, sizeof(double) * (size_t)2 * npairs * JPW * JPW));
  QB_TRY(ensure(ctx, ctx->Jint, sizeof(int) * (size_t)(2 * npairs + 2 * kp) + 64));
  QB_TRY(ensure(ctx, ctx->Jsig, sizeof(double) * (size_t)kp + 64));
  double* QBm = ctx->QB.d();
  const double* Bbar = ctx->Bbar.d();  // row-major k x n (ld ldb) == B̄^T column-major n x k
  QB_TRY(reset_flags(ctx));

  // 1. Q_B = orth(B̄^T), 256 columns at a time
  QB_CUDA(cudaMemcpy2DAsync(QBm, ldn * 8, Bbar, ctx->ldb * 8, n * 8, k, cudaMemcpyDeviceToDevice, ctx->stream));
  // 2. R (k x k, column-major, upper triangular) with B̄^T = Q_B R, from the projections of step 1
  //    (QB_SVD_RGEMM=1: the explicit product Q_B^T B̄^T instead)
  static const int rgemm = debug_env("QB_SVD_RGEMM");
  if (rgemm) {
    QB_TRY(orth_blocked(ctx, QBm, ldn, n, k));
    QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_COL, (int)k, (int)k, (int)n, QBm, ldn, Bbar, ctx->ldb, ctx->R.d(), ldk, false,
                nullptr));
  } else {
    QB_TRY(orth_blocked(ctx, QBm, ldn, n, k, ctx->R.d(), ldk));
  }
  double t_front = 0.0;
  if (debug_env("QB_JAC_TRACE")) {  // diagnostics: host time of the front end (orth of B̄^T, R)
    const double t0 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    t_front = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    fprintf(stderr, "[rqb_svd] front end done (waited %.2f ms)\n", t_front - t0);
  }
  // 3'. QR preconditioning (Drmac's preconditioned Jacobi): R^T = Q2 R2, Jacobi on R2^T instead
  // (default for k >= 2048, where it saves a sweep: T 224 -> 215 ms; at C4, k = 1152, the sweep count
  // is unchanged and the extra QR costs 1.6 ms; QB_SVD_PRECOND=0/1 forces it)
  static const char* precond_env = getenv("QB_SVD_PRECOND");
  const bool precond = precond_env ? atoi(precond_env) != 0 : k >= 2048;
  if (precond) {
    QB_TRY(ensure(ctx, ctx->Jq2, sizeof(double) * (size_t)(ldk * k)));
    dim3 grid((unsigned)((k + 31) / 32), (unsigned)((k + 31) / 32));
    transpose_kernel<double><<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->R.d(), ldk, k, k, ctx->Jq2.d(), ldk);
    QB_TRY(check_launch(ctx, "transpose"));  // Jq2 = R^T (column-major)
    // Jq2 = Q2 and R (column-major) <- R2, assembled from the projections (R^T = Q2 R2)
    QB_TRY(orth_blocked(ctx, ctx->Jq2.d(), ldk, k, k, ctx->R.d(), ldk));
  }
  // 3. one-sided Jacobi on X = R^T (kp x kp, zero-padded), J = I
  double* X = ctx->Jx.d();
  double* Jm = ctx->Jj.d();
  QB_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * (size_t)(kp * kp), ctx->stream));
  {
    dim3 grid((unsigned)((k + 31) / 32), (unsigned)((k + 31) / 32));
    transpose_kernel<double><<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->R.d(), ldk, k, k, X, kp);  // X(c, r) = R(r, c)
    QB_TRY(check_launch(ctx, "transpose"));
    qrcp_identity_kernel<<<(int)std::min<int64_t>((kp * kp + 255) / 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(
        Jm, kp, (int)kp);
    QB_TRY(check_launch(ctx, "identity"));
  }
  if (ctx->jac_pairs_nblk != nblk) {  // the tournament schedule, uploaded once per block count
    std::vector<int2> sched = round_robin(nblk);
    for (int p = 0; p < nblk / 2; ++p) sched.push_back(make_int2(2 * p, 2 * p + 1));  // QB_JAC_CROSS's first step
    QB_TRY(ensure(ctx, ctx->Jpairs, sizeof(int2) * sched.size()));
    QB_CUDA(cudaMemcpy(ctx->Jpairs.p, sched.data(), sizeof(int2) * sched.size(), cudaMemcpyHostToDevice));
    ctx->jac_pairs_nblk = nblk;
  }
  QB_SMEM_ATTR(jac_gram_kernel, JGRAM_SMEM);
  QB_SMEM_ATTR(jac_solve_kernel, JSOLVE_SMEM);
  QB_SMEM_ATTR(jac_update_kernel, JUPD_SMEM);
  int* jflag = static_cast<int*>(ctx->Jint.p);
  int* jrank = jflag + 2 * npairs;
  auto* offmax = reinterpret_cast<unsigned long long*>(ctx->Jsig.d() + kp);
  const int2* pairs = static_cast<const int2*>(ctx->Jpairs.p);
  // columns are orthogonal to this relative level at convergence (above the Gram's rounding ~ sqrt(k) u)
  // (the Gram entries carry rounding up to ~k u relative to the column norms, so the threshold scales
  // with k; at T, k u = 3e-13)
  const double tol = std::max(1e-14, (double)k * 0x1p-53);
  static const int inner = debug_env("QB_JAC_INNER") > 0 ? debug_env("QB_JAC_INNER") : 1;
  const int max_sweeps = 40;
  int sweeps = 0;
  double off = 1.0;
  // One sweep = nsteps x (Gram, solve, X update) on the main stream; the J update of step s runs on a
  // second stream beside the next step's Gram and solve (J is read by nothing else).  Δ and the flags
  // alternate between two slots: solve s+2 reuses slot s % 2 only after J update s (event).  The sweep
  // is captured once into a CUDA graph (private capture streams; nothing runs during capture) and
  // replayed per sweep on the context stream.
  if (!ctx->aux_stream) QB_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
  if (!ctx->jev[0])
    for (auto& e : ctx->jev) QB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const int nchj = nch;
  // Each sweep: a first step on the pairs (2p, 2p+1) with full inner sweeps (every within-block pair
  // of columns), then the tournament with cross-block rotations only (16 rotation steps per pair
  // instead of 31; T 249 -> 234 ms, C4 48 -> 42 ms, same sweep count).  QB_JAC_CROSS=0: full inner
  // sweeps on every tournament pair.
  static const int cross = getenv("QB_JAC_CROSS") ? atoi(getenv("QB_JAC_CROSS")) : 1;
  const int nst = nsteps + (cross ? 1 : 0);
  auto enqueue_sweep = [&](cudaStream_t st, cudaStream_t st2) -> qb_status {
    QB_CUDA(cudaMemsetAsync(offmax, 0, sizeof(unsigned long long), st));
    for (int s = 0; s < nst; ++s) {
      const int slot = s & 1;
      const int2* pr = (cross && s == 0) ? pairs + (size_t)nsteps * npairs : pairs + (size_t)(s - (cross ? 1 : 0)) * npairs;
      const int cross_only = (cross && s > 0) ? 1 : 0;
      double* Dsl = ctx->Jw.d() + (size_t)slot * npairs * JPW * JPW;
      int* fl = jflag + slot * npairs;
      jac_gram_kernel<<<dim3(npairs, nch), JTHREADS, JGRAM_SMEM, st>>>(X, kp, (int)k, pr, nch, ctx->Jpart.d());
      QB_TRY(check_launch(ctx, "jac_gram"));
      if (s >= 2) QB_CUDA(cudaStreamWaitEvent(st, ctx->jev[2 + slot], 0));  // J update s-2 read this slot
      jac_solve_kernel<<<npairs, JST, JSOLVE_SMEM, st>>>(ctx->Jpart.d(), nch, Dsl, fl, offmax, tol, inner, cross_only);
      QB_TRY(check_launch(ctx, "jac_solve"));
      QB_CUDA(cudaEventRecord(ctx->jev[slot], st));
      jac_update_kernel<<<dim3(npairs, nch), JTHREADS, JUPD_SMEM, st>>>(X, kp, (int)k, pr, Dsl, fl);
      QB_TRY(check_launch(ctx, "jac_update_x"));
      QB_CUDA(cudaStreamWaitEvent(st2, ctx->jev[slot], 0));
      jac_update_kernel<<<dim3(npairs, nchj), JTHREADS, JUPD_SMEM, st2>>>(Jm, kp, (int)k, pr, Dsl, fl);
      QB_TRY(check_launch(ctx, "jac_update_j"));
      QB_CUDA(cudaEventRecord(ctx->jev[2 + slot], st2));
    }
    QB_CUDA(cudaStreamWaitEvent(st, ctx->jev[2 + ((nst - 1) & 1)], 0));  // join the J branch
    return QB_OK;
  };
  static const int no_graph = debug_env("QB_JAC_NO_GRAPH");
  cudaGraphExec_t gexec = nullptr;
  const int per_sweep = 4 * nst;
  if (!no_graph && !debug_env("QB_DEBUG_SYNC")) {
    if (!ctx->cap_stream) QB_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    if (!ctx->cap_stream2) QB_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream2, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    QB_CUDA(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    // fork the second capture stream into the capture
    cudaError_t fe = cudaEventRecord(ctx->jev[4], ctx->cap_stream);
    if (fe == cudaSuccess) fe = cudaStreamWaitEvent(ctx->cap_stream2, ctx->jev[4], 0);
    const qb_status cs = fe == cudaSuccess ? enqueue_sweep(ctx->cap_stream, ctx->cap_stream2) : QB_ERR_CUDA;
    const cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
    if (cs != QB_OK || fe != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return cs != QB_OK ? cs : fail(ctx, QB_ERR_CUDA, "rqb_svd: graph capture fork: %s", cudaGetErrorString(fe));
    }
    QB_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiate(&gexec, graph, 0);
    cudaGraphDestroy(graph);
    QB_CUDA(ie);
    ctx->launches -= per_sweep;  // counted again per replay below
  } else {
    QB_CUDA(cudaEventRecord(ctx->jev[4], ctx->stream));  // the side stream starts after the setup
    QB_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->jev[4], 0));
  }
  for (; sweeps < max_sweeps && off > tol; ++sweeps) {
    if (gexec) {
      const cudaError_t le = cudaGraphLaunch(gexec, ctx->stream);
      if (le != cudaSuccess) {
        cudaGraphExecDestroy(gexec);
        QB_CUDA(le);
      }
      ctx->launches += per_sweep;
    } else {
      QB_TRY(enqueue_sweep(ctx->stream, ctx->aux_stream));
    }
    unsigned long long bits = 0;
    QB_CUDA(cudaMemcpyAsync(&bits, offmax, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&off, &bits, sizeof(off));
    static const int trace = debug_env("QB_JAC_TRACE");
    if (trace) {
      const double now = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
      fprintf(stderr, "[rqb_svd] sweep %d: max scaled off-diagonal %.3e, %.2f ms since the front end\n", sweeps, off,
              now - t_front);
    }
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  ctx->jac_sweeps = sweeps;
  if (off > tol) return fail(ctx, QB_ERR_UNSUPPORTED, "rqb_svd: Jacobi did not converge in %d sweeps (off %.3g)",
                             max_sweeps, off);
  // sorted triplets: S descending, Û (row-major, ld ldk) = X D^-1, J (row-major, ld ldk)
  double* sig = ctx->Jsig.d();
  jac_norms_kernel<<<(int)((k * 32 + 255) / 256), 256, 0, ctx->stream>>>(X, kp, (int)k, (int)k, sig);
  QB_TRY(check_launch(ctx, "jac_norms"));
  jac_rank_kernel<<<(int)((k + 255) / 256), 256, 0, ctx->stream>>>(sig, (int)k, jrank);
  QB_TRY(check_launch(ctx, "jac_rank"));
  jac_finish_kernel<<<(int)std::min<int64_t>((k * k + 255) / 256, 16 * ctx->num_sms), 256, 0, ctx->stream>>>(
      X, kp, Jm, kp, (int)k, sig, jrank, ctx->Ssv.d(), ctx->Ut.d(), ldk, ctx->Vt.d(), ldk);
  QB_TRY(check_launch(ctx, "jac_finish"));
  // 4. the kept rank: kkeep and / or the tail rule with eps
  int64_t kk = k;
  if (eps > 0.0) {
    auto* kdev = reinterpret_cast<long long*>(ctx->Jsig.d() + kp + 1);
    jac_tail_rank_kernel<<<1, 32, 0, ctx->stream>>>(ctx->Ssv.d(), (int)k, ctx->last_r2, eps * eps, kdev);
    QB_TRY(check_launch(ctx, "jac_tail_rank"));
    long long kh = k;
    QB_CUDA(cudaMemcpyAsync(&kh, kdev, sizeof(kh), cudaMemcpyDeviceToHost, ctx->stream));
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    kk = kh;
  }
  if (kkeep > 0 && kkeep < kk) kk = kkeep;
  if (kk_out) *kk_out = kk;
  const int64_t kkc = std::max<int64_t>(kk, 1);
  QB_TRY(ensure(ctx, ctx->Usv, sizeof(double) * (size_t)(ldm * kkc)));
  QB_TRY(ensure(ctx, ctx->Vsv, sizeof(double) * (size_t)(ldn * kkc)));
  if (kk > 0 && precond) {
    // R^T = Q2 R2 and R2^T J' = Û' D: B̄ = (Q2 J') D (Q_B Û')^T, so U = Q̄ (Q2 J'), V = Q_B Û'
    QB_TRY(ensure(ctx, ctx->Jm2, sizeof(double) * (size_t)(ldk * k)));
    QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_ROW, (int)k, (int)k, (int)k, ctx->Jq2.d(), ldk, ctx->Vt.d(), ldk, ctx->Jm2.d(),
                ldk, false, nullptr));  // row-major Q2 J'
    QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)m, (int)kk, (int)k, ctx->Qbar.d(), ctx->ldq, ctx->Jm2.d(), ldk,
                ctx->Usv.d(), ldm, false, nullptr));
    QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)n, (int)kk, (int)k, QBm, ldn, ctx->Ut.d(), ldk, ctx->Vsv.d(), ldn,
                false, nullptr));
  } else if (kk > 0) {
    QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)m, (int)kk, (int)k, ctx->Qbar.d(), ctx->ldq, ctx->Ut.d(), ldk,
                ctx->Usv.d(), ldm, false, nullptr));
    QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)n, (int)kk, (int)k, QBm, ldn, ctx->Vt.d(), ldk, ctx->Vsv.d(), ldn,
                false, nullptr));
  }
  QB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->status.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->h_status[4]) return fail(ctx, QB_ERR_ORTH_BREAKDOWN, "rqb_svd: CholeskyQR of B^T failed");
  const void* Up = ctx->Usv.p;
  const void* Sp = ctx->Ssv.p;
  const void* Vp = ctx->Vsv.p;
  if (ctx->dtype == QB_F32) {
    QB_TRY(ensure(ctx, ctx->Usv32, sizeof(float) * (size_t)(ldm * kkc)));
    QB_TRY(ensure(ctx, ctx->Vsv32, sizeof(float) * (size_t)(ldn * kkc)));
    QB_TRY(ensure(ctx, ctx->Ssv32, sizeof(float) * (size_t)ldk));
    QB_TRY(launch_convert(ctx, ctx->Usv.d(), ldm, m, kk, static_cast<float*>(ctx->Usv32.p), ldm));
    QB_TRY(launch_convert(ctx, ctx->Vsv.d(), ldn, n, kk, static_cast<float*>(ctx->Vsv32.p), ldn));
    QB_TRY(launch_convert(ctx, ctx->Ssv.d(), 1, 1, kk, static_cast<float*>(ctx->Ssv32.p), 1));
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    Up = ctx->Usv32.p;
    Sp = ctx->Ssv32.p;
    Vp = ctx->Vsv32.p;
  }
  if (U_out) *U_out = kk > 0 ? Up : nullptr;
  if (ldu_out) *ldu_out = ldm;
  if (S_out) *S_out = kk > 0 ? Sp : nullptr;
  if (V_out) *V_out = kk > 0 ? Vp : nullptr;
  if (ldv_out) *ldv_out = ldn;
  return QB_OK;
}

int qb_svd_sweeps(qb_ctx ctx) { return ctx ? ctx->jac_sweeps : 0; }

qb_status qb_pivoted_qr(qb_ctx ctx, int64_t* perm_out, const void** Qh_out, int64_t* ldqh_out, const void** R_out,
                        int64_t* ldr_out) {
  // QB -> partial pivoted QR: B P = Q~ R (Householder QR with column pivoting
  // of the l x n factor B), Q^ = Q Q~, so that A P ~ Q^ R.  FP64 internally.
  if (!ctx) return QB_ERR_INVALID_ARG;
  if (ctx->last_k < 0) return fail(ctx, QB_ERR_INVALID_ARG, "qb_pivoted_qr: no factorization to convert");
  if (ctx->nranks > 1 && !ctx->shard_rows)
    return fail(ctx, QB_ERR_UNSUPPORTED, "qb_pivoted_qr: column-sharded B̄ (distributed) not supported");
  const int64_t m = ctx->last_m, n = ctx->last_n, l = ctx->last_k;
  QB_CUDA(cudaSetDevice(ctx->device));
  if (l == 0) {
    if (perm_out)
      for (int64_t j = 0; j < n; ++j) perm_out[j] = j;
    if (Qh_out) *Qh_out = nullptr;
    if (R_out) *R_out = nullptr;
    if (ldqh_out) *ldqh_out = round_up(m, 16);
    if (ldr_out) *ldr_out = ctx->ldb;
    return QB_OK;
  }
  const int64_t ldr = ctx->ldb, ldm = round_up(m, 16), ldqt = round_up(l, 16);
  const int nchunks = (int)((l + QRCP_ROWS - 1) / QRCP_ROWS);
  const int64_t ldp = round_up(n, 16);
  QB_TRY(ensure(ctx, ctx->Rq, sizeof(double) * (size_t)(ldr * l)));
  QB_TRY(ensure(ctx, ctx->Qt, sizeof(double) * (size_t)(ldqt * l)));
  QB_TRY(ensure(ctx, ctx->Qh, sizeof(double) * (size_t)(ldm * l)));
  QB_TRY(ensure(ctx, ctx->qvn1, sizeof(double) * (size_t)n));
  QB_TRY(ensure(ctx, ctx->qvn2, sizeof(double) * (size_t)n));
  QB_TRY(ensure(ctx, ctx->qperm, sizeof(int) * (size_t)n));
  QB_TRY(ensure(ctx, ctx->qtau, sizeof(double) * (size_t)l));
  QB_TRY(ensure(ctx, ctx->qv, sizeof(double) * (size_t)l));
  QB_TRY(ensure(ctx, ctx->qparts, sizeof(double) * (size_t)(nchunks * ldp)));
  double* R = ctx->Rq.d();
  QB_CUDA(cudaMemcpyAsync(R, ctx->Bbar.p, sizeof(double) * (size_t)(ldr * l), cudaMemcpyDeviceToDevice, ctx->stream));
  double* vn1 = ctx->qvn1.d();
  double* vn2 = ctx->qvn2.d();
  int* perm = static_cast<int*>(ctx->qperm.p);
  double* tau = ctx->qtau.d();
  double* vb = ctx->qv.d();
  double* parts = ctx->qparts.d();
  const double tol3z = std::sqrt(0x1p-52);
  qrcp_init_kernel<<<(int)((n + QRCP_THREADS - 1) / QRCP_THREADS), QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l,
                                                                                                 (int)n, vn1, vn2, perm);
  QB_TRY(check_launch(ctx, "qrcp_init"));
  static const int unfused = debug_env("QB_QRCP_UNFUSED");
  static const int lookahead = debug_env("QB_QRCP_LOOKAHEAD");
  if (!unfused && !lookahead) {  // blocked (dlaqps): panels of QRCP_NB pivots, trailing GEMM per panel
    const int64_t nblk = (n + QRCP_THREADS - 1) / QRCP_THREADS + 8;
    const int64_t ldf = ldp, ldv = ldqt;
    QB_TRY(ensure(ctx, ctx->qw, sizeof(double) * (size_t)(QRCP_NB * ldf + QRCP_NB * ldv + 2 * nblk + 8)));
    double* F = ctx->qw.d();
    double* Vt = F + QRCP_NB * ldf;
    double* pmax = Vt + QRCP_NB * ldv;
    int* pidx = reinterpret_cast<int*>(pmax + nblk);
    int* piv = pidx + 2 * nblk;  // step i's pivot column
    const int kmin = (int)std::min<int64_t>(l, n);
    static const int ptrace = debug_env("QB_QRCP_TRACE");  // diagnostics: per-panel device time
    cudaEvent_t pev[2] = {nullptr, nullptr};
    if (ptrace) {
      cudaEventCreate(&pev[0]);
      cudaEventCreate(&pev[1]);
    }
    // one persistent cooperative launch per panel (qrcp_persist.cuh) when v fits in shared memory
    // and every CTA owns at most QP_THREADS columns
    static const int no_persist = debug_env("QB_QRCP_NO_PERSIST");
    const int G = ctx->num_sms;
    const int qp_cwp = (int)(((n + G - 1) / G + 1) | 1);  // odd stride: conflict-free F columns
    const size_t qp_smem = sizeof(double) * (size_t)(l + 2 * QP_THREADS + QRCP_NB * qp_cwp);
    bool persist = !no_persist && (n + G - 1) / G <= QP_THREADS && G <= QP_WARPS * QP_CPW && qp_smem <= QP_MAX_SMEM;
    if (persist) {
      QB_SMEM_ATTR(qrcp_panel_kernel, (int)QP_MAX_SMEM);  // the largest launch
      int per_sm = 0, coop = 0;
      QB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_panel_kernel, QP_THREADS, qp_smem));
      QB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
      persist = per_sm >= 1 && coop != 0;  // one co-resident CTA per SM, or the multi-kernel schedule
    }
    QrcpPanelArgs pa{};
    if (persist) {
      QB_TRY(ensure(ctx, ctx->qw2, sizeof(double) * (size_t)(QP_REP * (l + 8 + 35 * G) + 512)));
      double* pw = ctx->qw2.d();
      pa.B = R;
      pa.ldb = ldr;
      pa.l = (int)l;
      pa.n = (int)n;
      pa.vn1 = vn1;
      pa.vn2 = vn2;
      pa.perm = perm;
      pa.tau = tau;
      pa.F = F;
      pa.ldf = ldf;
      pa.xbuf = pw;
      pa.alpha = pa.xbuf + QP_REP * l;
      pa.ssp = pa.alpha + QP_REP;
      pa.auxp = pa.ssp + QP_REP * G;
      pa.pmax = pa.auxp + QP_REP * 32 * G;
      pa.pidx = reinterpret_cast<int*>(pa.pmax + QP_REP * G);
      pa.bar = reinterpret_cast<unsigned*>(pa.pmax + 2 * QP_REP * G);
      pa.tol3z = tol3z;
      pa.cwp = qp_cwp;
    }
    for (int i0 = 0; i0 < kmin; i0 += QRCP_NB) {
      const int nb = std::min(QRCP_NB, kmin - i0);
      if (ptrace) cudaEventRecord(pev[0], ctx->stream);
      if (persist) {
        pa.i0 = i0;
        pa.nb = nb;
        pa.first = i0 == 0;
        QB_CUDA(cudaMemsetAsync(pa.bar, 0, sizeof(unsigned), ctx->stream));
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3((unsigned)G);
        lc.blockDim = dim3(QP_THREADS);
        lc.dynamicSmemBytes = qp_smem;
        lc.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        static const int ptr = debug_env("QB_QRCP_PTRACE");  // diagnostics: phase marks of panels 0 and mid
        const bool trace_this = ptr && (i0 == 0 || i0 == (kmin / 2 / QRCP_NB) * QRCP_NB || i0 + QRCP_NB >= kmin);
        pa.trace = trace_this ? reinterpret_cast<unsigned long long*>(pa.pmax + 2 * QP_REP * G + 8) : nullptr;
        QB_CUDA(cudaLaunchKernelEx(&lc, qrcp_panel_kernel, pa));
        QB_TRY(check_launch(ctx, "qrcp_panel"));
        if (trace_this) {
          unsigned long long tr[64 + 320];
          QB_CUDA(cudaMemcpy(tr, pa.trace, sizeof(tr), cudaMemcpyDeviceToHost));
          for (int h = 0; h < 2; ++h) {  // arrival spread at the barriers of step 1 (h = 0: second, 1: first)
            const unsigned long long* ar = tr + 64 + 160 * h;
            unsigned long long mn = ~0ull, mx = 0;
            int cmx = 0;
            for (int cc = 0; cc < G; ++cc) {
              mn = std::min(mn, ar[cc]);
              if (ar[cc] > mx) {
                mx = ar[cc];
                cmx = cc;
              }
            }
            std::fprintf(stderr, "qrcp panel %d step 1 barrier %d arrival spread %.2f us (last CTA %d)\n", i0, 2 - h,
                         (double)(mx - mn) * 1e-3, cmx);
          }
          for (int s2 = 0; s2 < 4; ++s2) {
            std::fprintf(stderr, "qrcp panel %d step %d:", i0, s2);
            for (int k2 = 1; k2 <= 10; ++k2)
              std::fprintf(stderr, " %.2f", (double)(tr[s2 * 16 + k2] - tr[s2 * 16 + k2 - 1]) * 1e-3);
            std::fprintf(stderr, " | after barrier: loads %.2f sum %.2f us\n", (double)(tr[s2 * 16 + 11] - tr[s2 * 16 + 3]) * 1e-3,
                         (double)(tr[s2 * 16 + 12] - tr[s2 * 16 + 11]) * 1e-3);
          }
        }
      }
      for (int i = i0; i < i0 + nb && !persist; ++i) {
        const int npart = i > 0 ? (int)((n - i + QRCP_THREADS - 1) / QRCP_THREADS) : 0;
        qrcp_bk_pivot_kernel<<<1, BKP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, i0, vn1, tau, F, ldf, vb,
                                                                 piv, pmax, pidx, npart);
        QB_TRY(check_launch(ctx, "qrcp_bk_pivot"));
        if (i + 1 >= n) continue;  // then p = i: no swap is pending
        const int rch = (int)((l - i + QRCP_WROWS - 1) / QRCP_WROWS);
        dim3 wgrid((unsigned)((n - i0 + QRCP_THREADS - 1) / QRCP_THREADS), (unsigned)rch);
        qrcp_bk_w_kernel<<<wgrid, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, i0, vb, parts, ldp);
        QB_TRY(check_launch(ctx, "qrcp_bk_w"));
        const int rblocks = (int)((n - i - 1 + QRCP_THREADS - 1) / QRCP_THREADS);
        qrcp_bk_row_kernel<<<rblocks, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, i0, tau, parts, ldp,
                                                                      rch, F, ldf, vn1, vn2, perm, piv, tol3z, pmax, pidx);
        QB_TRY(check_launch(ctx, "qrcp_bk_row"));
      }
      // trailing block below and right of the panel: A -= V F^T (one GEMM; K = nb)
      const int r0 = i0 + nb;
      if (r0 < l && r0 < n) {
        const int rows = (int)(l - r0);
        qrcp_bk_vt_kernel<<<(int)std::min<int64_t>(((int64_t)rows * nb + 255) / 256, 4 * ctx->num_sms), 256, 0,
                            ctx->stream>>>(R, ldr, r0, rows, i0, nb, Vt, ldv);
        QB_TRY(check_launch(ctx, "qrcp_bk_vt"));
        QB_TRY(gemm(ctx, GEMM_NN, EPI_SUB_COL, (int)(n - r0), rows, nb, F + r0, ldf, Vt, ldv,
                    R + (int64_t)r0 * ldr + r0, ldr, false, nullptr));
      }
      if (ptrace) {
        float ms = 0.f;
        cudaEventRecord(pev[1], ctx->stream);
        cudaEventSynchronize(pev[1]);
        cudaEventElapsedTime(&ms, pev[0], pev[1]);
        std::fprintf(stderr, "qrcp panel %d: %.3f ms\n", i0, ms);
      }
    }
    if (ptrace) {
      cudaEventDestroy(pev[0]);
      cudaEventDestroy(pev[1]);
    }
  } else if (unfused) {  // reference schedule: reflector, w, rank-1 update, renorm per step
    for (int i = 0; i < (int)l; ++i) {
      qrcp_pivot_kernel<<<1, 1024, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, vn1, vn2, perm, tau, vb);
      QB_TRY(check_launch(ctx, "qrcp_pivot"));
      if (i + 1 >= n) continue;
      const int ncol = (int)(n - i - 1);
      const int rch = (int)((l - i + QRCP_ROWS - 1) / QRCP_ROWS);
      dim3 grid((unsigned)((ncol + QRCP_THREADS - 1) / QRCP_THREADS), (unsigned)rch);
      qrcp_w_kernel<<<grid, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, vb, parts, ldp);
      QB_TRY(check_launch(ctx, "qrcp_w"));
      qrcp_update_kernel<<<grid, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, vb, tau, parts, ldp, rch,
                                                                 vn1, vn2, tol3z);
      QB_TRY(check_launch(ctx, "qrcp_update"));
      qrcp_renorm_kernel<<<grid.x, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, vn1, vn2);
      QB_TRY(check_launch(ctx, "qrcp_renorm"));
    }
  } else {  // one-step lookahead: the trailing block is read and written once per step
    const int64_t nblk = (n + QRCP_THREADS - 1) / QRCP_THREADS + 8;
    QB_TRY(ensure(ctx, ctx->qw, sizeof(double) * (size_t)(n + 2 * l + 64 + 2 * nblk)));
    double* wprev = ctx->qw.d();
    double* vbs[2] = {vb, wprev + n};  // v_i alternates between two buffers (v_{i-1} still needed)
    // per-block (max partial norm, first index) of step i's updated norms: step i+1's pivot search
    double* pmax = wprev + n + 2 * l + 64;
    int* pidx = reinterpret_cast<int*>(pmax + nblk);
    QB_CUDA(cudaMemsetAsync(wprev, 0, sizeof(double) * (size_t)n, ctx->stream));
    for (int i = 0; i < (int)l; ++i) {
      double* vcur = vbs[i & 1];
      const double* vprev = vbs[(i + 1) & 1];
      const int npart = i > 0 && n - i > 0 ? (int)((n - i + QRCP_THREADS - 1) / QRCP_THREADS) : 0;
      qrcp_la_pivot_kernel<<<1, 1024, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, vn1, vn2, perm, tau, vprev, wprev,
                                                         vcur, pmax, pidx, npart);
      QB_TRY(check_launch(ctx, "qrcp_la_pivot"));
      if (i + 1 >= n) continue;
      const int ncol = (int)(n - i - 1);
      const int rch = (int)((l - i + QRCP_ROWS - 1) / QRCP_ROWS);
      dim3 grid((unsigned)((ncol + QRCP_THREADS - 1) / QRCP_THREADS), (unsigned)rch);
      qrcp_la_fw_kernel<<<grid, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, tau, vprev, wprev, vcur,
                                                                parts, ldp);
      QB_TRY(check_launch(ctx, "qrcp_la_fw"));
      qrcp_la_row_kernel<<<grid.x, QRCP_THREADS, 0, ctx->stream>>>(R, ldr, (int)l, (int)n, i, tau, vcur, parts, ldp,
                                                                   rch, wprev, vn1, vn2, tol3z, pmax, pidx);
      QB_TRY(check_launch(ctx, "qrcp_la_row"));
    }
    // the last deferred update reaches rows below l only: nothing left to apply
  }
  // Q~ = H_0 ... H_{l-1} (backward accumulation on the identity), then Q^ = Q̄ Q~
  double* Qt = ctx->Qt.d();
  qrcp_identity_kernel<<<(int)std::min<int64_t>((l * l + 255) / 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(
      Qt, ldqt, (int)l);
  QB_TRY(check_launch(ctx, "qrcp_identity"));
  static const int qtrace = debug_env("QB_QRCP_TRACE");
  cudaEvent_t qev[3] = {nullptr, nullptr, nullptr};
  if (qtrace) {
    for (auto& e : qev) cudaEventCreate(&e);
    cudaEventRecord(qev[0], ctx->stream);
  }
  static const int q_unblocked = debug_env("QB_QRCP_Q_UNBLOCKED");
  if (q_unblocked) {  // reference schedule: one reflector at a time
    for (int i = (int)l - 1; i >= 0; --i) {
      const int rch = (int)((l - i + QRCP_ROWS - 1) / QRCP_ROWS);
      dim3 grid((unsigned)((l - i + QRCP_THREADS - 1) / QRCP_THREADS), (unsigned)rch);
      qrcp_q_w_kernel<<<grid, QRCP_THREADS, 0, ctx->stream>>>(Qt, ldqt, (int)l, i, R, ldr, parts, ldp);
      QB_TRY(check_launch(ctx, "qrcp_q_w"));
      qrcp_q_update_kernel<<<grid, QRCP_THREADS, 0, ctx->stream>>>(Qt, ldqt, (int)l, i, R, ldr, tau, parts, ldp,
                                                                   rch);
      QB_TRY(check_launch(ctx, "qrcp_q_update"));
    }
  } else {  // panels of QRCP_NB reflectors, last to first: Q~(i0:, i0:) -= V (T (V^T Q~(i0:, i0:)))
    const int64_t ldw = ldqt;
    QB_TRY(ensure(ctx, ctx->qw, sizeof(double) * (size_t)(QRCP_NB * l + 3 * QRCP_NB * ldw + 2 * QRCP_NB * QRCP_NB)));
    double* Vx = ctx->qw.d();
    double* Vtp = Vx + QRCP_NB * l;
    double* Wt = Vtp + QRCP_NB * ldw;
    double* Zt = Wt + QRCP_NB * ldw;
    double* Tm = Zt + QRCP_NB * ldw;
    double* Gq = Tm + QRCP_NB * QRCP_NB;
    for (int i0 = (int)((l - 1) / QRCP_NB) * QRCP_NB; i0 >= 0; i0 -= QRCP_NB) {
      const int nb = (int)std::min<int64_t>(QRCP_NB, l - i0), rows = (int)(l - i0);
      qrcp_vpanel_kernel<<<(int)std::min<int64_t>(((int64_t)rows * QRCP_NB + 255) / 256, 4 * ctx->num_sms), 256, 0,
                           ctx->stream>>>(R, ldr, i0, rows, nb, Vx, Vtp, ldw);
      QB_TRY(check_launch(ctx, "qrcp_vpanel"));
      // G = V^T V (the DMMA GEMM on the column-major view of the row-major Vx), then T
      QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, QRCP_NB, QRCP_NB, rows, Vx, QRCP_NB, Vx, QRCP_NB, Gq, QRCP_NB, false,
                  nullptr));
      qrcp_tmat_kernel<<<1, 32, 0, ctx->stream>>>(Gq, nb, tau + i0, Tm);
      QB_TRY(check_launch(ctx, "qrcp_tmat"));
      // W^T = Q~(i0:, i0:)^T V (column-major views of the row-major Q~ and V)
      QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, rows, QRCP_NB, rows, Qt + (int64_t)i0 * ldqt + i0, ldqt, Vx, QRCP_NB,
                  Wt, ldw, false, nullptr));
      qrcp_tz_kernel<<<(rows + 127) / 128, 128, 0, ctx->stream>>>(Tm, Wt, ldw, rows, Zt);
      QB_TRY(check_launch(ctx, "qrcp_tz"));
      // Q~(i0:, i0:)^T -= Z^T V^T
      QB_TRY(gemm(ctx, GEMM_NN, EPI_SUB_COL, rows, rows, QRCP_NB, Zt, ldw, Vtp, ldw, Qt + (int64_t)i0 * ldqt + i0,
                  ldqt, false, nullptr));
    }
  }
  qrcp_zero_lower_kernel<<<(int)std::min<int64_t>((l * l + 255) / 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(
      R, ldr, (int)l);
  QB_TRY(check_launch(ctx, "qrcp_zero_lower"));
  QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)(16 * ctx->num_sms)));
  if (qtrace) cudaEventRecord(qev[1], ctx->stream);
  QB_TRY(gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)m, (int)l, (int)l, ctx->Qbar.d(), ctx->ldq, Qt, ldqt, ctx->Qh.d(), ldm,
              false, nullptr));
  if (qtrace) {
    float t1 = 0.f, t2 = 0.f;
    cudaEventRecord(qev[2], ctx->stream);
    cudaEventSynchronize(qev[2]);
    cudaEventElapsedTime(&t1, qev[0], qev[1]);
    cudaEventElapsedTime(&t2, qev[1], qev[2]);
    std::fprintf(stderr, "qrcp Q~ accumulation %.3f ms, Q^ = Q Q~ GEMM %.3f ms\n", t1, t2);
    for (auto& e : qev) cudaEventDestroy(e);
  }
  std::vector<int> hperm((size_t)n);
  QB_CUDA(cudaMemcpyAsync(hperm.data(), perm, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (perm_out)
    for (int64_t j = 0; j < n; ++j) perm_out[j] = hperm[(size_t)j];
  const void* Qp = ctx->Qh.p;
  const void* Rp = R;
  if (ctx->dtype == QB_F32) {
    QB_TRY(ensure(ctx, ctx->Qh32, sizeof(float) * (size_t)(ldm * l)));
    QB_TRY(ensure(ctx, ctx->Rq32, sizeof(float) * (size_t)(ldr * l)));
    QB_TRY(launch_convert(ctx, ctx->Qh.d(), ldm, m, l, static_cast<float*>(ctx->Qh32.p), ldm));
    QB_TRY(launch_convert(ctx, static_cast<const double*>(R), ldr, n, l, static_cast<float*>(ctx->Rq32.p), ldr));
    QB_CUDA(cudaStreamSynchronize(ctx->stream));
    Qp = ctx->Qh32.p;
    Rp = ctx->Rq32.p;
  }
  if (Qh_out) *Qh_out = Qp;
  if (ldqh_out) *ldqh_out = ldm;
  if (R_out) *R_out = Rp;
  if (ldr_out) *ldr_out = ldr;
  return QB_OK;
}

qb_status qb_fixed_rank(qb_ctx ctx, void* Ain, int64_t m, int64_t n, int64_t lda, int64_t l, int P, uint64_t seed,
                        unsigned flags, const void** Q_out, int64_t* ldq_out, const void** B_out, int64_t* ldb_out,
                        double* resid_out) {
  // randQB (Fig. 1) / randQB_p (Fig. 3), unblocked; the skip
  // variant of PAPER.md:919-927 under QB_SKIP_POWER_ORTH.
  if (!ctx) return QB_ERR_INVALID_ARG;
  ctx->stats.clear();
  ctx->last_k = -1;
  if (ctx->nranks > 1) return fail(ctx, QB_ERR_UNSUPPORTED, "qb_fixed_rank: distributed contexts not supported");
  const bool is_f32 = ctx->dtype == QB_F32;
  if (!Ain || m < 1 || n < 1 || lda < m || m > INT32_MAX || n > INT32_MAX || l < 1 || l > std::min(m, n) || P < 0)
    return fail(ctx, QB_ERR_INVALID_ARG, "qb_fixed_rank: bad arguments (m=%lld n=%lld lda=%lld l=%lld P=%d)",
                (long long)m, (long long)n, (long long)lda, (long long)l, P);
  QB_CUDA(cudaSetDevice(ctx->device));
  const size_t es = is_f32 ? 4 : 8;
  // A is only read, except for the optional residual: then it is updated in place (OVERWRITE)
  // or in a context-owned copy
  void* Av = Ain;
  int64_t ldA = lda;
  const bool aligned = (lda % (is_f32 ? 4 : 2) == 0) && ((reinterpret_cast<uintptr_t>(Ain) & 15) == 0);
  if (!aligned || (resid_out && !(flags & QB_OVERWRITE_A))) {
    ldA = round_up(m, 16);
    QB_TRY(ensure(ctx, ctx->Awork, es * (size_t)(ldA * n)));
    // an SM copy (the copy engine's device-to-device copy is slower); its sums of squares are unused
    const int grid = (int)std::min<int64_t>(n, 8 * ctx->num_sms);
    QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
    if (is_f32)
      copy_sumsq_kernel<float><<<grid, RED_THREADS, 0, ctx->stream>>>(static_cast<const float*>(Ain), lda, m, n,
                                                                       static_cast<float*>(ctx->Awork.p), ldA,
                                                                       ctx->parts.d());
    else
      copy_sumsq_kernel<double><<<grid, RED_THREADS, 0, ctx->stream>>>(static_cast<const double*>(Ain), lda, m, n,
                                                                        ctx->Awork.d(), ldA, ctx->parts.d());
    QB_TRY(check_launch(ctx, "copy"));
    Av = ctx->Awork.p;
  }
  double* A = static_cast<double*>(Av);
  float* A32 = static_cast<float*>(Av);
  const int64_t ldn = round_up(n, 16), lp = round_up(l, 16), ldm = round_up(m, 16);
  QB_TRY(grow_factors(ctx, m, n, l, l));
  double* Qd = ctx->Qbar.d();
  const int64_t ldq = ctx->ldq;
  double* Bd = ctx->Bbar.d();
  QB_TRY(ensure(ctx, ctx->Om, es * (size_t)(n * lp)));
  QB_TRY(ensure(ctx, ctx->T1, sizeof(double) * (size_t)(round_up(std::max(m, n), 16) * kMaxB)));
  const int64_t bp = round_up(kMaxB, 16);
  QB_TRY(ensure(ctx, ctx->G, sizeof(double) * bp * bp));
  QB_TRY(ensure(ctx, ctx->L, sizeof(double) * (bp * bp + 8 * 32 * 32)));
  QB_TRY(ensure(ctx, ctx->Rinv, sizeof(double) * bp * bp));
  QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)std::max<int64_t>(
                                     ((m + GEMM_BM - 1) / GEMM_BM) * ((n + kBN - 1) / kBN), 16 * ctx->num_sms)));
  if (P > 0) {
    QB_TRY(ensure(ctx, ctx->Z, sizeof(double) * (size_t)(ldn * l)));
    QB_TRY(ensure(ctx, ctx->Zt, es * (size_t)(n * lp)));
  }
  if (is_f32) QB_TRY(ensure(ctx, ctx->Q32, sizeof(float) * (size_t)(ldm * l)));
  float* X32 = static_cast<float*>(ctx->Q32.p);
  QB_TRY(reset_flags(ctx));

  // Y (into Q̄'s storage) = A X for the row-major n x l operand X (ld lp)
  auto sketch = [&](const void* X) -> qb_status {
    if (is_f32)
      return gemm_tf(ctx, GEMM_NN, TF_STORE_COL, (int)m, (int)l, (int)n, A32, ldA, static_cast<const float*>(X), lp,
                     Qd, ldq, false, nullptr);
    return gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)m, (int)l, (int)n, A, ldA, static_cast<const double*>(X), lp, Qd,
                ldq, false, nullptr);
  };
  // Z = A^T Q̄ (n x l, ld ldn)
  auto adjoint = [&]() -> qb_status {
    if (!is_f32)
      return gemm(ctx, GEMM_TN, EPI_STORE_COL, (int)n, (int)l, (int)m, A, ldA, Qd, ldq, ctx->Z.d(), ldn, false,
                  nullptr);
    QB_TRY(launch_convert(ctx, static_cast<const double*>(Qd), ldq, m, l, X32, ldm));
    return gemm_tf(ctx, GEMM_TN, TF_STORE_COL, (int)n, (int)l, (int)m, A32, ldA, X32, ldm, ctx->Z.d(), ldn, false,
                   nullptr);
  };
  auto transpose_z = [&]() -> qb_status {
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((l + 31) / 32));
    if (is_f32)
      transpose_kernel<float><<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->Z.d(), ldn, n, l,
                                                                      static_cast<float*>(ctx->Zt.p), lp);
    else
      transpose_kernel<double><<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->Z.d(), ldn, n, l, ctx->Zt.d(), lp);
    return check_launch(ctx, "transpose");
  };

  // Omega = randn(n, l): global columns 0..l-1, row-major (ld lp); FP32 contexts draw RN_32(Omega)
  QB_TRY(launch_omega(ctx, seed, 0, n, 0, l, ctx->Om.p, lp, is_f32 ? 1 : 0));
  QB_TRY(sketch(ctx->Om.p));  // Y = A Omega
  const bool skip_orth = skip_orth_flag(flags);
  if (skip_orth) {
    for (int j = 0; j < P; ++j) {  // Y = A (A^* Y)
      QB_TRY(adjoint());
      QB_TRY(transpose_z());
      QB_TRY(sketch(ctx->Zt.p));
    }
    QB_TRY(orth_blocked(ctx, Qd, ldq, m, l));
  } else {
    QB_TRY(orth_blocked(ctx, Qd, ldq, m, l));  // Q = orth(A Omega)
    for (int j = 0; j < P; ++j) {
      QB_TRY(adjoint());                                   // Z = A^* Q
      QB_TRY(orth_blocked(ctx, ctx->Z.d(), ldn, n, l));    // Z = orth(Z)
      QB_TRY(transpose_z());
      QB_TRY(sketch(ctx->Zt.p));                           // Q = A Z
      QB_TRY(orth_blocked(ctx, Qd, ldq, m, l));            // Q = orth(Q)
    }
  }
  // B = Q^* A (row-major l x n); FP32 contexts use RN_32(Q), the factor the caller receives
  int64_t nparts = 0;
  if (is_f32) {
    QB_TRY(launch_convert(ctx, static_cast<const double*>(Qd), ldq, m, l, static_cast<float*>(ctx->Qbar32.p), ldq));
    QB_TRY(gemm_tf(ctx, GEMM_TN, TF_STORE_ROW, (int)l, (int)n, (int)m, static_cast<const float*>(ctx->Qbar32.p), ldq,
                   A32, ldA, Bd, ctx->ldb, false, nullptr));
  } else {
    QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_ROW, (int)l, (int)n, (int)m, Qd, ldq, A, ldA, Bd, ctx->ldb, false, nullptr));
  }
  double r = 0.0;
  if (resid_out) {  // ||A - QB||_F, directly: A -= Q B with the fused sum of squares
    if (is_f32) {
      QB_TRY(ensure(ctx, ctx->B32, sizeof(float) * (size_t)(ctx->ldb * l)));
      QB_TRY(launch_convert(ctx, static_cast<const double*>(Bd), ctx->ldb, n, l, static_cast<float*>(ctx->B32.p),
                            ctx->ldb));
      QB_TRY(gemm_tf(ctx, GEMM_NN, TF_SUB_COL, (int)m, (int)n, (int)l, static_cast<const float*>(ctx->Qbar32.p), ldq,
                     static_cast<const float*>(ctx->B32.p), ctx->ldb, A32, ldA, true, &nparts));
    } else {
      QB_TRY(gemm(ctx, GEMM_NN, EPI_SUB_COL, (int)m, (int)n, (int)l, Qd, ldq, Bd, ctx->ldb, A, ldA, true, &nparts));
    }
    QB_TRY(reduce_to_scal(ctx, nparts, 0));
    QB_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->scal.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  QB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->status.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->h_status[4]) return fail(ctx, QB_ERR_ORTH_BREAKDOWN, "qb_fixed_rank: CholeskyQR failed even with the shift");
  ctx->last_r2 = 0.0;  // unknown unless requested: rqb_svd's tail rule then counts the kept triplets only
  if (resid_out) {
    r = std::sqrt(ctx->h_scal[0]);
    *resid_out = r;
    ctx->last_r2 = ctx->h_scal[0];
  }
  ctx->last_m = m;
  ctx->last_n = n;
  ctx->last_k = l;
  return publish_outputs(ctx, m, n, l, Q_out, ldq_out, B_out, ldb_out);
}

static qb_status factor_impl(qb_ctx ctx, void* Ain, int64_t m, int64_t n, int64_t lda, double eps, int64_t b, int q,
                             uint64_t seed, int64_t kmax, unsigned flags, int64_t* k_out, const void** Q_out,
                             int64_t* ldq_out, const void** B_out, int64_t* ldb_out, double* resid_out) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  ctx->stats.clear();
  if (!k_out) return fail(ctx, QB_ERR_INVALID_ARG, "k must not be NULL");
  *k_out = 0;
  const bool is_f32 = ctx->dtype == QB_F32;
  struct TfGram {  // set for the duration of this factorization
    qb_ctx c;
    explicit TfGram(qb_ctx c_, bool on) : c(c_) { c->tf_gram = on; }
    ~TfGram() { c->tf_gram = false; }
  } tf_gram_scope(ctx, is_f32);
  // empty A (m = 0 or n = 0, single-rank contexts): ||A||_F = 0 <= eps, so k = 0 (reading R3,
  // Algorithm 1 line (2)); A may be NULL.  Arguments b, q, eps are still validated.
  if (m >= 0 && n >= 0 && (m == 0 || n == 0) && ctx->nranks <= 1 && lda >= std::max<int64_t>(m, 1)) {
    if (b < 1 || b > kMaxB) return fail(ctx, QB_ERR_INVALID_ARG, "block size b=%lld outside [1, %lld]", (long long)b, (long long)kMaxB);
    if (q < 0) return fail(ctx, QB_ERR_INVALID_ARG, "q=%d < 0", q);
    if (!(eps >= 0.0)) return fail(ctx, QB_ERR_INVALID_ARG, "eps must be >= 0 (got %g)", eps);
    ctx->outQ = nullptr;
    ctx->outB = nullptr;
    ctx->last_m = m;
    ctx->last_n = n;
    ctx->last_k = 0;
    ctx->last_r2 = 0.0;
    if (resid_out) *resid_out = 0.0;
    if (Q_out) *Q_out = nullptr;
    if (ldq_out) *ldq_out = round_up(std::max<int64_t>(m, 1), 16);
    if (B_out) *B_out = nullptr;
    if (ldb_out) *ldb_out = round_up(std::max<int64_t>(n, 1), 16);
    return QB_OK;
  }
  if (!Ain || m < 1 || n < 1 || lda < m || m > INT32_MAX || n > INT32_MAX)
    return fail(ctx, QB_ERR_INVALID_ARG, "bad matrix arguments (m=%lld n=%lld lda=%lld)", (long long)m, (long long)n,
                (long long)lda);
  if (b < 1 || b > kMaxB) return fail(ctx, QB_ERR_INVALID_ARG, "block size b=%lld outside [1, %lld]", (long long)b, (long long)kMaxB);
  if (q < 0) return fail(ctx, QB_ERR_INVALID_ARG, "q=%d < 0", q);
  if (!(eps >= 0.0)) return fail(ctx, QB_ERR_INVALID_ARG, "eps must be >= 0 (got %g)", eps);
  // sharding: column shards allreduce Y (and the row-distributed Z's Gram);
  // row shards (NEXT-2) allreduce Grams, W, Z and B_i instead, and keep Y, Q_i local
  const bool rowsh = ctx->dist && ctx->shard_rows;
  const bool colsh = ctx->dist && !ctx->shard_rows;
  const int64_t n_glob = (colsh && ctx->nranks > 1) ? ctx->n_global : n;
  const int64_t m_glob = (rowsh && ctx->nranks > 1) ? ctx->m_global : m;
  const int64_t kmax_eff = (kmax <= 0) ? std::min(m_glob, n_glob) : std::min(kmax, std::min(m_glob, n_glob));
  QB_CUDA(cudaSetDevice(ctx->device));

  // ---- small problems: the whole loop in one cluster launch (small_loop.cuh)
  static const int no_small_loop = debug_env("QB_NO_SMALL_LOOP");
  SmallPlan plan;
  if (!no_small_loop && !is_f32 && !ctx->dist && !(flags & (QB_SKIP_POWER_ORTH | QB_FORCE_GENERAL)) &&
      small_plan(ctx, m, n, b, q, kmax_eff, &plan)) {
    NvtxRange nv("small_loop (whole factorization)");
    const bool overwrite = (flags & QB_OVERWRITE_A) != 0;
    QB_TRY(grow_factors(ctx, m, n, kmax_eff, kmax_eff));
    const int64_t nrec = (kmax_eff + b - 1) / b;
    QB_TRY(ensure(ctx, ctx->Srec, sizeof(double) * (size_t)(6 * nrec + 8)));
    SmallLoopArgs& a = plan.a;
    a.A = static_cast<const double*>(Ain);
    a.lda = lda;
    a.Aout = overwrite ? static_cast<double*>(Ain) : nullptr;
    a.ldo = lda;
    a.m = (int)m;
    a.n = (int)n;
    a.b = (int)b;
    a.q = q;
    a.kmax = (int)kmax_eff;
    a.reproj = (flags & QB_NO_REPROJ) ? 0 : 1;
    a.full_first = debug_env("QB_FULL_FIRST_ORTH") ? 1 : 0;
    a.eps2 = eps * eps;
    a.ns_tol2 = 1e-16;
    a.tol = 1e-13;
    a.seed = seed;
    a.Qbar = ctx->Qbar.d();
    a.ldq = ctx->ldq;
    a.Bbar = ctx->Bbar.d();
    a.ldb = ctx->ldb;
    a.out = ctx->Srec.d();
    a.rec = ctx->Srec.d() + 8;
    a.K = ctx->omega_consts;
    QB_CUDA(cudaFuncSetAttribute(small_loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem));
    static const int trace = debug_env("QB_SMALL_TRACE");
    a.trace = nullptr;
    if (trace) {
      QB_TRY(ensure(ctx, ctx->Strace, 32 * sizeof(unsigned long long)));
      QB_CUDA(cudaMemsetAsync(ctx->Strace.p, 0, 32 * sizeof(unsigned long long), ctx->stream));
      a.trace = static_cast<unsigned long long*>(ctx->Strace.p);
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(plan.cl, 1, 1);
    lc.blockDim = dim3(SL_THREADS, 1, 1);
    lc.dynamicSmemBytes = plan.smem;
    lc.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = plan.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    QB_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    QB_CUDA(cudaLaunchKernelEx(&lc, small_loop_kernel, a));
    QB_TRY(check_launch(ctx, "small_loop"));
    QB_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    std::vector<double> hrec((size_t)(6 * nrec + 8));
    QB_CUDA(cudaMemcpyAsync(hrec.data(), ctx->Srec.p, sizeof(double) * hrec.size(), cudaMemcpyDeviceToHost,
                            ctx->stream));
    QB_TRY(stream_wait(ctx));
    const double r2_0 = hrec[0], r2 = hrec[1];
    const int64_t k = (int64_t)hrec[2], nblk = (int64_t)hrec[5];
    if (trace) {
      unsigned long long tr[32];
      QB_CUDA(cudaMemcpy(tr, ctx->Strace.p, sizeof(tr), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[small_loop] cluster %d CTAs, %zu B smem; block 2 phases (us):", plan.cl, plan.smem);
      for (int i = 1; i < 12; ++i) fprintf(stderr, " %d:%.1f", i, tr[i] && tr[i - 1] ? (tr[i] - tr[i - 1]) * 1e-3 : -1.0);
      fprintf(stderr, "; first orth pass (us):");
      for (int i = 13; i < 19; ++i) fprintf(stderr, " %d:%.1f", i, tr[i] && tr[i - 1] ? (tr[i] - tr[i - 1]) * 1e-3 : -1.0);
      fprintf(stderr, "\n");
    }
    ctx->outQ = nullptr;
    ctx->outB = nullptr;
    if (!std::isfinite(r2_0)) return fail(ctx, QB_ERR_INVALID_ARG, "A contains NaN or Inf");
    if (hrec[4] != 0.0) return fail(ctx, QB_ERR_ORTH_BREAKDOWN, "CholeskyQR failed even with the shift");
    float total = 0.f;
    cudaEventElapsedTime(&total, ctx->ev0, ctx->ev1);
    for (int64_t i = 0; i < nblk; ++i) {
      qb_block_stats st{};
      st.ell = (int64_t)hrec[8 + 6 * i];
      st.w = (int64_t)hrec[8 + 6 * i + 1];
      st.r2 = hrec[8 + 6 * i + 2];
      st.ei = hrec[8 + 6 * i + 3];
      st.kappa_r = hrec[8 + 6 * i + 5] > 0.0 ? hrec[8 + 6 * i + 4] / hrec[8 + 6 * i + 5] : 0.0;
      st.ms = total / (double)nblk;  // one launch for all blocks: the mean
      st.fallback = i == nblk - 1 ? (int32_t)hrec[3] : 0;
      ctx->stats.push_back(st);
    }
    ctx->block_fallbacks = (int)hrec[3];
    if (resid_out) *resid_out = std::sqrt(r2);
    if (!std::isfinite(r2)) return fail(ctx, QB_ERR_CUDA, "non-finite residual");
    if (ctx->hout.Q && k > 0) {  // qb_factor_host: the factors to the caller's host buffers
      const int64_t kc = std::min(k, ctx->hout.kcap);
      QB_CUDA(cudaMemcpy2DAsync(ctx->hout.Q, ctx->hout.ldq * 8, ctx->Qbar.p, ctx->ldq * 8, m * 8, kc,
                                cudaMemcpyDeviceToHost, ctx->stream));
      QB_CUDA(cudaMemcpy2DAsync(ctx->hout.B, ctx->hout.ldb * 8, ctx->Bbar.p, ctx->ldb * 8, n * 8, kc,
                                cudaMemcpyDeviceToHost, ctx->stream));
      QB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    *k_out = k;
    ctx->last_m = m;
    ctx->last_n = n;
    ctx->last_k = k;
    ctx->last_r2 = r2;
    QB_TRY(publish_outputs(ctx, m, n, k, Q_out, ldq_out, B_out, ldb_out));
    return r2 <= eps * eps ? QB_OK : QB_NOT_CONVERGED;
  }

  // ---- residual workspace A^(0) = A (A^(j) overwrites A^(j-1), :112)
  // FP32 contexts ("FP32 path"): the residual stays FP32 and its contractions run
  // on the 3xTF32 tensor-core GEMM (gemm_tf32.cuh); the m x b panel work (CholeskyQR,
  // re-projection) and all norms are FP64.
  const size_t es = is_f32 ? 4 : 8;
  void* Av = Ain;
  int64_t ldA = lda;
  const bool inplace_ok = (flags & QB_OVERWRITE_A) && (lda % (is_f32 ? 4 : 2) == 0) &&
                          ((reinterpret_cast<uintptr_t>(Ain) & 15) == 0);
  if (!inplace_ok) {
    ldA = round_up(m, 16);
    QB_TRY(ensure(ctx, ctx->Awork, es * (size_t)(ldA * n)));
    Av = ctx->Awork.p;  // filled by a0's pass below
  }
  double* A = static_cast<double*>(Av);  // FP64 contexts
  float* A32 = static_cast<float*>(Av);  // FP32 contexts

  // ---- scratch
  const int64_t ldm = round_up(m, 16), ldn = round_up(n, 16), bp = round_up(kMaxB, 16);
  QB_TRY(ensure(ctx, ctx->Om, sizeof(double) * (size_t)(n * bp)));
  QB_TRY(ensure(ctx, ctx->Y, sizeof(double) * (size_t)(ldm * b)));
  QB_TRY(ensure(ctx, ctx->T1, sizeof(double) * (size_t)(round_up(std::max(m, n), 16) * kMaxB)));
  QB_TRY(ensure(ctx, ctx->G, sizeof(double) * bp * bp));
  QB_TRY(ensure(ctx, ctx->L, sizeof(double) * (bp * bp + 8 * 32 * 32)));
  QB_TRY(ensure(ctx, ctx->Rinv, sizeof(double) * bp * bp));
  if (q > 0) {
    QB_TRY(ensure(ctx, ctx->Z, sizeof(double) * (size_t)(ldn * b)));
    QB_TRY(ensure(ctx, ctx->Zt, sizeof(double) * (size_t)(n * bp)));
  }
  if (is_f32) {  // FP32 copies of the panel operands of the tensor-core GEMMs
    QB_TRY(ensure(ctx, ctx->Q32, sizeof(float) * (size_t)(ldm * b)));
    QB_TRY(ensure(ctx, ctx->B32, sizeof(float) * (size_t)(ldn * b)));
  }
  float* Q32 = static_cast<float*>(ctx->Q32.p);
  float* B32 = static_cast<float*>(ctx->B32.p);
  bool b32_copy_pending = false;  // qb_factor_host: B32 of the last block on its way to the host

  // per-CTA partials of the largest reduction (the downdate GEMM grid), sized once up front
  QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)std::max<int64_t>(
                                     ((m + GEMM_BM - 1) / GEMM_BM) * ((n + kBN - 1) / kBN), 16 * ctx->num_sms)));

  // ---- a0: r0^2 = ||A||_F^2; trivial exit (Algorithm 1 line (2), reading R3); fused with the
  // working copy when A is not factored in place (one pass over A instead of two)
  {
    const int grid = (int)std::min<int64_t>(n, 8 * ctx->num_sms);
    QB_TRY(ensure(ctx, ctx->parts, sizeof(double) * (size_t)grid));
    if (!inplace_ok) {
      if (is_f32)
        copy_sumsq_kernel<float><<<grid, RED_THREADS, 0, ctx->stream>>>(static_cast<const float*>(Ain), lda, m, n, A32,
                                                                         ldA, ctx->parts.d());
      else
        copy_sumsq_kernel<double><<<grid, RED_THREADS, 0, ctx->stream>>>(static_cast<const double*>(Ain), lda, m, n, A,
                                                                          ldA, ctx->parts.d());
    } else if (is_f32) {
      sumsq_kernel<float><<<grid, RED_THREADS, 0, ctx->stream>>>(A32, m, n, ldA, ctx->parts.d());
    } else {
      sumsq_kernel<double><<<grid, RED_THREADS, 0, ctx->stream>>>(A, m, n, ldA, ctx->parts.d());
    }
    QB_TRY(check_launch(ctx, "sumsq"));
    QB_TRY(reduce_to_scal(ctx, grid, 0));
    QB_TRY(allreduce_sum(ctx, ctx->scal.d(), 1));  // ||A||_F^2 over the column shards
    QB_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->scal.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    QB_TRY(stream_wait(ctx));
  }
  const double r2_0 = ctx->h_scal[0];
  if (!std::isfinite(r2_0)) return fail(ctx, QB_ERR_INVALID_ARG, "A contains NaN or Inf");
  const double eps2 = eps * eps;
  double r2 = r2_0, ei = r2_0;
  ctx->outQ = nullptr;
  ctx->outB = nullptr;
  if (resid_out) *resid_out = std::sqrt(r2_0);
  ctx->last_k = -1;
  if (r2_0 <= eps2) {
    ctx->last_r2 = r2_0;
    ctx->last_m = m;
    ctx->last_n = n;
    ctx->last_k = 0;
    QB_TRY(grow_factors(ctx, m, n, 1, std::max<int64_t>(kmax_eff, 1)));
    return publish_outputs(ctx, m, n, 0, Q_out, ldq_out, B_out, ldb_out);
  }

  int64_t ell = 0;
  // qb_factor_host: block [c0, c0 + wc) of Q̄ / B̄ still to be copied to the host
  struct {
    int64_t c0 = -1, wc = 0;
  } pending_copy;
  auto host_copy = [&]() -> qb_status {
    if (pending_copy.c0 < 0) return QB_OK;
    const int64_t c0 = pending_copy.c0, wc = pending_copy.wc;
    pending_copy.c0 = -1;
    const size_t es = is_f32 ? 4 : 8;
    const void* qsrc = is_f32 ? static_cast<const void*>(static_cast<const float*>(ctx->Qbar32.p) + c0 * ctx->ldq)
                              : static_cast<const void*>(ctx->Qbar.d() + c0 * ctx->ldq);
    const void* bsrc = is_f32 ? ctx->B32.p : static_cast<const void*>(ctx->Bbar.d() + c0 * ctx->ldb);
    QB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(ctx->hout.Q) + c0 * ctx->hout.ldq * es, ctx->hout.ldq * es, qsrc,
                              ctx->ldq * es, m * es, wc, cudaMemcpyDeviceToHost, ctx->copy_stream));
    QB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(ctx->hout.B) + c0 * ctx->hout.ldb * es, ctx->hout.ldb * es, bsrc,
                              ctx->ldb * es, n * es, wc, cudaMemcpyDeviceToHost, ctx->copy_stream));
    // FP32: B32 is rewritten by the next block's downdate, which waits for this copy first
    // (by then long done); everything else the copies read is final
    if (is_f32) {
      QB_CUDA(cudaEventRecord(ctx->ev_copy, ctx->copy_stream));
      b32_copy_pending = true;
    }
    return QB_OK;
  };
  static const int host_timing = debug_env("QB_HOST_TIMING");  // diagnostics: host time per block phase
  auto now_ms = [] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  while (ell < kmax_eff) {
    const double th0 = host_timing ? now_ms() : 0.0;
    const int64_t w = std::min<int64_t>(b, kmax_eff - ell);
    QB_TRY(grow_factors(ctx, m, n, ell + w, kmax_eff));
    QB_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    double gap_ms = -1.0;  // QB_HOST_TIMING: device idle between the previous block's end and this start
    if (host_timing) {
      if (!ctx->ev_gap) {
        QB_CUDA(cudaEventCreate(&ctx->ev_gap));
      } else if (ell > 0) {
        QB_CUDA(cudaEventSynchronize(ctx->ev0));
        float g = 0.f;
        if (cudaEventElapsedTime(&g, ctx->ev_gap, ctx->ev0) == cudaSuccess) gap_ms = g;
      }
    }
    QB_TRY(reset_flags(ctx));
    ctx->tused = 0;
    double* Qbar = ctx->Qbar.d();
    double* Qi = Qbar + ell * ctx->ldq;
    double* Bi = ctx->Bbar.d() + ell * ctx->ldb;

    // Y = A X for a row-major n x w operand X (ld bp): Ω_i or Z^T
    // FP32 contexts: Q̄32_i = RN_32(Q_i) is written by the orth passes themselves, and the sketch
    // leaves Y32 = RN_32(Y) in ctx->X32 for the first CholeskyQR pass (not on column shards, where
    // Y is the all-reduced sum of the local products)
    float* Qbar32 = static_cast<float*>(ctx->Qbar32.p);
    float* Qi32 = is_f32 ? Qbar32 + ell * ctx->ldq : nullptr;
    float* Y32 = nullptr;
    if (is_f32 && !colsh) {
      // sized for every CholeskyQR pass of the block (Y's and the power steps' Z), so that no
      // later ensure() moves the buffer under Y32
      QB_TRY(ensure(ctx, ctx->X32, sizeof(float) * (size_t)(std::max(ldm, ldn) * w)));
      Y32 = static_cast<float*>(ctx->X32.p);
    }
    auto sketch = [&](const void* X) -> qb_status {
      if (is_f32)
        return gemm_tf(ctx, GEMM_NN, TF_STORE_COL, (int)m, (int)w, (int)n, A32, ldA, static_cast<const float*>(X), bp,
                       ctx->Y.d(), ldm, false, nullptr, true, nullptr, Y32, ldm);
      return gemm(ctx, GEMM_NN, EPI_STORE_COL, (int)m, (int)w, (int)n, A, ldA, static_cast<const double*>(X), bp,
                  ctx->Y.d(), ldm, false, nullptr);
    };
    // Z = A^T X for a column-major m x w FP64 panel X (ld ldx)
    auto adjoint = [&](const double* X, int64_t ldx) -> qb_status {
      if (!is_f32)
        return gemm(ctx, GEMM_TN, EPI_STORE_COL, (int)n, (int)w, (int)m, A, ldA, X, ldx, ctx->Z.d(), ldn, false,
                    nullptr);
      QB_TRY(launch_convert(ctx, X, ldx, m, w, Q32, ldm));
      return gemm_tf(ctx, GEMM_TN, TF_STORE_COL, (int)n, (int)w, (int)m, A32, ldA, Q32, ldm, ctx->Z.d(), ldn, false,
                     nullptr);
    };
    // Z^T (row-major n x w, ld bp) in the residual's precision
    auto transpose_z = [&]() -> qb_status {
      dim3 grid((unsigned)((n + 31) / 32), (unsigned)((w + 31) / 32));
      if (is_f32)
        transpose_kernel<float><<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->Z.d(), ldn, n, w,
                                                                        static_cast<float*>(ctx->Zt.p), bp);
      else
        transpose_kernel<double><<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->Z.d(), ldn, n, w, ctx->Zt.d(), bp);
      return check_launch(ctx, "transpose");
    };

    // line (2): Ω_i = randn(n, w), global columns ell .. ell+w-1, row-major (ld bp); FP32
    // contexts draw RN_32(Ω_i) (reading R18)
    NvtxPhase phase;
    phase("K1 omega + K2 sketch (+C1)");
    QB_CUDA(cudaEventRecord(ctx->evp[0], ctx->stream));
    QB_TRY(launch_omega(ctx, seed, ctx->col_offset, ctx->col_offset + n, ell, w, ctx->Om.p, bp, is_f32 ? 1 : 0));
    // line (3): Y_i = A^(i-1) Ω_i ; Q_i = orth(Y_i)
    QB_TRY(sketch(ctx->Om.p));
    QB_TRY(host_copy());  // the previous block's Q_i / B_i (qb_factor_host)
    if (!rowsh) QB_TRY(allreduce_sum(ctx, ctx->Y.d(), (size_t)(ldm * w)));  // Y = sum_p A_p Omega_p (column shards)
    QB_CUDA(cudaEventRecord(ctx->evp[1], ctx->stream));
    // orth of line (3); a single CholeskyQR pass when the re-projection's orth follows (R11b)
    static const int full_first_orth = debug_env("QB_FULL_FIRST_ORTH");  // experiment: 1 = CholeskyQR2 always
    const bool reproj_follows = ell > 0 && !(flags & QB_NO_REPROJ) && !full_first_orth;
    // orth of a freshly sketched Y into Q_i (and Q̄32_i on FP32 contexts)
    auto orth_y_into = [&](bool single) -> qb_status {
      QB_TRY(span_mark(ctx, PH_ORTH));
      QB_TRY(cholqr2(ctx, ctx->Y.d(), ldm, Qi, ctx->ldq, m, (int)w, rowsh, single, Y32, ldm, Qi32, ctx->ldq));
      return span_mark(ctx, -1);
    };
    auto orth_y = [&]() -> qb_status { return orth_y_into(reproj_follows); };
    phase("K4 orth + K3 power steps");
    if (!(skip_orth_flag(flags) && q > 0)) {
      if (q == 0) QB_TRY(orth_y());
      else QB_TRY(orth_y_into(false));
    }
    // lines (4)-(7): power steps on the residual (reading R9), orth after each application (R10)
    const bool skip_orth = (flags & QB_SKIP_POWER_ORTH) != 0;
    for (int j = 0; j < q && skip_orth; ++j) {  // NEXT-3: Y = A (A^* Y), orth once
      QB_TRY(span_mark(ctx, PH_POWER));
      QB_TRY(adjoint(ctx->Y.d(), ldm));
      if (rowsh) QB_TRY(allreduce_sum(ctx, ctx->Z.d(), (size_t)(ldn * w)));  // Z = sum_p A_p^T Y_p
      QB_TRY(transpose_z());
      QB_TRY(sketch(ctx->Zt.p));
      if (!rowsh) QB_TRY(allreduce_sum(ctx, ctx->Y.d(), (size_t)(ldm * w)));
      QB_TRY(span_mark(ctx, -1));
    }
    if (skip_orth && q > 0) QB_TRY(orth_y());
    for (int j = 0; j < q && !skip_orth; ++j) {
      QB_TRY(span_mark(ctx, PH_POWER));
      QB_TRY(adjoint(Qi, ctx->ldq));
      if (rowsh) QB_TRY(allreduce_sum(ctx, ctx->Z.d(), (size_t)(ldn * w)));  // Z = sum_p A_p^T Q_p
      QB_TRY(span_mark(ctx, -1));
      QB_TRY(span_mark(ctx, PH_ORTH_Z));
      QB_TRY(cholqr2(ctx, ctx->Z.d(), ldn, ctx->Z.d(), ldn, n, (int)w, colsh));
      QB_TRY(span_mark(ctx, -1));
      QB_TRY(span_mark(ctx, PH_POWER));
      QB_TRY(transpose_z());
      QB_TRY(sketch(ctx->Zt.p));
      if (!rowsh) QB_TRY(allreduce_sum(ctx, ctx->Y.d(), (size_t)(ldm * w)));
      QB_TRY(span_mark(ctx, -1));
      if (j == q - 1) QB_TRY(orth_y());  // the last orth of the power scheme, line (6)
      else QB_TRY(orth_y_into(false));
    }
    // line (8) / (3'): Q_i = orth(Q_i - Q̄ (Q̄^* Q_i))  (one projection + orth, reading R11)
    if (ell > 0 && !(flags & QB_NO_REPROJ)) {
      phase("K5 re-projection + orth");
      QB_TRY(ensure(ctx, ctx->W, sizeof(double) * (size_t)(ell * bp)));
      QB_TRY(span_mark(ctx, PH_REPROJ));
      if (is_f32) {  // on the FP32 copies: W = Q̄^T Q_i, Q_i -= Q̄ W (3xTF32), then orth in FP64
        QB_TRY(ensure(ctx, ctx->W32, sizeof(float) * (size_t)(ell * bp)));
        QB_TRY(gemm_tf(ctx, GEMM_TN, TF_STORE_ROW, (int)ell, (int)w, (int)m, Qbar32, ctx->ldq, Qi32, ctx->ldq,
                       ctx->W.d(), bp, false, nullptr));
        if (rowsh) QB_TRY(allreduce_sum(ctx, ctx->W.d(), (size_t)(ell * bp)));  // W = sum_p Q̄_p^T Q_p
        QB_TRY(launch_convert(ctx, ctx->W.d(), bp, w, ell, static_cast<float*>(ctx->W32.p), bp));
        QB_TRY(gemm_tf(ctx, GEMM_NN, TF_SUB_COL, (int)m, (int)w, (int)ell, Qbar32, ctx->ldq,
                       static_cast<const float*>(ctx->W32.p), bp, Qi32, ctx->ldq, false, nullptr));
        // the projected panel to Y (FP64, for the Gram) and X32 (its FP32 source), so that the
        // CholeskyQR2 into Q_i / Q̄32_i is not in place and its usual single pass moves no data
        QB_TRY(ensure(ctx, ctx->X32, sizeof(float) * (size_t)(std::max(ldm, ldn) * w)));
        float* X32 = static_cast<float*>(ctx->X32.p);
        if (tf_gram_on(ctx) && !small_orth(m, (int)w, rowsh)) {  // the passes read only the FP32 copy (R18d)
          QB_TRY(launch_convert(ctx, static_cast<const float*>(Qi32), ctx->ldq, m, w, X32, ldm));
        } else {
          const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m * w + 255) / 256, 8 * ctx->num_sms));
          convert_dual_kernel<<<grid, 256, 0, ctx->stream>>>(Qi32, ctx->ldq, m, w, ctx->Y.d(), ldm, X32, ldm);
          QB_TRY(check_launch(ctx, "convert_dual"));
        }
        QB_TRY(span_mark(ctx, -1));
        QB_TRY(span_mark(ctx, PH_ORTH));
        QB_TRY(cholqr2(ctx, ctx->Y.d(), ldm, Qi, ctx->ldq, m, (int)w, rowsh, false, X32, ldm, Qi32, ctx->ldq));
        QB_TRY(span_mark(ctx, -1));
      } else {
        QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_ROW, (int)ell, (int)w, (int)m, Qbar, ctx->ldq, Qi, ctx->ldq, ctx->W.d(),
                    bp, false, nullptr));
        if (rowsh) QB_TRY(allreduce_sum(ctx, ctx->W.d(), (size_t)(ell * bp)));  // W = sum_p Q̄_p^T Q_p
        QB_TRY(gemm(ctx, GEMM_NN, EPI_SUB_COL, (int)m, (int)w, (int)ell, Qbar, ctx->ldq, ctx->W.d(), bp, Qi,
                    ctx->ldq, false, nullptr));
        QB_TRY(span_mark(ctx, -1));
        QB_TRY(span_mark(ctx, PH_ORTH));
        QB_TRY(cholqr2(ctx, Qi, ctx->ldq, Qi, ctx->ldq, m, (int)w, rowsh));
        QB_TRY(span_mark(ctx, -1));
      }
    }
    // line (9): B_i = Q_i^* A^(i-1) (reading R12), row-major into B̄, plus sum B_i^2 (the EI term)
    int64_t nb_parts = 0;
    phase("K6 B_i = Q_i^T A");
    QB_CUDA(cudaEventRecord(ctx->evp[2], ctx->stream));
    if (is_f32) {
      QB_TRY(gemm_tf(ctx, GEMM_TN, TF_STORE_ROW, (int)w, (int)n, (int)m, Qi32, ctx->ldq, A32, ldA, Bi, ctx->ldb,
                     !rowsh, &nb_parts));
    } else {
      QB_TRY(gemm(ctx, GEMM_TN, EPI_STORE_ROW, (int)w, (int)n, (int)m, Qi, ctx->ldq, A, ldA, Bi, ctx->ldb, !rowsh,
                  &nb_parts));
    }
    if (rowsh) {  // B_i = sum_p Q_p^T A_p, replicated; its norm from the reduced rows
      QB_TRY(allreduce_sum(ctx, Bi, (size_t)(w * ctx->ldb)));
      const int grid = (int)std::min<int64_t>(w, 4 * ctx->num_sms);
      sumsq_kernel<double><<<grid, RED_THREADS, 0, ctx->stream>>>(Bi, n, w, ctx->ldb, ctx->parts.d());
      QB_TRY(check_launch(ctx, "sumsq"));
      nb_parts = grid;
    }
    QB_CUDA(cudaEventRecord(ctx->evp[3], ctx->stream));
    QB_TRY(reduce_to_scal(ctx, nb_parts, 1));
    // line (10): A^(i) = A^(i-1) - Q_i B_i, with sum A^(i)^2 in the epilogue (the stop test, R1)
    int64_t na_parts = 0;
    phase("K7 downdate A -= Q_i B_i");
    QB_CUDA(cudaEventRecord(ctx->evp[4], ctx->stream));
    if (is_f32) {  // A -= RN32(Q_i) RN32(B_i): the residual of the factors the caller receives
      if (b32_copy_pending) {  // the previous block's B32 is still being copied to the host
        QB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copy, 0));
        b32_copy_pending = false;
      }
      QB_TRY(launch_convert(ctx, static_cast<const double*>(Bi), ctx->ldb, n, w, B32, ctx->ldb));
      QB_TRY(gemm_tf(ctx, GEMM_NN, TF_SUB_COL, (int)m, (int)n, (int)w, Qi32, ctx->ldq, B32, ctx->ldb, A32, ldA, true,
                     &na_parts));
    } else {
      QB_TRY(gemm(ctx, GEMM_NN, EPI_SUB_COL, (int)m, (int)n, (int)w, Qi, ctx->ldq, Bi, ctx->ldb, A, ldA, true,
                  &na_parts));
    }
    QB_CUDA(cudaEventRecord(ctx->evp[5], ctx->stream));
    phase("K8 stop test");
    QB_TRY(reduce_to_scal(ctx, na_parts, 0));
    // ||A^(i)||_F^2 (and, on column shards, ||B_i||_F^2) summed over the shards
    QB_TRY(allreduce_sum(ctx, ctx->scal.d(), rowsh ? 1 : 2));
    QB_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->scal.p, 6 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    QB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->status.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    QB_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    const double th1 = host_timing ? now_ms() : 0.0;
    double th_ev0 = 0.0;
    if (host_timing) {  // when did the block's first event complete on the device (host clock)?
      while (cudaEventQuery(ctx->ev0) == cudaErrorNotReady) {
      }
      th_ev0 = now_ms();
    }
    if (host_timing) QB_CUDA(cudaEventRecord(ctx->ev_gap, ctx->stream));  // this block's end on the device
    {
      NvtxRange nv("K8 stop test (host wait)");
      QB_TRY(stream_wait(ctx));
    }
    if (host_timing)
      fprintf(stderr, "[qb host] block at %lld: enqueue %.3f ms, block start +%.3f ms, wait %.3f ms, device gap %.3f ms\n",
              (long long)ell, th1 - th0, th_ev0 - th0, now_ms() - th1, gap_ms);
    if (ctx->h_status[4])
      return fail(ctx, QB_ERR_ORTH_BREAKDOWN, "CholeskyQR failed even with the shift in the block ending at %lld",
                  (long long)(ell + w));
    ctx->block_fallbacks = ctx->h_status[3];
    r2 = ctx->h_scal[0];
    ei -= ctx->h_scal[1];
    ell += w;
    qb_block_stats st{};
    st.ell = ell;
    st.w = w;
    st.r2 = r2;
    st.ei = ei;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    st.ms = ms;
    cudaEventElapsedTime(&ms, ctx->evp[0], ctx->evp[1]);
    st.ms_sketch = ms;
    cudaEventElapsedTime(&ms, ctx->evp[2], ctx->evp[3]);
    st.ms_bmat = ms;
    cudaEventElapsedTime(&ms, ctx->evp[4], ctx->evp[5]);
    st.ms_down = ms;
    st.fallback = ctx->block_fallbacks;
    st.kappa_r = (ctx->h_status[5] && ctx->h_scal[5] > 0.0) ? ctx->h_scal[4] / ctx->h_scal[5] : 0.0;
    {
      double acc[PH_N];
      span_collect(ctx, acc);
      st.ms_orth = acc[PH_ORTH];
      st.ms_orth_z = acc[PH_ORTH_Z];
      st.ms_reproj = acc[PH_REPROJ];
      st.ms_power = acc[PH_POWER];
    }
    ctx->stats.push_back(st);
    if (ctx->hout.Q && ell - w < ctx->hout.kcap) {
      // the block is final (host-synchronised above): its Q_i columns and B_i rows go to the
      // host on the copy stream while the next block computes; enqueued once the next block's
      // sketch is (host_copy below) — enqueued here, ahead of the next block, they held that
      // block's first operations back for the length of the copy (measured: +1.45 ms per block)
      pending_copy = {ell - w, std::min(w, ctx->hout.kcap - (ell - w))};
    }
    if (r2 <= eps2 || !std::isfinite(r2)) QB_TRY(host_copy());
    if (!std::isfinite(r2)) return fail(ctx, QB_ERR_CUDA, "non-finite residual after block ending at %lld", (long long)ell);
    if (r2 <= eps2) break;  // line (11): stop test (R1, R4)
  }
  QB_TRY(host_copy());  // kmax reached without the stop test firing
  *k_out = ell;
  ctx->last_r2 = r2;
  ctx->last_m = m;
  ctx->last_n = n;
  ctx->last_k = ell;
  QB_TRY(publish_outputs(ctx, m, n, ell, Q_out, ldq_out, B_out, ldb_out));
  if (resid_out) *resid_out = std::sqrt(r2);
  return r2 <= eps2 ? QB_OK : QB_NOT_CONVERGED;
}

qb_status qb_factor(qb_ctx ctx, void* Ain, int64_t m, int64_t n, int64_t lda, double eps, int64_t b, int q,
                    uint64_t seed, int64_t kmax, unsigned flags, int64_t* k_out, const void** Q_out,
                    int64_t* ldq_out, const void** B_out, int64_t* ldb_out, double* resid_out) {
  NvtxRange nv("qb_factor");
  const qb_status s = factor_impl(ctx, Ain, m, n, lda, eps, b, q, seed, kmax, flags, k_out, Q_out, ldq_out, B_out,
                                  ldb_out, resid_out);
  // a failed rank of an in-process loopback group releases its peers from the next barrier
  if (s != QB_OK && s != QB_NOT_CONVERGED && ctx && ctx->loop) ctx->loop->abort("a rank failed in qb_factor");
  return s;
}

qb_status qb_factor_host(qb_ctx ctx, const void* A_host, int64_t m, int64_t n, int64_t lda_host, double eps,
                         int64_t b, int q, uint64_t seed, int64_t kmax, int64_t* k, void* Q_host, int64_t ldq_host,
                         void* B_host, int64_t ldb_host, int64_t kcap_host, double* resid) {
  if (!ctx) return QB_ERR_INVALID_ARG;
  if (!A_host || !k || m < 1 || n < 1 || lda_host < m || kcap_host < 0 || (kcap_host > 0 && (!Q_host || !B_host)) ||
      (Q_host && ldq_host < m) || (B_host && ldb_host < n))
    return fail(ctx, QB_ERR_INVALID_ARG, "qb_factor_host: bad arguments");
  QB_CUDA(cudaSetDevice(ctx->device));
  const int64_t es = ctx->dtype == QB_F64 ? 8 : 4;
  const int64_t ldA = round_up(m, 16);
  DevBuf& dst = ctx->Astage;  // staged input, factored in place
  QB_TRY(ensure(ctx, dst, (size_t)(es * ldA * n)));
  QB_CUDA(cudaMemcpy2DAsync(dst.p, ldA * es, A_host, lda_host * es, m * es, n, cudaMemcpyHostToDevice, ctx->stream));
  const void* Qd = nullptr;
  const void* Bd = nullptr;
  int64_t ldq = 0, ldb = 0;
  if (!ctx->copy_stream) {
    QB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    QB_CUDA(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
  }
  // Q_i / B_i stream to the host block by block inside qb_factor (overlapping the next block)
  ctx->hout.Q = kcap_host > 0 ? Q_host : nullptr;
  ctx->hout.B = B_host;
  ctx->hout.ldq = ldq_host;
  ctx->hout.ldb = ldb_host;
  ctx->hout.kcap = kcap_host;
  qb_status s = qb_factor(ctx, dst.p, m, n, ldA, eps, b, q, seed, kmax, QB_OVERWRITE_A, k, &Qd, &ldq, &Bd, &ldb, resid);
  ctx->hout.Q = nullptr;
  ctx->hout.B = nullptr;
  const cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
  if (s != QB_OK && s != QB_NOT_CONVERGED) return s;
  if (ce != cudaSuccess) return fail(ctx, QB_ERR_CUDA, "qb_factor_host copies: %s", cudaGetErrorString(ce));
  QB_CUDA(cudaStreamSynchronize(ctx->stream));
  return s;
}

}  // extern "C"
