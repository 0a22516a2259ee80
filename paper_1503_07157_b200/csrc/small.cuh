// Small and bandwidth-bound kernels of the QB path:
//   sumsq_kernel       a0: partial sums of squares of A (||A||_F^2)
//   copy_sumsq_kernel  the same fused with the working copy of A
//   reduce_kernel      K8: fixed-order sum of per-CTA partials -> one FP64 scalar
//   splitk_reduce      fixed-order sum of split-K partials (+ sum of squares, the EI term)
//   transpose_kernel   column-major <-> row-major copy of a tall-skinny panel
//   chol_cluster_kernel  K4 core: the CholeskyQR factor T (R^-1, or a Newton-Schulz step) of
//                      a w x w Gram matrix on one 8-CTA cluster, shifted fallback (reading R8)
// All reductions run in a fixed order, so results are bitwise reproducible.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace qbk {

constexpr int RED_THREADS = 256;

// Per-block sum of squares of a column-major m x n matrix (ld), grid-stride over columns.
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) sumsq_kernel(const T* __restrict__ A, int64_t m, int64_t n,
                                                            int64_t lda, double* __restrict__ partials) {
  __shared__ double red[RED_THREADS / 32];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const T* col = A + j * lda;
    for (int64_t i = threadIdx.x; i < m; i += RED_THREADS) {
      const double v = static_cast<double>(col[i]);
      s = fma(v, v, s);
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

// out[slot] = sum of partials[0..count) in a fixed order (single CTA).
__global__ void __launch_bounds__(RED_THREADS) reduce_kernel(const double* __restrict__ partials, int64_t count,
                                                             double* __restrict__ out, int slot) {
  __shared__ double red[RED_THREADS / 32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += RED_THREADS) s += partials[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) t += red[w];
    out[slot] = t;
  }
}

// out[r*ldo + c] = sum_{s<S} P[s*stride + r*ldp + c] for r < rows, c < cols (any layout
// where "r" is the strided index), or out -= that sum when `subtract`.  Optional per-block
// sum of squares of the result.  `sub` (1, 2, 4 or 8) consecutive lanes share an output when there
// are few outputs and many splits: lane j of the group sums splits [j S/sub, (j+1) S/sub) in order
// and the group adds its partial sums in lane order — a fixed order either way.
__global__ void __launch_bounds__(RED_THREADS) splitk_reduce_kernel(const double* __restrict__ P, int S, int64_t stride,
                                                                    int64_t rows, int64_t cols, int64_t ldp,
                                                                    double* __restrict__ out, int64_t ldo,
                                                                    double* __restrict__ sq_partials,
                                                                    const int* __restrict__ gate, int subtract,
                                                                    float* __restrict__ out32 = nullptr,
                                                                    int64_t ld32 = 0, int sub = 1) {
  if (gate != nullptr && __ldcg(gate) == 0) return;
  __shared__ double red[RED_THREADS / 32];
  double sq = 0.0;
  const int64_t total = rows * cols, nthr = total * sub;
  const int lane = threadIdx.x & 31, part = lane % sub;
  const int s_lo = static_cast<int>((static_cast<int64_t>(S) * part) / sub);
  const int s_hi = static_cast<int>((static_cast<int64_t>(S) * (part + 1)) / sub);
  // warp-uniform trip count (the group sums shuffle)
  for (int64_t base = (blockIdx.x * static_cast<int64_t>(RED_THREADS) + threadIdx.x) - lane; base < nthr;
       base += static_cast<int64_t>(gridDim.x) * RED_THREADS) {
    const int64_t g = base + lane;
    const bool live = g < nthr;
    const int64_t idx = live ? g / sub : 0;
    const int64_t r = idx / cols, c = idx - r * cols;
    const double* src = P + r * ldp + c;
    double v = 0.0;
    if (live) {
#pragma unroll 8
      for (int s2 = s_lo; s2 < s_hi; ++s2) v += src[s2 * stride];
    }
    for (int k = 1; k < sub; ++k) {
      const double o = __shfl_down_sync(0xffffffffu, v, k);
      if (part == 0) v += o;  // ((p0 + p1) + p2) + ...
    }
    if (live && part == 0) {
      if (subtract) v = out[r * ldo + c] - v;  // C -= sum of the split products
      out[r * ldo + c] = v;
      if (out32 != nullptr) out32[r * ld32 + c] = static_cast<float>(v);  // FP32 contexts: RN_32 copy
      sq = fma(v, v, sq);
    }
  }
  if (sq_partials != nullptr) {
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < RED_THREADS / 32; ++w) t += red[w];
      sq_partials[blockIdx.x] = t;
    }
  }
}

// Lanes per output for splitk_reduce_kernel: more when the outputs alone leave most of the GPU idle
// and each lane would still sum at least 8 splits.
inline int splitk_sub(int64_t total, int S, int num_sms) {
  int sub = 1;
  while (sub < 8 && total * sub * 2 <= static_cast<int64_t>(4) * num_sms * RED_THREADS && S / (sub * 2) >= 8) sub *= 2;
  return sub;
}

// Loopback collective: out = sum_r in[r] in rank order, one kernel over the data
// of all in-process ranks (no rank's kernel waits on another's).
constexpr int LOOP_MAX = 8;
struct LoopPtrs {
  const double* p[LOOP_MAX];
};
__global__ void __launch_bounds__(256) loopback_sum_kernel(LoopPtrs in, int nranks, int64_t count,
                                                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < count; i += static_cast<int64_t>(gridDim.x) * 256) {
    double s = in.p[0][i];
    for (int r = 1; r < nranks; ++r) s += in.p[r][i];
    out[i] = s;
  }
}

// a0 fused with the working copy (qb_factor without QB_OVERWRITE_A): dst = src column by column
// and the same per-block sums of squares as sumsq_kernel, in the same order (bitwise equal r0^2).
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) copy_sumsq_kernel(const T* __restrict__ src, int64_t lds, int64_t m,
                                                                 int64_t n, T* __restrict__ dst, int64_t ldd,
                                                                 double* __restrict__ partials) {
  __shared__ double red[RED_THREADS / 32];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const T* col = src + j * lds;
    T* out = dst + j * ldd;
    for (int64_t i = threadIdx.x; i < m; i += RED_THREADS) {
      const T x = col[i];
      out[i] = x;
      const double v = static_cast<double>(x);
      s = fma(v, v, s);
    }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

// out[r*ldo + c] = in[r + c*ldi] for r < rows, c < cols (column-major -> row-major).
template <typename Tout>
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows,
                                                        int64_t cols, Tout* __restrict__ out, int64_t ldo) {
  __shared__ double t[32][33];
  const int64_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = r0 + threadIdx.x, c = c0 + j;
    if (r < rows && c < cols) t[j][threadIdx.x] = in[r + c * ldi];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < rows && c < cols) out[r * ldo + c] = static_cast<Tout>(t[threadIdx.x][j]);
  }
}

// out[r + c*ldo] = (Tout) in[r + c*ldi], column-major rows x cols (FP32 <-> FP64 staging of
// the FP32 path).
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) convert_kernel(const Tin* __restrict__ in, int64_t ldi, int64_t rows,
                                                      int64_t cols, Tout* __restrict__ out, int64_t ldo,
                                                      const int* __restrict__ gate) {
  if (gate != nullptr && __ldcg(gate) == 0) return;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    out[r + c * ldo] = static_cast<Tout>(in[r + c * ldi]);
  }
}

// p[0..n) = 0 (device flag words).  A kernel rather than cudaMemsetAsync: a memset may queue on
// a copy engine behind qb_factor_host's block copies to the host and stall the next block.
// status[0..7] = 0 and kappa[0..1] = 0 (the start of a block)
__global__ void reset_block_kernel(int* __restrict__ status, double* __restrict__ kappa) {
  if (threadIdx.x < 8) status[threadIdx.x] = 0;
  if (threadIdx.x < 2) kappa[threadIdx.x] = 0.0;
}

__global__ void zero_ints_kernel(int* __restrict__ p, int n) {
  if (static_cast<int>(threadIdx.x) < n) p[threadIdx.x] = 0;
}

// out = (double) in and out2 = in, column-major rows x cols (FP32 contexts: an FP32 panel and its
// FP64 copy for the Gram, R18c).
__global__ void __launch_bounds__(256) convert_dual_kernel(const float* __restrict__ in, int64_t ldi, int64_t rows,
                                                           int64_t cols, double* __restrict__ out, int64_t ldo,
                                                           float* __restrict__ out2, int64_t ldo2) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    const float v = in[r + c * ldi];
    out[r + c * ldo] = static_cast<double>(v);
    out2[r + c * ldo2] = v;
  }
}

// dst = src (column-major rows x cols) if *gate == 0, or if *gate != 0 with when_set (CholeskyQR2:
// moves the final pass's result from the scratch to the destination; see cholqr2).
__global__ void __launch_bounds__(256) gated_copy_kernel(const double* __restrict__ src, int64_t lds,
                                                         double* __restrict__ dst, int64_t ldd, int64_t rows,
                                                         int64_t cols, const int* __restrict__ gate,
                                                         const float* __restrict__ src32 = nullptr,
                                                         int64_t lds32 = 0, float* __restrict__ dst32 = nullptr,
                                                         int64_t ldd32 = 0, int when_set = 0) {
  if ((__ldcg(gate) != 0) != (when_set != 0)) return;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    dst[r + c * ldd] = src[r + c * lds];
    if (dst32 != nullptr) dst32[r + c * ldd32] = src32[r + c * lds32];  // and its FP32 copy
  }
}

// ---------------------------------------------------------------------------------------
// K4 core — chol_cluster_kernel: the CholeskyQR "T" of a w x w Gram matrix G = X^T X
// (column-major), w <= 256, on ONE thread-block cluster of 8 CTAs (one 32-column panel of the
// factor per CTA, kept in that CTA's shared memory; peers read it through distributed shared
// memory).  Writes T column-major into `Tout` (ld ldt) such that X T has orthonormal columns:
//   * Newton-Schulz: if ||G - I||_F <= sqrt(ns_tol2), X is orthonormal to first order and
//     T = I - (G - I)/2 (one step towards the polar factor, error (3/4)||G - I||^2).  status 3.
//   * Cholesky: right-looking over the 32-column panels.  Step p: warp 0 of CTA p factors its
//     32 x 32 diagonal block and inverts it in registers (lane = row, shuffles), the CTA solves
//     its panel below; the CTAs that own later panels copy the rows they need of panel p over
//     DSMEM and apply the rank-32 update.  Then CTA J forms block column J of L^-1 right-
//     looking over K = J.. (X_JJ = L_JJ^-1; X_KJ = -L_KK^-1 acc_K; acc_I += L_IK X_KJ for I > K,
//     one DSMEM copy of panel K per step) and writes Tout(row, col) = L^-1(row, col), i.e. read
//     ROW-major Tout is R^-1 = L^-T (upper triangular).  A pivot that is not > tol * G_jj (or
//     NaN) is a breakdown (reading R8): the cluster restarts once with the shifted-CholeskyQR
//     shift s = 11 (m w + w (w+1)) u trace(G).  status[0] = 0 ok / 1 shifted / 2 failed.
// Flags: status[1] = 1 when the shift was used (gates the extra CholeskyQR3 passes),
// status[2] = 1 when the Cholesky path ran (gates CholeskyQR's second pass; a Newton-Schulz
// first pass needs none), status[3] += 1 per shifted factorization, status[4] = 1 on failure.
// `gate` (may be null): the kernel does nothing unless *gate != 0.
constexpr int CHOL_MAXW = 256;
constexpr int CHOL_NB = 32;
constexpr int CHOL_CTAS = 8;
constexpr int CHOL_THREADS = 256;
constexpr int CHOL_PLD = CHOL_NB + 1;
constexpr int CHOL_SMEM = (3 * CHOL_MAXW * CHOL_PLD + 2 * CHOL_NB * CHOL_PLD) * 8;
constexpr int CHOL_ST_NS = 3;
#ifdef QB_CHOL_TIMING  // development instrumentation: phase timestamps of CTA 0 (not in product builds)
__device__ unsigned long long qb_chol_ts[64];
#define CHOL_TS(i)                                                                                     \
  do {                                                                                                 \
    if (threadIdx.x == 0 && cluster.block_rank() == 0) {                                               \
      unsigned long long t_;                                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                           \
      qb_chol_ts[(i)] = t_;                                                                            \
    }                                                                                                  \
  } while (0)
#else
#define CHOL_TS(i) do { } while (0)
#endif

// dst[i][k] = src[(r0 + i)][k] for i < n, k < 32 (row stride PLD), src in a peer's shared memory
// (DSMEM, generic loads): eight loads in flight per thread before the stores.
__device__ __forceinline__ void chol_copy_rows(double* __restrict__ dst, const double* __restrict__ src, int r0,
                                               int n) {
  constexpr int PLD = CHOL_PLD;
  const int total = n * CHOL_NB;
  for (int base = threadIdx.x; base < total; base += 8 * CHOL_THREADS) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * CHOL_THREADS;
      v[u] = idx < total ? src[(r0 + idx / CHOL_NB) * PLD + (idx % CHOL_NB)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * CHOL_THREADS;
      if (idx < total) dst[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = v[u];
    }
  }
}

// rows [r0, r1) of A (ld PLD) times B^T restricted to 32 columns: out(i, c) = sum_k A(i,k) B(c,k),
// four rows per warp pass (independent FMA chains); `op` consumes (i, c, value).
template <typename Op>
__device__ __forceinline__ void chol_rows_times_bt(const double* A, const double* B, int r0, int r1, int ncols,
                                                   Op op) {
  constexpr int PLD = CHOL_PLD;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane;
  for (int i = r0 + 4 * warp; i < r1; i += 4 * (CHOL_THREADS / 32)) {
    // 4 rows x 2 halves of k: 8 independent FMA chains (FP64 latency)
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
    const bool v1 = i + 1 < r1, v2 = i + 2 < r1, v3 = i + 3 < r1;
#pragma unroll 8
    for (int k = 0; k < CHOL_NB / 2; ++k) {
      const int kh = k + CHOL_NB / 2;
      const double b = B[c * PLD + k], bh = B[c * PLD + kh];
      a0 = fma(A[i * PLD + k], b, a0);
      e0 = fma(A[i * PLD + kh], bh, e0);
      if (v1) {
        a1 = fma(A[(i + 1) * PLD + k], b, a1);
        e1 = fma(A[(i + 1) * PLD + kh], bh, e1);
      }
      if (v2) {
        a2 = fma(A[(i + 2) * PLD + k], b, a2);
        e2 = fma(A[(i + 2) * PLD + kh], bh, e2);
      }
      if (v3) {
        a3 = fma(A[(i + 3) * PLD + k], b, a3);
        e3 = fma(A[(i + 3) * PLD + kh], bh, e3);
      }
    }
    __syncwarp();
    if (c < ncols) {
      op(i, c, a0 + e0);
      if (v1) op(i + 1, c, a1 + e1);
      if (v2) op(i + 2, c, a2 + e2);
      if (v3) op(i + 3, c, a3 + e3);
    }
  }
}

__global__ void __cluster_dims__(CHOL_CTAS, 1, 1) __launch_bounds__(CHOL_THREADS)
    chol_cluster_kernel(const double* __restrict__ G, int64_t ldg, int w, int64_t m_rows, double* __restrict__ Tout,
                        int64_t ldt, int* __restrict__ status, double tol, double ns_tol2,
                        const int* __restrict__ gate, double* __restrict__ kappa) {
  if (gate != nullptr && __ldcg(gate) == 0) return;  // same value in every CTA of the cluster
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int PLD = CHOL_PLD;
  extern __shared__ double sm[];
  double* P = sm;                      // [256][PLD] own panel: rows 32*cta.., columns 32*cta..+31
  double* X = P + CHOL_MAXW * PLD;     // [256][PLD] block column of L^-1 (accumulated)
  double* S = X + CHOL_MAXW * PLD;     // [256][PLD] staged rows of a peer panel
  double* Di = S + CHOL_MAXW * PLD;    // [32][PLD] L11^-1 (identity-padded), read by peers
  double* Dt = Di + CHOL_NB * PLD;     // [32][PLD] staged peer L_KK^-1
  __shared__ double red[2][CHOL_THREADS / 32];
  __shared__ double s_part[2], s_tot, s_shift;
  __shared__ int s_fail;
  __shared__ double s_lb[2][CHOL_NB];  // the pivot CTA's warp 0: pivot columns, then 1/diag
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = static_cast<int>(cluster.block_rank());
  const int nbk = (w + CHOL_NB - 1) / CHOL_NB;
  const bool active = cta < nbk;
  const int p0 = cta * CHOL_NB;
  const int rows = active ? w - p0 : 0, nb = active ? min(CHOL_NB, w - p0) : 0;
  CHOL_TS(0);

  // ---- Newton-Schulz test ||G - I||_F^2 and trace(G) over the own column block (rank order)
  double e2 = 0.0, tr = 0.0;
  for (int idx = tid; idx < w * nb; idx += CHOL_THREADS) {
    const int i = idx % w, j = p0 + idx / w;
    const double g = __ldcg(G + i + static_cast<int64_t>(j) * ldg);
    const double d = g - (i == j ? 1.0 : 0.0);
    e2 = fma(d, d, e2);
    if (i == j) tr += g;
  }
  e2 = warp_sum(e2);
  tr = warp_sum(tr);
  if (lane == 0) {
    red[0][warp] = e2;
    red[1][warp] = tr;
  }
  __syncthreads();
  if (tid == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int k = 0; k < CHOL_THREADS / 32; ++k) {
      t0 += red[0][k];
      t1 += red[1][k];
    }
    s_part[0] = t0;
    s_part[1] = t1;
  }
  cluster.sync();
  if (tid == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int r = 0; r < CHOL_CTAS; ++r) {
      const double* pr = cluster.map_shared_rank(s_part, r);
      t0 += pr[0];
      t1 += pr[1];
    }
    s_tot = t0;
    s_shift = 11.0 * (static_cast<double>(m_rows) * w + static_cast<double>(w) * (w + 1)) * 0x1p-53 * t1;
  }
  __syncthreads();
  if (ns_tol2 >= 0.0 && s_tot <= ns_tol2) {
    for (int idx = tid; idx < w * nb; idx += CHOL_THREADS) {
      const int i = idx % w, j = p0 + idx / w;  // T(i, j) = delta_ij - (G(i,j) - delta_ij)/2
      const double d = __ldcg(G + i + static_cast<int64_t>(j) * ldg) - (i == j ? 1.0 : 0.0);
      Tout[i + static_cast<int64_t>(j) * ldt] = (i == j ? 1.0 : 0.0) - 0.5 * d;
    }
    if (cta == 0 && tid == 0) status[0] = CHOL_ST_NS;
    cluster.sync();  // peers may still read s_part
    return;
  }
  // tolerance reference of the own diagonal block, lane = row
  const double gdiag = (lane < nb) ? __ldcg(G + (p0 + lane) + static_cast<int64_t>(p0 + lane) * ldg) : 1.0;

  int attempt = 0;
  bool failed = false;
  for (; attempt < 2; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : s_shift;
    // columns nb..31 of a narrow last panel are zero: the 32-wide products below multiply them
    // by the zero upper triangle of L11^-1, and stale shared memory could hold NaN patterns
    for (int idx = tid; idx < rows * CHOL_NB; idx += CHOL_THREADS) {
      const int i = idx % rows, j = idx / rows;
      double v = j < nb ? __ldcg(G + (p0 + i) + static_cast<int64_t>(p0 + j) * ldg) : 0.0;
      if (i == j) v += shift;
      P[i * PLD + j] = v;
    }
    // every 32-row block of this CTA's block column of L^-1 up to the last panel's, padding rows of a
    // narrow last block included (their zeros meet the identity padding of L_KK^-1)
    if (active)
      for (int idx = tid; idx < (nbk - cta) * CHOL_NB * CHOL_NB; idx += CHOL_THREADS)
        X[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = 0.0;
    if (tid == 0) s_fail = 0;
    CHOL_TS(1);
    cluster.sync();  // panels loaded; no peer still reads the previous attempt's panels
    CHOL_TS(2);
    failed = false;
    for (int p = 0; p < nbk; ++p) {
      if (cta == p) {
        if (warp == 0) {
          // Cholesky of the nb x nb diagonal block in registers: lane = row, a[c] = L(lane, c)
          double a[CHOL_NB];
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c)
            a[c] = (lane < nb && c < nb && c <= lane) ? P[lane * PLD + c] : (c == lane ? 1.0 : 0.0);
          // (dependent FP64 latency dominates this single-warp code: reciprocal square roots
          // instead of divisions, split accumulators in the substitution)
          if (p == 0) CHOL_TS(3);
          int bad = 0;
          double rdiag = 1.0;  // 1 / L(lane, lane)
          // pivot j: lane j checks its pivot against tol * G_jj; the column is scaled by 1/sqrt(d)
          auto pivot = [&](int j) -> double {
            const double d = __shfl_sync(0xffffffffu, a[j], j);
            if (lane == j && j < nb && (!(d > tol * gdiag) || !(d > 0.0))) bad = 1;
            const double ri = rsqrt(d);
            const double l = lane > j ? a[j] * ri : (lane == j ? d * ri : 0.0);
            if (lane == j) rdiag = ri;
            a[j] = l;
            return l;
          };
          // right-looking with a one-column lookahead: column jj+1 gets pivot jj's update first and
          // pivot jj+1 is formed before the rest of pivot jj's updates, so the dependent
          // pivot chain overlaps the independent column updates
#ifdef QB_CHOL_SHFL  // round-1 variant: the pivot column broadcast by shuffles (2 SHFL per FP64 value)
          double l = pivot(0);
#pragma unroll
          for (int jj = 0; jj < CHOL_NB; ++jj) {
            double lnext = 0.0;
            if (jj + 1 < CHOL_NB) {
              const double lc = __shfl_sync(0xffffffffu, l, jj + 1);
              if (lane >= jj + 1) a[jj + 1] = fma(-l, lc, a[jj + 1]);
              lnext = pivot(jj + 1);
            }
#pragma unroll
            for (int c = 0; c < CHOL_NB; ++c) {  // fixed bounds: a[] stays in registers
              if (c > jj + 1) {
                const double lc = __shfl_sync(0xffffffffu, l, c);
                if (lane >= c) a[c] = fma(-l, lc, a[c]);
              }
            }
            l = lnext;
          }
#else
          // the pivot column goes through shared memory (one store per lane, then broadcast loads:
          // the single warp's shuffle pipe was the bottleneck, 12 us per 32 x 32 block); two buffers,
          // because pivot jj+1 is formed (lookahead) before pivot jj's remaining updates read theirs
          double l = pivot(0);
          s_lb[0][lane] = l;
          __syncwarp();
#pragma unroll
          for (int jj = 0; jj < CHOL_NB; ++jj) {
            const double* sl = s_lb[jj & 1];
            double lnext = 0.0;
            if (jj + 1 < CHOL_NB) {
              const double lc = sl[jj + 1];
              if (lane >= jj + 1) a[jj + 1] = fma(-l, lc, a[jj + 1]);
              lnext = pivot(jj + 1);
              s_lb[(jj + 1) & 1][lane] = lnext;
            }
#pragma unroll
            for (int c = 0; c < CHOL_NB; ++c) {  // fixed bounds: a[] stays in registers
              if (c > jj + 1) {
                const double lc = sl[c];
                if (lane >= c) a[c] = fma(-l, lc, a[c]);
              }
            }
            __syncwarp();  // buffer jj & 1 is rewritten by pivot jj + 2
            l = lnext;
          }
#endif
          bad = __any_sync(0xffffffffu, bad);
          if (p == 0) CHOL_TS(4);
          // L11^-1, column `lane`, right-looking: x_r = v_r / L(r, r), then v_r2 -= L(r2, r) x_r for
          // r2 > r (L(r2, r) broadcast from lane r2); the dependent chain is two operations per row
          double x[CHOL_NB];
#pragma unroll
          for (int r = 0; r < CHOL_NB; ++r) x[r] = (r == lane) ? 1.0 : 0.0;
#ifdef QB_CHOL_SHFL
#pragma unroll
          for (int r = 0; r < CHOL_NB; ++r) {
            x[r] *= __shfl_sync(0xffffffffu, rdiag, r);
#pragma unroll
            for (int r2 = 0; r2 < CHOL_NB; ++r2)
              if (r2 > r) x[r2] = fma(-__shfl_sync(0xffffffffu, a[r], r2), x[r], x[r2]);
          }
#else
          // L (identity-padded) and 1/diag to shared memory (S is free on the pivot CTA during its
          // diagonal step); L(r2, r) is the same for every lane: broadcast loads
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c) S[lane * PLD + c] = (c <= lane) ? a[c] : 0.0;
          s_lb[0][lane] = rdiag;
          __syncwarp();
#pragma unroll
          for (int r = 0; r < CHOL_NB; ++r) {
            x[r] *= s_lb[0][r];
#pragma unroll
            for (int r2 = 0; r2 < CHOL_NB; ++r2)
              if (r2 > r) x[r2] = fma(-S[r2 * PLD + r], x[r], x[r2]);
          }
#endif
          if (p == 0) CHOL_TS(5);
#pragma unroll
          for (int r = 0; r < CHOL_NB; ++r) Di[r * PLD + lane] = (r >= lane) ? x[r] : 0.0;
          if (lane < nb) {
#pragma unroll
            for (int c = 0; c < CHOL_NB; ++c)
              if (c < nb) P[lane * PLD + c] = (c <= lane) ? a[c] : 0.0;
          }
          if (lane == 0) s_fail = bad;
        }
        __syncthreads();
        if (!s_fail) {  // panel below the diagonal block: L21 = P21 L11^-T, in place
          chol_rows_times_bt(P, Di, nb, rows, nb, [&](int i, int c, double v) { P[i * PLD + c] = v; });
        }
      }
      if (p == 0) CHOL_TS(6);
      cluster.sync();
      if (p == 0) CHOL_TS(7);
      if (*cluster.map_shared_rank(&s_fail, p)) {
        // every thread of every CTA has read CTA p's flag before any CTA passes this barrier, so
        // CTA p cannot reset it (next attempt) or reload its panel while a peer still reads them;
        // the flag is constant until then, so all threads take this branch together
        cluster.sync();
        failed = true;
        break;
      }
      if (active && cta > p) {  // rank-32 update of the own panel with panel p's rows p0.. (over DSMEM)
        chol_copy_rows(S, cluster.map_shared_rank(P, p), p0 - p * CHOL_NB, rows);
        __syncthreads();
        chol_rows_times_bt(S, S, 0, rows, nb, [&](int i, int c, double v) { P[i * PLD + c] -= v; });
      }
      // the block columns of L^-1 (T = R^-1 = L^-T) whose diagonal blocks are done advance by one
      // step while the later CTAs update their panels: CTA J's step K needs only L_KK^-1 and panel K
      if (active && cta <= p) {  // block column J = cta of L^-1: its step K = p (panel p is final)
        const int K = p;
        double* XK = X + (K - cta) * CHOL_NB * PLD;
        if (K == cta) {
          for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += CHOL_THREADS)
            XK[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = Di[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)];
        } else {  // X_KJ = -L_KK^-1 acc_K
          chol_copy_rows(Dt, cluster.map_shared_rank(Di, K), 0, CHOL_NB);
          __syncthreads();
          const int r = tid >> 3, c0 = (tid & 7) * 4;  // thread owns X_KJ(r, c0..c0+3)
          double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
#pragma unroll 8
          for (int t = 0; t < CHOL_NB / 2; ++t) {
            const int th = t + CHOL_NB / 2;
            const double d = Dt[r * PLD + t], dh = Dt[r * PLD + th];
            v0 = fma(d, XK[t * PLD + c0], v0);
            v1 = fma(d, XK[t * PLD + c0 + 1], v1);
            v2 = fma(d, XK[t * PLD + c0 + 2], v2);
            v3 = fma(d, XK[t * PLD + c0 + 3], v3);
            u0 = fma(dh, XK[th * PLD + c0], u0);
            u1 = fma(dh, XK[th * PLD + c0 + 1], u1);
            u2 = fma(dh, XK[th * PLD + c0 + 2], u2);
            u3 = fma(dh, XK[th * PLD + c0 + 3], u3);
          }
          __syncthreads();
          XK[r * PLD + c0] = -(v0 + u0);
          XK[r * PLD + c0 + 1] = -(v1 + u1);
          XK[r * PLD + c0 + 2] = -(v2 + u2);
          XK[r * PLD + c0 + 3] = -(v3 + u3);
        }
        const int below = w - (K + 1) * CHOL_NB;  // rows of panel K under its diagonal block
        if (below > 0) {
          chol_copy_rows(S, cluster.map_shared_rank(P, K), CHOL_NB, below);
          __syncthreads();
          // acc_I += L_IK X_KJ for the rows below block K: out(i, c) = sum_k S(i, k) XK(k, c)
          double* acc = X + (K + 1 - cta) * CHOL_NB * PLD;
          for (int i = 4 * warp; i < below; i += 4 * (CHOL_THREADS / 32)) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
            const bool q1 = i + 1 < below, q2 = i + 2 < below, q3 = i + 3 < below;
#pragma unroll 8
            for (int k = 0; k < CHOL_NB / 2; ++k) {
              const int kh = k + CHOL_NB / 2;
              const double xk = XK[k * PLD + lane], xh = XK[kh * PLD + lane];
              a0 = fma(S[i * PLD + k], xk, a0);
              e0 = fma(S[i * PLD + kh], xh, e0);
              if (q1) {
                a1 = fma(S[(i + 1) * PLD + k], xk, a1);
                e1 = fma(S[(i + 1) * PLD + kh], xh, e1);
              }
              if (q2) {
                a2 = fma(S[(i + 2) * PLD + k], xk, a2);
                e2 = fma(S[(i + 2) * PLD + kh], xh, e2);
              }
              if (q3) {
                a3 = fma(S[(i + 3) * PLD + k], xk, a3);
                e3 = fma(S[(i + 3) * PLD + kh], xh, e3);
              }
            }
            acc[i * PLD + lane] += a0 + e0;
            if (q1) acc[(i + 1) * PLD + lane] += a1 + e1;
            if (q2) acc[(i + 2) * PLD + lane] += a2 + e2;
            if (q3) acc[(i + 3) * PLD + lane] += a3 + e3;
          }
        }
        __syncthreads();
      }
      // no barrier here: the next step's pivot CTA reads only its own shared memory until the next
      // step's barrier publishes its panel, and nothing a peer reads is rewritten before that barrier
      CHOL_TS(8 + 2 * p);
      CHOL_TS(9 + 2 * p);
    }
    if (!failed) break;
  }
  if (cta == 0 && tid == 0) {
    // kappa-proxy of the block (qb_stats): max / min diagonal of the first factorization's R
    if (kappa != nullptr && attempt < 2 && atomicCAS(status + 5, 0, 1) == 0) {
      double dmax = 0.0, dmin = 1e300;
      for (int q = 0; q < nbk; ++q) {
        const double* Pq = cluster.map_shared_rank(P, q);
        const int nbq = min(CHOL_NB, w - q * CHOL_NB);
        for (int i = 0; i < nbq; ++i) {
          const double d = Pq[i * PLD + i];
          dmax = fmax(dmax, d);
          dmin = fmin(dmin, d);
        }
      }
      kappa[0] = dmax;
      kappa[1] = dmin;
    }
    status[0] = attempt;  // 0, 1, or 2 (= failed twice)
    status[2] = 1;
    if (attempt == 1) {
      status[1] = 1;
      atomicAdd(status + 3, 1);
    }
    if (attempt >= 2) status[4] = 1;
  }
  if (attempt >= 2) {
    cluster.sync();
    return;
  }

  CHOL_TS(30);
  // ---- L^-1 is complete (its block columns advanced inside the factor loop)
  if (active) {
    for (int idx = tid; idx < w * nb; idx += CHOL_THREADS) {
      const int row = idx % w, c = idx / w;
      Tout[row + static_cast<int64_t>(p0 + c) * ldt] = row >= p0 ? X[(row - p0) * PLD + c] : 0.0;
    }
  }
  CHOL_TS(31);
  cluster.sync();  // keep this CTA's shared memory alive while peers read it
  CHOL_TS(32);
}

}  // namespace qbk

namespace qbk {

// ---------------------------------------------------------------- whole CholeskyQR2 in one CTA
// For panels small enough to live in one CTA's shared memory (m w <= SCQR_MAX_ELEMS, w <= 64) the
// complete orth of cholqr2() — every pass, the Newton-Schulz shortcut (reading R7b), the shifted
// CholeskyQR3 fallback (R8) and the single-pass variant (R11b) — runs in ONE launch instead of the
// ~15 launches (Gram GEMM + split-K reduction, cluster Cholesky, X T GEMM, gated copies, gated
// fallback passes) of the general path, whose fixed costs dominate small problems (BASELINE
// configs[0]: 400 x 10 panels).  Same algorithm and flags as the general path:
//   pass:  G = X^T X (fixed-order sums);  ||G - I||_F^2 <= ns_tol2 -> T = I - (G - I)/2;  else
//          G = R^T R (pivot d > tol G_jj, else retry with the shift 11 (m w + w (w+1)) u tr(G)),
//          T = R^-1;  X <- X T.
//   order: pass 1; pass 2 if pass 1 factorised (or, single, if it shifted); two more passes if a
//          factorisation was shifted.  status[3] counts shifted retries, status[4] flags failure.
// The pieces are device functions of one CTA (all its threads call them) so that the cluster
// loop of small_loop.cuh runs the same arithmetic on a row-distributed panel.
constexpr int SCQR_MAX_W = 64;
constexpr int SCQR_MAX_ELEMS = 8192;
constexpr int SCQR_THREADS = 512;
constexpr int SCQR_GLD = SCQR_MAX_W + 1;
constexpr int SCQR_SMEM = (2 * SCQR_MAX_ELEMS + 2 * SCQR_MAX_W * SCQR_GLD) * 8;

// G (w x w, ld SCQR_GLD, symmetric) = P^T P for the column-major rows x w panel P (ld): one warp
// per entry i <= j, fixed-order warp sums.  Ends with __syncthreads.
__device__ __forceinline__ void scq_gram(const double* P, int ld, int rows, int w, double* G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  #pragma unroll 1
  for (int e = warp; e < w * w; e += nwarps) {
    const int i = e / w, j = e % w;
    if (i > j) continue;
    const double* xi = P + static_cast<int64_t>(i) * ld;
    const double* xj = P + static_cast<int64_t>(j) * ld;
    double s = 0.0;
    #pragma unroll 1
    for (int r = lane; r < rows; r += 32) s = fma(xi[r], xj[r], s);
    s = warp_sum(s);
    if (lane == 0) {
      G[i * SCQR_GLD + j] = s;
      G[j * SCQR_GLD + i] = s;
    }
  }
  __syncthreads();
}

// T (w x w, row-major, ld SCQR_GLD) from the full Gram G of an m_rows-row panel: the Newton-Schulz
// step when ||G - I||_F^2 <= ns_tol2, else R^-1 of G = R^T R with the shifted retry.  Updates the
// pass flags (factorised, shifted, fallback count); returns true on failure (both attempts broke
// down).  G is overwritten.  Uniform across the CTA; ends with __syncthreads.
__device__ bool scq_factor(double* G, double* T, int w, double m_rows, double ns_tol2, double tol, bool& f_fact,
                           bool& f_shift, int& fallbacks, double* kdiag = nullptr) {
  __shared__ double red[2][32];
  __shared__ double s_e2, s_shift;
  __shared__ int s_bad;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nthr = blockDim.x;
  double e2 = 0.0, tr = 0.0;
  #pragma unroll 1
  for (int e = t; e < w * w; e += nthr) {
    const int i = e / w, j = e % w;
    const double d = G[i * SCQR_GLD + j] - (i == j ? 1.0 : 0.0);
    e2 = fma(d, d, e2);
    if (i == j) tr += G[i * SCQR_GLD + j];
  }
  e2 = warp_sum(e2);
  tr = warp_sum(tr);
  if (lane == 0) {
    red[0][warp] = e2;
    red[1][warp] = tr;
  }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < (nthr >> 5); ++k) {
      a += red[0][k];
      b += red[1][k];
    }
    s_e2 = a;
    s_shift = 11.0 * (m_rows * w + static_cast<double>(w) * (w + 1)) * 0x1p-53 * b;
  }
  __syncthreads();
  if (ns_tol2 >= 0.0 && s_e2 <= ns_tol2) {  // Newton-Schulz step towards the polar factor
    #pragma unroll 1
    for (int e = t; e < w * w; e += nthr) {
      const int i = e / w, j = e % w;
      T[i * SCQR_GLD + j] = (i == j ? 1.0 : 0.0) - 0.5 * (G[i * SCQR_GLD + j] - (i == j ? 1.0 : 0.0));
    }
    __syncthreads();
    return false;
  }
  f_fact = true;
  // T keeps the Gram (pivot tolerance reference, and the retry's input)
  #pragma unroll 1
  for (int e = t; e < w * w; e += nthr) T[(e / w) * SCQR_GLD + e % w] = G[(e / w) * SCQR_GLD + e % w];
  __syncthreads();
  bool failed = false;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (attempt == 1) {
      #pragma unroll 1
      for (int e = t; e < w * w; e += nthr) {
        const int i = e / w, j = e % w;
        G[i * SCQR_GLD + j] = T[i * SCQR_GLD + j] + (i == j ? s_shift : 0.0);
      }
    }
    if (t == 0) s_bad = 0;
    __syncthreads();
    // right-looking Cholesky G = L L^T in place (lower triangle)
    for (int j = 0; j < w; ++j) {
      if (t == 0) {
        const double d = G[j * SCQR_GLD + j];
        if (!(d > tol * T[j * SCQR_GLD + j]) || !(d > 0.0)) s_bad = 1;
        G[j * SCQR_GLD + j] = sqrt(fmax(d, 0.0));
      }
      __syncthreads();
      if (s_bad) break;
      const double ljj = G[j * SCQR_GLD + j];
      for (int i = j + 1 + t; i < w; i += nthr) G[i * SCQR_GLD + j] /= ljj;
      __syncthreads();
      const int nt = w - j - 1;
      #pragma unroll 1
      for (int e = t; e < nt * nt; e += nthr) {
        const int i = j + 1 + e / nt, k = j + 1 + e % nt;
        if (k <= i) G[i * SCQR_GLD + k] = fma(-G[i * SCQR_GLD + j], G[k * SCQR_GLD + j], G[i * SCQR_GLD + k]);
      }
      __syncthreads();
    }
    const bool bad = s_bad != 0;
    __syncthreads();
    if (!bad) break;
    if (attempt == 0) {
      f_shift = true;
      ++fallbacks;
    } else {
      failed = true;
    }
  }
  if (failed) return true;
  if (kdiag != nullptr && t == 0) {  // max / min diagonal of R (the kappa-proxy of qb_stats)
    double dmax = 0.0, dmin = 1e300;
    for (int j = 0; j < w; ++j) {
      dmax = fmax(dmax, G[j * SCQR_GLD + j]);
      dmin = fmin(dmin, G[j * SCQR_GLD + j]);
    }
    kdiag[0] = dmax;
    kdiag[1] = dmin;
  }
  // T = R^-1 = L^-T: column c of L^-1 by forward substitution (thread c); T[c][i] = L^-1(i, c) = R^-1(c, i)
  for (int c = t; c < w; c += nthr) {
    #pragma unroll 1
    for (int i = 0; i < w; ++i) {
      if (i < c) {
        T[c * SCQR_GLD + i] = 0.0;
        continue;
      }
      double v = (i == c) ? 1.0 : 0.0;
      #pragma unroll 1
      for (int k = c; k < i; ++k) v = fma(-G[i * SCQR_GLD + k], T[c * SCQR_GLD + k], v);
      T[c * SCQR_GLD + i] = v / G[i * SCQR_GLD + i];
    }
  }
  __syncthreads();
  return false;
}

// P <- P T for the column-major rows x w panel P (ld), through the scratch X2 (ld rows).
__device__ __forceinline__ void scq_apply(double* P, int ld, int rows, int w, const double* T, double* X2) {
  const int t = threadIdx.x, nthr = blockDim.x;
  #pragma unroll 1
  for (int e = t; e < rows * w; e += nthr) {
    const int j = e / rows, r = e % rows;
    double s = 0.0;
    #pragma unroll 1
    for (int i = 0; i < w; ++i) s = fma(P[static_cast<int64_t>(i) * ld + r], T[i * SCQR_GLD + j], s);
    X2[e] = s;
  }
  __syncthreads();
  #pragma unroll 1
  for (int e = t; e < rows * w; e += nthr) P[static_cast<int64_t>(e / rows) * ld + e % rows] = X2[e];
  __syncthreads();
}

__global__ void __launch_bounds__(SCQR_THREADS) small_cholqr_kernel(const double* __restrict__ src, int64_t lds,
                                                                    double* __restrict__ dst, int64_t ldd, int m,
                                                                    int w, int single, double ns_tol2, double tol,
                                                                    int* __restrict__ status,
                                                                    float* __restrict__ dst32, int64_t ldd32,
                                                                    double* __restrict__ kappa) {
  extern __shared__ double scq[];
  double* X = scq;                         // [w][m] column-major (ld m)
  double* X2 = X + SCQR_MAX_ELEMS;         // product buffer
  double* G = X2 + SCQR_MAX_ELEMS;         // [w][GLD] Gram / Cholesky factor L (lower)
  double* T = G + SCQR_MAX_W * SCQR_GLD;   // [w][GLD] T (row-major)
  const int t = threadIdx.x;
  for (int idx = t; idx < m * w; idx += SCQR_THREADS) X[idx] = src[(idx / m) * lds + idx % m];
  __syncthreads();
  bool f_fact = false, f_shift = false, f_fail = false;
  int fallbacks = 0;
  __shared__ double kd[2];
  __shared__ int krec;
  if (t == 0) krec = (kappa != nullptr && atomicCAS(status + 5, 0, 1) == 0) ? 1 : 0;
  __syncthreads();
  bool kdone = krec == 0;
  auto pass = [&]() {
    scq_gram(X, m, m, w, G);
    const bool was_fact = f_fact;
    f_fail = scq_factor(G, T, w, static_cast<double>(m), ns_tol2, tol, f_fact, f_shift, fallbacks,
                        kdone ? nullptr : kd);
    if (!kdone && !was_fact && f_fact && !f_fail) {  // the first factorization of the block
      kdone = true;
      if (t == 0) {
        kappa[0] = kd[0];
        kappa[1] = kd[1];
      }
    }
    if (!f_fail) scq_apply(X, m, m, w, T, X2);
  };
  pass();
  if (!f_fail && (single ? f_shift : f_fact)) pass();
  if (!f_fail && f_shift) {
    pass();
    if (!f_fail) pass();
  }
  if (t == 0) {
    if (fallbacks) atomicAdd(status + 3, fallbacks);
    if (f_fail) status[4] = 1;
  }
  for (int idx = t; idx < m * w; idx += SCQR_THREADS) {
    const int j = idx / m, r = idx % m;
    dst[j * ldd + r] = X[idx];
    if (dst32 != nullptr) dst32[j * ldd32 + r] = static_cast<float>(X[idx]);
  }
}

}  // namespace qbk


namespace qbk {

// R(r, c) += W(r, c) for r < rows, c < cols: R column-major (ld ldr), W row-major (ld ldw) — the
// block Gram-Schmidt coefficients of one projection pass added into R's block column.
__global__ void __launch_bounds__(256) add_rowmajor_kernel(double* __restrict__ R, int64_t ldr,
                                                           const double* __restrict__ W, int64_t ldw, int64_t rows,
                                                           int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * 256ll + threadIdx.x; idx < total; idx += static_cast<int64_t>(gridDim.x) * 256) {
    const int64_t c = idx / rows, r = idx - c * rows;
    R[r + c * ldr] += W[r * ldw + c];
  }
}

}  // namespace qbk
