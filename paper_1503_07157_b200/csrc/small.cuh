// Small and bandwidth-bound kernels of the QB path:
//   sumsq_kernel       a0: partial sums of squares of A (||A||_F^2)
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
// sum of squares of the result.
__global__ void __launch_bounds__(RED_THREADS) splitk_reduce_kernel(const double* __restrict__ P, int S, int64_t stride,
                                                                    int64_t rows, int64_t cols, int64_t ldp,
                                                                    double* __restrict__ out, int64_t ldo,
                                                                    double* __restrict__ sq_partials,
                                                                    const int* __restrict__ gate, int subtract) {
  if (gate != nullptr && __ldcg(gate) == 0) return;
  __shared__ double red[RED_THREADS / 32];
  double sq = 0.0;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(RED_THREADS) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * RED_THREADS) {
    const int64_t r = idx / cols, c = idx - r * cols;
    const double* src = P + r * ldp + c;
    double v = 0.0;
    for (int s = 0; s < S; ++s) v += src[s * stride];
    if (subtract) v = out[r * ldo + c] - v;  // C -= sum of the split products
    out[r * ldo + c] = v;
    sq = fma(v, v, sq);
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
                                                      int64_t cols, Tout* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    out[r + c * ldo] = static_cast<Tout>(in[r + c * ldi]);
  }
}

// dst = src (column-major rows x cols) unless *gate != 0 (CholeskyQR: a first pass that took the
// Newton-Schulz step is final; its result moves from the scratch to the destination).
__global__ void __launch_bounds__(256) gated_copy_kernel(const double* __restrict__ src, int64_t lds,
                                                         double* __restrict__ dst, int64_t ldd, int64_t rows,
                                                         int64_t cols, const int* __restrict__ gate) {
  if (__ldcg(gate) != 0) return;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    dst[r + c * ldd] = src[r + c * lds];
  }
}

// ---------------------------------------------------------------------------------------
// K4 core — chol_cluster_kernel: the CholeskyQR "T" of a w x w Gram matrix G = X^T X
// (column-major), w <= 256, on ONE thread-block cluster of 8 CTAs (one 32-column panel of the
// factor per CTA, kept in that CTA's shared memory; peers read it through distributed shared
// memory).  Writes T column-major into `Tout` (ld ldt) such that X T has orthonormal columns:
//   * Newton-Schulz: if ||G - I||_F <= sqrt(ns_tol2), X is orthonormal to first order and
//     T = I - (G - I)/2 (one step towards the polar factor, error (3/4)||G - I||^2).  status 3.
//   * Cholesky: right-looking over the 32-column panels.  Step p: CTA p factors its 32 x 32
//     diagonal block (warp 0), inverts it, and solves its panel below; the CTAs that own later
//     panels copy the rows they need of panel p over DSMEM and apply the rank-32 update.  Then
//     CTA J forms block column J of L^-1 by blocked forward substitution
//     (X_JJ = L_JJ^-1, X_IJ = -L_II^-1 sum_{K=J}^{I-1} L_IK X_KJ), reading L_IK and L_II^-1 from
//     their owners, and writes it: Tout(row, col) = L^-1(row, col), i.e. read ROW-major Tout is
//     R^-1 = L^-T (upper triangular).  A pivot that is not > tol * G_jj (or NaN) is a breakdown
//     (reading R8): the cluster restarts once with the shifted-CholeskyQR shift
//     s = 11 (m w + w (w+1)) u trace(G).  status[0] = 0 ok / 1 shifted / 2 failed.
// Flags: status[1] = 1 when the shift was used (gates the extra CholeskyQR3 passes),
// status[2] = 1 when the Cholesky path ran (gates CholeskyQR's second pass; a Newton-Schulz
// first pass needs none), status[3] += 1 per shifted factorization, status[4] = 1 on failure.
// `gate` (may be null): the kernel does nothing unless *gate != 0.
constexpr int CHOL_MAXW = 256;
constexpr int CHOL_NB = 32;
constexpr int CHOL_CTAS = 8;
constexpr int CHOL_THREADS = 256;
constexpr int CHOL_PLD = CHOL_NB + 1;
constexpr int CHOL_SMEM = (2 * CHOL_MAXW * CHOL_PLD + 3 * CHOL_NB * CHOL_PLD) * 8;
constexpr int CHOL_ST_NS = 3;

__global__ void __cluster_dims__(CHOL_CTAS, 1, 1) __launch_bounds__(CHOL_THREADS)
    chol_cluster_kernel(const double* __restrict__ G, int64_t ldg, int w, int64_t m_rows, double* __restrict__ Tout,
                        int64_t ldt, int* __restrict__ status, double tol, double ns_tol2,
                        const int* __restrict__ gate) {
  if (gate != nullptr && __ldcg(gate) == 0) return;  // same value in every CTA of the cluster
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int PLD = CHOL_PLD;
  extern __shared__ double sm[];
  double* P = sm;                      // [256][PLD] own panel: rows 32*cta.., columns 32*cta..+31
  double* R = P + CHOL_MAXW * PLD;     // [256][PLD] staged rows of a peer panel; later X = L^-1 block column
  double* Dl = R + CHOL_MAXW * PLD;    // [32][PLD] diagonal block L11 (identity-padded) / staging
  double* Di = Dl + CHOL_NB * PLD;     // [32][PLD] L11^-1 (identity-padded), read by peers
  double* Tb = Di + CHOL_NB * PLD;     // [32][PLD] scratch
  __shared__ double red[CHOL_THREADS / 32];
  __shared__ double s_part, s_tot, s_shift;
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = static_cast<int>(cluster.block_rank());
  const int nbk = (w + CHOL_NB - 1) / CHOL_NB;
  const bool active = cta < nbk;
  const int p0 = cta * CHOL_NB;
  const int rows = active ? w - p0 : 0, nb = active ? min(CHOL_NB, w - p0) : 0;

  // ---- Newton-Schulz test: ||G - I||_F^2 over the own column block, summed in rank order
  double e2 = 0.0;
  for (int idx = tid; idx < w * nb; idx += CHOL_THREADS) {
    const int i = idx % w, j = p0 + idx / w;
    const double d = __ldcg(G + i + static_cast<int64_t>(j) * ldg) - (i == j ? 1.0 : 0.0);
    e2 = fma(d, d, e2);
  }
  e2 = warp_sum(e2);
  if (lane == 0) red[warp] = e2;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < CHOL_THREADS / 32; ++k) t += red[k];
    s_part = t;
    double tr = 0.0;
    for (int j = 0; j < w; ++j) tr += __ldcg(G + j + static_cast<int64_t>(j) * ldg);
    s_shift = 11.0 * (static_cast<double>(m_rows) * w + static_cast<double>(w) * (w + 1)) * 0x1p-53 * tr;
  }
  cluster.sync();
  if (tid == 0) {
    double t = 0.0;
    for (int r = 0; r < CHOL_CTAS; ++r) t += *cluster.map_shared_rank(&s_part, r);
    s_tot = t;
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

  int attempt = 0;
  bool failed = false;
  for (; attempt < 2; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : s_shift;
    for (int idx = tid; idx < rows * nb; idx += CHOL_THREADS) {
      const int i = idx % rows, j = idx / rows;
      double v = __ldcg(G + (p0 + i) + static_cast<int64_t>(p0 + j) * ldg);
      if (i == j) v += shift;
      P[i * PLD + j] = v;
    }
    if (tid == 0) s_fail = 0;
    cluster.sync();  // panels loaded; no peer still reads the previous attempt's panels
    failed = false;
    for (int p = 0; p < nbk; ++p) {
      if (cta == p) {
        // unblocked Cholesky of the nb x nb diagonal block (warp 0, lane = row)
        if (warp == 0) {
          int bad = 0;
          for (int jj = 0; jj < nb; ++jj) {
            const double d = P[jj * PLD + jj];
            const double g0 = __ldcg(G + (p0 + jj) + static_cast<int64_t>(p0 + jj) * ldg);
            if (!(d > tol * g0) || !(d > 0.0)) {
              bad = 1;
              break;
            }
            const double r = sqrt(d);
            __syncwarp();
            if (lane == jj) P[jj * PLD + jj] = r;
            if (lane > jj && lane < nb) P[lane * PLD + jj] /= r;
            __syncwarp();
            if (lane > jj && lane < nb) {
              const double lij = P[lane * PLD + jj];
              for (int c = jj + 1; c <= lane; ++c) P[lane * PLD + c] -= lij * P[c * PLD + jj];
            }
            __syncwarp();
          }
          if (lane == 0) s_fail = bad;
          if (!bad) {  // L11 -> Dl (identity-padded), L11^-1 -> Di by forward substitution, lane = column
            for (int r = 0; r < CHOL_NB; ++r)
              Dl[r * PLD + lane] =
                  (r < nb && lane < nb && lane <= r) ? P[r * PLD + lane] : (r == lane ? 1.0 : 0.0);
            __syncwarp();
            for (int r = 0; r < CHOL_NB; ++r) {
              double v = (r == lane) ? 1.0 : 0.0;
              for (int k = lane; k < r; ++k) v -= Dl[r * PLD + k] * Di[k * PLD + lane];
              Di[r * PLD + lane] = (r >= lane) ? v / Dl[r * PLD + r] : 0.0;
              __syncwarp();
            }
          }
        }
        __syncthreads();
        if (!s_fail) {  // panel below the diagonal block: L21 = P21 L11^-T
          const int c = lane;
          for (int i = nb + warp; i < rows; i += CHOL_THREADS / 32) {
            double v = 0.0;
            if (c < nb)
              for (int k = 0; k <= c; ++k) v = fma(P[i * PLD + k], Di[c * PLD + k], v);
            __syncwarp();
            if (c < nb) P[i * PLD + c] = v;
          }
        }
      }
      cluster.sync();
      if (*cluster.map_shared_rank(&s_fail, p)) {
        failed = true;
        break;
      }
      if (active && cta > p) {  // rank-32 update of the own panel with panel p's rows p0.. (over DSMEM)
        const double* Pp = cluster.map_shared_rank(P, p);
        const int off = p0 - p * CHOL_NB;
        for (int idx = tid; idx < rows * CHOL_NB; idx += CHOL_THREADS) {
          const int i = idx / CHOL_NB, k = idx % CHOL_NB;
          R[i * PLD + k] = Pp[(off + i) * PLD + k];
        }
        __syncthreads();
        const int c = lane;
        for (int i = warp; i < rows; i += CHOL_THREADS / 32) {
          if (c < nb) {
            double acc = 0.0;
#pragma unroll 8
            for (int k = 0; k < CHOL_NB; ++k) acc = fma(R[i * PLD + k], R[c * PLD + k], acc);
            P[i * PLD + c] -= acc;
          }
        }
      }
      cluster.sync();
    }
    if (!failed) break;
  }
  if (cta == 0 && tid == 0) {
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

  // ---- block column J = cta of L^-1 (X in R, rows 32J..w-1)
  if (active) {
    double* X = R;
    for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += CHOL_THREADS)
      X[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = Di[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)];
    const int r = tid >> 3, c0 = (tid & 7) * 4;  // thread owns T(r, c0..c0+3)
    for (int I = cta + 1; I < nbk; ++I) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
      for (int K = cta; K < I; ++K) {
        const double* PK = cluster.map_shared_rank(P, K);  // L_IK = rows 32(I-K).. of panel K
        __syncthreads();
        for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += CHOL_THREADS) {
          const int rr = idx / CHOL_NB, kk = idx % CHOL_NB;
          Dl[rr * PLD + kk] = (I * CHOL_NB + rr < w) ? PK[((I - K) * CHOL_NB + rr) * PLD + kk] : 0.0;
        }
        __syncthreads();
        const double* xb = X + (K - cta) * CHOL_NB * PLD;
#pragma unroll 4
        for (int kk = 0; kk < CHOL_NB; ++kk) {
          const double l = Dl[r * PLD + kk];
          const double* x = xb + kk * PLD + c0;
          t0 = fma(l, x[0], t0);
          t1 = fma(l, x[1], t1);
          t2 = fma(l, x[2], t2);
          t3 = fma(l, x[3], t3);
        }
      }
      const double* DI = cluster.map_shared_rank(Di, I);
      __syncthreads();
      Tb[r * PLD + c0] = t0;
      Tb[r * PLD + c0 + 1] = t1;
      Tb[r * PLD + c0 + 2] = t2;
      Tb[r * PLD + c0 + 3] = t3;
      for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += CHOL_THREADS)
        Dl[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = DI[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)];
      __syncthreads();
      double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
      for (int t = 0; t <= r; ++t) {
        const double d = Dl[r * PLD + t];
        v0 = fma(d, Tb[t * PLD + c0], v0);
        v1 = fma(d, Tb[t * PLD + c0 + 1], v1);
        v2 = fma(d, Tb[t * PLD + c0 + 2], v2);
        v3 = fma(d, Tb[t * PLD + c0 + 3], v3);
      }
      double* xo = X + ((I - cta) * CHOL_NB + r) * PLD + c0;
      xo[0] = -v0;
      xo[1] = -v1;
      xo[2] = -v2;
      xo[3] = -v3;
    }
    __syncthreads();
    for (int idx = tid; idx < w * nb; idx += CHOL_THREADS) {
      const int row = idx % w, c = idx / w;
      Tout[row + static_cast<int64_t>(p0 + c) * ldt] = row >= p0 ? X[(row - p0) * PLD + c] : 0.0;
    }
  }
  cluster.sync();  // keep this CTA's shared memory alive while peers read it
}

}  // namespace qbk
