// Small and bandwidth-bound kernels of the QB path:
//   sumsq_kernel       a0: partial sums of squares of A (||A||_F^2)
//   reduce_kernel      K8: fixed-order sum of per-CTA partials -> one FP64 scalar
//   splitk_reduce      fixed-order sum of split-K partials (+ sum of squares, the EI term)
//   transpose_kernel   column-major <-> row-major copy of a tall-skinny panel
//   chol_inv_kernel    K4 core: R^-1 of the Cholesky factor of a w x w Gram matrix,
//                      with the shifted-CholeskyQR fallback (reading R8)
// All reductions run in a fixed order, so results are bitwise reproducible.
#pragma once
#include "common.cuh"

namespace qbk {

constexpr int RED_THREADS = 256;

// Per-block sum of squares of a column-major m x n matrix (ld), grid-stride over columns.
__global__ void __launch_bounds__(RED_THREADS) sumsq_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                                            int64_t lda, double* __restrict__ partials) {
  __shared__ double red[RED_THREADS / 32];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const double* col = A + j * lda;
    for (int64_t i = threadIdx.x; i < m; i += RED_THREADS) s = fma(col[i], col[i], s);
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
// where "r" is the strided index).  Optional per-block sum of squares of the result.
__global__ void __launch_bounds__(RED_THREADS) splitk_reduce_kernel(const double* __restrict__ P, int S, int64_t stride,
                                                                    int64_t rows, int64_t cols, int64_t ldp,
                                                                    double* __restrict__ out, int64_t ldo,
                                                                    double* __restrict__ sq_partials) {
  __shared__ double red[RED_THREADS / 32];
  double sq = 0.0;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(RED_THREADS) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * RED_THREADS) {
    const int64_t r = idx / cols, c = idx - r * cols;
    const double* src = P + r * ldp + c;
    double v = 0.0;
    for (int s = 0; s < S; ++s) v += src[s * stride];
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
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows,
                                                        int64_t cols, double* __restrict__ out, int64_t ldo) {
  __shared__ double t[32][33];
  const int64_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = r0 + threadIdx.x, c = c0 + j;
    if (r < rows && c < cols) t[j][threadIdx.x] = in[r + c * ldi];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < rows && c < cols) out[r * ldo + c] = t[threadIdx.x][j];
  }
}

// ---------------------------------------------------------------------------------------
// chol_inv_kernel: one CTA, w <= CHOL_MAXW.
//   G (w x w, column-major, symmetric positive semi-definite Gram matrix X^T X)
//   -> L with L L^T = G + shift I (lower, column-major scratch `L`, ld ldl)
//   -> Rinv = L^-T written ROW-major (Rinv[i*ldr + j] = (L^-1)(j, i)), upper triangular,
//      so that Q = X Rinv is the CholeskyQR orthonormal factor.
// Attempt 0 uses shift 0.  A pivot that is not > tol * G_jj (or NaN) is a breakdown
// (reading R8); the kernel then restarts once with the shifted-CholeskyQR shift
// s = 11 (m w + w (w + 1)) u trace(G) (trace(G) = ||X||_F^2 >= ||X||_2^2) and reports it.
// status[0] = 0 ok / 1 shifted / 2 failed even with the shift.
constexpr int CHOL_MAXW = 256;
constexpr int CHOL_NB = 32;
constexpr int CHOL_THREADS = 512;
constexpr int CHOL_SMEM = (CHOL_MAXW * (CHOL_NB + 1) + CHOL_NB * (CHOL_MAXW + 1) + CHOL_MAXW) * 8 + 64;

__global__ void __launch_bounds__(CHOL_THREADS) chol_inv_kernel(const double* __restrict__ G, int64_t ldg, int w,
                                                                int64_t m_rows, double* __restrict__ L,
                                                                int64_t ldl, double* __restrict__ Rinv,
                                                                int64_t ldr, int* __restrict__ status,
                                                                double tol) {
  extern __shared__ double sm[];
  double* P = sm;                                   // [CHOL_MAXW][CHOL_NB + 1]
  double* LR = P + CHOL_MAXW * (CHOL_NB + 1);       // [CHOL_NB][CHOL_MAXW + 1]
  double* dg = LR + CHOL_NB * (CHOL_MAXW + 1);      // original diagonal of G
  __shared__ int s_fail;
  __shared__ double s_shift;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int PLD = CHOL_NB + 1, LRLD = CHOL_MAXW + 1;

  for (int j = tid; j < w; j += CHOL_THREADS) dg[j] = G[j + j * ldg];
  __syncthreads();
  if (tid == 0) {
    double tr = 0.0;
    for (int j = 0; j < w; ++j) tr += dg[j];
    const double u = 0x1p-53;
    s_shift = 11.0 * (static_cast<double>(m_rows) * w + static_cast<double>(w) * (w + 1)) * u * tr;
  }

  int attempt = 0;
  for (; attempt < 2; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : s_shift;
    if (tid == 0) s_fail = 0;
    __syncthreads();
    for (int p = 0; p < w; p += CHOL_NB) {
      const int nb = min(CHOL_NB, w - p), rows = w - p;
      // stage L(p + j, 0:p) and the panel G(p:w, p:p+nb)
      for (int idx = tid; idx < nb * p; idx += CHOL_THREADS) {
        const int j = idx % nb, k = idx / nb;
        LR[j * LRLD + k] = L[(p + j) + static_cast<int64_t>(k) * ldl];
      }
      for (int idx = tid; idx < rows * nb; idx += CHOL_THREADS) {
        const int i = idx % rows, j = idx / rows;
        double v = G[(p + i) + static_cast<int64_t>(p + j) * ldg];
        if (i == j) v += shift;
        P[i * PLD + j] = v;
      }
      __syncthreads();
      // left-looking update: P(i, j) -= sum_{k<p} L(p+i, k) L(p+j, k)
      if (p > 0) {
        const int half = tid >> 8, i = tid & 255;
        if (i < rows) {
          double acc[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) acc[jj] = 0.0;
          for (int k = 0; k < p; ++k) {
            const double l = L[(p + i) + static_cast<int64_t>(k) * ldl];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) acc[jj] = fma(l, LR[(half * 16 + jj) * LRLD + k], acc[jj]);
          }
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (half * 16 + jj < nb) P[i * PLD + half * 16 + jj] -= acc[jj];
        }
      }
      __syncthreads();
      // unblocked Cholesky of the nb x nb diagonal block (warp 0, lane = row)
      if (warp == 0) {
        for (int j = 0; j < nb; ++j) {
          const double d = P[j * PLD + j];
          const bool bad = !(d > tol * dg[p + j]) || !(d > 0.0);
          if (bad) {
            if (lane == 0) s_fail = 1;
            break;
          }
          const double r = sqrt(d);
          __syncwarp();
          if (lane == j) P[j * PLD + j] = r;
          if (lane > j && lane < nb) P[lane * PLD + j] /= r;
          __syncwarp();
          if (lane > j && lane < nb) {
            const double lij = P[lane * PLD + j];
            for (int c = j + 1; c <= lane; ++c) P[lane * PLD + c] -= lij * P[c * PLD + j];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (s_fail) break;
      // panel below the diagonal block: x L11^T = P(i, :), forward substitution per row
      for (int i = nb + tid; i < rows; i += CHOL_THREADS) {
        for (int j = 0; j < nb; ++j) {
          double v = P[i * PLD + j];
          for (int c = 0; c < j; ++c) v -= P[i * PLD + c] * P[j * PLD + c];
          P[i * PLD + j] = v / P[j * PLD + j];
        }
      }
      __syncthreads();
      for (int idx = tid; idx < rows * nb; idx += CHOL_THREADS) {
        const int i = idx % rows, j = idx / rows;
        if (i >= j) L[(p + i) + static_cast<int64_t>(p + j) * ldl] = P[i * PLD + j];
      }
      __syncthreads();
    }
    if (!s_fail) break;
  }
  if (attempt == 2) {
    if (tid == 0) status[0] = 2;
    return;
  }
  if (tid == 0) status[0] = attempt;
  __syncthreads();

  // ---- Linv = L^-1 (lower), stored column-major in Rinv (=> Rinv row-major = L^-T).
  // zero the strictly upper part
  for (int64_t idx = tid; idx < static_cast<int64_t>(w) * w; idx += CHOL_THREADS) {
    const int r = static_cast<int>(idx % w), c = static_cast<int>(idx / w);
    if (r < c) Rinv[r + static_cast<int64_t>(c) * ldr] = 0.0;
  }
  const int nbk = (w + CHOL_NB - 1) / CHOL_NB;
  // (a) diagonal blocks: warp jb inverts L_jb,jb by forward substitution, lane = column
  for (int jb = warp; jb < nbk; jb += CHOL_THREADS / 32) {
    const int o = jb * CHOL_NB, bs = min(CHOL_NB, w - o);
    double* X = P + jb * CHOL_NB * PLD;  // bs x bs scratch rows (fits: nbk*32 <= CHOL_MAXW rows)
    if (lane < bs) {
      for (int r = 0; r < bs; ++r) {
        double v = (r == lane) ? 1.0 : 0.0;
        if (r > lane) {
          for (int k = lane; k < r; ++k) v -= L[(o + r) + static_cast<int64_t>(o + k) * ldl] * X[k * PLD + lane];
        } else if (r < lane) {
          v = 0.0;
        }
        X[r * PLD + lane] = (r >= lane) ? v / L[(o + r) + static_cast<int64_t>(o + r) * ldl] : 0.0;
      }
      for (int r = 0; r < bs; ++r) Rinv[(o + r) + static_cast<int64_t>(o + lane) * ldr] = X[r * PLD + lane];
    }
  }
  __syncthreads();
  // (b) block rows I = 1..nbk-1: X_IJ = -X_II * sum_{K=J}^{I-1} L_IK X_KJ  for J < I
  double* T = LR;  // [I*CHOL_NB][CHOL_NB+1] scratch (I*32 <= CHOL_MAXW - 32 rows)
  for (int I = 1; I < nbk; ++I) {
    const int oI = I * CHOL_NB, bsI = min(CHOL_NB, w - oI);
    const int nel = I * CHOL_NB * CHOL_NB;
    for (int idx = tid; idx < nel; idx += CHOL_THREADS) {
      const int J = idx / (CHOL_NB * CHOL_NB), rem = idx % (CHOL_NB * CHOL_NB);
      const int r = rem / CHOL_NB, c = rem % CHOL_NB;
      double v = 0.0;
      if (r < bsI) {
        const int col = J * CHOL_NB + c;
        for (int k = J * CHOL_NB + c; k < oI; ++k)  // X(k, col) = 0 for k < col
          v += L[(oI + r) + static_cast<int64_t>(k) * ldl] * Rinv[k + static_cast<int64_t>(col) * ldr];
      }
      T[(J * CHOL_NB + r) * PLD + c] = v;
    }
    __syncthreads();
    for (int idx = tid; idx < nel; idx += CHOL_THREADS) {
      const int J = idx / (CHOL_NB * CHOL_NB), rem = idx % (CHOL_NB * CHOL_NB);
      const int r = rem / CHOL_NB, c = rem % CHOL_NB;
      if (r < bsI) {
        double v = 0.0;
        for (int t = 0; t <= r; ++t)
          v += Rinv[(oI + r) + static_cast<int64_t>(oI + t) * ldr] * T[(J * CHOL_NB + t) * PLD + c];
        Rinv[(oI + r) + static_cast<int64_t>(J * CHOL_NB + c) * ldr] = -v;
      }
    }
    __syncthreads();
  }
}

}  // namespace qbk
