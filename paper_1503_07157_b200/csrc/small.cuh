// Small and bandwidth-bound kernels of the QB path:
//   sumsq_kernel       a0: partial sums of squares of A (||A||_F^2)
//   reduce_kernel      K8: fixed-order sum of per-CTA partials -> one FP64 scalar
//   splitk_reduce      fixed-order sum of split-K partials (+ sum of squares, the EI term)
//   transpose_kernel   column-major <-> row-major copy of a tall-skinny panel
//   chol_kernel        K4 core: Cholesky factor of a w x w Gram matrix (one CTA) with the
//                      shifted-CholeskyQR fallback (reading R8)
//   trinv_kernel       K4 core: R^-1 = L^-T by blocked forward substitution (w/32 CTAs)
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
                                                                    double* __restrict__ sq_partials,
                                                                    const int* __restrict__ gate) {
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

// ---------------------------------------------------------------------------------------
// K4 core, step 1 — chol_kernel: one CTA, w <= CHOL_MAXW.  Given the w x w Gram matrix
// G = X^T X (column-major), produce T (row-major, in `Rinv`) such that X T is orthonormal:
//   * Newton-Schulz path: if ||G - I||_F <= ns_tol, X is already orthonormal to first order
//     and T = I - (G - I)/2 (one Newton-Schulz step towards the polar factor; the error is
//     (3/4)||G - I||^2, below u for ns_tol = 1e-8).  No factorization.   status[0] = 3.
//   * Cholesky path: L L^T = G (+ shift), written column-major to `L` with the inverses of its
//     32 x 32 diagonal blocks in `Dinv` (block J at Dinv + J*32*32, row-major); trinv_kernel
//     then writes T = R^-1 = L^-T.  Left-looking by 32-column panels, operands staged in
//     shared memory.  A pivot that is not > tol * G_jj (or NaN) is a breakdown (reading R8):
//     the kernel restarts once with the shifted-CholeskyQR shift s = 11 (m w + w (w+1)) u
//     trace(G) (trace(G) = ||X||_F^2 >= ||X||_2^2).  status[0] = 0 ok / 1 shifted / 2 failed.
// Block-level flags: status[1] = 1 when the shift was used (gates the extra CholeskyQR3
// passes), status[2] += 1 per shifted factorization, status[3] = 1 on failure.
// `gate` (may be null): the kernel does nothing unless *gate != 0.
constexpr int CHOL_MAXW = 256;
constexpr int CHOL_NB = 32;
constexpr int CHOL_THREADS = 512;
constexpr int CHOL_PLD = CHOL_NB + 1;
constexpr int CHOL_SMEM = (2 * CHOL_MAXW * CHOL_PLD + 2 * CHOL_NB * CHOL_PLD + CHOL_MAXW) * 8;
constexpr int CHOL_ST_NS = 3;

__global__ void __launch_bounds__(CHOL_THREADS) chol_kernel(const double* __restrict__ G, int64_t ldg, int w,
                                                            int64_t m_rows, double* __restrict__ L, int64_t ldl,
                                                            double* __restrict__ Dinv, double* __restrict__ Rinv,
                                                            int64_t ldr, int* __restrict__ status, double tol,
                                                            double ns_tol2, const int* __restrict__ gate) {
  if (gate != nullptr && __ldcg(gate) == 0) return;
  extern __shared__ double sm[];
  double* P = sm;                          // [CHOL_MAXW][PLD] current panel (rows p..w-1)
  double* Lc = P + CHOL_MAXW * CHOL_PLD;   // [CHOL_MAXW][PLD] staged L(p.., kc..kc+32)
  double* Dl = Lc + CHOL_MAXW * CHOL_PLD;  // [32][PLD] L11 of the panel
  double* Di = Dl + CHOL_NB * CHOL_PLD;    // [32][PLD] L11^-1
  double* dg = Di + CHOL_NB * CHOL_PLD;    // original diagonal of G
  constexpr int PLD = CHOL_PLD;
  __shared__ int s_fail;
  __shared__ double s_shift, s_e2;
  __shared__ double red[CHOL_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- Newton-Schulz test: e2 = ||G - I||_F^2 (fixed-order reduction)
  if (ns_tol2 >= 0.0) {
    double e2 = 0.0;
    for (int idx = tid; idx < w * w; idx += CHOL_THREADS) {
      const int i = idx % w, j = idx / w;
      const double d = __ldcg(G + i + static_cast<int64_t>(j) * ldg) - (i == j ? 1.0 : 0.0);
      e2 = fma(d, d, e2);
    }
    e2 = warp_sum(e2);
    if (lane == 0) red[warp] = e2;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int k = 0; k < CHOL_THREADS / 32; ++k) t += red[k];
      s_e2 = t;
    }
    __syncthreads();
    if (s_e2 <= ns_tol2) {
      for (int idx = tid; idx < w * w; idx += CHOL_THREADS) {
        const int i = idx / w, j = idx % w;
        const double d = __ldcg(G + i + static_cast<int64_t>(j) * ldg) - (i == j ? 1.0 : 0.0);
        Rinv[static_cast<int64_t>(i) * ldr + j] = (i == j ? 1.0 : 0.0) - 0.5 * d;
      }
      if (tid == 0) status[0] = CHOL_ST_NS;
      return;
    }
  }

  for (int j = tid; j < w; j += CHOL_THREADS) dg[j] = __ldcg(G + j + j * ldg);
  __syncthreads();
  if (tid == 0) {
    double tr = 0.0;
    for (int j = 0; j < w; ++j) tr += dg[j];
    s_shift = 11.0 * (static_cast<double>(m_rows) * w + static_cast<double>(w) * (w + 1)) * 0x1p-53 * tr;
  }
  int attempt = 0;
  for (; attempt < 2; ++attempt) {
    const double shift = attempt == 0 ? 0.0 : s_shift;
    if (tid == 0) s_fail = 0;
    __syncthreads();
    for (int p = 0; p < w; p += CHOL_NB) {
      const int nb = min(CHOL_NB, w - p), rows = w - p;
      for (int idx = tid; idx < rows * nb; idx += CHOL_THREADS) {
        const int i = idx % rows, j = idx / rows;
        double v = __ldcg(G + (p + i) + static_cast<int64_t>(p + j) * ldg);
        if (i == j) v += shift;
        P[i * PLD + j] = v;
      }
      // left-looking update P -= L(p:w, 0:p) L(p:p+nb, 0:p)^T, 32 columns of L at a time
      const int j = lane, i0 = warp;  // thread owns P(i0 + 16 r, j), r < 16
      double acc[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) acc[r] = 0.0;
      for (int kc = 0; kc < p; kc += CHOL_NB) {
        __syncthreads();
        for (int idx = tid; idx < rows * CHOL_NB; idx += CHOL_THREADS) {
          const int i = idx % rows, kk = idx / rows;
          Lc[i * PLD + kk] = __ldcg(L + (p + i) + static_cast<int64_t>(kc + kk) * ldl);
        }
        __syncthreads();
        if (j < nb) {
#pragma unroll 4
          for (int kk = 0; kk < CHOL_NB; ++kk) {
            const double lj = Lc[j * PLD + kk];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
              const int i = i0 + 16 * r;
              if (i < rows) acc[r] = fma(Lc[i * PLD + kk], lj, acc[r]);
            }
          }
        }
      }
      __syncthreads();
      if (j < nb) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int i = i0 + 16 * r;
          if (i < rows) P[i * PLD + j] -= acc[r];
        }
      }
      __syncthreads();
      // unblocked Cholesky of the nb x nb diagonal block (warp 0, lane = row)
      if (warp == 0) {
        for (int jj = 0; jj < nb; ++jj) {
          const double d = P[jj * PLD + jj];
          if (!(d > tol * dg[p + jj]) || !(d > 0.0)) {
            if (lane == 0) s_fail = 1;
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
        // L11 (lower) -> Dl, zero above; L11^-1 by forward substitution, lane = column
        if (!s_fail) {
          for (int r = 0; r < CHOL_NB; ++r) Dl[r * PLD + lane] = (r < nb && lane < nb && lane <= r) ? P[r * PLD + lane] : (r == lane ? 1.0 : 0.0);
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
      if (s_fail) break;
      // panel below the diagonal block: L21 = P21 L11^-T, L21(i, j) = sum_{c<=j} P(i, c) Di(j, c)
      {
        double out[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int i = nb + i0 + 16 * r;
          double v = 0.0;
          if (i < rows && j < nb)
            for (int c = 0; c <= j; ++c) v = fma(P[i * PLD + c], Di[j * PLD + c], v);
          out[r] = v;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int i = nb + i0 + 16 * r;
          if (i < rows && j < nb) P[i * PLD + j] = out[r];
        }
      }
      __syncthreads();
      for (int idx = tid; idx < rows * nb; idx += CHOL_THREADS) {
        const int i = idx % rows, jj = idx / rows;
        L[(p + i) + static_cast<int64_t>(p + jj) * ldl] = (i >= jj) ? P[i * PLD + jj] : 0.0;
      }
      for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += CHOL_THREADS)
        Dinv[(p / CHOL_NB) * CHOL_NB * CHOL_NB + idx] = Di[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)];
      __syncthreads();
    }
    if (!s_fail) break;
  }
  if (tid == 0) {
    status[0] = attempt;  // 0, 1, or 2 (= failed twice)
    if (attempt == 1) {
      status[1] = 1;
      atomicAdd(status + 2, 1);
    }
    if (attempt >= 2) status[3] = 1;
  }
}

// K4 core, step 2 — trinv_kernel: grid = ceil(w/32) CTAs, CTA J computes block column J of
// L^-1 (rows >= 32J) by blocked forward substitution
//   X_JJ = Dinv_J,  X_IJ = -Dinv_I sum_{K=J}^{I-1} L_IK X_KJ  (I > J)
// and writes it column-major into Rinv (ld ldr), zero above the diagonal, so that Rinv read
// ROW-major is R^-1 = L^-T, upper triangular: Q = X Rinv is the CholeskyQR factor.
constexpr int TRINV_THREADS = 256;
constexpr int TRINV_LRLD = CHOL_MAXW + 1;
constexpr int TRINV_SMEM = (CHOL_MAXW * CHOL_PLD + CHOL_NB * TRINV_LRLD + 2 * CHOL_NB * CHOL_PLD) * 8;

__global__ void __launch_bounds__(TRINV_THREADS) trinv_kernel(int w, const double* __restrict__ L, int64_t ldl,
                                                              const double* __restrict__ Dinv,
                                                              const int* __restrict__ status,
                                                              double* __restrict__ Rinv, int64_t ldr,
                                                              const int* __restrict__ gate) {
  if (gate != nullptr && __ldcg(gate) == 0) return;
  if (__ldcg(status) >= 2) return;  // failed, or the Newton-Schulz path already wrote T
  extern __shared__ double sm[];
  constexpr int PLD = CHOL_PLD;
  double* X = sm;                             // [CHOL_MAXW][PLD] rows oJ.. of block column J
  double* Lr = X + CHOL_MAXW * PLD;           // [32][TRINV_LRLD] L(oI.., oJ..oI)
  double* Tb = Lr + CHOL_NB * TRINV_LRLD;     // [32][PLD]
  double* Db = Tb + CHOL_NB * PLD;            // [32][PLD]
  const int tid = threadIdx.x;
  const int J = blockIdx.x, oJ = J * CHOL_NB, bsJ = min(CHOL_NB, w - oJ);
  const int nbk = (w + CHOL_NB - 1) / CHOL_NB;
  for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += TRINV_THREADS)
    X[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = __ldcg(Dinv + J * CHOL_NB * CHOL_NB + idx);
  const int r = tid >> 3, c0 = (tid & 7) * 4;  // thread owns T(r, c0..c0+3)
  for (int I = J + 1; I < nbk; ++I) {
    const int oI = I * CHOL_NB, bsI = min(CHOL_NB, w - oI), kl = oI - oJ;
    __syncthreads();
    for (int idx = tid; idx < CHOL_NB * kl; idx += TRINV_THREADS) {
      const int rr = idx % CHOL_NB, kk = idx / CHOL_NB;
      Lr[rr * TRINV_LRLD + kk] = rr < bsI ? __ldcg(L + (oI + rr) + static_cast<int64_t>(oJ + kk) * ldl) : 0.0;
    }
    for (int idx = tid; idx < CHOL_NB * CHOL_NB; idx += TRINV_THREADS)
      Db[(idx / CHOL_NB) * PLD + (idx % CHOL_NB)] = __ldcg(Dinv + I * CHOL_NB * CHOL_NB + idx);
    __syncthreads();
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
    for (int kk = 0; kk < kl; ++kk) {
      const double l = Lr[r * TRINV_LRLD + kk];
      const double* x = X + kk * PLD + c0;
      t0 = fma(l, x[0], t0);
      t1 = fma(l, x[1], t1);
      t2 = fma(l, x[2], t2);
      t3 = fma(l, x[3], t3);
    }
    Tb[r * PLD + c0] = t0;
    Tb[r * PLD + c0 + 1] = t1;
    Tb[r * PLD + c0 + 2] = t2;
    Tb[r * PLD + c0 + 3] = t3;
    __syncthreads();
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    for (int t = 0; t <= r; ++t) {
      const double d = Db[r * PLD + t];
      v0 = fma(d, Tb[t * PLD + c0], v0);
      v1 = fma(d, Tb[t * PLD + c0 + 1], v1);
      v2 = fma(d, Tb[t * PLD + c0 + 2], v2);
      v3 = fma(d, Tb[t * PLD + c0 + 3], v3);
    }
    double* xo = X + (kl + r) * PLD + c0;
    xo[0] = -v0;
    xo[1] = -v1;
    xo[2] = -v2;
    xo[3] = -v3;
  }
  __syncthreads();
  // write block column J of L^-1 (column-major, zeros above the diagonal block)
  for (int idx = tid; idx < w * bsJ; idx += TRINV_THREADS) {
    const int row = idx % w, c = idx / w;
    double v = 0.0;
    if (row >= oJ) v = X[(row - oJ) * PLD + c];
    Rinv[row + static_cast<int64_t>(oJ + c) * ldr] = v;
  }
}

}  // namespace qbk
