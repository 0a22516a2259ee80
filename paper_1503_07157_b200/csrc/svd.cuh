// svd.cuh — the k x k SVD core of rqb_svd (NEXT-1, QB -> partial SVD):
// block one-sided (Hestenes) Jacobi on X = R^T, R the triangular factor of B̄^T = Q_B R.
//
// One-sided Jacobi rotates pairs of columns of X until all columns are mutually orthogonal to a
// relative tolerance: X J = U D with J orthogonal (the accumulated rotations), D = column norms.
// It is relatively accurate — every rotation is computed from the Gram entries of the two columns
// it mixes, whose rounding is relative to those columns' norms — so the small singular values of a
// graded R (σ_k / σ_1 ~ 1e-9 at the target configuration) keep their relative accuracy, which a
// symmetric eigensolver of R R^T (absolute error u σ_1^2) would lose.
//
// Blocked for the GPU: the k columns are split into blocks of JNB = 16; a sweep visits every pair
// of blocks once (round-robin tournament, nblk - 1 steps of nblk / 2 disjoint pairs).  For one
// pair (I, J) the 32 x 32 Gram G = [X_I X_J]^T [X_I X_J] is formed (jac_gram_kernel, split over
// row chunks, summed in chunk order), diagonalised by cyclic two-sided Jacobi in shared memory
// (jac_solve_kernel, scaled threshold |G_ab| > tol sqrt(G_aa G_bb)), and the resulting rotation
// W = I + Δ is applied to the panel of X and of J as M += M Δ (jac_update_kernel).  Δ is
// accumulated directly (the rotation's c - 1 formed without cancellation), so a late, nearly
// trivial rotation perturbs X and J by its own size plus one rounding, not by a full 32-term
// product's rounding each time.  All reductions are in a fixed order: bitwise reproducible.
#pragma once
#include "common.cuh"

namespace qbk {

#ifndef QB_JAC_NB
#define QB_JAC_NB 16
#endif
constexpr int JNB = QB_JAC_NB;    // block width (16 or 32)
constexpr int JPW = 2 * JNB;      // pair width
#ifndef QB_JAC_RC
#define QB_JAC_RC 128
#endif
constexpr int JRC = QB_JAC_RC;     // rows per chunk (Gram partials, panel updates): 128 or 256
constexpr int JLDR = JRC + 4;     // row stride of a transposed chunk T[col][row] (= 4 mod 16 words:
                                  // conflict-free DMMA fragment loads)
constexpr int JLDD = JPW + 4;     // row stride of Δ in shared memory (= 4 mod 16 words)
constexpr int JGLD = JPW + 1;     // padded shared row of G / Δ in the solve
constexpr int JTHREADS = 256;
constexpr int JLOADS = JRC * JPW / JTHREADS;  // panel elements loaded per thread
constexpr int JGRAM_SMEM = JPW * JLDR * 8;
constexpr int JUPD_SMEM = (JPW * JLDR + JPW * JLDD) * 8;
constexpr int JTN = JPW / 8;                  // 8 x 8 DMMA tiles per dimension of a pair
constexpr int JTPW = JTN * JTN / (JTHREADS / 32);  // Gram tiles per warp (same row tile)
static_assert((JPW == 32 || JPW == 64) && JTHREADS == 256 && (JRC == 128 || JRC == 256),
              "fragment maps below assume these");
constexpr int JRT = JRC / 64;  // 8-row tiles per warp in the panel update

// Column j (0..JPW-1) of pair p's panel: block I or J of the pair, as a global column index.
__device__ __forceinline__ int jac_col(const int2 pr, int j) {
  return (j < JNB ? pr.x : pr.y) * JNB + (j & (JNB - 1));
}

// Rows [r0, r0 + rows) of pair pr's panel of M (column-major, ld) into T[JPW][JLDR] (transposed:
// T[j][r]), zero-padded; all loads of a thread are issued before its shared stores.
__device__ __forceinline__ void jac_load_panel(double* T, const double* __restrict__ M, int64_t ld, int2 pr, int r0,
                                               int rows, int t) {
  double v[JLOADS];
#pragma unroll
  for (int u = 0; u < JLOADS; ++u) {
    const int idx = t + u * JTHREADS, r = idx % JRC, j = idx / JRC;
    v[u] = r < rows ? __ldcg(M + static_cast<int64_t>(jac_col(pr, j)) * ld + r0 + r) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < JLOADS; ++u) {
    const int idx = t + u * JTHREADS, r = idx % JRC, j = idx / JRC;
    T[j * JLDR + r] = v[u];
  }
}

// Partial Gram of rows [c*JRC, min(nrows, (c+1)*JRC)) of pair p's panel of X (column-major,
// ld ldx): part[(p * nchunks + c) * JPW * JPW + i * JPW + j], on the FP64 tensor cores (DMMA
// m8n8k4: D(8x8) += A(8x4) B(4x8) with A = P^T, B = P over 4 rows at a time).  The 4 x 4 grid of
// 8 x 8 output tiles: warp w owns row tile w & 3 and column tiles 2 (w >> 2), 2 (w >> 2) + 1.
// grid = (npairs, nchunks).
__global__ void __launch_bounds__(JTHREADS) jac_gram_kernel(const double* __restrict__ X, int64_t ldx, int nrows,
                                                            const int2* __restrict__ pairs, int nchunks,
                                                            double* __restrict__ part) {
  extern __shared__ double jsm[];
  double* T = jsm;  // [JPW][JLDR]
  const int p = blockIdx.x, c = blockIdx.y, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int2 pr = pairs[p];
  const int r0 = c * JRC, rows = min(JRC, nrows - r0);
  jac_load_panel(T, X, ldx, pr, r0, rows, t);
  __syncthreads();
  const int ib = (w * JTPW) / JTN, jb0 = (w * JTPW) % JTN;
  const int m = lane >> 2, kk = lane & 3;
  double d[JTPW][2];
#pragma unroll
  for (int u = 0; u < JTPW; ++u) d[u][0] = d[u][1] = 0.0;
  const double* Ta = T + (8 * ib + m) * JLDR + kk;
  const double* Tb = T + (8 * jb0 + m) * JLDR + kk;
#pragma unroll 4
  for (int r = 0; r < JRC; r += 4) {  // zero-padded rows contribute nothing
    const double a = Ta[r];
#pragma unroll
    for (int u = 0; u < JTPW; ++u) dmma_8x8x4(d[u][0], d[u][1], a, Tb[u * 8 * JLDR + r]);
  }
  double* out = part + (static_cast<int64_t>(p) * nchunks + c) * JPW * JPW;
  const int gi = 8 * ib + m;
#pragma unroll
  for (int u = 0; u < JTPW; ++u) {
    const int gj = 8 * (jb0 + u) + 2 * kk;
    out[gi * JPW + gj] = d[u][0];
    out[gi * JPW + gj + 1] = d[u][1];
  }
}

// One pair per CTA of JST = 512 threads: G = sum of the chunk partials (chunk order); if some
// |G_ab| > tol sqrt(G_aa G_bb), diagonalise G by cyclic two-sided Jacobi (at most `inner` sweeps,
// round-robin parallel order) and write Δ = W - I of the accumulated rotation W (JPW x JPW,
// row-major) with flag[p] = 1; else flag[p] = 0 (nothing to apply).  Per rotation step the first
// 256 threads apply J^T G J to one 2 x 2 block each while the other 256 update two entries of Δ
// each, so a step is one angle phase and one update phase.  offmax receives max_ab |G_ab| /
// sqrt(G_aa G_bb) of the pair before rotating, as the bit pattern of a non-negative double
// (atomicMax on the bits is order-independent, so deterministic).
constexpr int JST = 512;
constexpr int JSOLVE_SMEM = 2 * JPW * JGLD * 8;
__global__ void __launch_bounds__(JST) jac_solve_kernel(const double* __restrict__ part, int nchunks,
                                                        double* __restrict__ Dout, int* __restrict__ flag,
                                                        unsigned long long* __restrict__ offmax, double tol,
                                                        int inner, int cross_only) {
  extern __shared__ double jsm[];
  constexpr int NP = JPW / 2;
  double* G = jsm;                    // [JPW][JGLD]
  double* Dl = G + JPW * JGLD;        // Δ = W - I
  __shared__ double cs[NP][3];        // c, s, c - 1
  __shared__ int prs[NP][2];
  __shared__ double red[JST / 32];
  __shared__ int any_rot;
  const int p = blockIdx.x, t = threadIdx.x;
  const double* src = part + static_cast<int64_t>(p) * nchunks * JPW * JPW;
  for (int idx = t; idx < JPW * JPW; idx += JST) {
    double s0 = 0.0, s1 = 0.0;  // chunk order: even chunks, odd chunks, then the pair (fixed)
    for (int c0 = 0; c0 < nchunks; c0 += 16) {  // sixteen partials in flight, summed in that order
      double x[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        x[u] = c0 + u < nchunks ? __ldcg(src + static_cast<int64_t>(c0 + u) * JPW * JPW + idx) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        if (c0 + u < nchunks) s0 += x[u];
        if (c0 + u + 1 < nchunks) s1 += x[u + 1];
      }
    }
    G[(idx / JPW) * JGLD + idx % JPW] = s0 + s1;
    Dl[(idx / JPW) * JGLD + idx % JPW] = 0.0;
  }
  __syncthreads();
  // scaled off-diagonal maximum (zero columns — padding — never rotate)
  double off = 0.0;
  for (int idx = t; idx < JPW * JPW; idx += JST) {
    const int a = idx / JPW, b = idx % JPW;
    if (a < b) {
      const double d = G[a * JGLD + a] * G[b * JGLD + b];
      if (d > 0.0) off = fmax(off, fabs(G[a * JGLD + b]) / sqrt(d));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
  if ((t & 31) == 0) red[t >> 5] = off;
  __syncthreads();
  if (t == 0) {
    double mx = 0.0;
    for (int w = 0; w < JST / 32; ++w) mx = fmax(mx, red[w]);
    red[0] = mx;
    atomicMax(offmax, static_cast<unsigned long long>(__double_as_longlong(mx)));
    flag[p] = mx > tol ? 1 : 0;
  }
  __syncthreads();
  if (!(red[0] > tol)) return;

  for (int sweep = 0; sweep < inner; ++sweep) {
    if (t == 0) any_rot = 0;
    __syncthreads();
    const int nsteps = cross_only ? NP : JPW - 1;
    for (int step = 0; step < nsteps; ++step) {
      if (t < NP) {
        // all pairs: circle method (step, JPW-1), (step + i, step - i) mod (JPW - 1); cross_only: the
        // NP^2 pairs between the two blocks, (i, NP + (i + step) mod NP)
        int a = cross_only ? t : (t == 0 ? step : (step + t) % (JPW - 1));
        int b = cross_only ? NP + (t + step) % NP : (t == 0 ? JPW - 1 : (step - t + (JPW - 1)) % (JPW - 1));
        if (a > b) {
          const int tmp = a;
          a = b;
          b = tmp;
        }
        const double al = G[a * JGLD + a], be = G[b * JGLD + b], ga = G[a * JGLD + b];
        double c = 1.0, s = 0.0, cm1 = 0.0;
        const double ab = al * be;
        if (ab > 0.0 && ga * ga > tol * tol * ab) {
          // x_a' = c x_a - s x_b, x_b' = s x_a + c x_b zeroes G_ab for t = s / c the small root of
          // t^2 + 2 zeta t - 1 = 0, zeta = d / h: t = sign(d) h / (|d| + sqrt(d^2 + h^2)).  Only the
          // orthogonality of the rotation (c^2 + s^2 = 1 to rounding) matters for accuracy; the
          // angle only steers convergence.
          const double d = be - al, h = 2.0 * ga;
          const double tt = copysign(1.0, d) * h / (fabs(d) + sqrt(fma(d, d, h * h)));
          c = rsqrt(fma(tt, tt, 1.0));
          s = c * tt;
          cm1 = -(s * s) / (1.0 + c);  // c - 1 = -s^2 / (1 + c), no cancellation
          any_rot = 1;
        }
        cs[t][0] = c;
        cs[t][1] = s;
        cs[t][2] = cm1;
        prs[t][0] = a;
        prs[t][1] = b;
      }
      __syncthreads();
      for (int idx = t; idx < NP * NP; idx += JST) {  // G <- J^T G J, the 2 x 2 block (pair qa rows, pair qb columns)
        const int qa = idx / NP, qb = idx % NP;
        const double c1 = cs[qa][0], s1 = cs[qa][1], c2 = cs[qb][0], s2 = cs[qb][1];
        if (s1 != 0.0 || s2 != 0.0) {
          const int a1 = prs[qa][0], b1 = prs[qa][1], a2 = prs[qb][0], b2 = prs[qb][1];
          const double g11 = G[a1 * JGLD + a2], g12 = G[a1 * JGLD + b2], g21 = G[b1 * JGLD + a2],
                       g22 = G[b1 * JGLD + b2];
          const double h11 = c2 * g11 - s2 * g12, h12 = s2 * g11 + c2 * g12;  // columns
          const double h21 = c2 * g21 - s2 * g22, h22 = s2 * g21 + c2 * g22;
          G[a1 * JGLD + a2] = c1 * h11 - s1 * h21;  // rows
          G[b1 * JGLD + a2] = s1 * h11 + c1 * h21;
          G[a1 * JGLD + b2] = c1 * h12 - s1 * h22;
          G[b1 * JGLD + b2] = s1 * h12 + c1 * h22;
        }
      }
      for (int idx = t; idx < JPW * NP; idx += JST) {  // Δ <- (I + Δ) J - I: row r of column pair q
        const int q = idx % NP, r = idx / NP;
        const double s = cs[q][1];
        if (s == 0.0) continue;
        const double cm1 = cs[q][2];
        const int a = prs[q][0], b = prs[q][1];
        const double da = Dl[r * JGLD + a], db = Dl[r * JGLD + b];
        double na = fma(cm1, da, da) - s * db, nb = fma(cm1, db, db) + s * da;
        if (r == a) {
          na += cm1;
          nb += s;
        } else if (r == b) {
          na -= s;
          nb += cm1;
        }
        Dl[r * JGLD + a] = na;
        Dl[r * JGLD + b] = nb;
      }
      __syncthreads();
    }
    if (!any_rot) break;
  }
  double* out = Dout + static_cast<int64_t>(p) * JPW * JPW;
  for (int idx = t; idx < JPW * JPW; idx += JST) out[idx] = Dl[(idx / JPW) * JGLD + idx % JPW];
}

// Apply each flagged pair's rotation to its panel of M (column-major, ld, nrows rows), in place,
// as M <- M + M Δ (the small update added last), on the FP64 tensor cores: the 128 x 32 chunk is
// 16 x 4 tiles of 8 x 8; warp w owns row tiles 2w, 2w + 1 and all 4 column tiles (K = 32: 8 DMMA
// k-steps).  grid = (npairs, ceil(nrows / JRC)).
__global__ void __launch_bounds__(JTHREADS) jac_update_kernel(double* __restrict__ M, int64_t ld, int nrows,
                                                              const int2* __restrict__ pairs,
                                                              const double* __restrict__ Dg,
                                                              const int* __restrict__ flag) {
  extern __shared__ double jsm[];
  double* T = jsm;                 // [JPW][JLDR]  (the chunk, transposed)
  double* D = T + JPW * JLDR;      // [JPW][JLDD]  (Δ, row-major)
  const int p = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (flag[p] == 0) return;
  const int2 pr = pairs[p];
  const int r0 = blockIdx.y * JRC, rows = min(JRC, nrows - r0);
  if (rows <= 0) return;
  const double* dsrc = Dg + static_cast<int64_t>(p) * JPW * JPW;
  constexpr int JDL = JPW * JPW / JTHREADS;  // Δ entries per thread, loaded with the panel (all in flight)
  double dv[JDL];
#pragma unroll
  for (int u = 0; u < JDL; ++u) dv[u] = __ldcg(dsrc + t + u * JTHREADS);
  jac_load_panel(T, M, ld, pr, r0, rows, t);
#pragma unroll
  for (int u = 0; u < JDL; ++u) {
    const int idx = t + u * JTHREADS;
    D[(idx / JPW) * JLDD + idx % JPW] = dv[u];
  }
  __syncthreads();
  const int m = lane >> 2, kk = lane & 3;
  double acc[JRT][JTN][2];
#pragma unroll
  for (int h = 0; h < JRT; ++h)
#pragma unroll
    for (int cb = 0; cb < JTN; ++cb) acc[h][cb][0] = acc[h][cb][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < JPW; ks += 4) {
    // A(m, kk) = chunk(8 rb + m, ks + kk) = T[ks + kk][8 rb + m];  B(kk, n) = Δ(ks + kk, 8 cb + n), n = lane >> 2
    double a[JRT];
#pragma unroll
    for (int h = 0; h < JRT; ++h) a[h] = T[(ks + kk) * JLDR + 8 * JRT * w + 8 * h + m];
#pragma unroll
    for (int cb = 0; cb < JTN; ++cb) {
      const double b = D[(ks + kk) * JLDD + 8 * cb + m];
#pragma unroll
      for (int h = 0; h < JRT; ++h) dmma_8x8x4(acc[h][cb][0], acc[h][cb][1], a[h], b);
    }
  }
  __syncthreads();  // every warp has read its A fragments: update T in place
#pragma unroll
  for (int h = 0; h < JRT; ++h)
#pragma unroll
    for (int cb = 0; cb < JTN; ++cb) {
      const int row = 8 * JRT * w + 8 * h + m, col = 8 * cb + 2 * kk;
      T[col * JLDR + row] += acc[h][cb][0];
      T[(col + 1) * JLDR + row] += acc[h][cb][1];
    }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < JLOADS; ++u) {
    const int idx = t + u * JTHREADS, r = idx % JRC, j = idx / JRC;
    if (r < rows) M[static_cast<int64_t>(jac_col(pr, j)) * ld + r0 + r] = T[j * JLDR + r];
  }
}

// Column norms sigma_j = ||X(:, j)||_2 (fixed order), j < ncols; one warp per column.
__global__ void __launch_bounds__(256) jac_norms_kernel(const double* __restrict__ X, int64_t ldx, int nrows,
                                                        int ncols, double* __restrict__ sig) {
  const int warp = (blockIdx.x * 256 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ncols) return;
  const double* col = X + static_cast<int64_t>(warp) * ldx;
  double s = 0.0;
  for (int i = lane; i < nrows; i += 32) s = fma(col[i], col[i], s);
  s = warp_sum(s);
  if (lane == 0) sig[warp] = sqrt(s);
}

// rank[j] = position of column j in descending order of sigma (ties: lower index first).
__global__ void __launch_bounds__(256) jac_rank_kernel(const double* __restrict__ sig, int n, int* __restrict__ rank) {
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= n) return;
  const double sj = sig[j];
  int r = 0;
  for (int i = 0; i < n; ++i) {
    const double si = sig[i];
    r += (si > sj || (si == sj && i < j)) ? 1 : 0;
  }
  rank[j] = r;
}

// Sorted outputs: S[rank_j] = sigma_j; Uhat (row-major k x k, ld ldu): Uhat[i][rank_j] = X(i, j) /
// sigma_j (0 for a zero column); Jrow (row-major, ld ldjr): Jrow[i][rank_j] = J(i, j); rows < k.
__global__ void __launch_bounds__(256) jac_finish_kernel(const double* __restrict__ X, int64_t ldx,
                                                         const double* __restrict__ Jm, int64_t ldj, int k,
                                                         const double* __restrict__ sig, const int* __restrict__ rank,
                                                         double* __restrict__ S, double* __restrict__ Uhat,
                                                         int64_t ldu, double* __restrict__ Jrow, int64_t ldjr) {
  const int64_t total = static_cast<int64_t>(k) * k;
  for (int64_t idx = blockIdx.x * 256ll + threadIdx.x; idx < total; idx += static_cast<int64_t>(gridDim.x) * 256) {
    const int j = static_cast<int>(idx / k), i = static_cast<int>(idx % k);
    const int rj = rank[j];
    const double sj = sig[j];
    Uhat[static_cast<int64_t>(i) * ldu + rj] = sj > 0.0 ? X[static_cast<int64_t>(j) * ldx + i] / sj : 0.0;
    Jrow[static_cast<int64_t>(i) * ldjr + rj] = Jm[static_cast<int64_t>(j) * ldj + i];
    if (i == 0) S[rj] = sj;
  }
}

// Tail rule: the smallest k' with resid2 + sum_{j >= k'} S_j^2 <= eps2 (S sorted
// descending); the suffix sums run from the smallest value up, in a fixed order.  One thread.
__global__ void jac_tail_rank_kernel(const double* __restrict__ S, int k, double resid2, double eps2,
                                     long long* __restrict__ kout) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double tail = resid2;
  int kk = k;
  for (int j = k - 1; j >= 0; --j) {
    const double nt = __dadd_rn(tail, __dmul_rn(S[j], S[j]));  // rounded like the oracle (no fma)
    if (nt > eps2) break;
    tail = nt;
    kk = j;
  }
  *kout = kk;
}

}  // namespace qbk
