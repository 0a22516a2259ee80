// QB -> partial pivoted QR (NEXT-4): B P = Q~ R by Householder QR with column
// pivoting on the l x n factor B (row-major, ld ldb: row r of B contiguous), then Q^ = Q Q~.
//
// Step i (LAPACK dlaqp2 order): the pivot is the first column of largest partial norm among
// j >= i; columns i and p are swapped; the Householder reflector H_i = I - tau v v^T (v_0 = 1)
// maps B(i:l, i) to (beta, 0, ..), beta = -sign(alpha) ||x||; the trailing columns get
// B(i:l, j) -= tau v (v^T B(i:l, j)); the partial norms are downdated with R(i, j) and
// recomputed from scratch when cancellation makes the downdate inaccurate (sqrt(eps) test).
// Row-major B makes the heavy pass coalesced over columns.  The rank-1 update of step i is
// deferred (one-step lookahead): the next step's fused pass applies it while it forms
// w_{i+1} = B(i+1:l, :)^T v_{i+1}, so every step reads and writes the trailing block once; row i
// (for the norm downdate) and the two swapped columns get the update first.  Reductions are
// fixed-order (per-row-chunk partials summed in chunk order).
#pragma once
#include "common.cuh"

namespace qbk {

constexpr int QRCP_THREADS = 256;  // columns per CTA in the trailing passes
constexpr int QRCP_ROWS = 32;      // rows per CTA in the trailing passes

// norms[j] = norms2[j] = ||B(0:l, j)||_2 (the partial norms vn1 / vn2 of dlaqp2), perm[j] = j
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_init_kernel(const double* __restrict__ B, int64_t ldb, int l,
                                                               int n, double* __restrict__ vn1,
                                                               double* __restrict__ vn2, int* __restrict__ perm) {
  const int j = blockIdx.x * QRCP_THREADS + threadIdx.x;
  if (j >= n) return;
  double s0 = 0.0, s1 = 0.0;
  int r = 0;
  for (; r + 1 < l; r += 2) {
    const double a = B[static_cast<int64_t>(r) * ldb + j], b = B[static_cast<int64_t>(r + 1) * ldb + j];
    s0 = fma(a, a, s0);
    s1 = fma(b, b, s1);
  }
  if (r < l) {
    const double a = B[static_cast<int64_t>(r) * ldb + j];
    s0 = fma(a, a, s0);
  }
  const double nr = sqrt(s0 + s1);
  vn1[j] = nr;
  vn2[j] = nr;
  perm[j] = j;
}

// One CTA: pivot (argmax of vn1 over j >= i, first index on ties), column swap, Householder of
// column i.  v (length l - i, v_0 = 1) goes to vbuf and below the diagonal of B; tau[i]; B(i,i) = beta.
__global__ void __launch_bounds__(1024) qrcp_pivot_kernel(double* __restrict__ B, int64_t ldb, int l, int n, int i,
                                                          double* __restrict__ vn1, double* __restrict__ vn2,
                                                          int* __restrict__ perm, double* __restrict__ tau,
                                                          double* __restrict__ vbuf) {
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ int s_p;
  __shared__ double s_red[32];
  __shared__ double s_beta, s_scale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // argmax (ties -> smallest index)
  double best = -1.0;
  int bi = n;
  for (int j = i + tid; j < n; j += blockDim.x) {
    const double v = vn1[j];
    if (v > best) {
      best = v;
      bi = j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_val[warp] = best;
    s_idx[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    double b = s_val[0];
    int x = s_idx[0];
    for (int w = 1; w < static_cast<int>(blockDim.x) / 32; ++w)
      if (s_val[w] > b || (s_val[w] == b && s_idx[w] < x)) {
        b = s_val[w];
        x = s_idx[w];
      }
    s_p = x;
  }
  __syncthreads();
  const int p = s_p;
  if (p != i) {  // swap columns i and p of B (all l rows) and their bookkeeping
    for (int r = tid; r < l; r += blockDim.x) {
      double* a = B + static_cast<int64_t>(r) * ldb;
      const double t = a[i];
      a[i] = a[p];
      a[p] = t;
    }
    if (tid == 0) {
      double t = vn1[i];
      vn1[i] = vn1[p];
      vn1[p] = t;
      t = vn2[i];
      vn2[i] = vn2[p];
      vn2[p] = t;
      const int q = perm[i];
      perm[i] = perm[p];
      perm[p] = q;
    }
  }
  __syncthreads();
  // Householder of x = B(i:l, i)
  double ss = 0.0;
  for (int r = i + 1 + tid; r < l; r += blockDim.x) {
    const double x = B[static_cast<int64_t>(r) * ldb + i];
    ss = fma(x, x, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) s_red[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x) / 32; ++w) t += s_red[w];
    const double alpha = B[static_cast<int64_t>(i) * ldb + i];
    if (t == 0.0) {  // already zero below the diagonal: H = I
      tau[i] = 0.0;
      s_beta = alpha;
      s_scale = 0.0;
    } else {
      const double nrm = sqrt(fma(alpha, alpha, t));
      const double beta = alpha >= 0.0 ? -nrm : nrm;
      tau[i] = (beta - alpha) / beta;
      s_beta = beta;
      s_scale = 1.0 / (alpha - beta);
    }
  }
  __syncthreads();
  const double scale = s_scale;
  for (int r = i + tid; r < l; r += blockDim.x) {
    double* a = B + static_cast<int64_t>(r) * ldb + i;
    if (r == i) {
      *a = s_beta;
      vbuf[0] = 1.0;
    } else {
      const double v = *a * scale;
      *a = v;
      vbuf[r - i] = v;
    }
  }
}

// partials[c][j] = sum_{r in row chunk c} v_{r-i} B(r, j) for the trailing columns j > i
// (grid: column blocks x row chunks of QRCP_ROWS rows starting at row i)
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_w_kernel(const double* __restrict__ B, int64_t ldb, int l, int n,
                                                            int i, const double* __restrict__ vbuf,
                                                            double* __restrict__ partials, int64_t ldp) {
  const int j = i + 1 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  const int r0 = i + blockIdx.y * QRCP_ROWS, r1 = min(l, r0 + QRCP_ROWS);
  if (j >= n) return;
  double s0 = 0.0, s1 = 0.0;
  int r = r0;
  for (; r + 1 < r1; r += 2) {
    s0 = fma(vbuf[r - i], B[static_cast<int64_t>(r) * ldb + j], s0);
    s1 = fma(vbuf[r + 1 - i], B[static_cast<int64_t>(r + 1) * ldb + j], s1);
  }
  if (r < r1) s0 = fma(vbuf[r - i], B[static_cast<int64_t>(r) * ldb + j], s0);
  partials[blockIdx.y * ldp + j] = s0 + s1;
}

// B(r, j) -= tau v_{r-i} w_j on this CTA's row chunk, w_j = sum of the chunk partials in chunk
// order; the chunk holding row i also downdates the partial norms (dlaqp2), recomputing a norm
// from the rows below i when the downdate lost accuracy.
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_update_kernel(double* __restrict__ B, int64_t ldb, int l, int n,
                                                                 int i, const double* __restrict__ vbuf,
                                                                 const double* __restrict__ tau,
                                                                 const double* __restrict__ partials, int64_t ldp,
                                                                 int nchunks, double* __restrict__ vn1,
                                                                 double* __restrict__ vn2, double tol3z) {
  const int j = i + 1 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  if (j >= n) return;
  const double t = tau[i];
  if (t == 0.0 && blockIdx.y != 0) return;
  double w = 0.0;
  for (int c = 0; c < nchunks; ++c) w += partials[c * ldp + j];
  const double tw = t * w;
  const int r0 = i + blockIdx.y * QRCP_ROWS, r1 = min(l, r0 + QRCP_ROWS);
  for (int r = r0; r < r1; ++r) {
    double* a = B + static_cast<int64_t>(r) * ldb + j;
    *a = fma(-vbuf[r - i], tw, *a);
  }
  if (blockIdx.y == 0) {  // row i is final: R(i, j); downdate the partial norm of column j
    const double rij = B[static_cast<int64_t>(i) * ldb + j];
    const double n1 = vn1[j];
    if (n1 != 0.0) {
      double temp = fabs(rij) / n1;
      temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
      const double ratio = n1 / vn2[j];
      const double temp2 = temp * ratio * ratio;
      if (temp2 <= tol3z) {
        // rows i+1.. of column j, read after this thread's own updates; the rows below this
        // chunk are updated by other CTAs, so the recompute is deferred to qrcp_renorm_kernel
        vn1[j] = -1.0;  // marker
      } else {
        vn1[j] = n1 * sqrt(temp);
      }
    }
  }
}

// Columns marked by qrcp_update_kernel (vn1 = -1): ||B(i+1:l, j)|| from scratch (rare).
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_renorm_kernel(const double* __restrict__ B, int64_t ldb, int l,
                                                                 int n, int i, double* __restrict__ vn1,
                                                                 double* __restrict__ vn2) {
  const int j = i + 1 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  if (j >= n || vn1[j] != -1.0) return;
  double s = 0.0;
  for (int r = i + 1; r < l; ++r) {
    const double a = B[static_cast<int64_t>(r) * ldb + j];
    s = fma(a, a, s);
  }
  vn1[j] = sqrt(s);
  vn2[j] = vn1[j];
}

// Q~ (l x l, row-major, ld ldq) <- H_i Q~ = Q~ - tau v (v^T Q~) restricted to rows i.. (backward
// accumulation of Q~ = H_0 ... H_{l-1} I); v is read from below the diagonal of B (column i).
// Before H_i is applied, Q~(i:, 0:i) = 0, so only the columns j >= i change.
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_q_w_kernel(const double* __restrict__ Qt, int64_t ldq, int l,
                                                              int i, const double* __restrict__ B, int64_t ldb,
                                                              double* __restrict__ partials, int64_t ldp) {
  const int j = i + blockIdx.x * QRCP_THREADS + threadIdx.x;
  const int r0 = i + blockIdx.y * QRCP_ROWS, r1 = min(l, r0 + QRCP_ROWS);
  if (j >= l) return;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int r = r0;
  for (; r + 3 < r1; r += 4) {
    double q[4], v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      q[u] = Qt[static_cast<int64_t>(r + u) * ldq + j];
      v[u] = r + u == i ? 1.0 : B[static_cast<int64_t>(r + u) * ldb + i];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = fma(v[u], q[u], s[u]);
  }
  for (; r < r1; ++r) {
    const double v = r == i ? 1.0 : B[static_cast<int64_t>(r) * ldb + i];
    s[0] = fma(v, Qt[static_cast<int64_t>(r) * ldq + j], s[0]);
  }
  partials[blockIdx.y * ldp + j] = (s[0] + s[2]) + (s[1] + s[3]);
}

__global__ void __launch_bounds__(QRCP_THREADS) qrcp_q_update_kernel(double* __restrict__ Qt, int64_t ldq, int l,
                                                                   int i, const double* __restrict__ B, int64_t ldb,
                                                                   const double* __restrict__ tau,
                                                                   const double* __restrict__ partials, int64_t ldp,
                                                                   int nchunks) {
  const int j = i + blockIdx.x * QRCP_THREADS + threadIdx.x;
  if (j >= l) return;
  double w = 0.0;
  for (int c = 0; c < nchunks; ++c) w += partials[c * ldp + j];
  const double tw = tau[i] * w;
  const int r0 = i + blockIdx.y * QRCP_ROWS, r1 = min(l, r0 + QRCP_ROWS);
  for (int r = r0; r < r1; ++r) {
    const double v = r == i ? 1.0 : B[static_cast<int64_t>(r) * ldb + i];
    double* q = Qt + static_cast<int64_t>(r) * ldq + j;
    *q = fma(-v, tw, *q);
  }
}

// Q~ = I (row-major l x l); R = the strictly-lower part of B zeroed (after Q~ is formed).
__global__ void qrcp_identity_kernel(double* __restrict__ Qt, int64_t ldq, int l) {
  const int64_t total = static_cast<int64_t>(l) * l;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / l, c = idx - r * l;
    Qt[r * ldq + c] = r == c ? 1.0 : 0.0;
  }
}

__global__ void qrcp_zero_lower_kernel(double* __restrict__ B, int64_t ldb, int l) {
  const int64_t total = static_cast<int64_t>(l) * l;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / l, c = idx - r * l;
    if (c < r) B[r * ldb + c] = 0.0;
  }
}

// ---------------------------------------------------------------- lookahead (fused) variant
// Step i: qrcp_la_pivot (apply the deferred U_{i-1} to the pivot column and column i, swap,
// reflector v_i), qrcp_la_fw (trailing rows >= i, columns > i: apply U_{i-1}, accumulate the
// partials of w_i), qrcp_la_row (w_i from the partials, row i += U_i -> R(i, :), norm downdate).

__global__ void __launch_bounds__(1024) qrcp_la_pivot_kernel(double* __restrict__ B, int64_t ldb, int l, int n, int i,
                                                             double* __restrict__ vn1, double* __restrict__ vn2,
                                                             int* __restrict__ perm, double* __restrict__ tau,
                                                             const double* __restrict__ vprev, double* __restrict__ wprev,
                                                             double* __restrict__ vbuf,
                                                             const double* __restrict__ pmax,
                                                             const int* __restrict__ pidx, int npart) {
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ int s_p;
  __shared__ double s_red[32];
  __shared__ double s_beta, s_scale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double best = -1.0;
  int bi = n;
  if (npart > 0) {
    // the previous step's qrcp_la_row left one (max, first index) per block of columns > i - 1
    for (int c = tid; c < npart; c += blockDim.x) {
      const double v = pmax[c];
      if (v > best || (v == best && pidx[c] < bi)) {
        best = v;
        bi = pidx[c];
      }
    }
  } else {
    for (int j = i + tid; j < n; j += blockDim.x) {
      const double v = vn1[j];
      if (v > best) {
        best = v;
        bi = j;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_val[warp] = best;
    s_idx[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    double b = s_val[0];
    int x = s_idx[0];
    for (int w = 1; w < static_cast<int>(blockDim.x) / 32; ++w)
      if (s_val[w] > b || (s_val[w] == b && s_idx[w] < x)) {
        b = s_val[w];
        x = s_idx[w];
      }
    s_p = x;
  }
  __syncthreads();
  const int p = s_p;
  // One pass over the two columns that move (rows >= i; each element is a separate DRAM row, so the
  // phases are latency-bound): the deferred update of step i-1, the swap, and the sum of squares of
  // the new column i below the diagonal; the first PIV_REG rows per thread stay in registers for
  // the scaling pass.  Rows < i of the swapped columns are swapped as they are (no pending update).
  constexpr int PIV_REG = 4;
  const double tp = i > 0 ? tau[i - 1] : 0.0;
  const double wi = i > 0 ? wprev[i] : 0.0, wp = i > 0 ? wprev[p] : 0.0;
  double keep[PIV_REG];
  double ss = 0.0;
  auto move = [&](int r) -> double {
    double* a = B + static_cast<int64_t>(r) * ldb;
    double xi = a[i], xp = a[p];
    if (i > 0) {
      const double tv = tp * vprev[r - (i - 1)];
      xi = fma(-tv, wi, xi);
      xp = fma(-tv, wp, xp);
    }
    if (p != i) a[p] = xi;
    const double x = p != i ? xp : xi;  // the new column i
    if (r > i) ss = fma(x, x, ss);
    return x;
  };
#pragma unroll
  for (int u = 0; u < PIV_REG; ++u) {
    const int r = i + tid + u * static_cast<int>(blockDim.x);
    keep[u] = r < l ? move(r) : 0.0;
  }
  for (int r = i + tid + PIV_REG * static_cast<int>(blockDim.x); r < l; r += blockDim.x)
    B[static_cast<int64_t>(r) * ldb + i] = move(r);  // re-read by the scaling pass
  if (p != i)
    for (int r = tid; r < i; r += blockDim.x) {
      double* a = B + static_cast<int64_t>(r) * ldb;
      const double t = a[i];
      a[i] = a[p];
      a[p] = t;
    }
  ss = warp_sum(ss);
  if (lane == 0) s_red[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    if (i > 0) {
      wprev[i] = 0.0;
      wprev[p] = 0.0;
    }
    if (p != i) {
      double t = vn1[i];
      vn1[i] = vn1[p];
      vn1[p] = t;
      t = vn2[i];
      vn2[i] = vn2[p];
      vn2[p] = t;
      const int q = perm[i];
      perm[i] = perm[p];
      perm[p] = q;
    }
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x) / 32; ++w) t += s_red[w];
    // alpha: the new B(i, i) — thread 0 holds it in keep[0] (row i is its first row)
    const double alpha = keep[0];
    if (t == 0.0) {
      tau[i] = 0.0;
      s_beta = alpha;
      s_scale = 0.0;
    } else {
      const double nrm = sqrt(fma(alpha, alpha, t));
      const double beta = alpha >= 0.0 ? -nrm : nrm;
      tau[i] = (beta - alpha) / beta;
      s_beta = beta;
      s_scale = 1.0 / (alpha - beta);
    }
  }
  __syncthreads();
  const double scale = s_scale;
  auto put = [&](int r, double x) {
    double* a = B + static_cast<int64_t>(r) * ldb + i;
    if (r == i) {
      *a = s_beta;
      vbuf[0] = 1.0;
    } else {
      const double v = x * scale;
      *a = v;
      vbuf[r - i] = v;
    }
  };
#pragma unroll
  for (int u = 0; u < PIV_REG; ++u) {
    const int r = i + tid + u * static_cast<int>(blockDim.x);
    if (r < l) put(r, keep[u]);
  }
  for (int r = i + tid + PIV_REG * static_cast<int>(blockDim.x); r < l; r += blockDim.x)
    put(r, B[static_cast<int64_t>(r) * ldb + i]);
}

// rows [r0, r1) of the trailing block (r >= i, columns j > i): B -= tau_{i-1} v_{i-1} w_{i-1}^T, then
// partials[c][j] = sum_r v_i[r - i] B(r, j)
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_la_fw_kernel(double* __restrict__ B, int64_t ldb, int l, int n,
                                                                int i, const double* __restrict__ tau,
                                                                const double* __restrict__ vprev,
                                                                const double* __restrict__ wprev,
                                                                const double* __restrict__ vcur,
                                                                double* __restrict__ partials, int64_t ldp) {
  const int j = i + 1 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  const int r0 = i + blockIdx.y * QRCP_ROWS, r1 = min(l, r0 + QRCP_ROWS);
  if (j >= n) return;
  const double tw = i > 0 ? tau[i - 1] * wprev[j] : 0.0;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int r = r0;
  for (; r + 3 < r1; r += 4) {  // four rows in flight (memory-level parallelism)
    double* a = B + static_cast<int64_t>(r) * ldb + j;
    double b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) b[u] = a[u * ldb];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i > 0) {
        b[u] = fma(-vprev[r + u - (i - 1)], tw, b[u]);
        a[u * ldb] = b[u];
      }
      s[u] = fma(vcur[r + u - i], b[u], s[u]);
    }
  }
  for (; r < r1; ++r) {
    double* a0 = B + static_cast<int64_t>(r) * ldb + j;
    double b0 = *a0;
    if (i > 0) {
      b0 = fma(-vprev[r - (i - 1)], tw, b0);
      *a0 = b0;
    }
    s[0] = fma(vcur[r - i], b0, s[0]);
  }
  const double s0 = s[0] + s[2], s1 = s[1] + s[3];
  partials[blockIdx.y * ldp + j] = s0 + s1;
}

// w_i[j] (chunk partials in order) -> wprev; row i: R(i, j) = B(i, j) - tau_i w_i[j]; partial-norm
// downdate (dlaqp2), recomputed from rows > i (with the deferred update applied) on cancellation.
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_la_row_kernel(double* __restrict__ B, int64_t ldb, int l, int n,
                                                                 int i, const double* __restrict__ tau,
                                                                 const double* __restrict__ vcur,
                                                                 const double* __restrict__ partials, int64_t ldp,
                                                                 int nchunks, double* __restrict__ wprev,
                                                                 double* __restrict__ vn1, double* __restrict__ vn2,
                                                                 double tol3z, double* __restrict__ pmax,
                                                                 int* __restrict__ pidx) {
  __shared__ double s_val[QRCP_THREADS / 32];
  __shared__ int s_idx[QRCP_THREADS / 32];
  const int j = i + 1 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  double best = -1.0;  // this column's new partial norm, for the next step's pivot search
  int bi = n;
  if (j < n) {
    double w = 0.0;
    for (int c = 0; c < nchunks; ++c) w += partials[c * ldp + j];
    wprev[j] = w;
    const double tw = tau[i] * w;
    double* bij = B + static_cast<int64_t>(i) * ldb + j;
    const double rij = *bij - tw;
    *bij = rij;
    double n1 = vn1[j];
    if (n1 != 0.0) {
      double temp = fabs(rij) / n1;
      temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
      const double ratio = n1 / vn2[j];
      if (temp * ratio * ratio <= tol3z) {
        double s = 0.0;
        for (int r = i + 1; r < l; ++r) {
          const double a = fma(-vcur[r - i], tw, B[static_cast<int64_t>(r) * ldb + j]);
          s = fma(a, a, s);
        }
        n1 = sqrt(s);
        vn2[j] = n1;
      } else {
        n1 = n1 * sqrt(temp);
      }
      vn1[j] = n1;
    }
    best = n1;
    bi = j;
  }
  if (pmax == nullptr) return;
  // (max, first index) over this block's columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_val[warp] = best;
    s_idx[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < QRCP_THREADS / 32; ++w2)
      if (s_val[w2] > best || (s_val[w2] == best && s_idx[w2] < bi)) {
        best = s_val[w2];
        bi = s_idx[w2];
      }
    pmax[blockIdx.x] = best;
    pidx[blockIdx.x] = bi;
  }
}

}  // namespace qbk
