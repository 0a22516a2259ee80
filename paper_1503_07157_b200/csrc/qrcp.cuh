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

namespace qbk {

// ---------------------------------------------------------------- blocked (dlaqps-style) schedule
// Panels of QRCP_NB pivots; inside a panel the trailing block is NOT updated.  The pending update of
// the panel's reflectors is carried by F (n x nb, F[kk * ldf + j] = F(j, kk)) as in LAPACK's
// dlaqps: the trailing block after kk reflectors is A - V F^T, with V the panel's Householder
// vectors.  Per step i = i0 + kk:
//   pivot: first column of largest partial norm; swap columns (and F rows); the pivot column gets
//          its pending update A(i:, i) -= A(i:, i0:i) F(i, 0:kk)^T; reflector (dlarfg);
//   w:     partials of A(i:, j)^T v over the (stale) trailing block — a read-only pass — and over
//          the panel's own columns (V(i:, q)^T v, for the incremental F update);
//   row:   aux(q) = -tau V(i:, q)^T v; F(j, kk) = tau w_j + F(j, 0:kk) aux; row i of the trailing block
//          A(i, j) -= A(i, i0:i) F(j, 0:kk)^T - F(j, kk); the dlaqp2 norm downdate (an exact norm
//          with the pending update applied on cancellation), and the next step's pivot partials.
// At the end of a panel the trailing block gets A -= V F^T as one GEMM.  Same pivots and R as the
// unblocked order in exact arithmetic; the trailing block is read once per step instead of read
// and written.
constexpr int QRCP_NB = 32;

constexpr int QRCP_WROWS = 64;   // rows per CTA of the blocked w pass (partials per column: (l - i) / 64)
constexpr int BKP_THREADS = 512;  // pivot kernel
constexpr int BKP_REG = 6;        // rows per pivot thread kept in registers (l - i <= 3072 fully)

// Step i's pivot (one CTA): the first column of largest partial norm p (from the previous row
// kernel's per-block maxima), published in piv[0]; columns i and p swapped in rows >= i only —
// rows < i (finished rows of R) are swapped by the row kernel, F's rows and the norms are read
// through the swap there too; the pivot column's pending update
// A(i:, i) = A(i:, p) - A(i:, i0:i) F(p, 0:kk)^T; the reflector (dlarfg): beta on the diagonal,
// v below it and in vbuf, tau[i].
__global__ void __launch_bounds__(BKP_THREADS) qrcp_bk_pivot_kernel(double* __restrict__ B, int64_t ldb, int l, int n,
                                                                    int i, int i0, const double* __restrict__ vn1,
                                                                    double* __restrict__ tau,
                                                                    const double* __restrict__ F, int64_t ldf,
                                                                    double* __restrict__ vbuf, int* __restrict__ piv,
                                                                    const double* __restrict__ pmax,
                                                                    const int* __restrict__ pidx, int npart) {
  __shared__ double s_val[BKP_THREADS / 32];
  __shared__ int s_idx[BKP_THREADS / 32];
  __shared__ int s_p;
  __shared__ double s_red[BKP_THREADS / 32];
  __shared__ double s_fi[QRCP_NB];
  __shared__ double s_alpha, s_beta, s_scale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = i - i0;
  double best = -1.0;
  int bi = n;
  if (npart > 0) {
    for (int c = tid; c < npart; c += BKP_THREADS) {
      const double v = pmax[c];
      if (v > best || (v == best && pidx[c] < bi)) {
        best = v;
        bi = pidx[c];
      }
    }
  } else {
    for (int j = i + tid; j < n; j += BKP_THREADS) {
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
    for (int w = 1; w < BKP_THREADS / 32; ++w)
      if (s_val[w] > b || (s_val[w] == b && s_idx[w] < x)) {
        b = s_val[w];
        x = s_idx[w];
      }
    s_p = x;
    piv[0] = x;
  }
  __syncthreads();
  const int p = s_p;
  if (tid < kk) s_fi[tid] = F[tid * ldf + p];  // F(i, :) after the swap = F(p, :) before it
  __syncthreads();
  // rows >= i: swap, the pending update of the new column i, the sum of squares below the diagonal
  double keep[BKP_REG], old[BKP_REG];
  double ss = 0.0;
#pragma unroll
  for (int u = 0; u < BKP_REG; ++u) {  // loads only (the swap's stores follow), so rows overlap
    const int r = i + tid + u * BKP_THREADS;
    keep[u] = 0.0;
    old[u] = 0.0;
    if (r < l) {
      const double* a = B + static_cast<int64_t>(r) * ldb;
      double x = a[p], y = 0.0;
      old[u] = a[i];
#pragma unroll
      for (int q = 0; q < QRCP_NB; q += 2)
        if (q < kk) {
          x = fma(-a[i0 + q], s_fi[q], x);
          if (q + 1 < kk) y = fma(-a[i0 + q + 1], s_fi[q + 1], y);
        }
      x += y;
      keep[u] = x;
      if (r == i) s_alpha = x;
      else ss = fma(x, x, ss);
    }
  }
  if (p != i)
#pragma unroll
    for (int u = 0; u < BKP_REG; ++u) {
      const int r = i + tid + u * BKP_THREADS;
      if (r < l) B[static_cast<int64_t>(r) * ldb + p] = old[u];
    }
  for (int r = i + tid + BKP_REG * BKP_THREADS; r < l; r += BKP_THREADS) {  // beyond the register rows
    double* a = B + static_cast<int64_t>(r) * ldb;
    double x = a[p];
    if (p != i) a[p] = a[i];
    for (int q = 0; q < kk; ++q) x = fma(-a[i0 + q], s_fi[q], x);
    a[i] = x;
    ss = fma(x, x, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) s_red[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < BKP_THREADS / 32; ++w) t += s_red[w];
    const double alpha = s_alpha;
    double tv;
    if (t == 0.0) {
      tv = 0.0;
      s_beta = alpha;
      s_scale = 0.0;
    } else {
      const double nrm = sqrt(fma(alpha, alpha, t));
      const double beta = alpha >= 0.0 ? -nrm : nrm;
      tv = (beta - alpha) / beta;
      s_beta = beta;
      s_scale = 1.0 / (alpha - beta);
    }
    tau[i] = tv;
  }
  __syncthreads();
  const double scale = s_scale;
#pragma unroll
  for (int u = 0; u < BKP_REG; ++u) {
    const int r = i + tid + u * BKP_THREADS;
    if (r < l) {
      const double v = r == i ? 1.0 : keep[u] * scale;
      B[static_cast<int64_t>(r) * ldb + i] = r == i ? s_beta : v;
      vbuf[r - i] = v;
    }
  }
  for (int r = i + tid + BKP_REG * BKP_THREADS; r < l; r += BKP_THREADS) {
    double* a = B + static_cast<int64_t>(r) * ldb;
    const double v = a[i] * scale;
    a[i] = v;
    vbuf[r - i] = v;
  }
}

// partials[c][j] = sum over chunk c (QRCP_WROWS rows from row i) of A(r, j) v_{r-i}, columns
// j >= j0 (j0 = the panel's first column: the panel's own columns give V(i:, q)^T v for F's
// incremental update).  Four rows in flight per thread.
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_bk_w_kernel(const double* __restrict__ B, int64_t ldb, int l,
                                                               int n, int i, int j0, const double* __restrict__ vbuf,
                                                               double* __restrict__ partials, int64_t ldp) {
  const int j = j0 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  const int r0 = i + blockIdx.y * QRCP_WROWS, r1 = min(l, r0 + QRCP_WROWS);
  if (j >= n) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int r = r0;
  for (; r + 3 < r1; r += 4) {
    const double* a = B + static_cast<int64_t>(r) * ldb + j;
    const double a0 = a[0], a1 = a[ldb], a2 = a[2 * ldb], a3 = a[3 * ldb];
    s0 = fma(vbuf[r - i], a0, s0);
    s1 = fma(vbuf[r + 1 - i], a1, s1);
    s2 = fma(vbuf[r + 2 - i], a2, s2);
    s3 = fma(vbuf[r + 3 - i], a3, s3);
  }
  for (; r < r1; ++r) s0 = fma(vbuf[r - i], B[static_cast<int64_t>(r) * ldb + j], s0);
  partials[blockIdx.y * ldp + j] = (s0 + s1) + (s2 + s3);
}

// Step i after the w pass, columns j > i (thread j reads F's row and the norms of column j
// through the pivot swap: from index i when j = p):
//   aux(q) = -tau_i V(i:, q)^T v (the panel columns' partials, fixed order);
//   F(j, kk) = tau_i w_j + F(j, 0:kk) aux;
//   row i: A(i, j) -= A(i, i0:i) F(j, 0:kk)^T + F(j, kk);
//   the dlaqp2 partial-norm downdate; where it lost accuracy, the exact norm of the updated column
//   ||A(i+1:, j) - V(i+1:, 0:kk+1) F(j, 0:kk+1)^T|| (the CTA's flagged columns packed into groups
//   of 32, all warps over slices of the rows: the trailing norms decay together, so over a stretch
//   of steps nearly every column needs this once);
//   per-block (max, first index) of the norms for the next pivot.
// Also the deferred swap of columns i and p in rows < i, and perm.
__global__ void __launch_bounds__(QRCP_THREADS) qrcp_bk_row_kernel(double* __restrict__ B, int64_t ldb, int l, int n,
                                                                 int i, int i0, const double* __restrict__ tau,
                                                                 const double* __restrict__ partials, int64_t ldp,
                                                                 int nchunks, double* __restrict__ F, int64_t ldf,
                                                                 double* __restrict__ vn1, double* __restrict__ vn2,
                                                                 int* __restrict__ perm, const int* __restrict__ piv,
                                                                 double tol3z, double* __restrict__ pmax,
                                                                 int* __restrict__ pidx) {
  __shared__ double s_val[QRCP_THREADS / 32];
  __shared__ int s_idx[QRCP_THREADS / 32];
  __shared__ double s_aux[QRCP_NB], s_ai[QRCP_NB];
  __shared__ double s_grp[QRCP_THREADS / 32][QRCP_NB];
  __shared__ int s_cnt[QRCP_THREADS / 32], s_list[QRCP_THREADS];
  __shared__ double s_part[QRCP_THREADS / 32][32], s_res[QRCP_THREADS];
  const int kk = i - i0;
  const int p = piv[0];
  const double t = tau[i];
  {
    const int q = threadIdx.x & 31, g = threadIdx.x >> 5;
    double a = 0.0;
    if (q < kk)
      for (int c = g; c < nchunks; c += QRCP_THREADS / 32) a += partials[c * ldp + i0 + q];
    s_grp[g][q] = a;
  }
  if (static_cast<int>(threadIdx.x) < kk)
    s_ai[threadIdx.x] = B[static_cast<int64_t>(i) * ldb + i0 + threadIdx.x];  // A(i, i0 + q): v entries
  if (p != i) {  // rows < i of columns i and p (finished rows of R)
    for (int r = blockIdx.x * QRCP_THREADS + threadIdx.x; r < i; r += gridDim.x * QRCP_THREADS) {
      double* a = B + static_cast<int64_t>(r) * ldb;
      const double x = a[i];
      a[i] = a[p];
      a[p] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const int x = perm[i];
      perm[i] = perm[p];
      perm[p] = x;
    }
  }
  __syncthreads();
  if (static_cast<int>(threadIdx.x) < kk) {
    double a = 0.0;
    for (int g = 0; g < QRCP_THREADS / 32; ++g) a += s_grp[g][threadIdx.x];
    s_aux[threadIdx.x] = -t * a;
  }
  __syncthreads();
  const int j = i + 1 + blockIdx.x * QRCP_THREADS + threadIdx.x;
  const int js = j == p ? i : j;  // where column j's F row and norms were before the swap
  double best = -1.0, n1 = 0.0, n2 = 0.0;
  int bi = n;
  bool recompute = false;
  if (j < n) {
    double w = 0.0;
#pragma unroll 16
    for (int c = 0; c < nchunks; ++c) w += partials[c * ldp + j];
    double f = t * w, rowsum = 0.0;
#pragma unroll
    for (int q = 0; q < QRCP_NB; ++q)
      if (q < kk) {
        const double fq = F[q * ldf + js];
        if (js != j) F[q * ldf + j] = fq;  // F's row follows the swap
        f = fma(fq, s_aux[q], f);
        rowsum = fma(s_ai[q], fq, rowsum);
      }
    F[kk * ldf + j] = f;
    double* bij = B + static_cast<int64_t>(i) * ldb + j;
    const double rij = *bij - rowsum - f;
    *bij = rij;
    n1 = vn1[js];
    n2 = vn2[js];
    if (n1 != 0.0) {
      double temp = fabs(rij) / n1;
      temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
      const double ratio = n1 / n2;
      if (temp * ratio * ratio <= tol3z) recompute = true;
      else n1 = n1 * sqrt(temp);
    }
  }
  // Exact norms for the flagged columns, packed 32 to a group (lanes over columns, the 8 warps over
  // slices of the rows), partial sums combined in warp order.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {
    const unsigned ballot = __ballot_sync(0xffffffffu, recompute);
    if (lane == 0) s_cnt[warp] = __popc(ballot);
    __syncthreads();
    int base = 0, total = 0;
    for (int w = 0; w < QRCP_THREADS / 32; ++w) {
      if (w < warp) base += s_cnt[w];
      total += s_cnt[w];
    }
    if (recompute) s_list[base + __popc(ballot & ((1u << lane) - 1u))] = threadIdx.x;
    __syncthreads();
    const int rows = l - i - 1, slice = (rows + QRCP_THREADS / 32 - 1) / (QRCP_THREADS / 32);
    const int ra = i + 1 + warp * slice, rz = min(l, ra + slice);
    for (int g = 0; g < total; g += 32) {
      const bool act = g + lane < total;
      const int tl = act ? s_list[g + lane] : 0;
      const int col = act ? i + 1 + blockIdx.x * QRCP_THREADS + tl : i;
      double f2[QRCP_NB];
#pragma unroll
      for (int q = 0; q < QRCP_NB; ++q) f2[q] = act && q <= kk ? F[q * ldf + col] : 0.0;
      double sa = 0.0, sb = 0.0;
      int r = ra;
      for (; r + 1 < rz; r += 2) {
        const double* a0 = B + static_cast<int64_t>(r) * ldb;
        const double* a1 = a0 + ldb;
        double x0 = a0[col], x1 = a1[col];
        const double2* v0 = reinterpret_cast<const double2*>(a0 + i0);
        const double2* v1 = reinterpret_cast<const double2*>(a1 + i0);
#pragma unroll
        for (int q = 0; q < QRCP_NB; q += 2)
          if (q <= kk) {
            const double2 u0 = v0[q / 2], u1 = v1[q / 2];
            x0 = fma(-u0.x, f2[q], x0);
            x1 = fma(-u1.x, f2[q], x1);
            x0 = fma(-u0.y, f2[q + 1], x0);
            x1 = fma(-u1.y, f2[q + 1], x1);
          }
        sa = fma(x0, x0, sa);
        sb = fma(x1, x1, sb);
      }
      if (r < rz) {
        const double* a0 = B + static_cast<int64_t>(r) * ldb;
        double x0 = a0[col];
        const double2* v0 = reinterpret_cast<const double2*>(a0 + i0);
#pragma unroll
        for (int q = 0; q < QRCP_NB; q += 2)
          if (q <= kk) {
            const double2 u0 = v0[q / 2];
            x0 = fma(-u0.x, f2[q], x0);
            x0 = fma(-u0.y, f2[q + 1], x0);
          }
        sa = fma(x0, x0, sa);
      }
      s_part[warp][lane] = sa + sb;
      __syncthreads();
      if (warp == 0 && act) {
        double t2 = 0.0;
        for (int w = 0; w < QRCP_THREADS / 32; ++w) t2 += s_part[w][lane];
        s_res[tl] = sqrt(t2);
      }
      __syncthreads();
    }
    if (recompute) {
      n1 = s_res[threadIdx.x];
      n2 = n1;
    }
  }
  if (j < n) {
    vn1[j] = n1;
    vn2[j] = n2;
    best = n1;
    bi = j;
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

// Vt[q][r'] = A(r0 + r', i0 + q), r' < rows, q < nb: the panel's Householder vectors below row r0,
// as the N-contiguous operand of the trailing GEMM.
__global__ void qrcp_bk_vt_kernel(const double* __restrict__ B, int64_t ldb, int r0, int rows, int i0, int nb,
                                  double* __restrict__ Vt, int64_t ldv) {
  const int64_t total = static_cast<int64_t>(rows) * nb;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx / nb), q = static_cast<int>(idx % nb);
    Vt[q * ldv + r] = B[static_cast<int64_t>(r0 + r) * ldb + i0 + q];
  }
}

}  // namespace qbk

namespace qbk {

// ---------------------------------------------------------------- blocked Q~ accumulation
// Q~ = H_0 ... H_{l-1} I backward by panels of QRCP_NB reflectors (LAPACK dorgqr/dlarft):
// H_{i0} ... H_{i0+nb-1} = I - V T V^T with T upper triangular (forward, columnwise), applied as
// Q~(i0:, i0:) -= V (T (V^T Q~(i0:, i0:))) — two GEMMs on the DMMA path per panel.

// V of the panel (rows i0.., unit diagonal, zero above it, the Householder vectors below — stored
// below R's diagonal) in two layouts: Vx[r'][q] (ld QRCP_NB) and Vt[q][r'] (ld ldv); q >= nb: 0.
__global__ void qrcp_vpanel_kernel(const double* __restrict__ B, int64_t ldb, int i0, int rows, int nb,
                                   double* __restrict__ Vx, double* __restrict__ Vt, int64_t ldv) {
  const int64_t total = static_cast<int64_t>(rows) * QRCP_NB;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx / QRCP_NB), q = static_cast<int>(idx % QRCP_NB);
    const double v = q >= nb || r < q ? 0.0 : (r == q ? 1.0 : B[static_cast<int64_t>(i0 + r) * ldb + i0 + q]);
    Vx[idx] = v;
    Vt[q * ldv + r] = v;
  }
}

// T (QRCP_NB x QRCP_NB, row-major, upper) of the panel from G = V^T V (column-major, ld QRCP_NB)
// and tau: the "UT transform" form of dlarft's T, T^{-1} = diag(1/tau) + striu(G) (Joffrain et al.
// 2006), solved by back substitution T(i, j) = tau_i (delta_ij - sum_{k>i} G(i, k) T(k, j)) — one
// warp, lane j owns column j in registers (tau_i = 0 gives a zero row, as dlarft does).
__global__ void __launch_bounds__(32) qrcp_tmat_kernel(const double* __restrict__ Gm, int nb,
                                                       const double* __restrict__ tau, double* __restrict__ Tm) {
  __shared__ double Gs[QRCP_NB][QRCP_NB + 1];
  __shared__ double ts[QRCP_NB];
  const int j = threadIdx.x;
  for (int i = 0; i < QRCP_NB; ++i) Gs[i][j] = Gm[i + j * QRCP_NB];  // G(i, j), column-major
  ts[j] = j < nb ? tau[j] : 0.0;
  __syncwarp();
  double t[QRCP_NB];
#pragma unroll
  for (int i = QRCP_NB - 1; i >= 0; --i) {
    double s = i == j ? 1.0 : 0.0;
#pragma unroll
    for (int k = i + 1; k < QRCP_NB; ++k) s = fma(-Gs[i][k], t[k], s);
    t[i] = i <= j ? ts[i] * s : 0.0;
  }
#pragma unroll
  for (int i = 0; i < QRCP_NB; ++i) Tm[i * QRCP_NB + j] = t[i];
}

// Zt[j' + q ldw] = sum_{s >= q} T(q, s) Wt[j' + s ldw] (Z = T W, stored transposed like W).
__global__ void qrcp_tz_kernel(const double* __restrict__ Tm, const double* __restrict__ Wt, int64_t ldw, int ncol,
                               double* __restrict__ Zt) {
  __shared__ double Ts[QRCP_NB * QRCP_NB];
  for (int e = threadIdx.x; e < QRCP_NB * QRCP_NB; e += blockDim.x) Ts[e] = Tm[e];
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncol) return;
  double w[QRCP_NB];
#pragma unroll
  for (int s = 0; s < QRCP_NB; ++s) w[s] = Wt[j + s * ldw];
#pragma unroll
  for (int q = 0; q < QRCP_NB; ++q) {
    double z = 0.0;
#pragma unroll
    for (int s = q; s < QRCP_NB; ++s) z = fma(Ts[q * QRCP_NB + s], w[s], z);
    Zt[j + q * ldw] = z;
  }
}

}  // namespace qbk
