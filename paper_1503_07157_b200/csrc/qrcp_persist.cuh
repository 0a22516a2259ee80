// qrcp_persist.cuh — one panel of the blocked pivoted QR (qrcp.cuh's dlaqps-style schedule) in ONE
// persistent cooperative launch: one CTA per SM, two grid-wide barriers per pivot step instead of
// three kernel boundaries, and the per-step work spread over the whole GPU.
//
// Per step i = i0 + kk (same arithmetic as qrcp_bk_*, LAPACK dlaqps/dlaqp2):
//   phase A (rows >= i partitioned over the CTAs, a warp per row):
//     p = argmax of the previous step's per-CTA maxima (first index on ties);
//     x_r = A(r, p) - A(r, i0:i) F(p, 0:kk)^T (the pivot column's pending update), the swap of
//     columns i and p in rows >= i (rows < i: the finished rows of R, swapped here too), perm;
//     per-CTA partials of sum_{r>i} x_r^2 and of V(r, q) x_r (for F's incremental update).
//   barrier
//   phase B (columns >= i0 partitioned over the CTAs):
//     every CTA forms the reflector (dlarfg) from the partials in the same order: beta, tau,
//     v = [1; x / (alpha - beta)], and aux(q) = -tau V(i:, q)^T v;
//     w_j = A(i:, j)^T v over the CTA's columns (the read-only pass over the stale trailing block);
//     F(j, kk) = tau w_j + F(j, 0:kk) aux; row i: A(i, j) -= A(i, i0:i) F(j, 0:kk)^T + F(j, kk);
//     the dlaqp2 norm downdate, exact recompute of flagged columns (CTA-wide, packed); the CTA's
//     (max, first index) for the next pivot; v into column i, beta on the diagonal.
//   barrier
// Data written by one CTA and read by another inside the launch is read with ld.global.cg (L2;
// the SMs' L1 is not coherent).
#pragma once

#include "common.cuh"
#include "qrcp.cuh"

namespace qbk {

constexpr int QP_THREADS = 512;
constexpr int QP_WARPS = QP_THREADS / 32;
constexpr int QP_MAX_SMEM = 200 * 1024;  // dynamic shared memory: v (l), w partials, F block
constexpr int QP_REP = 8;        // replicas of the data every CTA reads (spreads the L2 hot lines)
constexpr int QP_CPW = 16;       // CTAs per warp in the partial sums: gridDim.x <= QP_WARPS * QP_CPW

struct QrcpPanelArgs {
  double* B;
  int64_t ldb;
  int l, n, i0, nb;
  double* vn1;
  double* vn2;
  int* perm;
  double* tau;
  double* F;
  int64_t ldf;
  // exchanged between the CTAs, each in QP_REP replicas
  double* xbuf;   // QP_REP x l: x of the current step
  double* ssp;    // QP_REP x G: per-CTA sum of squares
  double* auxp;   // QP_REP x G x 32: per-CTA V^T x partials
  double* alpha;  // QP_REP: x_i
  double* pmax;   // QP_REP x G
  int* pidx;      // QP_REP x G
  unsigned* bar;  // grid barrier counter (zeroed before the launch)
  double tol3z;
  int cwp;        // row stride of the shared-memory F block (>= the columns a CTA owns)
  int first;      // step i0 == 0: pick the first pivot from vn1 itself
  unsigned long long* trace;  // diagnostics (QB_QRCP_PTRACE): %globaltimer marks of CTA 0, steps 0-3
};

#define QP_MARK(k)                                                                 \
  do {                                                                             \
    if (a.trace && c == 0 && tid == 0 && kk < 4) {                                 \
      unsigned long long t_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
      a.trace[kk * 16 + (k)] = t_;                                                 \
    }                                                                              \
  } while (0)

__device__ __forceinline__ void qp_grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (*reinterpret_cast<volatile unsigned*>(bar) < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__global__ void __launch_bounds__(QP_THREADS, 1) qrcp_panel_kernel(const QrcpPanelArgs a) {
  extern __shared__ __align__(16) double qp_sm[];
  double* xs = qp_sm;  // x / v (rows >= i), l - i entries, then the w partials
  __shared__ double s_red[QP_WARPS][33];
  __shared__ double s_aux[QRCP_NB], s_ai[QRCP_NB];
  __shared__ double s_scal[4];  // beta, tau, scale
  __shared__ int s_p;
  __shared__ double s_bv[QP_WARPS];
  __shared__ int s_bi[QP_WARPS];
  __shared__ int s_cnt[QP_WARPS], s_list[QP_THREADS];
  __shared__ double s_res[QP_THREADS];
  __shared__ double s_tot[33];
  __shared__ double s_fg[QRCP_NB + 1][32];  // flagged group: F rows (and scale F(j, kk)) per column
  __shared__ int s_col[32];

  double* __restrict__ B = a.B;
  const int64_t ldb = a.ldb, ldf = a.ldf;
  const int l = a.l, n = a.n, i0 = a.i0;
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // columns owned in phase B: [cj0, cj1), fixed for the panel
  const int ncols = n - i0, cw = (ncols + G - 1) / G;
  const int cj0 = i0 + c * cw, cj1 = min(n, cj0 + cw);
  unsigned target = 0;
  // thread tid owns column cj0 + tid for the whole panel: its norms in registers, its F row in
  // shared memory (F also goes to global memory for the trailing GEMM and the pivot swaps)
  const int jt = cj0 + tid;
  double n1r = jt < cj1 ? ldcg(a.vn1 + jt) : 0.0, n2r = jt < cj1 ? ldcg(a.vn2 + jt) : 1.0;
  double* sF = qp_sm + a.l + 2 * QP_THREADS;  // [QRCP_NB][cwp]
  const int cwp = a.cwp;
  const int rep = c % QP_REP;  // the replica of the exchanged data this CTA reads

  for (int kk = 0; kk < a.nb; ++kk) {
    const int i = i0 + kk;
    QP_MARK(0);
    // ---------------- phase A
    // this CTA's rows [ra, rz) of rows >= i; the first two per warp prefetched before the pivot is
    // known (their panel entries and A(r, i) do not depend on it)
    const int rcA = (l - i + G - 1) / G;
    const int raA = i + c * rcA, rzA = min(l, raA + rcA);
    double vq0[2], aiv0[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = raA + warp + u * QP_WARPS;
      const double* ar = B + static_cast<int64_t>(r < rzA ? r : i) * ldb;
      vq0[u] = r < rzA && lane < kk ? ldcg(ar + i0 + lane) : 0.0;
      aiv0[u] = r < rzA ? ldcg(ar + i) : 0.0;
    }
    int pv_;
    {
      double best = -1.0;
      int bi = n;
      if (a.first && kk == 0) {
        for (int j = i + tid; j < n; j += QP_THREADS) {
          const double v = ldcg(a.vn1 + j);
          if (v > best) {
            best = v;
            bi = j;
          }
        }
      } else {
        for (int q = tid; q < G; q += QP_THREADS) {
          const double v = ldcg(a.pmax + rep * G + q);
          const int x = __ldcg(a.pidx + rep * G + q);
          if (v > best || (v == best && x < bi)) {
            best = v;
            bi = x;
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
        s_bv[warp] = best;
        s_bi[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double b = s_bv[0];
        int x = s_bi[0];
        for (int w = 1; w < QP_WARPS; ++w)
          if (s_bv[w] > b || (s_bv[w] == b && s_bi[w] < x)) {
            b = s_bv[w];
            x = s_bi[w];
          }
        s_p = x;
      }
      __syncthreads();
      pv_ = s_p;
    }
    const int p = pv_;
    QP_MARK(1);
    const double fpl = lane < kk ? ldcg(a.F + lane * ldf + p) : 0.0;  // F(i, lane) after the swap
    // rows < i (finished rows of R): columns i and p to be swapped, at most one row per thread
    const int rc2 = (i + G - 1) / G, rsw = c * rc2 + tid;
    const bool swp = p != i && rsw < min(i, (c + 1) * rc2);
    const double sw_i = swp ? ldcg(B + static_cast<int64_t>(rsw) * ldb + i) : 0.0;
    const double sw_p = swp ? ldcg(B + static_cast<int64_t>(rsw) * ldb + p) : 0.0;
    {
      const int rows = l - i, rc = (rows + G - 1) / G;
      const int ra = i + c * rc, rz = min(l, ra + rc);
      double ss = 0.0, ax = 0.0;  // ax: lane q's sum of V(r, q) x_r
      for (int r0 = ra + warp; r0 < rz; r0 += 2 * QP_WARPS) {  // two rows per warp in flight
        double vq[2], ap[2], aiv[2];
        const bool pre = r0 == ra + warp;  // the prefetched pair
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = r0 + u * QP_WARPS;
          const double* ar = B + static_cast<int64_t>(min(r, rz - 1)) * ldb;
          vq[u] = pre ? vq0[u] : (lane < kk ? ldcg(ar + i0 + lane) : 0.0);
          ap[u] = ldcg(ar + p);
          aiv[u] = pre ? aiv0[u] : ldcg(ar + i);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = r0 + u * QP_WARPS;
          if (r >= rz) break;
          // lane 0's sum for every lane (the xor tree's lanes may differ in the last bit)
          const double x = __shfl_sync(0xffffffffu, ap[u] - warp_sum(vq[u] * fpl), 0);
          if (r > i) {
            if (lane == 0) ss = fma(x, x, ss);
            ax = fma(vq[u], x, ax);
          } else if (lane == 0) {
            for (int e = 0; e < QP_REP; ++e) a.alpha[e] = x;
          }
          if (lane < QP_REP) a.xbuf[lane * l + r - i] = x;
          if (lane == 0) {
            if (p != i) B[static_cast<int64_t>(r) * ldb + p] = aiv[u];
          }
        }
      }
      // rows < i (finished rows of R): columns i and p swapped
      if (swp) {
        B[static_cast<int64_t>(rsw) * ldb + i] = sw_p;
        B[static_cast<int64_t>(rsw) * ldb + p] = sw_i;
      }
      if (p != i) {
        if (c == 0 && tid == 0) {
          const int t = a.perm[i];
          a.perm[i] = a.perm[p];
          a.perm[p] = t;
        }
      }
      s_red[warp][lane] = ax;
      ss = warp_sum(ss);
      if (lane == 0) s_red[warp][32] = ss;
      __syncthreads();
      if (tid < 33) {
        double t = 0.0;
        for (int w = 0; w < QP_WARPS; ++w) t += s_red[w][tid];
        for (int e = 0; e < QP_REP; ++e) {
          if (tid < 32) a.auxp[(e * G + c) * 32 + tid] = t;
          else a.ssp[e * G + c] = t;
        }
      }
    }
    QP_MARK(2);
    if (a.trace && tid == 0 && kk == 1) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      a.trace[64 + 160 + c] = t_;
    }
    target += G;
    qp_grid_sync(a.bar, target);
    QP_MARK(3);

    // ---------------- phase B
    // this thread's column (independent of the reflector): F's row, A(i, j) and the norms, read
    // through the swap, issued before the reductions so that their latency overlaps them
    const int ja = max(cj0, i + 1), jn = cj1 - ja;
    const bool own = jt < cj1 && jt > i;
    const double bij_old = own ? ldcg(B + static_cast<int64_t>(i) * ldb + jt) : 0.0;
    if (own && jt == p) {  // the pivot swap: column p takes column i's F row and norms
      n1r = ldcg(a.vn1 + i);
      n2r = ldcg(a.vn2 + i);
      for (int q = 0; q < kk; ++q) sF[q * cwp + tid] = ldcg(a.F + q * ldf + i);
    }
    // the reflector's inputs, also independent of the reductions
    double alpha = 0.0, vi = 0.0;
    if (tid < 32) {
      alpha = ldcg(a.alpha + rep);
      if (tid < kk) vi = ldcg(B + static_cast<int64_t>(i) * ldb + i0 + tid);  // V(i, q)
    }
    // reflector and aux, every CTA in the same order: warp w sums the partials of CTAs
    // [w*cpw, (w+1)*cpw) (lane q: aux partial q; lane 0 also the sum of squares; all loads issued
    // together), then 33 threads sum the warps in order
    {
      const int cpw = (G + QP_WARPS - 1) / QP_WARPS, ca = warp * cpw, cz = min(G, ca + cpw);
      double pa_[QP_CPW];
#pragma unroll
      for (int u = 0; u < QP_CPW; ++u) {
        const int cc = ca + u;
        pa_[u] = cc < cz && lane < kk ? ldcg(a.auxp + (rep * G + cc) * 32 + lane) : 0.0;
      }
      const double ps_ = ca + lane < cz ? ldcg(a.ssp + rep * G + ca + lane) : 0.0;  // lane u: CTA ca + u
      // x (unscaled; 0 in row i, whose v entry is 1: w_j = A(i, j) + scale sum_{r>i} x_r A(r, j))
      {
        double xv[8];  // eight loads in flight per thread before the shared-memory stores
        int r = i + tid;
        for (; r + 7 * QP_THREADS < l; r += 8 * QP_THREADS) {
#pragma unroll
          for (int u = 0; u < 8; ++u) xv[u] = ldcg(a.xbuf + rep * l + r + u * QP_THREADS - i);
#pragma unroll
          for (int u = 0; u < 8; ++u) xs[r + u * QP_THREADS - i] = r + u * QP_THREADS == i ? 0.0 : xv[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = r + u * QP_THREADS < l ? ldcg(a.xbuf + rep * l + r + u * QP_THREADS - i) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (r + u * QP_THREADS < l) xs[r + u * QP_THREADS - i] = r + u * QP_THREADS == i ? 0.0 : xv[u];
      }
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < QP_CPW; ++u) t += pa_[u];
      const double s2 = __shfl_sync(0xffffffffu, warp_sum(ps_), 0);
      s_red[warp][lane] = t;
      if (lane == 0) s_red[warp][32] = s2;
      __syncthreads();
      QP_MARK(11);
      if (tid < 33) {
        double u2 = 0.0;
        for (int w = 0; w < QP_WARPS; ++w) u2 += s_red[w][tid];
        s_tot[tid] = u2;
      }
      __syncthreads();
      QP_MARK(12);
    }
    if (tid < 32) {
      const double t = s_tot[32], aq = s_tot[tid];
      double beta, tv, scale;
      if (t == 0.0) {
        tv = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        const double nrm = sqrt(fma(alpha, alpha, t));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tv = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      if (tid < kk) {
        s_ai[tid] = vi;
        s_aux[tid] = -tv * (vi + scale * aq);
      }
      if (tid == 0) {
        s_scal[0] = beta;
        s_scal[1] = tv;
        s_scal[2] = scale;
        if (c == 0) a.tau[i] = tv;
      }
    }
    __syncthreads();
    QP_MARK(4);
    const double beta = s_scal[0], tv = s_scal[1], scale = s_scal[2];
    QP_MARK(5);
    // v into column i (phase A's row partition), beta on the diagonal
    {
      const int rows = l - i, rc = (rows + G - 1) / G;
      const int ra = i + c * rc, rz = min(l, ra + rc);
      for (int r = ra + tid; r < rz; r += QP_THREADS)
        B[static_cast<int64_t>(r) * ldb + i] = r == i ? beta : xs[r - i] * scale;
    }
    // w over the owned columns j > i: warps over (32-column chunk, row split)
    const int nch = jn > 0 ? (jn + 31) / 32 : 0;
    const int S = nch > 0 ? max(1, QP_WARPS / nch) : 1;
    double* wp = xs + (l - i);  // S x nch*32 partials
    for (int u = warp; u < nch * S; u += QP_WARPS) {
      const int ch = u % nch, sp = u / nch;
      const int j = ja + ch * 32 + lane;
      const int jc = j < cj1 ? j : ja;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      const int rows = l - i, rs = (rows + S - 1) / S;
      const int r0 = i + sp * rs, r1 = min(l, r0 + rs);
      int r = r0;
      for (; r + 15 < r1; r += 16) {
        const double* ar = B + static_cast<int64_t>(r) * ldb + jc;
        double t[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) t[e] = ldcg(ar + e * ldb);
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          s0 = fma(xs[r + e - i], t[e], s0);
          s1 = fma(xs[r + e + 1 - i], t[e + 1], s1);
          s2 = fma(xs[r + e + 2 - i], t[e + 2], s2);
          s3 = fma(xs[r + e + 3 - i], t[e + 3], s3);
        }
      }
      for (; r < r1; ++r) s0 = fma(xs[r - i], ldcg(B + static_cast<int64_t>(r) * ldb + jc), s0);
      wp[sp * (nch * 32) + ch * 32 + lane] = (s0 + s1) + (s2 + s3);  // slot (row split, column)
    }
    __syncthreads();
    QP_MARK(6);
    // per owned column j > i (one per thread: a CTA owns at most QP_THREADS columns, checked on the
    // host): w, F, the row update, the norm downdate
    bool recompute = false;
    if (own) {
      double f0 = 0.0, rowsum = 0.0;  // F(j, 0:kk) aux and A(i, i0:i) F(j, 0:kk)^T
      for (int q = 0; q < kk; ++q) {
        const double fq = sF[q * cwp + tid];
        f0 = fma(fq, s_aux[q], f0);
        rowsum = fma(s_ai[q], fq, rowsum);
        if (jt == p) a.F[q * ldf + jt] = fq;  // F's row follows the swap
      }
      double w = 0.0;
      for (int sp = 0; sp < S; ++sp) w += wp[sp * (nch * 32) + (jt - ja)];
      w = fma(scale, w, bij_old);
      const double f = fma(tv, w, f0);
      sF[kk * cwp + tid] = f;
      a.F[kk * ldf + jt] = f;
      const double rij = bij_old - rowsum - f;
      B[static_cast<int64_t>(i) * ldb + jt] = rij;
      if (n1r != 0.0) {
        double temp = fabs(rij) / n1r;
        temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
        const double ratio = n1r / n2r;
        if (temp * ratio * ratio <= a.tol3z) recompute = true;
        else n1r = n1r * sqrt(temp);
      }
    }
    QP_MARK(7);
    // exact norms of the flagged columns (packed 32 to a group, warps over row slices)
    {
      const unsigned ballot = __ballot_sync(0xffffffffu, recompute);
      if (lane == 0) s_cnt[warp] = __popc(ballot);
      __syncthreads();
      int base = 0, total = 0;
      for (int w = 0; w < QP_WARPS; ++w) {
        if (w < warp) base += s_cnt[w];
        total += s_cnt[w];
      }
      if (recompute) s_list[base + __popc(ballot & ((1u << lane) - 1u))] = tid;
      __syncthreads();
      // lanes over rows (each lane's V row in registers, loaded once per pass), the group's columns
      // in passes of 8 (their F rows broadcast from shared memory, 8 loads in flight per lane);
      // per column: lane partials over the lane's rows, xor-tree warp sums, then warps in order
      for (int g = 0; g < total; g += 32) {
        const int gn = min(32, total - g);
        if (tid < 32) {
          const int tl = tid < gn ? s_list[g + tid] : 0;
          s_col[tid] = tid < gn ? cj0 + tl : i;
#pragma unroll
          for (int q = 0; q < QRCP_NB; ++q) s_fg[q][tid] = tid < gn && q < kk ? sF[q * cwp + tl] : 0.0;
          s_fg[QRCP_NB][tid] = tid < gn ? sF[kk * cwp + tl] * scale : 0.0;  // v_r = scale x_r
        }
        __syncthreads();
        for (int c0 = 0; c0 < gn; c0 += 8) {
          double acc[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[u] = 0.0;
          for (int rb = i + 1 + warp * 32; rb < l; rb += QP_WARPS * 32) {
            const int r = rb + lane;
            const bool rv = r < l;
            const double* ar = B + static_cast<int64_t>(rv ? r : i) * ldb;
            double v[QRCP_NB];
#pragma unroll
            for (int q = 0; q < QRCP_NB; q += 2) {
              double2 u2 = make_double2(0.0, 0.0);
              if (rv && q < kk) u2 = __ldcg(reinterpret_cast<const double2*>(ar + i0 + q));
              v[q] = u2.x;
              v[q + 1] = q + 1 < kk ? u2.y : 0.0;
            }
            const double xv = rv ? xs[r - i] : 0.0;
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = rv && c0 + u < gn ? ldcg(ar + s_col[c0 + u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              double y = fma(-xv, s_fg[QRCP_NB][c0 + u], x[u]);
#pragma unroll
              for (int q = 0; q < QRCP_NB; ++q)
                if (q < kk) y = fma(-v[q], s_fg[q][c0 + u], y);
              acc[u] = fma(y, y, acc[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double t2 = __shfl_sync(0xffffffffu, warp_sum(acc[u]), 0);
            if (lane == 0) s_red[warp][c0 + u] = t2;
          }
        }
        __syncthreads();
        if (tid < gn) {
          double t2 = 0.0;
          for (int w = 0; w < QP_WARPS; ++w) t2 += s_red[w][tid];
          s_res[s_list[g + tid]] = sqrt(t2);
        }
        __syncthreads();
      }
    }
    QP_MARK(8);
    double best = -1.0;
    int bi = n;
    if (own) {
      if (recompute) {
        n1r = s_res[tid];
        n2r = n1r;
      }
      a.vn1[jt] = n1r;
      a.vn2[jt] = n2r;
      best = n1r;
      bi = jt;
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
      s_bv[warp] = best;
      s_bi[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < QP_WARPS; ++w)
        if (s_bv[w] > best || (s_bv[w] == best && s_bi[w] < bi)) {
          best = s_bv[w];
          bi = s_bi[w];
        }
      for (int e = 0; e < QP_REP; ++e) {
        a.pmax[e * G + c] = best;
        a.pidx[e * G + c] = bi;
      }
    }
    QP_MARK(9);
    if (a.trace && tid == 0 && kk == 1) {  // every CTA's arrival time at the second barrier of step 1
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      a.trace[64 + c] = t_;
    }
    target += G;
    qp_grid_sync(a.bar, target);
    QP_MARK(10);
  }
}

}  // namespace qbk
