// small_loop.cuh — the whole adaptive blocked loop (Fig. 2 / Fig. 4) in
// ONE launch of one thread-block cluster, for problems whose A fits in the cluster's shared memory
// (BASELINE configs[0], 400 x 300).  The general path spends ~12 launches and a host round trip per
// block whose fixed latencies (TMA pipelines over long K with 10-column tiles, launch gaps) are
// 100x the block's arithmetic; here the residual never leaves shared memory, the block loop and
// its stop test run on the device (the paper: the Frobenius check "hardly adds at all to the
// execution time"), and the host reads the result once.
//
// Layout over the CL CTAs of the cluster (CL = 8 or 16):
//   A^(i):  CTA c holds columns [c nr, (c+1) nr) (all m rows) in shared memory, updated in place;
//   Ω_i:    CTA c draws its rows [c nr, (c+1) nr) of Ω_i (the same counter-based generator);
//   Y_i, Q_i: row-distributed, CTA c owns rows [c mr, (c+1) mr): Y_i = sum_c A_c Ω_c is summed over
//           DSMEM in CTA order; orth is the CholeskyQR2 of small.cuh with the Gram summed over the
//           CTAs (CTA order) and T computed on CTA 0 and read by the others; Z (power steps) is row-distributed like Ω;
//   Q̄:      CTA c keeps its rows of Q̄ in shared memory (the re-projection reads only those) and
//           writes them to global memory; B̄ rows go to global memory as blocks finish;
//   B_i = Q_i^T A_c and A_c -= Q_i B_i per CTA; r_i^2 and sum B_i^2 summed over CTAs in CTA order.
// Every sum has a fixed order, so results are bitwise reproducible.
#pragma once
#include <cooperative_groups.h>

#include "omega.cuh"
#include "small.cuh"

namespace qbk {

constexpr int SL_THREADS = 256;
constexpr int SL_MAXCL = 16;
constexpr int SL_CHUNK = 16;  // register accumulators per thread in the panel products

struct SmallLoopArgs {
  const double* A;
  int64_t lda;
  double* Aout;  // non-null: write the final residual back (QB_OVERWRITE_A)
  int64_t ldo;
  int m, n, b, q, kmax, reproj, full_first;
  double eps2, ns_tol2, tol;
  uint64_t seed;
  double* Qbar;
  int64_t ldq;
  double* Bbar;
  int64_t ldb;
  double* rec;  // per block: ell (after), w, r2, ei, max and min R diagonal of the first factorization
  double* out;  // [0] r2_0, [1] final r2, [2] k, [3] fallbacks, [4] 1 = orth breakdown, [5] blocks
  OmegaConsts K;
  int mr, nr;   // rows (of Y, Q) / columns (of A, rows of Ω, Z) per CTA
  // shared-memory carve-up, offsets in doubles
  int oA, oOm, oYp, oYs, oZs, oX2, oGp, oG, oT, oWp, oWr, oQc, oBc;
  unsigned long long* trace;  // diagnostics (QB_SMALL_TRACE): %globaltimer at phase marks of block 2
};

__device__ __forceinline__ unsigned long long sl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

namespace sl {
namespace cg = cooperative_groups;

// sum_k ptr_k[idx] over the cluster's CTAs in rank order, four remote loads in flight at a time
__device__ __noinline__ double rank_sum(cg::cluster_group& cl, const double* ptr, int idx, unsigned ncta) {
  double s = 0.0;
  for (unsigned k = 0; k < ncta; k += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (k + u < ncta) ? cl.map_shared_rank(ptr, k + u)[idx] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k + u < ncta) s += v[u];
  }
  return s;
}

// fixed-order CTA sum of a per-thread value (result valid in thread 0)
__device__ __forceinline__ double cta_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < SL_THREADS / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

// orth of a panel distributed over the cluster (CTA c: `rows` rows, column-major, ld `ld`):
// cholqr2()'s pass sequence with the Gram summed over the CTAs and T computed on CTA 0.
// Two cluster barriers per pass.  Returns true on breakdown (uniform over the cluster).
__device__ __noinline__ bool dist_orth(cg::cluster_group& cl, double* P, int ld, int rows, double global_rows, int w, bool single,
                          double* Gp, double* G, double* T, double* X2, const SmallLoopArgs& a, int* sf, int* sfl,
                          int& fallbacks, double* kap, int* kset) {
  const unsigned c = cl.block_rank(), ncta = cl.num_blocks();
  const int t = threadIdx.x;
  bool f_fact = false, f_shift = false, fail = false;
  unsigned long long* tr = (a.trace != nullptr && c == 0 && t == 0) ? a.trace : nullptr;
  auto pass = [&]() {
    if (tr && !tr[12]) tr[12] = sl_now();
    scq_gram(P, ld, rows, w, Gp);
    if (tr && !tr[13]) tr[13] = sl_now();
    cl.sync();  // every Gram partial is complete
    if (tr && !tr[14]) tr[14] = sl_now();
    if (c == 0) {
      #pragma unroll 1
      for (int e = t; e < w * w; e += SL_THREADS)
        G[(e / w) * SCQR_GLD + e % w] = rank_sum(cl, Gp, (e / w) * SCQR_GLD + e % w, ncta);
      __syncthreads();
      if (tr && !tr[15]) tr[15] = sl_now();
      bool ff = false, fs = false;
      int fb = 0;
      const bool first = *kset == 0;
      const bool fl = scq_factor(G, T, w, global_rows, a.ns_tol2, a.tol, ff, fs, fb, first ? kap : nullptr);
      if (t == 0) {
        sf[0] = ff;
        sf[1] = fs;
        sf[2] = fl;
        fallbacks += fb;
        if (first && ff && !fl) *kset = 1;  // kap holds the block's first factorization's R diagonal range
      }
    }
    if (tr && !tr[16]) tr[16] = sl_now();
    cl.sync();  // T and the flags of CTA 0 are ready (rewritten only after the next pass's first barrier)
    if (tr && !tr[17]) tr[17] = sl_now();
    if (t == 0) {
      const int* sf0 = cl.map_shared_rank(sf, 0);
      sfl[0] = sf0[0];
      sfl[1] = sf0[1];
      sfl[2] = sf0[2];
    }
    if (c != 0) {
      const double* T0 = cl.map_shared_rank(T, 0);
      #pragma unroll 1
      for (int e = t; e < w * w; e += SL_THREADS) T[(e / w) * SCQR_GLD + e % w] = T0[(e / w) * SCQR_GLD + e % w];
    }
    __syncthreads();
    f_fact |= sfl[0] != 0;
    f_shift |= sfl[1] != 0;
    fail = sfl[2] != 0;
    if (!fail) scq_apply(P, ld, rows, w, T, X2);
    if (tr && !tr[18]) tr[18] = sl_now();
  };
  pass();
  if (!fail && (single ? f_shift : f_fact)) pass();
  if (!fail && f_shift) {
    pass();
    if (!fail) pass();
  }
  return fail;
}

// Qf (m x w, ld m) = the full row-distributed panel (CTA r holds rows [r mr, ...) at Ys, ld mr).
__device__ __forceinline__ void gather_rows(cg::cluster_group& cl, double* Qf, const double* Ys, int m, int mr,
                                            int w) {
  const unsigned ncta = cl.num_blocks();
  #pragma unroll 1
  for (int e0 = threadIdx.x; e0 < m * w; e0 += 8 * SL_THREADS) {  // eight DSMEM loads in flight
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * SL_THREADS, tt = e / m, i = e % m;
      const unsigned r = static_cast<unsigned>(i / mr);
      v[u] = (e < m * w && r < ncta) ? cl.map_shared_rank(Ys, r)[tt * mr + (i - static_cast<int>(r) * mr)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * SL_THREADS, i = e % m;
      if (e < m * w && static_cast<unsigned>(i / mr) < ncta) Qf[e] = v[u];
    }
  }
  __syncthreads();
}

// Ys (own rows, ld mr) = sum over CTAs (in order) of their partials Yp (m x w, ld m).
__device__ __forceinline__ void sum_rows(cg::cluster_group& cl, double* Ys, const double* Yp, int m, int r0, int rr,
                                         int mr, int w) {
  const unsigned ncta = cl.num_blocks();
  #pragma unroll 1
  for (int e = threadIdx.x; e < rr * w; e += SL_THREADS) {
    const int tt = e / rr, r = e % rr;
    Ys[tt * mr + r] = rank_sum(cl, Yp, tt * m + r0 + r, ncta);
  }
  __syncthreads();
}

// Out (m x w, ld m) = M (m x k, ld m) X, X (k x w) with element (j, tt) at X[j * xs + tt * xt]:
// thread per row, SL_CHUNK accumulators in registers, the X entries broadcast.
__device__ __forceinline__ void rows_times(const double* M, int m, int k, const double* X, int xs, int xt, int w,
                                           double* Out) {
  #pragma unroll 1
  for (int t0 = 0; t0 < w; t0 += SL_CHUNK) {
    const int tw = min(SL_CHUNK, w - t0);
    #pragma unroll 1
    for (int i = threadIdx.x; i < m; i += SL_THREADS) {
      double acc[SL_CHUNK];
#pragma unroll
      for (int u = 0; u < SL_CHUNK; ++u) acc[u] = 0.0;
      #pragma unroll 1
      for (int j = 0; j < k; ++j) {
        const double v = M[j * m + i];
#pragma unroll
        for (int u = 0; u < SL_CHUNK; ++u)
          if (u < tw) acc[u] = fma(v, X[j * xs + (t0 + u) * xt], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < SL_CHUNK; ++u)
        if (u < tw) Out[(t0 + u) * m + i] = acc[u];
    }
  }
  __syncthreads();
}

// Out(jj, tt) = sum_i M(i, jj) P(i, tt) for the m x k M and m x w P (both ld m): warp per column jj,
// SL_CHUNK accumulators per lane, lane-strided rows, fixed xor-tree sums.  The callback receives
// (jj, tt, value) in lane 0.
template <typename F>
__device__ __forceinline__ void cols_dot(const double* M, int m, int k, const double* P, int w, F&& out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  #pragma unroll 1
  for (int t0 = 0; t0 < w; t0 += SL_CHUNK) {
    const int tw = min(SL_CHUNK, w - t0);
    #pragma unroll 1
    for (int jj = warp; jj < k; jj += SL_THREADS / 32) {
      double acc[SL_CHUNK];
#pragma unroll
      for (int u = 0; u < SL_CHUNK; ++u) acc[u] = 0.0;
      #pragma unroll 1
      for (int i = lane; i < m; i += 32) {
        const double v = M[jj * m + i];
#pragma unroll
        for (int u = 0; u < SL_CHUNK; ++u)
          if (u < tw) acc[u] = fma(v, P[(t0 + u) * m + i], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < SL_CHUNK; ++u) {
        if (u < tw) {
          const double s = warp_sum(acc[u]);
          if (lane == 0) out(jj, t0 + u, s);
        }
      }
    }
  }
  __syncthreads();
}

}  // namespace sl

__global__ void __launch_bounds__(SL_THREADS, 1) small_loop_kernel(const SmallLoopArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  double* Ac = sm + a.oA;
  double* Om = sm + a.oOm;
  double* Yp = sm + a.oYp;
  double* Ys = sm + a.oYs;
  double* Zs = sm + a.oZs;
  double* X2 = sm + a.oX2;
  double* Gp = sm + a.oGp;
  double* G = sm + a.oG;
  double* T = sm + a.oT;
  double* Wp = sm + a.oWp;
  double* Wr = sm + a.oWr;
  double* Qc = sm + a.oQc;  // this CTA's rows of Q̄ (ld mr)
  double* Bc = sm + a.oBc;
  __shared__ double red[SL_THREADS / 32];
  __shared__ double s_part[2];  // this CTA's r^2 and sum B^2 partials
  __shared__ double s_tot[2];
  __shared__ int sf[4];         // CTA 0: pass flags
  __shared__ int sfl[4];        // local copy of CTA 0's flags
  __shared__ double s_kap[2];   // CTA 0: R diagonal range of the block's first factorization
  __shared__ int s_kset;
  const unsigned c = cl.block_rank(), ncta = cl.num_blocks();
  const int t = threadIdx.x;
  const int m = a.m, n = a.n, mr = a.mr, nr = a.nr;
  const int r0 = static_cast<int>(c) * mr, rr = max(0, min(m, r0 + mr) - r0);
  const int c0 = static_cast<int>(c) * nr, cc = max(0, min(n, c0 + nr) - c0);
  int fallbacks = 0;

  // totals of the per-CTA partials s_part, in rank order (thread 0), broadcast in the CTA
  auto cluster_totals = [&](int nvals) {
    cl.sync();
    if (t == 0)
      for (int v = 0; v < nvals; ++v) {
        double s = 0.0;
        for (unsigned k = 0; k < ncta; ++k) s += cl.map_shared_rank(s_part, k)[v];
        s_tot[v] = s;
      }
    __syncthreads();
  };

  // A_c and r_0^2 = ||A||_F^2 (a0; Algorithm 1 line (2), reading R3)
  double s2 = 0.0;
  #pragma unroll 1
  for (int e = t; e < m * cc; e += SL_THREADS) {
    const double v = a.A[static_cast<int64_t>(c0 + e / m) * a.lda + e % m];
    Ac[e] = v;
    s2 = fma(v, v, s2);
  }
  s2 = sl::cta_sum(s2, red);
  if (t == 0) s_part[0] = s2;
  cluster_totals(1);
  const double r2_0 = s_tot[0];
  double r2 = r2_0, ei = r2_0;
  int ell = 0, nblk = 0;
  bool fail = false;
  bool stop = !(r2_0 > a.eps2);  // also stops on NaN (the host reports it)
  auto mark = [&](int i) {
    if (a.trace != nullptr && nblk == 2 && c == 0 && t == 0) a.trace[i] = sl_now();
  };
  cl.sync();  // s_part is rewritten below
  while (!stop && ell < a.kmax) {
    const int w = min(a.b, a.kmax - ell);
    mark(0);
    if (t == 0) {
      s_kset = 0;
      s_kap[0] = s_kap[1] = 0.0;
    }
    __syncthreads();
    const bool reproj_follows = ell > 0 && a.reproj && !a.full_first;
    // line (2): Ω_i rows [c0, c0 + cc) of global columns ell .. ell + w - 1 (row-major, ld w)
    if (cc > 0) {
      const int p0 = c0 >> 1, p1 = (c0 + cc - 1) >> 1;
      #pragma unroll 1
      for (int e = t; e < (p1 - p0 + 1) * w; e += SL_THREADS) {
        const int p = p0 + e / w, tt = e % w;
        double ev, od;
        gaussian_pair(a.seed, static_cast<uint64_t>(p), static_cast<uint64_t>(ell + tt), a.K, ev, od);
        if (2 * p >= c0 && 2 * p < c0 + cc) Om[(2 * p - c0) * w + tt] = ev;
        if (2 * p + 1 >= c0 && 2 * p + 1 < c0 + cc) Om[(2 * p + 1 - c0) * w + tt] = od;
      }
    }
    __syncthreads();
    mark(1);
    // line (3): Y_i = A^(i-1) Ω_i (partials over the column slabs, summed per row slab)
    sl::rows_times(Ac, m, cc, Om, w, 1, w, Yp);
    mark(2);
    cl.sync();
    sl::sum_rows(cl, Ys, Yp, m, r0, rr, mr, w);
    mark(3);
    fail = sl::dist_orth(cl, Ys, mr, rr, m, w, a.q == 0 ? reproj_follows : false, Gp, G, T, X2, a, sf, sfl,
                         fallbacks, s_kap, &s_kset);
    mark(4);
    // lines (4)-(7): power steps on the residual (readings R9, R10)
    for (int j = 0; j < a.q && !fail; ++j) {
      cl.sync();
      sl::gather_rows(cl, Yp, Ys, m, mr, w);  // Q_i in full (ld m)
      sl::cols_dot(Ac, m, cc, Yp, w, [&](int jj, int tt, double v) { Zs[tt * nr + jj] = v; });  // Z_c = A_c^T Q_i
      fail = sl::dist_orth(cl, Zs, nr, cc, n, w, false, Gp, G, T, X2, a, sf, sfl, fallbacks, s_kap, &s_kset);
      if (fail) break;
      sl::rows_times(Ac, m, cc, Zs, 1, nr, w, Yp);  // Y = A Z (partials); Yp free: every gather done
      cl.sync();
      sl::sum_rows(cl, Ys, Yp, m, r0, rr, mr, w);
      fail = sl::dist_orth(cl, Ys, mr, rr, m, w, j == a.q - 1 ? reproj_follows : false, Gp, G, T, X2, a, sf, sfl,
                           fallbacks, s_kap, &s_kset);
    }
    // line (8) / (3'): Q_i = orth(Q_i - Q̄ (Q̄^* Q_i)), on this CTA's rows of Q̄ (kept in Qc)
    if (!fail && ell > 0 && a.reproj) {
      #pragma unroll 1
      for (int e = t; e < ell * w; e += SL_THREADS) {  // W_c = Q̄(rows_c, :)^T Q_i(rows_c)
        const int tt = e / ell, l = e % ell;
        double s = 0.0;
        #pragma unroll 1
        for (int r = 0; r < rr; ++r) s = fma(Qc[l * mr + r], Ys[tt * mr + r], s);
        Wp[e] = s;
      }
      mark(5);
      cl.sync();
      // reduce-scatter: CTA k sums entries [k S, (k+1) S) over the ranks; then every CTA gathers W
      const int S = (ell * w + static_cast<int>(ncta) - 1) / static_cast<int>(ncta);
      #pragma unroll 1
      for (int e = t; e < S; e += SL_THREADS) {
        const int g = static_cast<int>(c) * S + e;
        if (g < ell * w) Wr[e] = sl::rank_sum(cl, Wp, g, ncta);
      }
      cl.sync();
      double* Wf = Yp;  // free until the gather below; ell <= m
      #pragma unroll 1
      for (int e = t; e < ell * w; e += SL_THREADS) Wf[e] = cl.map_shared_rank(Wr, e / S)[e % S];
      __syncthreads();
      #pragma unroll 1
      for (int e = t; e < rr * w; e += SL_THREADS) {  // Q_i(rows_c) -= Q̄(rows_c, :) W
        const int tt = e / rr, r = e % rr;
        double s = 0.0;
        #pragma unroll 1
        for (int l = 0; l < ell; ++l) s = fma(Qc[l * mr + r], Wf[tt * ell + l], s);
        Ys[tt * mr + r] -= s;
      }
      __syncthreads();
      mark(6);
      fail = sl::dist_orth(cl, Ys, mr, rr, m, w, false, Gp, G, T, X2, a, sf, sfl, fallbacks, s_kap, &s_kset);
    }
    mark(7);
    if (fail) break;
    // Q̄ = [Q̄ Q_i]: this CTA's rows (shared and global); Q_i in full for B_i and the downdate
    #pragma unroll 1
    for (int e = t; e < rr * w; e += SL_THREADS) {
      const int tt = e / rr, r = e % rr;
      const double v = Ys[tt * mr + r];
      Qc[(ell + tt) * mr + r] = v;
      a.Qbar[static_cast<int64_t>(ell + tt) * a.ldq + r0 + r] = v;
    }
    cl.sync();
    sl::gather_rows(cl, Yp, Ys, m, mr, w);
    mark(8);
    // line (9): B_i = Q_i^* A^(i-1) on this CTA's columns (reading R12), and sum B_i^2
    double bs = 0.0;
    sl::cols_dot(Ac, m, cc, Yp, w, [&](int jj, int tt, double v) {
      Bc[tt * nr + jj] = v;
      a.Bbar[static_cast<int64_t>(ell + tt) * a.ldb + c0 + jj] = v;
      bs = fma(v, v, bs);
    });
    mark(9);
    // line (10): A^(i) = A^(i-1) - Q_i B_i, and ||A^(i)||_F^2 (the stop test, reading R1): thread per row
    double as = 0.0;
    #pragma unroll 1
    for (int i = t; i < m; i += SL_THREADS) {
      #pragma unroll 1
      for (int t0 = 0; t0 < w; t0 += SL_CHUNK) {
        const int tw = min(SL_CHUNK, w - t0);
        double qrow[SL_CHUNK];
#pragma unroll
        for (int u = 0; u < SL_CHUNK; ++u) qrow[u] = u < tw ? Yp[(t0 + u) * m + i] : 0.0;
        const bool last = t0 + SL_CHUNK >= w;
        #pragma unroll 1
        for (int jj = 0; jj < cc; ++jj) {
          double s = 0.0;
#pragma unroll
          for (int u = 0; u < SL_CHUNK; ++u)
            if (u < tw) s = fma(qrow[u], Bc[(t0 + u) * nr + jj], s);
          const double v = Ac[jj * m + i] - s;
          Ac[jj * m + i] = v;
          if (last) as = fma(v, v, as);
        }
      }
    }
    mark(10);
    as = sl::cta_sum(as, red);
    bs = sl::cta_sum(bs, red);
    if (t == 0) {
      s_part[0] = as;
      s_part[1] = bs;
    }
    cluster_totals(2);
    r2 = s_tot[0];
    ei -= s_tot[1];
    ell += w;
    if (c == 0 && t == 0) {
      a.rec[6 * nblk + 0] = ell;
      a.rec[6 * nblk + 1] = w;
      a.rec[6 * nblk + 2] = r2;
      a.rec[6 * nblk + 3] = ei;
      a.rec[6 * nblk + 4] = s_kset ? s_kap[0] : 0.0;
      a.rec[6 * nblk + 5] = s_kset ? s_kap[1] : 0.0;
    }
    mark(11);
    ++nblk;
    stop = !(r2 > a.eps2);  // line (11): stop test (readings R1, R4); NaN stops too
    cl.sync();              // s_part and the gathered panel are reused next block
  }
  if (a.Aout != nullptr)
    #pragma unroll 1
    for (int e = t; e < m * cc; e += SL_THREADS) a.Aout[static_cast<int64_t>(c0 + e / m) * a.ldo + e % m] = Ac[e];
  if (c == 0 && t == 0) {
    a.out[0] = r2_0;
    a.out[1] = r2;
    a.out[2] = ell;
    a.out[3] = fallbacks;
    a.out[4] = fail ? 1.0 : 0.0;
    a.out[5] = nblk;
  }
  cl.sync();  // peers may still read this CTA's shared memory
}

}  // namespace qbk
