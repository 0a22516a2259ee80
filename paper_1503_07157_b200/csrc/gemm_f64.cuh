// FP64 GEMM for sm_100a (K2/K3/K4-Gram/K5/K6/K7 of DESIGN.md §5): TMA -> 128B-swizzled
// shared memory -> DMMA (mma.sync m8n8k4 f64) with register accumulators.
//
// tcgen05.mma has no FP64 kind on sm_100a (ptxas rejects .kind::f64), so the FP64
// contractions of the paper — Y = A Ω, B = Q^* A (:710), A -= Q B (:712),
// the power steps A^* Q / A Z (:868-870), the CholeskyQR Gram and Q = Y R^-1, and the
// re-projection Q - Q̄(Q̄^*Q) (:708) — run on the FP64 tensor pipe (SASS DMMA.8x8x4,
// 37.2 TFLOP/s measured, profiles/MEASURED_FP64.json) fed by TMA through an mbarrier ring.
//
// C(M x N) = sum_k opA(i, k) opB(k, j) with two operand layouts:
//   NN: opA(i,k) = A[i + k*lda] (M-contiguous), opB(k,j) = B[j + k*ldb] (N-contiguous)
//   TN: opA(i,k) = A[k + i*lda] (K-contiguous), opB(k,j) = B[k + j*ldb] (K-contiguous)
// CTA tile 128 x BN, k-tile 16; warp tile 64 x 32 = 8 x 4 DMMA 8x8 sub-tiles.
//
// Bank-conflict-free fragment loads: every operand stage is a set of TMA boxes whose 128-byte
// rows are XOR-swizzled (CU_TENSOR_MAP_SWIZZLE_128B).  For K-contiguous boxes (rows = m or
// n, 16 k per row) the 4 k of one DMMA are consecutive; for MN-contiguous boxes (rows = k,
// 16 m or n per row) the 4 k of one DMMA are {kq, kq+4, kq+8, kq+12}.  Either way a warp's
// 32 LDS.64 touch 16 distinct bank pairs twice: 2 wavefronts, the minimum for 256 bytes.
// The k permutation inside a 16-wide k-tile does not change the sum's terms.
#pragma once
#include "common.cuh"

namespace qbk {

enum GemmLayout { GEMM_NN = 0, GEMM_TN = 1 };
enum GemmEpi { EPI_STORE_COL = 0, EPI_STORE_ROW = 1, EPI_SUB_COL = 2 };

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 16;

struct GemmParams {
  int M, N, K;
  int tiles_m, tiles_n;
  int nkt;             // ceil(K / 16)
  int kt_per_split;    // k-tiles per split (gridDim.y splits)
  int raster_m_fast;   // 1: consecutive CTAs walk M first (they share the B panel)
  double* C;
  int64_t ldc;
  int64_t split_stride;  // elements between split partial outputs
  double* norm_partials; // EPI_SUB_COL: per-CTA sum of squares of the new C
  const int* gate;       // optional: the kernel does nothing unless *gate != 0
  int a3d, b3d;          // NN: operand maps are 3D {16, K, rows/16} -> one TMA per operand per stage
};

#ifndef QB_SUB_CTAS
#define QB_SUB_CTAS 3
#endif
#ifndef QB_ALL_CTAS
#define QB_ALL_CTAS 2
#endif
template <int BN, int EPI = 0>
struct GemmCfg {
  static constexpr int WARPS = (GEMM_BM / 64) * (BN / 32);
  static constexpr int THREADS = WARPS * 32;
  // subtract-updates (short K = b, epilogue-heavy) may run QB_SUB_CTAS CTAs per SM
  static constexpr bool SUB3 = BN == 64 && ((EPI == 2 && QB_SUB_CTAS == 3) || QB_ALL_CTAS == 3);
  static constexpr int STAGES = SUB3 ? 3 : (BN == 64 ? 4 : 5);
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 8;
  static constexpr int B_BYTES = BN * GEMM_BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + (2 * STAGES + 1) * 8 + WARPS * 8;
  // EPI_SUB_COL prefetches its C tile (128 x BN) by TMA into pipeline slots as they drain:
  // box {16 m, BN n}, C_PER_SLOT boxes per slot, C_GROUPS slots.
  static constexpr int C_BOX_BYTES = BN * 128;
  static constexpr int C_PER_SLOT = STAGE_BYTES / C_BOX_BYTES;
  static constexpr int C_GROUPS = (GEMM_BM / 16 + C_PER_SLOT - 1) / C_PER_SLOT;
  static_assert(C_PER_SLOT >= 1 && C_GROUPS <= STAGES, "C tile must fit in the drained pipeline slots");
  static constexpr int MIN_BLOCKS = SUB3 ? 3 : (BN == 64 ? 2 : 1);
};

template <int LAYOUT, int BN, int EPI>
__device__ __forceinline__ void gemm_issue_stage(const CUtensorMap* tA, const CUtensorMap* tB, uint8_t* sA,
                                                 uint8_t* sB, uint64_t* bar, int m0, int n0, int k0, int a3d,
                                                 int b3d) {
  using Cfg = GemmCfg<BN, EPI>;
  mbar_arrive_expect_tx(bar, Cfg::STAGE_BYTES);
  if (LAYOUT == GEMM_NN) {
    // the 16-row chunks of an MN-contiguous tile land at c * 2048 either way; a 3D map
    // {16, K, rows/16} moves them with one instruction when rows % 16 == 0
    if (a3d) {
      tma_load_3d(sA, tA, bar, 0, k0, m0 / 16);
    } else {
#pragma unroll
      for (int c = 0; c < GEMM_BM / 16; ++c) tma_load_2d(sA + c * 2048, tA, bar, m0 + 16 * c, k0);
    }
    if (b3d) {
      tma_load_3d(sB, tB, bar, 0, k0, n0 / 16);
    } else {
#pragma unroll
      for (int c = 0; c < BN / 16; ++c) tma_load_2d(sB + c * 2048, tB, bar, n0 + 16 * c, k0);
    }
  } else {
    tma_load_2d(sA, tA, bar, k0, m0);
    tma_load_2d(sB, tB, bar, k0, n0);
  }
}

// Issue the TMA loads of C-tile box group g (EPI_SUB_COL prefetch) into pipeline slot `slot`.
template <int BN, int EPI>
__device__ __forceinline__ void gemm_issue_c_group(const CUtensorMap* tC, uint8_t* smem, uint64_t* cbar, int g, int slot,
                                                   int m0, int n0) {
  using Cfg = GemmCfg<BN, EPI>;
#pragma unroll
  for (int j = 0; j < Cfg::C_PER_SLOT; ++j) {
    const int b = g * Cfg::C_PER_SLOT + j;
    if (b < GEMM_BM / 16) tma_load_2d(smem + slot * Cfg::STAGE_BYTES + j * Cfg::C_BOX_BYTES, tC, cbar, m0 + 16 * b, n0);
  }
}

template <int LAYOUT, int BN, int EPI>
__global__ void __launch_bounds__(GemmCfg<BN, EPI>::THREADS, GemmCfg<BN, EPI>::MIN_BLOCKS)
    gemm_f64_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                    const __grid_constant__ CUtensorMap tC, const GemmParams p) {
  using Cfg = GemmCfg<BN, EPI>;
  constexpr int STAGES = Cfg::STAGES;
  if (p.gate != nullptr && __ldcg(p.gate) == 0) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms, by pointer arithmetic on the __shared__
  // array so that the compiler keeps the shared address space (LDS, not generic LD).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* cbar = empty + STAGES;
  double* red = reinterpret_cast<double*>(cbar + 1);
  constexpr bool kPrefetchC = (EPI == EPI_SUB_COL);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;

  int tm, tn;
  if (p.raster_m_fast) {
    tm = blockIdx.x % p.tiles_m;
    tn = blockIdx.x / p.tiles_m;
  } else {
    tn = blockIdx.x % p.tiles_n;
    tm = blockIdx.x / p.tiles_n;
  }
  const int m0 = tm * GEMM_BM, n0 = tn * BN;
  const int kt0 = blockIdx.y * p.kt_per_split;
  const int kt1 = min(p.nkt, kt0 + p.kt_per_split);
  const int nk = max(kt1 - kt0, 0);

  if (tid == 0) {
    tma_prefetch_desc(&tA);
    tma_prefetch_desc(&tB);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::WARPS);
    }
    mbar_init(cbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (kPrefetchC) {
      tma_prefetch_desc(&tC);
      // pull the C tile towards L2 now; the shared-memory copy is taken when slots drain
      for (int b = 0; b < GEMM_BM / 16; ++b) tma_prefetch_l2_2d(&tC, m0 + 16 * b, n0);
      mbar_arrive_expect_tx(cbar, (GEMM_BM / 16) * Cfg::C_BOX_BYTES);
      // groups whose slot no k-tile ever uses go out right away
      for (int g = 0; g < Cfg::C_GROUPS; ++g) {
        const int t = nk - Cfg::C_GROUPS + g;
        if (t < 0) gemm_issue_c_group<BN, EPI>(&tC, smem, cbar, g, ((t % STAGES) + STAGES) % STAGES, m0, n0);
      }
    }
      for (int s = 0; s < STAGES && s < nk; ++s)
      gemm_issue_stage<LAYOUT, BN, EPI>(&tA, &tB, smem + s * Cfg::STAGE_BYTES, smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES,
                                   &full[s], m0, n0, (kt0 + s) * GEMM_BK, p.a3d, p.b3d);
  }

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Per-lane fragment offsets inside a stage (bytes), see the header comment.
  uint32_t offA[4][2], offB[4][2];
  if (LAYOUT == GEMM_NN) {
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      const int k = kq + 4 * (lane & 3);
      const int rsw = k & 7;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t o = k * 128 + ((((h * 4) + (lane >> 3)) ^ rsw) << 4) + (((lane >> 2) & 1) << 3);
        offA[kq][h] = o;
        offB[kq][h] = o;
      }
    }
  } else {
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      const int k = kq * 4 + (lane & 3);
      const uint32_t o = (lane >> 2) * 128 + ((((k >> 1) ^ (lane >> 2))) << 4) + ((k & 1) << 3);
      offA[kq][0] = offA[kq][1] = o;
      offB[kq][0] = offB[kq][1] = o;
    }
  }

  // Slot of k-tile j has been read by this warp: once every warp has, load k-tile j + STAGES
  // into it, or — past the last k-tile — a group of the EPI_SUB_COL C tile.
  auto refill = [&](int j) {
    const int slot = j % STAGES;
    const uint32_t par = (j / STAGES) & 1;
    if (j + STAGES < nk) {
      mbar_wait(&empty[slot], par);
      gemm_issue_stage<LAYOUT, BN, EPI>(&tA, &tB, smem + slot * Cfg::STAGE_BYTES,
                                   smem + slot * Cfg::STAGE_BYTES + Cfg::A_BYTES, &full[slot], m0, n0,
                                   (kt0 + j + STAGES) * GEMM_BK, p.a3d, p.b3d);
    } else if (kPrefetchC && j >= nk - Cfg::C_GROUPS) {
      mbar_wait(&empty[slot], par);
      gemm_issue_c_group<BN, EPI>(&tC, smem, cbar, j - (nk - Cfg::C_GROUPS), slot, m0, n0);
    }
  };

  for (int i = 0; i < nk; ++i) {
    const int slot = i % STAGES;
    const uint32_t par = (i / STAGES) & 1;
    mbar_wait(&full[slot], par);
    __syncwarp();
    const uint8_t* aS = smem + slot * Cfg::STAGE_BYTES;
    const uint8_t* bS = aS + Cfg::A_BYTES;
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      double a[8], b[4];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const uint32_t off = LAYOUT == GEMM_NN ? (wm * 4 + (mi >> 1)) * 2048 + offA[kq][mi & 1]
                                               : (wm * 64 + mi * 8) * 128 + offA[kq][0];
        a[mi] = *reinterpret_cast<const double*>(aS + off);
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const uint32_t off = LAYOUT == GEMM_NN ? (wn * 2 + (ni >> 1)) * 2048 + offB[kq][ni & 1]
                                               : (wn * 32 + ni * 8) * 128 + offB[kq][0];
        b[ni] = *reinterpret_cast<const double*>(bS + off);
      }
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    // Thread 0 refills the slot of the PREVIOUS k-tile: the other warps have usually released it
    // already, so the producer rarely stalls its own warp (STAGES-1 tiles stay in flight).
    if (tid == 0 && i >= 1) refill(i - 1);
  }
  if (tid == 0 && nk >= 1) refill(nk - 1);

  // ------------------------------------------------------------ epilogue
  const int mb = m0 + wm * 64 + (lane >> 2);
  const int nb = n0 + wn * 32 + 2 * (lane & 3);
  if (EPI == EPI_STORE_COL) {
    double* C = p.C + static_cast<int64_t>(blockIdx.y) * p.split_stride;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int m = mb + mi * 8;
      if (m >= p.M) continue;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = nb + ni * 8 + e;
          if (n < p.N) C[m + static_cast<int64_t>(n) * p.ldc] = acc[mi][ni][e];
        }
    }
    } else if (EPI == EPI_STORE_ROW) {
    double* C = p.C + static_cast<int64_t>(blockIdx.y) * p.split_stride;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int m = mb + mi * 8;
      if (m >= p.M) continue;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int n = nb + ni * 8;
        double* dst = C + static_cast<int64_t>(m) * p.ldc + n;
        if (n + 1 < p.N) {
          *reinterpret_cast<double2*>(dst) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        } else if (n < p.N) {
          dst[0] = acc[mi][ni][0];
        }
      }
    }
    } else {  // EPI_SUB_COL: C -= acc with C read from the prefetched smem tile, sum of squares
    mbar_wait(cbar, 0);
    double sq = 0.0, sq2 = 0.0;  // two independent FP64 chains (latency)
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int ml = wm * 64 + mi * 8 + (lane >> 2);
      const int b = ml >> 4, g = b / Cfg::C_PER_SLOT;
      const int slot = (((nk - Cfg::C_GROUPS + g) % STAGES) + STAGES) % STAGES;
      const uint8_t* box = smem + slot * Cfg::STAGE_BYTES + (b - g * Cfg::C_PER_SLOT) * Cfg::C_BOX_BYTES;
      const int m = m0 + ml;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int nl = wn * 32 + ni * 8 + 2 * (lane & 3) + e;
          const double c = *reinterpret_cast<const double*>(
              box + nl * 128 + ((((ml & 15) >> 1) ^ (nl & 7)) << 4) + ((ml & 1) << 3));
          const int n = n0 + nl;
          if (m < p.M && n < p.N) {
            const double v = c - acc[mi][ni][e];
            __stcg(p.C + m + static_cast<int64_t>(n) * p.ldc, v);
            if (e == 0) sq = fma(v, v, sq);
            else sq2 = fma(v, v, sq2);
          }
        }
    }
    if (p.norm_partials != nullptr) {
      sq = warp_sum(sq + sq2);
      if (lane == 0) red[warp] = sq;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < Cfg::WARPS; ++w) t += red[w];
        p.norm_partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
      }
    }
  }
}


}  // namespace qbk
