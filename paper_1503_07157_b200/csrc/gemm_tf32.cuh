// FP32 GEMM for sm_100a on the 5th-generation tensor cores (tcgen05.mma kind::tf32, TMEM
// accumulators), split "3xTF32" so that the products keep FP32 accuracy.  This is the FP32
// context's path for the contractions with the residual A (K2f/K5f/K6f):
// Y = A Ω, B = Q^* A (:710), A -= Q B (:712), the power steps A^* Q, A Z
// (:868-870), and on FP32 copies the re-projection Q_i -= Q̄ (Q̄^* Q_i) (:708) and CholeskyQR's
// X T (reading R18c).  The Grams and the Cholesky factorizations stay in FP64.
//
// Splitting (reading R18b): every operand x is written x = hi + lo with hi = RN_tf32(x) (10
// explicit mantissa bits, exactly representable in TF32) and lo = x - hi (exact in FP32,
// |lo| <= 2^-11 |x|); the tensor core forms hi*hi + hi*lo + lo*hi with FP32 accumulation.
// The dropped lo*lo term and the TF32 rounding of lo are below 2^-21 relative per product,
// under the FP32 accumulation error of the K-term sums.
//
// Accumulation (reading R18b): the tensor core's FP32 accumulation in TMEM is not
// round-to-nearest (measured: the error of a K-term sum grows like K^1.5, 1.4e-4 relative at
// K = 20000), so each chunk of TF_PROMO k-tiles (128 k) is accumulated in TMEM and then added
// into FP32 registers with IEEE rounding; two TMEM buffers let the MMAs of chunk c+1 run while
// chunk c is drained.
//
// Persistent CTAs (one per SM) walk the work units (tile x K-split) statically; CTA tile
// 128 x BN, k-tile 32 floats (one 128-byte swizzle row); 11 warps:
//   warp 0      TMA producer (one thread): raw FP32 tiles (and a pre-split B's hi / lo)
//   warp 1      TMEM allocator + MMA issuer (one thread): 4 k-steps x 3 tcgen05.mma per stage
//   warps 2..5  split the stage: A's row hi / lo into the stage's TMEM columns (TS, default) or
//               in place in shared memory (SS); B in place unless it arrives pre-split
//   warps 6..9  drain TMEM chunks into register accumulators, then the epilogue of the unit
//               (warp w reads TMEM lanes 32 (w % 4) .. + 31 = tile rows) while the MMAs of the
//               next unit run in the other TMEM buffer
//   warp 10     TF_SUB_COL only: TMA-loads the C tile, 128 x 32 at a time, into a ring that
//               the epilogue updates in place, and TMA-stores each sub-tile back once the
//               epilogue warps are done with it
// Barriers per stage: full (TMA bytes landed), conv (128 splitters done), empty (MMAs done,
// tcgen05.commit); per TMEM buffer: acc_full (chunk's MMAs done), acc_empty (drained); per C
// slot: cfull (loaded), cdone (updated by the 4 epilogue warps).
//
// gemm_tf32_sub_ares_kernel (end of file) is the short-K subtract-update variant whose A row
// block stays resident in TMEM across a CTA's run of tiles.
//
// Operand layouts in shared memory (UMMA canonical 128B-swizzle layouts):
//   K-major (TN): box {32 k, rows}: row r at r*128 B, 8-row groups at 1024 B (SBO), the k-th
//                 K=8 slice 32 B further (descriptor start + 2 per step)
//   MN-major (NN): chunks of 32 rows (128 B) x 32 k, chunk c at c*4096 B (LBO), 4-k groups at
//                 512 B (SBO) in the 32-byte-granule swizzle (SWIZZLE_128B_BASE32B, the only
//                 MN-major swizzle for 32-bit operands); the k-th K=8 slice 1024 B further
#pragma once
#include "common.cuh"

namespace qbk {

constexpr int TF_BM = 128;
constexpr int TF_BK = 32;
constexpr int TF_PROMO = 4;       // k-tiles (128 k) per TMEM accumulation chunk
constexpr int TF_THREADS = 352;   // 11 warps, see the header comment
constexpr int TF_CSUB = 32;       // TF_SUB_COL: C streams through shared memory 128 x 32 at a time
#ifndef QB_TF_CSLOTS
#define QB_TF_CSLOTS 4
#endif
constexpr int TF_CSLOTS = QB_TF_CSLOTS;  // ring of C sub-tiles

enum TfEpi { TF_STORE_COL = 0, TF_STORE_ROW = 1, TF_SUB_COL = 2 };

struct TfParams {
  int M, N, K;
  int tiles_m, tiles_n;
  int nkt;            // ceil(K / 32)
  int kt_per_split;
  int splits;         // work unit u: split u / tiles, tile u % tiles
  int raster_m_fast;
  void* C;            // STORE_*: double output (or split partials); SUB_COL: float C
  int64_t ldc;
  int64_t split_stride;
  double* norm_partials;  // SUB_COL: per-CTA sum of squares of the new C (FP64), one per CTA
  int a3d, b3d;       // NN: one 3D TMA per operand per stage ({32, K, rows/32} view)
  const int* gate;    // optional: the kernel does nothing unless *gate != 0
  int bsplit;         // TS: B arrives pre-split (tB = hi, tB2 = lo, tf32_split_kernel); no B split here
  float* C32;         // STORE_COL without split-K: optional FP32 copy of C (ld ldc32)
  int64_t ldc32;
};

// TS = true: the A operand goes to TMEM (hi and lo, 64 columns per stage, written by the
// splitters with tcgen05.st), so a stage's shared memory is [A raw][B_hi][B_lo] and more stages fit.
template <int BN, bool SUB = false, bool TS = false>
struct TfCfg {
  static constexpr int THREADS = TF_THREADS;
  static constexpr int A_BYTES = TF_BM * TF_BK * 4;
  static constexpr int B_BYTES = BN * TF_BK * 4;
  static constexpr int HI_BYTES = A_BYTES + B_BYTES;   // SS: [A_hi][B_hi], then [A_lo][B_lo]
  static constexpr int STAGE_BYTES = TS ? A_BYTES + 2 * B_BYTES : 2 * HI_BYTES;
  static constexpr int CSUB_BYTES = TF_BM * TF_CSUB * 4;
  static constexpr int C_BYTES = SUB ? TF_CSLOTS * CSUB_BYTES : 0;
  static constexpr int SMEM_STAGES = (224 * 1024 - C_BYTES) / STAGE_BYTES;
  static constexpr int TMEM_A_STAGES = (512 - 2 * BN) / 64;
  static constexpr int STAGES = TS ? (SMEM_STAGES < TMEM_A_STAGES ? SMEM_STAGES : TMEM_A_STAGES) : SMEM_STAGES;
  static constexpr int A_TMEM_COL = 2 * BN;  // TS: stage s holds A_hi at A_TMEM_COL + 64 s, A_lo 32 further
  static constexpr int TMEM_COLS = TS ? 512 : 2 * BN;  // two accumulator buffers (chunk c in buffer c & 1)
  static constexpr int SMEM_BYTES =
      1024 + STAGES * STAGE_BYTES + C_BYTES + (3 * STAGES + 4 + 2 * TF_CSLOTS) * 8 + 64;
  static_assert(STAGES >= 2, "at least double buffering");
  static_assert(BN == 64 || BN == 128, "BN: register accumulators of the promoter warps");
};

// Work unit u of a persistent CTA: tile origin and k-tile range.
struct TfUnit {
  int m0, n0, kt0, nk, split;
};

__device__ __forceinline__ TfUnit tf_unit(const TfParams& p, int u, int bn) {
  const int tiles = p.tiles_m * p.tiles_n;
  TfUnit r;
  r.split = u / tiles;
  const int t = u - r.split * tiles;
  int tm, tn;
  if (p.raster_m_fast) {
    tm = t % p.tiles_m;
    tn = t / p.tiles_m;
  } else {
    tn = t % p.tiles_n;
    tm = t / p.tiles_n;
  }
  r.m0 = tm * TF_BM;
  r.n0 = tn * bn;
  r.kt0 = r.split * p.kt_per_split;
  r.nk = max(min(p.nkt, r.kt0 + p.kt_per_split) - r.kt0, 0);
  return r;
}

// Shared-memory matrix descriptor: layout 2 = SWIZZLE_128B (K-major operands), 1 =
// SWIZZLE_128B_BASE32B (MN-major 32-bit operands: 32-byte granules of each 128-byte row XORed
// with the row index mod 4, the layout TMA writes with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, majors, N, M = 128.
template <int BN>
__host__ __device__ constexpr uint32_t tf32_idesc(int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(TF_BM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 consecutive TMEM columns of this thread's lane; the wait carries the registers as
// in/out operands so that no use of them can be scheduled before it.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// 32 consecutive TMEM columns of this thread's lane <- r (tcgen05.st 32x32b.x32)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// D[tmem] (+)= A[tmem] B[smem] (A K-major in TMEM: row = lane, one K element per column)
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void pin8(float (&t)[8]) {
  asm volatile("" : "+f"(t[0]), "+f"(t[1]), "+f"(t[2]), "+f"(t[3]), "+f"(t[4]), "+f"(t[5]), "+f"(t[6]), "+f"(t[7]));
}

// RN_tf32 with ties away from zero (= cvt.rna.tf32.f32 on finite x): add half an ulp of the
// 10-bit mantissa to the magnitude bits and truncate; two integer ops instead of cvt's four
// (cvt also keeps Inf/NaN; here Inf stays Inf and a NaN may become Inf, but lo = x - hi is NaN
// for both, so the products come out NaN either way)
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

template <int LAYOUT, int BN>
__device__ __forceinline__ void tf_load_b(const CUtensorMap* tB, uint8_t* sB, uint64_t* bar, int n0, int k0, int b3d) {
  if (LAYOUT == 0) {  // NN: MN-major chunks of 32 columns x 32 k
    if (b3d) {
      tma_load_3d(sB, tB, bar, 0, k0, n0 / 32);
    } else {
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tma_load_2d(sB + c * 4096, tB, bar, n0 + 32 * c, k0);
    }
  } else {  // TN: K-major rows
    tma_load_2d(sB, tB, bar, k0, n0);
  }
}

// One stage's raw A and B tiles; with bsplit, B's hi and lo tiles (tB, tB2) into sB and sB2.
template <int LAYOUT, int BN>
__device__ __forceinline__ void tf_issue_stage(const CUtensorMap* tA, const CUtensorMap* tB, const CUtensorMap* tB2,
                                               uint8_t* sA, uint8_t* sB, uint8_t* sB2, uint64_t* bar, int m0, int n0,
                                               int k0, int a3d, int b3d, int bsplit) {
  using Cfg = TfCfg<BN>;  // raw operand bytes do not depend on the epilogue or on TS
  mbar_arrive_expect_tx(bar, Cfg::HI_BYTES + (bsplit ? Cfg::B_BYTES : 0));
  if (LAYOUT == 0) {  // NN: MN-major chunks of 32 rows x 32 k
    if (a3d) {
      tma_load_3d(sA, tA, bar, 0, k0, m0 / 32);
    } else {
#pragma unroll
      for (int c = 0; c < TF_BM / 32; ++c) tma_load_2d(sA + c * 4096, tA, bar, m0 + 32 * c, k0);
    }
  } else {  // TN: K-major rows
    tma_load_2d(sA, tA, bar, k0, m0);
  }
  tf_load_b<LAYOUT, BN>(tB, sB, bar, n0, k0, b3d);
  if (bsplit) tf_load_b<LAYOUT, BN>(tB2, sB2, bar, n0, k0, b3d);
}

// hi = RN_tf32(x), lo = x - hi for a small operand that many tiles re-read (outer x inner,
// inner contiguous, leading dimension ld for all three arrays), split once instead of per tile.
__global__ void __launch_bounds__(256) tf32_split_kernel(const float* __restrict__ x, int64_t ld, int64_t outer,
                                                         int64_t inner, float* __restrict__ hi,
                                                         float* __restrict__ lo) {
  const int64_t total = outer * inner;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = idx / inner, i = idx - o * inner;
    const float v = x[o * ld + i];
    const float h = tf32_rna(v);
    hi[o * ld + i] = h;
    lo[o * ld + i] = v - h;
  }
}

// STORE_COL epilogue of one row (m) of a unit: FP64 C (or split partial) and the optional FP32
// copy; groups of 8 columns, pinned in order so that the compiler does not widen all BN
// accumulators to FP64 at once (register pressure)
template <int BN>
__device__ __forceinline__ void tf_store_col(const TfParams& p, const TfUnit& w, const float (&acc)[BN], int m,
                                             int ncols) {
  double* dst = static_cast<double*>(p.C) + static_cast<int64_t>(w.split) * p.split_stride + m +
                static_cast<int64_t>(w.n0) * p.ldc;
  float* dst32 = p.C32 != nullptr ? p.C32 + m + static_cast<int64_t>(w.n0) * p.ldc32 : nullptr;
#pragma unroll
  for (int c0 = 0; c0 < BN; c0 += 8) {
    float t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i] = acc[c0 + i];
    pin8(t);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (c0 + i < ncols) {
        *dst = static_cast<double>(t[i]);
        if (dst32 != nullptr) dst32[static_cast<int64_t>(c0 + i) * p.ldc32] = t[i];
      }
      dst += p.ldc;
    }
  }
}

template <int LAYOUT, int BN, int EPI, bool TS>
__global__ void __launch_bounds__(TF_THREADS, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                     const __grid_constant__ CUtensorMap tB2, const __grid_constant__ CUtensorMap tC,
                     const TfParams p) {
  if (p.gate != nullptr && __ldcg(p.gate) == 0) return;
  constexpr bool SUB = EPI == TF_SUB_COL;
  using Cfg = TfCfg<BN, SUB, TS>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* sC = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);  // SUB: ring of [32][128] sub-tiles
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::C_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint64_t* cfull = acc_empty + 2;      // [TF_CSLOTS]
  uint64_t* cdone = cfull + TF_CSLOTS;  // [TF_CSLOTS] the promoters are done with the slot's sub-tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cdone + TF_CSLOTS);
  double* red = reinterpret_cast<double*>(tmem_slot + 2);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int units = p.tiles_m * p.tiles_n * p.splits;

  if (tid == 0) {
    tma_prefetch_desc(&tA);
    tma_prefetch_desc(&tB);
    if (p.bsplit) tma_prefetch_desc(&tB2);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    for (int s = 0; s < TF_CSLOTS; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cdone[s], 4);  // one arrive per promoter warp
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- operand producer
    if (lane == 0) {
      int j = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const TfUnit w = tf_unit(p, u, BN);
        for (int kt = 0; kt < w.nk; ++kt, ++j) {
          const int slot = j % STAGES;
          if (j >= STAGES) mbar_wait(&empty[slot], ((j / STAGES) - 1) & 1);
          uint8_t* st = smem + slot * Cfg::STAGE_BYTES;
          // B lo: after B hi (TS: [A raw][B hi][B lo]) or in the lo half (SS: [A hi][B hi][A lo][B lo])
          uint8_t* sblo = TS ? st + Cfg::A_BYTES + Cfg::B_BYTES : st + Cfg::HI_BYTES + Cfg::A_BYTES;
          tf_issue_stage<LAYOUT, BN>(&tA, &tB, &tB2, st, st + Cfg::A_BYTES, sblo, &full[slot], w.m0, w.n0,
                                     (w.kt0 + kt) * TF_BK, p.a3d, p.b3d, p.bsplit);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc<BN>(LAYOUT == 0 ? 1 : 0, LAYOUT == 0 ? 1 : 0);
      // K-major: rows at 128 B, 8-row groups at 1024 B (SBO).  MN-major (BASE32B): 4-k groups
      // at 512 B (SBO), 32-row chunks at 4096 B (LBO)
      constexpr uint32_t LBO = LAYOUT == 0 ? 4096u : 16u;
      constexpr uint32_t SBO = LAYOUT == 0 ? 512u : 1024u;
      constexpr uint32_t LT = LAYOUT == 0 ? 1u : 2u;
      constexpr uint32_t KSTEP = LAYOUT == 0 ? 64u : 2u;  // descriptor units (16 B) per K=8 slice
      int j = 0, c = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int nk = tf_unit(p, u, BN).nk;
        uint32_t tacc = tmem_base;
        for (int kt = 0; kt < nk; ++kt, ++j) {
          const int slot = j % STAGES;
          const bool first = (kt % TF_PROMO) == 0;
          if (first) {
            // chunk c goes to accumulator buffer c & 1 once the promoters have drained it
            const int b = c & 1;
            if (c >= 2) mbar_wait(&acc_empty[b], ((c >> 1) - 1) & 1);
            tacc = tmem_base + static_cast<uint32_t>(b * BN);
          }
          mbar_wait(&conv[slot], (j / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (TS) {
            // A (hi, lo) in TMEM, K-major; B (hi, lo) in shared memory after the raw A
            constexpr uint32_t idesc_ts = tf32_idesc<BN>(0, LAYOUT == 0 ? 1 : 0);
            const uint32_t b_hi = smem_u32(smem + slot * Cfg::STAGE_BYTES) + Cfg::A_BYTES;
            const uint64_t dBh = umma_desc(b_hi, LBO, SBO, LT), dBl = umma_desc(b_hi + Cfg::B_BYTES, LBO, SBO, LT);
            const uint32_t ta = tmem_base + static_cast<uint32_t>(Cfg::A_TMEM_COL + 64 * slot);
#pragma unroll
            for (int kk = 0; kk < TF_BK / 8; ++kk) {
              const uint64_t adv = static_cast<uint64_t>(kk) * KSTEP;
              const uint32_t tah = ta + 8 * kk, tal = ta + 32 + 8 * kk;
              umma_tf32_ts(tacc, tah, dBh + adv, idesc_ts, (!first || kk > 0) ? 1u : 0u);
              umma_tf32_ts(tacc, tah, dBl + adv, idesc_ts, 1u);
              umma_tf32_ts(tacc, tal, dBh + adv, idesc_ts, 1u);
            }
          } else {
            const uint32_t a_hi = smem_u32(smem + slot * Cfg::STAGE_BYTES);
            const uint32_t b_hi = a_hi + Cfg::A_BYTES;
            const uint64_t dAh = umma_desc(a_hi, LBO, SBO, LT), dBh = umma_desc(b_hi, LBO, SBO, LT);
            const uint64_t dAl = umma_desc(a_hi + Cfg::HI_BYTES, LBO, SBO, LT);
            const uint64_t dBl = umma_desc(b_hi + Cfg::HI_BYTES, LBO, SBO, LT);
#pragma unroll
            for (int kk = 0; kk < TF_BK / 8; ++kk) {
              const uint64_t adv = static_cast<uint64_t>(kk) * KSTEP;
              umma_tf32(tacc, dAh + adv, dBh + adv, idesc, (!first || kk > 0) ? 1u : 0u);
              umma_tf32(tacc, dAh + adv, dBl + adv, idesc, 1u);
              umma_tf32(tacc, dAl + adv, dBh + adv, idesc, 1u);
            }
          }
          umma_commit(&empty[slot]);
          if ((kt % TF_PROMO) == TF_PROMO - 1 || kt == nk - 1) {
            umma_commit(&acc_full[c & 1]);
            ++c;
          }
        }
      }
    }
  } else if (warp < 6) {
    // ---------------------------------------------------------------- splitters
    const int t = tid - 64;
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int nk = tf_unit(p, u, BN).nk;
      for (int kt = 0; kt < nk; ++kt, ++j) {
        const int slot = j % STAGES;
        mbar_wait(&full[slot], (j / STAGES) & 1);
        uint8_t* st = smem + slot * Cfg::STAGE_BYTES;
        if (TS) {
          // A row r of the tile (TMEM lane r, this warp's quadrant): read its 32 k from the swizzled
          // raw stage, split, store hi / lo to the stage's TMEM columns
          const int quad = warp & 3, r = quad * 32 + lane;
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int k = 0; k < TF_BK; ++k) {
            const uint32_t off = LAYOUT == 0
                                     ? (r >> 5) * 4096 + k * 128 + ((((r & 31) >> 3) ^ (k & 3)) << 5) + ((r & 7) << 2)
                                     : r * 128 + ((((k >> 2) ^ (r & 7))) << 4) + ((k & 3) << 2);
            const float x = *reinterpret_cast<const float*>(st + off);
            const float h = tf32_rna(x);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(x - h);
          }
          const uint32_t ta = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                              static_cast<uint32_t>(Cfg::A_TMEM_COL + 64 * slot);
          tmem_st32(ta, hi);
          tmem_st32(ta + 32, lo);
          // B: hi in place, lo after it
          uint8_t* sb = st + Cfg::A_BYTES;
          if (!p.bsplit) {
#pragma unroll 4
            for (int i = t; i < Cfg::B_BYTES / 16; i += 128) {
              float4* hp = reinterpret_cast<float4*>(sb + i * 16);
              const float4 v = *hp;
              float4 h, l;
              h.x = tf32_rna(v.x);
              h.y = tf32_rna(v.y);
              h.z = tf32_rna(v.z);
              h.w = tf32_rna(v.w);
              l.x = v.x - h.x;
              l.y = v.y - h.y;
              l.z = v.z - h.z;
              l.w = v.w - h.w;
              *hp = h;
              *reinterpret_cast<float4*>(sb + Cfg::B_BYTES + i * 16) = l;
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // A's TMEM stores (overlapped with B)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        } else {
          // [A hi][B hi] split in place, lo halves after them; a pre-split B only needs A
          const int nsplit = p.bsplit ? Cfg::A_BYTES / 16 : Cfg::HI_BYTES / 16;
#pragma unroll 4
          for (int i = t; i < nsplit; i += 128) {
            float4* hp = reinterpret_cast<float4*>(st + i * 16);
            const float4 v = *hp;
            float4 h, l;
            h.x = tf32_rna(v.x);
            h.y = tf32_rna(v.y);
            h.z = tf32_rna(v.z);
            h.w = tf32_rna(v.w);
            l.x = v.x - h.x;
            l.y = v.y - h.y;
            l.z = v.z - h.z;
            l.w = v.w - h.w;
            *hp = h;
            *reinterpret_cast<float4*>(st + Cfg::HI_BYTES + i * 16) = l;
          }
          // generic-proxy writes -> visible to the tensor core (async proxy) before the MMA reads
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        mbar_arrive(&conv[slot]);
      }
    }
  } else if (warp < 10) {
    // ---------------------------------------------------------------- promoters + epilogue
    // Each K chunk of TF_PROMO k-tiles is accumulated by the tensor core in TMEM, then added
    // into FP32 registers here (round-to-nearest), which bounds the length of the tensor
    // core's own accumulation chain (reading R18b).  TMEM lane = tile row.  While this
    // epilogue runs, the MMAs of the next unit proceed in the other TMEM buffer.
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    double sq = 0.0;
    int c = 0, cs = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const TfUnit w = tf_unit(p, u, BN);
      float acc[BN];
#pragma unroll
      for (int i = 0; i < BN; ++i) acc[i] = 0.f;
      const int nchunks = (w.nk + TF_PROMO - 1) / TF_PROMO;
      for (int ch = 0; ch < nchunks; ++ch, ++c) {
        const int b = c & 1;
        mbar_wait(&acc_full[b], (c >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(trow + static_cast<uint32_t>(b * BN + c0), r);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[c0 + i] += __uint_as_float(r[i]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&acc_empty[b]);
      }

      const int m = w.m0 + row;
      if (EPI == TF_STORE_COL || EPI == TF_STORE_ROW) {
        if (m < p.M) {
          const int ncols = min(BN, p.N - w.n0);
          // groups of 8 columns, pinned in order so that the compiler does not widen all BN
          // accumulators to FP64 at once (register pressure)
          if (EPI == TF_STORE_COL) {
            tf_store_col<BN>(p, w, acc, m, ncols);
          } else {
            double* dst = static_cast<double*>(p.C) + static_cast<int64_t>(w.split) * p.split_stride +
                          static_cast<int64_t>(m) * p.ldc + w.n0;
            const bool vec = ncols == BN && (p.ldc & 1) == 0;
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 8) {
              float t[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) t[i] = acc[c0 + i];
              pin8(t);
              if (vec) {
#pragma unroll
                for (int i = 0; i < 8; i += 2)
                  *reinterpret_cast<double2*>(dst + c0 + i) = make_double2(t[i], t[i + 1]);
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  if (c0 + i < ncols) dst[c0 + i] = static_cast<double>(t[i]);
              }
            }
          }
        }
      } else {
        // TF_SUB_COL: C -= acc, 32 columns at a time through the shared-memory ring (sub-tile:
        // column n at n*128 floats; a warp touches 32 consecutive floats per column); FP64 sum
        // of squares of the new C; one thread TMA-stores each sub-tile (clipped to the matrix)
        const int ncols = m < p.M ? min(BN, p.N - w.n0) : 0;
#pragma unroll
        for (int sub = 0; sub < BN / TF_CSUB; ++sub, ++cs) {
          const int slot = cs % TF_CSLOTS;
          mbar_wait(&cfull[slot], (cs / TF_CSLOTS) & 1);
          float* cb = sC + slot * (TF_BM * TF_CSUB);
          // squares summed in FP32 over 8 entries (four chains), then in FP64: relative error
          // <= 8 * 2^-24 (positive terms), far below the FP32 residual's own rounding; FP64
          // conversions per entry cost 18 % of this kernel (R18)
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < TF_CSUB; ++i) {
            const float r = cb[i * TF_BM + row] - acc[sub * TF_CSUB + i];
            cb[i * TF_BM + row] = r;
            const float rv = sub * TF_CSUB + i < ncols ? r : 0.f;
            s4[i & 3] = fmaf(rv, rv, s4[i & 3]);
          }
          sq += (static_cast<double>(s4[0]) + static_cast<double>(s4[1])) +
                (static_cast<double>(s4[2]) + static_cast<double>(s4[3]));
          // generic-proxy writes -> visible to the TMA store the C warp issues after cdone
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&cdone[slot]);
        }
      }
    }
    if (SUB) {
      if (p.norm_partials != nullptr) {
        sq = warp_sum(sq);
        if (lane == 0) red[warp - 6] = sq;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 6 && lane == 0) p.norm_partials[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
      }
    }
  } else if (SUB) {
    // ---------------------------------------------------------------- C warp (warp 10)
    // Loads sub-tile cs into slot cs % TF_CSLOTS once the store of sub-tile cs - TF_CSLOTS (same
    // slot) has read it out; that store is issued here as soon as the promoters are done with
    // it (cdone), so the promoters never wait for a store.
    if (lane == 0) {
      tma_prefetch_desc(&tC);
      int cm[TF_CSLOTS] = {}, cn[TF_CSLOTS] = {};  // origin of the sub-tile held by each slot
      int cs = 0;
      auto store = [&](int t) {
        const int slot = t % TF_CSLOTS;
        mbar_wait(&cdone[slot], (t / TF_CSLOTS) & 1);
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                         reinterpret_cast<uint64_t>(&tC)),
                     "r"(smem_u32(sC + slot * (TF_BM * TF_CSUB))), "r"(cm[slot]), "r"(cn[slot])
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      };
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const TfUnit w = tf_unit(p, u, BN);
        for (int sub = 0; sub < BN / TF_CSUB; ++sub, ++cs) {
          const int slot = cs % TF_CSLOTS;
          if (cs >= TF_CSLOTS) {
            store(cs - TF_CSLOTS);
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          cm[slot] = w.m0;
          cn[slot] = w.n0 + sub * TF_CSUB;
          mbar_arrive_expect_tx(&cfull[slot], Cfg::CSUB_BYTES);
          tma_load_2d(sC + slot * (TF_BM * TF_CSUB), &tC, &cfull[slot], cm[slot], cn[slot]);
        }
      }
      for (int t = cs - TF_CSLOTS < 0 ? 0 : cs - TF_CSLOTS; t < cs; ++t) store(t);
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------------------
// Subtract-update C -= A B for a short K (<= 128, the block size b: the downdate A^(i) -= Q_i B_i
// and the re-projection Q_i -= Q̄ W) with the A row block RESIDENT in TMEM.  Each persistent CTA
// takes a contiguous run of tiles in n-fast order, so consecutive tiles share their 128 rows of
// A: those are loaded, split (hi, lo) and stored to TMEM once per row block instead of once
// per tile, and the only per-tile operand traffic is the pre-split B tile (hi, lo; L2-resident)
// besides C itself.  Warp roles as in gemm_tf32_kernel; the splitters only handle A.
template <int BN>
struct TfAresCfg {
  static constexpr int A_BYTES = TF_BM * TF_BK * 4;          // one 32-k slab of A (raw)
  static constexpr int B_BYTES = BN * TF_BK * 4;             // one 32-k slab of B (hi or lo)
  static constexpr int BSTAGE_BYTES = 2 * B_BYTES;
  static constexpr int CSUB_BYTES = TF_BM * TF_CSUB * 4;
  static constexpr int C_BYTES = TF_CSLOTS * CSUB_BYTES;
  static constexpr int ASTAGES = 2;
  static constexpr int BSTAGES = (224 * 1024 - C_BYTES - ASTAGES * A_BYTES) / BSTAGE_BYTES;
  static constexpr int A_TMEM_COL = 2 * BN;                  // slab s: hi at +64 s, lo at +64 s + 32
  static constexpr int TMEM_COLS = 512;
  static constexpr int NBAR = 2 * BSTAGES + 2 * ASTAGES + 2 + 4 + 2 * TF_CSLOTS;
  static constexpr int SMEM_BYTES = 1024 + BSTAGES * BSTAGE_BYTES + ASTAGES * A_BYTES + C_BYTES + NBAR * 8 + 64;
  static_assert(BSTAGES >= 2, "B double buffering");
  static_assert(A_TMEM_COL + 64 * 4 <= TMEM_COLS, "A (K <= 128) and two accumulators fit TMEM");
};

__device__ __forceinline__ void tf_ares_range(const TfParams& p, int& u0, int& u1) {
  const int64_t units = static_cast<int64_t>(p.tiles_m) * p.tiles_n;
  u0 = static_cast<int>(units * blockIdx.x / gridDim.x);
  u1 = static_cast<int>(units * (blockIdx.x + 1) / gridDim.x);
}

template <int BN>
__global__ void __launch_bounds__(TF_THREADS, 1)
    gemm_tf32_sub_ares_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tBh,
                              const __grid_constant__ CUtensorMap tBl, const __grid_constant__ CUtensorMap tC,
                              const TfParams p) {
  if (p.gate != nullptr && __ldcg(p.gate) == 0) return;
  using Cfg = TfAresCfg<BN>;
  constexpr int BS = Cfg::BSTAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sBst = smem;                                           // [BS][B hi | B lo]
  uint8_t* sAst = sBst + BS * Cfg::BSTAGE_BYTES;                  // [2][A slab]
  float* sC = reinterpret_cast<float*>(sAst + Cfg::ASTAGES * Cfg::A_BYTES);  // [TF_CSLOTS][32][128]
  uint64_t* bfull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sC) + Cfg::C_BYTES);
  uint64_t* bempty = bfull + BS;
  uint64_t* afull = bempty + BS;       // [2] A slab landed
  uint64_t* aempty = afull + 2;        // [2] A slab read by the 128 splitters
  uint64_t* a_ready = aempty + 2;      // A row block in TMEM (128 splitters)
  uint64_t* a_free = a_ready + 1;      // MMAs done with the row block (tcgen05.commit)
  uint64_t* acc_full = a_free + 1;     // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint64_t* cfull = acc_empty + 2;     // [TF_CSLOTS]
  uint64_t* cdone = cfull + TF_CSLOTS; // [TF_CSLOTS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cdone + TF_CSLOTS);
  double* red = reinterpret_cast<double*>(tmem_slot + 2);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int u0, u1;
  tf_ares_range(p, u0, u1);
  const int nkt = p.nkt;  // <= 4
  auto tile_m0 = [&](int u) { return (u / p.tiles_n) * TF_BM; };
  auto tile_n0 = [&](int u) { return (u % p.tiles_n) * BN; };

  if (tid == 0) {
    tma_prefetch_desc(&tA);
    tma_prefetch_desc(&tBh);
    tma_prefetch_desc(&tBl);
    for (int s = 0; s < BS; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 128);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    mbar_init(a_ready, 128);
    mbar_init(a_free, 1);
    for (int s = 0; s < TF_CSLOTS; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cdone[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer: A slabs per row block, B per tile
    if (lane == 0) {
      int jb = 0, ja = 0, prev_m = -1;
      for (int u = u0; u < u1; ++u) {
        const int m0 = tile_m0(u), n0 = tile_n0(u);
        if (m0 != prev_m) {
          for (int s = 0; s < nkt; ++s, ++ja) {
            const int slot = ja & 1;
            if (ja >= 2) mbar_wait(&aempty[slot], ((ja >> 1) - 1) & 1);
            uint8_t* sa = sAst + slot * Cfg::A_BYTES;
            mbar_arrive_expect_tx(&afull[slot], Cfg::A_BYTES);
            if (p.a3d) {
              tma_load_3d(sa, &tA, &afull[slot], 0, s * TF_BK, m0 / 32);
            } else {
#pragma unroll
              for (int c = 0; c < TF_BM / 32; ++c) tma_load_2d(sa + c * 4096, &tA, &afull[slot], m0 + 32 * c, s * TF_BK);
            }
          }
          prev_m = m0;
        }
        for (int kt = 0; kt < nkt; ++kt, ++jb) {
          const int slot = jb % BS;
          if (jb >= BS) mbar_wait(&bempty[slot], ((jb / BS) - 1) & 1);
          uint8_t* sb = sBst + slot * Cfg::BSTAGE_BYTES;
          mbar_arrive_expect_tx(&bfull[slot], 2 * Cfg::B_BYTES);
          tf_load_b<0, BN>(&tBh, sb, &bfull[slot], n0, kt * TF_BK, p.b3d);
          tf_load_b<0, BN>(&tBl, sb + Cfg::B_BYTES, &bfull[slot], n0, kt * TF_BK, p.b3d);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_ts = tf32_idesc<BN>(0, 1);  // A K-major in TMEM, B MN-major
      int jb = 0, c = 0, r = 0, prev_m = -1;
      for (int u = u0; u < u1; ++u) {
        const int m0 = tile_m0(u);
        if (m0 != prev_m) {
          mbar_wait(a_ready, r & 1);
          ++r;
          prev_m = m0;
        }
        const int b = c & 1;
        if (c >= 2) mbar_wait(&acc_empty[b], ((c >> 1) - 1) & 1);
        const uint32_t tacc = tmem_base + static_cast<uint32_t>(b * BN);
        for (int kt = 0; kt < nkt; ++kt, ++jb) {
          const int slot = jb % BS;
          mbar_wait(&bfull[slot], (jb / BS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t b_hi = smem_u32(sBst + slot * Cfg::BSTAGE_BYTES);
          const uint64_t dBh = umma_desc(b_hi, 4096u, 512u, 1u), dBl = umma_desc(b_hi + Cfg::B_BYTES, 4096u, 512u, 1u);
          const uint32_t ta = tmem_base + static_cast<uint32_t>(Cfg::A_TMEM_COL + 64 * kt);
#pragma unroll
          for (int kk = 0; kk < TF_BK / 8; ++kk) {
            const uint64_t adv = static_cast<uint64_t>(kk) * 64u;
            const uint32_t tah = ta + 8 * kk, tal = ta + 32 + 8 * kk;
            umma_tf32_ts(tacc, tah, dBh + adv, idesc_ts, (kt > 0 || kk > 0) ? 1u : 0u);
            umma_tf32_ts(tacc, tah, dBl + adv, idesc_ts, 1u);
            umma_tf32_ts(tacc, tal, dBh + adv, idesc_ts, 1u);
          }
          umma_commit(&bempty[slot]);
        }
        umma_commit(&acc_full[b]);
        ++c;
        if (u + 1 == u1 || tile_m0(u + 1) != m0) umma_commit(a_free);
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ splitters: A row block -> TMEM
    const int quad = warp & 3, rr = quad * 32 + lane;
    int ja = 0, r = 0, prev_m = -1;
    for (int u = u0; u < u1; ++u) {
      const int m0 = tile_m0(u);
      if (m0 == prev_m) continue;
      prev_m = m0;
      if (r > 0) {
        mbar_wait(a_free, (r - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      for (int s = 0; s < nkt; ++s, ++ja) {
        const int slot = ja & 1;
        mbar_wait(&afull[slot], (ja >> 1) & 1);
        const uint8_t* sa = sAst + slot * Cfg::A_BYTES;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < TF_BK; ++k) {
          const uint32_t off = (rr >> 5) * 4096 + k * 128 + ((((rr & 31) >> 3) ^ (k & 3)) << 5) + ((rr & 7) << 2);
          const float x = *reinterpret_cast<const float*>(sa + off);
          const float h = tf32_rna(x);
          hi[k] = __float_as_uint(h);
          lo[k] = __float_as_uint(x - h);
        }
        mbar_arrive(&aempty[slot]);
        const uint32_t ta = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                            static_cast<uint32_t>(Cfg::A_TMEM_COL + 64 * s);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(a_ready);
      ++r;
    }
  } else if (warp < 10) {
    // ------------------------------------------------------------ epilogue: C -= acc, sum of squares
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    double sq = 0.0;
    int c = 0, cs = 0;
    for (int u = u0; u < u1; ++u, ++c) {
      const int m0 = tile_m0(u), n0 = tile_n0(u);
      const int b = c & 1;
      mbar_wait(&acc_full[b], (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float acc[BN];
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(trow + static_cast<uint32_t>(b * BN + c0), v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[c0 + i] = __uint_as_float(v[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acc_empty[b]);
      const int ncols = m0 + row < p.M ? min(BN, p.N - n0) : 0;
#pragma unroll
      for (int sub = 0; sub < BN / TF_CSUB; ++sub, ++cs) {
        const int slot = cs % TF_CSLOTS;
        mbar_wait(&cfull[slot], (cs / TF_CSLOTS) & 1);
        float* cb = sC + slot * (TF_BM * TF_CSUB);
        float s4[4] = {0.f, 0.f, 0.f, 0.f};  // FP32 over 8 entries, then FP64 (R18)
#pragma unroll
        for (int i = 0; i < TF_CSUB; ++i) {
          const float x = cb[i * TF_BM + row] - acc[sub * TF_CSUB + i];
          cb[i * TF_BM + row] = x;
          const float xv = sub * TF_CSUB + i < ncols ? x : 0.f;
          s4[i & 3] = fmaf(xv, xv, s4[i & 3]);
        }
        sq += (static_cast<double>(s4[0]) + static_cast<double>(s4[1])) +
              (static_cast<double>(s4[2]) + static_cast<double>(s4[3]));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&cdone[slot]);
      }
    }
    if (p.norm_partials != nullptr) {
      sq = warp_sum(sq);
      if (lane == 0) red[warp - 6] = sq;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 6 && lane == 0) p.norm_partials[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
    }
  } else {
    // ------------------------------------------------------------ C warp: load / store the C ring
    if (lane == 0) {
      tma_prefetch_desc(&tC);
      int cm[TF_CSLOTS] = {}, cn[TF_CSLOTS] = {};
      int cs = 0;
      auto store = [&](int t) {
        const int slot = t % TF_CSLOTS;
        mbar_wait(&cdone[slot], (t / TF_CSLOTS) & 1);
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                         reinterpret_cast<uint64_t>(&tC)),
                     "r"(smem_u32(sC + slot * (TF_BM * TF_CSUB))), "r"(cm[slot]), "r"(cn[slot])
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      };
      for (int u = u0; u < u1; ++u) {
        for (int sub = 0; sub < BN / TF_CSUB; ++sub, ++cs) {
          const int slot = cs % TF_CSLOTS;
          if (cs >= TF_CSLOTS) {
            store(cs - TF_CSLOTS);
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          cm[slot] = tile_m0(u);
          cn[slot] = tile_n0(u) + sub * TF_CSUB;
          mbar_arrive_expect_tx(&cfull[slot], Cfg::CSUB_BYTES);
          tma_load_2d(sC + slot * (TF_BM * TF_CSUB), &tC, &cfull[slot], cm[slot], cn[slot]);
        }
      }
      for (int t = cs - TF_CSLOTS < 0 ? 0 : cs - TF_CSLOTS; t < cs; ++t) store(t);
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
  }
}

}  // namespace qbk
