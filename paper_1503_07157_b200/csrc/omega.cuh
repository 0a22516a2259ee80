// Ω_i generator (K1): counter-based Philox4x32-10 + Box-Muller, DESIGN.md §3.3.
//
// The paper draws Ω_i = randn(n, b), slices of one n x ℓ Gaussian
// (eq. (OmegaBlock), :479-484).  Reading R14/R15: column c is a pure function of
// (seed, c), so every block size, the unblocked scheme and every column sharding of A see
// the same Ω.  Only correctly rounded +, -, *, /, sqrt (the __d*_rn intrinsics, which nvcc
// never contracts into fma) are used, in the order the specification fixes, so the result
// is bit-identical to any other implementation of the specification.
#pragma once
#include "common.cuh"

namespace qbk {

struct OmegaConsts {
  double log_c[12];   // log_c[k] = RN(2/(2k+1)), k = 1..11 (index 0 unused); set on the host
  double log_c12;     // RN(2/25)
};

__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                              uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
}

// ln(x), x in (0, 1]: x = f 2^e with f in (sqrt2/2, sqrt2]; s = (f-1)/(f+1), z = s^2;
// ln x = e ln2_hi + (e ln2_lo + (2s + (s z) p)), p = 2/3 + 2z/5 + ... + 2z^11/25.
__device__ __forceinline__ double spec_log(double x, const OmegaConsts& K) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
  const int eraw = static_cast<int>((bits >> 52) & 0x7ffull);
  double f = __longlong_as_double(static_cast<long long>((bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
  double e = static_cast<double>(eraw - 1023);
  if (f > 0x1.6a09e667f3bcdp+0) {
    f = __dmul_rn(f, 0.5);
    e = __dadd_rn(e, 1.0);
  }
  const double s = __ddiv_rn(__dsub_rn(f, 1.0), __dadd_rn(f, 1.0));
  const double z = __dmul_rn(s, s);
  double p = K.log_c12;
#pragma unroll
  for (int k = 11; k >= 1; --k) p = __dadd_rn(__dmul_rn(p, z), K.log_c[k]);
  double t = __dmul_rn(s, z);
  t = __dmul_rn(t, p);
  const double lf = __dadd_rn(__dmul_rn(2.0, s), t);
  return __dadd_rn(__dmul_rn(e, 0x1.62e42fefa3800p-1), __dadd_rn(__dmul_rn(e, 0x1.ef35793c76730p-45), lf));
}

// (sin(pi t), cos(pi t)) for t in [0, 2): j = rint(2t), r = t - j/2, Taylor in r^2.
__device__ __forceinline__ void spec_sincospi(double t, double& sn_out, double& cn_out) {
  // cs[k] = RN((-1)^k pi^(2k+1)/(2k+1)!), cc[k] = RN((-1)^k pi^(2k)/(2k)!)
  const double cs[11] = {0x1.921fb54442d18p+1,  -0x1.4abbce625be53p+2, 0x1.466bc6775aae2p+1,
                         -0x1.32d2cce62bd86p-1, 0x1.50783487ee782p-4,  -0x1.e3074fde8871fp-8,
                         0x1.e8f434d018d63p-12, -0x1.6fadb9f155744p-16, 0x1.aaec32af93359p-21,
                         -0x1.8a404211f9547p-26, 0x1.2877020d52cf0p-31};
  const double cc[11] = {0x1.0000000000000p+0,  -0x1.3bd3cc9be45dep+2, 0x1.03c1f081b5ac4p+2,
                         -0x1.55d3c7e3cbffap+0, 0x1.e1f506891babbp-3,  -0x1.a6d1f2a204a8cp-6,
                         0x1.f9d38a3763cc3p-10, -0x1.b6e24f44b128fp-14, 0x1.20c62c2f2d7f5p-18,
                         -0x1.2a0c591af8314p-23, 0x1.ef6e308d6d1c4p-29};
  const double j = rint(__dmul_rn(2.0, t));
  const double r = __dsub_rn(t, __dmul_rn(0.5, j));
  const double r2 = __dmul_rn(r, r);
  double S = cs[10], C = cc[10];
#pragma unroll
  for (int k = 9; k >= 0; --k) {
    S = __dadd_rn(__dmul_rn(S, r2), cs[k]);
    C = __dadd_rn(__dmul_rn(C, r2), cc[k]);
  }
  const double sn = __dmul_rn(r, S), cn = C;
  const int q = static_cast<int>(j) & 3;
  sn_out = q == 0 ? sn : q == 1 ? cn : q == 2 ? -sn : -cn;
  cn_out = q == 0 ? cn : q == 1 ? -sn : q == 2 ? -cn : sn;
}

// Gaussian pair (rows 2p, 2p+1) of column c.
__device__ __forceinline__ void gaussian_pair(uint64_t seed, uint64_t p, uint64_t c, const OmegaConsts& K,
                                              double& even, double& odd) {
  uint32_t x = static_cast<uint32_t>(p), y = static_cast<uint32_t>(p >> 32);
  uint32_t z = static_cast<uint32_t>(c), w = static_cast<uint32_t>(c >> 32);
  philox4x32_10(x, y, z, w, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const uint64_t a = ((static_cast<uint64_t>(x) << 32) | y) >> 11;
  const uint64_t bb = ((static_cast<uint64_t>(z) << 32) | w) >> 11;
  const double u1 = __dmul_rn(__ull2double_rn(a + 1), 0x1p-53);
  const double u2 = __dmul_rn(__ull2double_rn(bb), 0x1p-53);
  const double rho = __dsqrt_rn(__dmul_rn(-2.0, spec_log(u1, K)));
  double sn, cn;
  spec_sincospi(__dmul_rn(2.0, u2), sn, cn);
  even = __dmul_rn(rho, cn);
  odd = __dmul_rn(rho, sn);
}

// out[(r - row0)*ldo + (c - col0)] = Ω(r, c) for r in [row0, row1), c in [col0, col0 + w).
// T = double with Round32 = true stores RN_32(Ω) widened back to FP64 (the FP32 path's Ω,
// DESIGN.md §3.3 rule 7, for FP64 arithmetic on FP32 data).
template <typename T, bool Round32 = false>
__global__ void __launch_bounds__(256) omega_kernel(uint64_t seed, int64_t row0, int64_t row1, int64_t col0,
                                                    int64_t w, T* __restrict__ out, int64_t ldo,
                                                    const OmegaConsts K) {
  const int64_t p0 = row0 >> 1;
  const int64_t npairs = ((row1 - 1) >> 1) - p0 + 1;
  const int64_t total = npairs * w;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pi = idx / w, ci = idx - pi * w;
    const int64_t p = p0 + pi;
    double ev, od;
    gaussian_pair(seed, static_cast<uint64_t>(p), static_cast<uint64_t>(col0 + ci), K, ev, od);
    if (Round32) {
      ev = static_cast<double>(static_cast<float>(ev));
      od = static_cast<double>(static_cast<float>(od));
    }
    const int64_t r_even = 2 * p, r_odd = 2 * p + 1;
    if (r_even >= row0 && r_even < row1) out[(r_even - row0) * ldo + ci] = static_cast<T>(ev);
    if (r_odd >= row0 && r_odd < row1) out[(r_odd - row0) * ldo + ci] = static_cast<T>(od);
  }
}

}  // namespace qbk
