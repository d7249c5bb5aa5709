// Counter-based Gaussian generator of the K4 sketches (gaussian.cu SIMT,
// gaussian_tc.cu tcgen05).  Extension: the reference rejects the "gaussian"
// family (pkg/src/levsketch/sketch.py:38-41, 74-75); BASELINE configs 1 and 5
// ask for it.  Z[j, i] (j < k sketch row, i global input row) is a
// bf16-rounded standard normal from Philox4x32-10 (Random123) with counter
// (i_lo, i_hi, j >> 2, 0) and key (seed_lo, seed_hi ^ 0x47415553), followed by
// Box-Muller whose log / sin / cos use only IEEE fp32 add/mul/div/sqrt (no FMA
// contraction), so the CPU oracle (oracle/levsketch_oracle.py: gaussian_z)
// reproduces every entry bit-for-bit.
#pragma once

#include "common.cuh"

namespace lvsk {

struct Philox {
  static constexpr uint32_t KEY_XOR = 0x47415553u;  // "GAUS"
  static constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  static constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
};

__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += Philox::W0;
      k1 += Philox::W1;
    }
    const uint64_t p0 = static_cast<uint64_t>(Philox::M0) * c[0];
    const uint64_t p1 = static_cast<uint64_t>(Philox::M1) * c[2];
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
  }
}

__device__ __forceinline__ float u01(uint32_t x) {
  return __fmul_rn(__uint2float_rn(((x >> 9) << 1) | 1u), 5.9604644775390625e-08f);  // * 2^-24
}

__device__ __forceinline__ float horner(float x2, float acc, float c) { return __fadd_rn(__fmul_rn(acc, x2), c); }

__device__ __forceinline__ float log_f32(float u) {
  uint32_t bits = __float_as_uint(u);
  int e = static_cast<int>((bits >> 23) & 0xFFu) - 127;
  uint32_t mb = (bits & 0x7FFFFFu) | 0x3F800000u;
  if (mb > 0x3FB504F3u) {
    mb -= 0x00800000u;
    e += 1;
  }
  const float m = __uint_as_float(mb);
  const float t = __fdiv_rn(__fsub_rn(m, 1.0f), __fadd_rn(m, 1.0f));
  const float t2 = __fmul_rn(t, t);
  float p = static_cast<float>(2.0 / 9.0);
  p = horner(t2, p, static_cast<float>(2.0 / 7.0));
  p = horner(t2, p, static_cast<float>(2.0 / 5.0));
  p = horner(t2, p, static_cast<float>(2.0 / 3.0));
  p = horner(t2, p, 2.0f);
  return __fadd_rn(__fmul_rn(static_cast<float>(e), static_cast<float>(0.6931471805599453)), __fmul_rn(t, p));
}

__device__ __forceinline__ void sincos_turns(float v, float& cs, float& sn) {
  const float f4 = __fmul_rn(v, 4.0f);
  const float q = floorf(f4);
  const float f = __fsub_rn(f4, q);
  const int qi = static_cast<int>(q);
  const float x = __fmul_rn(f, static_cast<float>(3.141592653589793 / 2.0));
  const float x2 = __fmul_rn(x, x);
  float s = static_cast<float>(-1.0 / 39916800.0);
  s = horner(x2, s, static_cast<float>(1.0 / 362880.0));
  s = horner(x2, s, static_cast<float>(-1.0 / 5040.0));
  s = horner(x2, s, static_cast<float>(1.0 / 120.0));
  s = horner(x2, s, static_cast<float>(-1.0 / 6.0));
  s = horner(x2, s, 1.0f);
  s = __fmul_rn(s, x);
  float c = static_cast<float>(1.0 / 479001600.0);
  c = horner(x2, c, static_cast<float>(-1.0 / 3628800.0));
  c = horner(x2, c, static_cast<float>(1.0 / 40320.0));
  c = horner(x2, c, static_cast<float>(-1.0 / 720.0));
  c = horner(x2, c, static_cast<float>(1.0 / 24.0));
  c = horner(x2, c, -0.5f);
  c = horner(x2, c, 1.0f);
  switch (qi) {
    case 0: cs = c; sn = s; break;
    case 1: cs = -s; sn = c; break;
    case 2: cs = -c; sn = -s; break;
    default: cs = s; sn = -c; break;
  }
}

__device__ __forceinline__ float bf16_rn(float z) {
  uint32_t b = __float_as_uint(z);
  b = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  return __uint_as_float(b);
}

// Four consecutive sketch rows j = 4q..4q+3 of column i.
__device__ __forceinline__ void gaussian4(uint64_t i, uint32_t q, uint32_t k0, uint32_t k1, float (&z)[4]) {
  uint32_t c[4] = {static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), q, 0u};
  philox4x32_10(c, k0, k1);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float u1 = u01(c[2 * h]), u2 = u01(c[2 * h + 1]);
    const float r = __fsqrt_rn(__fmul_rn(-2.0f, log_f32(u1)));
    float cs, sn;
    sincos_turns(u2, cs, sn);
    z[2 * h] = bf16_rn(__fmul_rn(r, cs));
    z[2 * h + 1] = bf16_rn(__fmul_rn(r, sn));
  }
}

// ---- tensor-core path (gaussian_tc.cu) -------------------------------------
struct GaussTcPlan {
  int ns, ktiles, dslabs;
  int64_t splits, rows_per_split;
};
GaussTcPlan plan_gauss_tc(int64_t n, int64_t d, int64_t k);
bool gaussian_tc_ok(const void* X, int64_t n, int64_t d, int64_t ldx, int64_t k);
// fp32 partials [splits][k][d] of Z X (unscaled)
int32_t gaussian_tc_bf16(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, int64_t k, uint64_t row0,
                         uint32_t k0, uint32_t k1, const GaussTcPlan& p, float* partial, cudaStream_t st);

}  // namespace lvsk
