// Counter-based Gaussian generator of the K4 sketches (gaussian.cu SIMT,
// gaussian_tc.cu tcgen05).  Extension: the reference rejects the "gaussian"
// family (pkg/src/levsketch/sketch.py:38-41, 74-75); BASELINE configs 1 and 5
// ask for it.
//
// Definition (restated bit-for-bit by oracle/levsketch_oracle.py gaussian_z):
//   Z[j, i], j = 8q + 2h + e (i = global input row): w = word h of
//   Philox4x32-10 (Random123) with counter (i_lo, i_hi, q, 0) and key
//   (seed_lo, seed_hi ^ 0x47415553); v1 = w & 0xFFFF, v2 = w >> 16;
//   radius  u1 = (v1 + 1/2) 2^-16 = 2^E f (f in [1,2), f0 = f truncated to 7
//           fraction bits, idx = those 7 bits), y = (f - f0) INV[idx],
//           ln u1 = E ln2 + (LN[idx] + (y - y*y/2)),  r = sqrt(-2 ln u1);
//   angle   v2 = 256 a + b,  (c, s) = (cos, sin)(2 pi a / 256 + 2 pi (b+1/2) / 2^16)
//           by the angle-addition formulas over the tables CSA[a], CSB[b];
//   Z = bf16_rn(r c) for e = 0, bf16_rn(r s) for e = 1.
// Every step is one IEEE fp32 operation (no FMA contraction: __fmul_rn /
// __fadd_rn) or an exact integer / table operation, so host numpy reproduces
// each entry exactly; the 1280-float table is built once on the host
// (lvsk_gaussian_tables exports it so the CPU tests pin it to the oracle's).
// One Philox call yields 8 entries; the transform is ~20 SASS instructions per
// entry (a division / polynomial Box-Muller costs ~110).
#pragma once

#include "common.cuh"

namespace lvsk {

struct Philox {
  static constexpr uint32_t KEY_XOR = 0x47415553u;  // "GAUS"
  static constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  static constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
};

// table layout (floats): INV[128] | LN[128] | CSA[256] (cos, sin) | CSB[256] (cos, sin)
constexpr int GT_INV = 0, GT_LN = 128, GT_CSA = 256, GT_CSB = 768, GT_SIZE = 1280;

const float* gaussian_table_device();  // device copy (built on first use)
void gaussian_table_host(float* out);  // GT_SIZE floats

__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += Philox::W0;
      k1 += Philox::W1;
    }
    const uint32_t hi0 = __umulhi(Philox::M0, c[0]), lo0 = Philox::M0 * c[0];
    const uint32_t hi1 = __umulhi(Philox::M1, c[2]), lo1 = Philox::M1 * c[2];
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
  }
}

// The pair (r cos, r sin) of one Philox word; tab = the GT_SIZE table.
__device__ __forceinline__ void box_muller16(uint32_t w, const float* __restrict__ tab, float& z0, float& z1) {
  const uint32_t v1 = w & 0xFFFFu, v2 = w >> 16;
  // exact int -> float via the 2^23 magic (keeps the XU free): v1 + 1/2, then * 2^-16
  const float v1h = __fsub_rn(__uint_as_float(0x4B000000u | v1), 8388607.5f);
  const float u1 = __fmul_rn(v1h, 1.52587890625e-05f);
  const uint32_t bits = __float_as_uint(u1);
  const float exf = __fsub_rn(__uint_as_float(0x4B000000u | (bits >> 23)), 8388735.0f);  // E = biased - 127
  const uint32_t idx = (bits >> 16) & 0x7Fu;
  const float f = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);
  const float f0 = __uint_as_float((bits & 0x007F0000u) | 0x3F800000u);
  const float y = __fmul_rn(__fsub_rn(f, f0), tab[GT_INV + idx]);
  const float t = __fsub_rn(y, __fmul_rn(__fmul_rn(y, y), 0.5f));
  const float lnf = __fadd_rn(tab[GT_LN + idx], t);
  const float lnu = __fadd_rn(__fmul_rn(exf, 0.693147182464599609375f), lnf);
  const float r = __fsqrt_rn(__fmul_rn(lnu, -2.0f));
  const float2 a = reinterpret_cast<const float2*>(tab + GT_CSA)[v2 >> 8];
  const float2 b = reinterpret_cast<const float2*>(tab + GT_CSB)[v2 & 0xFFu];
  const float c = __fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
  const float s = __fadd_rn(__fmul_rn(a.y, b.x), __fmul_rn(a.x, b.y));
  z0 = __fmul_rn(r, c);
  z1 = __fmul_rn(r, s);
}

// Entries Z[8q .. 8q+7, i] (fp32 before the bf16 rounding).
__device__ __forceinline__ void gaussian8(uint64_t i, uint32_t q, uint32_t k0, uint32_t k1,
                                          const float* __restrict__ tab, float (&z)[8]) {
  uint32_t c[4] = {static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), q, 0u};
  philox4x32_10(c, k0, k1);
#pragma unroll
  for (int h = 0; h < 4; ++h) box_muller16(c[h], tab, z[2 * h], z[2 * h + 1]);
}

__device__ __forceinline__ float bf16_rn(float z) { return __bfloat162float(__float2bfloat16_rn(z)); }

__device__ __forceinline__ void load_gaussian_table(float* dst, const float* __restrict__ src) {
  for (int e = threadIdx.x; e < GT_SIZE; e += blockDim.x) dst[e] = src[e];
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
