// Counter-based Gaussian generator of the K4 sketches (gaussian.cu SIMT,
// gaussian_tc.cu tcgen05).  Extension: the reference rejects the "gaussian"
// family (pkg/src/levsketch/sketch.py:38-41, 74-75); BASELINE configs 1 and 5
// ask for it.
//
// Definition (restated bit-for-bit by oracle/levsketch_oracle.py gaussian_z):
//   Z[8q + m, i] (i = global input row, m = 0..7) = TAB[f >> 4], f = the
//   16-bit field (m & 3) of the 64-bit word h_(m >> 2), where
//     h_w = mix64(key + phi * ((i << 24) | (q << 1) | w)),
//   mix64 the splitmix64 finaliser (the reference's _mix64, sketch.py:141-148),
//   phi = 0x9E3779B97F4A7C15 and key = (seed_hi ^ 'GAUS') << 32 | seed_lo —
//   i.e. splitmix64 output number (i << 24 | q << 1 | w) of the seeded
//   stream.  TAB is a 4096-level equiprobable Gaussian: TAB[j] =
//   bf16_rn(float(t_j / sqrt(mean t^2))), t_j = Phi^-1((j + 1/2) / 4096) by
//   bisection on erfc (antisymmetric: t_4095-j = -t_j), so E Z = 0 and
//   E Z^2 = 1 up to the bf16 rounding, tails at +-3.8 sigma.  Built once on
//   the host (lvsk_gaussian_tables exports it so the CPU tests pin it to the
//   oracle's).  Cost: two 64-bit hashes per 8 entries + one table read per
//   entry (~8 SASS instructions / entry; the earlier Philox4x32-10 + Box-Muller
//   definition cost ~40 and bounded K4-TC below the tensor-core rate).
#pragma once

#include "common.cuh"

namespace lvsk {

struct Philox {
  static constexpr uint32_t KEY_XOR = 0x47415553u;  // "GAUS"
};

constexpr int GT_SIZE = 4096;  // TAB: 4096 equiprobable Gaussian levels (bf16-valued floats)

const float* gaussian_table_device();  // device copy (built on first use)
void gaussian_table_host(float* out);  // GT_SIZE floats

// Entries Z[8q .. 8q+7, i] (exact bf16 values).
__device__ __forceinline__ void gaussian8(uint64_t i, uint32_t q, uint32_t k0, uint32_t k1,
                                          const float* __restrict__ tab, float (&z)[8]) {
  constexpr uint64_t PHI = 0x9E3779B97F4A7C15ull;
  const uint64_t key = (static_cast<uint64_t>(k1) << 32) | k0;
  const uint64_t base = key + PHI * ((i << 24) | (static_cast<uint64_t>(q) << 1));
  const uint64_t h0 = mix64(base), h1 = mix64(base + PHI);
  const uint32_t w[4] = {static_cast<uint32_t>(h0), static_cast<uint32_t>(h0 >> 32), static_cast<uint32_t>(h1),
                         static_cast<uint32_t>(h1 >> 32)};
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    z[2 * m] = tab[(w[m] >> 4) & 0xFFFu];
    z[2 * m + 1] = tab[w[m] >> 20];
  }
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
