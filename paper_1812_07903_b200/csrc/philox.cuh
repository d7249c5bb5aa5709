// Counter-based Gaussian generator of the K4 sketches (gaussian.cu SIMT,
// gaussian_tc.cu tcgen05).  Extension: the reference rejects the "gaussian"
// family (pkg/src/levsketch/sketch.py:38-41, 74-75); BASELINE configs 1 and 5
// ask for it.
//
// Definition (restated bit-for-bit by oracle/levsketch_oracle.py gaussian_z):
//   Z[8q + m, i] = TAB[32 b + c]  (i = global input row, m = 0..7), where
//     b = byte m of h = mix64(key + phi * ((i << 24) | (q << 1))),
//     c = (i >> 1) & 31,
//   mix64 the splitmix64 finaliser (the reference's _mix64, sketch.py:141-148),
//   phi = 0x9E3779B97F4A7C15, key = (seed_hi ^ 'GAUS') << 32 | seed_lo — i.e.
//   splitmix64 output number (i << 24 | q << 1) of the seeded stream, one
//   64-bit hash per 8 entries.  TAB[32 b + c], b < 128, is positive level
//   L = 32 b + c of an 8192-level equiprobable Gaussian, Phi^-1(1/2 + (L + 1/2)
//   / 8192), each column class c rescaled to unit second moment and bf16-
//   rounded; TAB[32 (b + 128) + c] = -TAB[32 b + c] (so every entry is
//   symmetric).  The class is the TC kernel's lane (lanes own input rows 2l,
//   2l+1 of a 64-row stage), so a warp's 32 table reads hit 32 different banks
//   and an entry costs a byte permute, an address and one shared load — ~4
//   SASS instructions including its share of the hash (the round-1 Philox +
//   Box-Muller definition cost ~40 and a 12-bit-indexed table ~3.5 shared
//   wavefronts per 32 reads; both bounded K4-TC below the tensor rate).
//   Built on the host (bisection on erfc, float64) with the same steps as the
//   oracle; lvsk_gaussian_tables exports the table so a CPU test pins the two.
#pragma once

#include "common.cuh"

namespace lvsk {

struct Philox {
  static constexpr uint32_t KEY_XOR = 0x47415553u;  // "GAUS"
};

constexpr int GT_SIZE = 8192;  // TAB[256 byte values][32 column classes] (bf16-valued floats)

const float* gaussian_table_device();  // device copy (built on first use)
void gaussian_table_host(float* out);  // GT_SIZE floats

// Entries Z[8q .. 8q+7, i] (exact bf16 values).
__device__ __forceinline__ void gaussian8(uint64_t i, uint32_t q, uint32_t k0, uint32_t k1,
                                          const float* __restrict__ tab, float (&z)[8]) {
  constexpr uint64_t PHI = 0x9E3779B97F4A7C15ull;
  const uint64_t key = (static_cast<uint64_t>(k1) << 32) | k0;
  const uint64_t h = mix64(key + PHI * ((i << 24) | (static_cast<uint64_t>(q) << 1)));
  const uint32_t w0 = static_cast<uint32_t>(h), w1 = static_cast<uint32_t>(h >> 32);
  const float* tc = tab + ((i >> 1) & 31u);  // this column class's bank
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    z[m] = tc[__byte_perm(w0, 0u, 0x4440u | m) * 32];
    z[4 + m] = tc[__byte_perm(w1, 0u, 0x4440u | m) * 32];
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
