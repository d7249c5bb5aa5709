// Counter-based Gaussian generator of the K4 sketches (gaussian.cu SIMT,
// gaussian_tc.cu tcgen05).  Extension: the reference rejects the "gaussian"
// family (pkg/src/levsketch/sketch.py:38-41, 74-75); BASELINE configs 1 and 5
// ask for S with i.i.d. N(0, 1/k) entries.
//
// Definition (restated bit-for-bit by oracle/levsketch_oracle.py gaussian_z):
//   Z[j, i] (sketch row j, global input row i) is the bf16 value with bits
//       MAG[w & 0x7FFF] | (w & 0x8000),
//   w = 16-bit field (j & 3) of h = mix64(key + phi * ((i << 24) | (j >> 2))),
//   mix64 the splitmix64 finaliser (the reference's _mix64, sketch.py:141-148),
//   phi = 0x9E3779B97F4A7C15, key = (seed_hi ^ 'GAUS') << 32 | seed_lo — i.e.
//   splitmix64 output number ((i << 24) | (j >> 2)) of the seeded stream, one
//   64-bit hash per 4 entries.  Bit 15 of w is the sign, bits 0-14 a uniform
//   level L, and MAG[L] = bf16_rn(Phi^-1(1/2 + (L + 1/2) / 65536)) — the
//   inverse normal CDF of a 16-bit uniform (65536 equiprobable levels,
//   |z| <= 4.33).  Every entry, whatever its row or column, has the same
//   distribution: N(0, 1) quantised to 16 bits, then rounded to bf16; entries
//   are independent up to the hash.  SX = Z X / sqrt(k).
//   MAG is built on the host (bisection on erfc, float64, the oracle's steps)
//   and held as bf16 bit patterns (64 KB); lvsk_gaussian_tables exports it so
//   a CPU test pins the two.  Cost per entry: its quarter of a mix64 (the
//   counter advances by constant adds), a field extract, one 16-bit shared
//   load (random bank: ~3.5 wavefronts per 32 reads) and one LOP3.
#pragma once

#include "common.cuh"

namespace lvsk {

constexpr uint32_t GAUSS_KEY_XOR = 0x47415553u;  // "GAUS"
constexpr int GT_LEVELS = 32768;                 // |z| levels (bf16 bit patterns)
constexpr uint64_t GAUSS_PHI = 0x9E3779B97F4A7C15ull;
constexpr int64_t GAUSS_MAX_K = int64_t{1} << 26;   // j >> 2 < 2^24
constexpr uint64_t GAUSS_MAX_ROW = uint64_t{1} << 40;  // i << 24 < 2^64

const uint16_t* gaussian_table_device();  // device copy for the current device (built on first use)
void gaussian_table_host(uint16_t* out);  // GT_LEVELS bf16 bit patterns

__host__ __device__ __forceinline__ uint64_t gauss_key(uint64_t seed) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(seed >> 32) ^ GAUSS_KEY_XOR) << 32) |
         static_cast<uint32_t>(seed);
}

// counter value of (input row i, quad t = j >> 2); consecutive quads differ
// by GAUSS_PHI, consecutive rows by GAUSS_PHI << 24
__device__ __forceinline__ uint64_t gauss_ctr(uint64_t key, uint64_t i, uint32_t t) {
  return key + GAUSS_PHI * ((i << 24) | t);
}

// bf16 bits (low 16) of entry m (= j & 3) of hash h
__device__ __forceinline__ uint32_t gauss_bits(uint64_t h, int m, const uint16_t* __restrict__ mag) {
  const uint32_t w = static_cast<uint32_t>(h >> (16 * m));
  return static_cast<uint32_t>(mag[w & 0x7FFFu]) | (w & 0x8000u);
}

__device__ __forceinline__ float bf16_bits_to_float(uint32_t b) { return __uint_as_float(b << 16); }

// Entries Z[4t .. 4t+3, i] as floats (exact bf16 values).
__device__ __forceinline__ void gaussian4(uint64_t key, uint64_t i, uint32_t t, const uint16_t* __restrict__ mag,
                                          float (&z)[4]) {
  const uint64_t h = mix64(gauss_ctr(key, i, t));
#pragma unroll
  for (int m = 0; m < 4; ++m) z[m] = bf16_bits_to_float(gauss_bits(h, m, mag));
}

__device__ __forceinline__ float bf16_rn(float z) { return __bfloat162float(__float2bfloat16_rn(z)); }

__device__ __forceinline__ void load_gaussian_table(uint16_t* dst, const uint16_t* __restrict__ src) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (int e = threadIdx.x; e < GT_LEVELS * 2 / 16; e += blockDim.x) d[e] = s[e];
}

// ---- tensor-core path (gaussian_tc.cu) -------------------------------------
struct GaussTcPlan {
  int ns, ktiles, dslabs;
  int64_t splits, rows_per_split;
  int64_t period;  // input row r is global row row0 + r mod period (stacked planes; = n otherwise)
};
GaussTcPlan plan_gauss_tc(int64_t n, int64_t d, int64_t k);
bool gaussian_tc_ok(const void* X, int64_t n, int64_t d, int64_t ldx, int64_t k);
// fp32 partials [splits][k][d] of Z X (unscaled)
int32_t gaussian_tc_bf16(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, int64_t k, uint64_t row0,
                         uint64_t key, const GaussTcPlan& p, float* partial, cudaStream_t st);

}  // namespace lvsk
