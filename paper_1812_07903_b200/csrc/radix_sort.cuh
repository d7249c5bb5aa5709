// Stable LSD radix sort of (key, value) pairs — the building block of the
// bucket grouping in K1 (hashed sketch) and of K7 (argsort for make_plan).
//
// Default ("onesweep"): one histogram kernel reads the keys once and counts
// the digits of every pass; then ONE kernel per 8-bit pass: each CTA takes
// the next tile in launch order, ranks its keys stably (__match_any_sync +
// per-warp digit counters; (warp, step, lane) order = index order), finds
// its per-digit global offsets by decoupled look-back over the preceding
// tiles' published counts, and writes its keys as contiguous per-digit runs
// staged through shared memory.  Used for small sorts (<= 2 tiles per SM),
// where launch count dominates; larger sorts use the three-kernel pass (tile
// histogram -> (digit, tile) scan -> scatter), whose per-pass cost beats the
// serial look-back latency at hundreds of tiles.
#pragma once

#include <cstdlib>

#include "common.cuh"

namespace lvsk {
namespace radix {

constexpr int THREADS = 256;
constexpr int ITEMS = 8;
constexpr int TILE = THREADS * ITEMS;  // 2048 keys per tile
constexpr int WARPS = THREADS / 32;
constexpr int WARP_ITEMS = TILE / WARPS;  // 256 contiguous keys per warp
constexpr int RADIX = 256;
constexpr int SCAN_THREADS = 1024;

inline int64_t num_tiles(int64_t n) { return (n + TILE - 1) / TILE; }

template <typename K>
__global__ void __launch_bounds__(THREADS) hist_kernel(const K* __restrict__ keys, int64_t n, int shift,
                                                       uint32_t mask, uint32_t* __restrict__ hist,
                                                       int64_t ntiles) {
  __shared__ uint32_t h[RADIX];
  for (int i = threadIdx.x; i < RADIX; i += THREADS) h[i] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * TILE;
#pragma unroll 4
  for (int j = 0; j < ITEMS; ++j) {
    int64_t i = base + j * THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[static_cast<uint32_t>(keys[i] >> shift) & mask], 1u);
  }
  __syncthreads();
  for (int dg = threadIdx.x; dg < RADIX; dg += THREADS) hist[dg * ntiles + blockIdx.x] = h[dg];
}

// Block-wide exclusive scan of one value per thread (THREADS threads).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* sh_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) sh_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < WARPS ? sh_warp[lane] : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, off);
      if (lane >= off) w += y;
    }
    if (lane < WARPS) sh_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  total = sh_warp[WARPS - 1];
  const uint32_t base = warp ? sh_warp[warp - 1] : 0u;
  __syncthreads();
  return base + x - v;
}

// Row scan: block d turns hist[d][0..ntiles) into its exclusive prefix and
// writes the row total to totals[d] (digit-major layout, one block per digit).
static __global__ void __launch_bounds__(THREADS) scan_rows_kernel(uint32_t* __restrict__ hist, int64_t ntiles,
                                                                   uint32_t* __restrict__ totals) {
  __shared__ uint32_t sh[WARPS];
  uint32_t* row = hist + static_cast<int64_t>(blockIdx.x) * ntiles;
  uint32_t run = 0;
  for (int64_t c0 = 0; c0 < ntiles; c0 += THREADS) {
    const int64_t i = c0 + threadIdx.x;
    const uint32_t v = i < ntiles ? row[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(v, sh, tot);
    if (i < ntiles) row[i] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = run;
}

// vals_in == nullptr means "value = item index" (argsort identity).
// offsets: row-scanned hist (exclusive within each digit row), totals: per-digit
// counts.  Items are ranked stably inside the tile, staged in shared memory in
// digit order and written out as contiguous per-digit runs (coalesced).
template <typename K, typename VIn, typename VOut>
__global__ void __launch_bounds__(THREADS) scatter_kernel(const K* __restrict__ keys_in,
                                                          const VIn* __restrict__ vals_in,
                                                          K* __restrict__ keys_out, VOut* __restrict__ vals_out,
                                                          int64_t n, int shift, uint32_t mask,
                                                          const uint32_t* __restrict__ offsets,
                                                          const uint32_t* __restrict__ totals, int64_t ntiles) {
  static_assert(THREADS == RADIX, "one thread per digit");
  __shared__ uint32_t cnt[WARPS][RADIX];
  __shared__ uint32_t loc_start[RADIX];
  __shared__ uint32_t gbase[RADIX];
  __shared__ uint32_t sh[WARPS];
  __shared__ K keys_s[TILE];
  __shared__ VOut vals_s[TILE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < WARPS * RADIX; i += THREADS) (&cnt[0][0])[i] = 0u;
  __syncthreads();
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * TILE;
  const int64_t base = tile0 + warp * WARP_ITEMS;
  const uint32_t lt = lanemask_lt();
  K k[ITEMS];
  VOut v[ITEMS];
  uint32_t rank[ITEMS];
  uint32_t dg[ITEMS];
  // all loads first (ITEMS independent DRAM requests in flight per thread)
#pragma unroll
  for (int t = 0; t < ITEMS; ++t) {
    const int64_t i = base + t * 32 + lane;
    if (i < n) {
      k[t] = keys_in[i];
      v[t] = vals_in ? static_cast<VOut>(vals_in[i]) : static_cast<VOut>(i);
    }
  }
#pragma unroll
  for (int t = 0; t < ITEMS; ++t) {
    const int64_t i = base + t * 32 + lane;
    const bool valid = i < n;
    uint32_t d = 0xFFFFFFFFu;
    if (valid) d = static_cast<uint32_t>(k[t] >> shift) & mask;
    dg[t] = d;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t before = valid ? cnt[warp][d] : 0u;
    __syncwarp();
    if (valid) {
      rank[t] = before + __popc(peers & lt);
      if (lane == __ffs(peers) - 1) cnt[warp][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: warp offsets inside the tile, tile count, local and global starts
  const int dd = threadIdx.x;
  uint32_t tile_cnt = 0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) {
    const uint32_t c = cnt[w][dd];
    cnt[w][dd] = tile_cnt;
    tile_cnt += c;
  }
  uint32_t tot_all;
  const uint32_t ls = block_exclusive_scan(tile_cnt, sh, tot_all);
  uint32_t dummy;
  const uint32_t db = block_exclusive_scan(totals[dd], sh, dummy);
  loc_start[dd] = ls;
  gbase[dd] = db + offsets[dd * ntiles + blockIdx.x];
  __syncthreads();
#pragma unroll
  for (int t = 0; t < ITEMS; ++t) {
    if (dg[t] != 0xFFFFFFFFu) {
      const uint32_t lp = loc_start[dg[t]] + cnt[warp][dg[t]] + rank[t];
      keys_s[lp] = k[t];
      vals_s[lp] = v[t];
    }
  }
  __syncthreads();
  const int64_t rem = n - tile0;
  const int tile_n = rem < TILE ? static_cast<int>(rem) : TILE;
  for (int i = threadIdx.x; i < tile_n; i += THREADS) {
    const K key = keys_s[i];
    const uint32_t d = static_cast<uint32_t>(key >> shift) & mask;
    const uint32_t pos = gbase[d] + (i - loc_start[d]);
    if (keys_out) keys_out[pos] = key;
    vals_out[pos] = vals_s[i];
  }
}

// ---- onesweep ----------------------------------------------------------------

constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_MASK = (1u << 30) - 1u;

// counts[p][d] += number of keys whose pass-p digit is d (all passes, one read of the keys)
template <typename K>
__global__ void __launch_bounds__(THREADS) global_hist_kernel(const K* __restrict__ keys, int64_t n, int passes,
                                                              int last_bits, uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[8][RADIX];
  for (int i = threadIdx.x; i < passes * RADIX; i += THREADS) (&h[0][0])[i] = 0u;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(THREADS) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * THREADS) {
    const K key = keys[i];
    for (int p = 0; p < passes; ++p) {
      const uint32_t mask = p == passes - 1 ? (1u << last_bits) - 1u : 0xFFu;
      atomicAdd(&h[p][static_cast<uint32_t>(key >> (8 * p)) & mask], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RADIX; i += THREADS) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&counts[i], c);
  }
}

// base[p][d] = exclusive scan of counts[p][.] (one block, one thread per digit)
static __global__ void __launch_bounds__(THREADS) digit_base_kernel(const uint32_t* __restrict__ counts, int passes,
                                                                    uint32_t* __restrict__ base) {
  __shared__ uint32_t sh[WARPS];
  for (int p = 0; p < passes; ++p) {
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(counts[p * RADIX + threadIdx.x], sh, tot);
    base[p * RADIX + threadIdx.x] = ex;
  }
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename K, typename VIn, typename VOut>
__global__ void __launch_bounds__(THREADS) onesweep_kernel(const K* __restrict__ keys_in,
                                                           const VIn* __restrict__ vals_in,
                                                           K* __restrict__ keys_out, VOut* __restrict__ vals_out,
                                                           int64_t n, int shift, uint32_t mask,
                                                           const uint32_t* __restrict__ base,
                                                           uint32_t* __restrict__ status,
                                                           uint32_t* __restrict__ tile_counter) {
  static_assert(THREADS == RADIX, "one thread per digit");
  __shared__ uint32_t cnt[WARPS][RADIX];
  __shared__ uint32_t loc_start[RADIX];
  __shared__ uint32_t gbase[RADIX];
  __shared__ uint32_t sh[WARPS];
  __shared__ K keys_s[TILE];
  __shared__ VOut vals_s[TILE];
  __shared__ uint32_t tile_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_counter, 1u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < WARPS * RADIX; i += THREADS) (&cnt[0][0])[i] = 0u;
  __syncthreads();
  const int64_t tile = tile_s;
  const int64_t tile0 = tile * TILE;
  const int64_t wbase = tile0 + warp * WARP_ITEMS;
  const uint32_t lt = lanemask_lt();
  K k[ITEMS];
  VOut v[ITEMS];
  uint32_t rank[ITEMS];
  uint32_t dg[ITEMS];
  // all loads first (ITEMS independent DRAM requests in flight per thread)
#pragma unroll
  for (int t = 0; t < ITEMS; ++t) {
    const int64_t i = wbase + t * 32 + lane;
    if (i < n) {
      k[t] = keys_in[i];
      v[t] = vals_in ? static_cast<VOut>(vals_in[i]) : static_cast<VOut>(i);
    }
  }
#pragma unroll
  for (int t = 0; t < ITEMS; ++t) {
    const int64_t i = wbase + t * 32 + lane;
    const bool valid = i < n;
    uint32_t d = 0xFFFFFFFFu;
    if (valid) d = static_cast<uint32_t>(k[t] >> shift) & mask;
    dg[t] = d;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t before = valid ? cnt[warp][d] : 0u;
    __syncwarp();
    if (valid) {
      rank[t] = before + __popc(peers & lt);
      if (lane == __ffs(peers) - 1) cnt[warp][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  const int dd = threadIdx.x;
  uint32_t tile_cnt = 0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) {
    const uint32_t c = cnt[w][dd];
    cnt[w][dd] = tile_cnt;
    tile_cnt += c;
  }
  // decoupled look-back over the preceding tiles, digit dd
  uint32_t* my = status + tile * RADIX + dd;
  uint32_t excl = 0;
  if (tile > 0) {
    st_release_u32(my, LB_AGG | tile_cnt);
    // windowed look-back: LW predecessors per hop, loaded independently, so a
    // tile far from the inclusive frontier pays ~distance / LW load latencies
    constexpr int LW = 16;
    int64_t j = tile - 1;
    for (;;) {
      const int64_t lo = j - (LW - 1) > 0 ? j - (LW - 1) : 0;
      const int nw = static_cast<int>(j - lo + 1);
      uint32_t w[LW];
#pragma unroll
      for (int q = 0; q < LW; ++q) w[q] = q < nw ? ld_acquire_u32(status + (j - q) * RADIX + dd) : LB_INC;
      bool done = false;
#pragma unroll
      for (int q = 0; q < LW; ++q) {
        if (!done && q < nw) {
          while ((w[q] & ~LB_MASK) == 0u) w[q] = ld_acquire_u32(status + (j - q) * RADIX + dd);
          excl += w[q] & LB_MASK;
          done = (w[q] & LB_INC) != 0u;
        }
      }
      if (done || lo == 0) break;
      j = lo - 1;
    }
  }
  st_release_u32(my, LB_INC | (excl + tile_cnt));
  uint32_t tot_all;
  const uint32_t ls = block_exclusive_scan(tile_cnt, sh, tot_all);
  loc_start[dd] = ls;
  gbase[dd] = base[dd] + excl;
  __syncthreads();
#pragma unroll
  for (int t = 0; t < ITEMS; ++t) {
    if (dg[t] != 0xFFFFFFFFu) {
      const uint32_t lp = loc_start[dg[t]] + cnt[warp][dg[t]] + rank[t];
      keys_s[lp] = k[t];
      vals_s[lp] = v[t];
    }
  }
  __syncthreads();
  const int64_t rem = n - tile0;
  const int tile_n = rem < TILE ? static_cast<int>(rem) : TILE;
  for (int i = threadIdx.x; i < tile_n; i += THREADS) {
    const K key = keys_s[i];
    const uint32_t d = static_cast<uint32_t>(key >> shift) & mask;
    const uint32_t pos = gbase[d] + (i - loc_start[d]);
    if (keys_out) keys_out[pos] = key;
    vals_out[pos] = vals_s[i];
  }
}

// start[b] = first position of bucket b in the sorted key array, start[k] = N.
template <typename I>
__global__ void bucket_bounds_kernel(const I* __restrict__ sorted, int64_t N, int64_t k, uint32_t* __restrict__ start) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t prev = i == 0 ? -1 : static_cast<int64_t>(sorted[i - 1]);
    const int64_t cur = i == N ? k : static_cast<int64_t>(sorted[i]);
    for (int64_t b = prev + 1; b <= cur && b <= k; ++b) start[b] = static_cast<uint32_t>(i);
  }
}

template <typename K>
struct Buffers {
  K* keys[2];
  uint32_t* vals[2];
  uint32_t* hist;
  uint32_t* totals;
  uint32_t* sweep;  // onesweep: counts[8][256] | base[8][256] | tile counters[8] | status[8][ntiles][256]
};

inline size_t sweep_words(int64_t n) { return 2 * 8 * RADIX + 8 + static_cast<size_t>(8) * RADIX * num_tiles(n); }

template <typename K>
inline void measure(Measure& m, int64_t n) {
  m.take<K>(n);
  m.take<K>(n);
  m.take<uint32_t>(n);
  m.take<uint32_t>(n);
  m.take<uint32_t>(static_cast<size_t>(RADIX) * num_tiles(n));
  m.take<uint32_t>(RADIX);
  m.take<uint32_t>(sweep_words(n));
}

template <typename K>
inline Buffers<K> carve(Carve& c, int64_t n) {
  Buffers<K> b;
  b.keys[0] = c.take<K>(n);
  b.keys[1] = c.take<K>(n);
  b.vals[0] = c.take<uint32_t>(n);
  b.vals[1] = c.take<uint32_t>(n);
  b.hist = c.take<uint32_t>(static_cast<size_t>(RADIX) * num_tiles(n));
  b.totals = c.take<uint32_t>(RADIX);
  b.sweep = c.take<uint32_t>(sweep_words(n));
  return b;
}

// Sort `n` pairs on key bits [0, nbits).  vals == nullptr: value = index.
// Final keys land in *keys_final (may be nullptr), final values in vals_final.
template <typename K, typename VOut>
int32_t sort_pairs(const K* keys, const uint32_t* vals, int64_t n, int nbits, Buffers<K>& b,
                   K* keys_final, VOut* vals_final, cudaStream_t st) {
  if (n <= 0) return LVSK_OK;
  if (n > 0xFFFFFFFFll) {
    set_error("radix sort supports at most 2^32-1 items, got %lld", (long long)n);
    return LVSK_ERR_CAPACITY;
  }
  const int64_t ntiles = num_tiles(n);
  const int passes = nbits <= 0 ? 1 : (nbits + 7) / 8;
  const K* kin = keys;
  const uint32_t* vin = vals;
  // onesweep wins when launches dominate (few tiles); with hundreds of tiles
  // per pass the serial look-back latency costs more than the classic
  // histogram + scan kernels (measured: 1e6 keys, 8 passes, 0.29 vs 0.23 ms)
  const bool sweep = getenv("LVSK_RADIX_ONESWEEP") != nullptr ||
                     (ntiles <= 2 * static_cast<int64_t>(num_sms()) && getenv("LVSK_RADIX_CLASSIC") == nullptr);
  if (n < (int64_t{1} << 30) && passes <= 8 && sweep) {
    uint32_t* counts = b.sweep;
    uint32_t* base = counts + 8 * RADIX;
    uint32_t* tiles = base + 8 * RADIX;
    uint32_t* status = tiles + 8;
    const int last_bits = nbits <= 0 ? 1 : nbits - 8 * (passes - 1);
    const size_t used = 2 * 8 * RADIX + 8 + static_cast<size_t>(passes) * RADIX * ntiles;
    cudaError_t e = cudaMemsetAsync(b.sweep, 0, used * sizeof(uint32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "radix memset");
    const int hgrid = static_cast<int>(ntiles < num_sms() * 4 ? ntiles : num_sms() * 4);
    global_hist_kernel<K><<<hgrid, THREADS, 0, st>>>(kin, n, passes, last_bits, counts);
    digit_base_kernel<<<1, THREADS, 0, st>>>(counts, passes, base);
    for (int p = 0; p < passes; ++p) {
      const int shift = 8 * p;
      const uint32_t mask = p == passes - 1 ? (1u << last_bits) - 1u : 0xFFu;
      uint32_t* stp = status + static_cast<size_t>(p) * RADIX * ntiles;
      if (p == passes - 1) {
        onesweep_kernel<K, uint32_t, VOut><<<static_cast<unsigned>(ntiles), THREADS, 0, st>>>(
            kin, vin, keys_final, vals_final, n, shift, mask, base + p * RADIX, stp, tiles + p);
      } else {
        K* ko = b.keys[p & 1];
        uint32_t* vo = b.vals[p & 1];
        onesweep_kernel<K, uint32_t, uint32_t><<<static_cast<unsigned>(ntiles), THREADS, 0, st>>>(
            kin, vin, ko, vo, n, shift, mask, base + p * RADIX, stp, tiles + p);
        kin = ko;
        vin = vo;
      }
      LVSK_CHECK_LAUNCH("radix onesweep pass");
    }
    return LVSK_OK;
  }
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    const int bits = nbits <= 0 ? 1 : min(8, nbits - shift);
    const uint32_t mask = (1u << bits) - 1u;
    const bool last = p == passes - 1;
    hist_kernel<K><<<static_cast<unsigned>(ntiles), THREADS, 0, st>>>(kin, n, shift, mask, b.hist, ntiles);
    scan_rows_kernel<<<RADIX, THREADS, 0, st>>>(b.hist, ntiles, b.totals);
    if (last) {
      scatter_kernel<K, uint32_t, VOut><<<static_cast<unsigned>(ntiles), THREADS, 0, st>>>(
          kin, vin, keys_final, vals_final, n, shift, mask, b.hist, b.totals, ntiles);
    } else {
      K* ko = b.keys[p & 1];
      uint32_t* vo = b.vals[p & 1];
      scatter_kernel<K, uint32_t, uint32_t><<<static_cast<unsigned>(ntiles), THREADS, 0, st>>>(
          kin, vin, ko, vo, n, shift, mask, b.hist, b.totals, ntiles);
      kin = ko;
      vin = vo;
    }
    LVSK_CHECK_LAUNCH("radix sort pass");
  }
  return LVSK_OK;
}

}  // namespace radix
}  // namespace lvsk
