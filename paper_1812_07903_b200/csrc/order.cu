// Ordering: scores_to_distribution + make_plan("dec"/"dec_swor") on device.
//
// Reference: order.py:51-63 (normalise with validation), order.py:84-90
// (dec = np.argsort(-p, kind="stable")), order.py:95-99 (dec_swor =
// np.argsort(Exp(1)/p, kind="stable")).  K7 is a stable LSD radix sort over
// an order-preserving uint64 image of the float64 keys (8 passes of 8 bits),
// values = indices, so ties keep ascending index exactly like numpy's stable
// sort.
//
// For n up to a few million the whole sort runs in ONE cooperative kernel
// (argsort_coop_kernel): the ping-pong key/index buffers (12 B per item) stay
// in the 126 MB L2, every CTA owns a contiguous index range, and a pass is
// chunk histogram -> grid barrier -> per-digit offsets from all CTAs'
// histograms -> stable in-chunk ranking + scatter -> grid barrier.  Passes
// whose 8-bit digit is the same for every key (found from the OR / AND of all
// keys; e.g. the sign and top exponent bits of a probability vector) are
// skipped — a stable pass on a constant digit is the identity.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "radix_sort.cuh"

namespace cg = cooperative_groups;

namespace lvsk {

constexpr int SUM_THREADS = 256;
constexpr int SUM_ITEMS = 8;
constexpr int64_t SUM_TILE = SUM_THREADS * SUM_ITEMS;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  // fixed-shape tree: deterministic for a given launch geometry
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
  }
  return v;
}

// stage 1: per-tile partial sums (+ validation flags)
__global__ void __launch_bounds__(SUM_THREADS) sum_stage1_kernel(const double* __restrict__ x, int64_t n,
                                                                 double* __restrict__ partial, int32_t* flags,
                                                                 int validate) {
  __shared__ double sh[SUM_THREADS / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * SUM_TILE;
  double v = 0.0;
  int bad = 0;
#pragma unroll
  for (int j = 0; j < SUM_ITEMS; ++j) {
    const int64_t i = base + j * SUM_THREADS + threadIdx.x;
    if (i < n) {
      const double s = x[i];
      if (validate) {
        if (!isfinite(s)) bad |= LVSK_FLAG_NONFINITE;
        else if (s < 0.0) bad |= LVSK_FLAG_NEGATIVE;
      }
      v += s;
    }
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (validate) {
    bad = __syncthreads_or(bad) ? bad : 0;
    if (bad) atomicOr(flags, bad);
  }
}

// stage 2: one block folds the partials in a fixed order
__global__ void __launch_bounds__(SUM_THREADS) sum_stage2_kernel(const double* __restrict__ partial, int64_t m,
                                                                 double* __restrict__ out) {
  __shared__ double sh[SUM_THREADS / 32];
  const int64_t per = (m + SUM_THREADS - 1) / SUM_THREADS;
  double v = 0.0;
  for (int64_t i = threadIdx.x * per; i < min(m, (threadIdx.x + 1) * per); ++i) v += partial[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) *out = v;
}

__global__ void divide_kernel(const double* __restrict__ s, int64_t n, const double* __restrict__ total,
                              double* __restrict__ p) {
  const double t = *total;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = s[i] / t;
}

// order-preserving uint64 image of a double (ascending), NaN last, -0 == +0
__device__ __forceinline__ uint64_t f64_key(double x) {
  if (isnan(x)) return ~0ull;
  if (x == 0.0) x = 0.0;
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void argsort_keys_kernel(const double* __restrict__ keys, int64_t n, int descending,
                                    uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = keys[i];
    out[i] = f64_key(descending ? -x : x);
  }
}

// ---- K7 cooperative (L2-resident) argsort ------------------------------------

constexpr int AS_THREADS = 512;
constexpr int AS_WARPS = AS_THREADS / 32;
constexpr int AS_ITEMS = 8;
constexpr int AS_SUB = AS_THREADS * AS_ITEMS;  // 4096 keys per ranking sub-tile
constexpr int AS_WARP_ITEMS = AS_SUB / AS_WARPS;
constexpr int AS_HALO = 64;                    // longest equal-prefix run the fix-up sorts locally
constexpr int AS_WIN = 4096;                   // fix-up window
constexpr int64_t AS_MAX_N = int64_t{8} << 20;
constexpr int AS_MAX_G = 1024;
constexpr int64_t AS_INFLIGHT_CHUNK = 8192;  // min keys per CTA with passes in flight
constexpr int AS_CHUNK_CAP = 12288;           // chunks up to this size are staged whole (longest output runs)
constexpr size_t AS_RANK_SMEM =
    sizeof(uint32_t) * AS_WARPS * 256 + (sizeof(uint64_t) + sizeof(uint32_t)) * AS_CHUNK_CAP;
constexpr size_t AS_FIX_SMEM = (sizeof(uint64_t) + sizeof(uint32_t)) * (AS_WIN + 2 * AS_HALO);
constexpr size_t AS_SMEM = AS_RANK_SMEM > AS_FIX_SMEM ? AS_RANK_SMEM : AS_FIX_SMEM;

struct AsArgs {
  const double* in;
  int64_t n;
  int descending;
  int64_t* out;
  uint64_t* kb[3];  // kb[0]: keys in index order (kept); kb[1], kb[2]: ping-pong
  uint32_t* vb[2];
  uint32_t* hist;   // [G][256] chunk histograms of the current pass
  uint32_t* totals; // [8][256] digit totals of every pass
  unsigned long long* orand;  // OR, AND of all keys
  unsigned int* bar;          // barrier arrivals
  unsigned int* flag;         // fix-up refused: redo with every digit
  unsigned long long* trace;  // optional phase timestamps (LVSK_SORT_TRACE)
};

__device__ __forceinline__ void as_stamp(const AsArgs& a, int slot) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[slot] = t;
  }
}

// exclusive scan of one value per thread over the first 256 threads (all 512 call)
__device__ __forceinline__ uint32_t scan256(uint32_t v, uint32_t* sh, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = threadIdx.x < 256 ? v : 0u;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31 && warp < 8) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < 8 ? sh[lane] : 0u;
#pragma unroll
    for (int off = 1; off < 8; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, off);
      if (lane >= off) w += y;
    }
    if (lane < 8) sh[lane] = w;
  }
  __syncthreads();
  total = sh[7];
  const uint32_t base = (warp > 0 && warp < 8) ? sh[warp - 1] : 0u;
  __syncthreads();
  return base + x - (threadIdx.x < 256 ? v : 0u);
}

// grid barrier on a monotone arrival counter (zeroed before the launch): the
// k-th barrier completes when count >= k * G.  One atomic per CTA, thread 0
// polls with ld.acquire.
__device__ __forceinline__ void as_barrier(unsigned int* count, unsigned int& nbar) {
  const unsigned int target = (++nbar) * gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Stable LSD passes over the active digits in [dlo, dhi] (8-bit digits of the
// keys in kb[0]).  The last active pass writes the indices (int64) to out and
// the keys in sorted order to the returned buffer.  No active digit: the
// identity.
__device__ const uint64_t* as_passes(const AsArgs& a, int dlo, int dhi, unsigned long long diff, unsigned int& nbar,
                                     uint8_t* smem, int64_t c0, int64_t c1) {
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);                  // [AS_WARPS][256]
  uint64_t* keys_s = reinterpret_cast<uint64_t*>(cnt + AS_WARPS * 256);  // [AS_CHUNK_CAP]
  uint32_t* vals_s = reinterpret_cast<uint32_t*>(keys_s + AS_CHUNK_CAP); // [AS_CHUNK_CAP]
  __shared__ uint32_t run[256], loc_start[256], sub_cnt[256], sh[16], cstart[256], crun[256];
  // a chunk that fits is staged whole in digit order before any global store,
  // so each digit leaves the CTA as one contiguous run (better write coalescing)
  const bool whole = c1 - c0 <= AS_CHUNK_CAP;
  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  int last = -1;
  for (int p = dlo; p <= dhi; ++p)
    if ((diff >> (8 * p)) & 0xFFull) last = p;
  if (last < 0) {
    for (int64_t i = c0 + threadIdx.x; i < c1; i += AS_THREADS) a.out[i] = i;
    as_barrier(a.bar, nbar);
    return a.kb[0];
  }
  const uint64_t* ksrc = a.kb[0];
  const uint32_t* vsrc = nullptr;  // identity on the first active pass
  uint64_t* kdst = a.kb[1];
  uint32_t* vdst = a.vb[0];
  for (int p = dlo; p <= last; ++p) {
    if (!((diff >> (8 * p)) & 0xFFull)) continue;
    const int shift = 8 * p;
    const bool fin = p == last;
    // (a) chunk histogram
    for (int i = threadIdx.x; i < 256; i += AS_THREADS) run[i] = 0u;
    __syncthreads();
    for (int64_t i = c0 + threadIdx.x; i < c1; i += AS_THREADS)
      atomicAdd(&run[static_cast<uint32_t>(__ldcg(ksrc + i) >> shift) & 0xFFu], 1u);
    __syncthreads();
    if (threadIdx.x < 256) a.hist[cta * 256 + threadIdx.x] = run[threadIdx.x];
    if (whole) {
      uint32_t ct;
      const uint32_t cs = scan256(threadIdx.x < 256 ? run[threadIdx.x] : 0u, sh, ct);
      if (threadIdx.x < 256) {
        cstart[threadIdx.x] = cs;
        crun[threadIdx.x] = cs;
      }
    }
    as_stamp(a, 4 * p + 2);
    as_barrier(a.bar, nbar);
    as_stamp(a, 4 * p + 3);
    // (b) start of this chunk's run of every digit: digit base (scan of the pass
    // totals) + the counts of the preceding chunks (16 rows in flight per thread)
    {
      const int d = threadIdx.x & 255, h = threadIdx.x >> 8;
      uint32_t acc = 0;
      for (int c = h; c < cta; c += 32) {
        uint32_t v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = c + 2 * u < cta ? __ldcg(a.hist + (c + 2 * u) * 256 + d) : 0u;
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u];
      }
      if (h == 1) loc_start[d] = acc;
      __syncthreads();
      const uint32_t before = h == 0 ? acc + loc_start[d] : 0u;
      uint32_t all;
      const uint32_t dbase = scan256(h == 0 ? __ldcg(a.totals + p * 256 + d) : 0u, sh, all);
      if (h == 0) run[d] = dbase + before;
      __syncthreads();
    }
    as_stamp(a, 4 * p + 4);
    // (c) stable scatter, sub-tile by sub-tile in index order
    for (int64_t s0 = c0; s0 < c1; s0 += AS_SUB) {
      for (int i = threadIdx.x; i < AS_WARPS * 256; i += AS_THREADS) cnt[i] = 0u;
      __syncthreads();
      const int64_t wb = s0 + warp * AS_WARP_ITEMS;
      uint64_t k[AS_ITEMS];
      uint32_t v[AS_ITEMS], rank[AS_ITEMS], dg[AS_ITEMS];
#pragma unroll
      for (int t = 0; t < AS_ITEMS; ++t) {
        const int64_t i = wb + t * 32 + lane;
        if (i < c1) {
          k[t] = __ldcg(ksrc + i);
          v[t] = vsrc ? __ldcg(vsrc + i) : static_cast<uint32_t>(i);
        }
      }
      // warp-level stable ranking: match_any groups the lanes of a digit, the
      // group leader bumps the warp's digit counter with one shared atomic
      // (a warp's atomics to one address apply in issue order = item order)
      // and broadcasts the old count; all items' matches and atomics are
      // independent, so they pipeline
      uint32_t peers[AS_ITEMS], old[AS_ITEMS];
#pragma unroll
      for (int t = 0; t < AS_ITEMS; ++t) {
        const int64_t i = wb + t * 32 + lane;
        dg[t] = i < c1 ? static_cast<uint32_t>(k[t] >> shift) & 0xFFu : 0xFFFFFFFFu;
        peers[t] = __match_any_sync(0xFFFFFFFFu, dg[t]);
      }
#pragma unroll
      for (int t = 0; t < AS_ITEMS; ++t) {
        old[t] = 0u;
        if (dg[t] != 0xFFFFFFFFu && lane == __ffs(peers[t]) - 1)
          old[t] = atomicAdd(&cnt[warp * 256 + dg[t]], static_cast<uint32_t>(__popc(peers[t])));
      }
#pragma unroll
      for (int t = 0; t < AS_ITEMS; ++t)
        rank[t] = __shfl_sync(0xFFFFFFFFu, old[t], __ffs(peers[t]) - 1) + __popc(peers[t] & lt);
      __syncthreads();
      uint32_t tc = 0;
      if (threadIdx.x < 256) {
#pragma unroll
        for (int w = 0; w < AS_WARPS; ++w) {
          const uint32_t c = cnt[w * 256 + threadIdx.x];
          cnt[w * 256 + threadIdx.x] = tc;
          tc += c;
        }
      }
      uint32_t tn;
      const uint32_t ls = scan256(tc, sh, tn);
      if (threadIdx.x < 256) {
        loc_start[threadIdx.x] = whole ? crun[threadIdx.x] : ls;
        sub_cnt[threadIdx.x] = tc;
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < AS_ITEMS; ++t) {
        if (dg[t] != 0xFFFFFFFFu) {
          const uint32_t lp = loc_start[dg[t]] + cnt[warp * 256 + dg[t]] + rank[t];
          keys_s[lp] = k[t];
          vals_s[lp] = v[t];
        }
      }
      __syncthreads();
      if (whole) {
        if (threadIdx.x < 256) crun[threadIdx.x] += sub_cnt[threadIdx.x];
        __syncthreads();
        continue;
      }
      for (int j = threadIdx.x; j < static_cast<int>(tn); j += AS_THREADS) {
        const uint64_t key = keys_s[j];
        const uint32_t d = static_cast<uint32_t>(key >> shift) & 0xFFu;
        const uint32_t pos = run[d] + (j - loc_start[d]);
        kdst[pos] = key;
        if (fin)
          a.out[pos] = vals_s[j];
        else
          vdst[pos] = vals_s[j];
      }
      __syncthreads();
      if (threadIdx.x < 256) run[threadIdx.x] += sub_cnt[threadIdx.x];
      __syncthreads();
    }
    if (whole) {
      const int len = static_cast<int>(c1 - c0);
      for (int j = threadIdx.x; j < len; j += AS_THREADS) {
        const uint64_t key = keys_s[j];
        const uint32_t d = static_cast<uint32_t>(key >> shift) & 0xFFu;
        const uint32_t pos = run[d] + (j - cstart[d]);
        kdst[pos] = key;
        if (fin)
          a.out[pos] = vals_s[j];
        else
          vdst[pos] = vals_s[j];
      }
    }
    as_stamp(a, 4 * p + 5);
    as_barrier(a.bar, nbar);
    if (fin) return kdst;
    ksrc = kdst;
    vsrc = vdst;
    kdst = kdst == a.kb[1] ? a.kb[2] : a.kb[1];
    vdst = vdst == a.vb[0] ? a.vb[1] : a.vb[0];
  }
  return ksrc;  // not reached
}

// Sort by the high 32 key bits only, then put every run of equal high bits in
// order locally (runs of <= AS_HALO keys, one thread each; in random data the
// runs hold 1-3 keys).  A disordered longer run raises *flag and the caller
// redoes the sort on every digit.
__device__ void as_fixup(const AsArgs& a, const uint64_t* ks, uint8_t* smem, int64_t c0, int64_t c1, int hs) {
  uint64_t* K = reinterpret_cast<uint64_t*>(smem);                     // [AS_WIN + 2 AS_HALO]
  uint32_t* I = reinterpret_cast<uint32_t*>(K + AS_WIN + 2 * AS_HALO);  // [AS_WIN + 2 AS_HALO]
  const int64_t n = a.n;
  for (int64_t w0 = c0; w0 < c1; w0 += AS_WIN) {
    const int wlen = static_cast<int>(c1 - w0 < AS_WIN ? c1 - w0 : AS_WIN);
    const int span = wlen + 2 * AS_HALO;
    for (int j = threadIdx.x; j < span; j += AS_THREADS) {
      const int64_t pos = w0 - AS_HALO + j;
      if (pos >= 0 && pos < n) {
        K[j] = __ldcg(ks + pos);
        I[j] = static_cast<uint32_t>(__ldcg(a.out + pos));
      }
    }
    __syncthreads();
    // detection (reads only); run starts in this window that need sorting
    int my_start[AS_WIN / AS_THREADS], my_len[AS_WIN / AS_THREADS], nmine = 0;
    bool bad = false;
    for (int t = threadIdx.x; t < wlen; t += AS_THREADS) {
      const int64_t pos = w0 + t;
      const int j = t + AS_HALO;
      const uint64_t hi = K[j] >> hs;
      const bool start = pos == 0 || (K[j - 1] >> hs) != hi;
      if (start) {
        int L = 1;
        bool dis = false;
        while (L <= AS_HALO && pos + L < n && (K[j + L] >> hs) == hi) {
          dis |= K[j + L] < K[j + L - 1];
          ++L;
        }
        if (L > AS_HALO) {
          bad |= dis;  // a run longer than the halo: only an ordered one is accepted
        } else if (dis) {
          my_start[nmine] = j;
          my_len[nmine] = L;
          ++nmine;
        }
      } else if (K[j] < K[j - 1]) {
        // disordered inside a run: fine if the run started within AS_HALO positions
        bool found = false;
        for (int q = 1; q <= AS_HALO && !found; ++q)
          found = pos - q < 0 || (K[j - q] >> hs) != hi;
        bad |= !found;
      }
    }
    if (bad) atomicOr(a.flag, 1u);
    __syncthreads();
    // fix: insertion sort of (key, index) over each short disordered run
    for (int m = 0; m < nmine; ++m) {
      const int j0 = my_start[m], L = my_len[m];
      for (int x = j0 + 1; x < j0 + L; ++x) {
        const uint64_t kx = K[x];
        const uint32_t ix = I[x];
        int y = x - 1;
        while (y >= j0 && (K[y] > kx || (K[y] == kx && I[y] > ix))) {
          K[y + 1] = K[y];
          I[y + 1] = I[y];
          --y;
        }
        K[y + 1] = kx;
        I[y + 1] = ix;
      }
      for (int x = j0; x < j0 + L; ++x) a.out[w0 - AS_HALO + x] = I[x];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(AS_THREADS, 1) argsort_coop_kernel(AsArgs a) {
  extern __shared__ __align__(16) uint8_t as_smem[];
  __shared__ unsigned long long red_or[AS_WARPS], red_and[AS_WARPS];
  unsigned int nbar = 0;
  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = a.n;
  const int64_t c0 = n * cta / G, c1 = n * (cta + 1) / G;

  // phase 0: order-preserving keys, OR / AND of all keys, and the digit totals
  // of every pass (a digit count does not depend on the order of the keys)
  uint32_t* h8 = reinterpret_cast<uint32_t*>(as_smem);  // [8][256]
  for (int i = threadIdx.x; i < 8 * 256; i += AS_THREADS) h8[i] = 0u;
  __syncthreads();
  unsigned long long o = 0ull, an = ~0ull;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += AS_THREADS) {
    const double x = a.in[i];
    const uint64_t k = f64_key(a.descending ? -x : x);
    a.kb[0][i] = k;
    o |= k;
    an &= k;
#pragma unroll
    for (int q = 0; q < 8; ++q) atomicAdd(&h8[q * 256 + ((k >> (8 * q)) & 0xFFu)], 1u);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    o |= __shfl_xor_sync(0xFFFFFFFFu, o, off);
    an &= __shfl_xor_sync(0xFFFFFFFFu, an, off);
  }
  if (lane == 0) {
    red_or[warp] = o;
    red_and[warp] = an;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += AS_THREADS)
    if (h8[i]) atomicAdd(a.totals + i, h8[i]);
  if (threadIdx.x == 0) {
    for (int w = 1; w < AS_WARPS; ++w) {
      o |= red_or[w];
      an &= red_and[w];
    }
    if (c1 > c0) {
      atomicOr(a.orand, o);
      atomicAnd(a.orand + 1, an);
    }
  }
  as_stamp(a, 0);
  as_barrier(a.bar, nbar);
  as_stamp(a, 1);
  const unsigned long long diff = __ldcg(a.orand) ^ __ldcg(a.orand + 1);
  if (diff == 0ull) {  // every key equal: the stable order is the identity
    for (int64_t i = c0 + threadIdx.x; i < c1; i += AS_THREADS) a.out[i] = i;
    return;
  }
  // fast path: the high 32 bits (digits 4..7) — 40 bits from 4M keys on, where
  // runs of equal high-32-bit keys outgrow the fix-up's halo (C5's 8e6
  // probabilities) — then the local fix-up of the runs
  const int dfirst = n >= (int64_t{1} << 22) ? 3 : 4;
  const int hs = 8 * dfirst;
  const uint64_t* ks = as_passes(a, dfirst, 7, diff, nbar, as_smem, c0, c1);
  if (diff & ((1ull << hs) - 1ull)) {
    as_stamp(a, 40);
    unsigned long long fx0 = 0;
    if (a.trace != nullptr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fx0));
    as_fixup(a, ks, as_smem, c0, c1, hs);
    if (a.trace != nullptr && threadIdx.x == 0) {
      unsigned long long fx1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(fx1));
      atomicMax(a.trace + 50, fx1 - fx0);
    }
    as_stamp(a, 41);
    as_barrier(a.bar, nbar);
    as_stamp(a, 42);
    if (__ldcg(a.flag) != 0u) as_passes(a, 0, 7, diff, nbar, as_smem, c0, c1);
  }
}

static int coop_grid() {
  const int per = resident_ctas(reinterpret_cast<const void*>(argsort_coop_kernel), AS_THREADS, static_cast<int>(AS_SMEM));
  int g = per >= 1 ? num_sms() * (per > 2 ? 2 : per) : 0;
  if (g > AS_MAX_G) g = AS_MAX_G;
  return g;
}

static int grid_cap(int64_t work) {
  int64_t g = (work + 255) / 256;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

static int32_t det_sum(const double* x, int64_t n, double* out, double* partial, int32_t* flags, int validate,
                       cudaStream_t st) {
  const int64_t tiles = (n + SUM_TILE - 1) / SUM_TILE;
  sum_stage1_kernel<<<static_cast<unsigned>(tiles), SUM_THREADS, 0, st>>>(x, n, partial, flags, validate);
  sum_stage2_kernel<<<1, SUM_THREADS, 0, st>>>(partial, tiles, out);
  LVSK_CHECK_LAUNCH("sum");
  return LVSK_OK;
}

}  // namespace lvsk

using namespace lvsk;

// ---- KM: merge of per-rank sorted runs (multi-rank "dec" order) ---------------
//
// Multi-rank ordering: every rank argsorts its own probabilities (K7, in
// parallel), rank 0 gathers the R sorted runs (keys in local sorted order +
// the local indices) — a streaming read, no random gathers — and merges them
// into the stable argsort of the concatenation — the same
// permutation lvsk_argsort_f64 returns for the gathered keys (runs are in rank
// = global row order, so a stable merge that takes the earlier run on ties
// reproduces numpy's stable tie order).  Pairwise merge-path rounds (ceil(log2 R))
// over (uint64 key image, uint32 global index) pairs; each CTA merges a
// 4096-output chunk of one pair through shared memory (its merge-path split
// found up front by km_split_kernel), each thread 8 outputs.
constexpr int KM_THREADS = 512;
constexpr int KM_ITEMS = 8;
constexpr int KM_CHUNK = KM_THREADS * KM_ITEMS;
constexpr int KM_MAX_RUNS = 512;

struct KmPairs {
  int64_t a0[KM_MAX_RUNS / 2 + 1], la[KM_MAX_RUNS / 2 + 1], lb[KM_MAX_RUNS / 2 + 1];
  int64_t r0[KM_MAX_RUNS / 2 + 1], r1[KM_MAX_RUNS / 2 + 1];  // round 1: global offsets of the pair's runs
  int64_t chunk0[KM_MAX_RUNS / 2 + 2];  // first chunk of each pair (prefix)
  int npairs;
};

// Element e of the working array: its uint64 key image and uint32 global
// index.  Round 1 (SRC = 1) reads the gathered runs directly — the double key
// sorted_keys[e] and the run-local index run_idx[e] (global = the run's offset
// + local; within a merged pair A is run 2i, B run 2i + 1) — so no expand pass;
// later rounds (SRC = 0) read the previous round's (image, index) pairs.
struct KmSrc {
  const uint64_t* kimg;
  const uint32_t* gidx;
  const double* skeys;
  const int32_t* ridx;
  int descending;
};
template <int SRC>
__device__ __forceinline__ uint64_t km_key(const KmSrc& S, int64_t e) {
  if constexpr (SRC == 0) {
    return S.kimg[e];
  } else {
    const double x = S.skeys[e];
    return f64_key(S.descending ? -x : x);
  }
}
template <int SRC>
__device__ __forceinline__ uint32_t km_idx(const KmSrc& S, int64_t e, int64_t run_off) {
  if constexpr (SRC == 0) return S.gidx[e];
  else return static_cast<uint32_t>(run_off + S.ridx[e]);
}

// merge-path split of every chunk boundary of a round: one warp per boundary,
// a 32-ary search (each step samples 32 positions and ballots the monotone
// predicate A[i] <= B[t-1-i], i.e. "A[i] is among the first t outputs")
template <int SRC>
__global__ void km_split_kernel(const __grid_constant__ KmPairs P, int64_t nchunks, KmSrc S,
                                int64_t* __restrict__ split) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (c >= nchunks) return;
  int q = 0;
  while (q + 1 < P.npairs && P.chunk0[q + 1] <= c) ++q;
  const int64_t a0 = P.a0[q], la = P.la[q], lb = P.lb[q], b0 = a0 + la;
  const int64_t t = (c - P.chunk0[q]) * KM_CHUNK;
  int64_t lo = t - lb > 0 ? t - lb : 0, hi = t < la ? t : la;  // answer in [lo, hi]
  while (hi > lo) {
    // candidates lo + (j + 1) * step - 1, j < 32, clipped to hi - 1
    const int64_t span = hi - lo;
    const int64_t step = (span + 31) / 32;
    int64_t i = lo + (lane + 1) * step - 1;
    if (i > hi - 1) i = hi - 1;
    const bool pr = km_key<SRC>(S, a0 + i) <= km_key<SRC>(S, b0 + t - 1 - i);
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, pr);  // a prefix of lanes (monotone)
    const int ntrue = __popc(m);
    // the first false candidate bounds the answer from above
    const int64_t nlo = ntrue == 0 ? lo : (lo + ntrue * step > hi ? hi : lo + ntrue * step);
    const int64_t cand_hi = ntrue == 32 ? hi : lo + (ntrue + 1) * step - 1;
    lo = nlo;
    hi = cand_hi < hi ? cand_hi : hi;
    if (step == 1) {  // every position in [old lo, old hi) was a candidate
      hi = lo;
    }
  }
  if (lane == 0) split[c] = lo;
}

template <int SRC, bool FINAL>
__global__ void __launch_bounds__(KM_THREADS) km_merge_kernel(const __grid_constant__ KmPairs P, KmSrc S,
                                                             const int64_t* __restrict__ split,
                                                             uint64_t* __restrict__ kout, uint32_t* __restrict__ iout,
                                                             int64_t* __restrict__ final_out) {
  __shared__ uint64_t sk[KM_CHUNK];
  __shared__ uint32_t si[KM_CHUNK];
  const int64_t chunk = blockIdx.x;
  int q = 0;
  while (q + 1 < P.npairs && P.chunk0[q + 1] <= chunk) ++q;
  const int64_t a0 = P.a0[q], la = P.la[q], lb = P.lb[q];
  const int64_t t0 = (chunk - P.chunk0[q]) * KM_CHUNK;
  const int64_t t1 = t0 + KM_CHUNK < la + lb ? t0 + KM_CHUNK : la + lb;
  const int64_t i0 = split[chunk];
  const int64_t i1 = chunk + 1 < P.chunk0[q + 1] ? split[chunk + 1] : la;  // a pair's last chunk ends with all of A
  const int na = static_cast<int>(i1 - i0), nb = static_cast<int>((t1 - i1) - (t0 - i0));
  const int tot = na + nb;
  // stage A[i0, i1) then B[t0 - i0, t1 - i1) (all loads issued before any is used)
#pragma unroll
  for (int u = 0; u < KM_ITEMS; ++u) {
    const int e = threadIdx.x + u * KM_THREADS;
    if (e < tot) {
      const bool inA = e < na;
      const int64_t src = inA ? a0 + i0 + e : a0 + la + (t0 - i0) + (e - na);
      sk[e] = km_key<SRC>(S, src);
      si[e] = km_idx<SRC>(S, src, inA ? P.r0[q] : P.r1[q]);
    }
  }
  __syncthreads();
  const int d0 = threadIdx.x * KM_ITEMS;
  uint64_t ok[KM_ITEMS];
  uint32_t oi[KM_ITEMS];
  if (d0 < tot) {
    // thread-level merge path inside the chunk
    int lo = d0 - nb > 0 ? d0 - nb : 0, hi = d0 < na ? d0 : na;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sk[mid] <= sk[na + d0 - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    int ia = lo, ib = d0 - lo;
#pragma unroll
    for (int j = 0; j < KM_ITEMS; ++j) {
      const bool takeA = ib >= nb || (ia < na && sk[ia] <= sk[na + ib]);
      const int src = takeA ? ia : na + ib;
      if (d0 + j < tot) {
        ok[j] = sk[src];
        oi[j] = si[src];
      }
      if (takeA) ++ia; else ++ib;
    }
  }
  // back through shared memory, so the stores below are coalesced
  __syncthreads();
#pragma unroll
  for (int j = 0; j < KM_ITEMS; ++j) {
    if (d0 + j < tot) {
      sk[d0 + j] = ok[j];
      si[d0 + j] = oi[j];
    }
  }
  __syncthreads();
  const int64_t o0 = a0 + t0;
#pragma unroll
  for (int u = 0; u < KM_ITEMS; ++u) {
    const int e = threadIdx.x + u * KM_THREADS;
    if (e < tot) {
      if (FINAL) {
        final_out[o0 + e] = static_cast<int64_t>(si[e]);
      } else {
        kout[o0 + e] = sk[e];
        iout[o0 + e] = si[e];
      }
    }
  }
}

// run-local indices outside their runs (one pass over run_idx; the merge
// itself never dereferences them)
struct KmOffsets {
  int64_t off[KM_MAX_RUNS + 1];
};
__global__ void km_check_kernel(const int32_t* __restrict__ run_idx, const __grid_constant__ KmOffsets O, int runs,
                                int64_t n, int32_t* flags) {
  const int64_t* off = O.off;
  bool bad = false;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = runs;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (off[mid] <= e) lo = mid; else hi = mid;
    }
    const int32_t li = run_idx[e];
    bad |= li < 0 || li >= off[lo + 1] - off[lo];
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, LVSK_FLAG_BADINDEX);
}

extern "C" size_t lvsk_normalize_workspace_bytes(int64_t n) {
  Measure m;
  m.take<double>((n + SUM_TILE - 1) / SUM_TILE + 1);
  return m.off;
}

extern "C" int32_t lvsk_sum_f64(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes,
                                void* stream) {
  LVSK_REQUIRE(n >= 1, LVSK_ERR_DEGENERATE, "empty input");
  Carve c(ws, ws_bytes);
  double* partial = c.take<double>((n + SUM_TILE - 1) / SUM_TILE + 1);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small");
  return det_sum(x, n, out, partial, nullptr, 0, as_stream(stream));
}

extern "C" int32_t lvsk_normalize_scores(const double* scores, int64_t n, double* p_out, double* total, void* ws,
                                         size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(n >= 1, LVSK_ERR_DEGENERATE, "scores must be a non-empty 1-D array");
  Carve c(ws, ws_bytes);
  double* partial = c.take<double>((n + SUM_TILE - 1) / SUM_TILE + 1);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small");
  cudaStream_t st = as_stream(stream);
  int32_t rc = det_sum(scores, n, total, partial, flags, 1, st);
  if (rc != LVSK_OK) return rc;
  divide_kernel<<<grid_cap(n), 256, 0, st>>>(scores, n, total, p_out);
  LVSK_CHECK_LAUNCH("normalize");
  return LVSK_OK;
}

extern "C" size_t lvsk_argsort_workspace_bytes(int64_t n) {
  Measure m;
  m.take<uint64_t>(n);
  radix::measure<uint64_t>(m, n);
  m.take<uint32_t>(static_cast<size_t>(256) * AS_MAX_G);  // coop: chunk histograms
  m.take<uint32_t>(8 * 256);                               // coop: digit totals of every pass
  m.take<unsigned long long>(4);                           // coop: OR, AND, barrier, flag
  return m.off;
}

extern "C" int32_t lvsk_argsort_f64(const double* keys, int64_t n, int32_t descending, int64_t* idx_out, void* ws,
                                    size_t ws_bytes, void* stream) {
  LVSK_REQUIRE(n >= 0, LVSK_ERR_DIMENSION, "negative length");
  if (n == 0) return LVSK_OK;
  Carve c(ws, ws_bytes);
  uint64_t* k64 = c.take<uint64_t>(n);
  auto rb = radix::carve<uint64_t>(c, n);
  uint32_t* chist = c.take<uint32_t>(static_cast<size_t>(256) * AS_MAX_G);
  uint32_t* totals = c.take<uint32_t>(8 * 256);
  unsigned long long* ctl = c.take<unsigned long long>(4);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  cudaStream_t st = as_stream(stream);
  int G = coop_grid();
  if (inflight_passes() >= 2) {
    // another pass runs concurrently: fuller CTAs leave SMs to it (the grid
    // barriers, not the key traffic, bound a pass at these sizes)
    const int64_t want = (n + AS_INFLIGHT_CHUNK - 1) / AS_INFLIGHT_CHUNK;
    if (want < G) G = static_cast<int>(want < 1 ? 1 : want);
  }
  if (n <= AS_MAX_N && G >= 1 && getenv("LVSK_ARGSORT_CLASSIC") == nullptr) {
    // ctl: [0] OR = 0, [1] AND = ~0, [2] barrier count = 0, [3] flag = 0
    cudaError_t e = cudaMemsetAsync(ctl, 0, 4 * sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctl + 1, 0xFF, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(totals, 0, 8 * 256 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "argsort memset");
    AsArgs a;
    a.in = keys;
    a.n = n;
    a.descending = descending;
    a.out = idx_out;
    a.kb[0] = k64;
    a.kb[1] = rb.keys[0];
    a.kb[2] = rb.keys[1];
    a.vb[0] = rb.vals[0];
    a.vb[1] = rb.vals[1];
    a.hist = chist;
    a.totals = totals;
    a.orand = ctl;
    a.bar = reinterpret_cast<unsigned int*>(ctl + 2);
    a.flag = reinterpret_cast<unsigned int*>(ctl + 3);
    static unsigned long long* trace = nullptr;
    const bool tracing = getenv("LVSK_SORT_TRACE") != nullptr;
    if (tracing && trace == nullptr) cudaMalloc(&trace, 512 * sizeof(unsigned long long));
    if (tracing) cudaMemsetAsync(trace, 0, 512 * sizeof(unsigned long long), st);
    a.trace = tracing ? trace : nullptr;
    void* args[] = {(void*)&a};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(argsort_coop_kernel), dim3(G), dim3(AS_THREADS), args,
                                    AS_SMEM, st);
    if (e != cudaSuccess) return cuda_status(e, "argsort coop launch");
    if (tracing) {
      unsigned long long h[64];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
      fprintf(stderr, "argsort n=%lld G=%d: phase0->bar %.1f us;", (long long)n, G, (h[1] - h[0]) / 1e3);
      for (int p = 0; p < 8; ++p)
        if (h[4 * p + 2])
          fprintf(stderr, " p%d hist-bar %.1f offs %.1f scatter %.1f |", p, (h[4 * p + 3] - h[4 * p + 2]) / 1e3,
                  (h[4 * p + 4] - h[4 * p + 3]) / 1e3, (h[4 * p + 5] - h[4 * p + 4]) / 1e3);
      if (h[40]) fprintf(stderr, " fixup %.1f (max over CTAs %.1f) bar %.1f", (h[41] - h[40]) / 1e3, h[50] / 1e3,
                         (h[42] - h[41]) / 1e3);
      fprintf(stderr, " total(from p0 end) %.1f\n", (h[42] ? h[42] : h[1]) > h[0] ? ((h[42] ? h[42] : h[1]) - h[0]) / 1e3 : 0.0);
    }
    return LVSK_OK;
  }
  argsort_keys_kernel<<<grid_cap(n), 256, 0, st>>>(keys, n, descending, k64);
  LVSK_CHECK_LAUNCH("argsort keys");
  return radix::sort_pairs<uint64_t, int64_t>(k64, nullptr, n, 64, rb, nullptr, idx_out, st);
}

extern "C" size_t lvsk_merge_runs_workspace_bytes(int64_t n, int32_t runs) {
  Measure m;
  m.take<uint64_t>(n);
  m.take<uint64_t>(n);
  m.take<uint32_t>(n);
  m.take<uint32_t>(n);
  m.take<int64_t>(static_cast<size_t>(n / KM_CHUNK + (runs < 1 ? 1 : runs) + 1));
  return m.off;
}

extern "C" int32_t lvsk_merge_argsort_runs(const double* sorted_keys, const int32_t* run_idx, const int64_t* run_off,
                                           int32_t runs, int32_t descending, int64_t* idx_out, void* ws,
                                           size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(runs >= 1 && runs <= KM_MAX_RUNS, LVSK_ERR_CONFIGURATION, "need 1 <= runs <= %d", KM_MAX_RUNS);
  LVSK_REQUIRE(run_off != nullptr && run_off[0] == 0, LVSK_ERR_CONFIGURATION, "run offsets must start at 0");
  for (int q = 0; q < runs; ++q)
    LVSK_REQUIRE(run_off[q + 1] >= run_off[q], LVSK_ERR_DIMENSION, "run offsets must be nondecreasing");
  const int64_t n = run_off[runs];
  LVSK_REQUIRE(n < (int64_t{1} << 32), LVSK_ERR_CAPACITY, "at most 2^32 keys");
  if (n == 0) return LVSK_OK;
  Carve c(ws, ws_bytes);
  uint64_t* k0 = c.take<uint64_t>(n);
  uint64_t* k1 = c.take<uint64_t>(n);
  uint32_t* i0 = c.take<uint32_t>(n);
  uint32_t* i1 = c.take<uint32_t>(n);
  int64_t* split = c.take<int64_t>(static_cast<size_t>(n / KM_CHUNK + runs + 1));
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  cudaStream_t st = as_stream(stream);
  // offsets travel as kernel parameters: no host-to-device copy (a pageable
  // copy would block the host until the stream drains)
  KmOffsets O;
  for (int q = 0; q <= runs; ++q) O.off[q] = run_off[q];
  km_check_kernel<<<grid_cap(n), 256, 0, st>>>(run_idx, O, runs, n, flags);
  LVSK_CHECK_LAUNCH("merge check");
  std::vector<int64_t> off(run_off, run_off + runs + 1);
  uint64_t *kin = k0, *kout = k1;
  uint32_t *iin = i0, *iout = i1;
  bool first = true;
  for (;;) {
    const int R = static_cast<int>(off.size()) - 1;
    const bool last = R <= 2;
    KmPairs P;
    std::vector<int64_t> noff;
    noff.push_back(0);
    int64_t chunks = 0;
    P.npairs = 0;
    for (int q = 0; q < R; q += 2) {
      const int64_t la = off[q + 1] - off[q], lb = q + 1 < R ? off[q + 2] - off[q + 1] : 0;
      P.a0[P.npairs] = off[q];
      P.la[P.npairs] = la;
      P.lb[P.npairs] = lb;
      P.r0[P.npairs] = off[q];
      P.r1[P.npairs] = off[q] + la;
      P.chunk0[P.npairs] = chunks;
      chunks += (la + lb + KM_CHUNK - 1) / KM_CHUNK;
      ++P.npairs;
      noff.push_back(off[q] + la + lb);
    }
    P.chunk0[P.npairs] = chunks;
    KmSrc S;
    S.kimg = kin;
    S.gidx = iin;
    S.skeys = sorted_keys;
    S.ridx = run_idx;
    S.descending = descending;
    if (chunks > 0) {
      const unsigned sg = static_cast<unsigned>((chunks * 32 + 255) / 256), mg = static_cast<unsigned>(chunks);
      if (first) {
        km_split_kernel<1><<<sg, 256, 0, st>>>(P, chunks, S, split);
        if (last)
          km_merge_kernel<1, true><<<mg, KM_THREADS, 0, st>>>(P, S, split, nullptr, nullptr, idx_out);
        else
          km_merge_kernel<1, false><<<mg, KM_THREADS, 0, st>>>(P, S, split, kout, iout, nullptr);
      } else {
        km_split_kernel<0><<<sg, 256, 0, st>>>(P, chunks, S, split);
        if (last)
          km_merge_kernel<0, true><<<mg, KM_THREADS, 0, st>>>(P, S, split, nullptr, nullptr, idx_out);
        else
          km_merge_kernel<0, false><<<mg, KM_THREADS, 0, st>>>(P, S, split, kout, iout, nullptr);
      }
      LVSK_CHECK_LAUNCH("merge round");
    }
    if (last) break;
    off.swap(noff);
    if (!first) {
      std::swap(kin, kout);
      std::swap(iin, iout);
    } else {  // round 1 wrote (k1, i1): read them next, write (k0, i0)
      kin = k1;
      iin = i1;
      kout = k0;
      iout = i0;
    }
    first = false;
  }
  return LVSK_OK;
}
