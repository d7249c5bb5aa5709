// K3 v3 (fp32 X) — SRHT in ONE pass over X: block WHT in shared memory +
// sampled combine in registers.  Reference: SketchState.data SRHT branch and
// fwht (pkg/src/levsketch/sketch.py:248-257, 364-385): SX = fwht(D X)[sample]
// / divisor, signs/sample drawn on the host exactly as sketch.py:220-224.
//
// Why a different factorisation.  H_m = H_hi (x) H_lo with the low B = 11
// row bits inside a block:  for sampled row p = (p_hi, p_lo)
//     SX[p] = sum_j (-1)^popc(p_hi & j) * W_j[p_lo],   W_j = H_2048 (D X)_block j
// The two-pass kernels (srht.cu) transform the low 16 bits completely and
// round-trip a 64 MB intermediate through L2/DRAM (3 x 2 GB of traffic at C3).
// Here the high bits are only ever evaluated at the k sampled rows, so the
// intermediate never leaves the SM: a persistent CTA owns one 8-column slab
// (32 B of every row) and keeps the k x 8 sampled outputs of that slab in
// fp32 registers (k <= 4096: 16 samples x 8 columns per thread), streams the
// 2048-row blocks of its slab with TMA (double-buffered), applies the row
// signs (bit-packed, XOR of the float sign bit), runs the 11-level WHT as two
// register passes through shared memory (row bits 2-7, then 0,1,8,9,10, with
// an XOR-swizzled layout that keeps both passes bank-conflict free), and adds
// (-1)^popc(p_hi & j) * W_j[p_lo] into its accumulators.  Every 128 blocks the
// fp32 accumulators are stored (store-only) as one partial run, and a final
// kernel sums the runs in a fixed order in fp64 and divides: the result is
// deterministic, error ~2e-7 relative (fp32 within a run, fp64 across runs).
//
// X is read exactly once.  Eight consecutive CTAs own the eight slabs of one
// 256-byte column segment and walk the same block sequence, so a 256 B L2
// line fetched for one of them is consumed by the other seven while it is
// still resident.  Algorithmic bytes: n*d*4 (+ k*d*8 written).
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace lvsk {
namespace srht3 {

constexpr int B = 11;                    // in-block row bits
constexpr int ROWS = 1 << B;             // 2048 rows per block
constexpr int W = 8;                     // fp32 columns per slab (32 B)
constexpr int OCT = 8;                   // slabs per 256 B column segment (CTAs per group)
constexpr int THREADS = 256;
constexpr int SPT = 16;                  // samples per thread
constexpr int KMAX = SPT * THREADS;      // 4096
constexpr int TILE_BYTES = ROWS * W * 4;  // 64 KB
constexpr int SIGN_BYTES = ROWS / 8;      // 256 B of sign bits per block
constexpr int STAGE_BYTES = TILE_BYTES + SIGN_BYTES;
constexpr int BOX_ROWS = 256;
constexpr int FLUSH = 128;               // blocks per fp32 accumulation run
constexpr int SMEM_BYTES = 2 * STAGE_BYTES + KMAX * 8 + 64 + 128;

// XOR swizzle of rows inside each 4-row group: bits 0,1 ^= bits 2,3
__device__ __forceinline__ int swz(int r) { return r ^ ((r >> 2) & 3); }

template <int N>
__device__ __forceinline__ void wht(float (&v)[N]) {
#pragma unroll
  for (int h = 1; h < N; h <<= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i & h) == 0) {
        const float a = v[i], b = v[i + h];
        v[i] = a + b;
        v[i + h] = a - b;
      }
    }
  }
}

// packed fp32 pairs (sm_100 FADD2 / FFMA2)
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0,%1}, rr;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "sub.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0,%1}, rr;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc, rr;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rr, ra, rb, rc;\n\tmov.b64 {%0,%1}, rr;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// WHT of the 2N values x[m] = v[m].x, x[m + N] = v[m].y: the butterflies over
// the low log2(N) index bits run packed, the top bit inside each pair.
template <int N>
__device__ __forceinline__ void wht_packed(float2 (&v)[N]) {
#pragma unroll
  for (int h = 1; h < N; h <<= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i & h) == 0) {
        const float2 a = v[i], b = v[i + h];
        v[i] = add2(a, b);
        v[i + h] = sub2(a, b);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = make_float2(v[i].x + v[i].y, v[i].x - v[i].y);
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

struct Params {
  const uint32_t* signbits;  // m/32 words, bit set = negative sign (nullptr: no flip)
  const uint2* slots;        // KMAX slots {(p & 2047) | (p >> 11) << 11, sample index t or ~0u}
  float* partial;            // [ctas][rmax][k][8] fp32 runs
  int64_t rmax;              // runs per CTA (capacity)
  int64_t k;
  int64_t jblocks;           // active 2048-row blocks (ceil(n / 2048))
  int64_t octets;            // ceil(slabs / 8)
  int64_t groups;            // CTA groups of 8
  int64_t j0;                // global index of the first block (row0 / 2048)
};

__device__ __forceinline__ void group_range(const Params& P, int64_t g, int64_t& lo, int64_t& hi) {
  const int64_t T = P.octets * P.jblocks;
  lo = g * T / P.groups;
  hi = (g + 1) * T / P.groups;
}

__global__ void __launch_bounds__(THREADS, 1) srht_sampled_kernel(const __grid_constant__ CUtensorMap mx, Params P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint32_t* meta_s = reinterpret_cast<uint32_t*>(smem + 2 * STAGE_BYTES);  // row | p_hi << 11
  uint32_t* samp_s = meta_s + KMAX;                                          // sample index or ~0u
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGE_BYTES + KMAX * 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t g = blockIdx.x / OCT;
  const int o = blockIdx.x % OCT;
  int64_t lo, hi;
  group_range(P, g, lo, hi);
  if (lo >= hi) return;

  const int k = static_cast<int>(P.k);
  for (int t = tid; t < KMAX; t += THREADS) {
    const uint2 e = P.slots[t];
    meta_s[t] = e.x;
    samp_s[t] = e.y;
  }
  if (tid == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint64_t pol = tc::l2_policy_evict_first();
  auto issue = [&](int64_t task, int s) {
    const int64_t oct = task / P.jblocks, j = task % P.jblocks;
    const int col = static_cast<int>((oct * OCT + o) * W);
    const int row0 = static_cast<int>(j * ROWS);
    tc::mbar_expect_tx(&full[s], P.signbits ? STAGE_BYTES : TILE_BYTES);
#pragma unroll
    for (int b = 0; b < ROWS / BOX_ROWS; ++b)
      tc::tma_load_2d(&mx, &full[s], smem + s * STAGE_BYTES + b * BOX_ROWS * W * 4, col, row0 + b * BOX_ROWS, pol);
    if (P.signbits) bulk_g2s(smem + s * STAGE_BYTES + TILE_BYTES, P.signbits + j * (ROWS / 32), SIGN_BYTES, &full[s]);
  };
  if (tid == 0) {
    issue(lo, 0);
    if (lo + 1 < hi) issue(lo + 1, 1);
  }

  float2 acc[SPT][W / 2];
#pragma unroll
  for (int u = 0; u < SPT; ++u)
#pragma unroll
    for (int c = 0; c < W / 2; ++c) acc[u][c] = make_float2(0.f, 0.f);

  int run = 0;           // fp32 partial runs written so far
  int runs = 0;          // blocks accumulated in the current run
  int64_t cur_oct = lo / P.jblocks;

  // store-only: each run of <= FLUSH blocks of one column segment becomes
  // one fp32 partial; the reduce kernel adds the runs in order in fp64
  auto flush = [&]() {
    float* base = P.partial + ((static_cast<int64_t>(blockIdx.x) * P.rmax + run) * P.k) * W;
    const int rot = (lane & 1) * 4;  // see the gather: odd lanes hold columns 4-7 first
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const uint32_t t = samp_s[tid + THREADS * u];
      if (t != ~0u) {
        float* p = base + static_cast<int64_t>(t) * W;
        *reinterpret_cast<float4*>(p + rot) = make_float4(acc[u][0].x, acc[u][0].y, acc[u][1].x, acc[u][1].y);
        *reinterpret_cast<float4*>(p + (rot ^ 4)) = make_float4(acc[u][2].x, acc[u][2].y, acc[u][3].x, acc[u][3].y);
      }
#pragma unroll
      for (int c = 0; c < W / 2; ++c) acc[u][c] = make_float2(0.f, 0.f);
    }
    ++run;
    runs = 0;
  };

  const int64_t jb = P.jblocks;
  int64_t oct = cur_oct;
  uint32_t j = static_cast<uint32_t>(lo - oct * jb);
  for (int64_t task = lo; task < hi; ++task, ++j) {
    const int it = static_cast<int>(task - lo);
    const int s = it & 1;
    if (j == jb) {
      j = 0;
      ++oct;
    }
    if (oct != cur_oct) {  // crossed into the next column segment
      if (runs > 0) flush();
      cur_oct = oct;
    }
    const uint32_t jg = j + static_cast<uint32_t>(P.j0);  // global block index (high row bits)
    tc::mbar_wait(&full[s], static_cast<uint32_t>((it >> 1) & 1));
    float* T = reinterpret_cast<float*>(smem + s * STAGE_BYTES);
    const uint32_t* sb = reinterpret_cast<const uint32_t*>(smem + s * STAGE_BYTES + TILE_BYTES);

    // ---- pass A: row bits 2..7 (lanes: column, bits 0-1; warps: bits 8-10)
    {
      const int c = lane & 7, b01 = lane >> 3;
      const int rbase = b01 + 256 * warp;
      float2 v[32];  // v[m] = (x[m], x[m + 32]), x[i] = row rbase + 4 i
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = make_float2(T[(rbase + 4 * m) * W + c], T[(rbase + 4 * (m + 32)) * W + c]);
      if (P.signbits) {
        uint32_t wv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) wv[q] = sb[8 * warp + q] >> b01;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
          const int i0 = m, i1 = m + 32;
          v[m].x = __uint_as_float(__float_as_uint(v[m].x) ^ ((wv[i0 >> 3] << (31 - 4 * (i0 & 7))) & 0x80000000u));
          v[m].y = __uint_as_float(__float_as_uint(v[m].y) ^ ((wv[i1 >> 3] << (31 - 4 * (i1 & 7))) & 0x80000000u));
        }
      }
      wht_packed<32>(v);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        T[(256 * warp + 4 * m + (b01 ^ (m & 3))) * W + c] = v[m].x;
        T[(256 * warp + 4 * (m + 32) + (b01 ^ (m & 3))) * W + c] = v[m].y;
      }
    }
    __syncthreads();
    // ---- pass B: row bits 0,1,8,9,10 (lanes: column, bits 2-3; warps: bits 4-6); the two
    // halves of row bit 7 are independent transforms and ride in the two lanes of each pair
    {
      const int c = lane & 7, b23 = lane >> 3;
      const int rb = 4 * b23 + 16 * warp;
      // u = 0..31 over row bits 0,1 (u & 3) and 8,9,10 (u >> 2)
      auto at = [&](int u) { return (rb + 256 * (u >> 2) + ((u & 3) ^ b23)) * W + c; };
      float2 v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = make_float2(T[at(u)], T[at(u) + 128 * W]);
#pragma unroll
      for (int h = 1; h < 32; h <<= 1) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if ((i & h) == 0) {
            const float2 x = v[i], y = v[i + h];
            v[i] = add2(x, y);
            v[i + h] = sub2(x, y);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        T[at(u)] = v[u].x;
        T[at(u) + 128 * W] = v[u].y;
      }
    }
    __syncthreads();
    // ---- sampled combine: acc[t] += (-1)^popc(p_hi & j) * W_j[p_lo]
    {
      const int h0 = lane & 1;
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        const uint32_t mt = meta_s[tid + THREADS * u];
        const int q = static_cast<int>(mt & (ROWS - 1));
        const uint32_t sbit = static_cast<uint32_t>(__popc((mt >> B) & jg) & 1) << 31;
        const float* row = T + swz(q) * W;
        const float4 a = *reinterpret_cast<const float4*>(row + 4 * h0);
        const float4 b = *reinterpret_cast<const float4*>(row + 4 * (h0 ^ 1));
        // lanes with h0 = 1 keep columns 4-7 in acc[u][0..3] (undone in flush)
        const float sg1 = __uint_as_float(0x3f800000u | sbit);
        const float2 sg = make_float2(sg1, sg1);
        acc[u][0] = fma2(make_float2(a.x, a.y), sg, acc[u][0]);
        acc[u][1] = fma2(make_float2(a.z, a.w), sg, acc[u][1]);
        acc[u][2] = fma2(make_float2(b.x, b.y), sg, acc[u][2]);
        acc[u][3] = fma2(make_float2(b.z, b.w), sg, acc[u][3]);
      }
    }
    __syncthreads();  // stage s is free
    if (tid == 0 && task + 2 < hi) issue(task + 2, s);
    if (++runs == FLUSH) flush();
  }
  if (runs > 0) flush();
}

// SX[t][col] = sum over the runs of the CTAs covering col's segment (fixed
// order: groups ascending, runs ascending) / divisor.  One thread per
// (8-column slab, sample), samples fastest (coalesced run reads); the run table of every (segment, group) is built
// in shared memory first.
__global__ void srht_sampled_reduce_kernel(Params P, int64_t d, double divisor, double* __restrict__ SX,
                                           int32_t* flags) {
  extern __shared__ int2 runs_s[];  // [octets][groups] = (first run, end run), empty if equal
  const int64_t G = P.groups;
  for (int64_t e = threadIdx.x; e < P.octets * G; e += blockDim.x) {
    const int64_t oct = e / G, g = e % G;
    int64_t lo, hi;
    group_range(P, g, lo, hi);
    int2 v = make_int2(0, 0);
    if (lo < hi) {
      const int64_t first = lo / P.jblocks, last = (hi - 1) / P.jblocks;
      if (oct >= first && oct <= last) {
        const int64_t b = (first + 1) * P.jblocks;
        const int64_t n0 = ((hi < b ? hi : b) - lo + FLUSH - 1) / FLUSH;
        v = oct == first ? make_int2(0, static_cast<int>(n0))
                         : make_int2(static_cast<int>(n0), static_cast<int>(n0 + (hi - b + FLUSH - 1) / FLUSH));
      }
    }
    runs_s[e] = v;
  }
  __syncthreads();
  const int64_t slabs = (d + W - 1) / W;
  const int64_t total = P.k * slabs;
  bool bad = false;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t slab = e / P.k, t = e % P.k, oct = slab / OCT, o = slab % OCT;
    double acc[W];
#pragma unroll
    for (int c = 0; c < W; ++c) acc[c] = 0.0;
    for (int64_t g = 0; g < G; ++g) {
      const int2 rr = runs_s[oct * G + g];
      const float* base = P.partial + ((g * OCT + o) * P.rmax * P.k + t) * W;
      for (int r = rr.x; r < rr.y; ++r) {
        const float4 a = *reinterpret_cast<const float4*>(base + static_cast<int64_t>(r) * P.k * W);
        const float4 b = *reinterpret_cast<const float4*>(base + static_cast<int64_t>(r) * P.k * W + 4);
        acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
        acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
      }
    }
    double* out = SX + t * d + slab * W;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      if (slab * W + c < d) {
        const double v = acc[c] / divisor;
        bad |= !isfinite(v);
        out[c] = v;
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
}

__global__ void srht_pack_kernel(const int8_t* __restrict__ signs, int64_t words, uint32_t* __restrict__ bits) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t b = 0;
    const int8_t* s = signs + w * 32;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) b |= static_cast<uint32_t>(s[i] < 0) << i;
    bits[w] = b;
  }
}

// Sample -> accumulator slot.  Slot s lives in thread s % 256, register set
// s / 256; in the gather, lane l reads its row halves in the order
// (l & 1, l & 1 ^ 1), so a quarter-warp is conflict-free when lane l's row
// sits in 4-row position (l >> 1) & 3 (bank group 2 * pos + half).  Samples
// go to slots of their own class while those last, the rest to free slots.
// (Which slot a sample lands in does not change its arithmetic, so atomics
// here keep the result deterministic.)
__global__ void __launch_bounds__(1024) srht_slots_kernel(const int64_t* __restrict__ sample, int64_t k, int64_t m,
                                                          uint2* __restrict__ slots, int32_t* flags) {
  constexpr int PER = KMAX / 4;
  __shared__ int cnt[4], ovf;
  __shared__ uint32_t over[2 * KMAX];
  if (threadIdx.x < 4) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) ovf = 0;
  for (int s = threadIdx.x; s < KMAX; s += blockDim.x) slots[s] = make_uint2(0u, ~0u);
  __syncthreads();
  auto slot_of = [](int c, int pos) { return (pos & 1) | (c << 1) | ((pos >> 1) << 3); };
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const int64_t p = sample[t];
    if (p < 0 || p >= m) atomicOr(flags, LVSK_FLAG_BADINDEX);
    const uint64_t pu = static_cast<uint64_t>(p) & (static_cast<uint64_t>(m) - 1);
    const uint32_t q = static_cast<uint32_t>(pu & (ROWS - 1));
    const uint2 e = make_uint2(q | static_cast<uint32_t>(pu >> B) << B, static_cast<uint32_t>(t));
    const int c = static_cast<int>((q ^ (q >> 2)) & 3);
    const int pos = atomicAdd(&cnt[c], 1);
    if (pos < PER) {
      slots[slot_of(c, pos)] = e;
    } else {
      const int i = atomicAdd(&ovf, 1);
      over[2 * i] = e.x;
      over[2 * i + 1] = e.y;
    }
  }
  __syncthreads();
  // the i-th overflow sample takes the i-th free slot (classes in order)
  for (int i = threadIdx.x; i < ovf; i += blockDim.x) {
    int rem = i;
    for (int c = 0; c < 4; ++c) {
      const int fr = cnt[c] < PER ? PER - cnt[c] : 0;
      if (rem < fr) {
        slots[slot_of(c, cnt[c] + rem)] = make_uint2(over[2 * i], over[2 * i + 1]);
        break;
      }
      rem -= fr;
    }
  }
}

struct Shape {
  int64_t jblocks, octets, groups, ctas, rmax;
};

static Shape shape(int64_t n, int64_t d) {
  Shape s;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  s.jblocks = (n + ROWS - 1) / ROWS;
  const int64_t slabs = (d + W - 1) / W;
  s.octets = (slabs + OCT - 1) / OCT;
  // a group's range spans at most two column segments: groups >= octets
  s.groups = sms / OCT > s.octets ? sms / OCT : s.octets;
  const int64_t T = s.octets * s.jblocks;
  if (s.groups > T) s.groups = T;
  s.ctas = s.groups * OCT;
  s.rmax = ((T + s.groups - 1) / s.groups + FLUSH - 1) / FLUSH + 1;
  return s;
}

}  // namespace srht3

// Usable for fp32 X with 16-byte aligned rows, m >= 2^11, k <= 4096.
bool srht_sampled_ok(const float* X, int64_t n, int64_t d, int64_t ldx, int64_t m, int64_t k, int64_t row0) {
  if (row0 % srht3::ROWS != 0 || row0 + n > m) return false;
  if (getenv("LVSK_SRHT_V2") != nullptr) return false;
  return m >= srht3::ROWS && k <= srht3::KMAX && d <= 4096 && m <= (int64_t{1} << 32) && n < (int64_t{1} << 31) &&
         d % 4 == 0 && ldx % 4 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0;
}

size_t srht_sampled_workspace(int64_t n, int64_t d, int64_t m, int64_t k) {
  const srht3::Shape s = srht3::shape(n, d);
  Measure ms;
  ms.take<uint32_t>(static_cast<size_t>(m / 32));
  ms.take<uint2>(srht3::KMAX);
  ms.take<float>(static_cast<size_t>(s.ctas) * s.rmax * k * srht3::W);
  return ms.off;
}

int32_t srht_sampled(const float* X, int64_t n, int64_t d, int64_t ldx, int64_t row0, int64_t m,
                     const int8_t* signs, const int64_t* sample, int64_t k, double divisor, double* SX, void* ws,
                     size_t ws_bytes, int32_t* flags, cudaStream_t st) {
  using namespace srht3;
  const Shape S = shape(n, d);
  Carve cv(ws, ws_bytes);
  uint32_t* bits = cv.take<uint32_t>(static_cast<size_t>(m / 32));
  uint2* slots = cv.take<uint2>(KMAX);
  float* partial = cv.take<float>(static_cast<size_t>(S.ctas) * S.rmax * k * W);
  LVSK_REQUIRE(cv.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", cv.off, ws_bytes);
  CUtensorMap mx;
  if (!tc::make_map(&mx, X, d, n, ldx * 4, W, BOX_ROWS, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    CU_TENSOR_MAP_SWIZZLE_NONE)) {
    set_error("cuTensorMapEncodeTiled failed (SRHT X)");
    return LVSK_ERR_CUDA;
  }
  const int64_t words = signs ? S.jblocks * (ROWS / 32) : 0;
  if (words) srht_pack_kernel<<<296, 256, 0, st>>>(signs + row0, words, bits);
  srht_slots_kernel<<<1, 1024, 0, st>>>(sample, k, m, slots, flags);
  LVSK_CHECK_LAUNCH("srht pack");
  const int32_t arc = ensure_smem_attr(reinterpret_cast<const void*>(srht_sampled_kernel), SMEM_BYTES,
                                       "srht sampled smem attribute");
  if (arc != LVSK_OK) return arc;
  Params P{signs ? bits : nullptr, slots, partial, S.rmax, k, S.jblocks, S.octets, S.groups, row0 / ROWS};
  srht_sampled_kernel<<<static_cast<unsigned>(S.ctas), THREADS, SMEM_BYTES, st>>>(mx, P);
  LVSK_CHECK_LAUNCH("srht sampled");
  const size_t rsm = static_cast<size_t>(S.octets * S.groups) * sizeof(int2);
  LVSK_REQUIRE(rsm <= 48 * 1024, LVSK_ERR_CONFIGURATION, "SRHT: d=%lld too wide for the run table", (long long)d);
  const int64_t rthreads = k * ((d + W - 1) / W);
  srht_sampled_reduce_kernel<<<static_cast<unsigned>((rthreads + 255) / 256), 256, rsm, st>>>(P, d, divisor, SX,
                                                                                               flags);
  LVSK_CHECK_LAUNCH("srht sampled reduce");
  return LVSK_OK;
}

}  // namespace lvsk

using namespace lvsk;

extern "C" int32_t lvsk_srht_rows(const float* X, int64_t n, int64_t d, int64_t ldx, int64_t row0, int64_t m,
                                  const int8_t* signs, const int64_t* sample, int64_t k, double divisor, double* SX,
                                  void* ws, size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(n >= 1 && d >= 1 && ldx >= d && row0 >= 0, LVSK_ERR_DIMENSION, "bad shape n=%lld d=%lld row0=%lld",
               (long long)n, (long long)d, (long long)row0);
  LVSK_REQUIRE(m >= row0 + n && (m & (m - 1)) == 0, LVSK_ERR_CONFIGURATION,
               "m=%lld must be a power of two >= row0 + n", (long long)m);
  LVSK_REQUIRE(k >= 1 && k <= m && divisor != 0.0, LVSK_ERR_CONFIGURATION, "SRHT needs 1 <= k <= m, divisor != 0");
  LVSK_REQUIRE(getenv("LVSK_SRHT_V2") == nullptr && srht_sampled_ok(X, n, d, ldx, m, k, row0), LVSK_ERR_UNSUPPORTED,
               "row-block SRHT needs fp32 16-byte aligned rows, d %% 4 == 0, d <= 4096, k <= 4096, row0 %% 2048 == 0");
  return srht_sampled(X, n, d, ldx, row0, m, signs, sample, k, divisor, SX, ws, ws_bytes, flags, as_stream(stream));
}
