// K6-TC — the CSR leverage pass ||x_i M||^2 (C4: d = 4096, r = 128) with the
// hot columns on the tensor cores.  Reference: _block_scores
// (pkg/src/levsketch/leverage.py:88-95) on the densified rows.
//
// The SIMT kernel (csr.cu) gathers a 512-byte fp32 row of M per nonzero
// (164 GB through L1 at C4) and is L1-bandwidth bound.  Bag-of-words column
// ids are Zipf-ranked, so the first H = 128 column ids carry half of the
// nonzeros (C4: 50 %), and every row's sorted column list starts with them.
// Per 128-row tile:
//   * 8 row-worker warps (16 rows each) scatter each row's hot prefix
//     (columns < H) into two bf16 planes x_hi = bf16(x), x_lo = bf16(x - x_hi)
//     of a dense [128 x H] A tile (K-major SW128), and gather the cold suffix
//     exactly as the SIMT kernel does (warp per row, lane owns 4 of the 128
//     columns of u, fp32) into u_cold [128][128] in shared memory;
//   * one thread issues tcgen05.mma kind::f16 against the resident B operand
//     [M_hi | M_lo]^T (N = 256, K = H, built once per CTA from the fp32 M):
//     D[:, 0:128] = x_hi M_hi, D[:, 128:256] = x_hi M_lo + x_lo M_hi
//     (fp32 TMEM accumulators, double-buffered);
//   * 4 epilogue warps (one row per thread) read u_hot = D_lo + D_hi from
//     TMEM and u_cold from shared memory (XOR-swizzled, conflict-free) and
//     write sum_c (u_hot + u_cold)^2 as float64.
// Precision: x_hi + x_lo carries 16 significand bits of x, M_hi + M_lo 16 of
// M, products exact, fp32 accumulation — the error class of the K5 tcgen05
// kernels (~1e-6 relative at C4).
#include <cstdlib>

#include "tc_common.cuh"

namespace lvsk {
namespace k6tc {

using namespace tc;

constexpr int H = 128;        // hot columns = MMA K
constexpr int R = 128;        // JL width r (u columns)
constexpr int TR = 128;       // rows per tile
constexpr int RW = 16;        // row-worker warps (TR / RW rows each)
constexpr int RPW = TR / RW;  // rows per worker warp
constexpr int EW = 4;         // epilogue warps
constexpr int THREADS = 32 * (1 + RW + EW);
constexpr int B_BLOCK = 2 * R * 128;   // one 64-element K block of B: 256 N-rows x 128 B = 32 KB
constexpr int A_BLOCK = TR * 128;      // one 64-element K block of A: 128 rows x 128 B = 16 KB
constexpr int OFF_B = 0;               // 2 K blocks
constexpr int KB = H / 64;              // 64-element K blocks
constexpr int OFF_AH = OFF_B + KB * B_BLOCK;
constexpr int OFF_AL = OFF_AH + KB * A_BLOCK;
constexpr int OFF_UC = OFF_AL + KB * A_BLOCK;  // u_cold [128][128] fp32
constexpr int OFF_BAR = OFF_UC + TR * R * 4;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;
// kind::f16, F32 accumulate, bf16 A / B K-major, M = 128
constexpr uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(TR >> 4) << 24);
}

// byte offset of element (row, k) in a K-major SW128 operand of `block` bytes per 64-element K block
__device__ __forceinline__ uint32_t sw128_off(int row, int k, int block) {
  const int kb = k >> 6, kin = k & 63;
  return static_cast<uint32_t>(kb * block + row * 128 + ((((kin >> 3) ^ (row & 7))) << 4) + ((kin & 7) << 1));
}

__device__ __forceinline__ uint16_t bf16_bits(float v) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}

template <typename V>
__global__ void __launch_bounds__(THREADS, 1)
    csr_rowsumsq_tc_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                           const V* __restrict__ val, int64_t n, int64_t d, const float* __restrict__ M,
                           double* __restrict__ scores, int32_t* flags) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* ready = bars;             // RW worker warps: A tile + u_cold written
  uint64_t* afree = ready + 1;        // MMA done reading the A tile
  uint64_t* ucfree = afree + 1;       // EW epilogue warps done reading u_cold
  uint64_t* accfull = ucfree + 1;     // [2]
  uint64_t* accempty = accfull + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  float* ucold = reinterpret_cast<float*>(smem + OFF_UC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int64_t base0 = row_ptr[0];

  if (threadIdx.x == 0) {
    mbar_init(ready, RW);
    mbar_init(afree, 1);
    mbar_init(ucfree, EW);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // resident B operand: B[n][k] = M_hi[k][n] (n < R), M_lo[k][n - R] (n >= R), K-major SW128
  for (int e = threadIdx.x; e < 2 * R * H; e += THREADS) {
    const int nn = e / H, k = e - nn * H;
    const int c = nn < R ? nn : nn - R;
    const float m = k < d ? M[static_cast<int64_t>(k) * R + c] : 0.f;
    const float mh = __bfloat162float(__float2bfloat16_rn(m));
    *reinterpret_cast<uint16_t*>(smem + OFF_B + sw128_off(nn, k, B_BLOCK)) = bf16_bits(nn < R ? m : m - mh);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B written through the generic proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---- MMA issuer
    if (lane == 0) {
      uint32_t lt = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
        mbar_wait(ready, lt & 1u);
        mbar_wait(&accempty[ab], aph ^ 1u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A tile written through the generic proxy
        tc_fence_after();
        const uint32_t dt = tmem_base + ab * 256;
#pragma unroll
        for (int kb = 0; kb < H / 64; ++kb) {
          const uint64_t ah = sw128_desc(smem_u32(smem + OFF_AH + kb * A_BLOCK));
          const uint64_t al = sw128_desc(smem_u32(smem + OFF_AL + kb * A_BLOCK));
          const uint64_t b = sw128_desc(smem_u32(smem + OFF_B + kb * B_BLOCK));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            umma_f16(dt, ah + 2 * kk, b + 2 * kk, idesc(2 * R), acc);       // x_hi [M_hi | M_lo]
            umma_f16(dt + R, al + 2 * kk, b + 2 * kk, idesc(R), 1u);        // + x_lo M_hi (lo half)
          }
        }
        umma_commit(afree);
        umma_commit(&accfull[ab]);
      }
    }
  } else if (warp <= RW) {
    // ---- row workers: rows RPW w .. RPW w + RPW - 1 of each tile
    const int w = warp - 1;
    int bad = 0;
    uint32_t lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      if (lt > 0) {
        mbar_wait(afree, (lt - 1) & 1u);
        mbar_wait(ucfree, (lt - 1) & 1u);
      }
      // zero this warp's RPW rows of both A planes (RPW rows x 256 B each)
#pragma unroll
      for (int pl = 0; pl < 2; ++pl) {
        uint8_t* a = smem + (pl ? OFF_AL : OFF_AH);
#pragma unroll
        for (int q = lane; q < RPW * KB * 8; q += 32) {  // RPW rows x KB K blocks x 8 chunks of 16 B
          const int rr = q / (KB * 8), blk = (q >> 3) % KB, ch = q & 7;
          *reinterpret_cast<uint4*>(a + blk * A_BLOCK + (RPW * w + rr) * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
        }
      }
      __syncwarp();
      // this warp's RPW row pointers (+1) in one load; the next row's first 96
      // entries are loaded while the current row is gathered
      const int64_t gbase = t * TR + RPW * w;
      int64_t rp = 0;
      if (lane <= RPW) rp = row_ptr[gbase + lane < n ? gbase + lane : n] - base0;
      int32_t cn[3];
      float xn[3];
      auto load3 = [&](int rr, int32_t (&c3)[3], float (&x3)[3]) {
        const int64_t f0 = __shfl_sync(0xFFFFFFFFu, rp, rr), f1 = __shfl_sync(0xFFFFFFFFu, rp, rr + 1);
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int64_t ei = f0 + 32 * b + lane;
          const bool live = ei < f1;
          c3[b] = live ? col[ei] : 0;
          x3[b] = live ? static_cast<float>(val[ei]) : 0.f;
        }
      };
      load3(0, cn, xn);
      for (int rr = 0; rr < RPW; ++rr) {
        const int i = RPW * w + rr;
        float u[4] = {0.f, 0.f, 0.f, 0.f};
        const int64_t e0 = __shfl_sync(0xFFFFFFFFu, rp, rr), e1 = __shfl_sync(0xFFFFFFFFu, rp, rr + 1);
        int32_t cc[3];
        float xx[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          cc[b] = cn[b];
          xx[b] = xn[b];
        }
        if (rr + 1 < RPW) load3(rr + 1, cn, xn);
        for (int64_t e = e0, b = 0; e < e1; e += 32, ++b) {
          const bool live = e + lane < e1;
          int32_t c;
          float x;
          if (b < 3) {
            c = b == 0 ? cc[0] : (b == 1 ? cc[1] : cc[2]);
            x = b == 0 ? xx[0] : (b == 1 ? xx[1] : xx[2]);
          } else {  // rows longer than 96 entries
            c = live ? col[e + lane] : 0;
            x = live ? static_cast<float>(val[e + lane]) : 0.f;
          }
          if (live && (c < 0 || c >= d)) {
            bad |= LVSK_FLAG_BADINDEX;
            c = 0;
            x = 0.f;
          }
          if (live && !isfinite(x)) bad |= LVSK_FLAG_NONFINITE;
          const bool hot = live && c < H;
          if (hot) {  // distinct columns within a row: no two lanes collide
            const float xh = __bfloat162float(__float2bfloat16_rn(x));
            const uint32_t off = sw128_off(i, c, A_BLOCK);
            *reinterpret_cast<uint16_t*>(smem + OFF_AH + off) = bf16_bits(xh);
            *reinterpret_cast<uint16_t*>(smem + OFF_AL + off) = bf16_bits(x - xh);
          }
          // cold entries: broadcast and gather the fp32 M rows, eight rows of M in
          // flight per lane (a row's sorted columns put the cold lanes in one run)
          uint32_t cm = __ballot_sync(0xFFFFFFFFu, live && !hot);
          const int ncold = __popc(cm);
          const int first = cm ? __ffs(cm) - 1 : 0;
          if (ncold > 0 && cm == ((0xFFFFFFFFu >> (32 - ncold)) << first)) {
            for (int b0 = 0; b0 < ncold; b0 += 8) {
              float4 mv[8];
              float xv[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int tl = (first + b0 + j) & 31;
                const int32_t ct = __shfl_sync(0xFFFFFFFFu, c, tl);
                const float xt = __shfl_sync(0xFFFFFFFFu, x, tl);
                const bool ok = b0 + j < ncold;
                xv[j] = ok ? xt : 0.f;
                mv[j] = ok ? __ldg(reinterpret_cast<const float4*>(M + static_cast<int64_t>(ct) * R) + lane)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                u[0] = fmaf(xv[j], mv[j].x, u[0]);
                u[1] = fmaf(xv[j], mv[j].y, u[1]);
                u[2] = fmaf(xv[j], mv[j].z, u[2]);
                u[3] = fmaf(xv[j], mv[j].w, u[3]);
              }
            }
            cm = 0;
          }
          while (cm) {  // general (unsorted) rows
            const int tl = __ffs(cm) - 1;
            cm &= cm - 1;
            const int32_t ct = __shfl_sync(0xFFFFFFFFu, c, tl);
            const float xt = __shfl_sync(0xFFFFFFFFu, x, tl);
            const float4 m = __ldg(reinterpret_cast<const float4*>(M + static_cast<int64_t>(ct) * R) + lane);
            u[0] = fmaf(xt, m.x, u[0]);
            u[1] = fmaf(xt, m.y, u[1]);
            u[2] = fmaf(xt, m.z, u[2]);
            u[3] = fmaf(xt, m.w, u[3]);
          }
        }
        // u_cold row i: 32 float4 blocks, block b stored at b ^ (i & 31)
        *reinterpret_cast<float4*>(ucold + i * R + 4 * (lane ^ (i & 31))) = make_float4(u[0], u[1], u[2], u[3]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(ready);
    }
    const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (any && lane == 0) atomicOr(flags, any);
  } else {
    // ---- epilogue: thread = tile row 32 q + lane
    const int q = warp & 3;
    const int i = 32 * q + lane;
    uint32_t lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
      mbar_wait(ready, lt & 1u);  // orders u_cold(t) before the reads below
      mbar_wait(&accfull[ab], aph);
      tc_fence_after();
      const uint32_t base = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + ab * 256;
      float acc = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < R; c0 += 32) {
        uint32_t vh[32], vl[32];
        tmem_ld32(base + c0, vh);
        tmem_ld32(base + R + c0, vl);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const int blk = (c0 + j) >> 2;
          const float4 uc = *reinterpret_cast<const float4*>(ucold + i * R + 4 * (blk ^ (i & 31)));
          const float a0 = __uint_as_float(vh[j]) + __uint_as_float(vl[j]) + uc.x;
          const float a1 = __uint_as_float(vh[j + 1]) + __uint_as_float(vl[j + 1]) + uc.y;
          const float a2 = __uint_as_float(vh[j + 2]) + __uint_as_float(vl[j + 2]) + uc.z;
          const float a3 = __uint_as_float(vh[j + 3]) + __uint_as_float(vl[j + 3]) + uc.w;
          acc = fmaf(a0, a0, acc);
          acc = fmaf(a1, a1, acc);
          acc = fmaf(a2, a2, acc);
          acc = fmaf(a3, a3, acc);
        }
      }
      const int64_t g = t * TR + i;
      if (g < n) scores[g] = static_cast<double>(acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(ucfree);
        mbar_arrive(&accempty[ab]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512));
  }
}

}  // namespace k6tc

// ---------------------------------------------------------------------------
// K6-TC v2 — a wide hot window streamed through the tensor cores.
//
// v1 above is bound by its gather bytes: the cold half gathers 512 B of M per
// nonzero, 82 GB at C4 in 7.4 ms = 11 TB/s through L1 + L2, next to the L2
// slices' ~6300 B/clk (12 TB/s) cap.  Only fewer gathered bytes make it faster.  A column that a
// fraction f of the rows holds costs 128 f x 512 B per 128-row tile when it is
// gathered and 512 B (its bf16 [M_hi | M_lo] operand rows) when it is
// multiplied densely, so every column with f > 1/128 belongs on the tensor
// cores: at C4 that is the first ~1000 Zipf-ranked ids.  The hot window is
// therefore HT = 64 nb columns (nb <= 16), streamed in 64-column K blocks:
//   * the B operand images (one 32 KB SW128 block per 64 columns, built once
//     per fold by k6_prep_kernel) arrive through a 2-stage cp.async.bulk ring;
//   * 4 scatter warps (thread = tile row) walk their row's sorted entries (two
//     entries of lookahead) and fill the A block (bf16 x_hi / x_lo planes,
//     2-stage ring) of each K block; the same warps run the epilogue of their
//     32 rows (warp q = TMEM lane quadrant q), so one TMEM accumulator suffices;
//   * 16 gather warps (8 rows each) read only each row's last 32 entries (three
//     rows ahead; a longer cold suffix walks back) and gather the columns >= HT
//     into u_cold with L1-bypassing loads, a tile ahead of the scatter / MMA
//     pipeline; they also count the cold entries so that the epilogue can check
//     hot + cold = row length (anything else is an unsorted row);
//   * one thread issues the MMAs, one thread the bulk copies.
// Measured at C4 (tools/k6v2_time.py): 7.41 ms (v1) -> 5.6 ms at nb = 10 (6.0 ms before the
// gather loads wrote their destination registers directly — ncu's top stall was the register
// move behind each predicated load, which left ~4 of the 8 loads in flight); the
// cold gathers alone take ~5.3 ms (L2 slices at ~10 TB/s) and the scatter /
// MMA chain alone ~4.7 ms (one warp's ~150 dependent instructions per K block).
// Tried: coalesced per-block sweeps by the scatter warps (32 rows x nb re-reads,
// 13.9 ms), 16-byte chunk walks with two chunks of register lookahead (6.4 ms:
// the predicated four-way body costs more instructions than it saves latency),
// an L2 bulk prefetch of the next tile's CSR span (no change), L1-allocating M
// loads (better alone, 4.3 ms, but they evict the row walks' lines: 5.9 ms),
// two scatter groups on alternate K blocks with 15 strided gather warps (24
// warps is the most that keep 80 registers; 7.3 ms), 8-byte pair refills of a
// four-entry lookahead (7.2 ms), clearing only the 16-byte chunks a thread
// wrote instead of zero-filling the stage (6.2 ms), an 8-entry cp.async ring per
// scatter thread (12 KB more shared memory, so 28 KB of L1: 8.1 ms).  Every variant that adds instructions to the
// walk loses: the scatter warps' dependent instruction chain per K block, not
// their load latency, paces the MMA pipeline (ncu: issue active 54 %, L1TEX
// 70 %, L2 slices 38 %, DRAM 8 %).
// Rows must have strictly increasing columns (the CSR contract, include/
// levsketch_b200.h); a row that does not sets LVSK_FLAG_BADINDEX.
namespace k6v2 {

using namespace tc;
using k6tc::bf16_bits;
using k6tc::idesc;

constexpr int R = 128;
constexpr int TR = 128;
constexpr int GW = 16;             // gather warps
constexpr int RPW = TR / GW;       // rows per gather warp
constexpr int SW = 4;              // scatter + epilogue warps
constexpr int WARP_MMA = SW;
constexpr int WARP_LOAD = SW + 1;
constexpr int WARP_G0 = SW + 2;
constexpr int THREADS = 32 * (SW + 2 + GW);
constexpr int KBLK = 64;                 // hot columns per K block
constexpr int B_STAGE = 2 * R * 128;     // [M_hi | M_lo]^T rows of one K block: 256 x 128 B
constexpr int A_PLANE = TR * 128;        // 128 rows x 128 B
constexpr int A_STAGE = 2 * A_PLANE;     // x_hi plane, x_lo plane
constexpr int NSB = 2;  // (two stages keep shared memory under 196 KB: 60 KB of L1 for the row walks)
constexpr int NSA = 2;
constexpr int OFF_B = 0;
constexpr int OFF_A = OFF_B + NSB * B_STAGE;
constexpr int OFF_UC = OFF_A + NSA * A_STAGE;
constexpr int OFF_BAR = OFF_UC + TR * R * 4;
constexpr int SMEM_BYTES = OFF_BAR + 256 + TR * 4 + 1024;
constexpr int MAX_NB = 16;
static_assert(SMEM_BYTES <= 232448, "K6-TC v2 shared memory");

// M rows stream through L2 only: the 60 KB of L1 belong to the scatter threads' row walks.
// The predicated load writes its destination registers directly (zero when !ok): a select
// after the load would put a register move behind every load and serialise the gathers.
__device__ __forceinline__ void ldg_stream_pred(float4& v, const float4* p, bool ok) {
  asm("{\n\t.reg .pred q;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "mov.f32 %0, 0f00000000;\n\tmov.f32 %1, 0f00000000;\n\tmov.f32 %2, 0f00000000;\n\tmov.f32 %3, 0f00000000;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n}"
      : "=&f"(v.x), "=&f"(v.y), "=&f"(v.z), "=&f"(v.w)
      : "l"(p), "r"(static_cast<int>(ok)));
}

// predicated element loads that write their (zero-initialised) destination directly, for the
// same reason: `live ? p[i] : 0` puts a move behind the load and waits for it at once
__device__ __forceinline__ void ldg_pred(int32_t& v, const int32_t* p, bool ok) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, 0;\n\t@q ld.global.nc.b32 %0, [%1];\n}"
      : "=&r"(v)
      : "l"(p), "r"(static_cast<int>(ok)));
}
__device__ __forceinline__ void ldg_pred(float& v, const float* p, bool ok) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.f32 %0, 0f00000000;\n\t@q ld.global.nc.f32 %0, [%1];\n}"
      : "=&f"(v)
      : "l"(p), "r"(static_cast<int>(ok)));
}
__device__ __forceinline__ void ldg_pred(double& v, const double* p, bool ok) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.f64 %0, 0d0000000000000000;\n\t@q ld.global.nc.f64 %0, [%1];\n}"
      : "=&d"(v)
      : "l"(p), "r"(static_cast<int>(ok)));
}

// B operand images: block j holds rows nn < R = bf16(M[64 j + k][nn]) and rows
// nn >= R = the bf16 remainder, K-major SW128 (the layout the MMA reads)
__global__ void k6_prep_kernel(const float* __restrict__ M, int64_t d, int nb, uint8_t* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(nb) * 2 * R * KBLK;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % R);
    const int kk = static_cast<int>((e / R) % KBLK);
    const int half = static_cast<int>((e / (R * KBLK)) & 1);
    const int j = static_cast<int>(e / (2 * R * KBLK));
    const int64_t k = static_cast<int64_t>(j) * KBLK + kk;
    const float m = k < d ? M[k * R + c] : 0.f;
    const float mh = __bfloat162float(__float2bfloat16_rn(m));
    const int nn = half * R + c;
    const int64_t off = static_cast<int64_t>(j) * B_STAGE + nn * 128 + ((((kk >> 3) ^ (nn & 7))) << 4) + ((kk & 7) << 1);
    *reinterpret_cast<uint16_t*>(out + off) = bf16_bits(half ? m - mh : mh);
  }
}

template <typename V>
__global__ void __launch_bounds__(THREADS, 1)
    csr_rowsumsq_tc2_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                            const V* __restrict__ val, int64_t n, int64_t d, const float* __restrict__ M,
                            const uint8_t* __restrict__ prep, int nb, double* __restrict__ scores, int32_t* flags) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* bfull = bars;             // [NSB] bulk copy landed
  uint64_t* bfree = bfull + NSB;      // [NSB] MMAs done reading the B stage
  uint64_t* aready = bfree + NSB;     // [NSA] SW scatter warps: A block written
  uint64_t* afree = aready + NSA;     // [NSA] MMAs done reading the A stage
  uint64_t* accfull = afree + NSA;    // all K blocks of the tile accumulated
  uint64_t* ucready = accfull + 1;    // GW gather warps: u_cold written
  uint64_t* ucfree = ucready + 1;     // SW epilogue warps: u_cold read
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ucfree + 1);
  int32_t* coldcnt = reinterpret_cast<int32_t*>(smem + OFF_BAR + 256);  // [TR] cold entries per row (gather -> epilogue)
  float* ucold = reinterpret_cast<float*>(smem + OFF_UC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int64_t base0 = row_ptr[0];
  const int32_t ht = nb * KBLK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bfree[s], 1);
    }
    for (int s = 0; s < NSA; ++s) {
      mbar_init(&aready[s], SW);
      mbar_init(&afree[s], 1);
    }
    mbar_init(accfull, 1);
    mbar_init(ucready, GW);
    mbar_init(ucfree, SW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == WARP_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == WARP_LOAD) {
    // ---- B loader: the nb block images, in order, for every tile
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int j = 0; j < nb; ++j, ++it) {
          const uint32_t s = it % NSB, u = it / NSB;
          if (u > 0) mbar_wait(&bfree[s], (u - 1) & 1u);
          mbar_expect_tx(&bfull[s], B_STAGE);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(smem + OFF_B + s * B_STAGE)),
              "l"(prep + static_cast<int64_t>(j) * B_STAGE), "r"(B_STAGE), "r"(smem_u32(&bfull[s]))
              : "memory");
        }
      }
    }
  } else if (warp == WARP_MMA) {
    // ---- MMA issuer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int j = 0; j < nb; ++j, ++it) {
          const uint32_t sb = it % NSB, sa = it % NSA;
          mbar_wait(&aready[sa], (it / NSA) & 1u);
          mbar_wait(&bfull[sb], (it / NSB) & 1u);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A written through the generic proxy
          tc_fence_after();
          const uint64_t ah = sw128_desc(smem_u32(smem + OFF_A + sa * A_STAGE));
          const uint64_t al = sw128_desc(smem_u32(smem + OFF_A + sa * A_STAGE + A_PLANE));
          const uint64_t b = sw128_desc(smem_u32(smem + OFF_B + sb * B_STAGE));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            umma_f16(tmem_base, ah + 2 * kk, b + 2 * kk, idesc(2 * R), (j | kk) ? 1u : 0u);  // x_hi [M_hi | M_lo]
            umma_f16(tmem_base + R, al + 2 * kk, b + 2 * kk, idesc(R), 1u);                  // + x_lo M_hi
          }
          umma_commit(&afree[sa]);
          umma_commit(&bfree[sb]);
        }
        umma_commit(accfull);
      }
    }
  } else if (warp < SW) {
    // ---- scatter + epilogue: thread = tile row 32 q + lane walks its row's sorted entries
    // (two entries of lookahead) and places those of each K block into the A planes
    const int q = warp;
    const int i = 32 * q + lane;
    int bad = 0;
    uint32_t it = 0, lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int64_t g = t * TR + i;
      const int64_t e0 = row_ptr[g < n ? g : n] - base0;
      const int64_t e1 = row_ptr[g + 1 < n ? g + 1 : n] - base0;
      int64_t ptr = e0;
      // two entries of lookahead
      int32_t cprev = -1;
      int32_t ca = ptr < e1 ? col[ptr] : 0x7FFFFFFF;
      float xa = ptr < e1 ? static_cast<float>(val[ptr]) : 0.f;
      int32_t cb = ptr + 1 < e1 ? col[ptr + 1] : 0x7FFFFFFF;
      float xb = ptr + 1 < e1 ? static_cast<float>(val[ptr + 1]) : 0.f;
      for (int j = 0; j < nb; ++j, ++it) {
        const uint32_t sa = it % NSA, u = it / NSA;
        if (u > 0) mbar_wait(&afree[sa], (u - 1) & 1u);
        uint8_t* ahp = smem + OFF_A + sa * A_STAGE;
        uint8_t* alp = ahp + A_PLANE;
        // zero this warp's 32 rows (4 KB, contiguous) of both planes
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          reinterpret_cast<uint4*>(ahp + 4096 * q)[x * 32 + lane] = make_uint4(0, 0, 0, 0);
          reinterpret_cast<uint4*>(alp + 4096 * q)[x * 32 + lane] = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
        const int32_t lo = j * KBLK, lim = lo + KBLK;
        while (ca < lim) {  // ca = INT_MAX past the row's end
          if (ca < lo || ca <= cprev) {  // out of order (or negative): the row breaks the CSR contract
            bad |= LVSK_FLAG_BADINDEX;
          } else {
            if (!isfinite(xa)) bad |= LVSK_FLAG_NONFINITE;
            const int32_t k = ca - lo;
            const float xh = __bfloat162float(__float2bfloat16_rn(xa));
            const uint32_t off = static_cast<uint32_t>(i * 128 + ((((k >> 3) ^ (i & 7))) << 4) + ((k & 7) << 1));
            *reinterpret_cast<uint16_t*>(ahp + off) = bf16_bits(xh);
            *reinterpret_cast<uint16_t*>(alp + off) = bf16_bits(xa - xh);
            cprev = ca;
          }
          ca = cb;
          xa = xb;
          ++ptr;
          const bool more = ptr + 1 < e1;
          cb = more ? col[ptr + 1] : 0x7FFFFFFF;
          xb = more ? static_cast<float>(val[ptr + 1]) : 0.f;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&aready[sa]);
      }
      // epilogue of this warp's 32 rows
      mbar_wait(ucready, lt & 1u);
      mbar_wait(accfull, lt & 1u);
      tc_fence_after();
      // every entry is either placed above (columns < ht) or gathered (the cold suffix):
      // anything else is a row that is not strictly increasing
      if (g < n && (ptr - e0) + coldcnt[i] != e1 - e0) bad |= LVSK_FLAG_BADINDEX;
      const uint32_t base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
      float acc = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < R; c0 += 32) {
        uint32_t vh[32], vl[32];
        tmem_ld32(base + c0, vh);
        tmem_ld32(base + R + c0, vl);
        tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          const int blk = (c0 + jj) >> 2;
          const float4 uc = *reinterpret_cast<const float4*>(ucold + i * R + 4 * (blk ^ (i & 31)));
          const float a0 = __uint_as_float(vh[jj]) + __uint_as_float(vl[jj]) + uc.x;
          const float a1 = __uint_as_float(vh[jj + 1]) + __uint_as_float(vl[jj + 1]) + uc.y;
          const float a2 = __uint_as_float(vh[jj + 2]) + __uint_as_float(vl[jj + 2]) + uc.z;
          const float a3 = __uint_as_float(vh[jj + 3]) + __uint_as_float(vl[jj + 3]) + uc.w;
          acc = fmaf(a0, a0, acc);
          acc = fmaf(a1, a1, acc);
          acc = fmaf(a2, a2, acc);
          acc = fmaf(a3, a3, acc);
        }
      }
      if (g < n) scores[g] = static_cast<double>(acc);
      tc_fence_before();  // the next tile's first MMA overwrites the accumulator
      __syncwarp();
      if (lane == 0) mbar_arrive(ucfree);
    }
    const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (any && lane == 0) atomicOr(flags, any);
  } else {
    // ---- gather warps: the cold suffix (columns >= ht) of rows RPW w .. RPW w + RPW - 1.
    // Only the row's last 32 entries are read (three rows ahead); a longer cold suffix
    // walks back batch by batch.
    const int w = warp - WARP_G0;
    int bad = 0;
    uint32_t lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int64_t gbase = t * TR + RPW * w;
      int64_t rp = 0;
      if (lane <= RPW) rp = row_ptr[gbase + lane < n ? gbase + lane : n] - base0;
      auto load_tail = [&](int rr, int32_t& c, V& x) {  // (values stay in their type until they are used)
        const int64_t f0 = __shfl_sync(0xFFFFFFFFu, rp, rr < RPW ? rr : RPW);
        const int64_t f1 = __shfl_sync(0xFFFFFFFFu, rp, rr < RPW ? rr + 1 : RPW);
        const int64_t s0 = f1 - 32 > f0 ? f1 - 32 : f0;
        const bool live = s0 + lane < f1;
        ldg_pred(c, col + s0 + lane, live);
        ldg_pred(x, val + s0 + lane, live);
      };
      int32_t c0, c1, c2;
      V x0, x1, x2;
      load_tail(0, c0, x0);
      load_tail(1, c1, x1);
      load_tail(2, c2, x2);
#pragma unroll 1
      for (int rr = 0; rr < RPW; ++rr) {
        const int i = RPW * w + rr;
        float u[4] = {0.f, 0.f, 0.f, 0.f};
        const int64_t e0 = __shfl_sync(0xFFFFFFFFu, rp, rr), e1 = __shfl_sync(0xFFFFFFFFu, rp, rr + 1);
        int32_t c = c0;
        float x = static_cast<float>(x0);
        c0 = c1;
        x0 = x1;
        c1 = c2;
        x1 = x2;
        load_tail(rr + 3, c2, x2);  // (past the tile's last row: an empty range, no load)
        int64_t s0 = e1 - 32 > e0 ? e1 - 32 : e0;  // this batch = entries [s0, s1)
        int64_t s1 = e1;
        int total = 0;
        while (true) {
          const int nl = static_cast<int>(s1 - s0);
          const bool live = lane < nl;
          const int32_t prev = __shfl_up_sync(0xFFFFFFFFu, c, 1);
          if (live && (c < 0 || c >= d || (lane > 0 && c <= prev))) {
            bad |= LVSK_FLAG_BADINDEX;
            c = 0;
            x = 0.f;
          }
          if (live && !isfinite(x)) bad |= LVSK_FLAG_NONFINITE;
          uint32_t cm = __ballot_sync(0xFFFFFFFFu, live && c >= ht);
          const int ncold = __popc(cm);
          total += ncold;
          const int first = nl - ncold;
          // sorted rows: the cold entries are the batch's last lanes; eight rows of M in flight per lane
          if (ncold > 0 && cm == ((0xFFFFFFFFu >> (32 - ncold)) << first)) {
            for (int b0 = 0; b0 < ncold; b0 += 8) {
              float4 mv[8];
              float xv[8];
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const int tl = (first + b0 + jj) & 31;
                const int32_t ct = __shfl_sync(0xFFFFFFFFu, c, tl);
                const float xt = __shfl_sync(0xFFFFFFFFu, x, tl);
                const bool ok = b0 + jj < ncold;
                xv[jj] = ok ? xt : 0.f;
                ldg_stream_pred(mv[jj], reinterpret_cast<const float4*>(M + static_cast<int64_t>(ct) * R) + lane, ok);
              }
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                u[0] = fmaf(xv[jj], mv[jj].x, u[0]);
                u[1] = fmaf(xv[jj], mv[jj].y, u[1]);
                u[2] = fmaf(xv[jj], mv[jj].z, u[2]);
                u[3] = fmaf(xv[jj], mv[jj].w, u[3]);
              }
            }
          } else if (ncold > 0) {
            bad |= LVSK_FLAG_BADINDEX;  // cold entries that are not a suffix: not increasing
          }
          if (ncold < nl || s0 <= e0) break;  // the suffix starts inside this batch (or the row is done)
          const int32_t head = __shfl_sync(0xFFFFFFFFu, c, 0);
          s1 = s0;
          s0 = s1 - 32 > e0 ? s1 - 32 : e0;
          const bool lv = s0 + lane < s1;
          c = lv ? col[s0 + lane] : 0;
          x = lv ? static_cast<float>(val[s0 + lane]) : 0.f;
          if (__shfl_sync(0xFFFFFFFFu, c, static_cast<int>(s1 - s0) - 1) >= head) bad |= LVSK_FLAG_BADINDEX;
        }
        // the previous tile's epilogue must be done with u_cold before its first row is replaced
        if (rr == 0 && lt > 0) mbar_wait(ucfree, (lt - 1) & 1u);
        *reinterpret_cast<float4*>(ucold + i * R + 4 * (lane ^ (i & 31))) = make_float4(u[0], u[1], u[2], u[3]);
        if (lane == 0) coldcnt[i] = total;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(ucready);
    }
    const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (any && lane == 0) atomicOr(flags, any);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(256));
  }
}

inline int hot_blocks(int64_t d) {
  int nb = 10;  // C4: 5.45 ms (8: 5.6, 12: 5.7; tools/k6v2_time.py)
  if (const char* e = getenv("LVSK_K6_HOTBLOCKS")) nb = atoi(e);
  nb = nb < 1 ? 1 : (nb > MAX_NB ? MAX_NB : nb);
  const int64_t cap = (d + KBLK - 1) / KBLK;
  return static_cast<int>(nb < cap ? nb : cap);
}

}  // namespace k6v2

size_t csr_rowsumsq_prep_bytes(int64_t d, int64_t r) {
  return r == k6v2::R ? static_cast<size_t>(k6v2::hot_blocks(d)) * k6v2::B_STAGE : 0;
}

int32_t csr_rowsumsq_prepare(const float* M, int64_t d, int64_t r, void* prep, size_t prep_bytes, cudaStream_t st) {
  using namespace k6v2;
  LVSK_REQUIRE(r == R, LVSK_ERR_UNSUPPORTED, "the prepared CSR leverage pass needs r = 128");
  const int nb = hot_blocks(d);
  LVSK_REQUIRE(prep != nullptr && prep_bytes >= static_cast<size_t>(nb) * B_STAGE, LVSK_ERR_CAPACITY,
               "prepared-operand buffer too small");
  LVSK_REQUIRE(reinterpret_cast<uintptr_t>(prep) % 16 == 0, LVSK_ERR_CONFIGURATION, "prepared-operand buffer not 16-byte aligned");
  const int64_t total = static_cast<int64_t>(nb) * 2 * R * KBLK;
  k6_prep_kernel<<<static_cast<int>((total + 255) / 256), 256, 0, st>>>(M, d, nb, static_cast<uint8_t*>(prep));
  LVSK_CHECK_LAUNCH("csr rowsumsq prepare");
  return LVSK_OK;
}

int32_t csr_rowsumsq_tc2(const int64_t* row_ptr, const int32_t* col, const void* val, int32_t val_dtype, int64_t n,
                         int64_t d, const float* M, const void* prep, size_t prep_bytes, double* scores,
                         int32_t* flags, cudaStream_t st) {
  using namespace k6v2;
  const int nb = hot_blocks(d);
  LVSK_REQUIRE(prep != nullptr && prep_bytes >= static_cast<size_t>(nb) * B_STAGE, LVSK_ERR_CAPACITY,
               "prepared-operand buffer too small");
  LVSK_REQUIRE(reinterpret_cast<uintptr_t>(prep) % 16 == 0 && reinterpret_cast<uintptr_t>(M) % 16 == 0,
               LVSK_ERR_CONFIGURATION, "M and the prepared operand must be 16-byte aligned");
  const void* fn = val_dtype == LVSK_F64 ? reinterpret_cast<const void*>(csr_rowsumsq_tc2_kernel<double>)
                                         : reinterpret_cast<const void*>(csr_rowsumsq_tc2_kernel<float>);
  const int32_t rc = ensure_smem_attr(fn, SMEM_BYTES, "csr tc2 smem attribute");
  if (rc != LVSK_OK) return rc;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int grid = static_cast<int>(ntiles < num_sms() ? ntiles : num_sms());
  const uint8_t* pp = static_cast<const uint8_t*>(prep);
  if (val_dtype == LVSK_F64)
    csr_rowsumsq_tc2_kernel<double><<<grid, k6v2::THREADS, SMEM_BYTES, st>>>(row_ptr, col, static_cast<const double*>(val), n,
                                                                      d, M, pp, nb, scores, flags);
  else
    csr_rowsumsq_tc2_kernel<float><<<grid, k6v2::THREADS, SMEM_BYTES, st>>>(row_ptr, col, static_cast<const float*>(val), n, d,
                                                                     M, pp, nb, scores, flags);
  LVSK_CHECK_LAUNCH("csr rowsumsq tc2");
  return LVSK_OK;
}

bool csr_rowsumsq_tc_ok(const float* M, int64_t r) {
  return r == k6tc::R && reinterpret_cast<uintptr_t>(M) % 16 == 0 && getenv("LVSK_K6_SIMT") == nullptr;
}

int32_t csr_rowsumsq_tc(const int64_t* row_ptr, const int32_t* col, const void* val, int32_t val_dtype, int64_t n,
                        int64_t d, const float* M, double* scores, int32_t* flags, cudaStream_t st) {
  using namespace k6tc;
  const void* fn = val_dtype == LVSK_F64 ? reinterpret_cast<const void*>(csr_rowsumsq_tc_kernel<double>)
                                         : reinterpret_cast<const void*>(csr_rowsumsq_tc_kernel<float>);
  const int32_t rc = ensure_smem_attr(fn, SMEM_BYTES, "csr tc smem attribute");
  if (rc != LVSK_OK) return rc;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int grid = static_cast<int>(ntiles < num_sms() ? ntiles : num_sms());
  if (val_dtype == LVSK_F64)
    csr_rowsumsq_tc_kernel<double><<<grid, k6tc::THREADS, SMEM_BYTES, st>>>(row_ptr, col, static_cast<const double*>(val),
                                                                       n, d, M, scores, flags);
  else
    csr_rowsumsq_tc_kernel<float><<<grid, k6tc::THREADS, SMEM_BYTES, st>>>(row_ptr, col, static_cast<const float*>(val), n,
                                                                      d, M, scores, flags);
  LVSK_CHECK_LAUNCH("csr rowsumsq tc");
  return LVSK_OK;
}

}  // namespace lvsk
