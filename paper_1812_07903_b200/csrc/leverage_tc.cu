// K5 on the 5th-gen tensor cores: scores[i] = || X[i,:] M ||^2, fp32 X,
// 3xTF32 split for fp32-level accuracy, accumulators in TMEM.
//
// Reference: _block_scores (pkg/src/levsketch/leverage.py:88-95).
//
// Per CTA (persistent, one per SM): row tiles of 256 rows = two M=128 UMMA
// sub-tiles; K streamed in 32-float (128 B) chunks through a 4-stage
// TMA -> smem ring (SWIZZLE_128B, K-major).  Per stage:
//   warp 0   TMA: X[256 x 32] + Mt_hi[N x 32] + Mt_lo[N x 32]     (full)
//   warp 1   MMA: acc += x.Mhi + x.Mlo         (tcgen05 kind::tf32) (xdone)
//   warps 2-5     x -> x_lo = x - tf32(x) in place (+ finiteness)    (loready)
//   warp 1   MMA: acc += x_lo.Mhi                                    (empty)
// and at the end of a row tile warps 2-5 drain the TMEM accumulator
// (tcgen05.ld 32x32b), square and row-reduce in registers and write float64
// scores.  Accumulators are double-buffered in TMEM so the epilogue of tile
// t overlaps the MMAs of tile t+1.  X is read from HBM exactly once.
#include <cstdlib>

#include "tc_common.cuh"

namespace lvsk {
namespace tc {


template <int N>
struct Cfg {
  static constexpr int STAGES = N <= 64 ? 4 : 3;
  static constexpr int X_BYTES = TILE_ROWS * BK * 4;  // 32 KB
  static constexpr int M_BYTES = N * BK * 4;
  static constexpr int STAGE_BYTES = X_BYTES + 2 * M_BYTES;
  static constexpr int ACC_COLS = SUB * N;
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  // instruction descriptor: F32 accum, A/B TF32, K-major both, N>>3, M>>4
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(BM >> 4) << 24);
};

template <int N>
__global__ void __launch_bounds__(THREADS, 1)
    leverage_tf32x3_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapHi,
                           const __grid_constant__ CUtensorMap mapLo, int64_t n, int kchunks,
                           double* __restrict__ scores, int32_t* flags) {
  using C = Cfg<N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays a shared-space pointer
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* xdone = bars + C::STAGES;
  uint64_t* loready = bars + 2 * C::STAGES;
  uint64_t* empty = bars + 3 * C::STAGES;
  uint64_t* accfull = bars + 4 * C::STAGES;
  uint64_t* accempty = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TILE_ROWS - 1) / TILE_ROWS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&xdone[s], 1);
      mbar_init(&loready[s], EPI_THREADS);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], EPI_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapHi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapLo) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_x = l2_policy_evict_first(), pol_m = l2_policy_evict_last();
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          tma_load_2d(&mapX, &full[s], st, kc * BK, static_cast<int>(t * TILE_ROWS), pol_x);
          tma_load_2d(&mapHi, &full[s], st + C::X_BYTES, kc * BK, 0, pol_m);
          tma_load_2d(&mapLo, &full[s], st + C::X_BYTES + C::M_BYTES, kc * BK, 0, pol_m);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      int64_t pend = -1;  // stage iteration whose x_lo MMAs are outstanding
      uint32_t pend_acc = 0;
      bool pend_last = false;
      auto issue_lo = [&](uint32_t pit, uint32_t acc_col, bool last) {
        const uint32_t ps = pit % C::STAGES, pph = (pit / C::STAGES) & 1u;
        mbar_wait(&loready[ps], pph);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + ps * C::STAGE_BYTES);
        const uint64_t bhi = sw128_desc(st + C::X_BYTES);
#pragma unroll
        for (int sub = 0; sub < SUB; ++sub) {
          const uint64_t a = sw128_desc(st + sub * (BM * 128));
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk)
            umma_tf32(tmem_base + acc_col + sub * N, a + 2 * kk, bhi + 2 * kk, C::IDESC, 1u);
        }
        umma_commit(&empty[ps]);
        if (last) umma_commit(&accfull[(acc_col / C::ACC_COLS) & 1u]);
      };
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
        const uint32_t acc_col = ab * C::ACC_COLS;
        mbar_wait(&accempty[ab], aph ^ 1u);
        tc_fence_after();
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1u;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * C::STAGE_BYTES);
          const uint64_t bhi = sw128_desc(st + C::X_BYTES);
          const uint64_t blo = sw128_desc(st + C::X_BYTES + C::M_BYTES);
#pragma unroll
          for (int sub = 0; sub < SUB; ++sub) {
            const uint64_t a = sw128_desc(st + sub * (BM * 128));
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t d = tmem_base + acc_col + sub * N;
              umma_tf32(d, a + 2 * kk, bhi + 2 * kk, C::IDESC, (kc | kk) ? 1u : 0u);
              umma_tf32(d, a + 2 * kk, blo + 2 * kk, C::IDESC, 1u);
            }
          }
          umma_commit(&xdone[s]);
          if (pend >= 0) issue_lo(static_cast<uint32_t>(pend), pend_acc, pend_last);
          pend = it;
          pend_acc = acc_col;
          pend_last = kc == kchunks - 1;
        }
      }
      if (pend >= 0) issue_lo(static_cast<uint32_t>(pend), pend_acc, pend_last);
    }
  } else {
    // ---------------- transform + epilogue (warps 2..5) ----------------
    const int et = threadIdx.x - 64;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    bool bad = false;
    uint32_t it = 0, lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1u;
        mbar_wait(&full[s], ph);
        mbar_wait(&xdone[s], ph);
        float4* xs = reinterpret_cast<float4*>(smem + s * C::STAGE_BYTES);
#pragma unroll 4
        for (int i = et; i < C::X_BYTES / 16; i += EPI_THREADS) {
          float4 v = xs[i];
          bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
          v.x -= __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          v.y -= __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          v.z -= __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          v.w -= __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          xs[i] = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&loready[s]);
      }
      // epilogue for tile t
      const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
      mbar_wait(&accfull[ab], aph);
      tc_fence_after();
#pragma unroll
      for (int sub = 0; sub < SUB; ++sub) {
        float acc = 0.f;
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ab * C::ACC_COLS + sub * N + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float u = __uint_as_float(v[j]);
            acc = fmaf(u, u, acc);
          }
        }
        const int64_t row = t * TILE_ROWS + sub * BM + quarter * 32 + lane;
        if (row < n) scores[row] = static_cast<double>(acc);
      }
      tc_fence_before();
      mbar_arrive(&accempty[ab]);
    }
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// v2 (r <= 64): main term x.[M_hi | M_lo] as ONE N=128 TF32 MMA (A read once
// for both halves), correction x_lo.M_hi as a BF16 MMA (x_lo written by the
// transform warps as bf16 into its own SW64 tile, M_hi in bf16 by TMA).  The
// x_lo / M_hi roundings to bf16 perturb a 2^-11-relative term by 2^-8, i.e.
// ~2^-19 of the result.  Per 256 x 32 stage the tensor core reads 88 KB of
// smem operands instead of 144 KB in v1.

// v2 runs 8 worker warps (two per TMEM lane quarter): all 8 make the x_lo
// tile of every stage (the transform is the kernel's longest per-stage chain),
// warps 2-5 read back sub-tile 0 and warps 6-9 sub-tile 1
constexpr int V2_EPI = 256;               // x_lo transform threads (all worker warps; 12 warps measured slower)
constexpr int V2_READ = 256;              // TMEM read-back threads (the first 8 worker warps)
constexpr int V2_THREADS = 64 + V2_EPI;

struct Cfg2 {
  static constexpr int N = 64;
  static constexpr int SX = 4;                             // X ring (the HBM stream)
  static constexpr int SB = 2;                             // M-chunk ring (L2 hits)
  static constexpr int SL = 2;                             // x_lo ring (produced on chip)
  static constexpr int X_BYTES = TILE_ROWS * BK * 4;       // 32 KB fp32, SW128
  static constexpr int B_BYTES = 2 * N * BK * 4;           // 16 KB: Mt_hi rows 0..63, Mt_lo rows 64..127
  static constexpr int BB_BYTES = N * BK * 2;              // 4 KB: Mt_hi bf16, SW64
  static constexpr int BSTAGE = B_BYTES + BB_BYTES;        // 20 KB
  static constexpr int XL_BYTES = TILE_ROWS * BK * 2;      // 16 KB: x_lo bf16, SW64
  static constexpr int OFF_B = SX * X_BYTES;
  static constexpr int OFF_XL = OFF_B + SB * BSTAGE;
  static constexpr int OFF_BAR = OFF_XL + SL * XL_BYTES;   // 200 KB
  static constexpr int ACC_COLS = SUB * 2 * N;             // 256 per accumulator buffer
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM_BYTES = OFF_BAR + 1024 + 512;
  static constexpr uint32_t IDESC_TF32 =
      (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t((2 * N) >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  static constexpr uint32_t IDESC_BF16 =
      (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(BM >> 4) << 24);
};

__global__ void __launch_bounds__(V2_THREADS, 1)
    leverage_v2_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapHi,
                       const __grid_constant__ CUtensorMap mapLo, const __grid_constant__ CUtensorMap mapHb,
                       int64_t n, int kchunks, double* __restrict__ scores, int32_t* flags) {
  using C = Cfg2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays a shared-space pointer
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* xfull = bars;                 // [SX] TMA complete_tx
  uint64_t* xempty = xfull + C::SX;       // [SX] main-MMA commit (1) + transform threads (128)
  uint64_t* bfull = xempty + C::SX;       // [SB]
  uint64_t* bempty = bfull + C::SB;       // [SB] lo-MMA commit
  uint64_t* xlfull = bempty + C::SB;      // [SL] transform threads
  uint64_t* xlempty = xlfull + C::SL;     // [SL] lo-MMA commit
  uint64_t* accfull = xlempty + C::SL;    // [2]
  uint64_t* accempty = accfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TILE_ROWS - 1) / TILE_ROWS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::SX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1 + V2_EPI);
    }
    for (int s = 0; s < C::SB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int s = 0; s < C::SL; ++s) {
      mbar_init(&xlfull[s], V2_EPI);
      mbar_init(&xlempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], V2_READ);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapHi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapLo) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapHb) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // lane 0 streams X (4 stages ahead), lane 1 streams the M chunks (2 ahead)
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::SX, ph = (it / C::SX) & 1u;
          mbar_wait(&xempty[s], ph ^ 1u);
          mbar_expect_tx(&xfull[s], C::X_BYTES);
          tma_load_2d(&mapX, &xfull[s], smem + s * C::X_BYTES, kc * BK, static_cast<int>(t * TILE_ROWS), pol);
        }
      }
    } else if (lane == 1) {
      const uint64_t pol = l2_policy_evict_last();
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::SB, ph = (it / C::SB) & 1u;
          mbar_wait(&bempty[s], ph ^ 1u);
          uint8_t* bs = smem + C::OFF_B + s * C::BSTAGE;
          mbar_expect_tx(&bfull[s], C::BSTAGE);
          tma_load_2d(&mapHi, &bfull[s], bs, kc * BK, 0, pol);
          tma_load_2d(&mapLo, &bfull[s], bs + C::B_BYTES / 2, kc * BK, 0, pol);
          tma_load_2d(&mapHb, &bfull[s], bs + C::B_BYTES, kc * BK, 0, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
        const uint32_t acc_col = ab * C::ACC_COLS;
        mbar_wait(&accempty[ab], aph ^ 1u);
        tc_fence_after();
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t sx = it % C::SX, phx = (it / C::SX) & 1u;
          const uint32_t sb = it % C::SB, phb = (it / C::SB) & 1u;
          const uint32_t sl = it % C::SL, phl = (it / C::SL) & 1u;
          mbar_wait(&xfull[sx], phx);
          mbar_wait(&bfull[sb], phb);
          tc_fence_after();
          const uint32_t xs = smem_u32(smem + sx * C::X_BYTES);
          const uint32_t bs = smem_u32(smem + C::OFF_B + sb * C::BSTAGE);
          const uint64_t bm = sw128_desc(bs);
#pragma unroll
          for (int sub = 0; sub < SUB; ++sub) {
            const uint64_t a = sw128_desc(xs + sub * (BM * 128));
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
              umma_tf32(tmem_base + acc_col + sub * 2 * C::N, a + 2 * kk, bm + 2 * kk, C::IDESC_TF32,
                        (kc | kk) ? 1u : 0u);
          }
          umma_commit(&xempty[sx]);
          mbar_wait(&xlfull[sl], phl);
          tc_fence_after();
          const uint64_t bb = sw64_desc(bs + C::B_BYTES);
          const uint32_t xls = smem_u32(smem + C::OFF_XL + sl * C::XL_BYTES);
#pragma unroll
          for (int sub = 0; sub < SUB; ++sub) {
            const uint64_t a = sw64_desc(xls + sub * (BM * 64));
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_f16(tmem_base + acc_col + sub * 2 * C::N, a + 2 * kk, bb + 2 * kk, C::IDESC_BF16, 1u);
          }
          umma_commit(&xlempty[sl]);
          umma_commit(&bempty[sb]);
          if (kc == kchunks - 1) umma_commit(&accfull[ab]);
        }
      }
    }
  } else {
    const int et = threadIdx.x - 64;
    const int quarter = warp & 3;
    const int my_sub = (warp - 2) >> 2;  // epilogue sub-tile of this warp
    bool bad = false;
    uint32_t it = 0, lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const uint32_t sx = it % C::SX, phx = (it / C::SX) & 1u;
        const uint32_t sl = it % C::SL, phl = (it / C::SL) & 1u;
        mbar_wait(&xfull[sx], phx);
        mbar_wait(&xlempty[sl], phl ^ 1u);
        const uint8_t* xsm = smem + sx * C::X_BYTES;
        uint8_t* xl = smem + C::OFF_XL + sl * C::XL_BYTES;
#pragma unroll 4
        for (int i = et; i < TILE_ROWS * 8; i += V2_EPI) {
          const int row = i >> 3, c = i & 7;
          const float4 v = *reinterpret_cast<const float4*>(xsm + row * 128 + ((c ^ (row & 7)) << 4));
          bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
          const float l0 = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          const float l1 = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          const float l2 = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          const float l3 = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          __nv_bfloat162 p0 = __floats2bfloat162_rn(l0, l1);
          __nv_bfloat162 p1 = __floats2bfloat162_rn(l2, l3);
          uint2 packed;
          packed.x = *reinterpret_cast<uint32_t*>(&p0);
          packed.y = *reinterpret_cast<uint32_t*>(&p1);
          *reinterpret_cast<uint2*>(xl + row * 64 + ((((c >> 1) ^ ((row >> 1) & 3))) << 4) + ((c & 1) << 3)) =
              packed;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&xlfull[sl]);
        mbar_arrive(&xempty[sx]);
      }
      if (my_sub >= SUB) continue;  // transform-only warps
      const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
      mbar_wait(&accfull[ab], aph);
      tc_fence_after();
      {
        const int sub = my_sub;
        float acc = 0.f;
        const uint32_t base = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ab * C::ACC_COLS + sub * 2 * C::N;
#pragma unroll
        for (int c0 = 0; c0 < C::N; c0 += 32) {
          uint32_t vh[32], vl[32];
          tmem_ld32(base + c0, vh);
          tmem_ld32(base + C::N + c0, vl);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float u = __uint_as_float(vh[j]) + __uint_as_float(vl[j]);
            acc = fmaf(u, u, acc);
          }
        }
        const int64_t row = t * TILE_ROWS + sub * BM + quarter * 32 + lane;
        if (row < n) scores[row] = static_cast<double>(acc);
      }
      tc_fence_before();
      mbar_arrive(&accempty[ab]);
    }
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// host side

template <int N>
static int32_t launch(const float* X, int64_t n, int64_t d, int64_t ldx, const float* Mt_hi, const float* Mt_lo,
                      int64_t r, double* scores, int32_t* flags, cudaStream_t st) {
  using C = Cfg<N>;
  CUtensorMap mx, mh, ml;
  if (!make_map(&mx, X, d, n, ldx * 4, BK, TILE_ROWS) || !make_map(&mh, Mt_hi, d, r, d * 4, BK, N) ||
      !make_map(&ml, Mt_lo, d, r, d * 4, BK, N)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t arc = ensure_smem_attr(reinterpret_cast<const void*>(leverage_tf32x3_kernel<N>), C::SMEM_BYTES,
                                       "leverage tc smem attribute");
  if (arc != LVSK_OK) return arc;
  const int64_t ntiles = (n + TILE_ROWS - 1) / TILE_ROWS;
  const int grid = static_cast<int>(ntiles < num_sms() ? ntiles : num_sms());
  const int kchunks = static_cast<int>((d + BK - 1) / BK);
  leverage_tf32x3_kernel<N><<<grid, THREADS, C::SMEM_BYTES, st>>>(mx, mh, ml, n, kchunks, scores, flags);
  LVSK_CHECK_LAUNCH("leverage tf32x3");
  return LVSK_OK;
}

static int32_t launch_v2(const float* X, int64_t n, int64_t d, int64_t ldx, const float* Mt_hi, const float* Mt_lo,
                         const __nv_bfloat16* Mt_hb, int64_t r, double* scores, int32_t* flags, cudaStream_t st) {
  using C = Cfg2;
  CUtensorMap mx, mh, ml, mb;
  if (!make_map(&mx, X, d, n, ldx * 4, BK, TILE_ROWS) || !make_map(&mh, Mt_hi, d, r, d * 4, BK, C::N) ||
      !make_map(&ml, Mt_lo, d, r, d * 4, BK, C::N) ||
      !make_map(&mb, Mt_hb, d, r, d * 2, BK, C::N, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_64B)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t arc = ensure_smem_attr(reinterpret_cast<const void*>(leverage_v2_kernel), C::SMEM_BYTES,
                                       "leverage v2 smem attribute");
  if (arc != LVSK_OK) return arc;
  const int64_t ntiles = (n + TILE_ROWS - 1) / TILE_ROWS;
  const int grid = static_cast<int>(ntiles < num_sms() ? ntiles : num_sms());
  const int kchunks = static_cast<int>((d + BK - 1) / BK);
  leverage_v2_kernel<<<grid, V2_THREADS, C::SMEM_BYTES, st>>>(mx, mh, ml, mb, n, kchunks, scores, flags);
  LVSK_CHECK_LAUNCH("leverage v2");
  return LVSK_OK;
}

}  // namespace tc
}  // namespace lvsk

using namespace lvsk;

extern "C" int32_t lvsk_leverage_tf32x3(const float* X, int64_t n, int64_t d, int64_t ldx, const float* Mt_hi,
                                        const float* Mt_lo, const void* Mt_hi_bf16, int64_t r, double* scores,
                                        int32_t* flags, void* stream) {
  LVSK_REQUIRE(n >= 0 && d >= 1 && ldx >= d && r >= 1, LVSK_ERR_DIMENSION, "bad shape");
  LVSK_REQUIRE(r <= 128, LVSK_ERR_UNSUPPORTED, "tensor-core leverage pass supports r <= 128 (got %lld)", (long long)r);
  LVSK_REQUIRE(reinterpret_cast<uintptr_t>(X) % 16 == 0 && (ldx * 4) % 16 == 0 && (d * 4) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(Mt_hi) % 16 == 0 && reinterpret_cast<uintptr_t>(Mt_lo) % 16 == 0,
               LVSK_ERR_UNSUPPORTED, "tensor-core leverage pass needs 16-byte aligned rows");
  LVSK_REQUIRE(n < (int64_t{1} << 31), LVSK_ERR_UNSUPPORTED, "n too large for one launch");
  if (n == 0) return LVSK_OK;
  cudaStream_t st = as_stream(stream);
  if (r <= 64 && Mt_hi_bf16 != nullptr && d % 8 == 0 && reinterpret_cast<uintptr_t>(Mt_hi_bf16) % 16 == 0 &&
      getenv("LVSK_K5_V1") == nullptr)
    return tc::launch_v2(X, n, d, ldx, Mt_hi, Mt_lo, static_cast<const __nv_bfloat16*>(Mt_hi_bf16), r, scores, flags,
                         st);
  if (r <= 64) return tc::launch<64>(X, n, d, ldx, Mt_hi, Mt_lo, r, scores, flags, st);
  return tc::launch<128>(X, n, d, ldx, Mt_hi, Mt_lo, r, scores, flags, st);
}
