// K5 for bf16 X on tcgen05 (BASELINE config 5: X stored in bf16, fp32
// accumulation, r = 128): scores[i] = || X[i,:] M ||^2 with M split
// M = M_hi + M_lo (both bf16, ~16 significant bits together) and ONE
// kind::f16 MMA of N = 2*r_pad per K-step: the accumulator holds x.M_hi in
// columns [0, r_pad) and x.M_lo in [r_pad, 2 r_pad); the epilogue adds the
// halves, squares and row-reduces.  bf16 X values are exact operands, so no
// transform warps are needed.
//
// Reference: _block_scores (pkg/src/levsketch/leverage.py:88-95).
//
// Persistent CTA per SM: warp 0 = TMA (lane 0: X ring of 6 x [128 x 64]
// bf16 SW128; lane 1: M ring of 2 x [N2 x 64]), warp 1 = MMA issuer, warps
// 2-5 = epilogue; 128-row tiles, accumulators double-buffered in TMEM.
#include <cstdlib>

#include "tc_common.cuh"

namespace lvsk {
namespace tc {

template <int N2>
struct CfgB {
  static constexpr int BKB = 64;                          // bf16 per 128-byte swizzle row
  static constexpr int SX = 6, SB = 2;
  static constexpr int X_BYTES = BM * BKB * 2;            // 16 KB
  static constexpr int B_BYTES = N2 * BKB * 2;            // up to 32 KB
  static constexpr int OFF_B = SX * X_BYTES;
  static constexpr int OFF_BAR = OFF_B + SB * B_BYTES;
  static constexpr int TMEM_COLS = 2 * N2 <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = OFF_BAR + 1024 + 256;
  static constexpr uint32_t IDESC =
      (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N2 >> 3) << 17) | (uint32_t(BM >> 4) << 24);
};

template <int N2>
__global__ void __launch_bounds__(THREADS, 1)
    leverage_bf16_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapM,
                         int64_t n, int kchunks, int r, double* __restrict__ scores) {
  using C = CfgB<N2>;
  constexpr int RP = N2 / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays a shared-space pointer
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* xfull = bars;
  uint64_t* xempty = xfull + C::SX;
  uint64_t* bfull = xempty + C::SX;
  uint64_t* bempty = bfull + C::SB;
  uint64_t* accfull = bempty + C::SB;
  uint64_t* accempty = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + BM - 1) / BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::SX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < C::SB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], EPI_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapM) : "memory");
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
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::SX, ph = (it / C::SX) & 1u;
          mbar_wait(&xempty[s], ph ^ 1u);
          mbar_expect_tx(&xfull[s], C::X_BYTES);
          tma_load_2d(&mapX, &xfull[s], smem + s * C::X_BYTES, kc * C::BKB, static_cast<int>(t * BM), pol);
        }
    } else if (lane == 1) {
      const uint64_t pol = l2_policy_evict_last();
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::SB, ph = (it / C::SB) & 1u;
          mbar_wait(&bempty[s], ph ^ 1u);
          mbar_expect_tx(&bfull[s], C::B_BYTES);
          tma_load_2d(&mapM, &bfull[s], smem + C::OFF_B + s * C::B_BYTES, kc * C::BKB, 0, pol);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
        mbar_wait(&accempty[ab], aph ^ 1u);
        tc_fence_after();
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t sx = it % C::SX, phx = (it / C::SX) & 1u;
          const uint32_t sb = it % C::SB, phb = (it / C::SB) & 1u;
          mbar_wait(&xfull[sx], phx);
          mbar_wait(&bfull[sb], phb);
          tc_fence_after();
          const uint64_t a = sw128_desc(smem_u32(smem + sx * C::X_BYTES));
          const uint64_t b = sw128_desc(smem_u32(smem + C::OFF_B + sb * C::B_BYTES));
#pragma unroll
          for (int kk = 0; kk < C::BKB / 16; ++kk)
            umma_f16(tmem_base + ab * N2, a + 2 * kk, b + 2 * kk, C::IDESC, (kc | kk) ? 1u : 0u);
          umma_commit(&xempty[sx]);
          umma_commit(&bempty[sb]);
          if (kc == kchunks - 1) umma_commit(&accfull[ab]);
        }
      }
    }
  } else {
    const int quarter = warp & 3;
    uint32_t lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
      mbar_wait(&accfull[ab], aph);
      tc_fence_after();
      const uint32_t base = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ab * N2;
      float acc = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < RP; c0 += 32) {
        uint32_t vh[32], vl[32];
        tmem_ld32(base + c0, vh);
        tmem_ld32(base + RP + c0, vl);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (c0 + j < r) {
            const float u = __uint_as_float(vh[j]) + __uint_as_float(vl[j]);
            acc = fmaf(u, u, acc);
          }
        }
      }
      const int64_t row = t * BM + quarter * 32 + lane;
      if (row < n) scores[row] = static_cast<double>(acc);
      tc_fence_before();
      mbar_arrive(&accempty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

// ---- CTA-pair variant (cta_group::2) -------------------------------------
// Two CTAs of a cluster form one M = 256 MMA: each holds its 128 rows of X
// (the A half) and HALF of the N2 columns of [M_hi | M_lo] (the B half), the
// leader (rank 0) issues tcgen05.mma.cta_group::2 and each CTA's TMEM
// receives its 128 rows x N2 accumulators.  Per CTA and k-chunk the shared
// memory then takes 16 KB of X + 16 KB of M (instead of 16 + 32 KB) and the
// MMA reads half of B from it: the 1-CTA kernel streams M through shared
// memory once per 128 rows, which bounds it at ~66 % of HBM (C5); the pair
// streams it once per 256 rows and reads half per SM.
template <int N2>
struct CfgP {
  static constexpr int BKB = 64;
  static constexpr int SX = 6;
  static constexpr int X_BYTES = BM * BKB * 2;             // 16 KB (this CTA's 128 rows)
  static constexpr int B_BYTES = (N2 / 2) * BKB * 2;       // 16 KB (this CTA's half of N2)
  static constexpr int STAGE = X_BYTES + B_BYTES;
  static constexpr int OFF_BAR = SX * STAGE;
  static constexpr int TMEM_COLS = 2 * N2 <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = OFF_BAR + 1024 + 256;
  // kind::f16, F32 accumulate, bf16 A / B, both K-major, N = N2, M = 256
  static constexpr uint32_t IDESC =
      (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N2 >> 3) << 17) | (uint32_t(256 >> 4) << 24);
};

template <int N2>
__global__ void __launch_bounds__(THREADS, 1)
    leverage_bf16_pair_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapM,
                              int64_t n, int kchunks, int r, double* __restrict__ scores) {
  using C = CfgP<N2>;
  constexpr int RP = N2 / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;              // leader: X + M bytes of both CTAs
  uint64_t* empty = full + C::SX;     // both: the pair's MMA released the slot
  uint64_t* accfull = empty + C::SX;  // both: tile accumulators ready
  uint64_t* accempty = accfull + 2;   // leader: both CTAs drained the accumulators
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t ntiles = (n + 2 * BM - 1) / (2 * BM);  // 256-row pair tiles

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::SX; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 2);  // one arrive per CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapM) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_pair();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t polx = l2_policy_evict_first(), polm = l2_policy_evict_last();
      uint32_t it = 0;
      for (int64_t t = pair; t < ntiles; t += npairs)
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::SX, ph = (it / C::SX) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          const uint32_t leader_full = mapa_rank(smem_u32(&full[s]), 0);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * C::STAGE);
          uint8_t* st = smem + s * C::STAGE;
          tma_load_2d_pair(&mapX, leader_full, st, kc * C::BKB, static_cast<int>(t * 2 * BM + rank * BM), polx);
          tma_load_2d_pair(&mapM, leader_full, st + C::X_BYTES, kc * C::BKB, static_cast<int>(rank * RP), polm);
        }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      uint32_t it = 0, lt = 0;
      for (int64_t t = pair; t < ntiles; t += npairs, ++lt) {
        const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
        mbar_wait(&accempty[ab], aph ^ 1u);
        tc_fence_after();
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const uint32_t s = it % C::SX, ph = (it / C::SX) & 1u;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a = sw128_desc(smem_u32(smem + s * C::STAGE));
          const uint64_t b = sw128_desc(smem_u32(smem + s * C::STAGE + C::X_BYTES));
#pragma unroll
          for (int kk = 0; kk < C::BKB / 16; ++kk)
            umma_f16_pair(tmem_base + ab * N2, a + 2 * kk, b + 2 * kk, C::IDESC, (kc | kk) ? 1u : 0u);
          umma_commit_mask(&empty[s], 3);
          if (kc == kchunks - 1) umma_commit_mask(&accfull[ab], 3);
        }
      }
    }
  } else {
    const int quarter = warp & 3;
    uint32_t lt = 0;
    const uint32_t leader_accempty = mapa_rank(smem_u32(&accempty[0]), 0);
    for (int64_t t = pair; t < ntiles; t += npairs, ++lt) {
      const uint32_t ab = lt & 1u, aph = (lt >> 1) & 1u;
      mbar_wait(&accfull[ab], aph);
      tc_fence_after();
      const uint32_t base = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ab * N2;
      float acc = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < RP; c0 += 32) {
        uint32_t vh[32], vl[32];
        tmem_ld32(base + c0, vh);
        tmem_ld32(base + RP + c0, vl);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (c0 + j < r) {
            const float u = __uint_as_float(vh[j]) + __uint_as_float(vl[j]);
            acc = fmaf(u, u, acc);
          }
        }
      }
      const int64_t row = t * 2 * BM + rank * BM + quarter * 32 + lane;
      if (row < n) scores[row] = static_cast<double>(acc);
      tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");  // this CTA's epilogue drained the buffer
      if (warp == 2 && lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_accempty + 8 * ab)
                     : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_pair();  // neither CTA frees TMEM / leaves while the pair's MMAs may still run
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

template <int N2>
static int32_t launch_bf16_pair(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, const __nv_bfloat16* Mt,
                                int r, double* scores, cudaStream_t st) {
  using C = CfgP<N2>;
  CUtensorMap mx, mm;
  if (!make_map(&mx, X, d, n, ldx * 2, C::BKB, BM, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) ||
      !make_map(&mm, Mt, d, N2, d * 2, C::BKB, N2 / 2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t arc = ensure_smem_attr(reinterpret_cast<const void*>(leverage_bf16_pair_kernel<N2>), C::SMEM_BYTES,
                                       "leverage bf16 pair smem attribute");
  if (arc != LVSK_OK) return arc;
  const int64_t ntiles = (n + 2 * BM - 1) / (2 * BM);
  const int64_t pairs = ntiles < num_sms() / 2 ? ntiles : num_sms() / 2;
  const int kchunks = static_cast<int>((d + C::BKB - 1) / C::BKB);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, leverage_bf16_pair_kernel<N2>, mx, mm, n, kchunks, r, scores);
  if (e != cudaSuccess) return cuda_status(e, "leverage bf16 pair launch");
  return LVSK_OK;
}

template <int N2>
static int32_t launch_bf16(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, const __nv_bfloat16* Mt,
                           int r, double* scores, cudaStream_t st) {
  using C = CfgB<N2>;
  CUtensorMap mx, mm;
  if (!make_map(&mx, X, d, n, ldx * 2, C::BKB, BM, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) ||
      !make_map(&mm, Mt, d, N2, d * 2, C::BKB, N2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t arc = ensure_smem_attr(reinterpret_cast<const void*>(leverage_bf16_kernel<N2>), C::SMEM_BYTES,
                                       "leverage bf16 smem attribute");
  if (arc != LVSK_OK) return arc;
  const int64_t ntiles = (n + BM - 1) / BM;
  const int grid = static_cast<int>(ntiles < num_sms() ? ntiles : num_sms());
  const int kchunks = static_cast<int>((d + C::BKB - 1) / C::BKB);
  leverage_bf16_kernel<N2><<<grid, THREADS, C::SMEM_BYTES, st>>>(mx, mm, n, kchunks, r, scores);
  LVSK_CHECK_LAUNCH("leverage bf16");
  return LVSK_OK;
}

}  // namespace tc
}  // namespace lvsk

using namespace lvsk;

extern "C" int32_t lvsk_leverage_bf16(const void* X, int64_t n, int64_t d, int64_t ldx, const void* Mt, int64_t r,
                                      int64_t r_pad, double* scores, int32_t* flags, void* stream) {
  (void)flags;  // bf16 inputs: finiteness of X is checked by the sketch kernel that precedes this pass
  LVSK_REQUIRE(n >= 0 && d >= 1 && ldx >= d && r >= 1 && r <= r_pad, LVSK_ERR_DIMENSION, "bad shape");
  LVSK_REQUIRE(r_pad == 32 || r_pad == 64 || r_pad == 128, LVSK_ERR_UNSUPPORTED,
               "bf16 tensor-core leverage pass needs r_pad in {32, 64, 128} (got %lld)", (long long)r_pad);
  LVSK_REQUIRE(reinterpret_cast<uintptr_t>(X) % 16 == 0 && (ldx * 2) % 16 == 0 && (d * 2) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(Mt) % 16 == 0,
               LVSK_ERR_UNSUPPORTED, "bf16 tensor-core leverage pass needs 16-byte aligned rows");
  if (n == 0) return LVSK_OK;
  cudaStream_t st = as_stream(stream);
  const auto* x = static_cast<const __nv_bfloat16*>(X);
  const auto* m = static_cast<const __nv_bfloat16*>(Mt);
  if (r_pad == 128 && getenv("LVSK_K5_SINGLE_CTA") == nullptr)  // C5: the CTA-pair kernel
    return tc::launch_bf16_pair<256>(x, n, d, ldx, m, static_cast<int>(r), scores, st);
  switch (r_pad) {
    case 32: return tc::launch_bf16<64>(x, n, d, ldx, m, static_cast<int>(r), scores, st);
    case 64: return tc::launch_bf16<128>(x, n, d, ldx, m, static_cast<int>(r), scores, st);
    default: return tc::launch_bf16<256>(x, n, d, ldx, m, static_cast<int>(r), scores, st);
  }
}
