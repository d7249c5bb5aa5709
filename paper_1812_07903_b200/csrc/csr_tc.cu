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
