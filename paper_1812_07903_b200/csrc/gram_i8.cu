// KG — the fold's Gram matrix G = SX^T SX in float64 on the int8 tensor cores
// (Ozaki scheme), replacing cuBLAS's sm80 DGEMM (cutlass_80_tensorop_d884:
// 9.7 ms at C4, d = 4096, at the fp64 peak).  Reference: the small
// factorisation of the sketch (pkg/src/levsketch/svd.py:30-37,
// leverage.py:75-85) — the certified Cholesky fold (factor.cu) factors G.
//
// Split: every column c of SX is scaled by 2^-e_c (e_c = exponent of its
// largest |entry|, so |t| < 1) and cut into T = 7 signed 7-bit slices,
//     t = sum_s a_s 2^(-7 (s + 1)) + r,   a_s in [-127, 127],  |r| < 2^-49,
// exactly in float64 (multiplications by powers of two and subtractions of
// integers).  Then
//     G[c][d] = 2^(e_c + e_d) sum_q 2^(-7 (q + 2)) C_q[c][d],
//     C_q = sum_{s + u = q} A_s^T A_u      (q = 0 .. T-1)
// and every C_q is an EXACT int32 dot product on the tensor cores
// (kind::i8, |C_q| <= 7 * k * 127^2 < 2^31 for k <= 16384 * 1.1).  Dropping
// the pairs with s + u >= T errs by < 2^-49 of sum_k |t_kc| |t_kd| — the
// error class of a float64 GEMM (k eps |SX_c| |SX_d|).  C_q is scaled and
// added into G in float64 in ascending q: deterministic.
//
// GEMM: M = N = d (columns of SX), K = k (rows).  The slices keep SX's
// row-major layout (k x d_pad int8), so both operands are MN-major SW128
// (128-byte boxes of 128 columns x BK rows; int8 MN-major UMMA operands).
// One CTA pair (tcgen05.mma.cta_group::2, M = 256) owns a 256 x 256 tile of
// the block upper triangle (and a K split when there are few tiles): each
// CTA holds its 128 A columns and half of the 256 B columns, the even rank
// issues kind::i8 MMAs (M = 256, N = 256, K = 32) into int32 TMEM
// accumulators double-buffered across q, and 4 epilogue warps per CTA scale
// and add each C_q tile into the float64 output (split partials are summed
// in a fixed order by a small reduce kernel).
#include <cstdlib>

#include "tc_common.cuh"

namespace lvsk {
namespace kg {

constexpr int EPI_WARPS_ = 8;
constexpr int T = 7;           // slices
constexpr int BK = 128;        // K rows per stage
constexpr int TILE = 256;      // output tile (M and N)
constexpr int S = 4;           // stages
constexpr int BOX = BK * 128;  // 16 KB: 128 int8 columns x BK rows
constexpr int STAGE = 2 * BOX; // A box + B box
constexpr int EPI_WARPS = EPI_WARPS_;           // two per TMEM lane quarter, 128 columns each
constexpr int OFF_EPI = S * STAGE;              // per epilogue warp: a 32 x 33 float64 transpose tile
constexpr int EPI_BYTES = EPI_WARPS * 32 * 33 * 8;
constexpr int OFF_BAR = OFF_EPI + EPI_BYTES;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;
constexpr int THREADS = 64 + 32 * EPI_WARPS_;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
// kind::i8: S32 accumulate, signed int8 A / B, both MN-major, N = 256, M = 256 (pair)
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (uint32_t(256 >> 3) << 17) |
                           (uint32_t(256 >> 4) << 24);

// MN-major SWIZZLE_128B for 8-bit data: 128-element x 8-row atoms; LBO =
// stride between 128-element MN blocks (one box), SBO = 8 K-rows (1024 B).
__device__ __forceinline__ uint64_t mn_desc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(BOX >> 4) << 16;
  d |= uint64_t{1024 >> 4} << 32;
  d |= uint64_t{1} << 46;
  d |= uint64_t{2} << 61;
  return d;
}

__device__ __forceinline__ void umma_i8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}

// per-column max |x| as ordered int64 bits (positive doubles order like ints)
__global__ void colmax_kernel(const double* __restrict__ X, int64_t k, int64_t d, int64_t ldx,
                              unsigned long long* __restrict__ cmax) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= d) return;
  const int64_t rpb = (k + gridDim.y - 1) / gridDim.y;  // rows per y block
  const int64_t r0 = blockIdx.y * rpb;
  const int64_t r1 = r0 + rpb < k ? r0 + rpb : k;
  unsigned long long m = 0;
  for (int64_t r = r0; r < r1; ++r) {
    const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(fabs(X[r * ldx + c])));
    m = v > m ? v : m;
  }
  atomicMax(cmax + c, m);
}

// e_c with max|x_c| < 2^e_c (0 for an all-zero column); non-finite -> flag
__global__ void colexp_kernel(const unsigned long long* __restrict__ cmax, int64_t d, int64_t dp,
                              int32_t* __restrict__ e, int32_t* flags) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= dp) return;
  if (c >= d) {
    e[c] = 0;
    return;
  }
  const double m = __longlong_as_double(static_cast<long long>(cmax[c]));
  if (!isfinite(m)) {
    atomicOr(flags, LVSK_FLAG_NONFINITE);
    e[c] = 0;
    return;
  }
  int ex = 0;
  if (m > 0.0) {
    frexp(m, &ex);  // m = f 2^ex, f in [0.5, 1)  ->  m < 2^ex
  }
  e[c] = ex;
}

// slices [T][kp][dp] int8 (zero padded): thread -> 4 consecutive columns of
// one row (coalesced float64 reads, 4-byte slice stores)
__global__ void slice_kernel(const double* __restrict__ X, int64_t k, int64_t d, int64_t ldx, int64_t kp, int64_t dp,
                             const int32_t* __restrict__ e, int8_t* __restrict__ sl) {
  const int64_t total = kp * dp;
  const int64_t c4 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 4;
  if (c4 >= dp) return;
  int ex[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) ex[j] = e[c4 + j];
  for (int64_t r = blockIdx.y; r < kp; r += gridDim.y) {
    double t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = c4 + j;
      t[j] = (r < k && c < d) ? ldexp(X[r * ldx + c], -ex[j]) : 0.0;
      if (!isfinite(t[j])) t[j] = 0.0;  // flagged by colexp_kernel
    }
#pragma unroll
    for (int s = 0; s < T; ++s) {
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double v = t[j] * 128.0;
        const double a = trunc(v);
        w |= (static_cast<uint32_t>(static_cast<int>(a)) & 0xFFu) << (8 * j);
        t[j] = v - a;
      }
      *reinterpret_cast<uint32_t*>(sl + static_cast<int64_t>(s) * total + r * dp + c4) = w;
    }
  }
}

struct Args {
  int64_t kp, dp;             // padded rows / columns of a slice
  int nt;                     // 256-column tiles
  int splits;                 // K splits per tile
  int64_t chunks_per_split;   // BK-row chunks per split
  const int32_t* e;           // column exponents
  double* out;                // [splits][dp][dp] (split 0 = G itself when splits == 1)
  int64_t ldo;
};

__device__ __forceinline__ void tile_of(int p, int nt, int& I, int& J) {
  // p-th (I, J), I <= J, row-major over the upper triangle
  int i = 0, rem = p;
  while (rem >= nt - i) {
    rem -= nt - i;
    ++i;
  }
  I = i;
  J = i + rem;
}

__global__ void __launch_bounds__(THREADS, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap map, const Args A) {
  using namespace tc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;             // leader: both CTAs' A + B bytes
  uint64_t* empty = full + S;        // both
  uint64_t* accfull = empty + S;     // both: C_q tile ready (2 buffers)
  uint64_t* accempty = accfull + 2;  // leader: both CTAs drained the buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int item = blockIdx.x >> 1;
  const int tile = item / A.splits, split = item % A.splits;
  int I, J;
  tile_of(tile, A.nt, I, J);
  const int64_t ch0 = static_cast<int64_t>(split) * A.chunks_per_split;
  const int64_t nch_total = A.kp / BK;
  const int64_t ch1 = ch0 + A.chunks_per_split < nch_total ? ch0 + A.chunks_per_split : nch_total;
  const int nch = static_cast<int>(ch1 - ch0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_pair();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // columns of this CTA's A half and B half; rows are slice-stacked: slice s row r -> s * kp + r
  const int acol = I * TILE + static_cast<int>(rank) * 128;
  const int bcol = J * TILE + static_cast<int>(rank) * 128;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      const uint32_t lead_full = mapa_rank(smem_u32(&full[0]), 0);
      uint32_t it = 0;
      for (int q = 0; q < T; ++q)
        for (int s = 0; s <= q; ++s)
          for (int c = 0; c < nch; ++c, ++it) {
            const uint32_t st = it % S, ph = (it / S) & 1u;
            mbar_wait(&empty[st], ph ^ 1u);
            if (rank == 0) mbar_expect_tx(&full[st], 2 * STAGE);
            const int64_t row = ch0 * BK + static_cast<int64_t>(c) * BK;
            uint8_t* dst = smem + st * STAGE;
            tma_load_2d_pair(&map, lead_full + 8 * st, dst, acol, static_cast<int>(s * A.kp + row), pol);
            tma_load_2d_pair(&map, lead_full + 8 * st, dst + BOX, bcol, static_cast<int>((q - s) * A.kp + row),
                             pol);
          }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      uint32_t it = 0;
      for (int q = 0; q < T; ++q) {
        const uint32_t ab = q & 1, aph = (q >> 1) & 1u;
        mbar_wait(&accempty[ab], aph ^ 1u);
        tc_fence_after();
        bool first = true;
        for (int s = 0; s <= q; ++s)
          for (int c = 0; c < nch; ++c, ++it) {
            const uint32_t st = it % S, ph = (it / S) & 1u;
            mbar_wait(&full[st], ph);
            tc_fence_after();
            const uint32_t base = smem_u32(smem + st * STAGE);
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk) {  // K = 32 per MMA: 32 rows x 128 B
              umma_i8_pair(tmem_base + ab * 256, mn_desc(base + kk * 4096), mn_desc(base + BOX + kk * 4096),
                           first ? 0u : 1u);
              first = false;
            }
            umma_commit_mask(&empty[st], 3);
          }
        umma_commit_mask(&accfull[ab], 3);
      }
    }
  } else {
    // ---- epilogue: this CTA's 128 rows (columns acol.. of SX) x 256 columns of
    //      the tile.  TMEM gives each thread one row; a per-warp shared-memory
    //      transpose turns that into row-contiguous (coalesced) float64
    //      read-modify-writes of the output
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int64_t rbase = acol + quarter * 32;  // first G row of this warp
    const int er = A.e[rbase + lane];
    const uint32_t lead_accempty = mapa_rank(smem_u32(&accempty[0]), 0);
    double* tb = reinterpret_cast<double*>(smem + OFF_EPI) + (warp - 2) * 32 * 33;
    double* obase = A.out + static_cast<int64_t>(split) * A.dp * A.ldo + rbase * A.ldo + J * TILE;
    const int32_t* ecol = A.e + J * TILE;
    for (int q = 0; q < T; ++q) {
      const uint32_t ab = q & 1, aph = (q >> 1) & 1u;
      mbar_wait(&accfull[ab], aph);
      tc_fence_after();
      const int sh = -7 * (q + 2) + er;
#pragma unroll 1
      for (int c0 = 128 * half; c0 < 128 * half + 128; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ab * 256 + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) tb[lane * 33 + j] = ldexp(static_cast<double>(static_cast<int32_t>(v[j])), sh);
        __syncwarp();
        const int ec = ecol[c0 + lane];
        double* o = obase + c0 + lane;  // row rbase + rr, column c0 + lane
        if (q == 0) {
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) o[rr * A.ldo] = ldexp(tb[rr * 33 + lane], ec);
        } else {
#pragma unroll
          for (int h = 0; h < 32; h += 16) {  // 16 loads in flight before the adds
            double old[16];
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) old[rr] = __ldcg(o + (h + rr) * A.ldo);
#pragma unroll
            for (int rr = 0; rr < 16; ++rr)
              o[(h + rr) * A.ldo] = old[rr] + ldexp(tb[(h + rr) * 33 + lane], ec);
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
      if (warp == 2 && lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lead_accempty + 8 * ab)
                     : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_pair();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512));
  }
}

// G[r][c] = sum over splits (fixed order), upper tiles only; lower tiles untouched
__global__ void split_reduce_kernel(const double* __restrict__ part, int splits, int64_t dp, int64_t d,
                                    double* __restrict__ G, int64_t ldg) {
  const int64_t total = d * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / d, c = i - r * d;
    if (r / TILE > c / TILE) continue;
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += part[(static_cast<int64_t>(p) * dp + r) * dp + c];
    G[r * ldg + c] = s;
  }
}

// copy the upper tiles of the (dp x dp) result into G when G is not the buffer itself
__global__ void copy_upper_kernel(const double* __restrict__ src, int64_t dp, int64_t d, double* __restrict__ G,
                                  int64_t ldg) {
  const int64_t total = d * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / d, c = i - r * d;
    if (r / TILE > c / TILE) continue;
    G[r * ldg + c] = src[r * dp + c];
  }
}

struct Plan {
  int64_t kp, dp;
  int nt, ntiles, splits;
  int64_t chunks_per_split;
};

inline Plan plan(int64_t k, int64_t d) {
  Plan p;
  p.kp = (k + BK - 1) / BK * BK;
  p.dp = (d + TILE - 1) / TILE * TILE;
  p.nt = static_cast<int>(p.dp / TILE);
  p.ntiles = p.nt * (p.nt + 1) / 2;
  const int64_t chunks = p.kp / BK;
  int64_t sp = (num_sms() / 2) / p.ntiles;  // CTA pairs per tile to fill the GPU
  if (sp < 1) sp = 1;
  if (sp > chunks / 8) sp = chunks / 8 > 0 ? chunks / 8 : 1;
  p.chunks_per_split = (chunks + sp - 1) / sp;
  p.splits = static_cast<int>((chunks + p.chunks_per_split - 1) / p.chunks_per_split);
  return p;
}

}  // namespace kg
}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_gram_workspace_bytes(int64_t k, int64_t d) {
  const kg::Plan p = kg::plan(k, d);
  Measure m;
  m.take<unsigned long long>(p.dp);
  m.take<int32_t>(p.dp);
  m.take<int8_t>(static_cast<size_t>(kg::T) * p.kp * p.dp);
  m.take<double>(static_cast<size_t>(p.splits) * p.dp * p.dp);
  return m.off;
}

extern "C" int32_t lvsk_gram_f64(const double* SX, int64_t k, int64_t d, int64_t ldsx, double* G, int64_t ldg,
                                 void* ws, size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(k >= 1 && d >= 1 && ldsx >= d && ldg >= d, LVSK_ERR_DIMENSION, "bad Gram shape k=%lld d=%lld",
               (long long)k, (long long)d);
  // exactness of the int32 accumulation: 7 slice pairs x k x 127^2 < 2^31
  LVSK_REQUIRE(k <= 18000, LVSK_ERR_UNSUPPORTED, "int8 Gram needs k <= 18000 (got %lld)", (long long)k);
  const kg::Plan p = kg::plan(k, d);
  Carve c(ws, ws_bytes);
  unsigned long long* cmax = c.take<unsigned long long>(p.dp);
  int32_t* e = c.take<int32_t>(p.dp);
  int8_t* sl = c.take<int8_t>(static_cast<size_t>(kg::T) * p.kp * p.dp);
  double* part = c.take<double>(static_cast<size_t>(p.splits) * p.dp * p.dp);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  cudaStream_t st = as_stream(stream);
  cudaError_t er = cudaMemsetAsync(cmax, 0, p.dp * sizeof(unsigned long long), st);
  if (er != cudaSuccess) return cuda_status(er, "gram memset");
  const int ysplit = static_cast<int>(k / 256 > 64 ? 64 : (k / 256 > 0 ? k / 256 : 1));
  kg::colmax_kernel<<<dim3(static_cast<unsigned>((d + 255) / 256), ysplit), 256, 0, st>>>(SX, k, d, ldsx, cmax);
  kg::colexp_kernel<<<static_cast<unsigned>((p.dp + 255) / 256), 256, 0, st>>>(cmax, d, p.dp, e, flags);
  const unsigned gx = static_cast<unsigned>((p.dp / 4 + 127) / 128);
  const unsigned gy = static_cast<unsigned>(p.kp < 4096 ? p.kp : 4096);
  kg::slice_kernel<<<dim3(gx, gy), 128, 0, st>>>(SX, k, d, ldsx, p.kp, p.dp, e, sl);
  LVSK_CHECK_LAUNCH("gram slicing");
  CUtensorMap map;
  if (!tc::make_map(&map, sl, p.dp, kg::T * p.kp, p.dp, 128, kg::BK, CU_TENSOR_MAP_DATA_TYPE_UINT8)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t rc = ensure_smem_attr(reinterpret_cast<const void*>(kg::gram_i8_kernel), kg::SMEM_BYTES,
                                      "gram smem attribute");
  if (rc != LVSK_OK) return rc;
  const bool direct = p.splits == 1 && G != nullptr && ldg == p.dp && d == p.dp;
  kg::Args a;
  a.kp = p.kp;
  a.dp = p.dp;
  a.nt = p.nt;
  a.splits = p.splits;
  a.chunks_per_split = p.chunks_per_split;
  a.e = e;
  a.out = direct ? G : part;
  a.ldo = p.dp;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * p.ntiles * p.splits));
  cfg.blockDim = dim3(kg::THREADS);
  cfg.dynamicSmemBytes = kg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  er = cudaLaunchKernelEx(&cfg, kg::gram_i8_kernel, map, a);
  if (er != cudaSuccess) return cuda_status(er, "gram launch");
  if (!direct) {
    const int64_t tot2 = d * d;
    const int g2 = static_cast<int>((tot2 + 255) / 256 < num_sms() * 16 ? (tot2 + 255) / 256 : num_sms() * 16);
    if (p.splits > 1)
      kg::split_reduce_kernel<<<g2, 256, 0, st>>>(part, p.splits, p.dp, d, G, ldg);
    else
      kg::copy_upper_kernel<<<g2, 256, 0, st>>>(part, p.dp, d, G, ldg);
  }
  LVSK_CHECK_LAUNCH("gram");
  return LVSK_OK;
}
