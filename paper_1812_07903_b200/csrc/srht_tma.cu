// K3 (fp32) — SRHT passes as persistent, warp-specialised TMA pipelines.
//
// Same algorithm and butterfly order as srht.cu (reference SketchState.data
// SRHT branch + fwht, pkg/src/levsketch/sketch.py:248-257, 364-385): a chunk
// of 2^(8+B2) rows is transformed over its low 8 bits in pass 1 (sign flip
// fused) into the L2-resident buffer T1, and over the next B2 bits in pass 2,
// which also applies the chunk's high-bit signs and accumulates the sampled
// rows into SX.  What changes is the data movement: one CTA per SM, a
// producer warp streams [256 rows x 32 columns] tiles with TMA into a 4-deep
// mbarrier ring (pass 1: a 2-D box of X; pass 2: a 3-D box of T1 viewed as
// [i2][q1][d], i.e. the 2^B2 rows q1 + 256 i2 of one residue in one box), and
// four compute warps run the 16 x 16 radix-2 WHT in registers, in place in
// the stage buffer, so loads, butterflies and stores of different tiles
// overlap instead of running as one-shot CTAs.  (Opt-in; see srht_tma_ok.)
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace lvsk {
namespace srht_tma {

constexpr int ROWS = 256;                 // tile rows (pass 1: the low 8 index bits)
constexpr int COLS = 32;                  // fp32 columns per tile (128 B)
constexpr int TILE_BYTES = ROWS * COLS * 4;  // 32 KB
constexpr int GROUPS = 3;                 // compute groups (4 warps each), one tile in flight per group
constexpr int STAGES = 2 * GROUPS;        // 6 x 32 KB ring
constexpr int CWARPS = 4 * GROUPS;        // compute warps
constexpr int NTHREADS = 32 * (CWARPS + 1);
constexpr int SMEM_BYTES = STAGES * TILE_BYTES + 1024 + 256;

// named barrier of one 128-thread compute group
__device__ __forceinline__ void bar_group(int g) { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); }

__device__ __forceinline__ void st_f4_keep(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}

template <int N>
__device__ __forceinline__ void wht_rows(float (&v)[N][4]) {
#pragma unroll
  for (int h = 1; h < N; h <<= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i & h) == 0) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float a = v[i][w], b = v[i + h][w];
          v[i][w] = a + b;
          v[i + h][w] = a - b;
        }
      }
    }
  }
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---- pass 1: T1[chunk-local rows] = WHT_8(sign * X[chunk rows]) ---------------
__global__ void __launch_bounds__(NTHREADS, 1)
    srht_p1_tma_kernel(const __grid_constant__ CUtensorMap mapX, int64_t row0, int64_t chunk_rows, int64_t d,
                       const int8_t* __restrict__ signs, float* __restrict__ T1, int32_t* flags) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rblocks = chunk_rows / ROWS;
  const int cblocks = static_cast<int>((d + COLS - 1) / COLS);
  const int64_t ntiles = rblocks * cblocks;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
  }
  __syncthreads();
  if (warp == CWARPS) {
    if (lane == 0) {
      const uint64_t pol = tc::l2_policy_evict_first();
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
        tc::mbar_wait(&empty[s], ph ^ 1u);
        tc::mbar_expect_tx(&full[s], TILE_BYTES);
        const int64_t rb = t / cblocks, cb = t - rb * cblocks;
        tc::tma_load_2d(&mapX, &full[s], smem + s * TILE_BYTES, static_cast<int>(cb * COLS),
                        static_cast<int>(row0 + rb * ROWS), pol);
      }
    }
    return;
  }
  const int grp = warp >> 2, tid = threadIdx.x & 127;  // compute group, thread in group
  const int q = tid & 7, rg = tid >> 3;  // column quad, row group
  const uint64_t keep = tc::l2_policy_evict_last();
  bool bad = false;
  uint32_t it = grp;
  for (int64_t t = blockIdx.x + static_cast<int64_t>(grp) * gridDim.x; t < ntiles;
       t += static_cast<int64_t>(GROUPS) * gridDim.x, it += GROUPS) {
    const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
    const int64_t rb = t / cblocks, cb = t - rb * cblocks;
    const int64_t grow0 = row0 + rb * ROWS;
    // signs of rows rg*16 .. rg*16+15 (16-byte aligned: grow0 is a multiple of 256)
    const int4 s16 = signs ? *reinterpret_cast<const int4*>(signs + grow0 + rg * 16)
                           : make_int4(0x01010101, 0x01010101, 0x01010101, 0x01010101);  // plain fwht
    const int8_t* sg = reinterpret_cast<const int8_t*>(&s16);
    tc::mbar_wait(&full[s], ph);
    float* tile = reinterpret_cast<float*>(smem + s * TILE_BYTES);
    float v[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float4 x = *reinterpret_cast<const float4*>(tile + (rg * 16 + j) * COLS + q * 4);
      const float f = sg[j] < 0 ? -1.f : 1.f;
      v[j][0] = f * x.x;
      v[j][1] = f * x.y;
      v[j][2] = f * x.z;
      v[j][3] = f * x.w;
      bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
    }
    wht_rows<16>(v);  // index bits 0-3
#pragma unroll
    for (int j = 0; j < 16; ++j)
      *reinterpret_cast<float4*>(tile + (rg * 16 + j) * COLS + q * 4) = make_float4(v[j][0], v[j][1], v[j][2], v[j][3]);
    bar_group(grp);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float4 x = *reinterpret_cast<const float4*>(tile + (rg + 16 * j) * COLS + q * 4);
      v[j][0] = x.x;
      v[j][1] = x.y;
      v[j][2] = x.z;
      v[j][3] = x.w;
    }
    wht_rows<16>(v);  // index bits 4-7
    const int64_t col = cb * COLS + q * 4;
    if (col < d) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        st_f4_keep(T1 + (rb * ROWS + rg + 16 * j) * d + col, make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), keep);
    }
    bar_group(grp);  // every thread of the group is done with the slot
    if (tid == 0) tc::mbar_arrive(&empty[s]);
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
}

// ---- pass 2: sampled rows of WHT over the next B2 bits, times the chunk sign --
template <int B2>
__global__ void __launch_bounds__(NTHREADS, 1)
    srht_p2_tma_kernel(const __grid_constant__ CUtensorMap mapT, int64_t d, int B1, int64_t chunk, int cbits,
                       const int64_t* __restrict__ sample, const uint32_t* __restrict__ order,
                       const uint32_t* __restrict__ qstart, double* __restrict__ SX, int first, double final_div) {
  constexpr int R = 1 << B2;
  constexpr int NA = R < 16 ? R : 16;
  constexpr int NB = R / NA;
  constexpr int BOX_BYTES = R * COLS * 4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cblocks = static_cast<int>((d + COLS - 1) / COLS);
  const int64_t nres = int64_t{1} << B1;
  const int64_t nitems = nres * cblocks;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapT) : "memory");
  }
  __syncthreads();
  if (warp == CWARPS) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < nitems; t += gridDim.x) {
        const int64_t q1 = t / cblocks, cb = t - q1 * cblocks;
        if (qstart[q1] == qstart[q1 + 1]) continue;  // no sampled row has this residue
        const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
        tc::mbar_wait(&empty[s], ph ^ 1u);
        tc::mbar_expect_tx(&full[s], BOX_BYTES);
        tma_load_3d(&mapT, &full[s], smem + s * TILE_BYTES, static_cast<int>(cb * COLS), static_cast<int>(q1), 0);
        ++it;
      }
    }
    return;
  }
  const int grp = warp >> 2, tid = threadIdx.x & 127;
  const int q = tid & 7, rg = tid >> 3;
  uint32_t it = 0;  // index of the non-empty item among this CTA's items; group grp takes it % GROUPS == grp
  for (int64_t t = blockIdx.x; t < nitems; t += gridDim.x) {
    const int64_t q1 = t / cblocks, cb = t - q1 * cblocks;
    const uint32_t e0 = qstart[q1], e1 = qstart[q1 + 1];
    if (e0 == e1) continue;
    const uint32_t mine = it++;
    if (mine % GROUPS != static_cast<uint32_t>(grp)) continue;
    const uint32_t s = mine % STAGES, ph = (mine / STAGES) & 1u;
    tc::mbar_wait(&full[s], ph);
    float* tile = reinterpret_cast<float*>(smem + s * TILE_BYTES);
    float v[NA][4];
    if (rg < R / NA) {
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        const float4 x = *reinterpret_cast<const float4*>(tile + (rg * NA + j) * COLS + q * 4);
        v[j][0] = x.x;
        v[j][1] = x.y;
        v[j][2] = x.z;
        v[j][3] = x.w;
      }
      wht_rows<NA>(v);  // index bits 8 .. 8+log2(NA)-1
#pragma unroll
      for (int j = 0; j < NA; ++j)
        *reinterpret_cast<float4*>(tile + (rg * NA + j) * COLS + q * 4) =
            make_float4(v[j][0], v[j][1], v[j][2], v[j][3]);
    }
    bar_group(grp);
    if constexpr (NB > 1) {
      float u[NB][4];
      if (rg < NA) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const float4 x = *reinterpret_cast<const float4*>(tile + (rg + NA * j) * COLS + q * 4);
          u[j][0] = x.x;
          u[j][1] = x.y;
          u[j][2] = x.z;
          u[j][3] = x.w;
        }
        wht_rows<NB>(u);  // the remaining bits
#pragma unroll
        for (int j = 0; j < NB; ++j)
          *reinterpret_cast<float4*>(tile + (rg + NA * j) * COLS + q * 4) =
              make_float4(u[j][0], u[j][1], u[j][2], u[j][3]);
      }
      bar_group(grp);
    }
    // scatter: SX[t] (+)= (-1)^popc(p_hi & chunk) * row q2 of the tile; 4 rows x 32 columns per sweep
    const int c = tid & 31;
    const int64_t col = cb * COLS + c;
    for (uint32_t e = e0 + (tid >> 5); e < e1; e += 4) {
      const uint32_t tt = order[e];
      const uint64_t p = static_cast<uint64_t>(sample[tt]);
      const int q2 = static_cast<int>((p >> B1) & static_cast<uint64_t>(R - 1));
      const bool neg = __popcll((p >> cbits) & static_cast<uint64_t>(chunk)) & 1;
      if (col < d) {
        double val = static_cast<double>(tile[q2 * COLS + c]);
        if (neg) val = -val;
        double* dst = SX + static_cast<int64_t>(tt) * d + col;
        double acc = first ? val : *dst + val;
        if (final_div != 0.0) acc = acc / final_div;
        *dst = acc;
      }
    }
    bar_group(grp);
    if (tid == 0) tc::mbar_arrive(&empty[s]);
  }
}

}  // namespace srht_tma

// Runs pass 1 + pass 2 of one chunk with the TMA kernels; false if the shape
// is not covered (caller keeps the one-shot kernels).
// Opt-in (LVSK_SRHT_TMA=1): measured on C3 (2^21 x 256) pass 1 23 us vs 25 us
// one-shot per 64 MB chunk, but pass 2 35 us vs 26 us — the 3-D residue box is
// 256 separate 128-byte rows, which the TMA engine serves slower than the
// one-shot kernel's direct L2 loads; the default stays the one-shot pair.
bool srht_tma_ok(const float* X, int64_t d, int64_t ldx, int B1) {
  if (getenv("LVSK_SRHT_TMA") == nullptr) return false;
  return B1 == 8 && d % 4 == 0 && ldx % 4 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0;
}

int32_t srht_tma_chunk(const float* X, int64_t n, int64_t d, int64_t ldx, int B1, int B2, int64_t chunk, int cbits,
                       const int8_t* signs, float* T1, const int64_t* sample, const uint32_t* order,
                       const uint32_t* qstart, double* SX, int first, double final_div, int32_t* flags,
                       cudaStream_t st) {
  using namespace srht_tma;
  const int64_t chunk_rows = int64_t{1} << (B1 + B2);
  CUtensorMap mx, mt;
  // X: [rows][d] (rows past n read as zero: the reference's zero padding)
  if (!tc::make_map(&mx, X, d, n, ldx * 4, COLS, ROWS, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    CU_TENSOR_MAP_SWIZZLE_NONE)) {
    set_error("cuTensorMapEncodeTiled failed (SRHT X)");
    return LVSK_ERR_CUDA;
  }
  {  // T1 as [i2][q1][d]: box {32 columns, 1 residue, 2^B2 rows}
    tc::EncodeFn enc = tc::encode_fn();
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(int64_t{1} << B1),
                          static_cast<cuuint64_t>(int64_t{1} << B2)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(d * 4), static_cast<cuuint64_t>((int64_t{1} << B1) * d * 4)};
    cuuint32_t box[3] = {COLS, 1, static_cast<cuuint32_t>(1 << B2)};
    cuuint32_t es[3] = {1, 1, 1};
    if (!enc || enc(&mt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, T1, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (SRHT T1)");
      return LVSK_ERR_CUDA;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(srht_p1_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
#define LVSK_P2A(BB) \
  cudaFuncSetAttribute(srht_p2_tma_kernel<BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    LVSK_P2A(1) LVSK_P2A(2) LVSK_P2A(3) LVSK_P2A(4) LVSK_P2A(5) LVSK_P2A(6) LVSK_P2A(7) LVSK_P2A(8)
#undef LVSK_P2A
    attr = true;
  }
  const int grid = num_sms();
  srht_p1_tma_kernel<<<grid, NTHREADS, SMEM_BYTES, st>>>(mx, chunk * chunk_rows, chunk_rows, d, signs, T1, flags);
  switch (B2) {
#define LVSK_P2(BB)                                                                                          \
  case BB:                                                                                                   \
    srht_p2_tma_kernel<BB><<<grid, NTHREADS, SMEM_BYTES, st>>>(mt, d, B1, chunk, cbits, sample, order, qstart, \
                                                               SX, first, final_div);                      \
    break;
    LVSK_P2(1) LVSK_P2(2) LVSK_P2(3) LVSK_P2(4) LVSK_P2(5) LVSK_P2(6) LVSK_P2(7) LVSK_P2(8)
#undef LVSK_P2
    default:
      set_error("SRHT TMA path needs 1 <= B2 <= 8 (got %d)", B2);
      return LVSK_ERR_CONFIGURATION;
  }
  LVSK_CHECK_LAUNCH("srht tma passes");
  return LVSK_OK;
}

}  // namespace lvsk
