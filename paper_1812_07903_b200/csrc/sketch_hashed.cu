// K1 — CountSketch / OSNAP on dense rows, as an owner-computes gather.
//
// Reference: SketchState._update_hashed -> _scatter_add -> _two_sum
// (pkg/src/levsketch/sketch.py:260-266, 173-191, 166-170), driven by
// consume_rows (sketch.py:289-312).
//
// B200 design: instead of scattering rows into buckets (atomics, order-
// dependent), the row -> bucket map (pure integer hash of the GLOBAL row
// index) is inverted with a stable radix sort, and one warp owns one
// (bucket, 32*VEC-column chunk).  The warp walks its bucket's rows in
// ascending global index and applies each contribution as a TwoSum into
// float64 (hi, lo) registers — exactly the reference's per-bucket operation
// sequence — so SX is bit-identical to the reference, with no atomics.  X is
// read once per block j (s times for OSNAP), in 512-byte warp-contiguous
// row segments; the accumulator never round-trips HBM.
#include <cstdlib>

#include <cstdio>

#include "radix_sort.cuh"

namespace lvsk {

constexpr int KEYGEN_MAX_BLOCKS = 64;

struct KeygenBlocks {
  uint64_t a[KEYGEN_MAX_BLOCKS];
  uint64_t b[KEYGEN_MAX_BLOCKS];
  uint64_t key[KEYGEN_MAX_BLOCKS];
  uint32_t offset[KEYGEN_MAX_BLOCKS];
  uint32_t size[KEYGEN_MAX_BLOCKS];
};

// keys[j*n + r] = global bucket of row r in block j; vals = (r << 1) | negative
__global__ void hashed_keygen_kernel(int64_t n, uint64_t row0, int j0, int nb, KeygenBlocks P,
                                     uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t total = n * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int jj = static_cast<int>(t / n);
    const int64_t r = t - static_cast<int64_t>(jj) * n;
    const uint64_t g = row0 + static_cast<uint64_t>(r);
    const uint32_t bk = P.offset[jj] + bucket_hash(g, P.a[jj], P.b[jj], P.size[jj]);
    const bool neg = sign_negative(g, P.key[jj]);
    const int64_t o = static_cast<int64_t>(j0 + jj) * n + r;
    keys[o] = bk;
    vals[o] = (static_cast<uint32_t>(r) << 1) | (neg ? 1u : 0u);
  }
}

template <typename T, int VEC>
struct VecLoad;
template <>
struct VecLoad<float, 4> {
  using V = float4;
  __device__ static void load(const float* p, float (&o)[4]) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  __device__ static void load_smem(const float* p, float (&o)[4]) {
    float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
};
template <>
struct VecLoad<double, 2> {
  __device__ static void load(const double* p, double (&o)[2]) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = v.x; o[1] = v.y;
  }
  __device__ static void load_smem(const double* p, double (&o)[2]) {
    double2 v = *reinterpret_cast<const double2*>(p);
    o[0] = v.x; o[1] = v.y;
  }
};
template <>
struct VecLoad<__nv_bfloat16, 8> {
  __device__ static void load(const __nv_bfloat16* p, __nv_bfloat16 (&o)[8]) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = h[i];
  }
  __device__ static void load_smem(const __nv_bfloat16* p, __nv_bfloat16 (&o)[8]) {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = h[i];
  }
};
template <typename T>
struct VecLoad<T, 1> {
  __device__ static void load(const T* p, T (&o)[1]) { o[0] = p[0]; }
};

constexpr int GATHER_UNROLL = 8;  // rows in flight per lane (memory-level parallelism)

template <typename T, int VEC>
__global__ void __launch_bounds__(256, 3) hashed_gather_kernel(
    const T* __restrict__ X, int64_t ldx, int64_t d, int nchunks, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ start, int64_t k, double scale, const double* hi_in, const double* lo_in,
    double* hi_out, double* lo_out, int32_t* flags) {
  const int64_t unit = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (unit >= k * nchunks) return;  // warp-uniform
  const int64_t b = unit / nchunks;
  const int64_t col0 = (unit - b * nchunks) * (32 * VEC) + lane * VEC;
  const bool active = col0 < d;
  double h[VEC], l[VEC];
  const int64_t so = b * d + col0;
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    h[v] = (hi_in != nullptr && active && col0 + v < d) ? hi_in[so + v] : 0.0;  // NULL state: zeros
    l[v] = (lo_in != nullptr && active && col0 + v < d) ? lo_in[so + v] : 0.0;
  }
  const uint32_t p0 = start[b], p1 = start[b + 1];
  bool bad = false;
  for (uint32_t base = p0; base < p1; base += 32) {
    const uint32_t cnt = min(32u, p1 - base);
    const uint32_t mine = lane < cnt ? vals[base + lane] : 0u;
    for (uint32_t t = 0; t < cnt; t += GATHER_UNROLL) {
      T xs[GATHER_UNROLL][VEC];
#pragma unroll
      for (int u = 0; u < GATHER_UNROLL; ++u) {
        const uint32_t vv = __shfl_sync(0xFFFFFFFFu, mine, (t + u) & 31);
        if (t + u < cnt && active) VecLoad<T, VEC>::load(X + static_cast<int64_t>(vv >> 1) * ldx + col0, xs[u]);
      }
#pragma unroll
      for (int u = 0; u < GATHER_UNROLL; ++u) {
        const uint32_t vv = __shfl_sync(0xFFFFFFFFu, mine, (t + u) & 31);
        if (t + u < cnt && active) {
          const double sg = (vv & 1u) ? -scale : scale;  // (sign * scale), exact
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double xv = to_f64<T>(xs[u][v]);
            bad |= !isfinite(xv);
            double s, e;
            two_sum(h[v], __dmul_rn(sg, xv), s, e);
            h[v] = s;
            l[v] = __dadd_rn(l[v], e);
          }
        }
      }
    }
  }
  if (active) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      if (col0 + v < d) {
        if (lo_out != nullptr) {
          hi_out[so + v] = h[v];
          lo_out[so + v] = l[v];
        } else {  // the folded sketch hi + lo (lvsk_fold_compensated's value)
          hi_out[so + v] = __dadd_rn(h[v], l[v]);
        }
      }
    }
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------
// Bulk-copy gather (default when rows are 16-byte aligned): one CTA owns one
// (bucket, 2 KB column group).  A producer warp streams the bucket's row
// segments into a 6-slot x 2-row shared-memory ring with cp.async.bulk (TMA 1-D,
// mbarrier complete_tx), so 24 KB per CTA (~190 KB per SM) are in flight;
// two consumer warps apply the rows in ascending index order, TwoSum into
// float64 (hi, lo) registers, exactly as the reference does per bucket.
constexpr int BULK_RPS = 2;     // rows per ring slot (one mbarrier round trip per pair of rows)
// 6 slots x 2 rows x 2 KB = 24 KB ring and <= 78 registers (launch bound of 8
// CTAs/SM): 8 CTAs per SM, 0.452 -> 0.426 ms at C2 vs 8 slots / 88 registers
constexpr int BULK_SLOTS = 6;
constexpr int BULK_SEG = 2048;  // bytes per row segment
// each consumer lane owns 32 B of the segment (8 fp32 / 4 fp64 / 16 bf16
// values = independent TwoSum chains per lane; 16 B and 64 B measured slower)
template <typename T>
constexpr int bulk_lane_bytes() { return 32; }
template <typename T>
constexpr int bulk_consumers() { return BULK_SEG / (32 * bulk_lane_bytes<T>()); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni BW_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}

// x with its sign flipped when neg, on the raw bits (exact; no fp64 op)
template <typename T>
__device__ __forceinline__ T flip_sign(T x, bool neg);
template <>
__device__ __forceinline__ float flip_sign<float>(float x, bool neg) {
  return __uint_as_float(__float_as_uint(x) ^ (static_cast<uint32_t>(neg) << 31));
}
template <>
__device__ __forceinline__ double flip_sign<double>(double x, bool neg) {
  return __longlong_as_double(__double_as_longlong(x) ^ (static_cast<long long>(neg) << 63));
}
template <>
__device__ __forceinline__ __nv_bfloat16 flip_sign<__nv_bfloat16>(__nv_bfloat16 x, bool neg) {
  return __ushort_as_bfloat16(__bfloat16_as_ushort(x) ^ static_cast<unsigned short>(neg << 15));
}

// contribution (sign * scale) * x as float64; UNIT: scale == 1 -> exact sign flip
template <typename T, bool UNIT>
__device__ __forceinline__ double contrib(T x, bool neg, double scale) {
  if constexpr (UNIT) {
    return to_f64<T>(flip_sign<T>(x, neg));
  } else {
    return __dmul_rn(neg ? -scale : scale, to_f64<T>(x));
  }
}

template <typename T, bool UNIT>
__global__ void __launch_bounds__(32 * (bulk_consumers<T>() + 1), 8) hashed_gather_bulk_kernel(
    const T* __restrict__ X, int64_t ldx, int64_t d, int ngroups, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ start, int64_t k, double scale, const double* hi_in, const double* lo_in,
    double* hi_out, double* lo_out, int32_t* flags) {
  constexpr int BULK_CONSUMERS = bulk_consumers<T>();
  constexpr int VEC = bulk_lane_bytes<T>() / static_cast<int>(sizeof(T));
  constexpr int NQ = bulk_lane_bytes<T>() / 16;  // 16-byte shared loads per lane and row
  __shared__ alignas(128) uint8_t ring[BULK_SLOTS][BULK_RPS][BULK_SEG];
  __shared__ uint64_t full[BULK_SLOTS], empty[BULK_SLOTS];
  __shared__ uint32_t slot_neg[BULK_SLOTS];
  const int64_t b = blockIdx.x / ngroups;
  const int g = blockIdx.x - static_cast<int>(b * ngroups);
  constexpr int SEG_ELEMS = BULK_SEG / static_cast<int>(sizeof(T));
  const int64_t c0 = static_cast<int64_t>(g) * SEG_ELEMS;
  const int64_t cols = d - c0 < SEG_ELEMS ? d - c0 : SEG_ELEMS;
  const uint32_t seg_bytes = static_cast<uint32_t>(cols * sizeof(T));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < BULK_SLOTS; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], BULK_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t p0 = start[b], p1 = start[b + 1];
  const uint32_t cnt = p1 - p0;
  if (warp == BULK_CONSUMERS) {  // producer: one lane, one bulk copy per row; the row's sign goes to the slot
    if (lane == 0) {
      for (uint32_t q = 0; q * BULK_RPS < cnt; ++q) {
        const uint32_t s = q % BULK_SLOTS, ph = (q / BULK_SLOTS) & 1u;
        const uint32_t nr = cnt - q * BULK_RPS < BULK_RPS ? cnt - q * BULK_RPS : BULK_RPS;
        uint32_t v[BULK_RPS];
        uint32_t negs = 0;
#pragma unroll
        for (int r = 0; r < BULK_RPS; ++r) {
          v[r] = r < static_cast<int>(nr) ? vals[p0 + q * BULK_RPS + r] : 0u;
          negs |= (v[r] & 1u) << r;
        }
        bar_wait(&empty[s], ph ^ 1u);
        slot_neg[s] = negs;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[s])),
                     "r"(seg_bytes * nr)
                     : "memory");
#pragma unroll
        for (int r = 0; r < BULK_RPS; ++r) {
          if (r < static_cast<int>(nr)) {
            const T* src = X + static_cast<int64_t>(v[r] >> 1) * ldx + c0;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(ring[s][r])),
                "l"(src), "r"(seg_bytes), "r"(smem_addr(&full[s]))
                : "memory");
          }
        }
      }
    }
    return;
  }
  const int64_t col = static_cast<int64_t>(warp * 32 + lane) * VEC;  // within the segment
  const bool active = col < cols;  // cols is a multiple of 16 B / sizeof(T); VEC spans 32 B
  const int nv = active ? (cols - col >= VEC ? VEC : static_cast<int>(cols - col)) : 0;
  double h[VEC], l[VEC];
  const int64_t so = b * d + c0 + col;
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    h[v] = (hi_in != nullptr && v < nv) ? hi_in[so + v] : 0.0;  // NULL state: zeros
    l[v] = (lo_in != nullptr && v < nv) ? lo_in[so + v] : 0.0;
  }
  bool bad = false;
  auto apply_row = [&](const uint8_t* seg, bool neg) {
    if (nv) {
      T xs[VEC];
      const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(seg) + col);
      uint4 w[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q)  // nv is a multiple of 16 B
        w[q] = q * (16 / static_cast<int>(sizeof(T))) < nv ? src[q] : make_uint4(0u, 0u, 0u, 0u);
      const T* wv = reinterpret_cast<const T*>(w);
#pragma unroll
      for (int v = 0; v < VEC; ++v) xs[v] = wv[v];
      if constexpr (UNIT) {
        // the row's sign is warp-uniform: pick TwoSum(h, x) or TwoSum(h, -x)
        if (neg) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double cval = to_f64<T>(xs[v]);
            if constexpr (sizeof(T) == 8) bad |= !isfinite(cval);
            double sum, e;
            two_sum_neg(h[v], cval, sum, e);
            h[v] = sum;
            l[v] = __dadd_rn(l[v], e);
          }
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double cval = to_f64<T>(xs[v]);
            if constexpr (sizeof(T) == 8) bad |= !isfinite(cval);
            double sum, e;
            two_sum(h[v], cval, sum, e);
            h[v] = sum;
            l[v] = __dadd_rn(l[v], e);
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double cval = contrib<T, UNIT>(xs[v], neg, scale);
          if constexpr (sizeof(T) == 8) bad |= !isfinite(cval);
          double sum, e;
          two_sum(h[v], cval, sum, e);
          h[v] = sum;
          l[v] = __dadd_rn(l[v], e);
        }
      }
    }
  };
  for (uint32_t q = 0; q * BULK_RPS < cnt; ++q) {
    const uint32_t s = q % BULK_SLOTS, ph = (q / BULK_SLOTS) & 1u;
    bar_wait(&full[s], ph);
    const uint32_t negs = slot_neg[s];  // written by the producer before its (release) arrive
    apply_row(ring[s][0], (negs & 1u) != 0u);
    if (q * BULK_RPS + 1 < cnt) apply_row(ring[s][1], (negs & 2u) != 0u);
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[s]);
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    if (v < nv) {
      if (lo_out != nullptr) {
        hi_out[so + v] = h[v];
        lo_out[so + v] = l[v];
      } else {  // the folded sketch hi + lo (lvsk_fold_compensated's value)
        hi_out[so + v] = __dadd_rn(h[v], l[v]);
      }
      // fp32 / bf16 inputs cannot overflow a float64 sum: a non-finite state
      // means a non-finite input (checked once here instead of per element)
      if constexpr (sizeof(T) < 8) bad |= !(isfinite(h[v]) && isfinite(l[v]));
    }
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
}

// copies hi/lo rows of buckets that no row touched when in != out
__global__ void copy_f64_kernel(const double* __restrict__ a, double* __restrict__ b, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

__global__ void merge_kernel(const double* hi1, const double* lo1, const double* hi2, const double* lo2,
                             double* hi_out, double* lo_out, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s, e;
    two_sum(hi1[i], hi2[i], s, e);
    const double l = __dadd_rn(__dadd_rn(lo1[i], lo2[i]), e);  // (lo1 + lo2) + e, sketch.py:355
    hi_out[i] = s;
    lo_out[i] = l;
  }
}

__global__ void hash_rows_kernel(const uint64_t* __restrict__ idx, int64_t n, int nb, KeygenBlocks P, int j0,
                                 int64_t* __restrict__ buckets, double* __restrict__ signs) {
  const int64_t total = n * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int jj = static_cast<int>(t / n);
    const int64_t r = t - static_cast<int64_t>(jj) * n;
    const uint64_t g = idx[r];
    const int64_t o = static_cast<int64_t>(j0 + jj) * n + r;
    buckets[o] = static_cast<int64_t>(P.offset[jj]) + bucket_hash(g, P.a[jj], P.b[jj], P.size[jj]);
    signs[o] = sign_negative(g, P.key[jj]) ? -1.0 : 1.0;
  }
}

static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(num_sms()) * 32;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

static int ceil_log2(int64_t v) {
  int b = 0;
  while ((int64_t{1} << b) < v) ++b;
  return b;
}

static void fill_blocks(KeygenBlocks& P, const lvsk_hash_block* blocks, int j0, int nb) {
  for (int jj = 0; jj < nb; ++jj) {
    const lvsk_hash_block& B = blocks[j0 + jj];
    P.a[jj] = B.a;
    P.b[jj] = B.b;
    P.key[jj] = B.sign_key;
    P.offset[jj] = static_cast<uint32_t>(B.offset);
    P.size[jj] = static_cast<uint32_t>(B.size);
  }
}

template <typename T, int VEC_UNUSED>
static void launch_gather_bulk(const void* X, int64_t ldx, int64_t d, const uint32_t* vals, const uint32_t* start,
                               int64_t k, double scale, const double* hi_in, const double* lo_in, double* hi_out,
                               double* lo_out, int32_t* flags, cudaStream_t st) {
  const int ngroups = static_cast<int>((d * static_cast<int64_t>(sizeof(T)) + BULK_SEG - 1) / BULK_SEG);
  const unsigned grid = static_cast<unsigned>(k * ngroups);
  if (scale == 1.0)
    hashed_gather_bulk_kernel<T, true><<<grid, 32 * (bulk_consumers<T>() + 1), 0, st>>>(
        static_cast<const T*>(X), ldx, d, ngroups, vals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags);
  else
    hashed_gather_bulk_kernel<T, false><<<grid, 32 * (bulk_consumers<T>() + 1), 0, st>>>(
        static_cast<const T*>(X), ldx, d, ngroups, vals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags);
}

template <typename T, int VEC>
static void launch_gather(const void* X, int64_t ldx, int64_t d, const uint32_t* vals, const uint32_t* start,
                          int64_t k, double scale, const double* hi_in, const double* lo_in, double* hi_out,
                          double* lo_out, int32_t* flags, cudaStream_t st) {
  const int nchunks = static_cast<int>((d + 32 * VEC - 1) / (32 * VEC));
  const int64_t threads = k * nchunks * 32;
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  hashed_gather_kernel<T, VEC><<<grid, 256, 0, st>>>(static_cast<const T*>(X), ldx, d, nchunks, vals, start, k,
                                                     scale, hi_in, lo_in, hi_out, lo_out, flags);
}

// ---------------------------------------------------------------------------
// Bucket grouping in ONE cooperative kernel (k <= GC_MAX_K): a stable counting
// sort of the (row, block) items by bucket.  CTA c owns a contiguous item range
// and each of its 8 warps a contiguous sub-range, so stable order = (CTA, warp,
// 32-item step, lane):
//   1. hash every item once (bucket, value kept in shared memory when the
//      chunk fits), per-warp bucket counts, CTA histogram -> ghist[b][cta]
//   2. grid barrier; CTA c turns the rows of its ~k/G buckets into prefix
//      counts over the CTAs (one warp scan per bucket) and bucket totals
//   3. grid barrier; every CTA scans the totals (bucket starts, written by
//      CTA 0 as `start`), adds its prefix and its warps' prefixes, and each
//      warp writes its items' values in order (match_any ranks equal buckets
//      within a step; the warp's own counter orders the steps)
// Replaces keygen + two radix passes + bucket bounds (7 launches).
constexpr int GC_THREADS = 256;
constexpr int GC_WARPS = GC_THREADS / 32;
constexpr int64_t GC_MAX_K = 4096;
constexpr int GC_MAX_G = 256;
constexpr int GC_PER = static_cast<int>(GC_MAX_K / GC_THREADS);  // buckets per thread in the base scan
constexpr int GC_CAP = 7168;                                       // items cached per CTA
constexpr size_t GC_SMEM = sizeof(uint32_t) * ((GC_WARPS + 2) * GC_MAX_K + 2 * GC_CAP);

__device__ __forceinline__ void gc_barrier(unsigned int* count, unsigned int& nbar) {
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

// item t = (block jj, row r) with t = jj * n + r; callers walk t in steps of
// 32 and carry (jj, r) along instead of a 64-bit division per item
__device__ __forceinline__ void gc_split(int64_t t, int64_t n, int& jj, int64_t& r) {
  jj = static_cast<int>(t / n);
  r = t - static_cast<int64_t>(jj) * n;
}
__device__ __forceinline__ void gc_step(int64_t n, int& jj, int64_t& r) {
  r += 32;
  while (r >= n) {  // (n >= 1; at most one wrap per step unless n < 32)
    r -= n;
    ++jj;
  }
}
__device__ __forceinline__ void gc_item(int jj, int64_t r, uint64_t row0, const KeygenBlocks& P, uint32_t& bk,
                                        uint32_t& val) {
  const uint64_t g = row0 + static_cast<uint64_t>(r);
  bk = P.offset[jj] + bucket_hash(g, P.a[jj], P.b[jj], P.size[jj]);
  val = (static_cast<uint32_t>(r) << 1) | (sign_negative(g, P.key[jj]) ? 1u : 0u);
}

__global__ void __launch_bounds__(GC_THREADS, 1) group_coop_kernel(int64_t n, int nb, uint64_t row0, KeygenBlocks P,
                                                                   int64_t k, uint32_t* __restrict__ svals,
                                                                   uint32_t* __restrict__ start, uint32_t* ghist,
                                                                   uint32_t* gtot, uint32_t* pre, unsigned int* bar,
                                                                   unsigned long long* trace) {
  auto stamp = [&](int slot) {
    if (trace != nullptr && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[slot + (blockIdx.x == 0 ? 0 : 8)] = t;
    }
  };
  stamp(0);
  extern __shared__ uint32_t gc_smem[];
  uint32_t* hw = gc_smem;                     // [GC_WARPS][k] per-warp counts, then per-warp write offsets
  uint32_t* base = gc_smem + GC_WARPS * k;    // [k]
  uint32_t* prow = base + k;                  // [k] this CTA's prefix row
  uint32_t* items = prow + k;                 // [GC_CAP][2] (bucket, value) in item order
  __shared__ uint32_t sh[GC_WARPS];
  unsigned int nbar = 0;
  const int G = gridDim.x, cta = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = n * nb;
  const int64_t c0 = N * cta / G, c1 = N * (cta + 1) / G;
  const bool cached = c1 - c0 <= GC_CAP;
  const int64_t w0 = c0 + (c1 - c0) * warp / GC_WARPS, w1 = c0 + (c1 - c0) * (warp + 1) / GC_WARPS;
  for (int64_t i = threadIdx.x; i < GC_WARPS * k; i += GC_THREADS) hw[i] = 0u;
  __syncthreads();
  // 1. hash, per-warp counts
  int ij;
  int64_t ir;
  gc_split(w0 + lane, n, ij, ir);
  for (int64_t t = w0 + lane; t < w1; t += 32, gc_step(n, ij, ir)) {
    uint32_t bk, val;
    gc_item(ij, ir, row0, P, bk, val);
    if (cached) {
      items[2 * (t - c0)] = bk;
      items[2 * (t - c0) + 1] = val;
    }
    atomicAdd(&hw[warp * k + bk], 1u);
  }
  __syncthreads();
  for (int64_t b = threadIdx.x; b < k; b += GC_THREADS) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < GC_WARPS; ++w) {
      const uint32_t c = hw[w * k + b];
      hw[w * k + b] = run;  // prefix over the CTA's earlier warps
      run += c;
    }
    ghist[b * G + cta] = run;  // bucket-major: a bucket's CTA counts are contiguous
  }
  stamp(1);
  gc_barrier(bar, nbar);
  stamp(2);
  // 2. prefix over CTAs for my buckets: one warp per bucket, all loads up front
  {
    const int64_t b0 = k * cta / G, b1 = k * (cta + 1) / G;
    for (int64_t b = b0 + warp; b < b1; b += GC_WARPS) {
      const uint32_t* row = ghist + b * G;
      uint32_t v[GC_MAX_G / 32];
#pragma unroll
      for (int q = 0; q < GC_MAX_G / 32; ++q) v[q] = q * 32 + lane < G ? __ldcg(row + q * 32 + lane) : 0u;
      uint32_t carry = 0;
#pragma unroll
      for (int q = 0; q < GC_MAX_G / 32; ++q) {
        if (q * 32 >= G) break;
        uint32_t x = v[q];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
          if (lane >= off) x += y;
        }
        if (q * 32 + lane < G) pre[static_cast<int64_t>(q * 32 + lane) * k + b] = carry + x - v[q];
        carry += __shfl_sync(0xFFFFFFFFu, x, 31);
      }
      if (lane == 0) gtot[b] = carry;
    }
  }
  stamp(3);
  gc_barrier(bar, nbar);
  stamp(4);
  // 3. bucket starts: totals and this CTA's prefix row staged through shared
  // memory with coalesced loads, then thread t scans buckets [t*PER, (t+1)*PER)
  {
    uint32_t tv[GC_PER], pv[GC_PER];  // all 2 x GC_PER loads in flight before any store
#pragma unroll
    for (int q = 0; q < GC_PER; ++q) {
      const int64_t b = threadIdx.x + static_cast<int64_t>(q) * GC_THREADS;
      tv[q] = b < k ? __ldcg(gtot + b) : 0u;
      pv[q] = b < k ? __ldcg(pre + static_cast<int64_t>(cta) * k + b) : 0u;
    }
#pragma unroll
    for (int q = 0; q < GC_PER; ++q) {
      const int64_t b = threadIdx.x + static_cast<int64_t>(q) * GC_THREADS;
      if (b < k) {
        base[b] = tv[q];
        prow[b] = pv[q];
      }
    }
  }
  __syncthreads();
  {
    const int64_t b0 = static_cast<int64_t>(threadIdx.x) * GC_PER;
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < GC_PER; ++q) run += b0 + q < k ? base[b0 + q] : 0u;
    uint32_t x = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    uint32_t acc = x - run;
    for (int w = 0; w < warp; ++w) acc += sh[w];
    uint32_t tv[GC_PER];
#pragma unroll
    for (int q = 0; q < GC_PER; ++q) tv[q] = b0 + q < k ? base[b0 + q] : 0u;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GC_PER; ++q) {
      if (b0 + q < k) base[b0 + q] = acc;  // bucket start
      acc += tv[q];
    }
  }
  __syncthreads();
  for (int64_t b = threadIdx.x; b < k; b += GC_THREADS) {  // consecutive buckets per warp: no bank conflicts
    const uint32_t st0 = base[b];
    if (cta == 0) start[b] = st0;
    const uint32_t o = st0 + prow[b];
#pragma unroll
    for (int w = 0; w < GC_WARPS; ++w) hw[w * k + b] += o;
  }
  if (cta == 0 && threadIdx.x == 0) start[k] = static_cast<uint32_t>(N);
  __syncthreads();
  stamp(5);
  // 4. stable scatter of the values, warp by warp
  const uint32_t lt = lanemask_lt();
  uint32_t* my = hw + warp * k;
  gc_split(w0 + lane, n, ij, ir);
  for (int64_t t0 = w0; t0 < w1; t0 += 32, gc_step(n, ij, ir)) {
    const int64_t t = t0 + lane;
    const bool valid = t < w1;
    uint32_t bk = 0xFFFFFFFFu, val = 0u;
    if (valid) {
      if (cached) {
        bk = items[2 * (t - c0)];
        val = items[2 * (t - c0) + 1];
      } else {
        gc_item(ij, ir, row0, P, bk, val);
      }
    }
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, bk);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0u;
    if (valid && lane == leader) {
      old = my[bk];
      my[bk] = old + __popc(peers);
    }
    old = __shfl_sync(0xFFFFFFFFu, old, leader);
    if (valid) svals[old + __popc(peers & lt)] = val;
    __syncwarp();
  }
  __syncthreads();
  stamp(6);
}

static int gc_grid() {
  const int per = resident_ctas(reinterpret_cast<const void*>(group_coop_kernel), GC_THREADS, static_cast<int>(GC_SMEM));
  int g = per >= 1 ? num_sms() : 0;
  if (g > GC_MAX_G) g = GC_MAX_G;
  return g;
}

}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_hashed_workspace_bytes(int64_t n, int32_t s, int64_t k) {
  Measure m;
  const int64_t N = n * s;
  m.take<uint32_t>(N);  // keys
  m.take<uint32_t>(N);  // vals
  m.take<uint32_t>(N);  // sorted keys
  m.take<uint32_t>(N);  // sorted vals
  m.take<uint32_t>(k + 1);
  radix::measure<uint32_t>(m, N);
  if (k <= GC_MAX_K) {  // cooperative grouping: CTA histograms and prefixes, bucket totals, barrier
    m.take<uint32_t>(static_cast<size_t>(GC_MAX_G) * k);
    m.take<uint32_t>(static_cast<size_t>(GC_MAX_G) * k);
    m.take<uint32_t>(k);
    m.take<uint32_t>(4);
  }
  return m.off;
}

extern "C" int32_t lvsk_hashed_sketch(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx,
                                      uint64_t row0, const lvsk_hash_block* blocks, int32_t s, double scale,
                                      const double* hi_in, const double* lo_in, double* hi_out, double* lo_out,
                                      int64_t k, void* ws, size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(n >= 0 && d >= 1 && ldx >= d, LVSK_ERR_DIMENSION, "bad shape n=%lld d=%lld ldx=%lld",
               (long long)n, (long long)d, (long long)ldx);
  LVSK_REQUIRE(s >= 1 && k >= s, LVSK_ERR_CONFIGURATION, "need 1 <= s <= k (s=%d, k=%lld)", s, (long long)k);
  LVSK_REQUIRE(k < (int64_t{1} << 31), LVSK_ERR_CAPACITY, "k=%lld too large", (long long)k);
  LVSK_REQUIRE(n < (int64_t{1} << 31) && n * s < 0xFFFFFFFFll, LVSK_ERR_CAPACITY,
               "row block of %lld rows x s=%d too large for one call; split it", (long long)n, s);
  LVSK_REQUIRE(dtype == LVSK_F32 || dtype == LVSK_F64 || dtype == LVSK_BF16, LVSK_ERR_CONFIGURATION,
               "unknown dtype %d", dtype);
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    if (hi_in == nullptr || lo_in == nullptr) {
      cudaError_t e = cudaMemsetAsync(hi_out, 0, static_cast<size_t>(k * d) * sizeof(double), st);
      if (e == cudaSuccess) e = cudaMemsetAsync(lo_out, 0, static_cast<size_t>(k * d) * sizeof(double), st);
      if (e != cudaSuccess) return cuda_status(e, "hashed zero state");
      return LVSK_OK;
    }
    if (hi_in != hi_out) copy_f64_kernel<<<grid_for(k * d, 256), 256, 0, st>>>(hi_in, hi_out, k * d);
    if (lo_in != lo_out) copy_f64_kernel<<<grid_for(k * d, 256), 256, 0, st>>>(lo_in, lo_out, k * d);
    LVSK_CHECK_LAUNCH("hashed copy");
    return LVSK_OK;
  }
  const int64_t N = n * s;
  Carve c(ws, ws_bytes);
  uint32_t* keys = c.take<uint32_t>(N);
  uint32_t* vals = c.take<uint32_t>(N);
  uint32_t* skeys = c.take<uint32_t>(N);
  uint32_t* svals = c.take<uint32_t>(N);
  uint32_t* start = c.take<uint32_t>(k + 1);
  auto rb = radix::carve<uint32_t>(c, N);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);

  const int G = k <= GC_MAX_K && s <= KEYGEN_MAX_BLOCKS ? gc_grid() : 0;
  if (G >= 1 && getenv("LVSK_GROUP_RADIX") == nullptr) {
    uint32_t* ghist = c.take<uint32_t>(static_cast<size_t>(GC_MAX_G) * k);  // [k][G]
    uint32_t* pre = c.take<uint32_t>(static_cast<size_t>(GC_MAX_G) * k);    // [G][k]
    uint32_t* gtot = c.take<uint32_t>(k);
    uint32_t* bar = c.take<uint32_t>(4);
    LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
    cudaError_t e = cudaMemsetAsync(bar, 0, 4 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "group memset");
    KeygenBlocks P;
    fill_blocks(P, blocks, 0, s);
    int nb = s;
    unsigned int* barp = bar;
    static unsigned long long* trace = nullptr;
    const bool tracing = getenv("LVSK_GROUP_TRACE") != nullptr;
    if (tracing && trace == nullptr) cudaMalloc(&trace, 16 * sizeof(unsigned long long));
    unsigned long long* tr = tracing ? trace : nullptr;
    void* args[] = {(void*)&n, (void*)&nb, (void*)&row0, (void*)&P, (void*)&k, (void*)&svals, (void*)&start,
                    (void*)&ghist, (void*)&gtot, (void*)&pre, (void*)&barp, (void*)&tr};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(group_coop_kernel), dim3(G), dim3(GC_THREADS), args,
                                    static_cast<size_t>(sizeof(uint32_t) * ((GC_WARPS + 2) * k + 2 * GC_CAP)), st);
    if (e != cudaSuccess) return cuda_status(e, "group coop launch");
    if (tracing) {
      unsigned long long h[16];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
      for (int c = 0; c < 2; ++c) {
        const unsigned long long* q = h + 8 * c;
        fprintf(stderr, "group cta %s: count %.1f bar %.1f colscan %.1f bar %.1f bases %.1f scatter %.1f us\n",
                c ? "last" : "0", (q[1] - q[0]) / 1e3, (q[2] - q[1]) / 1e3, (q[3] - q[2]) / 1e3, (q[4] - q[3]) / 1e3,
                (q[5] - q[4]) / 1e3, (q[6] - q[5]) / 1e3);
      }
    }
  } else {
    for (int j0 = 0; j0 < s; j0 += KEYGEN_MAX_BLOCKS) {
      const int nb = s - j0 < KEYGEN_MAX_BLOCKS ? s - j0 : KEYGEN_MAX_BLOCKS;
      KeygenBlocks P;
      fill_blocks(P, blocks, j0, nb);
      hashed_keygen_kernel<<<grid_for(n * nb, 256), 256, 0, st>>>(n, row0, j0, nb, P, keys, vals);
    }
    LVSK_CHECK_LAUNCH("hashed keygen");
    int32_t rc = radix::sort_pairs<uint32_t, uint32_t>(keys, vals, N, ceil_log2(k), rb, skeys, svals, st);
    if (rc != LVSK_OK) return rc;
    radix::bucket_bounds_kernel<uint32_t><<<grid_for(N + 1, 256), 256, 0, st>>>(skeys, N, k, start);
    LVSK_CHECK_LAUNCH("bucket bounds");
  }

  const uintptr_t xa = reinterpret_cast<uintptr_t>(X);
  const bool bulk = getenv("LVSK_K1_REGS") == nullptr;  // register-path gather kept for A/B checks
  switch (dtype) {
    case LVSK_F32:
      if (bulk && xa % 16 == 0 && (ldx * 4) % 16 == 0 && d % 4 == 0)
        launch_gather_bulk<float, 4>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags, st);
      else if (xa % 16 == 0 && (ldx * 4) % 16 == 0 && d % 4 == 0)
        launch_gather<float, 4>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags, st);
      else
        launch_gather<float, 1>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags, st);
      break;
    case LVSK_F64:
      if (bulk && xa % 16 == 0 && (ldx * 8) % 16 == 0 && d % 2 == 0)
        launch_gather_bulk<double, 2>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags, st);
      else if (xa % 16 == 0 && (ldx * 8) % 16 == 0 && d % 2 == 0)
        launch_gather<double, 2>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags, st);
      else
        launch_gather<double, 1>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags, st);
      break;
    default:
      if (bulk && xa % 16 == 0 && (ldx * 2) % 16 == 0 && d % 8 == 0)
        launch_gather_bulk<__nv_bfloat16, 8>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags,
                                              st);
      else if (xa % 16 == 0 && (ldx * 2) % 16 == 0 && d % 8 == 0)
        launch_gather<__nv_bfloat16, 8>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags,
                                         st);
      else
        launch_gather<__nv_bfloat16, 1>(X, ldx, d, svals, start, k, scale, hi_in, lo_in, hi_out, lo_out, flags,
                                         st);
  }
  LVSK_CHECK_LAUNCH("hashed gather");
  return LVSK_OK;
}

extern "C" int32_t lvsk_hash_rows(const uint64_t* idx, int64_t n, const lvsk_hash_block* blocks, int32_t s,
                                  int64_t* buckets_out, double* signs_out, void* stream) {
  LVSK_REQUIRE(n >= 0 && s >= 1, LVSK_ERR_CONFIGURATION, "bad arguments");
  cudaStream_t st = as_stream(stream);
  for (int j0 = 0; j0 < s; j0 += KEYGEN_MAX_BLOCKS) {
    const int nb = s - j0 < KEYGEN_MAX_BLOCKS ? s - j0 : KEYGEN_MAX_BLOCKS;
    KeygenBlocks P;
    fill_blocks(P, blocks, j0, nb);
    if (n > 0) hash_rows_kernel<<<grid_for(n * nb, 256), 256, 0, st>>>(idx, n, nb, P, j0, buckets_out, signs_out);
  }
  LVSK_CHECK_LAUNCH("hash rows");
  return LVSK_OK;
}

extern "C" int32_t lvsk_merge_compensated(const double* hi1, const double* lo1, const double* hi2,
                                          const double* lo2, double* hi_out, double* lo_out, int64_t count,
                                          void* stream) {
  if (count <= 0) return LVSK_OK;
  merge_kernel<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(hi1, lo1, hi2, lo2, hi_out, lo_out, count);
  LVSK_CHECK_LAUNCH("merge");
  return LVSK_OK;
}

namespace lvsk {
__global__ void fold_kernel(const double* hi, const double* lo, double* out, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __dadd_rn(hi[i], lo[i]);
}
}  // namespace lvsk

extern "C" int32_t lvsk_fold_compensated(const double* hi, const double* lo, double* out, int64_t count,
                                         void* stream) {
  if (count <= 0) return LVSK_OK;
  fold_kernel<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(hi, lo, out, count);
  LVSK_CHECK_LAUNCH("fold");
  return LVSK_OK;
}
