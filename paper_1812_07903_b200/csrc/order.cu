// Ordering: scores_to_distribution + make_plan("dec"/"dec_swor") on device.
//
// Reference: order.py:51-63 (normalise with validation), order.py:84-90
// (dec = np.argsort(-p, kind="stable")), order.py:95-99 (dec_swor =
// np.argsort(Exp(1)/p, kind="stable")).  K7 is a stable LSD radix sort over
// an order-preserving uint64 image of the float64 keys (8 passes of 8 bits),
// values = indices, so ties keep ascending index exactly like numpy's stable
// sort.
#include "radix_sort.cuh"

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
  return m.off;
}

extern "C" int32_t lvsk_argsort_f64(const double* keys, int64_t n, int32_t descending, int64_t* idx_out, void* ws,
                                    size_t ws_bytes, void* stream) {
  LVSK_REQUIRE(n >= 0, LVSK_ERR_DIMENSION, "negative length");
  if (n == 0) return LVSK_OK;
  Carve c(ws, ws_bytes);
  uint64_t* k64 = c.take<uint64_t>(n);
  auto rb = radix::carve<uint64_t>(c, n);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  cudaStream_t st = as_stream(stream);
  argsort_keys_kernel<<<grid_cap(n), 256, 0, st>>>(keys, n, descending, k64);
  LVSK_CHECK_LAUNCH("argsort keys");
  return radix::sort_pairs<uint64_t, int64_t>(k64, nullptr, n, 64, rb, nullptr, idx_out, st);
}
