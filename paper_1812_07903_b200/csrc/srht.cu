// K3 — SRHT: SX = (H_m D X)[sample] / divisor, fused sign flip + WHT + row
// subsampling.  Reference: SketchState.data SRHT branch and fwht
// (pkg/src/levsketch/sketch.py:248-257, 364-385; signs/sample drawn on the
// host exactly as sketch.py:220-224).
//
// B200 design.  m = 2^L rows are split as  i = (i_hi, i2, i1)  with
// i1 = low B1 (<= 8) bits, i2 = next B2 (<= 8) bits, i_hi = top a bits.  One
// chunk = 2^(B1+B2) consecutive rows, sized so its fp32 intermediate stays
// L2-resident (<= 64 MB).  Per chunk:
//   pass 1: CTA = 2^B1 consecutive rows x 128 B of columns; rows are loaded
//           once from HBM (sign flip and zero padding fused into the load),
//           transformed over i1 in registers (bits 0-3) and through shared
//           memory (bits 4-7), written to the chunk buffer T1;
//   pass 2: CTA = one residue q1 of i1 x 128 B of columns; loads the 2^B2
//           rows q1 + 2^B1*i2 of T1 (L2 hits), transforms over i2, and for
//           every sampled row p with p_lo == (q2, q1) adds
//           (-1)^popcount(p_hi & chunk) * value into SX[t] (float64).
// The butterflies run low bit first like the reference, so float64 input
// reproduces the reference up to the reassociation of the top a bits.
#include <cstdlib>
#include <type_traits>

#include "radix_sort.cuh"

namespace lvsk {

constexpr int SRHT_THREADS = 128;
constexpr size_t SRHT_CHUNK_BYTES = size_t{64} << 20;

template <typename C>
struct SrhtCfg {
  static constexpr int W = 16 / sizeof(C);      // values per 16-byte vector
  static constexpr int DC = 128 / sizeof(C);    // columns per CTA (128 B)
  static constexpr int Q = DC / W;              // vectors per row segment (8)
  static constexpr int PAD = W;                 // one vector of padding per smem row
};

// in-register radix-2 WHT over N rows of W-wide vectors, low bit first
template <typename C, int N, int W>
__device__ __forceinline__ void reg_wht(C (&v)[N][W]) {
#pragma unroll
  for (int h = 1; h < N; h <<= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i & h) == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const C a = v[i][w], b = v[i + h][w];
          v[i][w] = a + b;
          v[i + h][w] = a - b;
        }
      }
    }
  }
}

__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_f4_hint(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_f4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// W consecutive values of row `row` starting at column `col` (zero past d / n)
template <typename T, typename C, bool VECTOR>
__device__ __forceinline__ void load_row_vec(const T* X, int64_t ldx, int64_t n, int64_t d, int64_t row, int64_t col,
                                             uint64_t pol, C (&out)[SrhtCfg<C>::W]) {
  constexpr int W = SrhtCfg<C>::W;
  if (row >= n) {
#pragma unroll
    for (int w = 0; w < W; ++w) out[w] = C(0);
    return;
  }
  const T* p = X + row * ldx + col;
  if constexpr (VECTOR && sizeof(T) == sizeof(C)) {
    if (col + W <= d) {
      if constexpr (sizeof(C) == 4) {
        float4 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(p), "l"(pol));
        out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
      } else {
        double2 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(v.x), "=d"(v.y)
                     : "l"(p), "l"(pol));
        out[0] = v.x; out[1] = v.y;
      }
      return;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) out[w] = (col + w < d) ? static_cast<C>(to_f64<T>(p[w])) : C(0);
}

// Pass 1: rows [chunk_row0 + blockIdx.x*2^B, +2^B) -> T1 (chunk-local rows),
// sign flip and zero padding fused into the load.
template <typename T, typename C, int B, bool VECTOR>
__global__ void __launch_bounds__(SRHT_THREADS) srht_pass1_kernel(const T* __restrict__ X, int64_t n, int64_t d,
                                                                  int64_t ldx, int64_t chunk_row0,
                                                                  const int8_t* __restrict__ signs,
                                                                  C* __restrict__ T1, int32_t* flags) {
  using G = SrhtCfg<C>;
  constexpr int W = G::W, Q = G::Q;
  constexpr int R = 1 << B;
  constexpr int BA = B < 4 ? B : 4;
  constexpr int NA = 1 << BA;
  constexpr int NB = 1 << (B - BA);
  __shared__ alignas(16) C S[R][G::DC + G::PAD];
  const int64_t col0 = static_cast<int64_t>(blockIdx.y) * G::DC;
  const int64_t lrow0 = static_cast<int64_t>(blockIdx.x) * R;  // chunk-local
  const uint64_t pol = evict_first_policy();
  const uint64_t pol_keep = evict_last_policy();  // T1 is re-read by pass 2 from L2
  bool bad = false;
  for (int g = threadIdx.x; g < (R / NA) * Q; g += SRHT_THREADS) {
    const int q = g % Q, rh = g / Q;
    const int64_t grow0 = chunk_row0 + lrow0 + rh * NA;
    C v[NA][W];
#pragma unroll
    for (int j = 0; j < NA; ++j) load_row_vec<T, C, VECTOR>(X, ldx, n, d, grow0 + j, col0 + q * W, pol, v[j]);
    if (signs) {
      int8_t sg[NA];
      if constexpr (NA == 16) {
        const int4 s16 = *reinterpret_cast<const int4*>(signs + grow0);
        const int8_t* sp = reinterpret_cast<const int8_t*>(&s16);
#pragma unroll
        for (int j = 0; j < NA; ++j) sg[j] = sp[j];
      } else {
#pragma unroll
        for (int j = 0; j < NA; ++j) sg[j] = signs[grow0 + j];
      }
#pragma unroll
      for (int j = 0; j < NA; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) v[j][w] = sg[j] < 0 ? -v[j][w] : v[j][w];
    }
#pragma unroll
    for (int j = 0; j < NA; ++j)
#pragma unroll
      for (int w = 0; w < W; ++w) bad |= !isfinite(static_cast<double>(v[j][w]));
    reg_wht<C, NA, W>(v);
#pragma unroll
    for (int j = 0; j < NA; ++j)
#pragma unroll
      for (int w = 0; w < W; ++w) S[rh * NA + j][q * W + w] = v[j][w];
  }
  __syncthreads();
  for (int g = threadIdx.x; g < NA * Q; g += SRHT_THREADS) {
    const int q = g % Q, rl = g / Q;
    C v[NB][W];
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int w = 0; w < W; ++w) v[j][w] = S[rl + NA * j][q * W + w];
    reg_wht<C, NB, W>(v);
    const int64_t col = col0 + q * W;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      C* dst = T1 + (lrow0 + rl + NA * j) * d + col;
      if (col + W <= d && d % W == 0) {
        if constexpr (sizeof(C) == 4) {
          st_f4_hint(reinterpret_cast<float*>(dst), make_float4(v[j][0], v[j][1], v[j][2], v[j][3]), pol_keep);
        } else {
          *reinterpret_cast<double2*>(dst) = make_double2(v[j][0], v[j][1]);
        }
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (col + w < d) dst[w] = v[j][w];
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
}

// Pass 2: residue q1 = blockIdx.x of the low B1 bits; WHT over the next B2
// bits; every sampled row with that residue gets (-1)^popc(p_hi & chunk) x
// its value added into SX (float64).
template <typename C, int B2>
__global__ void __launch_bounds__(SRHT_THREADS) srht_pass2_kernel(const C* __restrict__ T1, int64_t d, int B1,
                                                                  int64_t chunk, int cb,
                                                                  const int64_t* __restrict__ sample,
                                                                  const uint32_t* __restrict__ order,
                                                                  const uint32_t* __restrict__ qstart,
                                                                  double* __restrict__ SX, int first,
                                                                  double final_div) {
  using G = SrhtCfg<C>;
  constexpr int W = G::W, Q = G::Q;
  constexpr int R = 1 << B2;
  constexpr int BA = B2 < 4 ? B2 : 4;
  constexpr int NA = 1 << BA;
  constexpr int NB = 1 << (B2 - BA);
  __shared__ alignas(16) C S[R][G::DC + G::PAD];
  const int64_t q1 = blockIdx.x;
  const uint32_t e0 = qstart[q1], e1 = qstart[q1 + 1];
  if (e0 == e1) return;  // no sampled row has this residue (block-uniform)
  const int64_t col0 = static_cast<int64_t>(blockIdx.y) * G::DC;
  const int64_t stride = int64_t{1} << B1;
  const uint64_t pol_drop = evict_first_policy();  // last use of T1
  for (int g = threadIdx.x; g < (R / NA) * Q; g += SRHT_THREADS) {
    const int q = g % Q, rh = g / Q;
    const int64_t col = col0 + q * W;
    C v[NA][W];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      const C* src = T1 + (q1 + stride * (rh * NA + j)) * d + col;
      if (col + W <= d && d % W == 0) {
        if constexpr (sizeof(C) == 4) {
          const float4 t = ld_f4_hint(reinterpret_cast<const float*>(src), pol_drop);
          v[j][0] = t.x; v[j][1] = t.y; v[j][2] = t.z; v[j][3] = t.w;
        } else {
          const double2 t = *reinterpret_cast<const double2*>(src);
          v[j][0] = t.x; v[j][1] = t.y;
        }
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) v[j][w] = col + w < d ? src[w] : C(0);
      }
    }
    reg_wht<C, NA, W>(v);
#pragma unroll
    for (int j = 0; j < NA; ++j)
#pragma unroll
      for (int w = 0; w < W; ++w) S[rh * NA + j][q * W + w] = v[j][w];
  }
  __syncthreads();
  if (NB > 1) {
    for (int g = threadIdx.x; g < NA * Q; g += SRHT_THREADS) {
      const int q = g % Q, rl = g / Q;
      C v[NB][W];
#pragma unroll
      for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) v[j][w] = S[rl + NA * j][q * W + w];
      reg_wht<C, NB, W>(v);
#pragma unroll
      for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) S[rl + NA * j][q * W + w] = v[j][w];
    }
    __syncthreads();
  }
  // scatter the sampled outputs: SX[t] (+)= sign * S[q2]
  const int q = threadIdx.x % Q;
  const int64_t col = col0 + q * W;
  if (col >= d) return;
  for (uint32_t e = e0 + threadIdx.x / Q; e < e1; e += SRHT_THREADS / Q) {
    const uint32_t t = order[e];
    const uint64_t p = static_cast<uint64_t>(sample[t]);
    const int q2 = static_cast<int>((p >> B1) & static_cast<uint64_t>(R - 1));
    const bool neg = __popcll((p >> cb) & static_cast<uint64_t>(chunk)) & 1;
    double* dst = SX + static_cast<int64_t>(t) * d + col;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      if (col + w >= d) break;
      double v = static_cast<double>(S[q2][q * W + w]);
      if (neg) v = -v;
      double acc = first ? v : dst[w] + v;
      if (final_div != 0.0) acc = acc / final_div;
      dst[w] = acc;
    }
  }
}

__global__ void srht_keys_kernel(const int64_t* __restrict__ sample, int64_t k, uint64_t mask,
                                 uint32_t* __restrict__ keys, int64_t m, int32_t* bad) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < k;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = sample[t];
    if (p < 0 || p >= m) atomicOr(bad, LVSK_FLAG_BADINDEX);
    keys[t] = static_cast<uint32_t>(static_cast<uint64_t>(p) & mask);
  }
}

struct SrhtPlan {
  int L, B1, B2, cb;
  int64_t chunks;
};

static SrhtPlan plan_srht(int64_t m, int64_t d, size_t csize) {
  SrhtPlan p;
  p.L = 0;
  while ((int64_t{1} << p.L) < m) ++p.L;
  if (p.L <= 8) {
    p.B1 = p.L;
    p.B2 = 0;
  } else {
    p.B1 = 8;
    int maxcb = 8;
    size_t cap = SRHT_CHUNK_BYTES;
    if (const char* e = getenv("LVSK_SRHT_CHUNK_MB")) cap = static_cast<size_t>(atoi(e)) << 20;
    while (maxcb < 16 && (size_t{1} << (maxcb + 1)) * static_cast<size_t>(d) * csize <= cap) ++maxcb;
    int cb = p.L < maxcb ? p.L : maxcb;
    p.B2 = cb - 8;
  }
  p.cb = p.B1 + p.B2;
  p.chunks = int64_t{1} << (p.L - p.cb);
  return p;
}

template <typename T, typename C, bool VECTOR>
static void launch_pass1(int B, dim3 grid, cudaStream_t st, const T* X, int64_t n, int64_t d, int64_t ldx,
                         int64_t row0, const int8_t* signs, C* T1, int32_t* flags) {
#define LVSK_P1(BB)                                                                                              \
  case BB:                                                                                                       \
    srht_pass1_kernel<T, C, BB, VECTOR><<<grid, SRHT_THREADS, 0, st>>>(X, n, d, ldx, row0, signs, T1, flags); \
    break;
  switch (B) {
    LVSK_P1(0) LVSK_P1(1) LVSK_P1(2) LVSK_P1(3) LVSK_P1(4) LVSK_P1(5) LVSK_P1(6) LVSK_P1(7) LVSK_P1(8)
  }
#undef LVSK_P1
}

template <typename C>
static void launch_pass2(int B2, dim3 grid, cudaStream_t st, const C* T1, int64_t d, int B1, int64_t chunk, int cb,
                         const int64_t* sample, const uint32_t* order, const uint32_t* qstart, double* SX, int first,
                         double fd) {
#define LVSK_P2(BB)                                                                                            \
  case BB:                                                                                                     \
    srht_pass2_kernel<C, BB><<<grid, SRHT_THREADS, 0, st>>>(T1, d, B1, chunk, cb, sample, order, qstart, SX, \
                                                            first, fd);                                        \
    break;
  switch (B2) {
    LVSK_P2(0) LVSK_P2(1) LVSK_P2(2) LVSK_P2(3) LVSK_P2(4) LVSK_P2(5) LVSK_P2(6) LVSK_P2(7) LVSK_P2(8)
  }
#undef LVSK_P2
}

bool srht_sampled_ok(const float* X, int64_t n, int64_t d, int64_t ldx, int64_t m, int64_t k, int64_t row0);
size_t srht_sampled_workspace(int64_t n, int64_t d, int64_t m, int64_t k);
int32_t srht_sampled(const float* X, int64_t n, int64_t d, int64_t ldx, int64_t row0, int64_t m,
                     const int8_t* signs, const int64_t* sample, int64_t k, double divisor, double* SX, void* ws,
                     size_t ws_bytes, int32_t* flags, cudaStream_t st);
template <typename T, typename C>
static int32_t run_srht(const T* X, int64_t n, int64_t d, int64_t ldx, int64_t m, const int8_t* signs,
                        const int64_t* sample, int64_t k, double divisor, double* SX, void* ws, size_t ws_bytes,
                        int32_t* flags, cudaStream_t st) {
  if constexpr (std::is_same<T, float>::value) {
    if (srht_sampled_ok(X, n, d, ldx, m, k, 0))
      return srht_sampled(X, n, d, ldx, 0, m, signs, sample, k, divisor, SX, ws, ws_bytes, flags, st);
  }
  const SrhtPlan P = plan_srht(m, d, sizeof(C));
  Carve c(ws, ws_bytes);
  C* T1 = c.take<C>((size_t{1} << P.cb) * static_cast<size_t>(d));
  uint32_t* keys = c.take<uint32_t>(k);
  uint32_t* order = c.take<uint32_t>(k);
  uint32_t* qstart = c.take<uint32_t>((size_t{1} << P.B1) + 1);
  auto rb = radix::carve<uint32_t>(c, k);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  // group sampled rows by residue q1 = p & (2^B1 - 1)
  const uint64_t mask = (uint64_t{1} << P.B1) - 1;
  srht_keys_kernel<<<static_cast<unsigned>((k + 255) / 256), 256, 0, st>>>(sample, k, mask, keys, m, flags);
  int32_t rc = radix::sort_pairs<uint32_t, uint32_t>(keys, nullptr, k, P.B1, rb, rb.keys[1], order, st);
  if (rc != LVSK_OK) return rc;
  // qstart from the sorted residues
  radix::bucket_bounds_kernel<uint32_t><<<static_cast<unsigned>((k + 256) / 256), 256, 0, st>>>(rb.keys[1], k, int64_t{1} << P.B1,
                                                                               qstart);
  LVSK_CHECK_LAUNCH("srht sample grouping");
  const int64_t chunk_rows = int64_t{1} << P.cb;
  int64_t last = (n + chunk_rows - 1) / chunk_rows - 1;  // chunks past n are all padding
  if (last < 0) last = 0;
  if (last > P.chunks - 1) last = P.chunks - 1;
  const unsigned ycols = static_cast<unsigned>((d + SrhtCfg<C>::DC - 1) / SrhtCfg<C>::DC);
  const bool vector_ok = reinterpret_cast<uintptr_t>(X) % 16 == 0 && (ldx * sizeof(T)) % 16 == 0 &&
                         (d * sizeof(C)) % 16 == 0 && (d * sizeof(T)) % 16 == 0;
  for (int64_t ch = 0; ch <= last; ++ch) {
    dim3 g1(static_cast<unsigned>(chunk_rows >> P.B1), ycols);
    if (vector_ok)
      launch_pass1<T, C, true>(P.B1, g1, st, X, n, d, ldx, ch * chunk_rows, signs, T1, flags);
    else
      launch_pass1<T, C, false>(P.B1, g1, st, X, n, d, ldx, ch * chunk_rows, signs, T1, flags);
    dim3 g2(static_cast<unsigned>(int64_t{1} << P.B1), ycols);
    launch_pass2<C>(P.B2, g2, st, T1, d, P.B1, ch, P.cb, sample, order, qstart, SX, ch == 0 ? 1 : 0,
                    ch == last ? divisor : 0.0);
  }
  LVSK_CHECK_LAUNCH("srht passes");
  return LVSK_OK;
}

}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_srht_workspace_bytes(int64_t m, int64_t d, int32_t dtype, int64_t k) {
  const size_t cs = dtype == LVSK_F64 ? 8 : 4;
  const SrhtPlan P = plan_srht(m, d, cs);
  Measure ms;
  ms.take<char>((size_t{1} << P.cb) * static_cast<size_t>(d) * cs);
  ms.take<uint32_t>(k);
  ms.take<uint32_t>(k);
  ms.take<uint32_t>((size_t{1} << P.B1) + 1);
  radix::measure<uint32_t>(ms, k);
  if (dtype == LVSK_F32) {
    const size_t s3 = srht_sampled_workspace(m, d, m, k);
    if (s3 > ms.off) return s3;
  }
  return ms.off;
}

extern "C" int32_t lvsk_srht(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx, int64_t m,
                             const int8_t* signs, const int64_t* sample, int64_t k, double divisor, double* SX,
                             void* ws, size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(n >= 1 && d >= 1 && ldx >= d, LVSK_ERR_DIMENSION, "bad shape n=%lld d=%lld", (long long)n,
               (long long)d);
  LVSK_REQUIRE(m >= n && (m & (m - 1)) == 0, LVSK_ERR_CONFIGURATION, "m=%lld must be a power of two >= n",
               (long long)m);
  LVSK_REQUIRE(k >= 1 && k <= m, LVSK_ERR_CONFIGURATION, "SRHT needs 1 <= k <= m (k=%lld, m=%lld)", (long long)k,
               (long long)m);
  LVSK_REQUIRE(divisor != 0.0, LVSK_ERR_CONFIGURATION, "divisor must be nonzero");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case LVSK_F32:
      return run_srht<float, float>(static_cast<const float*>(X), n, d, ldx, m, signs, sample, k, divisor, SX, ws,
                                    ws_bytes, flags, st);
    case LVSK_F64:
      return run_srht<double, double>(static_cast<const double*>(X), n, d, ldx, m, signs, sample, k, divisor, SX,
                                      ws, ws_bytes, flags, st);
    case LVSK_BF16:
      return run_srht<__nv_bfloat16, float>(static_cast<const __nv_bfloat16*>(X), n, d, ldx, m, signs, sample, k,
                                            divisor, SX, ws, ws_bytes, flags, st);
  }
  set_error("unknown dtype %d", dtype);
  return LVSK_ERR_CONFIGURATION;
}
