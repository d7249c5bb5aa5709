// K5 — leverage pass: scores[i] = || X[i,:] M ||^2 (fused row sum of squares).
//
// Reference: _block_scores (pkg/src/levsketch/leverage.py:88-95): u = rows @
// basis; einsum("ij,ij->i", u, u).  X is read once; the d x r product never
// leaves registers.  This file holds the SIMT kernel (any d, r, dtype; fp32
// FFMA for fp32/bf16 inputs, fp64 for fp64 inputs).  The tcgen05 / TMEM
// 3xTF32 kernel for the fp32 r in {64,128} hot configurations lives in
// leverage_tc.cu and is selected by lvsk_rowsumsq_gemm.
#include "common.cuh"

namespace lvsk {

constexpr int L_BM = 64, L_BN = 64, L_BK = 32;

template <typename T, typename A>
__global__ void __launch_bounds__(256) rowsumsq_simt_kernel(const T* __restrict__ X, int64_t n, int64_t d,
                                                            int64_t ldx, const A* __restrict__ M, int64_t r,
                                                            double* __restrict__ scores, int32_t* flags) {
  __shared__ A Xs[L_BK][L_BM + 1];
  __shared__ A Ms[L_BK][L_BN];
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * L_BM;
  A rowsq[4] = {A(0), A(0), A(0), A(0)};
  bool bad = false;
  for (int64_t n0 = 0; n0 < r; n0 += L_BN) {
    A acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = A(0);
    for (int64_t k0 = 0; k0 < d; k0 += L_BK) {
      for (int e = tid; e < L_BM * L_BK; e += 256) {
        const int rr = e / L_BK, kk = e % L_BK;
        const int64_t row = row0 + rr, col = k0 + kk;
        A v = A(0);
        if (row < n && col < d) {
          v = static_cast<A>(to_f64<T>(X[row * ldx + col]));
          if (n0 == 0) bad |= !isfinite(static_cast<double>(v));
        }
        Xs[kk][rr] = v;
      }
      for (int e = tid; e < L_BK * L_BN; e += 256) {
        const int kk = e / L_BN, cc = e % L_BN;
        const int64_t kr = k0 + kk, c = n0 + cc;
        Ms[kk][cc] = (kr < d && c < r) ? M[kr * r + c] : A(0);
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < L_BK; ++kk) {
        A a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = Xs[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Ms[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) rowsq[i] += acc[i][j] * acc[i][j];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    A v = rowsq[i];
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    const int64_t row = row0 + ty + 16 * i;
    if (tx == 0 && row < n) scores[row] = static_cast<double>(v);
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(flags, LVSK_FLAG_NONFINITE);
}

}  // namespace lvsk

using namespace lvsk;

namespace lvsk {

// K5 operand split of a float64 fold M (d x r) in one launch (was a chain of
// small framework kernels on the fold's critical path):
//   tf32 mode:  Mt_hi = M^T with the low 13 mantissa bits of fp32(M) cleared
//               (exact TF32), Mt_lo = fp32(M^T - Mt_hi), Mt_hb = bf16(Mt_hi)
//   bf16 mode:  out rows [0, r) = bf16(fp32(M^T)), rows [r_pad, r_pad + r) =
//               bf16(fp32(M^T - hi))   (the other rows stay as they are)
__global__ void split_fold_kernel(const double* __restrict__ M, int64_t d, int64_t r, int bf16_mode, int64_t r_pad,
                                  float* __restrict__ hi, float* __restrict__ lo, __nv_bfloat16* __restrict__ hb) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < d * r;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / r, c = idx - i * r;
    const double m = M[idx];
    if (bf16_mode) {
      const __nv_bfloat16 h = __float2bfloat16_rn(__double2float_rn(m));
      const __nv_bfloat16 l = __float2bfloat16_rn(__double2float_rn(m - static_cast<double>(__bfloat162float(h))));
      hb[c * d + i] = h;
      hb[(r_pad + c) * d + i] = l;
    } else {
      const float h = __uint_as_float(__float_as_uint(__double2float_rn(m)) & ~0x1FFFu);
      hi[c * d + i] = h;
      lo[c * d + i] = __double2float_rn(m - static_cast<double>(h));
      if (hb != nullptr) hb[c * d + i] = __float2bfloat16_rn(h);
    }
  }
}

}  // namespace lvsk

extern "C" int32_t lvsk_split_fold(const double* M, int64_t d, int64_t r, int32_t bf16_mode, int64_t r_pad,
                                   float* Mt_hi, float* Mt_lo, void* Mt_bf16, void* stream) {
  using namespace lvsk;
  LVSK_REQUIRE(d >= 1 && r >= 1 && M, LVSK_ERR_DIMENSION, "bad fold shape d=%lld r=%lld", (long long)d, (long long)r);
  LVSK_REQUIRE(bf16_mode ? (Mt_bf16 != nullptr && r_pad >= r) : (Mt_hi != nullptr && Mt_lo != nullptr),
               LVSK_ERR_CONFIGURATION, "missing split outputs");
  const int64_t work = d * r;
  const unsigned grid = static_cast<unsigned>(work < 256 * 1184 ? (work + 255) / 256 : 1184);
  split_fold_kernel<<<grid, 256, 0, as_stream(stream)>>>(M, d, r, bf16_mode, r_pad, Mt_hi, Mt_lo,
                                                         static_cast<__nv_bfloat16*>(Mt_bf16));
  LVSK_CHECK_LAUNCH("split fold");
  return LVSK_OK;
}

extern "C" int32_t lvsk_rowsumsq_gemm(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx,
                                      const void* M, const void* M_lo, int64_t r, double* scores, int32_t* flags,
                                      void* stream) {
  LVSK_REQUIRE(n >= 0 && d >= 1 && ldx >= d && r >= 1, LVSK_ERR_DIMENSION, "bad shape n=%lld d=%lld r=%lld",
               (long long)n, (long long)d, (long long)r);
  if (n == 0) return LVSK_OK;
  cudaStream_t st = as_stream(stream);
  const unsigned grid = static_cast<unsigned>((n + L_BM - 1) / L_BM);
  switch (dtype) {
    case LVSK_F32: {
      rowsumsq_simt_kernel<float, float><<<grid, 256, 0, st>>>(static_cast<const float*>(X), n, d, ldx,
                                                               static_cast<const float*>(M), r, scores, flags);
      break;
    }
    case LVSK_F64:
      rowsumsq_simt_kernel<double, double><<<grid, 256, 0, st>>>(static_cast<const double*>(X), n, d, ldx,
                                                                 static_cast<const double*>(M), r, scores, flags);
      break;
    case LVSK_BF16:
      rowsumsq_simt_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>(
          static_cast<const __nv_bfloat16*>(X), n, d, ldx, static_cast<const float*>(M), r, scores, flags);
      break;
    default:
      set_error("unknown dtype %d", dtype);
      return LVSK_ERR_CONFIGURATION;
  }
  LVSK_CHECK_LAUNCH("rowsumsq");
  return LVSK_OK;
}
