// KD — the Gram G = SX^T SX of the fold for d < 2048 (C1-C3, C5) on the
// float64 tensor cores.  Reference: the float64 products inside _approx_basis
// / truncate (pkg/src/levsketch/leverage.py:75-85, svd.py:30-54); the
// Cholesky fold (factor.cu) reads G's upper triangle, the spectral routes
// symmetrise it.
//
// Only the 64 x 64 block upper triangle (tiles bi <= bj) is formed — half the
// flops of the full DGEMM the pipeline ran before (cuBLAS's sm80 d884 kernel):
// C2 (k 4096, d 512) 77 -> 60 us, C5 (2048, 1024) 132 -> 99 us, C3 34 -> 27 us
// (tools/gram_kd_time.py; ~20 TF/s, about half the DMMA peak: each warp's
// 32 x 16 block loads 6 fragment values per 8 DMMAs, two CTAs per SM).  The k summation is split into S row slices so the small
// tile count (36 tiles at d = 512) still fills the GPU: CTA (pair, s) stages
// 32-row chunks of the two 64-column panels of SX with cp.async
// (three stages, 16-byte copies, L2-resident SX) and accumulates At^T B on DMMA
// (mma.m8n8k4.f64, the KF tile product's fragment layout); the S partial
// tiles are then added in a fixed slice order, so G is deterministic.
#include "common.cuh"

namespace lvsk {
namespace kd {

constexpr int T = 64;        // tile edge
constexpr int BK = 32;       // rows per staged chunk
constexpr int LD = T + 4;    // smem row stride (= 4 mod 16: conflict-free fragment loads)
constexpr int THREADS = 256;
constexpr int NS = 3;                       // cp.async stages (two chunks in flight)
constexpr int SMEM = NS * 2 * BK * LD * 8;  // (A, B) x stages: 104 KB, two CTAs per SM

struct Args {
  const double* SX;
  int64_t k, d, ld;
  double* part;  // [S][npairs][T*T] (S > 1)
  double* G;
  int64_t ldg;
  int ntile, npairs, S;
  int64_t rows_per;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

// pair index -> (bi, bj), bi <= bj, row-major over the upper triangle
__device__ __forceinline__ void pair_of(int p, int nt, int& bi, int& bj) {
  int i = 0;
  while (p >= nt - i) {
    p -= nt - i;
    ++i;
  }
  bi = i;
  bj = i + p;
}

__global__ void __launch_bounds__(THREADS) syrk_kernel(Args a) {
  extern __shared__ __align__(16) double kd_smem[];
  double* As = kd_smem;                  // [NS][BK][LD]
  double* Bs = kd_smem + NS * BK * LD;   // [NS][BK][LD]
  int bi, bj;
  pair_of(blockIdx.x, a.ntile, bi, bj);
  const bool diag = bi == bj;
  const int s = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(s) * a.rows_per;
  const int64_t r1 = r0 + a.rows_per < a.k ? r0 + a.rows_per : a.k;
  const int nchunks = r1 > r0 ? static_cast<int>((r1 - r0 + BK - 1) / BK) : 0;
  const int64_t ci = static_cast<int64_t>(bi) * T, cj = static_cast<int64_t>(bj) * T;
  // 16-byte copies when every row start of SX is 16-byte aligned and d is even
  const bool vec = ((reinterpret_cast<uintptr_t>(a.SX) | static_cast<uintptr_t>(a.ld * 8)) & 15) == 0 && (a.d & 1) == 0;

  auto stage_panel = [&](double* D, int64_t rb, int64_t c0) {
    if (vec) {
      for (int e = threadIdx.x; e < BK * T / 2; e += THREADS) {
        const int row = e >> 5, col = 2 * (e & 31);
        const int64_t r = rb + row;
        if (r < r1 && c0 + col < a.d) cp_async16(D + row * LD + col, a.SX + r * a.ld + c0 + col);
        else *reinterpret_cast<double2*>(D + row * LD + col) = make_double2(0.0, 0.0);
      }
    } else {
      for (int e = threadIdx.x; e < BK * T; e += THREADS) {
        const int row = e >> 6, col = e & 63;
        const int64_t r = rb + row;
        if (r < r1 && c0 + col < a.d) cp_async8(D + row * LD + col, a.SX + r * a.ld + c0 + col);
        else D[row * LD + col] = 0.0;
      }
    }
  };
  auto stage = [&](int c) {
    if (c < nchunks) {
      const int64_t rb = r0 + static_cast<int64_t>(c) * BK;
      const int buf = c % NS;
      stage_panel(As + buf * BK * LD, rb, ci);
      if (!diag) stage_panel(Bs + buf * BK * LD, rb, cj);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (empty groups keep the count uniform)
  };

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rb = (w & 1) * 32, cb = (w >> 1) * 16;
  const int qr = lane >> 2, qc = lane & 3;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int c = 0; c < NS - 1; ++c) stage(c);
  for (int c = 0; c < nchunks; ++c) {
    stage(c + NS - 1);  // refills the buffer read at c - 1 (released by the barrier below)
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
    __syncthreads();
    const double* A = As + (c % NS) * BK * LD;
    const double* B = diag ? A : Bs + (c % NS) * BK * LD;
#pragma unroll
    for (int k0 = 0; k0 < BK; k0 += 4) {
      const double* ar = A + (k0 + qc) * LD + rb + qr;
      const double* br = B + (k0 + qc) * LD + cb + qr;
      double av[4], bv[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = ar[8 * i];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = br[8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();  // buffer c % NS is restaged at c + NS
  }

#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int row = rb + 8 * i + qr, col = cb + 8 * j + 2 * qc;
      if (a.S == 1) {
        if (ci + row < a.d) {
          double* g = a.G + (ci + row) * a.ldg + cj + col;
          if (cj + col < a.d) g[0] = acc[i][j][0];
          if (cj + col + 1 < a.d) g[1] = acc[i][j][1];
        }
      } else {
        double* p = a.part + (static_cast<int64_t>(s) * a.npairs + blockIdx.x) * (T * T) + row * T + col;
        *reinterpret_cast<double2*>(p) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
}

// G tile = sum of the S slice partials in slice order (deterministic)
__global__ void reduce_kernel(Args a) {
  const int64_t total = static_cast<int64_t>(a.npairs) * T * T;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(e / (T * T));
    const int rc = static_cast<int>(e % (T * T)), row = rc / T, col = rc % T;
    int bi, bj;
    pair_of(p, a.ntile, bi, bj);
    const int64_t gr = static_cast<int64_t>(bi) * T + row, gc = static_cast<int64_t>(bj) * T + col;
    if (gr >= a.d || gc >= a.d) continue;
    double v = 0.0;
    for (int s = 0; s < a.S; ++s) v += a.part[(static_cast<int64_t>(s) * a.npairs + p) * (T * T) + rc];
    a.G[gr * a.ldg + gc] = v;
  }
}

struct Plan {
  int ntile, npairs, S;
  int64_t rows_per;
};

static Plan plan(int64_t k, int64_t d) {
  Plan p;
  p.ntile = static_cast<int>((d + T - 1) / T);
  p.npairs = p.ntile * (p.ntile + 1) / 2;
  // about two CTAs per SM, slices of at least 128 rows
  const int64_t want = (2 * 148 + p.npairs - 1) / p.npairs;
  const int64_t maxs = (k + 127) / 128;
  int64_t S = want < maxs ? want : maxs;
  if (S < 1) S = 1;
  p.rows_per = (k + S - 1) / S;
  p.rows_per = (p.rows_per + BK - 1) / BK * BK;
  p.S = static_cast<int>((k + p.rows_per - 1) / p.rows_per);
  if (p.S < 1) p.S = 1;
  return p;
}

}  // namespace kd
}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_syrk_workspace_bytes(int64_t k, int64_t d) {
  if (k < 1 || d < 1) return 0;
  const kd::Plan p = kd::plan(k, d);
  return p.S > 1 ? static_cast<size_t>(p.S) * p.npairs * kd::T * kd::T * sizeof(double) : 0;
}

extern "C" int32_t lvsk_syrk_f64(const double* SX, int64_t k, int64_t d, int64_t ldsx, double* G, int64_t ldg,
                                 void* ws, size_t ws_bytes, void* stream) {
  LVSK_REQUIRE(k >= 1 && d >= 1 && ldsx >= d && ldg >= d, LVSK_ERR_DIMENSION, "bad Gram shape k=%lld d=%lld",
               (long long)k, (long long)d);
  LVSK_REQUIRE(d <= 64 * 512, LVSK_ERR_CAPACITY, "d too large for the SYRK tile table");
  LVSK_REQUIRE(SX && G, LVSK_ERR_CONFIGURATION, "null pointer argument");
  const kd::Plan p = kd::plan(k, d);
  const size_t need = lvsk_syrk_workspace_bytes(k, d);
  LVSK_REQUIRE(ws_bytes >= need && (need == 0 || ws), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu",
               need, ws_bytes);
  cudaStream_t st = as_stream(stream);
  kd::Args a;
  a.SX = SX;
  a.k = k;
  a.d = d;
  a.ld = ldsx;
  a.part = static_cast<double*>(ws);
  a.G = G;
  a.ldg = ldg;
  a.ntile = p.ntile;
  a.npairs = p.npairs;
  a.S = p.S;
  a.rows_per = p.rows_per;
  const int32_t rc = ensure_smem_attr(reinterpret_cast<const void*>(kd::syrk_kernel), kd::SMEM, "syrk smem attribute");
  if (rc != LVSK_OK) return rc;
  kd::syrk_kernel<<<dim3(p.npairs, p.S), kd::THREADS, kd::SMEM, st>>>(a);
  LVSK_CHECK_LAUNCH("syrk");
  if (p.S > 1) {
    const int64_t total = static_cast<int64_t>(p.npairs) * kd::T * kd::T;
    const int64_t g = (total + 255) / 256;
    kd::reduce_kernel<<<static_cast<unsigned>(g < 4096 ? g : 4096), 256, 0, st>>>(a);
    LVSK_CHECK_LAUNCH("syrk reduce");
  }
  return LVSK_OK;
}
