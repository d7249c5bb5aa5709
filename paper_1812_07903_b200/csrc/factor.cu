// KF — the certified Cholesky fold in one cooperative kernel.
//
// Replaces the cuSOLVER potrf + two trsm chains of the fold (leverage.py
// _chol_body; oracle fold_r, the JL-fold definition M = R^-1 Pi with R the
// positive-diagonal triangular factor of SX, R^T R = G = SX^T SX).  Inputs:
// G (d x d, float64, symmetric; the upper triangle is read) and Pi (d x r).
// Outputs: M = R^-1 Pi (d x r, float64) and diag = [info, trace(G),
// trace(G^-1)] with trace(G^-1) = ||R^-1||_F^2 (the truncation certificate of
// leverage.chol_certified).
//
// B200 design.  The d x d problem is latency-bound (d <= a few thousand), so
// one persistent cooperative kernel (<= 1 CTA per SM, 256 threads) walks the
// blocked algorithm over 64 x 64 float64 tiles held in global memory (L2
// resident: d = 512 is 2 MB) with a grid barrier between dependent phases:
//   Cholesky step j:  B(j) panel solves  U_jk = U_jj^-T A_jk        (k > j)
//                     C(j) trailing updates A_kl -= U_jk^T U_jl   (j < k <= l),
//                          the task owning (j+1, j+1) also factors it
//   back substitution X = U^-1 [Pi | I]:  step i updates W_l,c -= U_li X_ic
//                          (l < i), the task owning (i-1, c) also solves it
// Each tile op runs from shared memory: 64-step substitutions / factorization
// with one __syncthreads per step, and 4 x 4 register-blocked float64 tile
// GEMMs.  Padding rows (d % 64) carry an identity so no branch reaches the
// math.  Zero tiles of the identity right-hand side (U^-1 is triangular) are
// skipped.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lvsk {

constexpr int FT = 64;          // tile edge
constexpr int FLD = FT + 1;     // smem row stride (transposed loads stay ~conflict-free)
constexpr int FTHREADS = 256;
constexpr int FTILE_SMEM = FT * FLD * 8;

struct FactorArgs {
  const double* G;
  int64_t d, ldg;
  const double* Pi;
  int64_t r;
  double* M;  // d x r, row-major
  double* diag;
  double* A;  // dp x dp working copy (upper tiles)
  double* W;  // dp x wc right-hand sides, overwritten by X
  double* partial;
  int32_t* info;
  int nb, rt, ct;  // tiles per edge, Pi column tiles, total RHS column tiles (rt + nb)
  int64_t dp, wc;
};

// ---- tile movement -----------------------------------------------------------

__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld) {
  for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
    const int m = e >> 6, c = e & 63;
    s[m * FLD + c] = g[m * ld + c];
  }
}
__device__ __forceinline__ void load_tile_t(double* s, const double* g, int64_t ld) {
  for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
    const int m = e >> 6, c = e & 63;
    s[c * FLD + m] = g[m * ld + c];
  }
}
__device__ __forceinline__ void store_tile(double* g, int64_t ld, const double* s) {
  for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
    const int m = e >> 6, c = e & 63;
    g[m * ld + c] = s[m * FLD + c];
  }
}

// ---- tile math ---------------------------------------------------------------

// C (global, 64 x 64) -= At^T B with At[p][m], B[p][c] in smem; the result is
// also left in smem tile `out` when out != nullptr.
__device__ __forceinline__ void gemm_sub(double* gC, int64_t ldc, const double* At, const double* B, double* out) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = gC[(ty + 16 * a) * ldc + tx + 16 * b];
#pragma unroll 4
  for (int p = 0; p < FT; ++p) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = At[p * FLD + ty + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = B[p * FLD + tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(-av[a], bv[b], acc[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (out)
        out[(ty + 16 * a) * FLD + tx + 16 * b] = acc[a][b];
      else
        gC[(ty + 16 * a) * ldc + tx + 16 * b] = acc[a][b];
    }
}

// In-place Cholesky of the upper triangle of s (s = U^T U, U upper with a
// positive diagonal); the strict lower triangle is zeroed.  Returns through
// *bad a nonzero value when a pivot is not positive and finite.
__device__ void chol_tile(double* s, int32_t* bad) {
  const int c = threadIdx.x & 63, g = threadIdx.x >> 6;
  for (int p = 0; p < FT; ++p) {
    __syncthreads();
    const double piv = s[p * FLD + p];
    if (c > p) {
      const double w = s[p * FLD + c] / piv;
      for (int m = p + 1 + ((g - (p + 1)) & 3); m <= c; m += 4) s[m * FLD + c] = fma(-s[p * FLD + m], w, s[m * FLD + c]);
    }
  }
  __syncthreads();
  // scale rows: U[p][c] = a[p][c] / sqrt(a[p][p]); reads of the diagonal must
  // finish before any row is rewritten
  double dg[FT / 4];
  for (int i = 0; i < FT / 4; ++i) {
    const int m = g + 4 * i;
    dg[i] = s[m * FLD + m];
  }
  __syncthreads();
  for (int i = 0; i < FT / 4; ++i) {
    const int m = g + 4 * i;
    const double piv = dg[i];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (c == 0) atomicOr(bad, 1);
    }
    const double v = s[m * FLD + c];
    s[m * FLD + c] = c >= m ? v / sqrt(piv) : 0.0;
  }
  __syncthreads();
}

// Y = U^-T B (forward substitution with the lower U^T): B in smem (destroyed),
// Y written to smem `y`.
__device__ void solve_lower_t(const double* U, double* b, double* y) {
  const int c = threadIdx.x & 63, g = threadIdx.x >> 6;
  for (int p = 0; p < FT; ++p) {
    __syncthreads();
    const double x = b[p * FLD + c] / U[p * FLD + p];
    if (g == 0) y[p * FLD + c] = x;
    for (int m = p + 1 + ((g - (p + 1)) & 3); m < FT; m += 4) b[m * FLD + c] = fma(-U[p * FLD + m], x, b[m * FLD + c]);
  }
  __syncthreads();
}

// X = U^-1 B (backward substitution with the upper U): B in smem (destroyed).
__device__ void solve_upper(const double* U, double* b, double* x_out) {
  const int c = threadIdx.x & 63, g = threadIdx.x >> 6;
  for (int p = FT - 1; p >= 0; --p) {
    __syncthreads();
    const double x = b[p * FLD + c] / U[p * FLD + p];
    if (g == 0) x_out[p * FLD + c] = x;
    for (int m = g; m < p; m += 4) b[m * FLD + c] = fma(-U[m * FLD + p], x, b[m * FLD + c]);
  }
  __syncthreads();
}

// ---- the kernel ----------------------------------------------------------------

__device__ __forceinline__ double* atile(const FactorArgs& a, int k, int l) {
  return a.A + static_cast<int64_t>(k) * FT * a.dp + static_cast<int64_t>(l) * FT;
}
__device__ __forceinline__ double* wtile(const FactorArgs& a, int i, int c) {
  return a.W + static_cast<int64_t>(i) * FT * a.wc + static_cast<int64_t>(c) * FT;
}

// identity column tile c (c >= rt) has nonzero X rows only for i <= c - rt
__device__ __forceinline__ bool x_live(const FactorArgs& a, int i, int c) { return c < a.rt || i <= c - a.rt; }

__global__ void __launch_bounds__(FTHREADS, 1) chol_fold_kernel(FactorArgs a) {
  extern __shared__ double fsm[];
  double* s0 = fsm;
  double* s1 = fsm + FT * FLD;
  double* s2 = fsm + 2 * FT * FLD;
  cg::grid_group grid = cg::this_grid();
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int nb = a.nb;

  // phase 0: working copies (padding: identity on the diagonal, zeros elsewhere)
  {
    const int64_t dp = a.dp;
    const int64_t total = dp * dp + dp * a.wc;
    for (int64_t e = static_cast<int64_t>(cta) * FTHREADS + threadIdx.x; e < total;
         e += static_cast<int64_t>(ncta) * FTHREADS) {
      if (e < dp * dp) {
        const int64_t m = e / dp, c = e - m * dp;
        double v;
        if (m < a.d && c < a.d)
          v = m <= c ? a.G[m * a.ldg + c] : 0.0;
        else
          v = m == c ? 1.0 : 0.0;
        a.A[e] = v;
      } else {
        const int64_t f = e - dp * dp;
        const int64_t m = f / a.wc, c = f - m * a.wc;
        const int64_t rp = static_cast<int64_t>(a.rt) * FT;
        double v;
        if (c < rp)
          v = (m < a.d && c < a.r) ? a.Pi[m * a.r + c] : 0.0;
        else
          v = (c - rp) == m ? 1.0 : 0.0;
        a.W[f] = v;
      }
    }
    if (cta == 0) {
      // trace(G) in a fixed order (one warp, then lane 0)
      if (threadIdx.x < 32) {
        double t = 0.0;
        for (int64_t i = threadIdx.x; i < a.d; i += 32) t += a.G[i * a.ldg + i];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, o);
        if (threadIdx.x == 0) {
          a.diag[1] = t;
          *a.info = 0;
        }
      }
    }
  }
  grid.sync();
  if (cta == 0) {
    load_tile(s0, atile(a, 0, 0), a.dp);
    chol_tile(s0, a.info);
    store_tile(atile(a, 0, 0), a.dp, s0);
  }
  grid.sync();

  // ---- blocked Cholesky
  for (int j = 0; j < nb - 1; ++j) {
    // B(j): U_jk = U_jj^-T A_jk
    for (int k = j + 1 + cta; k < nb; k += ncta) {
      load_tile(s0, atile(a, j, j), a.dp);
      load_tile(s1, atile(a, j, k), a.dp);
      solve_lower_t(s0, s1, s2);
      store_tile(atile(a, j, k), a.dp, s2);
      __syncthreads();
    }
    grid.sync();
    // C(j): A_kl -= U_jk^T U_jl for j < k <= l; task 0 is (j+1, j+1) + factor
    const int m = nb - j - 1;
    const int ntask = m * (m + 1) / 2;
    for (int t = cta; t < ntask; t += ncta) {
      // t -> (k, l): row-major over the upper triangle starting at (j+1, j+1)
      int k = 0, rem = t;
      while (rem >= m - k) {
        rem -= m - k;
        ++k;
      }
      const int kk = j + 1 + k, ll = kk + rem;
      load_tile(s0, atile(a, j, kk), a.dp);
      load_tile(s1, atile(a, j, ll), a.dp);
      __syncthreads();
      if (t == 0) {
        gemm_sub(atile(a, kk, ll), a.dp, s0, s1, s2);
        chol_tile(s2, a.info);
        store_tile(atile(a, kk, ll), a.dp, s2);
      } else {
        gemm_sub(atile(a, kk, ll), a.dp, s0, s1, nullptr);
      }
      __syncthreads();
    }
    grid.sync();
  }

  // ---- back substitution X = U^-1 W, in place in W
  const int ct = a.ct;
  for (int c = cta; c < ct; c += ncta) {
    if (!x_live(a, nb - 1, c)) continue;
    load_tile(s0, atile(a, nb - 1, nb - 1), a.dp);
    load_tile(s1, wtile(a, nb - 1, c), a.wc);
    solve_upper(s0, s1, s2);
    store_tile(wtile(a, nb - 1, c), a.wc, s2);
    __syncthreads();
  }
  grid.sync();
  for (int i = nb - 1; i >= 1; --i) {
    // tasks (l, c), l < i; the l = i-1 tasks (update + solve) are enumerated first
    const int ntask = i * ct;
    for (int t = cta; t < ntask; t += ncta) {
      const int l = i - 1 - t / ct, c = t % ct;
      const bool solve = l == i - 1;
      if (solve && !x_live(a, l, c)) continue;
      const bool upd = x_live(a, i, c);
      if (!upd && !solve) continue;
      if (upd) {
        load_tile_t(s0, atile(a, l, i), a.dp);
        load_tile(s1, wtile(a, i, c), a.wc);
        __syncthreads();
        gemm_sub(wtile(a, l, c), a.wc, s0, s1, solve ? s2 : nullptr);
      } else {
        load_tile(s2, wtile(a, l, c), a.wc);
      }
      if (solve) {
        __syncthreads();
        load_tile(s0, atile(a, l, l), a.dp);
        solve_upper(s0, s2, s1);
        store_tile(wtile(a, l, c), a.wc, s1);
      }
      __syncthreads();
    }
    grid.sync();
  }

  // ---- outputs: M (Pi columns) and per-tile sums of squares of U^-1
  {
    const int ntask = nb * ct;
    for (int t = cta; t < ntask; t += ncta) {
      const int i = t / ct, c = t % ct;
      const double* x = wtile(a, i, c);
      if (c < a.rt) {
        for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
          const int64_t m = static_cast<int64_t>(i) * FT + (e >> 6);
          const int64_t q = static_cast<int64_t>(c) * FT + (e & 63);
          if (m < a.d && q < a.r) a.M[m * a.r + q] = x[(e >> 6) * a.wc + (e & 63)];
        }
      } else {
        double ss = 0.0;
        if (x_live(a, i, c)) {
          for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
            const int64_t m = static_cast<int64_t>(i) * FT + (e >> 6);
            const int64_t q = static_cast<int64_t>(c - a.rt) * FT + (e & 63);
            if (m < a.d && q < a.d) {
              const double v = x[(e >> 6) * a.wc + (e & 63)];
              ss = fma(v, v, ss);
            }
          }
        }
        // fixed-order block reduction
        __shared__ double red[FTHREADS / 32];
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xFFFFFFFFu, ss, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
          double tsum = 0.0;
          for (int w = 0; w < FTHREADS / 32; ++w) tsum += red[w];
          a.partial[t] = tsum;
        }
        __syncthreads();
      }
    }
  }
  grid.sync();
  if (cta == 0 && threadIdx.x == 0) {
    double tr = 0.0;
    for (int t = 0; t < nb * ct; ++t)
      if (t % ct >= a.rt) tr += a.partial[t];
    a.diag[2] = tr;
    a.diag[0] = static_cast<double>(*a.info);
  }
}

struct FactorPlan {
  int nb, rt, ct;
  int64_t dp, wc;
};

static FactorPlan plan_factor(int64_t d, int64_t r) {
  FactorPlan p;
  p.nb = static_cast<int>((d + FT - 1) / FT);
  p.rt = static_cast<int>((r + FT - 1) / FT);
  p.ct = p.rt + p.nb;
  p.dp = static_cast<int64_t>(p.nb) * FT;
  p.wc = static_cast<int64_t>(p.ct) * FT;
  return p;
}

}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_chol_fold_workspace_bytes(int64_t d, int64_t r) {
  if (d < 1 || r < 1) return 0;
  const FactorPlan P = plan_factor(d, r);
  Measure ms;
  ms.take<double>(static_cast<size_t>(P.dp) * P.dp);
  ms.take<double>(static_cast<size_t>(P.dp) * P.wc);
  ms.take<double>(static_cast<size_t>(P.nb) * P.ct);
  ms.take<int32_t>(1);
  return ms.off;
}

extern "C" int32_t lvsk_chol_fold(const double* G, int64_t d, int64_t ldg, const double* Pi, int64_t r, double* M,
                                  double* diag, void* ws, size_t ws_bytes, void* stream) {
  LVSK_REQUIRE(d >= 1 && r >= 1 && ldg >= d, LVSK_ERR_DIMENSION, "bad fold shape d=%lld r=%lld ldg=%lld",
               (long long)d, (long long)r, (long long)ldg);
  LVSK_REQUIRE(G && Pi && M && diag, LVSK_ERR_CONFIGURATION, "null pointer argument");
  const FactorPlan P = plan_factor(d, r);
  Carve c(ws, ws_bytes);
  FactorArgs a;
  a.G = G;
  a.d = d;
  a.ldg = ldg;
  a.Pi = Pi;
  a.r = r;
  a.M = M;
  a.diag = diag;
  a.A = c.take<double>(static_cast<size_t>(P.dp) * P.dp);
  a.W = c.take<double>(static_cast<size_t>(P.dp) * P.wc);
  a.partial = c.take<double>(static_cast<size_t>(P.nb) * P.ct);
  a.info = c.take<int32_t>(1);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  a.nb = P.nb;
  a.rt = P.rt;
  a.ct = P.ct;
  a.dp = P.dp;
  a.wc = P.wc;
  const int smem = 3 * FTILE_SMEM;
  static int grid_cap = 0;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(chol_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "chol_fold smem attribute");
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, chol_fold_kernel, FTHREADS, smem);
    grid_cap = sms * (per < 1 ? 1 : (per > 1 ? 1 : per));
    if (grid_cap < 1) grid_cap = 1;
  }
  // more CTAs than the widest phase only adds barrier cost
  int64_t widest = static_cast<int64_t>(P.nb) * P.ct;
  const int64_t tri = static_cast<int64_t>(P.nb) * (P.nb + 1) / 2;
  if (tri > widest) widest = tri;
  const int grid = static_cast<int>(widest < grid_cap ? widest : grid_cap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(FTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, chol_fold_kernel, a);
  if (e != cudaSuccess) return cuda_status(e, "chol_fold launch");
  return LVSK_OK;
}
