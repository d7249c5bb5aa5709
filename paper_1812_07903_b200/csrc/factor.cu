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
//   Cholesky step j:  B(j) panels  U_jk = T_j^T A_jk  (T_j = U_jj^-1)  (k > j)
//                     C(j) trailing updates A_kl -= U_jk^T U_jl   (j < k <= l),
//                          the task owning (j+1, j+1) also factors and inverts it
//   back substitution X = U^-1 [Pi | I]:  step i updates W_l,c -= U_li X_ic
//                          (l < i), the task owning (i-1, c) then sets X = T W
// The only sequential tile op is the diagonal one (chol_inv_tile: 64-pivot
// Cholesky + the 64-step inverse of its factor, columns register-resident,
// one __syncthreads per pivot); panels and the substitution are 4 x 4
// register-blocked float64 tile GEMMs against those inverses.  Padding rows (d % 64) carry an identity so no branch reaches the
// math.  Zero tiles of the identity right-hand side (U^-1 is triangular) are
// skipped.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

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
  double* T;  // nb tiles 64 x 64: inverses of the diagonal tiles of U
  double* partial;
  int32_t* info;
  unsigned long long* trace;  // optional phase timestamps (LVSK_KF_TRACE), else null
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

// acc = (SUB ? C - At^T B : At^T B) with At[p][m], B[p][c] in smem (C read from
// global when SUB); the result goes to smem `out` when out != nullptr, else
// back to global C.  4 x 4 register blocking, 256 threads.
template <bool SUB>
__device__ __forceinline__ void gemm_tile(double* gC, int64_t ldc, const double* At, const double* B, double* out) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = SUB ? gC[(ty + 16 * a) * ldc + tx + 16 * b] : 0.0;
  const double sg = SUB ? -1.0 : 1.0;
#pragma unroll 4
  for (int p = 0; p < FT; ++p) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = sg * At[p * FLD + ty + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = B[p * FLD + tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
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

// Cholesky of the 64 x 64 tile s (upper triangle used; s = U^T U) and the
// inverse T = U^-1, both upper triangular, written to s and t.  One 64-step
// elimination on the augmented tile [A | I]: the row operations that take A
// to D L^T take I to L^-1, so U = D^-1/2 (D L^T) and T = L^-T D^-1/2.  Thread
// (column c, group g) keeps rows g, g+4, .. of column c of both halves in
// registers; one __syncthreads per pivot (pivot rows published through
// `rowbuf`).  *bad |= 1 on a pivot that is not positive and finite.
__device__ __noinline__ void chol_inv_tile(double* s, double* t, double* scratch, int32_t* bad) {
  const int c = threadIdx.x & 63, g = threadIdx.x >> 6;
  const int cw0 = c & 32;            // first column of this warp
  double* rowbuf = scratch;          // [2][2][64]: (A row, B row) per parity
  double* rsd = scratch + 4 * FT;    // [64] 1 / sqrt(pivot)
  double a[FT / 4], bm[FT / 4];
#pragma unroll
  for (int i = 0; i < FT / 4; ++i) {
    a[i] = s[(g + 4 * i) * FLD + c];
    bm[i] = (g + 4 * i == c) ? 1.0 : 0.0;
  }
  bool badp = false;
#pragma unroll
  for (int p = 0; p < FT; ++p) {
    double* ra = rowbuf + (p & 1) * 2 * FT;
    double* rb = ra + FT;
    if (g == (p & 3)) {
      ra[c] = a[p >> 2];
      rb[c] = bm[p >> 2];
    }
    __syncthreads();
    const double piv = ra[p];
    // 1/sqrt(piv): SFU approximation + one Newton step (rel. error ~1e-15)
    double rs;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(piv));
    rs = rs * fma(-0.5 * piv, rs * rs, 1.5);
    const double inv = rs * rs;
    // row m -= (a[p][m] / piv) row p, on both halves; columns left of the pivot
    // keep zero in the A half, columns right of it in the B half (L^-1 lower)
    const double wa = cw0 + 31 > p ? ra[c] * inv : 0.0;
    const double wb = cw0 <= p ? rb[c] * inv : 0.0;
#pragma unroll
    for (int i = 0; i < FT / 4; ++i) {
      if (g + 4 * i > p) {
        const double l = ra[g + 4 * i];
        a[i] = fma(-l, wa, a[i]);
        bm[i] = fma(-l, wb, bm[i]);
      }
    }
    if (g == (p & 3)) a[p >> 2] = c >= p ? a[p >> 2] * rs : 0.0;
    if (c == p && g == 0) {
      badp = !(piv > 0.0) || !isfinite(piv);
      rsd[p] = rs;
    }
  }
  if (badp) atomicOr(bad, 1);
#pragma unroll
  for (int i = 0; i < FT / 4; ++i) s[(g + 4 * i) * FLD + c] = a[i];
  __syncthreads();
  // T[c][m] = L^-1[m][c] / sqrt(D_m)
#pragma unroll
  for (int i = 0; i < FT / 4; ++i) t[c * FLD + g + 4 * i] = bm[i] * rsd[g + 4 * i];
  __syncthreads();
}

// ---- the kernel ----------------------------------------------------------------

__device__ __forceinline__ double* atile(const FactorArgs& a, int k, int l) {
  return a.A + static_cast<int64_t>(k) * FT * a.dp + static_cast<int64_t>(l) * FT;
}
__device__ __forceinline__ double* ttile(const FactorArgs& a, int j) { return a.T + static_cast<int64_t>(j) * FT * FT; }
__device__ __forceinline__ double* wtile(const FactorArgs& a, int i, int c) {
  return a.W + static_cast<int64_t>(i) * FT * a.wc + static_cast<int64_t>(c) * FT;
}

// identity column tile c (c >= rt) has nonzero X rows only for i <= c - rt
__device__ __forceinline__ bool x_live(const FactorArgs& a, int i, int c) { return c < a.rt || i <= c - a.rt; }

__device__ __forceinline__ void kf_mark(const FactorArgs& a, int& ph) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[ph] = t;
  }
  ++ph;
}

__global__ void __launch_bounds__(FTHREADS, 1) chol_fold_kernel(FactorArgs a) {
  int ph = 0;
  extern __shared__ double fsm[];
  double* s0 = fsm;
  double* s1 = fsm + FT * FLD;
  double* s2 = fsm + 2 * FT * FLD;
  double* scratch = fsm + 3 * FT * FLD;  // 5 x 64 doubles
  cg::grid_group grid = cg::this_grid();
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int nb = a.nb;

  // phase 0: working copies (padding: identity on the diagonal, zeros elsewhere);
  // one warp per row, no integer division
  {
    const int64_t dp = a.dp, wc = a.wc;
    const int64_t rp = static_cast<int64_t>(a.rt) * FT;
    const int wid = (cta * FTHREADS + threadIdx.x) >> 5, nw = (ncta * FTHREADS) >> 5, lane = threadIdx.x & 31;
    for (int64_t m = wid; m < 2 * dp; m += nw) {
      if (m < dp) {
        double* row = a.A + m * dp;
        for (int64_t c = lane; c < dp; c += 32)
          row[c] = (m < a.d && c < a.d) ? (m <= c ? a.G[m * a.ldg + c] : 0.0) : (m == c ? 1.0 : 0.0);
      } else {
        const int64_t mm = m - dp;
        double* row = a.W + mm * wc;
        for (int64_t c = lane; c < wc; c += 32)
          row[c] = c < rp ? ((mm < a.d && c < a.r) ? a.Pi[mm * a.r + c] : 0.0) : ((c - rp) == mm ? 1.0 : 0.0);
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
  kf_mark(a, ph);
  if (cta == 0) {
    load_tile(s0, atile(a, 0, 0), a.dp);
    chol_inv_tile(s0, s1, scratch, a.info);
    store_tile(atile(a, 0, 0), a.dp, s0);
    store_tile(ttile(a, 0), FT, s1);
  }
  grid.sync();
  kf_mark(a, ph);

  // ---- blocked Cholesky (T_j = U_jj^-1 from the task that factored U_jj)
  for (int j = 0; j < nb - 1; ++j) {
    // B(j): U_jk = T_j^T A_jk
    for (int k = j + 1 + cta; k < nb; k += ncta) {
      load_tile(s0, ttile(a, j), FT);
      load_tile(s1, atile(a, j, k), a.dp);
      __syncthreads();
      gemm_tile<false>(atile(a, j, k), a.dp, s0, s1, nullptr);
      __syncthreads();
    }
    grid.sync();
    kf_mark(a, ph);
    // C(j): A_kl -= U_jk^T U_jl for j < k <= l; task 0 is (j+1, j+1) + factor + inverse
    const int m = nb - j - 1;
    const int ntask = m * (m + 1) / 2;
    for (int t = cta; t < ntask; t += ncta) {
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
        unsigned long long t0, t1, t2, t3;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        gemm_tile<true>(atile(a, kk, ll), a.dp, s0, s1, s2);
        __syncthreads();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        chol_inv_tile(s2, s0, scratch, a.info);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
        store_tile(atile(a, kk, ll), a.dp, s2);
        store_tile(ttile(a, kk), FT, s0);
        __syncthreads();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
        if (a.trace != nullptr && threadIdx.x == 0) {
          a.trace[512 + 3 * j] = t1 - t0;
          a.trace[513 + 3 * j] = t2 - t1;
          a.trace[514 + 3 * j] = t3 - t2;
        }
      } else {
        gemm_tile<true>(atile(a, kk, ll), a.dp, s0, s1, nullptr);
      }
      __syncthreads();
    }
    grid.sync();
    kf_mark(a, ph);
  }

  // ---- back substitution X = U^-1 W, in place in W:  X_i = T_i (W_i - sum_{l>i} U_il X_l)
  const int ct = a.ct;
  for (int c = cta; c < ct; c += ncta) {
    if (!x_live(a, nb - 1, c)) continue;
    load_tile_t(s0, ttile(a, nb - 1), FT);
    load_tile(s1, wtile(a, nb - 1, c), a.wc);
    __syncthreads();
    gemm_tile<false>(wtile(a, nb - 1, c), a.wc, s0, s1, nullptr);
    __syncthreads();
  }
  grid.sync();
  kf_mark(a, ph);
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
        gemm_tile<true>(wtile(a, l, c), a.wc, s0, s1, solve ? s2 : nullptr);
      } else {
        load_tile(s2, wtile(a, l, c), a.wc);
      }
      if (solve) {
        __syncthreads();
        load_tile_t(s0, ttile(a, l), FT);
        __syncthreads();
        gemm_tile<false>(wtile(a, l, c), a.wc, s0, s2, nullptr);
      }
      __syncthreads();
    }
    grid.sync();
    kf_mark(a, ph);
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
  kf_mark(a, ph);
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
  ms.take<double>(static_cast<size_t>(P.nb) * FT * FT);
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
  a.T = c.take<double>(static_cast<size_t>(P.nb) * FT * FT);
  a.partial = c.take<double>(static_cast<size_t>(P.nb) * P.ct);
  a.info = c.take<int32_t>(1);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  a.nb = P.nb;
  a.rt = P.rt;
  a.ct = P.ct;
  a.dp = P.dp;
  a.wc = P.wc;
  const int smem = 3 * FTILE_SMEM + 5 * FT * 8;
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
  static unsigned long long* trace = nullptr;
  const bool tracing = getenv("LVSK_KF_TRACE") != nullptr;
  if (tracing && trace == nullptr) cudaMalloc(&trace, 1024 * sizeof(unsigned long long));
  a.trace = tracing ? trace : nullptr;
  cudaError_t e = cudaLaunchKernelEx(&cfg, chol_fold_kernel, a);
  if (e != cudaSuccess) return cuda_status(e, "chol_fold launch");
  if (tracing) {
    unsigned long long h[1024];
    const int nph = 4 + 2 * (P.nb - 1) + P.nb;
    cudaStreamSynchronize(cfg.stream);
    cudaMemcpy(h, trace, nph * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    fprintf(stderr, "KF d=%lld r=%lld grid=%d phases(us):", (long long)d, (long long)r, grid);
    for (int i = 1; i < nph; ++i) fprintf(stderr, " %.1f", (h[i] - h[i - 1]) / 1000.0);
    cudaMemcpy(h + 512, trace + 512, 3 * P.nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    fprintf(stderr, "\n  diag task gemm/chol_inv/store(us):");
    for (int j = 0; j + 1 < P.nb && j < 8; ++j)
      fprintf(stderr, " %.1f/%.1f/%.1f", h[512 + 3 * j] / 1000.0, h[513 + 3 * j] / 1000.0, h[514 + 3 * j] / 1000.0);
    fprintf(stderr, "\n");
  }
  return LVSK_OK;
}
