// KF — the certified Cholesky fold in one cooperative dataflow kernel.
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
// one persistent cooperative kernel (<= 1 CTA per SM, 256 threads) runs the
// blocked algorithm over 64 x 64 float64 tiles (global memory, L2 resident:
// d = 512 is 2 MB) as a DATAFLOW graph: every tile carries a version counter,
// a task waits (acquire) for the versions it reads and publishes (release)
// the one it writes, so no grid barrier separates the steps and step j+1
// starts while step j's trailing updates still run.  With U = R (upper) and
// Y = U^-T (lower), step j is
//   CHAIN(j+1)  U_j,j+1 = T_j^T A_j,j+1;  A_j+1,j+1 -= U^T U;  factor + invert
//               it (T_j+1 = U_j+1,j+1^-1, Y_j+1,j+1 = T_j+1^T) — the critical
//               path, run back to back by CTA 0 with T_j kept in shared memory
//   PANEL       U_jk = T_j^T A_jk                         (k > j + 1)
//   YROW        Y_jm = T_j^T W_jm                         (m < j)
//   UPD         A_kl -= U_jk^T U_jl                       (j < k <= l)
//   WUPD        W_km -= U_jk^T Y_jm                       (m <= j < k)
//   MACC        M_i  += Y_ji^T Pi_j                       (i <= j)
// i.e. the forward substitution U^T Y = I rides along the factorisation and
// M = U^-1 Pi = Y^T Pi accumulates as rows of Y complete, so there is no
// separate back substitution.  The other CTAs pull the remaining tasks from
// an atomic queue in topological order (deadlock-free: a task only waits on
// lower-numbered tasks or on CTA 0's chain, which only waits on tasks two
// steps back).  The only sequential tile op is the diagonal one
// (chol_inv_tile: 64-pivot Cholesky + the inverse of its factor, columns
// register-resident, one __syncthreads per pivot); everything else is a
// 4 x 4 register-blocked float64 tile GEMM.  Mutable tiles are read with
// ld.global.cg (L2) so no stale L1 line survives a version change.  Padding
// rows (d % 64) carry an identity so no branch reaches the math.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lvsk {

constexpr int FT = 64;          // tile edge
constexpr int FLD = FT + 4;     // smem row stride, = 4 mod 16: DMMA fragment loads are conflict-free
constexpr int FTHREADS = 256;
constexpr int FTILE_SMEM = FT * FLD * 8;
constexpr int KF_INFLIGHT_GRID = 24;

struct FactorArgs {
  const double* G;
  int64_t d, ldg;
  const double* Pi;
  int64_t r;
  double* M;  // d x r, row-major
  double* diag;
  double cert_limit;   // certificate: trace(G) * trace(G^-1) < cert_limit
  int32_t* cert_fail;  // optional counter, +1 when the certificate fails
  double* A;   // dp x dp: upper tiles, A -> U in place
  double* W;   // dp x dp: lower tiles, W -> Y = U^-T in place
  double* T;   // nb tiles 64 x 64: inverses of the diagonal tiles of U
  double* P;   // dp x rp: Pi, zero padded
  double* Ma;  // dp x rp: partial M = Y^T Pi
  double* partial;  // nb x nb: ||Y_km||_F^2 (valid entries)
  int32_t* verA;    // nb x nb tile versions
  int32_t* verW;    // nb x nb
  int32_t* verM;    // nb x rt
  int32_t* ctl;     // [0] queue head, [1] finished Y tiles, [2] info, [3] the chain CTA's SM
  unsigned long long* trace;  // optional chain timestamps (LVSK_KF_TRACE), else null
  int nb, rt;
  int64_t dp, rp;
};

// ---- synchronisation -----------------------------------------------------------

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// thread 0 spins until *f >= v; the CTA proceeds after the barrier
__device__ __forceinline__ void wait_ge(const int32_t* f, int v) {
  if (threadIdx.x == 0) {
    while (ld_acquire(f) < v) __nanosleep(32);
  }
}
// publish: every thread's tile stores are ordered before the flag — the CTA
// barrier orders them before thread 0's release, and a gpu-scope release is
// cumulative (the CUTLASS semaphore pattern), so no separate fence.sc
__device__ __forceinline__ void signal(int32_t* f, int v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(f, v);
}

// ---- tile movement (mutable tiles through L2 only) ------------------------------

__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld) {
  for (int e = threadIdx.x; e < FT * FT / 2; e += FTHREADS) {
    const int m = e >> 5, c = 2 * (e & 31);
    *reinterpret_cast<double2*>(s + m * FLD + c) = __ldcg(reinterpret_cast<const double2*>(g + m * ld + c));
  }
}
__device__ __forceinline__ void store_tile(double* g, int64_t ld, const double* s) {
  for (int e = threadIdx.x; e < FT * FT / 2; e += FTHREADS) {
    const int m = e >> 5, c = 2 * (e & 31);
    *reinterpret_cast<double2*>(g + m * ld + c) = *reinterpret_cast<const double2*>(s + m * FLD + c);
  }
}
__device__ __forceinline__ void store_tile_t(double* g, int64_t ld, const double* s) {
  for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
    const int m = e >> 6, c = e & 63;
    g[m * ld + c] = s[c * FLD + m];
  }
}

// ---- tile math ---------------------------------------------------------------

// one float64 tensor-core product (mma.m8n8k4: A 8x4 row-major — lane l holds
// A[l / 4][l % 4]; B 4x8 column-major — B[l % 4][l / 4]; C 8x8 — C[l / 4][2 (l % 4) + i])
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// out = At^T B (MODE 0), C - At^T B (MODE 1) or C + At^T B (MODE 2); At[p][m],
// B[p][c] in smem (row stride FLD); C (ldc) read through L2 when CG, else
// from smem; out (ldo) may be smem or global.  On the float64 tensor cores
// (DMMA): warp w owns rows 32 (w & 1) .. +31 and columns 16 (w >> 1) .. +15 as
// 4 x 2 fragments of 8 x 8; per k-step of 4 it loads 4 A and 2 B fragment
// values (FLD = 4 mod 16 keeps both loads bank-conflict free) for 8 DMMAs.
// SHAPE 1: At is upper triangular, so row block i stops at k = its last row
// (the skipped products are exact zeros); SHAPE 2: only the fragments that
// hold upper-triangle entries of the (symmetric) result are formed.
template <int MODE, bool CG, int SHAPE = 0>
__device__ __forceinline__ void gemm_tile(const double* At, const double* B, const double* C, int64_t ldc, double* out,
                                          int64_t ldo) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rb = (w & 1) * 32, cb = (w >> 1) * 16;
  const int qr = lane >> 2, qc = lane & 3;
  auto need = [&](int i, int j) { return SHAPE != 2 || cb + 8 * j + 7 >= rb + 8 * i; };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      acc[i][j][0] = acc[i][j][1] = 0.0;
      if (MODE != 0 && need(i, j)) {
        const double* cp = C + (rb + 8 * i + qr) * ldc + cb + 8 * j + 2 * qc;
        const double2 v = CG ? __ldcg(reinterpret_cast<const double2*>(cp)) : *reinterpret_cast<const double2*>(cp);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      }
    }
  const double sg = MODE == 1 ? -1.0 : 1.0;
  const int kend = SHAPE == 1 ? rb + 32 : FT;
#pragma unroll 4
  for (int k0 = 0; k0 < kend; k0 += 4) {
    const double* ar = At + (k0 + qc) * FLD + rb + qr;
    const double* br = B + (k0 + qc) * FLD + cb + qr;
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sg * ar[8 * i];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = br[8 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (need(i, j) && (SHAPE != 1 || k0 <= rb + 8 * i + 7)) dmma(acc[i][j], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (need(i, j))
        *reinterpret_cast<double2*>(out + (rb + 8 * i + qr) * ldo + cb + 8 * j + 2 * qc) =
            make_double2(acc[i][j][0], acc[i][j][1]);
}

// fixed-order sum of squares of the valid (rows < nr, cols < nc) entries of a
// smem tile (TRANS: entry (m, c) read as s[c][m]); result on thread 0
template <bool TRANS>
__device__ double tile_sumsq(const double* s, int nr, int nc, double* red) {
  double ss = 0.0;
  for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
    const int m = e >> 6, c = e & 63;
    if (m < nr && c < nc) {
      const double v = TRANS ? s[c * FLD + m] : s[m * FLD + c];
      ss = fma(v, v, ss);
    }
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xFFFFFFFFu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < FTHREADS / 32; ++w) t += red[w];
  __syncthreads();
  return t;
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

// ---- tiles -------------------------------------------------------------------

__device__ __forceinline__ double* atile(const FactorArgs& a, int k, int l) {
  return a.A + static_cast<int64_t>(k) * FT * a.dp + static_cast<int64_t>(l) * FT;
}
__device__ __forceinline__ double* wtile(const FactorArgs& a, int k, int m) {
  return a.W + static_cast<int64_t>(k) * FT * a.dp + static_cast<int64_t>(m) * FT;
}
__device__ __forceinline__ double* ttile(const FactorArgs& a, int j) { return a.T + static_cast<int64_t>(j) * FT * FT; }
__device__ __forceinline__ double* ptile(const FactorArgs& a, int k, int c) {
  return a.P + static_cast<int64_t>(k) * FT * a.rp + static_cast<int64_t>(c) * FT;
}
__device__ __forceinline__ double* mtile(const FactorArgs& a, int i, int c) {
  return a.Ma + static_cast<int64_t>(i) * FT * a.rp + static_cast<int64_t>(c) * FT;
}

__device__ __forceinline__ void kf_stamp(const FactorArgs& a, int slot) {
  if (a.trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[slot] = t;
  }
}

enum : int { T_PANEL = 0, T_YROW = 1, T_UPD = 2, T_WUPD = 3, T_MACC = 4, T_FINAL = 5, T_NONE = 6, T_YDIAG = 7 };

// queue task t -> (type, j, x, y); per step j: YDIAG(j), PANEL(j, k >= j+2), YROW(j, m < j),
// UPD(j; k <= l) without (j+1, j+1) — row j+1 first, WUPD(j; k, m <= j) — row
// j+1 first, MACC(j; i <= j, c); then FINAL.  UPD and WUPD come in row
// segments of up to KF_SEG consecutive tiles that share the left operand U_jk
// (one load of U_jk and one queue pull per segment; each tile still publishes
// its own version): x = type | count << 4, (y, z, w) = (j, k, first l or m).
constexpr int KF_SEG = 4;

// sum_{c=1..n} ceil(c / KF_SEG)
__host__ __device__ inline int kf_seg_sum(int n) {
  if (n <= 0) return 0;
  const int q = n / KF_SEG, r = n % KF_SEG;
  return KF_SEG * q * (q + 1) / 2 + r * (q + 1);
}

__host__ __device__ inline int4 kf_decode(int t, int nb, int rt) {
  for (int j = 0; j < nb; ++j) {
    const int m = nb - j - 1;
    const int np = m > 1 ? m - 1 : 0;
    const int ny = j;
    // UPD rows: row j+1 has m - 1 tiles (l = j+2..), row j+1+kk (kk >= 1) has m - kk
    const int nu = m >= 1 ? (m - 1 + KF_SEG - 1) / KF_SEG + kf_seg_sum(m - 1) : 0;
    const int wseg = (j + 1 + KF_SEG - 1) / KF_SEG;
    const int nw = m * wseg;
    const int nm = (j + 1) * rt;
    if (t == 0) return make_int4(T_YDIAG, j, 0, 0);
    t -= 1;
    if (t < np) return make_int4(T_PANEL, j, j + 2 + t, 0);
    t -= np;
    if (t < ny) return make_int4(T_YROW, j, t, 0);
    t -= ny;
    if (t < nu) {
      for (int kk = 0; kk < m; ++kk) {
        const int l0 = kk == 0 ? j + 2 : j + 1 + kk;
        const int cnt = nb - l0;
        const int ns = (cnt + KF_SEG - 1) / KF_SEG;
        if (t < ns) {
          const int first = l0 + t * KF_SEG;
          const int c = nb - first < KF_SEG ? nb - first : KF_SEG;
          return make_int4(T_UPD | (c << 4), j, j + 1 + kk, first);
        }
        t -= ns;
      }
    }
    t -= nu;
    if (t < nw) {
      const int first = (t % wseg) * KF_SEG;
      const int c = j + 1 - first < KF_SEG ? j + 1 - first : KF_SEG;
      return make_int4(T_WUPD | (c << 4), j, j + 1 + t / wseg, first);
    }
    t -= nw;
    if (t < nm) return make_int4(T_MACC, j, t / rt, t % rt);
    t -= nm;
  }
  return make_int4(t == 0 ? T_FINAL : T_NONE, 0, 0, 0);
}

static int kf_queue_tasks(int nb, int rt) {
  int n = 0;
  for (int j = 0; j < nb; ++j) {
    const int m = nb - j - 1;
    const int nu = m >= 1 ? (m - 1 + KF_SEG - 1) / KF_SEG + kf_seg_sum(m - 1) : 0;
    n += 1 + (m > 1 ? m - 1 : 0) + j + nu + m * ((j + 1 + KF_SEG - 1) / KF_SEG) + (j + 1) * rt;
  }
  return n + 1;
}

// T_j (smem t) -> global; publish.  U_jj itself is never read again, and
// Y_jj = T_j^T with its trace share is a queue task (YDIAG), off the chain.
__device__ __forceinline__ void finish_diag(const FactorArgs& a, int j, const double* t) {
  store_tile(ttile(a, j), FT, t);
  signal(a.verA + j * a.nb + j, j + 1);
}

// NT = 4 smem tiles, one CTA per SM (d <= 1024: the chain is the critical
// path and keeps its next diagonal tile loaded ahead); NT = 3, two CTAs per
// SM (large d: the queue's tile updates are the bound, and a second CTA per SM
// overlaps one CTA's tile loads and dependency waits with the other's DMMAs;
// the chain then loads its diagonal tile after the panel product).
template <int NT>
__global__ void __launch_bounds__(FTHREADS, NT == 3 ? 2 : 1) chol_fold_kernel(FactorArgs a) {
  extern __shared__ double fsm[];
  double* b0 = fsm;
  double* b1 = fsm + FT * FLD;
  double* b2 = fsm + 2 * FT * FLD;
  double* b3 = NT == 4 ? fsm + 3 * FT * FLD : nullptr;
  double* scratch = fsm + NT * FT * FLD;  // 5 x 64 doubles (chol_inv_tile)
  double* red = scratch + 5 * FT;        // 8 doubles
  __shared__ int4 s_task;
  cg::grid_group grid = cg::this_grid();
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int nb = a.nb, rt = a.rt;
  const int64_t dp = a.dp, rp = a.rp;

  // phase 0: working copies (padding: identity on the diagonal), flags; one warp per row
  {
    const int wid = (cta * FTHREADS + threadIdx.x) >> 5, nw = (ncta * FTHREADS) >> 5, lane = threadIdx.x & 31;
    for (int64_t m = wid; m < 3 * dp; m += nw) {
      if (m < dp) {
        double* row = a.A + m * dp;
        for (int64_t c = lane; c < dp; c += 32)
          row[c] = (m < a.d && c < a.d) ? (m <= c ? a.G[m * a.ldg + c] : 0.0) : (m == c ? 1.0 : 0.0);
      } else if (m < 2 * dp) {
        double* row = a.W + (m - dp) * dp;
        for (int64_t c = lane; c < dp; c += 32) row[c] = 0.0;
      } else {
        const int64_t mm = m - 2 * dp;
        double* row = a.P + mm * rp;
        for (int64_t c = lane; c < rp; c += 32) row[c] = (mm < a.d && c < a.r) ? a.Pi[mm * a.r + c] : 0.0;
      }
    }
    const int gt = cta * FTHREADS + threadIdx.x, gn = ncta * FTHREADS;
    for (int i = gt; i < nb * nb; i += gn) {
      a.verA[i] = 0;
      a.verW[i] = 0;
    }
    for (int i = gt; i < nb * rt; i += gn) a.verM[i] = 0;
    if (gt < 3) a.ctl[gt] = 0;
    if (cta == 0 && threadIdx.x == 0) {  // the chain CTA's SM (read after the grid barrier)
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      a.ctl[3] = static_cast<int32_t>(sm);
    }
    if (cta == 0 && threadIdx.x < 32) {
      // trace(G) in a fixed order (one warp, then lane 0)
      double t = 0.0;
      for (int64_t i = threadIdx.x; i < a.d; i += 32) t += a.G[i * a.ldg + i];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, o);
      if (threadIdx.x == 0) a.diag[1] = t;
    }
  }
  grid.sync();

  if (cta == 0 && NT == 4) {
    // ---- the critical chain: DIAG(0), then CHAIN(1..nb-1), T_j kept in smem
    double *T = b0, *x = b1, *y = b2, *z = b3;
    kf_stamp(a, 0);
    load_tile(y, atile(a, 0, 0), dp);
    __syncthreads();
    chol_inv_tile(y, T, scratch, a.ctl + 2);
    finish_diag(a, 0, T);
    kf_stamp(a, 1);
    for (int j = 0; j + 1 < nb; ++j) {
      wait_ge(a.verA + j * nb + j + 1, j);
      wait_ge(a.verA + (j + 1) * nb + j + 1, j);
      __syncthreads();
      kf_stamp(a, 2 + 3 * j);
      load_tile(x, atile(a, j, j + 1), dp);
      load_tile(y, atile(a, j + 1, j + 1), dp);
      __syncthreads();
      kf_stamp(a, 600 + 4 * j);
      gemm_tile<0, false, 1>(T, x, nullptr, 0, z, FLD);  // U_j,j+1 = T_j^T A_j,j+1 (T_j upper)
      __syncthreads();
      kf_stamp(a, 601 + 4 * j);
      store_tile(atile(a, j, j + 1), dp, z);
      signal(a.verA + j * nb + j + 1, j + 1);
      kf_stamp(a, 602 + 4 * j);
      gemm_tile<1, false, 2>(z, z, y, FLD, x, FLD);  // A_j+1,j+1 - U^T U (upper triangle)
      __syncthreads();
      kf_stamp(a, 3 + 3 * j);
      chol_inv_tile(x, y, scratch, a.ctl + 2);  // x = U_j+1,j+1, y = T_j+1
      finish_diag(a, j + 1, y);
      kf_stamp(a, 4 + 3 * j);
      double* freed = T;
      T = y;
      y = freed;
    }
    return;
  }
  if (cta == 0 && NT == 3) {
    // ---- the chain in three tiles: T_j, the panel / diagonal tile, U_j,j+1
    double *T = b0, *x = b1, *z = b2;
    kf_stamp(a, 0);
    load_tile(x, atile(a, 0, 0), dp);
    __syncthreads();
    chol_inv_tile(x, T, scratch, a.ctl + 2);
    finish_diag(a, 0, T);
    kf_stamp(a, 1);
    for (int j = 0; j + 1 < nb; ++j) {
      wait_ge(a.verA + j * nb + j + 1, j);
      wait_ge(a.verA + (j + 1) * nb + j + 1, j);
      __syncthreads();
      kf_stamp(a, 2 + 3 * j);
      load_tile(x, atile(a, j, j + 1), dp);
      __syncthreads();
      kf_stamp(a, 600 + 4 * j);
      gemm_tile<0, false, 1>(T, x, nullptr, 0, z, FLD);  // U_j,j+1 = T_j^T A_j,j+1
      __syncthreads();
      kf_stamp(a, 601 + 4 * j);
      store_tile(atile(a, j, j + 1), dp, z);
      load_tile(x, atile(a, j + 1, j + 1), dp);
      signal(a.verA + j * nb + j + 1, j + 1);  // (its __syncthreads also orders the load)
      kf_stamp(a, 602 + 4 * j);
      gemm_tile<1, false, 2>(z, z, x, FLD, x, FLD);  // in place (each thread owns its C fragment)
      __syncthreads();
      kf_stamp(a, 3 + 3 * j);
      chol_inv_tile(x, z, scratch, a.ctl + 2);  // x = U_j+1,j+1, z = T_j+1
      finish_diag(a, j + 1, z);
      kf_stamp(a, 4 + 3 * j);
      double* freed = T;
      T = z;
      z = freed;
    }
    return;
  }

  // ---- everything else from the queue, in topological order.  Two CTAs per
  // SM (NT = 3): the queue CTA that shares the chain CTA's SM leaves, so the
  // latency-bound chain (its 64-pivot eliminations, DFMA on the same fp64
  // pipe as the queue's DMMA) has the SM to itself — chol_inv 30-43 us per
  // tile beside a queue CTA vs 12.5 us alone (LVSK_KF_TRACE at d = 4096)
  if (NT == 3) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if (static_cast<int32_t>(sm) == __ldcg(a.ctl + 3)) return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_task = kf_decode(atomicAdd(a.ctl, 1), nb, rt);
    __syncthreads();
    const int4 tk = s_task;
    __syncthreads();
    if (tk.x == T_NONE) break;
    const int j = tk.y;
    if (tk.x == T_YDIAG) {  // Y_jj = T_j^T and its share of trace(G^-1)
      wait_ge(a.verA + j * nb + j, j + 1);
      __syncthreads();
      load_tile(b0, ttile(a, j), FT);
      __syncthreads();
      store_tile_t(wtile(a, j, j), dp, b0);
      const int nv = static_cast<int>(a.d - static_cast<int64_t>(j) * FT);
      const double ss = tile_sumsq<true>(b0, nv, nv, red);
      if (threadIdx.x == 0) a.partial[j * nb + j] = ss;
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(a.verW + j * nb + j, 1);
        atomicAdd(a.ctl + 1, 1);
      }
    } else if (tk.x == T_PANEL) {  // U_jk = T_j^T A_jk
      const int k = tk.z;
      wait_ge(a.verA + j * nb + j, j + 1);
      wait_ge(a.verA + j * nb + k, j);
      __syncthreads();
      load_tile(b0, ttile(a, j), FT);
      load_tile(b1, atile(a, j, k), dp);
      __syncthreads();
      gemm_tile<0, false, 1>(b0, b1, nullptr, 0, atile(a, j, k), dp);
      signal(a.verA + j * nb + k, j + 1);
    } else if (tk.x == T_YROW) {  // Y_jm = T_j^T W_jm
      const int m = tk.z;
      wait_ge(a.verA + j * nb + j, j + 1);
      wait_ge(a.verW + j * nb + m, j - m);
      __syncthreads();
      load_tile(b0, ttile(a, j), FT);
      load_tile(b1, wtile(a, j, m), dp);
      __syncthreads();
      gemm_tile<0, false, 1>(b0, b1, nullptr, 0, b2, FLD);
      __syncthreads();
      store_tile(wtile(a, j, m), dp, b2);
      const double ss = tile_sumsq<false>(b2, static_cast<int>(a.d - static_cast<int64_t>(j) * FT),
                                          static_cast<int>(a.d - static_cast<int64_t>(m) * FT), red);
      if (threadIdx.x == 0) a.partial[j * nb + m] = ss;
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(a.verW + j * nb + m, j - m + 1);
        atomicAdd(a.ctl + 1, 1);
      }
    } else if ((tk.x & 15) == T_UPD) {  // A_kl -= U_jk^T U_jl, l = w .. w + count - 1
      const int k = tk.z, cnt = tk.x >> 4;
      wait_ge(a.verA + j * nb + k, j + 1);
      __syncthreads();
      load_tile(b0, atile(a, j, k), dp);
      for (int q = 0; q < cnt; ++q) {
        const int l = tk.w + q;
        wait_ge(a.verA + j * nb + l, j + 1);
        wait_ge(a.verA + k * nb + l, j);
        __syncthreads();  // also: the previous tile's gemm is done with b1
        if (l != k) load_tile(b1, atile(a, j, l), dp);
        __syncthreads();
        if (l != k)
          gemm_tile<1, true>(b0, b1, atile(a, k, l), dp, atile(a, k, l), dp);
        else  // diagonal tile: only its upper triangle is ever read
          gemm_tile<1, true, 2>(b0, b0, atile(a, k, l), dp, atile(a, k, l), dp);
        signal(a.verA + k * nb + l, j + 1);
      }
    } else if ((tk.x & 15) == T_WUPD) {  // W_km -= U_jk^T Y_jm, m = w .. w + count - 1
      const int k = tk.z, cnt = tk.x >> 4;
      wait_ge(a.verA + j * nb + k, j + 1);
      __syncthreads();
      load_tile(b0, atile(a, j, k), dp);
      for (int q = 0; q < cnt; ++q) {
        const int m = tk.w + q;
        wait_ge(a.verW + j * nb + m, j - m + 1);
        wait_ge(a.verW + k * nb + m, j - m);
        __syncthreads();
        load_tile(b1, wtile(a, j, m), dp);
        __syncthreads();
        gemm_tile<1, true>(b0, b1, wtile(a, k, m), dp, wtile(a, k, m), dp);
        signal(a.verW + k * nb + m, j - m + 1);
      }
    } else if (tk.x == T_MACC) {  // M_ic += Y_ji^T Pi_jc
      const int i = tk.z, c = tk.w;
      wait_ge(a.verW + j * nb + i, j - i + 1);
      wait_ge(a.verM + i * rt + c, j - i);
      __syncthreads();
      load_tile(b0, wtile(a, j, i), dp);
      load_tile(b1, ptile(a, j, c), rp);
      __syncthreads();
      if (j + 1 < nb) {
        if (j == i)
          gemm_tile<0, false>(b0, b1, nullptr, 0, mtile(a, i, c), rp);
        else
          gemm_tile<2, true>(b0, b1, mtile(a, i, c), rp, mtile(a, i, c), rp);
        signal(a.verM + i * rt + c, j - i + 1);
      } else {
        if (j == i)
          gemm_tile<0, false>(b0, b1, nullptr, 0, b2, FLD);
        else
          gemm_tile<2, true>(b0, b1, mtile(a, i, c), rp, b2, FLD);
        __syncthreads();
        for (int e = threadIdx.x; e < FT * FT; e += FTHREADS) {
          const int64_t row = static_cast<int64_t>(i) * FT + (e >> 6);
          const int64_t col = static_cast<int64_t>(c) * FT + (e & 63);
          if (row < a.d && col < a.r) a.M[row * a.r + col] = b2[(e >> 6) * FLD + (e & 63)];
        }
        __syncthreads();
      }
    } else {  // FINAL: trace(G^-1) = ||Y||_F^2 in a fixed order, info
      if (threadIdx.x == 0) {
        while (ld_acquire(a.ctl + 1) < nb * (nb + 1) / 2) __nanosleep(64);
        double tr = 0.0;
        for (int k = 0; k < nb; ++k)
          for (int m = 0; m <= k; ++m) tr += a.partial[k * nb + m];
        a.diag[2] = tr;
        const int32_t info = ld_acquire(a.ctl + 2);
        a.diag[0] = static_cast<double>(info);
        // trace(G) was written before the grid barrier of phase 0
        const double trg = a.diag[1];
        const bool ok = info == 0 && isfinite(trg) && isfinite(tr) && trg > 0.0 && tr > 0.0 && trg * tr < a.cert_limit;
        if (!ok && a.cert_fail != nullptr) atomicAdd(a.cert_fail, 1);
      }
      __syncthreads();
    }
  }
}

struct FactorPlan {
  int nb, rt;
  int64_t dp, rp;
};

static FactorPlan plan_factor(int64_t d, int64_t r) {
  FactorPlan p;
  p.nb = static_cast<int>((d + FT - 1) / FT);
  p.rt = static_cast<int>((r + FT - 1) / FT);
  p.dp = static_cast<int64_t>(p.nb) * FT;
  p.rp = static_cast<int64_t>(p.rt) * FT;
  return p;
}

template <typename Alloc>
static void kf_layout(Alloc& c, const FactorPlan& P, FactorArgs* a) {
  const size_t nb2 = static_cast<size_t>(P.nb) * P.nb;
  auto A = c.template take<double>(static_cast<size_t>(P.dp) * P.dp);
  auto W = c.template take<double>(static_cast<size_t>(P.dp) * P.dp);
  auto T = c.template take<double>(static_cast<size_t>(P.nb) * FT * FT);
  auto Pp = c.template take<double>(static_cast<size_t>(P.dp) * P.rp);
  auto Ma = c.template take<double>(static_cast<size_t>(P.dp) * P.rp);
  auto part = c.template take<double>(nb2);
  auto vA = c.template take<int32_t>(nb2);
  auto vW = c.template take<int32_t>(nb2);
  auto vM = c.template take<int32_t>(static_cast<size_t>(P.nb) * P.rt);
  auto ctl = c.template take<int32_t>(4);
  if (a) {
    a->A = A;
    a->W = W;
    a->T = T;
    a->P = Pp;
    a->Ma = Ma;
    a->partial = part;
    a->verA = vA;
    a->verW = vW;
    a->verM = vM;
    a->ctl = ctl;
  }
}

// Measure::take returns void; a typed twin so kf_layout serves both
struct MeasureT {
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    off += count * sizeof(T);
    return nullptr;
  }
};

}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_chol_fold_workspace_bytes(int64_t d, int64_t r) {
  if (d < 1 || r < 1) return 0;
  const FactorPlan P = plan_factor(d, r);
  MeasureT ms;
  kf_layout(ms, P, nullptr);
  return ms.off;
}

extern "C" int32_t lvsk_chol_fold(const double* G, int64_t d, int64_t ldg, const double* Pi, int64_t r, double* M,
                                  double* diag, double cert_limit, int32_t* cert_fail, void* ws, size_t ws_bytes,
                                  void* stream) {
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
  a.cert_limit = cert_limit;
  a.cert_fail = cert_fail;
  kf_layout(c, P, &a);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  a.nb = P.nb;
  a.rt = P.rt;
  a.dp = P.dp;
  a.rp = P.rp;
  // large d: three-tile CTAs, two per SM (the queue's tile updates dominate)
  const bool wide = P.nb > 16;
  const void* fn = wide ? reinterpret_cast<const void*>(chol_fold_kernel<3>) : reinterpret_cast<const void*>(chol_fold_kernel<4>);
  const int smem = (wide ? 3 : 4) * FTILE_SMEM + (5 * FT + 8) * 8;
  const int32_t arc = ensure_smem_attr(fn, smem, "chol_fold smem attribute");
  if (arc != LVSK_OK) return arc;
  const int per_sm = resident_ctas(fn, FTHREADS, smem);
  const int grid_cap = per_sm >= 1 ? num_sms() * (wide && per_sm >= 2 ? 2 : 1) : 0;
  if (grid_cap < 2) return cuda_status(cudaErrorInvalidConfiguration, "chol_fold needs two co-resident CTAs");
  // CTA 0 runs the chain; more queue CTAs than tasks only add polling
  const int ntask = kf_queue_tasks(P.nb, P.rt);
  int grid = 1 + (ntask < grid_cap - 1 ? ntask : grid_cap - 1);
  // passes in flight on other streams (lvsk_set_inflight): at d <= 1024 the
  // chain, not the queue, bounds KF, and 24 CTAs keep its pace (C2: +14 us
  // alone) while the other SMs run the concurrent pass's HBM-bound kernels
  if (inflight_passes() >= 2 && !wide && grid > KF_INFLIGHT_GRID) grid = KF_INFLIGHT_GRID;
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
  cudaError_t e = wide ? cudaLaunchKernelEx(&cfg, chol_fold_kernel<3>, a) : cudaLaunchKernelEx(&cfg, chol_fold_kernel<4>, a);
  if (e != cudaSuccess) return cuda_status(e, "chol_fold launch");
  if (tracing) {
    unsigned long long h[1024];
    const int nst = P.nb < 300 ? P.nb : 300;
    cudaStreamSynchronize(cfg.stream);
    cudaMemcpy(h, trace, (2 + 3 * nst) * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    fprintf(stderr, "KF d=%lld r=%lld grid=%d tasks=%d diag0 %.1f us; chain wait/gemm/chol_inv (us):", (long long)d,
            (long long)r, grid, ntask, (h[1] - h[0]) / 1000.0);
    unsigned long long prev = h[1];
    for (int j = 0; j + 1 < nst && j < 16; ++j) {
      fprintf(stderr, " %.1f/%.1f/%.1f", (h[2 + 3 * j] - prev) / 1000.0, (h[3 + 3 * j] - h[2 + 3 * j]) / 1000.0,
              (h[4 + 3 * j] - h[3 + 3 * j]) / 1000.0);
      prev = h[4 + 3 * j];
    }
    fprintf(stderr, "\n  load/gemm1/store+signal/gemm2 (us):");
    cudaMemcpy(h + 600, trace + 600, 4 * 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    for (int j = 0; j + 1 < nst && j < 8; ++j)
      fprintf(stderr, " %.1f/%.1f/%.1f/%.1f", (h[600 + 4 * j] - h[2 + 3 * j]) / 1000.0,
              (h[601 + 4 * j] - h[600 + 4 * j]) / 1000.0, (h[602 + 4 * j] - h[601 + 4 * j]) / 1000.0,
              (h[3 + 3 * j] - h[602 + 4 * j]) / 1000.0);
    fprintf(stderr, "\n");
  }
  return LVSK_OK;
}
