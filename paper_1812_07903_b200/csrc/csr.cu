// K2 / K6 — the hashed sketch and the leverage pass on CSR rows (BASELINE
// config 4: OSNAP on a bag-of-words-like CSR matrix).  Extension G2: the
// reference only takes dense rows (matrix.py:30-39); its semantics on a CSR
// matrix are those of consume_rows on the densified rows (sketch.py:289-312),
// which these kernels reproduce exactly: a zero entry contributes +-0 to a
// TwoSum and leaves (hi, lo) unchanged, so skipping it is bit-exact.
//
// K2: rows are grouped by bucket with the same keygen + stable radix sort as
// K1; one warp owns one (bucket, 1024-column group) and keeps its float64
// (hi, lo) slice in shared memory (16 KB), walking the bucket's rows in
// ascending index and applying each nonzero of its column range as a TwoSum
// (canonical CSR: strictly increasing columns inside a row, so the lanes of a
// warp never touch the same column within a row).
// K6: one warp per row; lane l owns r/32 consecutive columns of u = x M and
// gathers the M rows of the row's nonzeros (L1/L2-resident), fp32 FMA, then
// the squared norm is reduced across the warp.
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <cstring>

#include "radix_sort.cuh"

namespace lvsk {

constexpr int CSR_GROUP = 1024;  // columns per warp-owned SX slice (16 KB of hi/lo)
constexpr int CSR_WARPS = 4;

struct CsrBlocks {
  uint64_t a[64], b[64], key[64];
  uint32_t offset[64], size[64];
};

__global__ void csr_keygen_kernel(int64_t n, uint64_t row0, int j0, int nb, CsrBlocks P, uint32_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals) {
  const int64_t total = n * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int jj = static_cast<int>(t / n);
    const int64_t r = t - static_cast<int64_t>(jj) * n;
    const uint64_t g = row0 + static_cast<uint64_t>(r);
    keys[static_cast<int64_t>(j0 + jj) * n + r] = P.offset[jj] + bucket_hash(g, P.a[jj], P.b[jj], P.size[jj]);
    vals[static_cast<int64_t>(j0 + jj) * n + r] =
        (static_cast<uint32_t>(r) << 1) | (sign_negative(g, P.key[jj]) ? 1u : 0u);
  }
}

template <typename V>
__global__ void __launch_bounds__(32 * CSR_WARPS) csr_gather_kernel(
    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const V* __restrict__ val, int64_t d,
    int ngroups, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ start, int64_t units, double scale,
    const double* hi_in, const double* lo_in, double* hi_out, double* lo_out, int32_t* flags) {
  extern __shared__ double csr_dyn[];  // [CSR_WARPS][2][CSR_GROUP]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = static_cast<int64_t>(blockIdx.x) * CSR_WARPS + warp;
  if (unit >= units) return;
  const int64_t b = unit / ngroups;
  const int64_t c0 = (unit - b * ngroups) * CSR_GROUP;
  const int64_t width = d - c0 < CSR_GROUP ? d - c0 : CSR_GROUP;
  double* hi = csr_dyn + static_cast<int64_t>(warp) * 2 * CSR_GROUP;
  double* lo = hi + CSR_GROUP;
  for (int64_t c = lane; c < width; c += 32) {
    hi[c] = hi_in ? hi_in[b * d + c0 + c] : 0.0;
    lo[c] = lo_in ? lo_in[b * d + c0 + c] : 0.0;
  }
  __syncwarp();
  const int64_t base0 = row_ptr[0];
  const uint32_t p0 = start[b], p1 = start[b + 1];
  int bad = 0;
  for (uint32_t p = p0; p < p1; ++p) {
    const uint32_t vv = vals[p];
    const int64_t r = vv >> 1;
    const double sg = (vv & 1u) ? -scale : scale;
    const int64_t e0 = row_ptr[r] - base0, e1 = row_ptr[r + 1] - base0;
    int32_t prev_last = -1;
    for (int64_t e = e0; e < e1; e += 32) {
      const int64_t ei = e + lane;
      const bool live = ei < e1;
      const int32_t c = live ? col[ei] : INT32_MAX;
      const double x = live ? static_cast<double>(val[ei]) : 0.0;
      // canonical CSR check: strictly increasing columns in range
      const int32_t cprev = __shfl_up_sync(0xFFFFFFFFu, c, 1);
      const int32_t before = lane == 0 ? prev_last : cprev;
      if (live) {
        if (c < 0 || c >= d) bad |= LVSK_FLAG_BADINDEX;
        else if (c <= before) bad |= LVSK_FLAG_BADINDEX;
        if (!isfinite(x)) bad |= LVSK_FLAG_NONFINITE;
      }
      prev_last = __shfl_sync(0xFFFFFFFFu, c, 31);
      const int64_t lc = static_cast<int64_t>(c) - c0;
      if (live && lc >= 0 && lc < width) {
        double s, er;
        two_sum(hi[lc], __dmul_rn(sg, x), s, er);
        hi[lc] = s;
        lo[lc] = __dadd_rn(lo[lc], er);
      }
    }
    __syncwarp();
  }
  for (int64_t c = lane; c < width; c += 32) {
    if (lo_out) {
      hi_out[b * d + c0 + c] = hi[c];
      lo_out[b * d + c0 + c] = lo[c];
    } else {  // the folded sketch hi + lo (lvsk_fold_compensated's value)
      hi_out[b * d + c0 + c] = hi[c] + lo[c];
    }
  }
  const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (any && lane == 0) atomicOr(flags, any);
}

// ---------------------------------------------------------------------------
// csr_prep_kernel turns the bucket-sorted (row, sign) pairs into per-pair
// (source offset, length) so the sketch kernel never chases row pointers.
constexpr int ST_COLS = 4096;  // columns per CTA-owned SX slice (one 32 KB float64 partial row per warp)

__device__ __forceinline__ uint32_t csr_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void csr_prep_kernel(const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ svals, int64_t N,
                                int64_t* __restrict__ msrc, int32_t* __restrict__ mlen) {
  const int64_t base0 = row_ptr[0];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = svals[i] >> 1;
    const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
    msrc[i] = e0 - base0;
    mlen[i] = static_cast<int32_t>(e1 - e0);
  }
}

// ---------------------------------------------------------------------------
// K2 v4 (default): self-loading applier warps.  One CTA owns one (bucket,
// <= 4096-column group); each of its W warps owns a private float64 partial
// row (32 KB) and a private ring of NB batches of 8 row slots, and takes the
// bucket's pairs p0 + w, p0 + w + W, ... in ascending order.  Copy: four
// lanes per row copy the 16-byte aligned supersets of the row's columns and
// values into its slot with cp.async (LDGSTS.128; a batch is one commit
// group, NB - 1 batches in flight per warp; rows longer than a slot are read
// straight from global memory when their turn comes).  Apply: the row's
// entries are striped over the lanes; one row's columns are distinct, so the
// plain float64 load-add-stores never collide.  No loader warp and no
// cross-warp hand-off: round 2's design (one loader warp feeding two applier
// warps through mbarrier stages) kept its appliers waiting; the partial rows
// cap a CTA at five warps, so the per-row instruction count and the overlap
// of consecutive rows are what set the speed (ncu: ~25 % issue-active, memory
// system ~25 % busy).  The CTA ends with the TwoSum fold of (hi_in, lo_in,
// P_0 .. P_W-1) in warp order: deterministic.
constexpr int K2_SLOT_DEFAULT = 124;  // ring slot capacity in entries (rows of up to 118 entries are staged)
constexpr int K2_BATCH = 8;   // rows per copy batch (4 lanes per row)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(csr_smem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int k2_smem_bytes(int w, int nb, int vsz, int slot = K2_SLOT_DEFAULT) {
  return w * (ST_COLS * 8 + nb * K2_BATCH * slot * (4 + vsz) + nb * K2_BATCH * 24);
}

template <typename V, int W, int NB, bool POW2, bool ONEG, int K2_SLOT = K2_SLOT_DEFAULT>
__global__ void __launch_bounds__(32 * W) csr_sketch_kernel(
    const int32_t* __restrict__ col, const V* __restrict__ val, int64_t d, int ngroups,
    const uint32_t* __restrict__ svals, const int64_t* __restrict__ msrc, const int32_t* __restrict__ mlen,
    const uint32_t* __restrict__ start, double scale, const double* hi_in, const double* lo_in,
    double* hi_out, double* lo_out, int32_t* flags, int64_t validate_below) {
  extern __shared__ __align__(128) uint8_t k2_smem[];
  constexpr int VPC = 16 / sizeof(V);  // values per 16-byte chunk
  constexpr int RS = NB * K2_BATCH;    // row slots per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbase = k2_smem + warp * (ST_COLS * 8 + RS * K2_SLOT * (4 + sizeof(V)) + RS * 24);
  double* mine = reinterpret_cast<double*>(wbase);                              // [ST_COLS]
  int32_t* cr = reinterpret_cast<int32_t*>(mine + ST_COLS);                     // [RS][K2_SLOT]
  V* vr = reinterpret_cast<V*>(cr + RS * K2_SLOT);                              // [RS][K2_SLOT]
  int4* mt = reinterpret_cast<int4*>(vr + RS * K2_SLOT);                        // [RS]
  int64_t* ds = reinterpret_cast<int64_t*>(mt + RS);                            // [RS] (direct rows)
  const int64_t b = blockIdx.x / ngroups;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x - b * ngroups) * ST_COLS;
  const int width = static_cast<int>(d - c0 < ST_COLS ? d - c0 : ST_COLS);
  for (int c = 2 * lane; c < ST_COLS; c += 64) *reinterpret_cast<double2*>(mine + c) = make_double2(0.0, 0.0);

  const uint32_t p0 = start[b], p1 = start[b + 1];
  const int cnt = static_cast<int>(p1 - p0) > warp ? (static_cast<int>(p1 - p0) - warp + W - 1) / W : 0;
  const int nbat = (cnt + K2_BATCH - 1) / K2_BATCH;
  // metadata of my rows, 32 at a time (lane l: row base + l), one block ahead
  int64_t bsrc = 0, nsrc = 0;
  int32_t blen = 0, nlen = 0;
  uint32_t bsv = 0, nsv = 0;
  auto fetch = [&](int base, int64_t& s_, int32_t& l_, uint32_t& v_) {
    l_ = 0;
    if (base + lane < cnt) {
      const uint32_t q = p0 + warp + static_cast<uint32_t>(W) * static_cast<uint32_t>(base + lane);
      s_ = msrc[q];
      l_ = mlen[q];
      v_ = svals[q];
    }
  };
  fetch(0, bsrc, blen, bsv);
  fetch(32, nsrc, nlen, nsv);
  const int rr = lane >> 2, sub = lane & 3;  // copy: row of the batch, chunk phase
  auto produce = [&](int t) {
    if (t < nbat) {
      const int i0 = t * K2_BATCH;  // first row of the batch (a multiple of 8)
      if ((i0 & 31) == 0 && i0 > 0) {
        bsrc = nsrc;
        blen = nlen;
        bsv = nsv;
        fetch(i0 + 32, nsrc, nlen, nsv);
      }
      const int ml = (i0 & 31) + rr;
      const int64_t src = __shfl_sync(0xFFFFFFFFu, bsrc, ml);
      const int32_t len = __shfl_sync(0xFFFFFFFFu, blen, ml);
      const uint32_t sv = __shfl_sync(0xFFFFFFFFu, bsv, ml);
      const int slot = (t % NB) * K2_BATCH + rr;
      const uintptr_t ca = reinterpret_cast<uintptr_t>(col + src), va = reinterpret_cast<uintptr_t>(val + src);
      const int padc = static_cast<int>((ca & 15) >> 2), padv = static_cast<int>((va & 15) / sizeof(V));
      const int nchc = (padc + len + 3) >> 2, nchv = (padv + len + VPC - 1) / VPC;
      const bool direct = 4 * nchc > K2_SLOT || VPC * nchv > K2_SLOT;
      if (!direct && len > 0) {
        const char* gc = reinterpret_cast<const char*>(ca & ~uintptr_t{15});
        const char* gv = reinterpret_cast<const char*>(va & ~uintptr_t{15});
        int32_t* dc = cr + slot * K2_SLOT;
        V* dv = vr + slot * K2_SLOT;
        const int nch = nchc > nchv ? nchc : nchv;
        for (int ch = sub; ch < nch; ch += 4) {
          if (ch < nchc) cp_async16(dc + 4 * ch, gc + 16 * ch);
          if (ch < nchv) cp_async16(dv + VPC * ch, gv + 16 * ch);
        }
      }
      if (sub == 0) {
        mt[slot] = make_int4(padc, padv, len, static_cast<int>(sv & 1u) | (direct ? 2 : 0));
        ds[slot] = src;
      }
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int t = 0; t < NB - 1; ++t) produce(t);

  // one row: lane l takes entries l, l + 32, l + 64, l + 96 (entry e sits at
  // column slot padc + e and value slot padv + e); the next row's metadata is
  // read two rows ahead and its entries one row ahead, so the loads overlap
  // this row's read-add-store chain (shared accesses of one warp execute in
  // order, so the next row's partial loads see this row's stores).  32-bit
  // index math; one OSNAP column group (ONEG, d <= 4096) needs no range check
  // (a valid column is in range; an invalid one is masked into the partial
  // and flagged by block 0's checks); the sign (and a power-of-two scale,
  // applied in the fold) rides in one DFMA; only OSNAP block 0's buckets run
  // the checks (VALIDATE: every row meets block 0 exactly once).
  const int c0i = static_cast<int>(c0);
  auto rows = [&](auto vt) {
    constexpr bool VALIDATE = decltype(vt)::value;
    int bad = 0;
    int32_t carry = -1;
    auto apply4 = [&](const int32_t (&c)[4], const V (&x)[4], const int e0, const int len, const double sg) {
      if constexpr (VALIDATE) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool live = e0 + 32 * u + lane < len;
          const int32_t cprev = __shfl_up_sync(0xFFFFFFFFu, c[u], 1);
          const int32_t before = lane == 0 ? carry : cprev;
          carry = __shfl_sync(0xFFFFFFFFu, c[u], 31);
          if (live && (c[u] < 0 || c[u] >= d || c[u] <= before)) bad |= LVSK_FLAG_BADINDEX;
          if (live && !isfinite(static_cast<double>(x[u]))) bad |= LVSK_FLAG_NONFINITE;
        }
      }
      int lc[4];
      double xd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool live = e0 + 32 * u + lane < len;
        if constexpr (ONEG) {
          lc[u] = live ? (c[u] & (ST_COLS - 1)) : -1;
        } else {
          const int l = c[u] - c0i;
          lc[u] = (live && static_cast<unsigned>(l) < static_cast<unsigned>(width)) ? l : -1;
        }
        xd[u] = static_cast<double>(x[u]);
        if constexpr (!POW2) xd[u] = __dmul_rn(sg, xd[u]);
      }
      double old[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) old[u] = lc[u] >= 0 ? mine[lc[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (lc[u] >= 0) {
          if constexpr (POW2)
            mine[lc[u]] = fma(xd[u], sg, old[u]);  // sg = +-1: exact, = old +- x
          else
            mine[lc[u]] = __dadd_rn(old[u], xd[u]);
        }
      }
    };
    auto sgn_of = [&](const int4& m) { return POW2 ? ((m.w & 1) ? -1.0 : 1.0) : ((m.w & 1) ? -scale : scale); };
    auto load_row = [&](int slot, const int4& m, int32_t (&c)[4], V (&x)[4]) {
      const int32_t* cb = cr + slot * K2_SLOT + m.x;
      const V* vb = vr + slot * K2_SLOT + m.y;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = cb[32 * u + lane];  // slot reads past the row stay inside shared memory; masked by len
        x[u] = vb[32 * u + lane];
      }
    };
#pragma unroll 1
    for (int t = 0; t < nbat; ++t) {
      produce(t + NB - 1);
      cp_async_wait<NB - 1>();
      __syncwarp();
      const int base = (t % NB) * K2_BATCH;
      const int nr = cnt - t * K2_BATCH < K2_BATCH ? cnt - t * K2_BATCH : K2_BATCH;
      int4 m = mt[base];
      int4 mn = mt[base + 1];  // (stale past nr: never used)
      int32_t c[4];
      V x[4];
      load_row(base, m, c, x);
#pragma unroll 1
      for (int q = 0; q < nr; ++q) {
        const int4 mc = m;
        int32_t cc[4];
        V xc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cc[u] = c[u];
          xc[u] = x[u];
        }
        if (q + 1 < nr) {
          m = mn;
          if (q + 2 < nr) mn = mt[base + q + 2];
          load_row(base + q + 1, m, c, x);
        }
        if (!(mc.w & 2)) {
          if constexpr (VALIDATE) carry = -1;
          apply4(cc, xc, 0, mc.z, sgn_of(mc));
        } else {  // a long row, straight from global memory, 128 entries per step
          const int64_t src = ds[base + q];
          const int len = mc.z;
          if constexpr (VALIDATE) carry = -1;
          for (int s0 = 0; s0 < len; s0 += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int e = s0 + 32 * u + lane;
              cc[u] = e < len ? __ldg(col + src + e) : INT32_MAX;
              xc[u] = e < len ? __ldg(val + src + e) : V(0);
            }
            apply4(cc, xc, s0, len, sgn_of(mc));
            __syncwarp();
          }
        }
      }
      __syncwarp();  // slots of batch t are refilled next iteration
    }
    return bad;
  };
  const int bad = b < validate_below ? rows(std::true_type{}) : rows(std::false_type{});
  cp_async_wait<0>();
  const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (any && lane == 0) atomicOr(flags, any);
  __syncthreads();
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    double h = 0.0, l = 0.0;  // NULL input state = zeros (no read)
    if (hi_in) {
      h = hi_in[b * d + c0 + c];
      l = lo_in[b * d + c0 + c];
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const double* pw = reinterpret_cast<const double*>(k2_smem + w * (ST_COLS * 8 + RS * K2_SLOT * (4 + sizeof(V)) + RS * 24));
      double su, er;
      two_sum(h, POW2 ? pw[c] * scale : pw[c], su, er);
      h = su;
      l = __dadd_rn(l, er);
    }
    if (lo_out) {
      hi_out[b * d + c0 + c] = h;
      lo_out[b * d + c0 + c] = l;
    } else {  // the folded sketch hi + lo (lvsk_fold_compensated's value)
      hi_out[b * d + c0 + c] = h + l;
    }
  }
}

// K6: one warp per row, lane owns RPL = r/32 consecutive columns of u
template <typename V, int RPL, bool VEC4>
__global__ void __launch_bounds__(256) csr_rowsumsq_kernel(const int64_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col,
                                                           const V* __restrict__ val, int64_t n, int64_t d,
                                                           const float* __restrict__ M, int64_t r,
                                                           double* __restrict__ scores, int32_t* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t base0 = row_ptr[0];
  int bad = 0;
  for (int64_t row = warp0; row < n; row += nw) {
    const int64_t e0 = row_ptr[row] - base0, e1 = row_ptr[row + 1] - base0;
    float u[RPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j) u[j] = 0.f;
    for (int64_t e = e0; e < e1; e += 32) {
      const int64_t ei = e + lane;
      const bool live = ei < e1;
      int32_t c = live ? col[ei] : 0;
      float x = live ? static_cast<float>(val[ei]) : 0.f;
      if (live && (c < 0 || c >= d)) {
        bad |= LVSK_FLAG_BADINDEX;
        c = 0;
        x = 0.f;
      }
      if (live && !isfinite(x)) bad |= LVSK_FLAG_NONFINITE;
      const int cnt = static_cast<int>(e1 - e < 32 ? e1 - e : 32);
      for (int t = 0; t < cnt; ++t) {
        const int32_t ct = __shfl_sync(0xFFFFFFFFu, c, t);
        const float xt = __shfl_sync(0xFFFFFFFFu, x, t);
        const float* mrow = M + static_cast<int64_t>(ct) * r + lane * RPL;
        if constexpr (VEC4) {
#pragma unroll
          for (int j = 0; j < RPL; j += 4) {
            const float4 m = __ldg(reinterpret_cast<const float4*>(mrow + j));
            u[j] = fmaf(xt, m.x, u[j]);
            u[j + 1] = fmaf(xt, m.y, u[j + 1]);
            u[j + 2] = fmaf(xt, m.z, u[j + 2]);
            u[j + 3] = fmaf(xt, m.w, u[j + 3]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < RPL; ++j)
            if (lane * RPL + j < r) u[j] = fmaf(xt, __ldg(mrow + j), u[j]);
        }
      }
    }
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < RPL; ++j) acc = fmaf(u[j], u[j], acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
    if (lane == 0) scores[row] = static_cast<double>(acc);
  }
  const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (any && lane == 0) atomicOr(flags, any);
}

static int csr_grid(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 32;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

static int ceil_log2_csr(int64_t v) {
  int b = 0;
  while ((int64_t{1} << b) < v) ++b;
  return b;
}

}  // namespace lvsk

using namespace lvsk;

extern "C" size_t lvsk_hashed_csr_workspace_bytes(int64_t n, int32_t s, int64_t k) {
  Measure m;
  const int64_t N = n * s;
  m.take<uint32_t>(N);
  m.take<uint32_t>(N);
  m.take<uint32_t>(N);
  m.take<uint32_t>(N);
  m.take<uint32_t>(k + 1);
  m.take<int64_t>(N);
  m.take<int32_t>(N);
  radix::measure<uint32_t>(m, N);
  return m.off;
}

extern "C" int32_t lvsk_hashed_sketch_csr(const int64_t* row_ptr, const int32_t* col, const void* val,
                                          int32_t val_dtype, int64_t n, int64_t d, uint64_t row0,
                                          const lvsk_hash_block* blocks, int32_t s, double scale, const double* hi_in,
                                          const double* lo_in, double* hi_out, double* lo_out, int64_t k, void* ws,
                                          size_t ws_bytes, int32_t* flags, void* stream) {
  LVSK_REQUIRE(n >= 1 && d >= 1, LVSK_ERR_DIMENSION, "bad shape n=%lld d=%lld", (long long)n, (long long)d);
  LVSK_REQUIRE(d < (int64_t{1} << 31), LVSK_ERR_DIMENSION, "d too large for int32 column indices");
  LVSK_REQUIRE(s >= 1 && s <= 64 && k >= s, LVSK_ERR_CONFIGURATION, "need 1 <= s <= min(64, k)");
  LVSK_REQUIRE(n < (int64_t{1} << 31) && n * s < 0xFFFFFFFFll, LVSK_ERR_CAPACITY, "row block too large");
  LVSK_REQUIRE(val_dtype == LVSK_F32 || val_dtype == LVSK_F64, LVSK_ERR_CONFIGURATION, "values must be f32 or f64");
  cudaStream_t st = as_stream(stream);
  const int64_t N = n * s;
  Carve c(ws, ws_bytes);
  uint32_t* keys = c.take<uint32_t>(N);
  uint32_t* vals = c.take<uint32_t>(N);
  uint32_t* skeys = c.take<uint32_t>(N);
  uint32_t* svals = c.take<uint32_t>(N);
  uint32_t* start = c.take<uint32_t>(k + 1);
  int64_t* msrc = c.take<int64_t>(N);
  int32_t* mlen = c.take<int32_t>(N);
  auto rb = radix::carve<uint32_t>(c, N);
  LVSK_REQUIRE(c.ok(), LVSK_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
  CsrBlocks P;
  for (int j = 0; j < s; ++j) {
    P.a[j] = blocks[j].a;
    P.b[j] = blocks[j].b;
    P.key[j] = blocks[j].sign_key;
    P.offset[j] = static_cast<uint32_t>(blocks[j].offset);
    P.size[j] = static_cast<uint32_t>(blocks[j].size);
  }
  csr_keygen_kernel<<<csr_grid(N, 256), 256, 0, st>>>(n, row0, 0, s, P, keys, vals);
  LVSK_CHECK_LAUNCH("csr keygen");
  // every row meets the first block exactly once: its buckets validate the rows
  const int64_t validate_below = blocks[0].offset == 0 ? blocks[0].size : k;
  int32_t rc = radix::sort_pairs<uint32_t, uint32_t>(keys, vals, N, ceil_log2_csr(k), rb, skeys, svals, st);
  if (rc != LVSK_OK) return rc;
  radix::bucket_bounds_kernel<uint32_t><<<csr_grid(N + 1, 256), 256, 0, st>>>(skeys, N, k, start);
  const int ngroups = static_cast<int>((d + CSR_GROUP - 1) / CSR_GROUP);
  const int64_t units = k * ngroups;
  const unsigned grid = static_cast<unsigned>((units + CSR_WARPS - 1) / CSR_WARPS);
  const int smem = CSR_WARPS * 2 * CSR_GROUP * static_cast<int>(sizeof(double));
  rc = val_dtype == LVSK_F64
           ? ensure_smem_attr(reinterpret_cast<const void*>(csr_gather_kernel<double>), smem, "csr gather smem attribute")
           : ensure_smem_attr(reinterpret_cast<const void*>(csr_gather_kernel<float>), smem, "csr gather smem attribute");
  if (rc != LVSK_OK) return rc;
  if (getenv("LVSK_K2_DETERMINISTIC") == nullptr) {
    csr_prep_kernel<<<csr_grid(N, 256), 256, 0, st>>>(row_ptr, svals, N, msrc, mlen);
    const int sgroups = static_cast<int>((d + ST_COLS - 1) / ST_COLS);
    const unsigned sgrid = static_cast<unsigned>(k * sgroups);
    // K2 v4: W self-loading warps x NB copy batches of 8 row slots (float
    // values: 5 warps x 2 batches of 96-entry slots, one CTA per SM — the
    // fastest of the measured shapes (2x2, 2x3, 4x3 with 124-entry slots:
    // 7.4 / 7.8 / 8.1 ms against 6.9 ms at C4); float64 values: 4 x 2)
    int sexp = 0;
    const bool pow2 = std::frexp(scale, &sexp) == 0.5;  // scale = 2^k: applied exactly in the fold
#define LVSK_K2_GO(V, W_, D_, S_, P_, O_)                                                                       \
  do {                                                                                                          \
    const int sm = k2_smem_bytes(W_, D_, static_cast<int>(sizeof(V)), S_);                                     \
    auto kern = csr_sketch_kernel<V, W_, D_, P_, O_, S_>;                                                       \
    rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), sm, "csr sketch smem attribute");               \
    if (rc != LVSK_OK) return rc;                                                                               \
    kern<<<sgrid, 32 * W_, sm, st>>>(col, static_cast<const V*>(val), d, sgroups, svals, msrc, mlen, start,     \
                                     scale, hi_in, lo_in, hi_out, lo_out, flags, validate_below);               \
  } while (0)
#define LVSK_K2_LAUNCH(V, W_, D_, S_)            \
  do {                                           \
    if (pow2 && sgroups == 1)                    \
      LVSK_K2_GO(V, W_, D_, S_, true, true);     \
    else if (pow2)                               \
      LVSK_K2_GO(V, W_, D_, S_, true, false);    \
    else if (sgroups == 1)                       \
      LVSK_K2_GO(V, W_, D_, S_, false, true);    \
    else                                         \
      LVSK_K2_GO(V, W_, D_, S_, false, false);   \
  } while (0)
    if (val_dtype == LVSK_F32)
      LVSK_K2_LAUNCH(float, 5, 2, 96);
    else
      LVSK_K2_LAUNCH(double, 4, 2, 96);
#undef LVSK_K2_GO
#undef LVSK_K2_LAUNCH
  } else if (val_dtype == LVSK_F32)
    csr_gather_kernel<float><<<grid, 32 * CSR_WARPS, smem, st>>>(row_ptr, col, static_cast<const float*>(val), d,
                                                              ngroups, svals, start, units, scale, hi_in, lo_in,
                                                              hi_out, lo_out, flags);
  else
    csr_gather_kernel<double><<<grid, 32 * CSR_WARPS, smem, st>>>(row_ptr, col, static_cast<const double*>(val), d,
                                                               ngroups, svals, start, units, scale, hi_in, lo_in,
                                                               hi_out, lo_out, flags);
  LVSK_CHECK_LAUNCH("csr gather");
  return LVSK_OK;
}

namespace lvsk {
bool csr_rowsumsq_tc_ok(const float* M, int64_t r);
int32_t csr_rowsumsq_tc(const int64_t* row_ptr, const int32_t* col, const void* val, int32_t val_dtype, int64_t n,
                        int64_t d, const float* M, double* scores, int32_t* flags, cudaStream_t st);
size_t csr_rowsumsq_prep_bytes(int64_t d, int64_t r);
int32_t csr_rowsumsq_prepare(const float* M, int64_t d, int64_t r, void* prep, size_t prep_bytes, cudaStream_t st);
int32_t csr_rowsumsq_tc2(const int64_t* row_ptr, const int32_t* col, const void* val, int32_t val_dtype, int64_t n,
                         int64_t d, const float* M, const void* prep, size_t prep_bytes, double* scores,
                         int32_t* flags, cudaStream_t st);
}  // namespace lvsk

// K6-TC v2 (csr_tc.cu): the fold's M is turned once into bf16 operand images of
// the hot column window (lvsk_rowsumsq_csr_prepare); every leverage pass over
// CSR rows with that M then streams them through the tensor cores.
extern "C" size_t lvsk_rowsumsq_csr_prep_bytes(int64_t d, int64_t r) {
  return d >= 1 && getenv("LVSK_K6_SIMT") == nullptr && getenv("LVSK_K6_V1") == nullptr ? csr_rowsumsq_prep_bytes(d, r) : 0;
}

extern "C" int32_t lvsk_rowsumsq_csr_prepare(const float* M, int64_t d, int64_t r, void* prep, size_t prep_bytes,
                                             void* stream) {
  LVSK_REQUIRE(d >= 1 && r >= 1 && M != nullptr, LVSK_ERR_DIMENSION, "bad shape");
  return csr_rowsumsq_prepare(M, d, r, prep, prep_bytes, as_stream(stream));
}

extern "C" int32_t lvsk_rowsumsq_csr_prepared(const int64_t* row_ptr, const int32_t* col, const void* val,
                                              int32_t val_dtype, int64_t n, int64_t d, const float* M, int64_t r,
                                              const void* prep, size_t prep_bytes, double* scores, int32_t* flags,
                                              void* stream) {
  LVSK_REQUIRE(n >= 0 && d >= 1 && r == 128, LVSK_ERR_DIMENSION, "bad shape (the prepared pass needs r = 128)");
  LVSK_REQUIRE(val_dtype == LVSK_F32 || val_dtype == LVSK_F64, LVSK_ERR_CONFIGURATION, "values must be f32 or f64");
  if (n == 0) return LVSK_OK;
  return csr_rowsumsq_tc2(row_ptr, col, val, val_dtype, n, d, M, prep, prep_bytes, scores, flags, as_stream(stream));
}

extern "C" int32_t lvsk_rowsumsq_csr(const int64_t* row_ptr, const int32_t* col, const void* val, int32_t val_dtype,
                                     int64_t n, int64_t d, const float* M, int64_t r, double* scores, int32_t* flags,
                                     void* stream) {
  LVSK_REQUIRE(n >= 0 && d >= 1 && r >= 1, LVSK_ERR_DIMENSION, "bad shape");
  LVSK_REQUIRE(val_dtype == LVSK_F32 || val_dtype == LVSK_F64, LVSK_ERR_CONFIGURATION, "values must be f32 or f64");
  if (n == 0) return LVSK_OK;
  cudaStream_t st = as_stream(stream);
  // r = 128 (C4): the hot columns on the tensor cores (csr_tc.cu); LVSK_K6_SIMT=1 forces the SIMT kernel
  if (csr_rowsumsq_tc_ok(M, r)) return csr_rowsumsq_tc(row_ptr, col, val, val_dtype, n, d, M, scores, flags, st);
  const int grid = csr_grid(n * 32, 256);
  const bool aligned = reinterpret_cast<uintptr_t>(M) % 16 == 0;
#define LVSK_K6(RPL, V4)                                                                                         \
  do {                                                                                                           \
    if (val_dtype == LVSK_F32)                                                                                   \
      csr_rowsumsq_kernel<float, RPL, V4><<<grid, 256, 0, st>>>(row_ptr, col, static_cast<const float*>(val), n, \
                                                                d, M, r, scores, flags);                         \
    else                                                                                                         \
      csr_rowsumsq_kernel<double, RPL, V4><<<grid, 256, 0, st>>>(row_ptr, col, static_cast<const double*>(val), \
                                                                 n, d, M, r, scores, flags);                     \
  } while (0)
  if (r == 128 && aligned)
    LVSK_K6(4, true);
  else if (r <= 32)
    LVSK_K6(1, false);
  else if (r <= 64)
    LVSK_K6(2, false);
  else if (r <= 128)
    LVSK_K6(4, false);
  else if (r <= 256)
    LVSK_K6(8, false);
  else {
    set_error("CSR leverage pass supports r <= 256 (got %lld)", (long long)r);
    return LVSK_ERR_UNSUPPORTED;
  }
#undef LVSK_K6
  LVSK_CHECK_LAUNCH("csr rowsumsq");
  return LVSK_OK;
}
