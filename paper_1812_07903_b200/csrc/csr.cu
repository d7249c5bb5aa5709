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
#include <cstdlib>

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
    hi_out[b * d + c0 + c] = hi[c];
    lo_out[b * d + c0 + c] = lo[c];
  }
  const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (any && lane == 0) atomicOr(flags, any);
}

// ---------------------------------------------------------------------------
// K2 streaming variant (default).  csr_prep_kernel turns the bucket-sorted
// (row, sign) pairs into per-pair (source offset, length) so nothing
// downstream chases row pointers.  csr_stream_kernel: one CTA owns one
// (bucket, <= 4096-column group) with its float64 (hi, lo) slice in shared
// memory (64 KB); warp 0 streams the bucket's rows in chunks (<= 64 row
// segments / 1024 entries; longer rows are split, harmless since one row's
// entries have distinct columns) with cp.async into a 4-deep ring signalled
// by cp.async.mbarrier.arrive; warps 1..8 apply the chunk's segments
// concurrently (segment q by warp q mod 5), each into its OWN float64 row of
// partial sums in shared memory (5 x 32 KB): a segment's entries have distinct
// columns, so a warp's 32 lanes never collide and every update is a plain
// load-add-store — no atomics (the first version used returning shared fp64
// atomics, CAS loops that serialised on the Zipf-hot columns: 17.6 ms at C4).
// At the end hi_out + lo_out = TwoSum fold of (hi_in, lo_in, P_0 .. P_4) in
// warp order.  Deterministic; equal to the reference's compensated state to
// ~1e-16 relative instead of bit-for-bit (LVSK_K2_DETERMINISTIC=1 selects the
// ordered csr_gather_kernel, which is bit-exact).  The same warps validate
// their segments (strictly increasing in-range columns, finite values).
constexpr int ST_COLS = 4096;
constexpr int ST_ECAP = 1024;
constexpr int ST_RMAX = 64;
constexpr int ST_STAGES = 4;
// smem of a csr_stream_kernel<V, APPLY> CTA: APPLY private fp64 partial rows + the ring
constexpr int st_smem_bytes(int apply, int vsz) {
  return apply * ST_COLS * 8 + ST_STAGES * ST_ECAP * (vsz + 4) + ST_STAGES * ST_RMAX * 16 + ST_STAGES * 4 +
         2 * ST_STAGES * 8;
}

__device__ __forceinline__ uint32_t csr_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct SegInfo {
  int32_t off, len;  // position of the first column index in the stage buffer, entry count
  int32_t flags;     // bit0 negative sign, bit1 continuation of the previous segment's row
  int32_t voff;      // position of the first value (the two arrays' 16-byte alignments differ)
};

// Stage slot of a row piece of `len` entries: its 16-byte aligned superset in
// either array (<= 3 leading + <= 3 trailing entries) rounded to 4 entries.
__device__ __forceinline__ int32_t st_slot(int64_t len) { return static_cast<int32_t>((len + 9) & ~int64_t{3}); }

__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   csr_smem(dst)),
               "l"(src), "r"(bytes), "r"(csr_smem(bar))
               : "memory");
}

// Issue the aligned-superset copies of entries [src, src + len) of col / val
// into the stage at slot position pos; returns the SegInfo offsets.  A
// 16-byte aligned chunk holding one valid byte cannot cross a page, so the
// superset reads are always safe.
template <typename V>
__device__ __forceinline__ void st_issue(const int32_t* col, const V* val, int64_t src, int64_t len, int32_t pos,
                                         int32_t* cbuf, V* vbuf, uint64_t* bar, int32_t& coff, int32_t& voff) {
  const uintptr_t ca = reinterpret_cast<uintptr_t>(col + src), va = reinterpret_cast<uintptr_t>(val + src);
  const int32_t padc = static_cast<int32_t>((ca & 15) >> 2);
  const int32_t padv = static_cast<int32_t>((va & 15) / sizeof(V));
  constexpr int VW = 16 / sizeof(V);
  const uint32_t cbytes = static_cast<uint32_t>(((padc + len + 3) & ~int64_t{3}) * 4);
  const uint32_t vbytes = static_cast<uint32_t>(((padv + len + VW - 1) / VW) * 16);
  bulk_copy_g2s(cbuf + pos, reinterpret_cast<const void*>(ca & ~uintptr_t{15}), cbytes, bar);
  bulk_copy_g2s(vbuf + pos, reinterpret_cast<const void*>(va & ~uintptr_t{15}), vbytes, bar);
  coff = pos + padc;
  voff = pos + padv;
}
template <typename V>
__device__ __forceinline__ uint32_t st_bytes(const int32_t* col, const V* val, int64_t src, int64_t len) {
  const uintptr_t ca = reinterpret_cast<uintptr_t>(col + src), va = reinterpret_cast<uintptr_t>(val + src);
  const int64_t padc = (ca & 15) >> 2, padv = (va & 15) / sizeof(V);
  constexpr int VW = 16 / sizeof(V);
  return static_cast<uint32_t>(((padc + len + 3) & ~int64_t{3}) * 4 + ((padv + len + VW - 1) / VW) * 16);
}
__device__ __forceinline__ void st_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(csr_smem(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(csr_smem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(csr_smem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void st_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni SW_%=;\n}" ::"r"(csr_smem(b)),
      "r"(parity)
      : "memory");
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

// APPLY applier warps (private partial rows): 5 fills one SM per CTA; 2
// leaves room for two CTAs (two loaders) per SM.  Buckets below
// `validate_below` (OSNAP block 0: every row meets it exactly once)
// validate their segments; the other blocks' warps skip the per-entry
// checks.
template <typename V, int ST_APPLY>
__global__ void __launch_bounds__(32 * (1 + ST_APPLY)) csr_stream_kernel(
    const int32_t* __restrict__ col, const V* __restrict__ val, int64_t d, int ngroups,
    const uint32_t* __restrict__ svals, const int64_t* __restrict__ msrc, const int32_t* __restrict__ mlen,
    const uint32_t* __restrict__ start, double scale, const double* hi_in, const double* lo_in, double* hi_out,
    double* lo_out, int32_t* flags, int64_t validate_below) {
  extern __shared__ __align__(128) uint8_t st_smem[];
  double* part = reinterpret_cast<double*>(st_smem);                     // [ST_APPLY][ST_COLS]
  V* bval = reinterpret_cast<V*>(part + ST_APPLY * ST_COLS);             // [ST_STAGES][ST_ECAP]
  int32_t* bcol = reinterpret_cast<int32_t*>(bval + ST_STAGES * ST_ECAP);  // [ST_STAGES][ST_ECAP]
  SegInfo* seg = reinterpret_cast<SegInfo*>(bcol + ST_STAGES * ST_ECAP);  // [ST_STAGES][ST_RMAX]
  int32_t* nseg = reinterpret_cast<int32_t*>(seg + ST_STAGES * ST_RMAX);  // [ST_STAGES]
  uint64_t* full = reinterpret_cast<uint64_t*>(nseg + ST_STAGES);         // 8-aligned: ST_STAGES even
  uint64_t* empty = full + ST_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x / ngroups;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x - b * ngroups) * ST_COLS;
  const int64_t width = d - c0 < ST_COLS ? d - c0 : ST_COLS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(csr_smem(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(csr_smem(&empty[s])), "r"(ST_APPLY));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int c = threadIdx.x; c < ST_APPLY * ST_COLS; c += blockDim.x) part[c] = 0.0;
  __syncthreads();
  const uint32_t p0 = start[b], p1 = start[b + 1];
  if (warp == 0) {
    // ---- loader: 32 rows at a time, one lane per row — a warp scan places
    //      each row's 16-byte aligned superset in the stage and the lane
    //      issues its two cp.async.bulk copies; a row longer than a whole
    //      stage is streamed in pieces by lane 0
    uint32_t pb = p0;          // next pair batch
    int bcnt = 0, bq = 0;      // pairs in the current batch / consumed
    int64_t my_src = 0;
    int32_t my_len = 0;
    uint32_t my_v = 0;
    // the next batch's (src, len, sign), loaded one batch ahead so the
    // global-load latency overlaps the current batch's copies
    int64_t nx_src = 0;
    int32_t nx_len = 0;
    uint32_t nx_v = 0;
    if (lane < static_cast<int>(p1 - p0)) {
      nx_src = msrc[p0 + lane];
      nx_len = mlen[p0 + lane];
      nx_v = svals[p0 + lane];
    }
    int64_t lsrc = 0, lrem = 0;  // long row in progress (lane-uniform)
    uint32_t lneg = 0;
    bool lcont = false;
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it % ST_STAGES, ph = (it / ST_STAGES) & 1u;
      st_wait(&empty[s], ph ^ 1u);
      int32_t* cbuf = bcol + s * ST_ECAP;
      V* vbuf = bval + s * ST_ECAP;
      int ns = 0, ne = 0;
      bool done = false;
      while (ns < ST_RMAX) {
        if (lrem > 0) {
          const int64_t room = ST_ECAP - ne - 6;
          if (room < 1) break;
          const int64_t plen = lrem < room ? lrem : room;
          if (lane == 0) {
            st_expect(&full[s], st_bytes<V>(col, val, lsrc, plen));
            SegInfo si;
            st_issue<V>(col, val, lsrc, plen, ne, cbuf, vbuf, &full[s], si.off, si.voff);
            si.len = static_cast<int32_t>(plen);
            si.flags = static_cast<int32_t>(lneg | (lcont ? 2u : 0u));
            seg[s * ST_RMAX + ns] = si;
          }
          ++ns;
          ne += st_slot(plen);
          lsrc += plen;
          lrem -= plen;
          lcont = true;
          continue;
        }
        if (bq == bcnt) {  // fetch the next 32 pairs' (src, len, sign) in parallel
          if (pb >= p1) {
            done = true;
            break;
          }
          bcnt = p1 - pb < 32u ? static_cast<int>(p1 - pb) : 32;
          my_src = nx_src;
          my_len = nx_len;
          my_v = nx_v;
          pb += bcnt;
          bq = 0;
          if (pb + lane < p1) {
            nx_src = msrc[pb + lane];
            nx_len = mlen[pb + lane];
            nx_v = svals[pb + lane];
          }
        }
        const bool pend = lane >= bq && lane < bcnt;
        const bool longrow = pend && st_slot(my_len) > ST_ECAP;
        const uint32_t lm = __ballot_sync(0xFFFFFFFFu, longrow);
        const int first_long = lm ? __ffs(lm) - 1 : 32;
        const bool cand = pend && lane < first_long;
        const int32_t S = cand && my_len > 0 ? st_slot(my_len) : 0;
        const int32_t R = S > 0 ? 1 : 0;
        int32_t incl = S, rincl = R;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o), tr = __shfl_up_sync(0xFFFFFFFFu, rincl, o);
          if (lane >= o) {
            incl += t;
            rincl += tr;
          }
        }
        const bool fits = ne + incl <= ST_ECAP && ns + rincl <= ST_RMAX;
        const uint32_t nf = __ballot_sync(0xFFFFFFFFu, cand && !fits);
        int stop = nf ? __ffs(nf) - 1 : first_long;  // first lane not taken
        if (stop > bcnt) stop = bcnt;
        const bool take = cand && lane < stop;
        const uint32_t bytes = take && S > 0 ? st_bytes<V>(col, val, my_src, my_len) : 0u;
        const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, bytes);
        if (lane == 0 && total) st_expect(&full[s], total);
        __syncwarp();
        if (take && S > 0) {
          SegInfo si;
          st_issue<V>(col, val, my_src, my_len, ne + incl - S, cbuf, vbuf, &full[s], si.off, si.voff);
          si.len = my_len;
          si.flags = static_cast<int32_t>(my_v & 1u);
          seg[s * ST_RMAX + ns + rincl - 1] = si;
        }
        const int last_take = stop - 1;  // >= bq - 1
        if (last_take >= bq) {
          ne += __shfl_sync(0xFFFFFFFFu, incl, last_take);
          ns += __shfl_sync(0xFFFFFFFFu, rincl, last_take);
        }
        bq = stop;
        if (nf) break;  // the stage is full
        if (first_long < bcnt && bq == first_long) {  // hand the long row to the piece path
          lsrc = __shfl_sync(0xFFFFFFFFu, my_src, first_long);
          lrem = __shfl_sync(0xFFFFFFFFu, my_len, first_long);
          lneg = __shfl_sync(0xFFFFFFFFu, my_v, first_long) & 1u;
          lcont = false;
          ++bq;
        }
      }
      if (lane == 0) nseg[s] = done && ns == 0 ? -1 : ns;
      if (done && ns > 0 && lane == 0) nseg[s] = ns | (1 << 30);  // last chunk
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(csr_smem(&full[s])) : "memory");
      if (done) break;
    }
  } else {
    // ---- appliers
    const int aw = warp - 1;
    const bool validate = b < validate_below;
    int bad = 0;
    int32_t lastcol = -1;
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it % ST_STAGES, ph = (it / ST_STAGES) & 1u;
      st_wait(&full[s], ph);
      const int raw = nseg[s];
      if (raw < 0) break;
      const bool last = (raw >> 30) & 1;
      const int ns = raw & ((1 << 30) - 1);
      const V* vb = bval + s * ST_ECAP;
      const int32_t* cb = bcol + s * ST_ECAP;
      // segments are independent and this warp's partial row is private, so
      // every entry is a plain load-add-store (lanes hold distinct columns)
      double* mine = part + aw * ST_COLS;
      for (int q = aw; q < ns; q += ST_APPLY) {
        const SegInfo si = seg[s * ST_RMAX + q];
        const double sg = (si.flags & 1) ? -scale : scale;
        int32_t carry = -1;
        if (validate && (si.flags & 2)) {
          if (q > 0) {
            const SegInfo sp = seg[s * ST_RMAX + q - 1];
            carry = cb[sp.off + sp.len - 1];
          } else {
            carry = lastcol;
          }
        }
        // four 32-entry chunks at a time: one row's entries have distinct
        // columns, so their loads / adds / stores are independent (ILP)
        for (int e0v = 0; e0v < si.len; e0v += 128) {
          int32_t cc[4];
          double xx[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0v + 32 * u + lane;
            const bool live = e < si.len;
            const int32_t c = live ? cb[si.off + e] : INT32_MAX;
            const V xv = live ? vb[si.voff + e] : V(0);
            if (validate) {  // warp-uniform
              const int32_t cprev = __shfl_up_sync(0xFFFFFFFFu, c, 1);
              const int32_t before = lane == 0 ? carry : cprev;
              carry = __shfl_sync(0xFFFFFFFFu, c, 31);
              if (live) {
                if (c < 0 || c >= d || c <= before) bad |= LVSK_FLAG_BADINDEX;
                if (!isfinite(static_cast<double>(xv))) bad |= LVSK_FLAG_NONFINITE;
              }
            }
            const int64_t lc = static_cast<int64_t>(c) - c0;
            cc[u] = (live && lc >= 0 && lc < width) ? static_cast<int32_t>(lc) : -1;
            xx[u] = __dmul_rn(sg, static_cast<double>(xv));
          }
          double old[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) old[u] = cc[u] >= 0 ? mine[cc[u]] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cc[u] >= 0) mine[cc[u]] = __dadd_rn(old[u], xx[u]);
        }
        __syncwarp();  // the next segment may hit the same columns from other lanes
      }
      if (ns > 0) {
        const SegInfo sl = seg[s * ST_RMAX + ns - 1];
        lastcol = cb[sl.off + sl.len - 1];
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(csr_smem(&empty[s])) : "memory");
      if (last) break;
    }
    const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (any && lane == 0) atomicOr(flags, any);
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < width; c += blockDim.x) {
    double h = 0.0, l = 0.0;  // NULL input state = zeros (no read)
    if (hi_in) {
      h = hi_in[b * d + c0 + c];
      l = lo_in[b * d + c0 + c];
    }
#pragma unroll
    for (int w = 0; w < ST_APPLY; ++w) {
      double su, er;
      two_sum(h, part[w * ST_COLS + c], su, er);
      h = su;
      l = __dadd_rn(l, er);
    }
    hi_out[b * d + c0 + c] = h;
    lo_out[b * d + c0 + c] = l;
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
    const int vsz = val_dtype == LVSK_F64 ? 8 : 4;
    // applier warps per CTA (each with a private 32 KB partial row): 2 fits two
    // CTAs (two loader warps) per SM, 1 three; LVSK_K2_APPLY overrides (A/B)
    const int apply = getenv("LVSK_K2_APPLY") ? atoi(getenv("LVSK_K2_APPLY")) : 2;
    const unsigned sgrid = static_cast<unsigned>(k * sgroups);
    const int64_t vbelow = validate_below;
#define LVSK_K2_LAUNCH(V, A)                                                                                       \
  do {                                                                                                             \
    const int sm = st_smem_bytes(A, static_cast<int>(sizeof(V)));                                                 \
    rc = ensure_smem_attr(reinterpret_cast<const void*>(csr_stream_kernel<V, A>), sm, "csr stream smem attribute"); \
    if (rc != LVSK_OK) return rc;                                                                                  \
    csr_stream_kernel<V, A><<<sgrid, 32 * (1 + A), sm, st>>>(col, static_cast<const V*>(val), d, sgroups, svals,  \
                                                             msrc, mlen, start, scale, hi_in, lo_in, hi_out,      \
                                                             lo_out, flags, vbelow);                              \
  } while (0)
    if (val_dtype == LVSK_F32) {
      if (apply == 1)
        LVSK_K2_LAUNCH(float, 1);
      else if (apply == 3)
        LVSK_K2_LAUNCH(float, 3);
      else if (apply == 5)
        LVSK_K2_LAUNCH(float, 5);
      else
        LVSK_K2_LAUNCH(float, 2);
    } else {
      if (apply == 1)
        LVSK_K2_LAUNCH(double, 1);
      else if (apply == 3)
        LVSK_K2_LAUNCH(double, 3);
      else if (apply == 5)
        LVSK_K2_LAUNCH(double, 5);
      else
        LVSK_K2_LAUNCH(double, 2);
    }
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
}  // namespace lvsk

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
