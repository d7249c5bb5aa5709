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
    hi[c] = hi_in[b * d + c0 + c];
    lo[c] = lo_in[b * d + c0 + c];
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
// K2 staged variant (default): one CTA (8 warps) owns one (bucket, <= 4096-
// column group) with its float64 (hi, lo) slice in shared memory (64 KB).
// The bucket's rows are staged in chunks of <= 64 rows / 2048 entries: warp 0
// plans a chunk from 32 rows' pointers fetched in parallel (rows longer than
// the buffer are split into segments, which is harmless: one row's entries
// have distinct columns), all warps copy it with cp.async (LDGSTS) into one of
// two buffers while the previous chunk is applied; the apply walks the rows
// in ascending index and warp w applies the entries of its 512 columns
// (TwoSum into hi / lo), the validation (strictly increasing in-range columns,
// finite values) is spread over the warps by row.
constexpr int SG_COLS = 4096;
constexpr int SG_WARPS = 8;
constexpr int SG_ECAP = 2048;  // entries per staging buffer
constexpr int SG_RMAX = 64;    // rows (segments) per staging buffer

struct SegInfo {
  int64_t src;      // first entry (relative to base0)
  int32_t off, len;  // position in the buffer, entry count
  int32_t flags;     // bit0 negative sign, bit1 continuation of the previous segment's row
};

__device__ __forceinline__ uint32_t csr_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(csr_smem(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(csr_smem(dst)), "l"(src) : "memory");
}

template <typename V>
__global__ void __launch_bounds__(32 * SG_WARPS) csr_staged_kernel(
    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const V* __restrict__ val, int64_t d,
    int ngroups, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ start, double scale,
    const double* hi_in, const double* lo_in, double* hi_out, double* lo_out, int32_t* flags) {
  extern __shared__ __align__(128) uint8_t sg_smem[];
  double* hi = reinterpret_cast<double*>(sg_smem);
  double* lo = hi + SG_COLS;
  V* bval = reinterpret_cast<V*>(lo + SG_COLS);                       // [2][SG_ECAP]
  int32_t* bcol = reinterpret_cast<int32_t*>(bval + 2 * SG_ECAP);     // [2][SG_ECAP]
  SegInfo* seg = reinterpret_cast<SegInfo*>(bcol + 2 * SG_ECAP);      // [2][SG_RMAX]
  __shared__ int nseg_s[2];
  __shared__ int more_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x / ngroups;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x - b * ngroups) * SG_COLS;
  const int64_t width = d - c0 < SG_COLS ? d - c0 : SG_COLS;
  for (int64_t c = threadIdx.x; c < width; c += blockDim.x) {
    hi[c] = hi_in[b * d + c0 + c];
    lo[c] = lo_in[b * d + c0 + c];
  }
  const int64_t base0 = row_ptr[0];
  const uint32_t p0 = start[b], p1 = start[b + 1];

  // ---- planner state (warp 0): a batch of 32 prefetched rows + the row in progress
  uint32_t pb = p0;        // first row of the prefetched batch
  int bq = 32;             // next batch slot to consume (32 = batch empty)
  int64_t e0 = 0, e1 = 0;  // this lane's batch row
  uint32_t vv = 0;
  int64_t cur = 0, cur_end = 0;  // segment cursor of the row in progress (lane-uniform)
  uint32_t cur_neg = 0;
  bool cur_live = false, cont = false;

  auto plan = [&](int buf) -> int {  // warp 0 only; returns the number of segments
    int ns = 0, ne = 0;
    while (ns < SG_RMAX && ne < SG_ECAP) {
      if (!cur_live) {
        if (bq == 32) {
          if (pb >= p1) break;
          const uint32_t p = pb + lane;
          const bool valid = p < p1;
          vv = valid ? vals[p] : 0u;
          const int64_t r = vv >> 1;
          e0 = valid ? row_ptr[r] - base0 : 0;
          e1 = valid ? row_ptr[r + 1] - base0 : 0;
          bq = 0;
        }
        const uint32_t p = pb + bq;
        if (p >= p1) break;
        cur = __shfl_sync(0xFFFFFFFFu, e0, bq);
        cur_end = __shfl_sync(0xFFFFFFFFu, e1, bq);
        cur_neg = __shfl_sync(0xFFFFFFFFu, vv, bq) & 1u;
        cur_live = true;
        cont = false;
        if (++bq == 32) pb += 32;
      }
      const int64_t room = SG_ECAP - ne;
      const int64_t len = cur_end - cur < room ? cur_end - cur : room;
      if (len == 0 && cur_end > cur) break;  // buffer full
      if (lane == 0) {
        SegInfo si;
        si.src = cur;
        si.off = ne;
        si.len = static_cast<int32_t>(len);
        si.flags = static_cast<int32_t>(cur_neg | (cont ? 2u : 0u));
        seg[buf * SG_RMAX + ns] = si;
      }
      ++ns;
      ne += static_cast<int>(len);
      cur += len;
      if (cur >= cur_end) {
        cur_live = false;
      } else {
        cont = true;
      }
    }
    return ns;
  };
  auto issue = [&](int buf, int ns) {  // all warps: copy the planned segments
    for (int q = warp; q < ns; q += SG_WARPS) {
      const SegInfo si = seg[buf * SG_RMAX + q];
      for (int e = lane; e < si.len; e += 32) {
        cp_async4(bcol + buf * SG_ECAP + si.off + e, col + si.src + e);
        if constexpr (sizeof(V) == 8)
          cp_async8(bval + buf * SG_ECAP + si.off + e, val + si.src + e);
        else
          cp_async4(bval + buf * SG_ECAP + si.off + e, val + si.src + e);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  if (warp == 0) {
    const int ns = plan(0);
    if (lane == 0) {
      nseg_s[0] = ns;
      more_s = cur_live || (pb + (bq == 32 ? 0 : bq)) < p1;
    }
  }
  __syncthreads();
  issue(0, nseg_s[0]);
  int bad = 0;
  int32_t lastcol = -1;  // last column of the previous chunk (a row continued across chunks)
  const int64_t lo_c = static_cast<int64_t>(warp) * (SG_COLS / SG_WARPS), hi_c = lo_c + SG_COLS / SG_WARPS;
  for (int it = 0;; ++it) {
    const int buf = it & 1;
    const bool more = more_s;
    __syncthreads();  // every thread has read more_s / nseg_s before the planner rewrites them
    if (more) {
      if (warp == 0) {
        const int ns = plan(buf ^ 1);
        if (lane == 0) {
          nseg_s[buf ^ 1] = ns;
          more_s = cur_live || (pb + (bq == 32 ? 0 : bq)) < p1;
        }
      }
      __syncthreads();
      issue(buf ^ 1, nseg_s[buf ^ 1]);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // chunk `it` has landed for every thread's copies
    const int ns = nseg_s[buf];
    const V* vb = bval + buf * SG_ECAP;
    const int32_t* cb = bcol + buf * SG_ECAP;
    for (int q = 0; q < ns; ++q) {
      const SegInfo si = seg[buf * SG_RMAX + q];
      const double sg = (si.flags & 1) ? -scale : scale;
      for (int e = lane; e < si.len; e += 32) {
        const int64_t lc = static_cast<int64_t>(cb[si.off + e]) - c0;
        if (lc >= lo_c && lc < hi_c && lc < width) {
          double su, er;
          two_sum(hi[lc], __dmul_rn(sg, static_cast<double>(vb[si.off + e])), su, er);
          hi[lc] = su;
          lo[lc] = __dadd_rn(lo[lc], er);
        }
      }
      __syncwarp();  // the next row may hit the same columns from other lanes
      if (q % SG_WARPS == warp) {  // validation of this segment
        int32_t carry = (si.flags & 2) ? (q > 0 ? cb[si.off - 1] : lastcol) : -1;
        for (int e0v = 0; e0v < si.len; e0v += 32) {
          const int e = e0v + lane;
          const bool live = e < si.len;
          const int32_t c = live ? cb[si.off + e] : INT32_MAX;
          const double x = live ? static_cast<double>(vb[si.off + e]) : 0.0;
          const int32_t cprev = __shfl_up_sync(0xFFFFFFFFu, c, 1);
          const int32_t before = lane == 0 ? carry : cprev;
          if (live) {
            if (c < 0 || c >= d || c <= before) bad |= LVSK_FLAG_BADINDEX;
            if (!isfinite(x)) bad |= LVSK_FLAG_NONFINITE;
          }
          carry = __shfl_sync(0xFFFFFFFFu, c, 31);
        }
      }
    }
    if (ns > 0) {
      const SegInfo sl = seg[buf * SG_RMAX + ns - 1];
      if (sl.len > 0) lastcol = cb[sl.off + sl.len - 1];
    }
    if (!more) break;
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < width; c += blockDim.x) {
    hi_out[b * d + c0 + c] = hi[c];
    lo_out[b * d + c0 + c] = lo[c];
  }
  const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (any && lane == 0) atomicOr(flags, any);
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
  int32_t rc = radix::sort_pairs<uint32_t, uint32_t>(keys, vals, N, ceil_log2_csr(k), rb, skeys, svals, st);
  if (rc != LVSK_OK) return rc;
  radix::bucket_bounds_kernel<uint32_t><<<csr_grid(N + 1, 256), 256, 0, st>>>(skeys, N, k, start);
  const int ngroups = static_cast<int>((d + CSR_GROUP - 1) / CSR_GROUP);
  const int64_t units = k * ngroups;
  const unsigned grid = static_cast<unsigned>((units + CSR_WARPS - 1) / CSR_WARPS);
  const int smem = CSR_WARPS * 2 * CSR_GROUP * static_cast<int>(sizeof(double));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(csr_gather_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(csr_gather_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  if (getenv("LVSK_K2_SIMPLE") == nullptr) {
    const int sgroups = static_cast<int>((d + SG_COLS - 1) / SG_COLS);
    const int vsz = val_dtype == LVSK_F64 ? 8 : 4;
    const int ssmem = 2 * SG_COLS * 8 + 2 * SG_ECAP * (vsz + 4) + 2 * SG_RMAX * static_cast<int>(sizeof(SegInfo));
    static bool sattr = false;
    if (!sattr) {
      cudaFuncSetAttribute(csr_staged_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           2 * SG_COLS * 8 + 2 * SG_ECAP * 8 + 2 * SG_RMAX * static_cast<int>(sizeof(SegInfo)));
      cudaFuncSetAttribute(csr_staged_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           2 * SG_COLS * 8 + 2 * SG_ECAP * 12 + 2 * SG_RMAX * static_cast<int>(sizeof(SegInfo)));
      sattr = true;
    }
    const unsigned sgrid = static_cast<unsigned>(k * sgroups);
    if (val_dtype == LVSK_F32)
      csr_staged_kernel<float><<<sgrid, 32 * SG_WARPS, ssmem, st>>>(row_ptr, col, static_cast<const float*>(val), d,
                                                                   sgroups, svals, start, scale, hi_in, lo_in,
                                                                   hi_out, lo_out, flags);
    else
      csr_staged_kernel<double><<<sgrid, 32 * SG_WARPS, ssmem, st>>>(row_ptr, col, static_cast<const double*>(val),
                                                                    d, sgroups, svals, start, scale, hi_in, lo_in,
                                                                    hi_out, lo_out, flags);
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

extern "C" int32_t lvsk_rowsumsq_csr(const int64_t* row_ptr, const int32_t* col, const void* val, int32_t val_dtype,
                                     int64_t n, int64_t d, const float* M, int64_t r, double* scores, int32_t* flags,
                                     void* stream) {
  LVSK_REQUIRE(n >= 0 && d >= 1 && r >= 1, LVSK_ERR_DIMENSION, "bad shape");
  LVSK_REQUIRE(val_dtype == LVSK_F32 || val_dtype == LVSK_F64, LVSK_ERR_CONFIGURATION, "values must be f32 or f64");
  if (n == 0) return LVSK_OK;
  cudaStream_t st = as_stream(stream);
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
