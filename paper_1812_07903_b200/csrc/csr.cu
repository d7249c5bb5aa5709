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
// K2 ring variant (default for float32 values): one CTA owns one (bucket, <= 4096-column group) with its
// float64 (hi, lo) slice in shared memory; a producer warp streams the
// bucket's CSR row pieces (16-byte aligned supersets, <= 64 entries each;
// rounding out to 16-byte granules never leaves the allocation's page) into a
// 32-slot ring; four consumer warps each apply one quarter of the columns
// into a 64-slot ring with cp.async.bulk, so ~100 rows are in flight per CTA;
// a consumer warp applies them in ascending row order.
constexpr int RING_SLOTS = 32;
constexpr int RING_CONSUMERS = 4;  // consumer warps, each owning a quarter of the column group
constexpr int SLOT_ELEMS = 64;
constexpr int RING_GROUP = 4096;

struct SlotMeta {
  int32_t first, last;  // valid element range inside the slot
  uint32_t flags;       // bit0: negative sign, bit1: first piece of its row
};

__device__ __forceinline__ uint32_t csr_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void csr_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni CW_%=;\n}" ::"r"(csr_smem(b)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(32 * (1 + RING_CONSUMERS)) csr_ring_kernel(const int64_t* __restrict__ row_ptr,
                                                      const int32_t* __restrict__ col, const float* __restrict__ val,
                                                      int64_t shift, int64_t d, int ngroups, const uint32_t* __restrict__ vals,
                                                      const uint32_t* __restrict__ start, double scale,
                                                      const double* hi_in, const double* lo_in, double* hi_out,
                                                      double* lo_out, int32_t* flags) {
  extern __shared__ __align__(128) uint8_t csr_ring_smem[];
  double* hi = reinterpret_cast<double*>(csr_ring_smem);
  double* lo = hi + RING_GROUP;
  int32_t* rcol = reinterpret_cast<int32_t*>(lo + RING_GROUP);     // [RING_SLOTS][SLOT_ELEMS]
  float* rval = reinterpret_cast<float*>(rcol + RING_SLOTS * SLOT_ELEMS);
  SlotMeta* meta = reinterpret_cast<SlotMeta*>(rval + RING_SLOTS * SLOT_ELEMS);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + RING_SLOTS);
  uint64_t* empty = full + RING_SLOTS;
  const int64_t b = blockIdx.x / ngroups;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x - b * ngroups) * RING_GROUP;
  const int64_t width = d - c0 < RING_GROUP ? d - c0 : RING_GROUP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING_SLOTS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(csr_smem(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(csr_smem(&empty[s])), "r"(RING_CONSUMERS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int64_t c = threadIdx.x; c < width; c += blockDim.x) {
    hi[c] = hi_in[b * d + c0 + c];
    lo[c] = lo_in[b * d + c0 + c];
  }
  __syncthreads();
  // element indices are relative to the 16-byte aligned col / val bases
  const int64_t base0 = row_ptr[0] - shift;
  const uint32_t p0 = start[b], p1 = start[b + 1];
  if (warp == 0) {  // producer: 32 rows' pointers fetched in parallel, lane 0 issues the copies
    uint32_t j = 0;
    for (uint32_t pb = p0; pb < p1; pb += 32) {
      const uint32_t p = pb + lane;
      const bool valid = p < p1;
      const uint32_t vv = valid ? vals[p] : 0u;
      const int64_t r = vv >> 1;
      const int64_t e0 = valid ? row_ptr[r] - base0 : 0, e1 = valid ? row_ptr[r + 1] - base0 : 0;
      const int cnt = p1 - pb < 32u ? static_cast<int>(p1 - pb) : 32;
      for (int q = 0; q < cnt; ++q) {
        const int64_t re0 = __shfl_sync(0xFFFFFFFFu, e0, q), re1 = __shfl_sync(0xFFFFFFFFu, e1, q);
        const uint32_t neg = __shfl_sync(0xFFFFFFFFu, vv, q) & 1u;
        if (lane == 0) {
          const int64_t a0 = re0 & ~int64_t{3};
          const int64_t a_end = (re1 + 3) & ~int64_t{3};
          int64_t s0 = a0;
          do {
            const int64_t s1 = s0 + SLOT_ELEMS < a_end ? s0 + SLOT_ELEMS : a_end;
            const uint32_t slot = j % RING_SLOTS, ph = (j / RING_SLOTS) & 1u;
            csr_wait(&empty[slot], ph ^ 1u);
            SlotMeta m;
            m.first = static_cast<int32_t>((re0 > s0 ? re0 : s0) - s0);
            m.last = static_cast<int32_t>((re1 < s1 ? re1 : s1) - s0);
            m.flags = neg | (s0 == a0 ? 2u : 0u);
            meta[slot] = m;
            const uint32_t nb = static_cast<uint32_t>((s1 - s0) * 4);
            if (nb > 0) {
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(csr_smem(&full[slot])),
                           "r"(2 * nb)
                           : "memory");
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      csr_smem(rcol + slot * SLOT_ELEMS)),
                  "l"(col + s0), "r"(nb), "r"(csr_smem(&full[slot]))
                  : "memory");
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      csr_smem(rval + slot * SLOT_ELEMS)),
                  "l"(val + s0), "r"(nb), "r"(csr_smem(&full[slot]))
                  : "memory");
            } else {
              asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(csr_smem(&full[slot])) : "memory");
            }
            ++j;
            s0 = s1;
          } while (s0 < a_end);
        }
      }
    }
    if (lane == 0) {  // end-of-stream marker
      const uint32_t slot = j % RING_SLOTS, ph = (j / RING_SLOTS) & 1u;
      csr_wait(&empty[slot], ph ^ 1u);
      SlotMeta m;
      m.first = m.last = 0;
      m.flags = 4u;
      meta[slot] = m;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(csr_smem(&full[slot])) : "memory");
    }
  } else {  // consumers: slots in order until the end marker (row starts carry flag bit 1);
           // warp w applies the columns [w, w+1) * RING_GROUP / RING_CONSUMERS of the group,
           // warp 1 also validates every entry
    const int cw = warp - 1;
    const int64_t lo_c = static_cast<int64_t>(cw) * (RING_GROUP / RING_CONSUMERS);
    const int64_t hi_c = lo_c + RING_GROUP / RING_CONSUMERS;
    int bad = 0;
    int32_t prev_last = -1;
    for (uint32_t j = 0;; ++j) {
      const uint32_t slot = j % RING_SLOTS, ph = (j / RING_SLOTS) & 1u;
      csr_wait(&full[slot], ph);
      const SlotMeta m = meta[slot];
      if (m.flags & 4u) break;
      if (m.flags & 2u) prev_last = -1;
      const double sg = (m.flags & 1u) ? -scale : scale;
      int32_t c[SLOT_ELEMS / 32];
      float x[SLOT_ELEMS / 32];
      bool live[SLOT_ELEMS / 32];
#pragma unroll
      for (int h = 0; h < SLOT_ELEMS / 32; ++h) {
        const int idx = h * 32 + lane;
        live[h] = idx >= m.first && idx < m.last;
        c[h] = live[h] ? rcol[slot * SLOT_ELEMS + idx] : INT32_MAX;
        x[h] = live[h] ? rval[slot * SLOT_ELEMS + idx] : 0.f;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(csr_smem(&empty[slot])) : "memory");
      if (cw == 0) {
#pragma unroll
        for (int h = 0; h < SLOT_ELEMS / 32; ++h) {
          const int idx = h * 32 + lane;
          const int32_t cprev = __shfl_up_sync(0xFFFFFFFFu, c[h], 1);
          const bool prev_live = lane > 0 && (idx - 1) >= m.first;
          const int32_t before = prev_live ? cprev : prev_last;
          if (live[h]) {
            if (c[h] < 0 || c[h] >= d || c[h] <= before) bad |= LVSK_FLAG_BADINDEX;
            if (!isfinite(x[h])) bad |= LVSK_FLAG_NONFINITE;
          }
          const uint32_t lm = __ballot_sync(0xFFFFFFFFu, live[h]);
          if (lm) prev_last = __shfl_sync(0xFFFFFFFFu, c[h], 31 - __clz(lm));
        }
      }
      // the entries of one row have distinct columns: both halves' updates are independent
      double hv[SLOT_ELEMS / 32], lv[SLOT_ELEMS / 32];
      int64_t lc[SLOT_ELEMS / 32];
      bool mine[SLOT_ELEMS / 32];
#pragma unroll
      for (int h = 0; h < SLOT_ELEMS / 32; ++h) {
        lc[h] = static_cast<int64_t>(c[h]) - c0;
        mine[h] = live[h] && lc[h] >= lo_c && lc[h] < hi_c && lc[h] < width;
        if (mine[h]) {
          hv[h] = hi[lc[h]];
          lv[h] = lo[lc[h]];
        }
      }
#pragma unroll
      for (int h = 0; h < SLOT_ELEMS / 32; ++h) {
        if (mine[h]) {
          double su, er;
          two_sum(hv[h], __dmul_rn(sg, static_cast<double>(x[h])), su, er);
          hi[lc[h]] = su;
          lo[lc[h]] = __dadd_rn(lv[h], er);
        }
      }
      __syncwarp();  // the next row may update the same columns from other lanes
    }
    const int any = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (any && lane == 0) atomicOr(flags, any);
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < width; c += blockDim.x) {
    hi_out[b * d + c0 + c] = hi[c];
    lo_out[b * d + c0 + c] = lo[c];
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
  // the ring reads 16-byte aligned supersets of each row; col and val must
  // share their misalignment so one element index addresses both
  const int mis = static_cast<int>(reinterpret_cast<uintptr_t>(col) % 16);
  const bool ring = val_dtype == LVSK_F32 && mis % 4 == 0 &&
                    mis == static_cast<int>(reinterpret_cast<uintptr_t>(val) % 16) &&
                    getenv("LVSK_K2_SIMPLE") == nullptr;
  if (ring) {
    const int rgroups = static_cast<int>((d + RING_GROUP - 1) / RING_GROUP);
    const int rsmem = 2 * RING_GROUP * 8 + RING_SLOTS * SLOT_ELEMS * 8 + RING_SLOTS * static_cast<int>(sizeof(SlotMeta)) +
                      2 * RING_SLOTS * 8;
    static bool rattr = false;
    if (!rattr) {
      cudaFuncSetAttribute(csr_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem);
      rattr = true;
    }
    csr_ring_kernel<<<static_cast<unsigned>(k * rgroups), 32 * (1 + RING_CONSUMERS), rsmem, st>>>(
        row_ptr, col - mis / 4, static_cast<const float*>(val) - mis / 4, mis / 4, d, rgroups, svals, start, scale, hi_in, lo_in, hi_out, lo_out,
        flags);
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
