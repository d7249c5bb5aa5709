// K4-TC — Gaussian sketch SX = Z X / sqrt(k) on the tensor cores for bf16 X
// (BASELINE config 5), Z generated on the fly (gauss_gen.cuh) and never stored
// in global memory.  Extension: the reference rejects "gaussian"
// (pkg/src/levsketch/sketch.py:38-41, 74-75).
//
// GEMM shape: SX (k x d) = Z (k x n) . X (n x d), contraction over the input
// rows n.  One CTA owns a (128 sketch rows) x (NS <= 512 columns) output
// tile for one split of the rows (split-K; the fp32 partials are reduced in
// float64 by gaussian.cu's reduce kernel), accumulating in TMEM
// (NS fp32 columns).  Per 64-row stage:
//   warp 0   TMA: X[64 rows][NS cols] as NS/64 SW128 boxes.  X is the MMA's
//            B operand in MN-major layout (rows of X = K, contiguous columns
//            = N), so no transpose pass exists anywhere;
//   warps 2-17 generate the Z tile [128 x 64] (gauss_gen.cuh: one mix64
//            per 4 entries, a 16-bit inverse-CDF table lookup per entry,
//            bit-identical to the SIMT path and the oracle) straight into
//            the K-major SW128 A layout in shared memory and arrive (the MMA
//            thread issues the generic->async proxy fence once per stage);
//   warp 1   issues 4 x (NS/256) tcgen05.mma kind::f16 (M = 128, N = 256,
//            K = 16) and commits the stage back to both producers.
// After the last stage warps 2-17 drain TMEM (tcgen05.ld 32x32b) into the
// split's fp32 partial.  X traffic: each X element is read once per 128
// sketch rows (ceil(k/128) times, L2-shared across the CTAs of one
// (split, column slab) which are launched adjacently); each Z entry is
// generated ceil(d/NS) times.
#include <cstdlib>

#include "gauss_gen.cuh"
#include "tc_common.cuh"

namespace lvsk {
namespace tc {

template <int NS>
struct CfgG {
  static constexpr int BKN = 64;                // input rows per stage (MMA K)
  static constexpr int NB = NS / 64;            // 64-column TMA boxes per stage
  static constexpr int NMMA = NS / 256;         // N = 256 MMAs per K16 step
  static constexpr int BOX_BYTES = BKN * 64 * 2;  // 8 KB
  static constexpr int X_BYTES = NB * BOX_BYTES;
  static constexpr int Z_BYTES = BM * BKN * 2;  // 16 KB
  static constexpr int S = NS == 512 ? 2 : 4;  // X stages
  static constexpr int SZ = 2;                  // Z stages (the 64 KB table leaves room for two)
  static constexpr int OFF_Z = S * X_BYTES;
  static constexpr int OFF_BAR = OFF_Z + SZ * Z_BYTES;
  static constexpr int OFF_TAB = OFF_BAR + 256;
  static constexpr int SMEM_BYTES = OFF_TAB + GT_LEVELS * 2 + 1024;
  static constexpr int GEN_WARPS = 16;  // one per 8-row octet of the 128-row tile
  static constexpr int NTHREADS = 64 + 32 * GEN_WARPS;
  // kind::f16: F32 accumulate, A = B = bf16, B MN-major, N = 256, M = 128
  static constexpr uint32_t IDESC =
      (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(256 >> 3) << 17) | (uint32_t(BM >> 4) << 24);
};

// MN-major SWIZZLE_128B: 64-element x 8-row atoms; LBO = stride between
// 64-element MN blocks, SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(lbo_bytes >> 4) << 16;
  d |= uint64_t{1024 >> 4} << 32;
  d |= uint64_t{1} << 46;
  d |= uint64_t{2} << 61;
  return d;
}

__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t map_peer(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// 4-byte store into a peer CTA's shared memory that completes 4 bytes of the
// transaction count of the peer's mbarrier (no release fence: the barrier
// carries the ordering)
__device__ __forceinline__ void st_async_b32(uint32_t remote_addr, uint32_t v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(remote_addr), "r"(v),
               "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                               uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
      : "memory");
}

// MX = 2: the two CTAs of a cluster are consecutive k tiles of the same
// (column slab, split); each issues half of every X stage's boxes with TMA
// multicast to both, so X crosses L2 -> SM once per pair, and a slot is
// refilled only after both CTAs' MMAs released it (commit multicast).
// CL = 2 (d in (NS, 2 NS]): the two column slabs of a k tile form a cluster
// and share its Z tile: each CTA generates half of the tile's rows and writes
// them into its own shared memory (st.shared) and into the peer's
// (st.async, completing bytes of the peer's zfull transaction count), so
// every Z entry is generated once per k tile instead of once per slab — the
// 16-bit table lookups (random banks, ~3.5 wavefronts per warp read) are the
// kernel's shared-memory bound.  Round 1's version of this signalled the
// peer with cluster-scope release arrives and lost (5.25 vs 3.68 ms); the
// transaction-count form needs no fence.
// Otherwise one CTA per (k tile, column slab, split), generating its whole Z
// tile.  CL and MX are not combined.
template <int NS, int CL, int MX>
__global__ void __launch_bounds__(CfgG<NS>::NTHREADS, 1)
    gaussian_tc_kernel(const __grid_constant__ CUtensorMap mapX, int64_t n, int64_t d, int64_t k, uint64_t row0,
                       uint64_t key, int ktiles, int dslabs, int64_t rows_per_split, int64_t period,
                       const uint16_t* __restrict__ gmag, float* __restrict__ partial) {
  using C = CfgG<NS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, stays a shared-space pointer
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* xfull = bars;
  uint64_t* empty = xfull + C::S;  // X slots
  uint64_t* zfull = empty + C::S;
  uint64_t* zempty = zfull + C::SZ;
  uint64_t* accfull = zempty + C::SZ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);
  uint16_t* mag = reinterpret_cast<uint16_t*>(smem + C::OFF_TAB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int item = blockIdx.x;
  int ktile, dslab;
  int64_t split;
  if constexpr (CL == 1) {
    ktile = item % ktiles;
    dslab = (item / ktiles) % dslabs;
    split = item / (ktiles * dslabs);
  } else {  // cluster rank = column slab
    dslab = item % CL;
    ktile = (item / CL) % ktiles;
    split = item / (CL * ktiles);
  }
  const int64_t r_begin = split * rows_per_split;
  const int64_t r_end = r_begin + rows_per_split < n ? r_begin + rows_per_split : n;
  const int nstages = static_cast<int>((r_end - r_begin + C::BKN - 1) / C::BKN);
  const int col0 = dslab * NS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&empty[s], MX);
    }
    for (int s = 0; s < C::SZ; ++s) {
      mbar_init(&zfull[s], C::GEN_WARPS);  // + (CL = 2) the peer's half of the tile as transaction bytes
      mbar_init(&zempty[s], CL);           // every CTA's MMA that reads the slot
    }
    mbar_init(accfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
  }
  load_gaussian_table(mag, gmag);
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(NS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (CL > 1 || MX > 1) cluster_sync_all();  // peers' barriers are initialised before any remote arrive
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_normal();
      for (int t = 0; t < nstages; ++t) {
        const uint32_t s = t % C::S, ph = (t / C::S) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_expect_tx(&xfull[s], C::X_BYTES);
        const int row = static_cast<int>(r_begin + static_cast<int64_t>(t) * C::BKN);
        if constexpr (MX > 1) {
          const int rk = ktile % MX;  // cluster rank
#pragma unroll
          for (int b = rk; b < C::NB; b += MX)
            tma_load_2d_mc(&mapX, &xfull[s], smem + s * C::X_BYTES + b * C::BOX_BYTES, col0 + b * 64, row,
                           static_cast<uint16_t>((1u << MX) - 1u), pol);
        } else {
#pragma unroll
          for (int b = 0; b < C::NB; ++b)
            tma_load_2d(&mapX, &xfull[s], smem + s * C::X_BYTES + b * C::BOX_BYTES, col0 + b * 64, row, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int t = 0; t < nstages; ++t) {
        const uint32_t s = t % C::S, ph = (t / C::S) & 1u;
        const uint32_t sz = t % C::SZ, phz = (t / C::SZ) & 1u;
        mbar_wait(&xfull[s], ph);
        if constexpr (CL > 1)
          mbar_wait_cluster(&zfull[sz], phz);  // half of the tile came from the peer
        else
          mbar_wait(&zfull[sz], phz);
        // the Z tile was written through the generic proxy; one proxy fence
        // here, after the acquire, orders it before the tensor core's
        // async-proxy reads (instead of one per producer warp)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_after();
        const uint64_t a = sw128_desc(smem_u32(smem + C::OFF_Z + sz * C::Z_BYTES));
#pragma unroll
        for (int kk = 0; kk < C::BKN / 16; ++kk) {
#pragma unroll
          for (int h = 0; h < C::NMMA; ++h) {
            const uint64_t b = sw128_mn_desc(smem_u32(smem + s * C::X_BYTES + h * 4 * C::BOX_BYTES + kk * 2048),
                                             C::BOX_BYTES);
            umma_f16(tmem_base + h * 256, a + 2 * kk, b, C::IDESC, (t | kk) ? 1u : 0u);
          }
        }
        if constexpr (MX > 1)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[s])),
              "h"(static_cast<uint16_t>((1u << MX) - 1u))
              : "memory");
        else
          umma_commit(&empty[s]);
        if constexpr (CL > 1)  // both CTAs write this Z slot: both MMAs release it
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&zempty[sz])),
              "h"(static_cast<uint16_t>((1u << CL) - 1u))
              : "memory");
        else
          umma_commit(&zempty[sz]);
      }
      umma_commit(accfull);
    }
  } else {
    const int gw = warp - 2;
    constexpr uint64_t ROW = GAUSS_PHI << 24;    // next input row
    constexpr uint64_t STAGE = GAUSS_PHI << 30;  // 64 input rows on
    const uint32_t mbase = smem_u32(mag);
    if constexpr (CL == 1) {
      // ---- Z generation: warp gw -> sketch rows 8gw .. 8gw+7 of the tile
      //      (quads t0, t0 + 1), lane -> input rows 2*lane, 2*lane+1 of the
      //      stage: four mix64 per lane per stage, counters advanced by
      //      constant adds (gauss_ctr is linear in (i << 24) | t)
      const uint32_t t0 = static_cast<uint32_t>(ktile * (BM / 4) + 2 * gw);
      // Row r of the stacked input is global row row0 + (r mod period): the
      // fp32 path stacks its three bf16 planes (period = padded plane rows,
      // a multiple of 64, so a stage never straddles two planes)
      int64_t rr = r_begin % period;
      const uint64_t wrap = static_cast<uint64_t>(period) * ROW;
      uint64_t ctr = gauss_ctr(key, row0 + static_cast<uint64_t>(rr + 2 * lane), t0);
      for (int t = 0; t < nstages; ++t, ctr += STAGE, rr += C::BKN) {
        if (rr == period) rr = 0, ctr -= wrap;
        const uint32_t s = t % C::SZ, ph = (t / C::SZ) & 1u;
        // h[r][q]: input row 2 lane + r, quad t0 + q
        const uint64_t h00 = mix64(ctr), h01 = mix64(ctr + GAUSS_PHI);
        const uint64_t h10 = mix64(ctr + ROW), h11 = mix64(ctr + ROW + GAUSS_PHI);
        uint32_t w[8];  // sketch row 8 gw + r8: bf16 pair (input row 2 lane, 2 lane + 1)
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
          const uint64_t ha = r8 < 4 ? h00 : h01, hb = r8 < 4 ? h10 : h11;
          const uint32_t fa = static_cast<uint32_t>(ha >> (16 * (r8 & 3)));
          const uint32_t fb = static_cast<uint32_t>(hb >> (16 * (r8 & 3)));
          uint16_t ma, mb;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(ma) : "r"(mbase + 2 * (fa & 0x7FFFu)));
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(mb) : "r"(mbase + 2 * (fb & 0x7FFFu)));
          w[r8] = (static_cast<uint32_t>(ma) | (fa & 0x8000u)) | ((static_cast<uint32_t>(mb) | (fb & 0x8000u)) << 16);
        }
        mbar_wait(&zempty[s], ph ^ 1u);
        uint8_t* zt = smem + C::OFF_Z + s * C::Z_BYTES;
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
          const int j = 8 * gw + r8;
          // row j: 128 B = 8 swizzled 16-byte chunks; lane owns bytes [4 lane, 4 lane + 4)
          const int off = j * 128 + ((((lane >> 2) ^ (j & 7))) << 4) + (lane & 3) * 4;
          *reinterpret_cast<uint32_t*>(zt + off) = w[r8];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&zfull[s]);
      }
    } else {
      // ---- Z generation, cluster of 2: this CTA (rank = dslab) makes tile
      //      rows [64 rank, 64 rank + 64): warp gw -> rows 64 rank + 4 gw ..
      //      +3 (one quad), lane -> input rows 2 lane, 2 lane + 1; each word
      //      goes to both CTAs' Z slot
      const uint32_t peer = static_cast<uint32_t>(dslab ^ 1);
      const int jbase = 64 * dslab + 4 * gw;
      const uint32_t t0 = static_cast<uint32_t>(ktile * (BM / 4) + jbase / 4);
      // stacked-plane row wrap, as in the CL == 1 loop
      int64_t rr = r_begin % period;
      const uint64_t wrap = static_cast<uint64_t>(period) * ROW;
      uint64_t ctr = gauss_ctr(key, row0 + static_cast<uint64_t>(rr + 2 * lane), t0);
      const uint32_t zloc = smem_u32(smem + C::OFF_Z);
      const uint32_t zrem = map_peer(zloc, peer);
      const uint32_t fullrem = map_peer(smem_u32(&zfull[0]), peer);
      for (int t = 0; t < nstages; ++t, ctr += STAGE, rr += C::BKN) {
        if (rr == period) rr = 0, ctr -= wrap;
        const uint32_t s = t % C::SZ, ph = (t / C::SZ) & 1u;
        const uint64_t h0 = mix64(ctr), h1 = mix64(ctr + ROW);
        uint32_t w[4];
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
          const uint32_t fa = static_cast<uint32_t>(h0 >> (16 * r4));
          const uint32_t fb = static_cast<uint32_t>(h1 >> (16 * r4));
          uint16_t ma, mb;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(ma) : "r"(mbase + 2 * (fa & 0x7FFFu)));
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(mb) : "r"(mbase + 2 * (fb & 0x7FFFu)));
          w[r4] = (static_cast<uint32_t>(ma) | (fa & 0x8000u)) | ((static_cast<uint32_t>(mb) | (fb & 0x8000u)) << 16);
        }
        mbar_wait_cluster(&zempty[s], ph ^ 1u);  // both CTAs' MMAs are done with this slot
        const uint32_t slot = static_cast<uint32_t>(s * C::Z_BYTES);
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
          const int j = jbase + r4;
          const uint32_t off = slot + j * 128 + ((((lane >> 2) ^ (j & 7))) << 4) + (lane & 3) * 4;
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(zloc + off), "r"(w[r4]) : "memory");
          st_async_b32(zrem + off, w[r4], fullrem + 8 * s);
        }
        __syncwarp();
        if (lane == 0) {
          if (gw == 0)  // this CTA's arrival also announces the peer's 8 KB half
            mbar_expect_tx(&zfull[s], 64 * 128);
          else
            mbar_arrive(&zfull[s]);
        }
      }
    }
    // ---- epilogue: TMEM -> fp32 partial
    mbar_wait(accfull, 0);
    tc_fence_after();
    constexpr int PARTS = C::GEN_WARPS / 4;  // warps per TMEM lane quarter
    const int quarter = warp & 3, part = gw >> 2;
    const int64_t j = static_cast<int64_t>(ktile) * BM + quarter * 32 + lane;
    float* out = partial + split * k * d + j * d;
#pragma unroll 1
    for (int c = part * (NS / PARTS); c < (part + 1) * (NS / PARTS); c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + c, v);
      tmem_wait_ld();
      const int64_t dc = col0 + c;
      if (j < k) {
        if (dc + 32 <= d && (d & 3) == 0) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(out + dc + e) =
                make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                            __uint_as_float(v[e + 3]));
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (dc + e < d) out[dc + e] = __uint_as_float(v[e]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(NS));
  }
  if constexpr (CL > 1 || MX > 1) cluster_sync_all();  // no CTA leaves while its peer may still write into it
}

// ---- cluster of four: a CTA pair (cta_group::2) x two column slabs --------
// Ranks 2 slab + kt: the two k tiles 2p, 2p + 1 of a k-tile pair form one
// M = 256 MMA (each CTA holds its 128 Z rows = the A half, and 256 of its
// slab's 512 X columns = the B half: 128 of each N = 256 instruction), and
// the two slabs share every Z tile as in CL = 2 (each CTA generates 64 of
// its 128 Z rows, the slab partner rank ^ 2 the other 64, over st.async).
// Per CTA and stage the shared memory takes 32 KB of X (not 64) and the MMA
// reads half of B from it — the 1-CTA kernel is shared-memory-bandwidth
// bound (TMA writes + UMMA operand reads + the generator's table loads) —
// and the freed space deepens the Z ring (the generators run up to four
// stages ahead; with two the pair measured slower than CL = 2).  Measured at
// C5 (1e6 rows, one box): 3.22 ms (S = 3, SZ = 4) vs 3.75 (2, 4), 4.82
// (4, 2), 3.93 CL = 2, 4.31 X multicast; all bitwise equal.
template <int NS, int S_ = 3, int SZ_ = 4>
struct CfgGP {
  static constexpr int BKN = 64;
  static constexpr int NBH = NS / 128;            // 64-column boxes per CTA per stage (half of the slab)
  static constexpr int BOX_BYTES = BKN * 64 * 2;  // 8 KB
  static constexpr int X_BYTES = NBH * BOX_BYTES;
  static constexpr int Z_BYTES = BM * BKN * 2;    // 16 KB
  static constexpr int S = S_, SZ = SZ_;
  static constexpr int OFF_Z = S * X_BYTES;
  static constexpr int OFF_BAR = OFF_Z + SZ * Z_BYTES;
  static constexpr int OFF_TAB = OFF_BAR + 256;
  static constexpr int SMEM_BYTES = OFF_TAB + GT_LEVELS * 2 + 1024;
  static constexpr int GEN_WARPS = 16;
  static constexpr int NTHREADS = 64 + 32 * GEN_WARPS;
  // kind::f16: F32 accumulate, bf16 A (K-major) / B (MN-major), N = 256, M = 256 (pair)
  static constexpr uint32_t IDESC =
      (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(256 >> 3) << 17) | (uint32_t(256 >> 4) << 24);
};

template <int NS, int S_, int SZ_>
__global__ void __launch_bounds__(CfgGP<NS, S_, SZ_>::NTHREADS, 1)
    gaussian_tc_pair_kernel(const __grid_constant__ CUtensorMap mapX, int64_t n, int64_t d, int64_t k, uint64_t row0,
                            uint64_t key, int kpairs, int64_t rows_per_split, int64_t period,
                            const uint16_t* __restrict__ gmag,
                            float* __restrict__ partial) {
  using C = CfgGP<NS, S_, SZ_>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* xfull = bars;             // leader: both CTAs' X bytes
  uint64_t* xempty = xfull + C::S;    // the pair's MMA released the X slot
  uint64_t* zfull = xempty + C::S;    // 16 local arrivals + the slab partner's 8 KB
  uint64_t* zpeer = zfull + C::SZ;    // leader: the odd CTA's Z tile is complete
  uint64_t* zempty = zpeer + C::SZ;   // both pairs' MMAs released the Z slot
  uint64_t* accfull = zempty + C::SZ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);
  uint16_t* mag = reinterpret_cast<uint16_t*>(smem + C::OFF_TAB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t kt = rank & 1u, slab = rank >> 1, lead = rank & ~1u;
  const uint16_t pair_mask = static_cast<uint16_t>(3u << lead);
  const int64_t cid = blockIdx.x >> 2;
  const int ktile = static_cast<int>(2 * (cid % kpairs) + kt);
  const int64_t split = cid / kpairs;
  const int64_t r_begin = split * rows_per_split;
  const int64_t r_end = r_begin + rows_per_split < n ? r_begin + rows_per_split : n;
  const int nstages = static_cast<int>((r_end - r_begin + C::BKN - 1) / C::BKN);
  const int col0 = static_cast<int>(slab) * NS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::S; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < C::SZ; ++s) {
      mbar_init(&zfull[s], C::GEN_WARPS);
      mbar_init(&zpeer[s], 1);
      mbar_init(&zempty[s], 2);
    }
    mbar_init(accfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
  }
  load_gaussian_table(mag, gmag);
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(NS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_normal();
      const uint32_t lead_xfull = mapa_rank(smem_u32(&xfull[0]), lead);
      for (int t = 0; t < nstages; ++t) {
        const uint32_t s = t % C::S, ph = (t / C::S) & 1u;
        mbar_wait(&xempty[s], ph ^ 1u);
        if (kt == 0) mbar_expect_tx(&xfull[s], 2 * C::X_BYTES);
        const int row = static_cast<int>(r_begin + static_cast<int64_t>(t) * C::BKN);
#pragma unroll
        for (int b = 0; b < C::NBH; ++b) {  // instruction h = b / 2 takes columns [256 h + 128 kt, +128)
          const int col = col0 + 256 * (b >> 1) + 128 * static_cast<int>(kt) + 64 * (b & 1);
          tma_load_2d_pair(&mapX, lead_xfull + 8 * s, smem + s * C::X_BYTES + b * C::BOX_BYTES, col, row, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      if (kt == 0) {  // the pair's MMA issuer
        for (int t = 0; t < nstages; ++t) {
          const uint32_t s = t % C::S, ph = (t / C::S) & 1u;
          const uint32_t sz = t % C::SZ, phz = (t / C::SZ) & 1u;
          mbar_wait(&xfull[s], ph);
          mbar_wait_cluster(&zfull[sz], phz);
          mbar_wait_cluster(&zpeer[sz], phz);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_fence_after();
          const uint64_t a = sw128_desc(smem_u32(smem + C::OFF_Z + sz * C::Z_BYTES));
#pragma unroll
          for (int kk = 0; kk < C::BKN / 16; ++kk) {
#pragma unroll
            for (int h = 0; h < NS / 256; ++h) {
              const uint64_t b = sw128_mn_desc(smem_u32(smem + s * C::X_BYTES + h * 2 * C::BOX_BYTES + kk * 2048),
                                               C::BOX_BYTES);
              umma_f16_pair(tmem_base + h * 256, a + 2 * kk, b, C::IDESC, (t | kk) ? 1u : 0u);
            }
          }
          umma_commit_mask(&xempty[s], pair_mask);
          umma_commit_mask(&zempty[sz], 0xF);  // both slabs' generators write this pair's Z slots
        }
        umma_commit_mask(accfull, pair_mask);
      } else {  // odd CTA: tell the leader when this CTA's half of the A operand is complete
        const uint32_t lead_zpeer = mapa_rank(smem_u32(&zpeer[0]), lead);
        for (int t = 0; t < nstages; ++t) {
          const uint32_t sz = t % C::SZ, phz = (t / C::SZ) & 1u;
          mbar_wait_cluster(&zfull[sz], phz);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lead_zpeer + 8 * sz)
                       : "memory");
        }
      }
    }
  } else {
    const int gw = warp - 2;
    constexpr uint64_t ROW = GAUSS_PHI << 24;
    constexpr uint64_t STAGE = GAUSS_PHI << 30;
    const uint32_t mbase = smem_u32(mag);
    // ---- Z generation: tile rows [64 slab, 64 slab + 64) of k tile `ktile`:
    //      warp gw -> rows 64 slab + 4 gw .. +3 (one quad), lane -> input rows
    //      2 lane, 2 lane + 1; each word to this CTA's and the slab partner's Z slot
    const uint32_t partner = rank ^ 2u;
    const int jbase = 64 * static_cast<int>(slab) + 4 * gw;
    const uint32_t t0 = static_cast<uint32_t>(ktile * (BM / 4) + jbase / 4);
    // stacked-plane row wrap, as in gaussian_tc_kernel
    int64_t rr = r_begin % period;
    const uint64_t wrap = static_cast<uint64_t>(period) * ROW;
    uint64_t ctr = gauss_ctr(key, row0 + static_cast<uint64_t>(rr + 2 * lane), t0);
    const uint32_t zloc = smem_u32(smem + C::OFF_Z);
    const uint32_t zrem = mapa_rank(zloc, partner);
    const uint32_t fullrem = mapa_rank(smem_u32(&zfull[0]), partner);
    for (int t = 0; t < nstages; ++t, ctr += STAGE, rr += C::BKN) {
      if (rr == period) rr = 0, ctr -= wrap;
      const uint32_t s = t % C::SZ, ph = (t / C::SZ) & 1u;
      const uint64_t h0 = mix64(ctr), h1 = mix64(ctr + ROW);
      uint32_t w[4];
#pragma unroll
      for (int r4 = 0; r4 < 4; ++r4) {
        const uint32_t fa = static_cast<uint32_t>(h0 >> (16 * r4));
        const uint32_t fb = static_cast<uint32_t>(h1 >> (16 * r4));
        uint16_t ma, mb;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(ma) : "r"(mbase + 2 * (fa & 0x7FFFu)));
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(mb) : "r"(mbase + 2 * (fb & 0x7FFFu)));
        w[r4] = (static_cast<uint32_t>(ma) | (fa & 0x8000u)) | ((static_cast<uint32_t>(mb) | (fb & 0x8000u)) << 16);
      }
      mbar_wait_cluster(&zempty[s], ph ^ 1u);
      const uint32_t slot = static_cast<uint32_t>(s * C::Z_BYTES);
#pragma unroll
      for (int r4 = 0; r4 < 4; ++r4) {
        const int j = jbase + r4;
        const uint32_t off = slot + j * 128 + ((((lane >> 2) ^ (j & 7))) << 4) + (lane & 3) * 4;
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(zloc + off), "r"(w[r4]) : "memory");
        st_async_b32(zrem + off, w[r4], fullrem + 8 * s);
      }
      __syncwarp();
      if (lane == 0) {
        if (gw == 0)
          mbar_expect_tx(&zfull[s], 64 * 128);
        else
          mbar_arrive(&zfull[s]);
      }
    }
    // ---- epilogue: this CTA's 128 rows (k tile `ktile`) x NS columns -> fp32 partial
    mbar_wait(accfull, 0);
    tc_fence_after();
    constexpr int PARTS = C::GEN_WARPS / 4;
    const int quarter = warp & 3, part = gw >> 2;
    const int64_t j = static_cast<int64_t>(ktile) * BM + quarter * 32 + lane;
    float* out = partial + split * k * d + j * d;
#pragma unroll 1
    for (int c = part * (NS / PARTS); c < (part + 1) * (NS / PARTS); c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + c, v);
      tmem_wait_ld();
      const int64_t dc = col0 + c;
      if (j < k) {
        if (dc + 32 <= d && (d & 3) == 0) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(out + dc + e) =
                make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                            __uint_as_float(v[e + 3]));
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (dc + e < d) out[dc + e] = __uint_as_float(v[e]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(NS));
  }
}

}  // namespace tc

GaussTcPlan plan_gauss_tc(int64_t n, int64_t d, int64_t k) {
  GaussTcPlan p;
  p.ns = d > 256 ? 512 : 256;
  p.ktiles = static_cast<int>((k + tc::BM - 1) / tc::BM);
  p.dslabs = static_cast<int>((d + p.ns - 1) / p.ns);
  const int64_t pairs = static_cast<int64_t>(p.ktiles) * p.dslabs;
  int64_t splits = num_sms() / pairs;
  const int64_t maxs = (n + 255) / 256;
  if (splits > maxs) splits = maxs;
  if (splits < 1) splits = 1;
  p.rows_per_split = ((n + splits - 1) / splits + 63) / 64 * 64;
  p.splits = (n + p.rows_per_split - 1) / p.rows_per_split;
  p.period = n;
  return p;
}

bool gaussian_tc_ok(const void* X, int64_t n, int64_t d, int64_t ldx, int64_t k) {
  if (getenv("LVSK_NO_TC") != nullptr) return false;
  if (reinterpret_cast<uintptr_t>(X) % 16 != 0 || (ldx * 2) % 16 != 0) return false;
  if (n > (int64_t{1} << 31) - (int64_t{1} << 20) || d < 1 || k < 1) return false;
  return true;
}

template <int NS, int CL, int MX>
static int32_t launch_gauss_tc(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, int64_t k, uint64_t row0,
                               uint64_t key, const GaussTcPlan& p, float* partial, cudaStream_t st) {
  using C = tc::CfgG<NS>;
  CUtensorMap mx;
  if (!tc::make_map(&mx, X, d, n, ldx * 2, 64, C::BKN, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t rc = ensure_smem_attr(reinterpret_cast<const void*>(tc::gaussian_tc_kernel<NS, CL, MX>), C::SMEM_BYTES,
                                      "gaussian tc smem attribute");
  if (rc != LVSK_OK) return rc;
  const int64_t items = static_cast<int64_t>(p.ktiles) * p.dslabs * p.splits;
  const uint16_t* gmag = gaussian_table_device();
  if (gmag == nullptr) {
    set_error("cannot allocate the Gaussian generator table");
    return LVSK_ERR_CUDA;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(items));
  cfg.blockDim = dim3(C::NTHREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CL * MX;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc::gaussian_tc_kernel<NS, CL, MX>, mx, n, d, k, row0, key, p.ktiles,
                                     p.dslabs, p.rows_per_split, p.period, gmag, partial);
  if (e != cudaSuccess) return cuda_status(e, "gaussian tc launch");
  return LVSK_OK;
}

template <int S_, int SZ_>
static int32_t launch_gauss_tc_pair(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, int64_t k,
                                    uint64_t row0, uint64_t key, const GaussTcPlan& p, float* partial,
                                    cudaStream_t st) {
  using C = tc::CfgGP<512, S_, SZ_>;
  CUtensorMap mx;
  if (!tc::make_map(&mx, X, d, n, ldx * 2, 64, C::BKN, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16)) {
    set_error("cuTensorMapEncodeTiled failed");
    return LVSK_ERR_CUDA;
  }
  const int32_t rc = ensure_smem_attr(reinterpret_cast<const void*>(tc::gaussian_tc_pair_kernel<512, S_, SZ_>), C::SMEM_BYTES,
                                      "gaussian tc pair smem attribute");
  if (rc != LVSK_OK) return rc;
  const uint16_t* gmag = gaussian_table_device();
  if (gmag == nullptr) {
    set_error("cannot allocate the Gaussian generator table");
    return LVSK_ERR_CUDA;
  }
  const int kpairs = p.ktiles / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(4 * kpairs * p.splits));
  cfg.blockDim = dim3(C::NTHREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 4;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc::gaussian_tc_pair_kernel<512, S_, SZ_>, mx, n, d, k, row0, key, kpairs,
                                           p.rows_per_split, p.period, gmag, partial);
  if (e != cudaSuccess) return cuda_status(e, "gaussian tc pair launch");
  return LVSK_OK;
}

int32_t gaussian_tc_bf16(const __nv_bfloat16* X, int64_t n, int64_t d, int64_t ldx, int64_t k, uint64_t row0,
                         uint64_t key, const GaussTcPlan& p, float* partial, cudaStream_t st) {
  // LVSK_K4_VARIANT: A/B switch between equivalent kernels (identical results;
  // tests/test_gpu_parity.py runs every one): 3 = pair x shared Z (default),
  // 2 = shared Z, 1 = X multicast, 0 = plain
  const char* v = getenv("LVSK_K4_VARIANT");
  const int want = v ? atoi(v) : 3;
  if (want >= 3 && p.ns == 512 && p.dslabs == 2 && p.ktiles % 2 == 0)
    return launch_gauss_tc_pair<3, 4>(X, n, d, ldx, k, row0, key, p, partial, st);
  if (want >= 2 && p.ns == 512 && p.dslabs == 2)
    return launch_gauss_tc<512, 2, 1>(X, n, d, ldx, k, row0, key, p, partial, st);
  if (want >= 1 && p.ns == 512 && p.ktiles % 2 == 0)
    return launch_gauss_tc<512, 1, 2>(X, n, d, ldx, k, row0, key, p, partial, st);
  return p.ns == 512 ? launch_gauss_tc<512, 1, 1>(X, n, d, ldx, k, row0, key, p, partial, st)
                     : launch_gauss_tc<256, 1, 1>(X, n, d, ldx, k, row0, key, p, partial, st);
}

}  // namespace lvsk
