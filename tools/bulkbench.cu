// K1-shaped microbenchmark (tools only): CTA per bucket streams ~244 random
// 2 KB rows through a SLOTS-deep cp.async.bulk ring (one producer lane), two
// consumer warps touch each row (optionally with the TwoSum work) and release
// the slot.  Separates the bulk-copy stream limit from the consumer limit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulkbench tools/bulkbench.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra.uni W_%=;\n}" ::"r"(
          sa(b)),
      "r"(ph)
      : "memory");
}

template <int SLOTS, bool WORK>
__global__ void __launch_bounds__(96) bulk_rows(const float* __restrict__ x, const int* __restrict__ perm,
                                                const int* __restrict__ start, double* out) {
  __shared__ alignas(128) uint8_t ring[SLOTS][2048];
  __shared__ uint64_t full[SLOTS], empty[SLOTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(sa(&empty[s])));
    }
  }
  __syncthreads();
  const int p0 = start[blockIdx.x], p1 = start[blockIdx.x + 1], cnt = p1 - p0;
  if (warp == 2) {
    if (lane == 0)
      for (int j = 0; j < cnt; ++j) {
        const int s = j % SLOTS;
        const uint32_t ph = (j / SLOTS) & 1;
        wait(&empty[s], ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 2048;" ::"r"(sa(&full[s])) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                sa(ring[s])),
            "l"(x + (long long)perm[p0 + j] * 512), "r"(sa(&full[s]))
            : "memory");
      }
    return;
  }
  double h[8] = {0, 0, 0, 0, 0, 0, 0, 0}, l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int j = 0; j < cnt; ++j) {
    const int s = j % SLOTS;
    const uint32_t ph = (j / SLOTS) & 1;
    wait(&full[s], ph);
    const float4* src = reinterpret_cast<const float4*>(ring[s]) + (warp * 32 + lane) * 2;
    const float4 a = src[0], b = src[1];
    if (WORK) {
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double c = (double)v[i];
        const double sm = h[i] + c, bp = sm - h[i];
        const double e = (h[i] - (sm - bp)) + (c - bp);
        h[i] = sm;
        l[i] += e;
      }
    } else {
      h[0] += a.x + b.y;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
  double t = 0;
  for (int i = 0; i < 8; ++i) t += h[i] + l[i];
  if (t == 1234.5) *out = t;
}

template <int SLOTS, bool STATEIO, bool BALLOT, bool BATCH>
__global__ void __launch_bounds__(96) k1_like(const float* __restrict__ x, const int* __restrict__ perm,
                                              const int* __restrict__ start, double* hi_io, double* lo_io,
                                              double* out) {
  __shared__ alignas(128) uint8_t ring[SLOTS][2048];
  __shared__ uint64_t full[SLOTS], empty[SLOTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(sa(&empty[s])));
    }
  }
  __syncthreads();
  const int p0 = start[blockIdx.x], p1 = start[blockIdx.x + 1], cnt = p1 - p0;
  if (warp == 2 && !BATCH) {
    if (lane == 0)
      for (int j = 0; j < cnt; ++j) {
        const int s = j % SLOTS;
        const uint32_t ph = (j / SLOTS) & 1;
        wait(&empty[s], ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 2048;" ::"r"(sa(&full[s])) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                sa(ring[s])),
            "l"(x + (long long)perm[p0 + j] * 512), "r"(sa(&full[s]))
            : "memory");
      }
    return;
  }
  if (warp == 2) {
    for (int jb = 0; jb < cnt; jb += 32) {
      const int mine = jb + lane < cnt ? perm[p0 + jb + lane] : 0;
      const int nb = cnt - jb < 32 ? cnt - jb : 32;
      for (int q = 0; q < nb; ++q) {
        const int v = __shfl_sync(0xFFFFFFFFu, mine, q);
        if (lane == 0) {
          const int j = jb + q, s = j % SLOTS;
          const uint32_t ph = (j / SLOTS) & 1;
          wait(&empty[s], ph ^ 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 2048;" ::"r"(sa(&full[s])) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                  sa(ring[s])),
              "l"(x + (long long)v * 512), "r"(sa(&full[s]))
              : "memory");
        }
      }
    }
    return;
  }
  const long long so = (long long)blockIdx.x * 512 + (warp * 32 + lane) * 8;
  double h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h[i] = STATEIO ? hi_io[so + i] : 0.0;
    l[i] = STATEIO ? lo_io[so + i] : 0.0;
  }
  uint32_t signs = 0;
  for (int j = 0; j < cnt; ++j) {
    const int s = j % SLOTS;
    const uint32_t ph = (j / SLOTS) & 1;
    if (BALLOT && (j & 31) == 0) signs = __ballot_sync(0xFFFFFFFFu, j + lane < cnt && (perm[p0 + j + lane] & 1));
    const bool neg = (signs >> (j & 31)) & 1u;
    wait(&full[s], ph);
    const float4* src = reinterpret_cast<const float4*>(ring[s]) + (warp * 32 + lane) * 2;
    const float4 a = src[0], b = src[1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double c = neg ? -(double)v[i] : (double)v[i];
      const double sm = h[i] + c, bp = sm - h[i];
      const double e = (h[i] - (sm - bp)) + (c - bp);
      h[i] = sm;
      l[i] += e;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
  if (STATEIO) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hi_io[so + i] = h[i];
      lo_io[so + i] = l[i];
    }
  } else {
    double t = 0;
    for (int i = 0; i < 8; ++i) t += h[i] + l[i];
    if (t == 1234.5) *out = t;
  }
}

int main() {
  const int nrows = 1 << 20, k = 4096;
  float* x;
  int *perm, *start;
  double* out;
  cudaMalloc(&x, (size_t)nrows * 2048);
  {
    std::vector<float> hx((size_t)nrows * 512);
    unsigned r = 7;
    for (size_t i = 0; i < hx.size(); ++i) {
      r = r * 1664525u + 1013904223u;
      hx[i] = (float)(r >> 8) * (1.0f / 16777216.0f) - 0.5f;
    }
    cudaMemcpy(x, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&perm, nrows * 4);
  cudaMalloc(&start, (k + 1) * 4);
  cudaMalloc(&out, 8);
  std::vector<int> h(nrows), st(k + 1);
  unsigned s = 12345;
  for (int i = 0; i < nrows; ++i) h[i] = i;
  for (int i = nrows - 1; i > 0; --i) {
    s = s * 1664525u + 1013904223u;
    int j = s % (i + 1);
    int t = h[i];
    h[i] = h[j];
    h[j] = t;
  }
  for (int b = 0; b <= k; ++b) st[b] = (int)((long long)nrows * b / k);
  cudaMemcpy(perm, h.data(), nrows * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(start, st.data(), (k + 1) * 4, cudaMemcpyHostToDevice);
  // K1's real order: rows hashed to buckets, each bucket in ascending row order
  std::vector<int> hb(nrows), cnt(k + 1, 0), bk(nrows), st2(k + 1, 0);
  const unsigned long long ha = 0xd855bac60e2f2043ull | 1ull, hbb = 0xa6cfae49d58dfd30ull;
  for (int i = 0; i < nrows; ++i) {
    const unsigned long long v = ha * (unsigned long long)i + hbb;  // the reference's multiply-shift bucket hash
    bk[i] = (int)(((v >> 32) * (unsigned long long)k) >> 32);
    ++cnt[bk[i] + 1];
  }
  for (int b = 0; b < k; ++b) cnt[b + 1] += cnt[b];
  st2 = cnt;
  for (int i = 0; i < nrows; ++i) hb[cnt[bk[i]]++] = i;
  int *perm2, *start2;
  cudaMalloc(&perm2, nrows * 4);
  cudaMalloc(&start2, (k + 1) * 4);
  cudaMemcpy(perm2, hb.data(), nrows * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(start2, st2.data(), (k + 1) * 4, cudaMemcpyHostToDevice);
  auto run2 = [&](const char* name, auto kern) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) kern<<<k, 96>>>(x, perm2, start2, out);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) kern<<<k, 96>>>(x, perm2, start2, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-36s %7.1f GB/s (%.3f ms)  %s\n", name, (double)nrows * 2048 * 10 / (ms * 1e-3) / 1e9, ms / 10,
           cudaGetErrorString(cudaGetLastError()));
  };
  auto run = [&](const char* name, auto kern) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) kern<<<k, 96>>>(x, perm, start, out);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) kern<<<k, 96>>>(x, perm, start, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-36s %7.1f GB/s (%.3f ms)  %s\n", name, (double)nrows * 2048 * 10 / (ms * 1e-3) / 1e9, ms / 10,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("bulk 2KB rows, 16 slots, no work", bulk_rows<16, false>);
  run("bulk 2KB rows, 16 slots, TwoSum", bulk_rows<16, true>);
  run("bulk 2KB rows, 20 slots, TwoSum", bulk_rows<20, true>);
  run("bulk 2KB rows, 8 slots, TwoSum", bulk_rows<8, true>);
  run2("hashed buckets ascending, 16, TwoSum", bulk_rows<16, true>);
  run2("hashed buckets ascending, 16, no work", bulk_rows<16, false>);
  double *hio, *lio;
  cudaMalloc(&hio, (size_t)k * 512 * 8);
  cudaMalloc(&lio, (size_t)k * 512 * 8);
  cudaMemset(hio, 0, (size_t)k * 512 * 8);
  cudaMemset(lio, 0, (size_t)k * 512 * 8);
  auto runk = [&](const char* name, auto kern) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) kern<<<k, 96>>>(x, perm2, start2, hio, lio, out);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) kern<<<k, 96>>>(x, perm2, start2, hio, lio, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-36s %7.1f GB/s (%.3f ms)  %s\n", name, (double)nrows * 2048 * 10 / (ms * 1e-3) / 1e9, ms / 10,
           cudaGetErrorString(cudaGetLastError()));
  };
  runk("K1-like all", k1_like<16, true, true, true>);
  runk("K1-like no stateio", k1_like<16, false, true, true>);
  runk("K1-like no ballot", k1_like<16, true, false, true>);
  runk("K1-like no batch", k1_like<16, true, true, false>);
  runk("K1-like none", k1_like<16, false, false, false>);
  runk("K1-like stateio only", k1_like<16, true, false, false>);
  return 0;
}
