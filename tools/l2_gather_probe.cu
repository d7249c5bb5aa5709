// L2 -> SM gather bandwidth probe (the roofline of K6's cold M-row gathers):
// warps gather random 512-byte rows (one float4 per lane) of an L2-resident
// table (4096 x 128 fp32 = 2 MB, K6's M at C4), IN_FLIGHT rows per lane
// outstanding, and FMA them into registers (as K6 does).  Also: the same with
// Zipf-like row ids (C4's cold columns) and a coalesced-stream baseline.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2g tools/l2_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cmath>

template <int IN_FLIGHT>
__global__ void gather_kernel(const float4* __restrict__ M, const int* __restrict__ ids, int64_t nids, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = warp * 32; base < nids; base += nw * 32) {
    const int my = ids[base + lane];
#pragma unroll
    for (int b0 = 0; b0 < 32; b0 += IN_FLIGHT) {
      float4 mv[IN_FLIGHT];
#pragma unroll
      for (int j = 0; j < IN_FLIGHT; ++j) {
        const int ct = __shfl_sync(0xFFFFFFFFu, my, b0 + j);
        mv[j] = __ldg(M + (int64_t)ct * 32 + lane);
      }
#pragma unroll
      for (int j = 0; j < IN_FLIGHT; ++j) {
        u.x = fmaf(1.0001f, mv[j].x, u.x);
        u.y = fmaf(1.0001f, mv[j].y, u.y);
        u.z = fmaf(1.0001f, mv[j].z, u.z);
        u.w = fmaf(1.0001f, mv[j].w, u.w);
      }
    }
  }
  if (u.x + u.y + u.z + u.w == 12345.f) out[0] = u.x;
}

int main() {
  const int rows = 4096, r = 128;
  const int64_t nids = int64_t(1) << 26;  // 64M gathered rows = 32 GB of gather traffic
  std::vector<float> hM((size_t)rows * r, 1.f);
  std::vector<int> uni(nids), zipf(nids);
  std::mt19937_64 g(1);
  std::uniform_int_distribution<int> U(0, rows - 1);
  for (int64_t i = 0; i < nids; ++i) uni[i] = U(g);
  // Zipf(1.1) over the cold columns 128..4095 (K6-TC's gathered set at C4)
  std::vector<double> cdf(rows);
  double s = 0;
  for (int i = 0; i < rows; ++i) { s += (i >= 128) ? std::pow(i + 1.0, -1.1) : 0.0; cdf[i] = s; }
  std::uniform_real_distribution<double> R(0, s);
  for (int64_t i = 0; i < nids; ++i) zipf[i] = int(std::lower_bound(cdf.begin(), cdf.end(), R(g)) - cdf.begin());
  float4* dM; int* dI; float* dO;
  cudaMalloc(&dM, hM.size() * 4); cudaMalloc(&dI, nids * 4); cudaMalloc(&dO, 4);
  cudaMemcpy(dM, hM.data(), hM.size() * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int which = 0; which < 2; ++which) {
    cudaMemcpy(dI, which ? zipf.data() : uni.data(), nids * 4, cudaMemcpyHostToDevice);
    for (int blocks_per_sm : {4, 8}) {
      for (int inflight : {8, 16}) {
        auto launch = [&]() {
          if (inflight == 8) gather_kernel<8><<<sms * blocks_per_sm, 256>>>(dM, dI, nids, dO);
          else gather_kernel<16><<<sms * blocks_per_sm, 256>>>(dM, dI, nids, dO);
        };
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int it = 0; it < 5; ++it) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        const double bytes = double(nids) * 512 + double(nids) * 4;
        printf("%s ids, %d CTAs/SM x 256 thr, %d rows in flight/lane: %.3f ms, gather %.2f TB/s (%.1f B/clk/SM @1.965 GHz)\n",
               which ? "zipf-cold" : "uniform", blocks_per_sm, inflight, ms, bytes / ms / 1e9,
               bytes / (ms * 1e-3) / sms / 1.965e9);
      }
    }
  }
  return 0;
}
