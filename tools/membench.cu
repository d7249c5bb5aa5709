// HBM read-pattern microbenchmark (tools only, not product): how much DRAM
// bandwidth do the access patterns of K1 (row gather) and K5 (K-chunked row
// tiles) get on this B200, compared with a contiguous stream?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench tools/membench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void stream_read(const float4* __restrict__ x, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldg(x + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) *out = acc;
}

// each warp reads `seg` bytes from row perm[r] (row = 2 KB), rows in permuted order
template <int SEG_F4>
__global__ void gather_rows(const float4* __restrict__ x, const int* __restrict__ perm, int nrows, int row_f4,
                            float* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int segs = row_f4 / SEG_F4;
  float acc = 0.f;
  for (long long u = warp; u < (long long)nrows * segs; u += nw) {
    const int r = perm[u / segs], s = u % segs;
    const float4* p = x + (size_t)r * row_f4 + s * SEG_F4;
#pragma unroll
    for (int j = lane; j < SEG_F4; j += 32) {
      float4 v = __ldg(p + j);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 1234.5f) *out = acc;
}

// K5-like: CTA owns 256-row tiles; reads column chunk kc (128 B) of all 256 rows, kc = 0..15
__global__ void tile_chunks(const float4* __restrict__ x, int nrows, int row_f4, float* out) {
  float acc = 0.f;
  const int ntiles = nrows / 256;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int kc = 0; kc < row_f4 / 8; ++kc) {
      // 256 rows x 8 float4 = 2048 float4 per chunk, 256 threads x 8
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = j * 256 + threadIdx.x;
        const int r = e / 8, c = e % 8;
        float4 v = __ldg(x + (size_t)(t * 256 + r) * row_f4 + kc * 8 + c);
        acc += v.x + v.y + v.z + v.w;
      }
    }
  }
  if (acc == 1234.5f) *out = acc;
}

int main() {
  const int nrows = 1 << 20, row_f4 = 128;  // 1M rows x 2 KB = 2 GB
  const size_t n4 = (size_t)nrows * row_f4;
  float4* x;
  float* out;
  int* perm;
  cudaMalloc(&x, n4 * 16);
  cudaMalloc(&out, 4);
  cudaMalloc(&perm, nrows * 4);
  cudaMemset(x, 0, n4 * 16);
  std::vector<int> h(nrows);
  for (int i = 0; i < nrows; ++i) h[i] = i;
  srand(1);
  for (int i = nrows - 1; i > 0; --i) {
    int j = rand() % (i + 1);
    std::swap(h[i], h[j]);
  }
  cudaMemcpy(perm, h.data(), nrows * 4, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(a);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.1f GB/s  (%.3f ms)\n", name, n4 * 16.0 * reps / (ms * 1e-3) / 1e9, ms / reps);
  };
  timeit("stream contiguous (grid 8x SMs)", [&] { stream_read<<<sms * 8, 256>>>(x, n4, out); });
  timeit("stream contiguous (grid 32x SMs)", [&] { stream_read<<<sms * 32, 256>>>(x, n4, out); });
  timeit("gather random rows, 512 B/warp", [&] { gather_rows<32><<<sms * 16, 256>>>(x, perm, nrows, row_f4, out); });
  timeit("gather random rows, 2 KB/warp", [&] { gather_rows<128><<<sms * 16, 256>>>(x, perm, nrows, row_f4, out); });
  timeit("gather random rows, 128 B/warp", [&] { gather_rows<8><<<sms * 16, 256>>>(x, perm, nrows, row_f4, out); });
  timeit("tile chunks 256 rows x 128 B (1 CTA/SM)", [&] { tile_chunks<<<sms, 256>>>(x, nrows, row_f4, out); });
  timeit("tile chunks 256 rows x 128 B (4 CTA/SM)", [&] { tile_chunks<<<sms * 4, 256>>>(x, nrows, row_f4, out); });
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
