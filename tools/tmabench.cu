// TMA streaming microbenchmark (tools only): DRAM bandwidth of a K-major
// [ROWS x 32 fp32] SWIZZLE_128B box stream (the K5 X stream) as a function of
// box height and ring depth, one CTA per SM, single producer thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmabench tools/tmabench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int ROWS, int STAGES>
__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap map, int nrows, int kchunks,
                                                    float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + STAGES * ROWS * 128);
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
  __syncthreads();
  const int ntiles = nrows / ROWS;
  float acc = 0.f;
  if (threadIdx.x == 0) {
    uint32_t it = 0, issued = 0;
    // prologue + steady state: keep STAGES boxes in flight
    int t = blockIdx.x, kc = 0;
    auto issue = [&](uint32_t i) {
      const uint32_t s = i % STAGES;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(ROWS * 128));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
              "r"(sa(sm + s * ROWS * 128)),
          "l"(&map), "r"(kc * 32), "r"(t * ROWS), "r"(sa(&full[s]))
          : "memory");
      if (++kc == kchunks) { kc = 0; t += gridDim.x; }
    };
    const uint32_t total = (uint32_t)(((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * kchunks);
    for (; issued < STAGES && issued < total; ++issued) issue(issued);
    for (it = 0; it < total; ++it) {
      const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra.uni W_%=;\n}" ::"r"(
              sa(&full[s])),
          "r"(ph)
          : "memory");
      acc += *(float*)(sm + s * ROWS * 128);
      if (issued < total) issue(issued++);
    }
  }
  if (acc == 1234.5f) *out = acc;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int ROWS, int STAGES>
void run(EncodeFn enc, float* x, int nrows, int d, float* out, int sms) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  cuuint32_t box[2] = {32, ROWS};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = STAGES * ROWS * 128 + 1024 + 256;
  cudaFuncSetAttribute(tma_stream<ROWS, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) tma_stream<ROWS, STAGES><<<sms, 64, smem>>>(m, nrows, d / 32, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) tma_stream<ROWS, STAGES><<<sms, 64, smem>>>(m, nrows, d / 32, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("box %3d rows x 128 B, %2d stages (%3d KB in flight): %7.1f GB/s  %s\n", ROWS, STAGES,
         STAGES * ROWS * 128 / 1024, (double)nrows * d * 4 * 5 / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int nrows = 1 << 20, d = 512;
  float *x, *out;
  cudaMalloc(&x, (size_t)nrows * d * 4);
  cudaMalloc(&out, 4);
  cudaMemset(x, 0, (size_t)nrows * d * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  run<256, 4>(enc, x, nrows, d, out, sms);
  run<256, 6>(enc, x, nrows, d, out, sms);
  run<128, 8>(enc, x, nrows, d, out, sms);
  run<128, 12>(enc, x, nrows, d, out, sms);
  run<64, 16>(enc, x, nrows, d, out, sms);
  run<64, 24>(enc, x, nrows, d, out, sms);
  run<32, 32>(enc, x, nrows, d, out, sms);
  return 0;
}
