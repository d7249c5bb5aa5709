// Yardstick only (not product code): CUB onesweep SortPairs on 64-bit keys +
// 32-bit values, the shape of K7 (argsort for make_plan), event-timed.
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>

int main() {
  for (int n : {100000, 1000000, 4000000}) {
    std::vector<uint64_t> hk(n);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hk[i] = (0x3EBull << 52) | (x >> 12); }
    uint64_t *k0, *k1; uint32_t *v0, *v1;
    cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    cudaMemcpy(k0, hk.data(), n * 8, cudaMemcpyHostToDevice);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, n, 0, 64);
    void* tmp; cudaMalloc(&tmp, tb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bits : {64, 56}) {
      cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, bits);
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, bits);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("cub SortPairs n=%d bits=%d: %.1f us\n", n, bits, ms / 20 * 1000);
    }
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tmp);
  }
  return 0;
}
