// Shared helpers for the levsketch_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/levsketch_b200.h"

namespace lvsk {

// ---------------------------------------------------------------------------
// host-side error plumbing (thread-local last error)

void set_error(const char* fmt, ...);
int32_t cuda_status(cudaError_t e, const char* what);

#define LVSK_CHECK_LAUNCH(what)                                  \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::lvsk::cuda_status(_e, what); \
  } while (0)

#define LVSK_REQUIRE(cond, code, ...)       \
  do {                                      \
    if (!(cond)) {                          \
      ::lvsk::set_error(__VA_ARGS__);       \
      return code;                          \
    }                                       \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Carve {
  char* base;
  size_t cap;
  size_t off = 0;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// size-only twin of Carve, for *_workspace_bytes queries
struct Measure {
  size_t off = 0;
  template <typename T>
  void take(size_t count) {
    off = align_up(off, 256);
    off += count * sizeof(T);
  }
};

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  // splitmix64 finaliser (reference sketch.py:141-148)
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint32_t bucket_hash(uint64_t idx, uint64_t a, uint64_t b, uint64_t size) {
  // multiply-shift on the top 32 bits (reference sketch.py:151-154)
  uint64_t v = a * idx + b;
  return static_cast<uint32_t>(((v >> 32) * size) >> 32);
}

__device__ __forceinline__ bool sign_negative(uint64_t idx, uint64_t key) {
  // sign = 1 - 2*(mix64(idx ^ key) & 1)  (reference sketch.py:157-159)
  return (mix64(idx ^ key) & 1ull) != 0ull;
}

// Knuth TwoSum with explicit round-to-nearest adds (no contraction).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& err) {
  s = __dadd_rn(a, b);
  double bp = __dsub_rn(s, a);
  err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bp)), __dsub_rn(b, bp));
}

// Same (s, err) as two_sum — the rounding error of a + b is unique, so any
// exact method gives the identical bits — via Fast2Sum on the operands ordered
// by magnitude: 3 fp64 adds + one compare, the ordering done with integer
// selects (for finite inputs; a non-finite input is caught by the callers).
__device__ __forceinline__ void two_sum_ordered(double a, double b, double& s, double& err) {
  s = __dadd_rn(a, b);
  const bool a_big = fabs(a) >= fabs(b);
  const double big = a_big ? a : b, small = a_big ? b : a;
  err = __dsub_rn(small, __dsub_rn(s, big));
}

// two_sum(a, -c) with the same bits, without negating c: the sign of a CountSketch
// row is uniform across the warp, so it selects this variant instead of flipping
// every element (negation is exact and round-to-nearest is symmetric).
__device__ __forceinline__ void two_sum_neg(double a, double c, double& s, double& err) {
  s = __dsub_rn(a, c);
  double bp = __dsub_rn(s, a);
  err = __dsub_rn(__dsub_rn(a, __dsub_rn(s, bp)), __dadd_rn(c, bp));
}

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f32<double>(double v) { return static_cast<float>(v); }

template <typename T>
__device__ __forceinline__ double to_f64(T v) { return static_cast<double>(to_f32<T>(v)); }
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }
__device__ __forceinline__ bool finite_f(double v) { return isfinite(v); }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per-device launch facts, cached per (device, kernel) so a process that
// drives several GPUs (torch.cuda.set_device switches) stays correct (capi.cu).
int num_sms();  // SMs of the current device
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
int32_t ensure_smem_attr(const void* fn, int smem_bytes, const char* what);
// co-resident CTAs per SM of `fn` at (threads, smem) on the current device
// (after ensure_smem_attr); 0 when the attribute or the query failed
int resident_ctas(const void* fn, int threads, int smem_bytes);
// passes the caller keeps in flight on separate streams (lvsk_set_inflight);
// >= 2 makes the latency-bound cooperative kernels (KF, K7) take fewer SMs
int inflight_passes();

}  // namespace lvsk
