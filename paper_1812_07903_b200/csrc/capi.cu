// C-ABI plumbing shared by every entry point: thread-local error message and
// CUDA status mapping (include/levsketch_b200.h).
#include <atomic>
#include <cstdarg>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace lvsk {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int32_t cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return LVSK_ERR_CUDA;
}

static std::atomic<int> g_inflight{1};
int inflight_passes() { return g_inflight.load(std::memory_order_relaxed); }

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev;
}

int num_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int v = 148;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
  cache[dev] = v;
  return v;
}

int32_t ensure_smem_attr(const void* fn, int smem_bytes, const char* what) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int>, int> done;  // (kernel, device) -> bytes set
  const auto key = std::make_tuple(fn, current_device());
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem_bytes) return LVSK_OK;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return cuda_status(e, what);
  done[key] = smem_bytes;
  return LVSK_OK;
}

int resident_ctas(const void* fn, int threads, int smem_bytes) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> cache;
  const auto key = std::make_tuple(fn, current_device(), threads, smem_bytes);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per = 0;
  if (ensure_smem_attr(fn, smem_bytes, "kernel shared-memory attribute") != LVSK_OK ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem_bytes) != cudaSuccess)
    per = 0;
  std::lock_guard<std::mutex> g(mu);
  cache[key] = per;
  return per;
}

}  // namespace lvsk

extern "C" const char* lvsk_last_error(void) { return lvsk::g_last_error; }

extern "C" int32_t lvsk_set_inflight(int32_t passes) {
  if (passes < 1 || passes > 64) {
    lvsk::set_error("lvsk_set_inflight: passes must be in [1, 64], got %d", passes);
    return LVSK_ERR_CONFIGURATION;
  }
  lvsk::g_inflight.store(passes, std::memory_order_relaxed);
  return LVSK_OK;
}

extern "C" int32_t lvsk_get_inflight(void) { return lvsk::inflight_passes(); }

extern "C" int32_t lvsk_abi_version(void) { return 1; }
