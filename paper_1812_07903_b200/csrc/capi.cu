// C-ABI plumbing shared by every entry point: thread-local error message and
// CUDA status mapping (include/levsketch_b200.h).
#include <cstdarg>

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

}  // namespace lvsk

extern "C" const char* lvsk_last_error(void) { return lvsk::g_last_error; }

extern "C" int32_t lvsk_abi_version(void) { return 1; }
