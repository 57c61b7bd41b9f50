// Error reporting of the C-ABI: a thread-local message plus sg_status codes.
#include <cstdarg>
#include <cstdio>

#include "sg_device.cuh"

namespace sg {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SG_ECUDA;
  }
  return SG_OK;
}

}  // namespace sg

extern "C" int sg_abi_version(void) { return SG_ABI_VERSION; }

extern "C" const char* sg_last_error(void) { return sg::g_last_error; }
