// fv_util.cu -- error reporting, launch accounting and ABI version.
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "fv_common.cuh"

namespace fv {

static thread_local char g_last_error[512] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(FV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  count_launch();  // successful launches only
  return FV_OK;
}

}  // namespace fv

extern "C" {

int fv_version(void) { return 100; }

const char* fv_last_error(void) { return fv::g_last_error; }

uint64_t fv_launch_count(void) { return fv::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
