// ghn_abi.cu -- error reporting and version for the C ABI (include/ghn.h).
#include <atomic>
#include <stdarg.h>
#include <stdio.h>

#include "ghn_common.cuh"

namespace ghn {

static thread_local char g_last_error[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int32_t cuda_status(cudaError_t e, const char *where) {
    set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
    return GHN_ERR_CUDA;
}

}  // namespace ghn

extern "C" const char *ghn_last_error(void) { return ghn::g_last_error; }

extern "C" int32_t ghn_abi_version(void) { return 100; }

extern "C" uint64_t ghn_launch_count(void) { return ghn::g_launches.load(); }
