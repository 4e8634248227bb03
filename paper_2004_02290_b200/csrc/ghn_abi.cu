// ghn_abi.cu -- error reporting and version for the C ABI (include/ghn.h).
#include <atomic>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

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

// Streaming multiprocessors of the current device (grid sizing), cached per
// device; 148 on B200.
int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
    if (dev < 64) {
        const int c = cache[dev].load(std::memory_order_relaxed);
        if (c > 0) return c;
    }
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
    if (dev < 64) cache[dev].store(v, std::memory_order_relaxed);
    return v;
}

#ifdef GHN_TUNING_KNOBS
double knob(const char *name, double dflt) {
    const char *e = getenv(name);
    return e ? atof(e) : dflt;
}
#endif

int32_t cuda_status(cudaError_t e, const char *where) {
    set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
    return GHN_ERR_CUDA;
}

}  // namespace ghn

extern "C" const char *ghn_last_error(void) { return ghn::g_last_error; }

extern "C" int32_t ghn_abi_version(void) { return 200; }

extern "C" int32_t ghn_build_flags(void) {
    int32_t f = 0;
#ifdef GHN_TUNING_KNOBS
    f |= 1;
#endif
#ifdef GHN_FB_REASONS
    f |= 2;
#endif
    return f;
}

extern "C" uint64_t ghn_launch_count(void) { return ghn::g_launches.load(); }
