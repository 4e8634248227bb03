// ghn_common.cuh -- shared device helpers for the GHN sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ghn.h"

#define GHN_FULL 0xffffffffu

namespace ghn {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int32_t cuda_status(cudaError_t e, const char *where);

#define GHN_CUDA_CHECK(expr)                                           \
    do {                                                               \
        cudaError_t _e = (expr);                                       \
        if (_e != cudaSuccess) return ::ghn::cuda_status(_e, #expr);   \
    } while (0)

void count_launch();
int sm_count();   // SMs of the current device (cached)

// Measurement knobs: environment overrides exist only in a tuning build
// (-DGHN_TUNING_KNOBS); the product library always uses the defaults.
#ifdef GHN_TUNING_KNOBS
double knob(const char *name, double dflt);
#else
inline double knob(const char *, double dflt) { return dflt; }
#endif

#define GHN_LAUNCH_CHECK(where)                                        \
    do {                                                               \
        ::ghn::count_launch();                                         \
        cudaError_t _e = cudaGetLastError();                           \
        if (_e != cudaSuccess) return ::ghn::cuda_status(_e, where);   \
    } while (0)

// ---------------------------------------------------------------- numerics
// Cell id: floor(x / w) in IEEE fp64 (grid.py:125, explore.py:91).  When w is
// a power of two, x * (1/w) is the same exactly-representable real value and
// rounds identically, so the reciprocal multiply is bit-exact.
__device__ __forceinline__ int64_t cell_id(double x, double w, double inv_w, bool pow2) {
    double t = pow2 ? __dmul_rn(x, inv_w) : __ddiv_rn(x, w);
    double f = floor(t);
    // clamp far outliers (|id| >= 2^62) so integer arithmetic cannot overflow
    f = fmin(fmax(f, -4.6116860184273879e18), 4.6116860184273879e18);
    return (int64_t)f;
}

// Squared L2 key in numpy's einsum('ij,ij->i') order (core.py:80):
// two SSE2 lanes (even / odd coordinates); each 8-wide chunk is folded as a
// reversed chain of 4 pairs; remaining pairs forward; lane0 + lane1; no FMA.
template <int D>
__device__ __forceinline__ double key_numpy_order(const double (&diff)[D]) {
    double a0 = 0.0, a1 = 0.0;
    int j = 0;
#pragma unroll
    for (int c = 0; c < D / 8; ++c, j += 8) {
#pragma unroll
        for (int p = 3; p >= 0; --p) {
            a0 = __dadd_rn(__dmul_rn(diff[j + 2 * p], diff[j + 2 * p]), a0);
            a1 = __dadd_rn(__dmul_rn(diff[j + 2 * p + 1], diff[j + 2 * p + 1]), a1);
        }
    }
#pragma unroll
    for (; j < D; j += 2) {
        a0 = __dadd_rn(__dmul_rn(diff[j], diff[j]), a0);
        if (j + 1 < D) a1 = __dadd_rn(__dmul_rn(diff[j + 1], diff[j + 1]), a1);
    }
    return __dadd_rn(a0, a1);
}

// Runtime-d variant (d <= GHN_MAX_DIM), same order.
__device__ __forceinline__ double key_numpy_order_rt(const double *diff, int d) {
    double a0 = 0.0, a1 = 0.0;
    int j = 0;
    for (; d - j >= 8; j += 8) {
        for (int p = 3; p >= 0; --p) {
            a0 = __dadd_rn(__dmul_rn(diff[j + 2 * p], diff[j + 2 * p]), a0);
            a1 = __dadd_rn(__dmul_rn(diff[j + 2 * p + 1], diff[j + 2 * p + 1]), a1);
        }
    }
    for (; j < d; j += 2) {
        a0 = __dadd_rn(__dmul_rn(diff[j], diff[j]), a0);
        if (j + 1 < d) a1 = __dadd_rn(__dmul_rn(diff[j + 1], diff[j + 1]), a1);
    }
    return __dadd_rn(a0, a1);
}

// numpy pairwise summation (add.reduce over a contiguous row) of |diff|:
// the manhattan key np.abs(diff).sum(axis=1) (core.py:81-82).  d <= 16.
__device__ __forceinline__ double pairwise_abs_sum(const double *v, int n) {
    if (n < 8) {
        double r = fabs(v[0]);
        for (int i = 1; i < n; ++i) r = __dadd_rn(r, fabs(v[i]));
        return r;
    }
    double acc[8];
    for (int t = 0; t < 8; ++t) acc[t] = fabs(v[t]);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int t = 0; t < 8; ++t) acc[t] = __dadd_rn(acc[t], fabs(v[i + t]));
    double r = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                         __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
    for (; i < n; ++i) r = __dadd_rn(r, fabs(v[i]));
    return r;
}

// Ordering key of a difference vector for a metric (core.py:72-86).
template <int D>
__device__ __forceinline__ double metric_key(const double (&diff)[D], int metric) {
    if (metric == GHN_METRIC_EUCLIDEAN) return key_numpy_order<D>(diff);
    if (metric == GHN_METRIC_MANHATTAN) return pairwise_abs_sum(diff, D);
    double m = fabs(diff[0]);
#pragma unroll
    for (int j = 1; j < D; ++j) m = fmax(m, fabs(diff[j]));
    return m;
}

__device__ __forceinline__ double metric_key_rt(const double *diff, int d, int metric) {
    if (metric == GHN_METRIC_EUCLIDEAN) return key_numpy_order_rt(diff, d);
    if (metric == GHN_METRIC_MANHATTAN) return pairwise_abs_sum(diff, d);
    double m = fabs(diff[0]);
    for (int j = 1; j < d; ++j) m = fmax(m, fabs(diff[j]));
    return m;
}

// Guaranteed-stop bound key for layer l (explore.py:124-125) and the
// reported distance of a key (core.py:89-91).
__device__ __forceinline__ double bound_key(int64_t l, double min_w, int metric) {
    const double b = __dmul_rn((double)l, min_w);
    return metric == GHN_METRIC_EUCLIDEAN ? __dmul_rn(b, b) : b;
}
__device__ __forceinline__ double key_to_dist(double key, int metric) {
    return metric == GHN_METRIC_EUCLIDEAN ? sqrt(key) : key;
}

// (key, index) lexicographic order (explore.py:114).
__device__ __forceinline__ bool pair_less(double ka, int32_t ia, double kb, int32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(GHN_FULL, v, src);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(GHN_FULL, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GHN_FULL, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T u = __shfl_xor_sync(GHN_FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T u = __shfl_xor_sync(GHN_FULL, v, o);
        v = u > v ? u : v;
    }
    return v;
}

__device__ __forceinline__ double to_double(float x) { return (double)x; }
__device__ __forceinline__ double to_double(double x) { return x; }

// ---------------------------------------------------------------- TMA 1-D
// Bulk global -> shared copies (cp.async.bulk, SASS UBLKCP) completing on a
// CTA-local mbarrier: one thread arms the barrier with the byte count and
// issues the copies; every thread waits on the phase.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// bytes: multiple of 16; src / dst 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Issue a copy of any 16-byte multiple in pieces of at most 32 KB.
__device__ __forceinline__ void bulk_g2s_all(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    for (uint32_t o = 0; o < bytes; o += 32768u) {
        const uint32_t b = bytes - o < 32768u ? bytes - o : 32768u;
        bulk_g2s((char *)dst + o, (const char *)src + o, b, bar);
    }
}

// Order-preserving encoding of doubles into uint64 (for atomicMin).
__device__ __forceinline__ unsigned long long dbl_order_key(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dbl_from_order_key(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    memcpy(&v, &b, sizeof(v));
    return v;
}

inline bool is_pow2_width(double w, double *inv) {
    int e;
    double m = frexp(w, &e);
    if (m != 0.5) return false;
    *inv = ldexp(1.0, 1 - e);
    return (*inv) * w == 1.0 && isfinite(*inv) && *inv != 0.0;
}

// ---------------------------------------------------------------- scan / sort
// Device-wide exclusive scan of int32 (in may alias out).  Workspace bytes:
size_t scan_workspace_bytes(int64_t len);
int32_t exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t len, void *ws, cudaStream_t s);

// Stable LSD radix sort of (uint32 key, int32 value) pairs over key bits
// [0, bits).  vals_in == NULL means "values are 0..n-1".  Results land in
// (keys_out, vals_out); the *_tmp buffers are ping-pong scratch.
size_t radix_workspace_bytes(int64_t n);
int32_t radix_sort_pairs(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out,
                         int32_t *vals_out, uint32_t *keys_tmp, int32_t *vals_tmp, int64_t n,
                         int bits, void *ws, cudaStream_t s);

}  // namespace ghn
