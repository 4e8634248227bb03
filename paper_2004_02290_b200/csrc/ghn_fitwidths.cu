// ghn_fitwidths.cu -- max-splits cell-width fit on the device (K7).
//
// Replaces grid.fit_cell_measurements / _max_splits_1d (grid.py:47-109).
// Per dimension:
//   1. order-preserving integer keys of the fp64 values, LSD radix sort
//      (32-bit keys for fp32 data, two 32-bit halves for fp64);
//   2. distinct values u (np.unique), gaps g = diff(u) (np.diff, fp64),
//      max gap, span = u[-1] - u[0];
//   3. s_hi = min(#distinct, ceil(2 span / max_gap), cap) on the host;
//   4. the gaps wider than span / s_hi (a superset of every smaller s's
//      "wide" set, grid.py:75-76) are compacted with their end points;
//   5. candidate split counts s = s_hi, s_hi-1, ... are checked in parallel
//      batches: s passes iff every gap g > span/s keeps
//      bin(right) - bin(left) <= 1 with bin(v) = min(floor(((v - lo) * s) / span), s - 1)
//      (grid.py:47-49, 79-82); the largest passing s wins, exactly what the
//      reference's descending loop returns.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "ghn_common.cuh"

namespace ghn {
namespace {

constexpr int FW_THREADS = 256;

__device__ __forceinline__ uint64_t dkey(double v) {
    uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
__global__ void keys_kernel(const T *__restrict__ X, int64_t n, int d, int j, uint32_t *lo, uint32_t *hi) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = dkey(to_double(X[i * d + j]));
        lo[i] = (uint32_t)k;
        if (hi) hi[i] = (uint32_t)(k >> 32);
    }
}

// fp32 data: the float's own order-preserving 32-bit key.
__global__ void keys32_kernel(const float *__restrict__ X, int64_t n, int d, int j, uint32_t *k32) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = __float_as_uint(X[i * d + j]);
        k32[i] = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    }
}

__global__ void gather_u32_kernel(const uint32_t *__restrict__ src, const int32_t *__restrict__ idx, int64_t n,
                                  uint32_t *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

template <typename T>
__global__ void sorted_values_kernel(const T *__restrict__ X, int64_t n, int d, int j,
                                     const int32_t *__restrict__ perm, double *__restrict__ vs,
                                     int32_t *__restrict__ flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = to_double(X[(int64_t)perm[i] * d + j]);
        vs[i] = v;
        flags[i] = i == 0 || v != to_double(X[(int64_t)perm[i - 1] * d + j]) ? 1 : 0;
    }
}

__global__ void compact_distinct_kernel(const double *__restrict__ vs, const int32_t *__restrict__ flags,
                                        const int32_t *__restrict__ pos, int64_t n, double *__restrict__ u) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (flags[i]) u[pos[i]] = vs[i];
}

__global__ void max_gap_kernel(const double *__restrict__ u, int64_t m, unsigned long long *out) {
    double best = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < m;
         i += (int64_t)gridDim.x * blockDim.x)
        best = fmax(best, __dsub_rn(u[i + 1], u[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(GHN_FULL, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

__global__ void wide_flags_kernel(const double *__restrict__ u, int64_t m, double thr, int32_t *__restrict__ flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < m;
         i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = __dsub_rn(u[i + 1], u[i]) > thr ? 1 : 0;
}

__global__ void wide_compact_kernel(const double *__restrict__ u, int64_t m, const int32_t *__restrict__ flags,
                                    const int32_t *__restrict__ pos, double *__restrict__ wl,
                                    double *__restrict__ wr, double *__restrict__ wg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < m;
         i += (int64_t)gridDim.x * blockDim.x)
        if (flags[i]) {
            const int32_t p = pos[i];
            wl[p] = u[i];
            wr[p] = u[i + 1];
            wg[p] = __dsub_rn(u[i + 1], u[i]);
        }
}

__device__ __forceinline__ double bin_of(double v, double lo, double s, double span, double smax) {
    // grid.py:49: np.minimum(np.floor((values - lo) * s / span), s - 1)
    return fmin(floor(__ddiv_rn(__dmul_rn(__dsub_rn(v, lo), s), span)), smax);
}

// ok[t] for s = s_top - t: every wide gap (g > span / s) keeps bins adjacent.
__global__ void check_splits_kernel(const double *__restrict__ wl, const double *__restrict__ wr,
                                    const double *__restrict__ wg, int64_t W, double lo, double span,
                                    int64_t s_top, int64_t count, uint8_t *__restrict__ ok) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t si = s_top - t;
        const double s = (double)si;
        const double thr = __ddiv_rn(span, s);
        const double smax = (double)(si - 1);
        bool good = true;
        for (int64_t e = 0; e < W && good; ++e) {
            if (wg[e] > thr)
                good = bin_of(wr[e], lo, s, span, smax) - bin_of(wl[e], lo, s, span, smax) <= 1.0;
        }
        ok[t] = good ? 1 : 0;
    }
}

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

unsigned grid_of(int64_t n) {
    int64_t b = (n + FW_THREADS - 1) / FW_THREADS;
    if (b > sm_count() * 16) b = sm_count() * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

constexpr int64_t CHECK_BATCH = 1 << 16;

template <typename T>
int32_t fit_widths_impl(const T *X, int64_t n, int d, int64_t cap, double *widths, int64_t *splits,
                        double *origin, char *ws, cudaStream_t s) {
    const size_t n4 = a256((size_t)n * 4), n8 = a256((size_t)n * 8);
    uint32_t *klo = (uint32_t *)ws;
    uint32_t *khi = (uint32_t *)(ws + n4);
    uint32_t *ksort = (uint32_t *)(ws + 2 * n4);
    uint32_t *ktmp = (uint32_t *)(ws + 3 * n4);
    int32_t *p1 = (int32_t *)(ws + 4 * n4);
    int32_t *p2 = (int32_t *)(ws + 5 * n4);
    int32_t *vtmp = (int32_t *)(ws + 6 * n4);
    int32_t *flags = (int32_t *)(ws + 7 * n4);
    int32_t *pos = (int32_t *)(ws + 8 * n4);
    double *vs = (double *)(ws + 9 * n4);
    double *u = (double *)(ws + 9 * n4 + n8);
    double *wl = (double *)(ws + 9 * n4 + 2 * n8);
    double *wr = (double *)(ws + 9 * n4 + 3 * n8);
    double *wg = (double *)(ws + 9 * n4 + 4 * n8);
    unsigned long long *dmax = (unsigned long long *)(ws + 9 * n4 + 5 * n8);
    uint8_t *ok = (uint8_t *)(ws + 9 * n4 + 5 * n8 + 256);
    char *rws = ws + 9 * n4 + 5 * n8 + 256 + a256(CHECK_BATCH);
    char *sws = rws + a256(radix_workspace_bytes(n));
    const unsigned g = grid_of(n);
    static uint8_t hok[CHECK_BATCH];
    for (int j = 0; j < d; ++j) {
        // 1. sort the column (order-preserving keys; fp64 needs two 32-bit passes)
        const bool wide = sizeof(T) == 8;
        int32_t *perm = p1;
        int32_t rc;
        if (wide) {
            keys_kernel<T><<<g, FW_THREADS, 0, s>>>(X, n, d, j, klo, khi);
            GHN_LAUNCH_CHECK("keys_kernel");
            rc = radix_sort_pairs(klo, nullptr, ksort, p1, ktmp, vtmp, n, 32, rws, s);
            if (rc) return rc;
            gather_u32_kernel<<<g, FW_THREADS, 0, s>>>(khi, p1, n, klo);
            GHN_LAUNCH_CHECK("gather_u32_kernel");
            rc = radix_sort_pairs(klo, p1, ksort, p2, ktmp, vtmp, n, 32, rws, s);
            if (rc) return rc;
            perm = p2;
        } else {
            keys32_kernel<<<g, FW_THREADS, 0, s>>>((const float *)X, n, d, j, klo);
            GHN_LAUNCH_CHECK("keys32_kernel");
            rc = radix_sort_pairs(klo, nullptr, ksort, p1, ktmp, vtmp, n, 32, rws, s);
            if (rc) return rc;
        }
        // 2. distinct values, gaps, span
        sorted_values_kernel<T><<<g, FW_THREADS, 0, s>>>(X, n, d, j, perm, vs, flags);
        GHN_LAUNCH_CHECK("sorted_values_kernel");
        rc = exclusive_scan_i32(flags, pos, n, sws, s);
        if (rc) return rc;
        compact_distinct_kernel<<<g, FW_THREADS, 0, s>>>(vs, flags, pos, n, u);
        GHN_LAUNCH_CHECK("compact_distinct_kernel");
        int32_t lastpos = 0, lastflag = 0;
        GHN_CUDA_CHECK(cudaMemcpyAsync(&lastpos, pos + n - 1, 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaMemcpyAsync(&lastflag, flags + n - 1, 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        const int64_t m = (int64_t)lastpos + lastflag;
        GHN_CUDA_CHECK(cudaMemcpyAsync(&origin[j], u, 8, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        if (m == 1) {   // constant feature (grid.py:60-61)
            splits[j] = 1;
            widths[j] = 1.0;
            continue;
        }
        double ulo = 0.0, uhi = 0.0;
        GHN_CUDA_CHECK(cudaMemsetAsync(dmax, 0, 8, s));
        max_gap_kernel<<<grid_of(m), FW_THREADS, 0, s>>>(u, m, dmax);
        GHN_LAUNCH_CHECK("max_gap_kernel");
        unsigned long long hmax = 0;
        GHN_CUDA_CHECK(cudaMemcpyAsync(&ulo, u, 8, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaMemcpyAsync(&uhi, u + m - 1, 8, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaMemcpyAsync(&hmax, dmax, 8, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        double max_gap;
        memcpy(&max_gap, &hmax, 8);
        const double lo = ulo, span = uhi - ulo;
        // 3. s_hi (grid.py:67-70)
        int64_t s_hi = (int64_t)ceil(2.0 * span / max_gap);
        if (m < s_hi) s_hi = m;
        if (cap > 0 && cap < s_hi) s_hi = cap;
        if (s_hi < 2) {
            splits[j] = 1;
            widths[j] = span;
            continue;
        }
        // 4. the gaps wider than span / s_hi
        wide_flags_kernel<<<grid_of(m), FW_THREADS, 0, s>>>(u, m, span / (double)s_hi, flags);
        GHN_LAUNCH_CHECK("wide_flags_kernel");
        rc = exclusive_scan_i32(flags, pos, m - 1, sws, s);
        if (rc) return rc;
        wide_compact_kernel<<<grid_of(m), FW_THREADS, 0, s>>>(u, m, flags, pos, wl, wr, wg);
        GHN_LAUNCH_CHECK("wide_compact_kernel");
        GHN_CUDA_CHECK(cudaMemcpyAsync(&lastpos, pos + m - 2, 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaMemcpyAsync(&lastflag, flags + m - 2, 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        const int64_t W = (int64_t)lastpos + lastflag;
        // 5. descending candidates, in parallel batches
        int64_t best = -1;
        for (int64_t top = s_hi; top >= 2 && best < 0; top -= CHECK_BATCH) {
            const int64_t count = top - 1 < CHECK_BATCH ? top - 1 : CHECK_BATCH;
            check_splits_kernel<<<grid_of(count), FW_THREADS, 0, s>>>(wl, wr, wg, W, lo, span, top, count, ok);
            GHN_LAUNCH_CHECK("check_splits_kernel");
            GHN_CUDA_CHECK(cudaMemcpyAsync(hok, ok, (size_t)count, cudaMemcpyDeviceToHost, s));
            GHN_CUDA_CHECK(cudaStreamSynchronize(s));
            for (int64_t t = 0; t < count; ++t)
                if (hok[t]) {
                    best = top - t;
                    break;
                }
        }
        if (best < 0) {
            splits[j] = 1;
            widths[j] = span;
        } else {
            splits[j] = best;
            widths[j] = span / (double)best;
        }
    }
    return GHN_OK;
}

}  // namespace
}  // namespace ghn

using namespace ghn;

extern "C" size_t ghn_fit_widths_workspace_size(int64_t n) {
    const size_t n4 = a256((size_t)(n > 0 ? n : 1) * 4), n8 = a256((size_t)(n > 0 ? n : 1) * 8);
    return 9 * n4 + 5 * n8 + 256 + a256(CHECK_BATCH) + a256(radix_workspace_bytes(n > 0 ? n : 1)) +
           scan_workspace_bytes(n > 0 ? n : 1) + 256;
}

extern "C" int32_t ghn_fit_widths(const void *X, int32_t dtype, int64_t n, int32_t d, int64_t max_splits,
                                  double *widths, int64_t *splits, double *origin, void *workspace,
                                  size_t workspace_bytes, void *stream) {
    if (n <= 0) {
        set_error("empty dataset");
        return GHN_ERR_VALUE;
    }
    if (d < 1 || d > GHN_MAX_DIM) {
        set_error("d=%d unsupported", d);
        return GHN_ERR_UNSUPPORTED;
    }
    if (n > 0x7ffffffeLL) {
        set_error("n=%lld too large", (long long)n);
        return GHN_ERR_UNSUPPORTED;
    }
    if (workspace_bytes < ghn_fit_widths_workspace_size(n)) {
        set_error("fit_widths workspace too small");
        return GHN_ERR_VALUE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == GHN_F32)
        return fit_widths_impl<float>((const float *)X, n, d, max_splits, widths, splits, origin,
                                      (char *)workspace, s);
    return fit_widths_impl<double>((const double *)X, n, d, max_splits, widths, splits, origin,
                                   (char *)workspace, s);
}
