// ghn_sort.cu -- device-wide exclusive scan and stable LSD radix sort.
//
// These replace np.lexsort's stable grouping (grid.py:188-189): an LSD radix
// sort is stable, and its input is in point-index order, so equal cell keys
// keep input order -- exactly the in-bucket order of the reference.
//
// Radix pass = upsweep (per-tile digit histogram) -> exclusive scan of the
// digit-major count matrix -> downsweep (per-warp in-order ranking with
// __match_any_sync, then scatter).  Tile = 256 threads x 16 keys.
#include <stdio.h>

#include "ghn_common.cuh"

namespace ghn {

// ------------------------------------------------------------------- scan
namespace {
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_IPT;

__device__ __forceinline__ int block_exclusive_scan(int v, int *total) {
    __shared__ int warp_sums[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = warp_inclusive_scan(v);
    if (lane == 31) warp_sums[w] = inc;
    __syncthreads();
    if (w == 0) {
        int s = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
        int si = warp_inclusive_scan(s);
        if (lane < SCAN_THREADS / 32) warp_sums[lane] = si - s;
        if (lane == SCAN_THREADS / 32 - 1) *total = si;
    }
    __syncthreads();
    int r = warp_sums[w] + inc - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const int32_t *in, int64_t len,
                                                                   int32_t *partials) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        int64_t e = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
        if (e < len) s += in[e];
    }
    s = warp_sum(s);
    __shared__ int ws[SCAN_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w) t += ws[w];
        partials[blockIdx.x] = t;
    }
}

// VEC: a thread's 8 elements move as two 16-byte words (in / out 16-byte
// aligned; full tiles only -- the caller routes the tail tile to VEC=false).
template <bool VEC>
__global__ void __launch_bounds__(SCAN_THREADS) scan_downsweep_kernel(const int32_t *in, int32_t *out,
                                                                      int64_t len,
                                                                      const int32_t *partials,
                                                                      int64_t tile0 = 0) {
    const int64_t tile = tile0 + blockIdx.x;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    int v[SCAN_IPT];
    int s = 0;
    if (VEC) {
        const int4 a = reinterpret_cast<const int4 *>(in + base)[0];
        const int4 b = reinterpret_cast<const int4 *>(in + base)[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
#pragma unroll
        for (int i = 0; i < SCAN_IPT; ++i) s += v[i];
    } else {
#pragma unroll
        for (int i = 0; i < SCAN_IPT; ++i) {
            int64_t e = base + i;
            v[i] = e < len ? in[e] : 0;
            s += v[i];
        }
    }
    int total;
    int ex = block_exclusive_scan(s, &total);
    int run = ex + (partials ? partials[tile] : 0);
    if (VEC) {
        int r[SCAN_IPT];
#pragma unroll
        for (int i = 0; i < SCAN_IPT; ++i) {
            r[i] = run;
            run += v[i];
        }
        reinterpret_cast<int4 *>(out + base)[0] = make_int4(r[0], r[1], r[2], r[3]);
        reinterpret_cast<int4 *>(out + base)[1] = make_int4(r[4], r[5], r[6], r[7]);
    } else {
#pragma unroll
        for (int i = 0; i < SCAN_IPT; ++i) {
            int64_t e = base + i;
            if (e < len) out[e] = run;
            run += v[i];
        }
    }
}
static_assert(SCAN_IPT == 8, "the VEC downsweep moves 8 elements per thread");
}  // namespace

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t scan_workspace_bytes(int64_t len) {
    size_t bytes = 0;
    int64_t m = len;
    while (m > SCAN_TILE) {
        m = ceil_div(m, SCAN_TILE);
        bytes += ((size_t)m * 4 + 255) & ~(size_t)255;
    }
    return bytes + 256;
}

int32_t exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t len, void *ws, cudaStream_t s) {
    if (len <= 0) return GHN_OK;
    int64_t nb = ceil_div(len, SCAN_TILE);
    if (nb == 1) {
        scan_downsweep_kernel<false><<<1, SCAN_THREADS, 0, s>>>(in, out, len, nullptr);
        GHN_LAUNCH_CHECK("scan_downsweep_kernel");
        return GHN_OK;
    }
    int32_t *partials = (int32_t *)ws;
    void *ws_next = (char *)ws + (((size_t)nb * 4 + 255) & ~(size_t)255);
    scan_reduce_kernel<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, len, partials);
    GHN_LAUNCH_CHECK("scan_reduce_kernel");
    int32_t rc = exclusive_scan_i32(partials, partials, nb, ws_next, s);
    if (rc != GHN_OK) return rc;
    const int64_t full = len / SCAN_TILE;   // complete tiles
    if ((((uintptr_t)in | (uintptr_t)out) & 15) == 0 && full > 0) {
        scan_downsweep_kernel<true><<<(unsigned)full, SCAN_THREADS, 0, s>>>(in, out, len, partials);
        GHN_LAUNCH_CHECK("scan_downsweep_kernel");
        if (full < nb) {
            scan_downsweep_kernel<false><<<(unsigned)(nb - full), SCAN_THREADS, 0, s>>>(in, out, len, partials, full);
            GHN_LAUNCH_CHECK("scan_downsweep_kernel");
        }
        return GHN_OK;
    }
    scan_downsweep_kernel<false><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, len, partials);
    GHN_LAUNCH_CHECK("scan_downsweep_kernel");
    return GHN_OK;
}

// ------------------------------------------------------------------- radix
namespace {
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_IPT = 16;                       // keys per lane
constexpr int RS_TILE = RS_THREADS * RS_IPT;     // 4096 keys per CTA
constexpr int RS_MAX_BITS = 8;

__global__ void __launch_bounds__(RS_THREADS) radix_upsweep_kernel(const uint32_t *keys, int64_t n,
                                                                   int shift, int nbits,
                                                                   int32_t *counts, int nb) {
    __shared__ int hist[1 << RS_MAX_BITS];
    const int radix = 1 << nbits;
    const uint32_t mask = (uint32_t)radix - 1u;
    for (int i = threadIdx.x; i < radix; i += RS_THREADS) hist[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int i = 0; i < RS_IPT; ++i) {
        int64_t e = base + (int64_t)i * RS_THREADS + threadIdx.x;
        if (e < n) atomicAdd(&hist[(keys[e] >> shift) & mask], 1);
    }
    __syncthreads();
    for (int dg = threadIdx.x; dg < radix; dg += RS_THREADS)
        counts[(int64_t)dg * nb + blockIdx.x] = hist[dg];
}

template <bool IDENT>
__global__ void __launch_bounds__(RS_THREADS) radix_downsweep_kernel(
    const uint32_t *__restrict__ kin, const int32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    int32_t *__restrict__ vout, int64_t n, int shift, int nbits, const int32_t *__restrict__ offsets,
    int nb) {
    __shared__ int cnt[RS_WARPS][1 << RS_MAX_BITS];
    __shared__ int gbase[1 << RS_MAX_BITS];
    const int radix = 1 << nbits;
    const uint32_t mask = (uint32_t)radix - 1u;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * (1 << RS_MAX_BITS); i += RS_THREADS) (&cnt[0][0])[i] = 0;
    for (int dg = threadIdx.x; dg < radix; dg += RS_THREADS)
        gbase[dg] = offsets[(int64_t)dg * nb + blockIdx.x];
    __syncthreads();
    // warp w owns keys [base, base + 32*RS_IPT) of the tile, ranked in order
    const int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * 32 * RS_IPT;
    uint32_t key[RS_IPT];
    int32_t val[RS_IPT];
    int rank[RS_IPT];
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < RS_IPT; ++r) {
        const int64_t e = base + r * 32 + lane;
        const bool act = e < n;
        const unsigned am = __ballot_sync(GHN_FULL, act);
        if (act) {
            key[r] = kin[e];
            val[r] = IDENT ? (int32_t)e : vin[e];
            const int dg = (int)((key[r] >> shift) & mask);
            const unsigned peers = __match_any_sync(am, dg);
            const int before = __popc(peers & lt);
            rank[r] = cnt[w][dg] + before;
            __syncwarp(am);
            if (before == 0) cnt[w][dg] += __popc(peers);
            __syncwarp(am);
        }
    }
    __syncthreads();
    for (int dg = threadIdx.x; dg < radix; dg += RS_THREADS) {
        int s = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            int c = cnt[ww][dg];
            cnt[ww][dg] = s;
            s += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_IPT; ++r) {
        const int64_t e = base + r * 32 + lane;
        if (e < n) {
            const int dg = (int)((key[r] >> shift) & mask);
            const int64_t pos = (int64_t)gbase[dg] + cnt[w][dg] + rank[r];
            kout[pos] = key[r];
            vout[pos] = val[r];
        }
    }
}

__global__ void iota_kernel(int32_t *v, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
}
}  // namespace

size_t radix_workspace_bytes(int64_t n) {
    int64_t nb = ceil_div(n > 0 ? n : 1, RS_TILE);
    int64_t cnt = nb << RS_MAX_BITS;
    return (((size_t)cnt * 4 + 255) & ~(size_t)255) + scan_workspace_bytes(cnt);
}

int32_t radix_sort_pairs(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out,
                         int32_t *vals_out, uint32_t *keys_tmp, int32_t *vals_tmp, int64_t n,
                         int bits, void *ws, cudaStream_t s) {
    if (n <= 0) return GHN_OK;
    if (bits <= 0) {
        GHN_CUDA_CHECK(cudaMemcpyAsync(keys_out, keys_in, n * 4, cudaMemcpyDeviceToDevice, s));
        if (vals_in) {
            GHN_CUDA_CHECK(cudaMemcpyAsync(vals_out, vals_in, n * 4, cudaMemcpyDeviceToDevice, s));
        } else {
            iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(vals_out, n);
            GHN_LAUNCH_CHECK("iota_kernel");
        }
        return GHN_OK;
    }
    const int passes = (bits + RS_MAX_BITS - 1) / RS_MAX_BITS;
    const int per = (bits + passes - 1) / passes;
    const int64_t nb = ceil_div(n, RS_TILE);
    if (nb > 0x7fffffff / (1 << RS_MAX_BITS)) {
        set_error("radix_sort_pairs: n=%lld too large", (long long)n);
        return GHN_ERR_UNSUPPORTED;
    }
    int32_t *counts = (int32_t *)ws;
    void *scan_ws = (char *)ws + ((((size_t)nb << RS_MAX_BITS) * 4 + 255) & ~(size_t)255);
    const uint32_t *ksrc = keys_in;
    const int32_t *vsrc = vals_in;
    for (int p = 0; p < passes; ++p) {
        const int shift = p * per;
        const int nbits = (bits - shift) < per ? (bits - shift) : per;
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        uint32_t *kdst = to_out ? keys_out : keys_tmp;
        int32_t *vdst = to_out ? vals_out : vals_tmp;
        radix_upsweep_kernel<<<(unsigned)nb, RS_THREADS, 0, s>>>(ksrc, n, shift, nbits, counts, (int)nb);
        GHN_LAUNCH_CHECK("radix_upsweep_kernel");
        int32_t rc = exclusive_scan_i32(counts, counts, nb << nbits, scan_ws, s);
        if (rc != GHN_OK) return rc;
        if (vsrc == nullptr)
            radix_downsweep_kernel<true><<<(unsigned)nb, RS_THREADS, 0, s>>>(
                ksrc, nullptr, kdst, vdst, n, shift, nbits, counts, (int)nb);
        else
            radix_downsweep_kernel<false><<<(unsigned)nb, RS_THREADS, 0, s>>>(
                ksrc, vsrc, kdst, vdst, n, shift, nbits, counts, (int)nb);
        GHN_LAUNCH_CHECK("radix_downsweep_kernel");
        ksrc = kdst;
        vsrc = vdst;
    }
    return GHN_OK;
}

}  // namespace ghn
