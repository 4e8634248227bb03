// ghn_fit.cu -- grid build (fit) for sm_100a.
//
// Replaces grid.build (grid.py:165-195):
//   K1 bounds   per-dim min/max of floor(x/w), origin = min coordinate,
//               non-finite check (core.py:35-36)                 [HBM read n*d]
//   K2 keys     row-major linear cell key over the id bounding box
//               (dim 0 most significant == lexicographic order)   [read n*d, write 4n]
//   K5 sort     stable LSD radix sort of (key, index)  == lexsort((arange, ids...))
//   K6 cells    run boundaries -> cell_start / cell_ids (== cell_array, buckets)
//   K4 dense    ne_off (non-empty prefix) and pt_off (slot prefix) over E cells
//   gather      permuted SoA coordinates coords[j*n + slot]
// LIST layout (huge sparse boxes): one stable radix sort per dimension,
// last dimension first (the lexsort key order), no dense tables.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "ghn_common.cuh"

namespace ghn {
namespace {

constexpr int FIT_THREADS = 256;

struct DimParams {
    double w[GHN_MAX_DIM];
    double inv[GHN_MAX_DIM];
    int64_t lo[GHN_MAX_DIM];
    int64_t ext[GHN_MAX_DIM];
    uint32_t pow2;   // bit j: widths[j] is a power of two
    int32_t d;
    // bit j: fp32 coordinates get their id as floor(x * inv) in fp32 --
    // identical to the fp64 division: 1/w is a power of two >= 1, so the
    // product is exact in fp32 (no rounding, no underflow) and |id| < 2^30
    uint32_t fast32;
    float inv32[GHN_MAX_DIM];
};

static DimParams make_dims(int d, const double *widths, const int64_t *lo, const int64_t *ext) {
    DimParams p;
    memset(&p, 0, sizeof(p));
    p.d = d;
    for (int j = 0; j < d; ++j) {
        p.w[j] = widths[j];
        double inv = 0.0;
        if (is_pow2_width(widths[j], &inv)) {
            p.pow2 |= 1u << j;
            p.inv[j] = inv;
        }
        if (lo) p.lo[j] = lo[j];
        if (ext) p.ext[j] = ext[j];
        if (lo && ext && ((p.pow2 >> j) & 1u) && inv >= 1.0 && inv <= 0x1p100 && lo[j] > -(1LL << 30) &&
            lo[j] + ext[j] < (1LL << 30)) {
            p.fast32 |= 1u << j;
            p.inv32[j] = (float)inv;
        }
    }
    return p;
}

__global__ void bounds_init_kernel(int64_t *bounds, unsigned long long *origin_key, int32_t *flags,
                                   int d) {
    int j = threadIdx.x;
    if (j < d) {   // order keys of the min (origin_key) and max (bounds[d + j]) coordinates
        bounds[j] = 0;
        bounds[d + j] = 0;
        origin_key[j] = ~0ull;
    }
    if (j == 0) *flags = 0;
}

// K1: D > 0 compile-time dims.  floor(x / w) is monotone in x, so the id
// bounds are the ids of the per-dimension min / max coordinates: the pass
// only reduces min / max (and the non-finite flag) in the input type, and
// origin_decode_kernel turns them into ids.  Keys staged as order-preserving
// uint64 (min in origin_key, max in bounds[d + j]).
template <typename T, int D>
__global__ void __launch_bounds__(FIT_THREADS) bounds_kernel(const T *__restrict__ X, int64_t n,
                                                             DimParams p, int64_t *bounds,
                                                             unsigned long long *origin_key,
                                                             int32_t *flags) {
    T mn[D], mx[D];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        mn[j] = (T)INFINITY;
        mx[j] = (T)-INFINITY;
    }
    // BU points per thread per iteration, loads issued first
    constexpr int BU = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (BU - 1) * stride < n; i += BU * stride) {
        T v[BU][D];
#pragma unroll
        for (int u = 0; u < BU; ++u)
#pragma unroll
            for (int j = 0; j < D; ++j) v[u][j] = __ldcs(X + (i + u * stride) * D + j);
#pragma unroll
        for (int u = 0; u < BU; ++u)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                bad |= !isfinite(v[u][j]);
                mn[j] = fmin(mn[j], v[u][j]);
                mx[j] = fmax(mx[j], v[u][j]);
            }
    }
    for (; i < n; i += stride) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const T x = X[i * D + j];
            bad |= !isfinite(x);
            mn[j] = fmin(mn[j], x);
            mx[j] = fmax(mx[j], x);
        }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double m = to_double(mn[j]), M = to_double(mx[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m = fmin(m, __shfl_xor_sync(GHN_FULL, m, o));
            M = fmax(M, __shfl_xor_sync(GHN_FULL, M, o));
        }
        if ((threadIdx.x & 31) == 0) {
            if (m != INFINITY) atomicMin(&origin_key[j], dbl_order_key(m));
            if (M != -INFINITY) atomicMax((unsigned long long *)&bounds[D + j], dbl_order_key(M));
        }
    }
    if (__any_sync(GHN_FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
}

// K1 for runtime d (up to GHN_MAX_DIM): element-parallel with global atomics per warp-run.
template <typename T>
__global__ void __launch_bounds__(FIT_THREADS) bounds_kernel_rt(const T *__restrict__ X, int64_t n,
                                                                DimParams p, int64_t *bounds,
                                                                unsigned long long *origin_key,
                                                                int32_t *flags) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int j = 0; j < d; ++j) {
            double x = to_double(X[i * d + j]);
            if (!isfinite(x)) {
                atomicOr(flags, 1);
                continue;
            }
            atomicMin(&origin_key[j], dbl_order_key(x));
            atomicMax((unsigned long long *)&bounds[d + j], dbl_order_key(x));
        }
    }
}

__global__ void origin_decode_kernel(const unsigned long long *origin_key, double *origin, int64_t *bounds,
                                     DimParams p) {
    const int j = threadIdx.x, d = p.d;
    if (j < d) {
        const double mn = dbl_from_order_key(origin_key[j]);
        const double mx = dbl_from_order_key((unsigned long long)bounds[d + j]);
        origin[j] = mn;
        bounds[j] = cell_id(mn, p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
        bounds[d + j] = cell_id(mx, p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
    }
}

// K2: linear key over the bbox, row-major with dim 0 most significant.
template <typename T>
__global__ void __launch_bounds__(FIT_THREADS) linear_key_kernel(const T *__restrict__ X, int64_t n,
                                                                 DimParams p,
                                                                 uint32_t *__restrict__ keys) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = 0;
        for (int j = 0; j < d; ++j) {
            int64_t c = cell_id(to_double(X[i * d + j]), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
            key = key * (uint64_t)p.ext[j] + (uint64_t)(c - p.lo[j]);
        }
        keys[i] = (uint32_t)key;
    }
}

// LIST layout: relative id of dimension j for the point at slot i of perm.
template <typename T>
__global__ void __launch_bounds__(FIT_THREADS) dim_key_kernel(const T *__restrict__ X, int64_t n,
                                                              DimParams p, int j,
                                                              const int32_t *__restrict__ perm,
                                                              uint32_t *__restrict__ keys) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t src = perm ? perm[i] : i;
        int64_t c = cell_id(to_double(X[src * d + j]), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
        keys[i] = (uint32_t)(c - p.lo[j]);
    }
}

// K6 (DENSE): boundary flags from sorted linear keys.
__global__ void dense_flags_kernel(const uint32_t *__restrict__ skeys, int64_t n, int32_t *flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1 : 0;
}

__global__ void dense_emit_kernel(const uint32_t *__restrict__ skeys, int64_t n,
                                  const int32_t *__restrict__ cidx, DimParams p,
                                  int32_t *__restrict__ cell_start, int32_t *__restrict__ cell_ids,
                                  int32_t *__restrict__ n_cells, int32_t *__restrict__ ne_flag) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool head = (i == 0 || skeys[i] != skeys[i - 1]);
        if (head) {
            int32_t c = cidx[i];
            cell_start[c] = (int32_t)i;
            uint64_t rem = skeys[i];
            for (int j = d - 1; j >= 0; --j) {
                cell_ids[(int64_t)c * d + j] = (int32_t)(rem % (uint64_t)p.ext[j]);
                rem /= (uint64_t)p.ext[j];
            }
            if (ne_flag) ne_flag[skeys[i]] = 1;
        }
        if (i == n - 1) {
            int32_t total = cidx[i] + 1;
            *n_cells = total;
            cell_start[total] = (int32_t)n;
        }
    }
}

// K6 (LIST): boundary flags by comparing the id tuples of consecutive slots.
template <typename T>
__global__ void list_flags_kernel(const T *__restrict__ X, int64_t n, DimParams p,
                                  const int32_t *__restrict__ perm, int32_t *flags) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int f = 0;
        if (i == 0) {
            f = 1;
        } else {
            int64_t a = perm[i], b = perm[i - 1];
            for (int j = 0; j < d; ++j) {
                bool pw = (p.pow2 >> j) & 1u;
                if (cell_id(to_double(X[a * d + j]), p.w[j], p.inv[j], pw) !=
                    cell_id(to_double(X[b * d + j]), p.w[j], p.inv[j], pw)) {
                    f = 1;
                    break;
                }
            }
        }
        flags[i] = f;
    }
}

template <typename T>
__global__ void list_emit_kernel(const T *__restrict__ X, int64_t n, DimParams p,
                                 const int32_t *__restrict__ perm, const int32_t *__restrict__ cidx,
                                 int32_t *__restrict__ cell_start, int32_t *__restrict__ cell_ids,
                                 int32_t *__restrict__ n_cells) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = cidx[i];
        int32_t cnext = (i + 1 < n) ? cidx[i + 1] : -1;
        bool head = (i == 0) || (cidx[i - 1] != c);
        (void)cnext;
        if (head) {
            cell_start[c] = (int32_t)i;
            int64_t a = perm[i];
            for (int j = 0; j < d; ++j) {
                int64_t id = cell_id(to_double(X[a * d + j]), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
                cell_ids[(int64_t)c * d + j] = (int32_t)(id - p.lo[j]);
            }
        }
        if (i == n - 1) {
            *n_cells = c + 1;
            cell_start[c + 1] = (int32_t)n;
        }
    }
}

// inclusive-to-cell-index: cidx[i] = (# heads in [0, i]) - 1, from an exclusive scan of flags.
__global__ void excl_to_cidx_kernel(const int32_t *__restrict__ flags_excl,
                                    const int32_t *__restrict__ flags, int32_t *cidx, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        cidx[i] = flags_excl[i] + flags[i] - 1;
}

// K4 (DENSE): pt_off[c] = cell_start[ne_off[c]] for c in [0, E].
__global__ void pt_off_kernel(const int32_t *__restrict__ ne_off, const int32_t *__restrict__ cell_start,
                              int32_t *__restrict__ pt_off, int64_t len) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < len;
         c += (int64_t)gridDim.x * blockDim.x)
        pt_off[c] = cell_start[ne_off[c]];
}

// Permuted SoA coordinates (+ labels in slot order when requested): one
// random gather per point; a point's d coordinates are adjacent in X.
template <typename T>
__global__ void __launch_bounds__(FIT_THREADS) gather_coords_kernel(const T *__restrict__ X, int64_t n,
                                                                    int d,
                                                                    const int32_t *__restrict__ perm,
                                                                    T *__restrict__ out,
                                                                    const int32_t *__restrict__ lab_in,
                                                                    int32_t *__restrict__ lab_out) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = perm[s];
        if (d == 2 && sizeof(T) == 4) {
            const float2 v = reinterpret_cast<const float2 *>(X)[src];
            out[s] = (T)v.x;
            out[n + s] = (T)v.y;
        } else {
            for (int j = 0; j < d; ++j) out[(int64_t)j * n + s] = X[src * d + j];
        }
        if (lab_out) lab_out[s] = lab_in[src];
    }
}

// ------------------------------------------------------------------
// Counting-scatter fit (DENSE, cells of <= FAST_MAX_CELL points).
// hist -> scan -> scatter of (coords, label, index) records through per-cell
// atomic cursors (arbitrary order inside a cell) -> in-cell fix-up that ranks
// each record by point index, restoring the stable input order of
// np.lexsort (grid.py:188-189), and writes the SoA outputs near-sequentially.
constexpr int FAST_MAX_CELL = 256;

// X is streamed (evict-first) so the L2 keeps the per-cell counters / cursors
// that the atomics hit.
template <typename T, bool STREAM = true>
__device__ __forceinline__ uint32_t point_key(const T *__restrict__ X, int64_t i, const DimParams &p) {
    uint64_t key = 0;
    for (int j = 0; j < p.d; ++j) {
        const T x = STREAM ? __ldcs(X + i * p.d + j) : X[i * p.d + j];
        const int64_t c = cell_id(to_double(x), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
        key = key * (uint64_t)p.ext[j] + (uint64_t)(c - p.lo[j]);
    }
    return (uint32_t)key;
}

// These histograms serve the sets the streaming fit leaves (a key range too
// heavy for a CTA: cfg3 puts 36M of its 50M points in one cell), so lanes of
// a warp often share a cell: one atomic per distinct key and warp
// (__match_any_sync), not 32 serialised ones on the same counter.
__device__ __forceinline__ void hist_add_agg(uint32_t *ctr, uint32_t key, uint32_t slot, uint32_t unit) {
    const unsigned peers = __match_any_sync(__activemask(), key);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(ctr + slot, unit * (uint32_t)__popc(peers));
}

template <typename T>
__global__ void __launch_bounds__(FIT_THREADS) hist_kernel(const T *__restrict__ X, int64_t n, DimParams p,
                                                           int32_t *__restrict__ counts) {
    constexpr int BU = 4;   // independent points per iteration (loads and atomics in flight)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (BU - 1) * stride < n; i += BU * stride) {
        uint32_t key[BU];
#pragma unroll
        for (int u = 0; u < BU; ++u) key[u] = point_key(X, i + u * stride, p);
#pragma unroll
        for (int u = 0; u < BU; ++u) hist_add_agg((uint32_t *)counts, key[u], key[u], 1u);
    }
    for (; i < n; i += stride) atomicAdd(&counts[point_key(X, i, p)], 1);
}

// The same histogram with two 16-bit counters per word: half the counter
// footprint (33 MB at cfg4), so the atomics stay in L2 instead of thrashing
// the 67 MB int32 table out to HBM.  A cell of >= 65536 points carries into
// its neighbour (or out of the word): the decoded counts then sum to less
// than n, which the caller checks (pt_off[E] after the scan) before redoing
// the int32 histogram.
template <typename T>
__global__ void __launch_bounds__(FIT_THREADS) hist16_kernel(const T *__restrict__ X, int64_t n, DimParams p,
                                                             uint32_t *__restrict__ packed) {
    constexpr int BU = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (BU - 1) * stride < n; i += BU * stride) {
        uint32_t key[BU];
#pragma unroll
        for (int u = 0; u < BU; ++u) key[u] = point_key(X, i + u * stride, p);
#pragma unroll
        for (int u = 0; u < BU; ++u) hist_add_agg(packed, key[u], key[u] >> 1, 1u << (16 * (key[u] & 1u)));
    }
    for (; i < n; i += stride) {
        const uint32_t key = point_key(X, i, p);
        atomicAdd(&packed[key >> 1], 1u << (16 * (key & 1u)));
    }
}

__global__ void unpack16_kernel(const uint32_t *__restrict__ packed, int64_t E, int32_t *__restrict__ counts) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= E;
         c += (int64_t)gridDim.x * blockDim.x)
        counts[c] = c < E ? (int32_t)((packed[c >> 1] >> (16 * (c & 1))) & 0xffffu) : 0;
}

__global__ void max_count_kernel(const int32_t *__restrict__ off, int64_t E, int32_t *out) {
    int m = 0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < E;
         c += (int64_t)gridDim.x * blockDim.x)
        m = max(m, off[c + 1] - off[c]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Record: d coordinates (T), label, point index -- RW words of 4 bytes.
template <typename T, int RW>
__global__ void __launch_bounds__(FIT_THREADS) scatter_records_kernel(
    const T *__restrict__ X, int64_t n, DimParams p, int32_t *__restrict__ cursor,
    const int32_t *__restrict__ labels, uint32_t *__restrict__ rec) {
    const int d = p.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t key = point_key(X, i, p);
        const int32_t slot = atomicAdd(&cursor[key], 1);
        uint32_t w[RW];
#pragma unroll
        for (int t = 0; t < RW; ++t) w[t] = 0u;
        const uint32_t *xs = reinterpret_cast<const uint32_t *>(X + i * d);
        const int cw = d * (int)(sizeof(T) / 4);
#pragma unroll
        for (int t = 0; t < RW - 2; ++t)
            if (t < cw) w[t] = __ldcs(xs + t);
        w[RW - 2] = labels ? (uint32_t)__ldcs(labels + i) : 0u;
        w[RW - 1] = (uint32_t)i;
        uint4 *dst = reinterpret_cast<uint4 *>(rec + (int64_t)slot * RW);
#pragma unroll
        for (int t = 0; t < RW / 4; ++t)
            __stcs(dst + t, make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]));
    }
}

// Locality pass before the cell scatter: a partition of the points by the
// high bits of their cell key (<= 1024 key-range buckets, 4 rows of cells at
// cfg4; measured against 256 and 4096: fewer buckets widen the scatter's
// write window beyond L2, more shorten the partition's write runs).  Each CTA
// takes a contiguous chunk of points (8K: 512 threads x 16; the counting
// phase loads X through L2 so the writing phase re-reads it from there --
// cfg4 fit 7.75 -> 7.3 ms against 64K-point chunks with streamed loads; 16-byte
// cell records instead of 32 measured 7.7 ms, tools/fit_sweep.sh),
// counts its buckets in shared memory, reserves one range per bucket with a
// single global atomic, and writes compact records (coords, label, index)
// into those ranges.  The cell scatter that follows then walks the points
// bucket by bucket: its cursor atomics and its record writes stay inside one
// bucket's window (L2-resident) instead of hitting all of HBM at random.
constexpr int PART_BUCKETS = 1024;
#ifndef PART_THR
#define PART_THR 512
#endif
constexpr int PART_THREADS = PART_THR;
#ifndef PART_CHUNK_K
#define PART_CHUNK_K 16
#endif
#ifndef PART_P1_STREAM
#define PART_P1_STREAM 0
#endif
constexpr int PART_CHUNK = PART_CHUNK_K * PART_THREADS;

template <typename T, int RWP>
__global__ void __launch_bounds__(PART_THREADS) partition_kernel(const T *__restrict__ X, int64_t n, DimParams p,
                                                                 int shift, const int32_t *__restrict__ labels,
                                                                 int32_t *__restrict__ bcur,
                                                                 uint32_t *__restrict__ part) {
    __shared__ int cnt[PART_BUCKETS];
    __shared__ int base[PART_BUCKETS];
    const int64_t i0 = (int64_t)blockIdx.x * PART_CHUNK;
    const int64_t i1 = i0 + PART_CHUNK < n ? i0 + PART_CHUNK : n;
    for (int b = threadIdx.x; b < PART_BUCKETS; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) atomicAdd(&cnt[point_key<T, PART_P1_STREAM>(X, i, p) >> shift], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < PART_BUCKETS; b += blockDim.x) {
        const int c = cnt[b];
        base[b] = c ? atomicAdd(&bcur[b], c) : 0;
        cnt[b] = 0;
    }
    __syncthreads();
    const int d = p.d;
    const int cw = d * (int)(sizeof(T) / 4);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const uint32_t b = point_key(X, i, p) >> shift;
        const int64_t pos = (int64_t)base[b] + atomicAdd(&cnt[b], 1);
        uint32_t w[RWP];
#pragma unroll
        for (int t = 0; t < RWP; ++t) w[t] = 0u;
        const uint32_t *xs = reinterpret_cast<const uint32_t *>(X + i * d);
#pragma unroll
        for (int t = 0; t < RWP - 2; ++t)
            if (t < cw) w[t] = __ldcs(xs + t);
        w[RWP - 2] = labels ? (uint32_t)__ldcs(labels + i) : 0u;
        w[RWP - 1] = (uint32_t)i;
        uint4 *dst = reinterpret_cast<uint4 *>(part + pos * RWP);
#pragma unroll
        for (int t = 0; t < RWP / 4; ++t) dst[t] = make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]);
    }
}

__global__ void bucket_start_kernel(const int32_t *__restrict__ pt_off, int shift, int nbuck,
                                    int32_t *__restrict__ bcur) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbuck; b += gridDim.x * blockDim.x)
        bcur[b] = pt_off[(int64_t)b << shift];
}

// The cell scatter over the partitioned records (bucket order).
template <typename T, int RWP, int RW>
__global__ void __launch_bounds__(FIT_THREADS) scatter_part_kernel(const uint32_t *__restrict__ part, int64_t n,
                                                                   DimParams p, int32_t *__restrict__ cursor,
                                                                   uint32_t *__restrict__ rec) {
    const int d = p.d;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[RW];
#pragma unroll
        for (int t = 0; t < RW; ++t) w[t] = 0u;
        const uint4 *src = reinterpret_cast<const uint4 *>(part + s * RWP);
#pragma unroll
        for (int t = 0; t < RWP / 4; ++t) {
            const uint4 v = __ldcs(src + t);
            w[4 * t] = v.x;
            w[4 * t + 1] = v.y;
            w[4 * t + 2] = v.z;
            w[4 * t + 3] = v.w;
        }
        const uint32_t lab = w[RWP - 2], idx = w[RWP - 1];
        w[RWP - 2] = 0u;
        w[RWP - 1] = 0u;
        w[RW - 2] = lab;
        w[RW - 1] = idx;
        const T *xc = reinterpret_cast<const T *>(w);
        uint64_t key = 0;
        for (int j = 0; j < d; ++j) {
            const int64_t c = cell_id(to_double(xc[j]), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
            key = key * (uint64_t)p.ext[j] + (uint64_t)(c - p.lo[j]);
        }
        const int32_t slot = atomicAdd(&cursor[key], 1);
        uint4 *dst = reinterpret_cast<uint4 *>(rec + (int64_t)slot * RW);
#pragma unroll
        for (int t = 0; t < RW / 4; ++t) dst[t] = make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]);
    }
}

template <typename T, int RW>
__global__ void __launch_bounds__(FIT_THREADS) fixup_records_kernel(
    const uint32_t *__restrict__ rec, int64_t n, DimParams p, const int32_t *__restrict__ pt_off,
    T *__restrict__ coords, int32_t *__restrict__ perm, int32_t *__restrict__ labels_out) {
    const int d = p.d;
    const int cw = d * (int)(sizeof(T) / 4);
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rec + s * RW);
        uint32_t w[RW];
#pragma unroll
        for (int t = 0; t < RW / 4; ++t) {
            const uint4 v = src[t];
            w[4 * t] = v.x;
            w[4 * t + 1] = v.y;
            w[4 * t + 2] = v.z;
            w[4 * t + 3] = v.w;
        }
        const T *xc = reinterpret_cast<const T *>(w);
        uint64_t key = 0;
        for (int j = 0; j < d; ++j) {
            const int64_t c = cell_id(to_double(xc[j]), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
            key = key * (uint64_t)p.ext[j] + (uint64_t)(c - p.lo[j]);
        }
        const int32_t c0 = pt_off[key], c1 = pt_off[key + 1];
        const uint32_t me = w[RW - 1];
        int rank = 0;
        for (int32_t t = c0; t < c1; ++t) rank += rec[(int64_t)t * RW + RW - 1] < me;
        const int64_t o = (int64_t)c0 + rank;
        for (int j = 0; j < d; ++j) coords[(int64_t)j * n + o] = xc[j];
        perm[o] = (int32_t)me;
        if (labels_out) labels_out[o] = (int32_t)w[RW - 2];
        (void)cw;
    }
}

// ------------------------------------------------------------------
// Streaming fit (DENSE; the default when every key-range bucket fits a CTA).
// Final buckets are runs of 2^shift consecutive cell keys (<= 32768 of
// them, a few thousand points each).
//   count  : points per final bucket (shared-memory histogram)   [read X]
//   part1  : records (coords, label, index) by the bucket's top bits (<= 128
//            level-1 buckets); each CTA counting-sorts an 8K-point chunk in
//            shared memory and writes one contiguous run per level-1 bucket
//                                                   [read X + labels, write records]
//   part2  : the same over the level-1 output by the low 8 bits (a chunk
//            spans <= 2 level-1 buckets, so <= 512 digits)  [read + write records]
//   local  : one CTA per final bucket, entirely in shared memory: the
//            bucket's records, cell histogram -> scan -> pt_off, slots
//            grouped by cell, each cell's slots ordered by point index (the
//            stable in-cell order of np.lexsort, grid.py:188-189), coalesced
//            SoA coordinates / perm / labels            [read records, write outputs]
// Every global write is a burst of consecutive records, so no HBM sector
// is written partially (the scattered 16-byte writes of a one-level
// partition into 8K buckets cost ~2x their bytes in read-modify-write).
constexpr int SF_MAX_BUCKETS = 32768;
constexpr int SF_L2_BITS = 8;
constexpr int SF_MAX_L1 = SF_MAX_BUCKETS >> SF_L2_BITS;   // 128
constexpr int SF_MAX_CELLS = 8192;       // cells per final bucket (shared histogram)
constexpr int SF_COUNT_THREADS = 1024;
constexpr int SF_PART_THREADS = 256;
#ifndef SF_LOCAL_THR
#define SF_LOCAL_THR 512
#endif
constexpr int SF_LOCAL_THREADS = SF_LOCAL_THR;
constexpr int SF_MAX_POINTS = 65535;     // per final bucket (16-bit record positions)

// Cell id of a coordinate of the training set (inside [lo, hi] by construction).
template <typename T>
__device__ __forceinline__ int64_t fit_cell_id(T x, const DimParams &p, int j) {
    if (sizeof(T) == 4 && ((p.fast32 >> j) & 1u)) return (int64_t)__float2int_rd((float)x * p.inv32[j]);
    return cell_id(to_double(x), p.w[j], p.inv[j], (p.pow2 >> j) & 1u);
}

template <typename T, int D>
__device__ __forceinline__ uint32_t sf_key_d(const T (&x)[D > 0 ? D : 1], const DimParams &p) {
    uint64_t key = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const int64_t c = fit_cell_id<T>(x[j], p, j);
        key = key * (uint64_t)p.ext[j] + (uint64_t)(c - p.lo[j]);
    }
    return (uint32_t)key;
}

// Final-bucket histogram.  D > 0: compile-time dims, 4 points in flight per
// thread; D == 0: point_key.
template <typename T, int D>
__global__ void __launch_bounds__(SF_COUNT_THREADS) sf_count_kernel(const T *__restrict__ X, int64_t n, DimParams p,
                                                                   int shift, int nb, int32_t *__restrict__ bcount) {
    extern __shared__ int sf_hist[];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) sf_hist[b] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (D > 0) {
        constexpr int DD = D > 0 ? D : 1;
        constexpr int BU = 8;
        for (; i + (BU - 1) * stride < n; i += BU * stride) {
            T v[BU][DD];
#pragma unroll
            for (int u = 0; u < BU; ++u)
#pragma unroll
                for (int j = 0; j < DD; ++j) v[u][j] = __ldcs(X + (i + u * stride) * DD + j);
#pragma unroll
            for (int u = 0; u < BU; ++u) atomicAdd(&sf_hist[sf_key_d<T, DD>(v[u], p) >> shift], 1);
        }
    }
    for (; i < n; i += stride) atomicAdd(&sf_hist[point_key<T, true>(X, i, p) >> shift], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        if (sf_hist[b]) atomicAdd(&bcount[b], sf_hist[b]);
}

template <int RWP>
__device__ __forceinline__ void sf_load_record(const uint32_t *__restrict__ src, int64_t r, uint32_t (&w)[RWP]) {
    const uint4 *q = reinterpret_cast<const uint4 *>(src + r * RWP);
#pragma unroll
    for (int t = 0; t < RWP / 4; ++t) {
        const uint4 v = q[t];
        w[4 * t] = v.x;
        w[4 * t + 1] = v.y;
        w[4 * t + 2] = v.z;
        w[4 * t + 3] = v.w;
    }
}

template <int RWP>
__device__ __forceinline__ void sf_store_record(uint32_t *__restrict__ dst, int64_t r, const uint32_t (&w)[RWP]) {
    uint4 *q = reinterpret_cast<uint4 *>(dst + r * RWP);
#pragma unroll
    for (int t = 0; t < RWP / 4; ++t) q[t] = make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]);
}

// Cell key of a record; the loop is unrolled to the most coordinates a
// record of RWP words holds, so the record stays in registers.
template <typename T, int RWP>
__device__ __forceinline__ uint32_t sf_record_key(const uint32_t (&w)[RWP], const DimParams &p) {
    constexpr int MAXD = (RWP - 2) * 4 / (int)sizeof(T);
    uint64_t key = 0;
#pragma unroll
    for (int j = 0; j < MAXD; ++j) {
        if (j < p.d) {
            int64_t c;
            if (sizeof(T) == 4) c = fit_cell_id<float>(__uint_as_float(w[j]), p, j);
            else c = fit_cell_id<double>(__hiloint2double((int)w[2 * j + 1], (int)w[2 * j]), p, j);
            key = key * (uint64_t)p.ext[j] + (uint64_t)(c - p.lo[j]);
        }
    }
    return (uint32_t)key;
}

// Block-wide exclusive scan of a[0..len) in shared memory; returns the total.
__device__ __forceinline__ int sf_block_scan(int *a, int len, int *warp_tot) {
    const int per = (len + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per;
    int sum = 0;
    for (int t = 0; t < per; ++t)
        if (b0 + t < len) sum += a[b0 + t];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int incl = warp_inclusive_scan(sum);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = (int)(blockDim.x >> 5);
        const int v = lane < nw ? warp_tot[lane] : 0;
        const int vi = warp_inclusive_scan(v);
        if (lane < nw) warp_tot[lane] = vi - v;
        if (lane == 31) warp_tot[32] = vi;
    }
    __syncthreads();
    int run = incl - sum + warp_tot[wid];
    for (int t = 0; t < per; ++t)
        if (b0 + t < len) {
            const int v = a[b0 + t];
            a[b0 + t] = run;
            run += v;
        }
    const int total = warp_tot[32];
    __syncthreads();
    return total;
}

// Level-2 chunks never straddle a level-1 bucket: chunk prefix per level-1
// bucket (cpre[b1] = chunks before bucket b1), one warp.
__global__ void sf_chunk_prefix_kernel(const int32_t *__restrict__ bbase, int nb, int nb1, int ch,
                                       int32_t *__restrict__ cpre) {
    int run = 0;
    for (int b0 = 0; b0 < nb1; b0 += 32) {
        const int b1 = b0 + (int)threadIdx.x;
        int c = 0;
        if (b1 < nb1) {
            const int32_t st = bbase[b1 << SF_L2_BITS];
            const int32_t en = bbase[min((b1 + 1) << SF_L2_BITS, nb)];
            c = (en - st + ch - 1) / ch;
        }
        const int incl = warp_inclusive_scan(c);
        if (b1 < nb1) cpre[b1] = run + incl - c;
        run += __shfl_sync(GHN_FULL, incl, 31);
    }
    if (threadIdx.x == 0) cpre[nb1] = run;
}

// One level of the partition over a chunk of CH items, staged through shared
// memory: the chunk's input arrives by 1-D TMA (cp.async.bulk) into the
// staging area, each thread takes ITEMS items into registers with their
// digit and rank (shared atomics), then the items are counting-sorted into
// the staging area and every digit's run leaves in one burst of consecutive
// 16-byte stores at [reserved base, ...).
//   LEVEL 1: items = points of X (+ labels), digit = final bucket >> 8,
//            chunk = blockIdx.x;
//   LEVEL 2: items = level-1 records of one level-1 bucket b1 (chunks from
//            cpre), digit = final bucket & 255.
template <typename T, int RWP, int LEVEL, int ITEMS>
__global__ void __launch_bounds__(SF_PART_THREADS, 4) sf_part_kernel(const T *__restrict__ X, const int32_t *__restrict__ labels,
                                                                 const uint32_t *__restrict__ in, int64_t n, DimParams p,
                                                                 int shift, const int32_t *__restrict__ bbase,
                                                                 const int32_t *__restrict__ cpre, int nb, int nb1,
                                                                 int32_t *__restrict__ cursor,
                                                                 uint32_t *__restrict__ out) {
    constexpr int CH = ITEMS * SF_PART_THREADS;
    constexpr int ND = LEVEL == 1 ? SF_MAX_L1 : (1 << SF_L2_BITS);
    extern __shared__ uint4 sf_stage4[];
    uint32_t *stage = reinterpret_cast<uint32_t *>(sf_stage4);       // CH records
    uint16_t *sdig = reinterpret_cast<uint16_t *>(stage + CH * RWP);  // CH digits
    __shared__ int cnt[ND], off[ND], gbase[ND];
    __shared__ int warp_tot[33];
    __shared__ int64_t s_i0, s_i1;
    __shared__ int s_b1;
    __shared__ alignas(8) uint64_t bar;
    const int d = p.d;
    if (threadIdx.x == 0) {
        int64_t i0, i1;
        int b1 = 0;
        if (LEVEL == 1) {
            i0 = (int64_t)blockIdx.x * CH;
            i1 = i0 + CH < n ? i0 + CH : n;
        } else {
            // the level-1 bucket holding this chunk: last b1 with cpre[b1] <= blockIdx.x
            int lo = 0, hi = nb1;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (cpre[mid] <= (int)blockIdx.x) lo = mid;
                else hi = mid;
            }
            b1 = lo;
            const int64_t st = bbase[b1 << SF_L2_BITS], en = bbase[min((b1 + 1) << SF_L2_BITS, nb)];
            i0 = st + (int64_t)((int)blockIdx.x - cpre[b1]) * CH;
            i1 = i0 + CH < en ? i0 + CH : en;
            if ((int)blockIdx.x >= cpre[nb1]) i0 = i1 = 0;
        }
        s_i0 = i0;
        s_i1 = i1;
        s_b1 = b1;
        mbar_init(&bar, 1);
    }
    for (int b = threadIdx.x; b < ND; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    const int64_t i0 = s_i0, i1 = s_i1;
    const int m = (int)(i1 - i0);
    if (m <= 0) return;
    // ---- chunk input into the staging area (TMA when 16-byte sized)
    const uint32_t xbytes = LEVEL == 1 ? (uint32_t)m * d * sizeof(T) : (uint32_t)m * RWP * 4;
    const uint32_t lbytes = (LEVEL == 1 && labels) ? (uint32_t)m * 4 : 0u;
    uint32_t *lab_s = stage + ((xbytes + 15) / 16) * 4;      // labels after the coordinates
    const void *xsrc = LEVEL == 1 ? (const void *)(X + i0 * d) : (const void *)(in + i0 * RWP);
    const bool bulk = xbytes % 16 == 0 && lbytes % 16 == 0;
    if (bulk) {
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&bar, xbytes + lbytes);
            bulk_g2s_all(stage, xsrc, xbytes, &bar);
            if (lbytes) bulk_g2s_all(lab_s, labels + i0, lbytes, &bar);
        }
        mbar_wait_parity(&bar, 0);
    } else {
        for (uint32_t q = threadIdx.x; q < xbytes / 4; q += blockDim.x) stage[q] = ((const uint32_t *)xsrc)[q];
        for (uint32_t q = threadIdx.x; q < lbytes / 4; q += blockDim.x) lab_s[q] = (uint32_t)labels[i0 + q];
        __syncthreads();
    }
    const int cw = d * (int)(sizeof(T) / 4);
    const int fb = LEVEL == 2 ? s_b1 << SF_L2_BITS : 0;
    uint32_t w[ITEMS][RWP];
    int dig[ITEMS], rank[ITEMS];
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
        const int t = threadIdx.x + u * SF_PART_THREADS;
        dig[u] = -1;
        if (t < m) {
            if (LEVEL == 1) {
#pragma unroll
                for (int q = 0; q < RWP; ++q) w[u][q] = 0u;
                if (cw == 2) {
                    const uint2 v = reinterpret_cast<const uint2 *>(stage)[t];
                    w[u][0] = v.x;
                    w[u][1] = v.y;
                } else {
#pragma unroll
                    for (int q = 0; q < RWP - 2; ++q)
                        if (q < cw) w[u][q] = stage[t * cw + q];
                }
                w[u][RWP - 2] = lbytes ? lab_s[t] : 0u;
                w[u][RWP - 1] = (uint32_t)(i0 + t);
                dig[u] = (int)((sf_record_key<T, RWP>(w[u], p) >> shift) >> SF_L2_BITS);
            } else {
#pragma unroll
                for (int q = 0; q < RWP; q += 4) {
                    const uint4 v = sf_stage4[(t * RWP + q) / 4];
                    w[u][q] = v.x;
                    w[u][q + 1] = v.y;
                    w[u][q + 2] = v.z;
                    w[u][q + 3] = v.w;
                }
                dig[u] = (int)(sf_record_key<T, RWP>(w[u], p) >> shift) - fb;
            }
            rank[u] = atomicAdd(&cnt[dig[u]], 1);
        }
    }
    __syncthreads();   // the staging area's input is consumed
    for (int b = threadIdx.x; b < ND; b += blockDim.x) off[b] = cnt[b];
    __syncthreads();
    sf_block_scan(off, ND, warp_tot);
    for (int b = threadIdx.x; b < ND; b += blockDim.x) {
        const int c = cnt[b];
        gbase[b] = c ? atomicAdd(&cursor[fb + b], c) : 0;
    }
#pragma unroll
    for (int u = 0; u < ITEMS; ++u)
        if (dig[u] >= 0) {
            const int sl = off[dig[u]] + rank[u];
#pragma unroll
            for (int q = 0; q < RWP; q += 4)
                sf_stage4[(sl * RWP + q) / 4] = make_uint4(w[u][q], w[u][q + 1], w[u][q + 2], w[u][q + 3]);
            sdig[sl] = (uint16_t)dig[u];
        }
    __syncthreads();
    // RWP / 4 uint4 per record: consecutive threads store consecutive 16-byte words of a run
    for (int q = threadIdx.x; q < m * (RWP / 4); q += blockDim.x) {
        const int sl = q / (RWP / 4), part = q % (RWP / 4);
        const int b = sdig[sl];
        const int64_t g = (int64_t)gbase[b] + (sl - off[b]);
        reinterpret_cast<uint4 *>(out + g * RWP)[part] = sf_stage4[q];
    }
}

template <typename T, int RWP>
__global__ void __launch_bounds__(SF_LOCAL_THREADS) sf_local_kernel(const uint32_t *__restrict__ part,
                                                                   const int32_t *__restrict__ bbase, int shift,
                                                                   int64_t E, int64_t n, DimParams p,
                                                                   T *__restrict__ coords, int32_t *__restrict__ perm,
                                                                   int32_t *__restrict__ labels_out,
                                                                   int32_t *__restrict__ pt_off) {
    extern __shared__ uint4 sf_lm4[];
    __shared__ int warp_tot[33];
    const int b = blockIdx.x;
    const int32_t r0 = bbase[b], m = bbase[b + 1] - r0;
    const int64_t c0 = (int64_t)b << shift;
    const int ncell = (int)min((int64_t)1 << shift, E - c0);
    uint32_t *rec = reinterpret_cast<uint32_t *>(sf_lm4);        // m records
    int *hist = reinterpret_cast<int *>(rec + (size_t)m * RWP);     // ncell
    int32_t *sidx = hist + ncell;                                   // m point indices, grouped by cell
    uint16_t *spos = reinterpret_cast<uint16_t *>(sidx + m);        // m record positions, grouped by cell
    __shared__ alignas(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        if (m > 0) {   // the bucket's records by 1-D TMA
            mbar_arrive_expect_tx(&bar, (uint32_t)m * RWP * 4);
            bulk_g2s_all(rec, part + (int64_t)r0 * RWP, (uint32_t)m * RWP * 4, &bar);
        }
    }
    for (int c = threadIdx.x; c < ncell; c += blockDim.x) hist[c] = 0;
    __syncthreads();
    if (m > 0) mbar_wait_parity(&bar, 0);
    auto load = [&](int t, uint32_t (&w)[RWP]) {
#pragma unroll
        for (int u = 0; u < RWP; u += 4) {
            const uint4 v = sf_lm4[(t * RWP + u) / 4];
            w[u] = v.x, w[u + 1] = v.y, w[u + 2] = v.z, w[u + 3] = v.w;
        }
    };
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
        uint32_t w[RWP];
        load(t, w);
        atomicAdd(&hist[sf_record_key<T, RWP>(w, p) - (uint32_t)c0], 1);
    }
    __syncthreads();
    sf_block_scan(hist, ncell, warp_tot);
    for (int c = threadIdx.x; c < ncell; c += blockDim.x) pt_off[c0 + c] = r0 + hist[c];
    __syncthreads();
    // records grouped by cell (arbitrary order inside a cell); hist[c] ends as the end of cell c
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
        uint32_t w[RWP];
        load(t, w);
        const int slot = atomicAdd(&hist[sf_record_key<T, RWP>(w, p) - (uint32_t)c0], 1);
        sidx[slot] = (int32_t)w[RWP - 1];
        spos[slot] = (uint16_t)t;
    }
    __syncthreads();
#ifndef SF_SORT
#define SF_SORT 1
#endif
#if SF_SORT
    // each cell's slots by point index (insertion sort; cells hold a few points)
    for (int c = threadIdx.x; c < ncell; c += blockDim.x) {
        const int s0 = c ? hist[c - 1] : 0, s1 = hist[c];
        for (int s = s0 + 1; s < s1; ++s) {
            const int32_t ki = sidx[s];
            const uint16_t kp = spos[s];
            int u = s - 1;
            while (u >= s0 && sidx[u] > ki) {
                sidx[u + 1] = sidx[u];
                spos[u + 1] = spos[u];
                --u;
            }
            sidx[u + 1] = ki;
            spos[u + 1] = kp;
        }
    }
    __syncthreads();
    const int d = p.d;
    for (int s = threadIdx.x; s < m; s += blockDim.x) {
        const uint32_t *w = rec + (size_t)spos[s] * RWP;
        const T *xc = reinterpret_cast<const T *>(w);
        const int64_t o = (int64_t)r0 + s;
        for (int j = 0; j < d; ++j) __stcs(coords + (int64_t)j * n + o, xc[j]);
        __stcs(perm + o, sidx[s]);
        if (labels_out) __stcs(labels_out + o, (int32_t)w[RWP - 2]);
    }
#else
    // slot s goes to its cell's start + its rank by point index inside the
    // cell (the stable in-cell order of np.lexsort, grid.py:188-189)
    const int d = p.d;
    for (int s = threadIdx.x; s < m; s += blockDim.x) {
        uint32_t w[RWP];
        load(spos[s], w);
        const int c = (int)(sf_record_key<T, RWP>(w, p) - (uint32_t)c0);
        const int s0 = c ? hist[c - 1] : 0, s1 = hist[c];
        const int32_t me = sidx[s];
        int rank = 0;
        for (int u = s0; u < s1; ++u) rank += sidx[u] < me;
        const T *xc = reinterpret_cast<const T *>(w);
        const int64_t o = (int64_t)r0 + s0 + rank;
        for (int j = 0; j < d; ++j) __stcs(coords + (int64_t)j * n + o, xc[j]);
        __stcs(perm + o, me);
        if (labels_out) __stcs(labels_out + o, (int32_t)w[RWP - 2]);
    }
#endif
}

__global__ void sf_tail_kernel(int32_t *pt_off, int64_t E, int64_t n) { pt_off[E] = (int32_t)n; }

// Cell table from the offsets: non-empty flags -> (scan) -> cell_start / ids.
__global__ void ne_flag_kernel(const int32_t *__restrict__ pt_off, int64_t E, int32_t *__restrict__ ne) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= E;
         c += (int64_t)gridDim.x * blockDim.x)
        ne[c] = (c < E && pt_off[c + 1] > pt_off[c]) ? 1 : 0;
}

__global__ void cells_from_offsets_kernel(const int32_t *__restrict__ pt_off,
                                          const int32_t *__restrict__ ne_off, int64_t E, int64_t n,
                                          DimParams p, int32_t *__restrict__ cell_start,
                                          int32_t *__restrict__ cell_ids, int32_t *__restrict__ n_cells) {
    const int d = p.d;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < E;
         c += (int64_t)gridDim.x * blockDim.x) {
        if (pt_off[c + 1] > pt_off[c]) {
            const int32_t idx = ne_off[c];
            cell_start[idx] = pt_off[c];
            if (E <= 0xffffffffLL) {   // 32-bit divisions (the 64-bit ones are a software loop)
                uint32_t rem = (uint32_t)c;
                for (int j = d - 1; j >= 0; --j) {
                    const uint32_t e = (uint32_t)p.ext[j];
                    const uint32_t q = rem / e;
                    cell_ids[(int64_t)idx * d + j] = (int32_t)(rem - q * e);
                    rem = q;
                }
            } else {
                uint64_t rem = (uint64_t)c;
                for (int j = d - 1; j >= 0; --j) {
                    cell_ids[(int64_t)idx * d + j] = (int32_t)(rem % (uint64_t)p.ext[j]);
                    rem /= (uint64_t)p.ext[j];
                }
            }
        }
        if (c == 0) {
            *n_cells = ne_off[E];
            cell_start[ne_off[E]] = (int32_t)n;
        }
    }
}

// Records are one full 32-byte DRAM sector: a random scatter of half-sector
// records costs a read-modify-write per sector (measured: 13 GB of traffic
// for 100M 16-byte records vs 3.2 GB written here).
static int record_words(int d, int dtype) {
    const int cw = d * (dtype == GHN_F32 ? 1 : 2);
    if (cw + 2 <= 8) return 8;   // full 32-byte sectors: partial-sector scatter writes cost a DRAM read each
    return 0;   // no fast path
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Partition records: 16 bytes when (coords, label, index) fit, else 32.
static int part_words(int d, int dtype) {
    const int cw = d * (dtype == GHN_F32 ? 1 : 2);
    return cw + 2 <= 4 ? 4 : 8;
}

// Counting-scatter workspace tail: partition records, then bucket cursors.
static size_t fast_part_off(const ghn_fit_plan *plan) {
    const int RW = record_words(plan->d, plan->dtype);
    return plan->fast_rec_off + align256((size_t)plan->n * RW * 4);
}
static size_t fast_bcur_off(const ghn_fit_plan *plan) {
    return fast_part_off(plan) + align256((size_t)plan->n * part_words(plan->d, plan->dtype) * 4);
}

static unsigned grid_for(int64_t n, int threads = FIT_THREADS) {
    int64_t b = (n + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count() * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (unsigned)b;
}

static int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}


template <typename T>
int32_t bounds_launch(const T *X, int64_t n, int d, const DimParams &p, int64_t *bounds,
                      unsigned long long *okey, int32_t *flags, cudaStream_t s) {
    unsigned g = grid_for(n);
    switch (d) {
#define GHN_BCASE(DD) \
    case DD: bounds_kernel<T, DD><<<g, FIT_THREADS, 0, s>>>(X, n, p, bounds, okey, flags); break;
        GHN_BCASE(1) GHN_BCASE(2) GHN_BCASE(3) GHN_BCASE(4)
        GHN_BCASE(5) GHN_BCASE(6) GHN_BCASE(7) GHN_BCASE(8)
#undef GHN_BCASE
        default: bounds_kernel_rt<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, bounds, okey, flags);
    }
    GHN_LAUNCH_CHECK("bounds_kernel");
    return GHN_OK;
}

// Streaming fit host side (see sf_*): returns GHN_ERR_UNSUPPORTED without
// touching the outputs when a final bucket spans too many cells or holds
// more points than a CTA's shared memory takes.
template <typename T, int RWP>
int32_t fit_stream_rw(const ghn_fit_plan *plan, const T *X, const ghn_fit_out *out, char *ws, char *sws,
                      const DimParams &p, cudaStream_t s) {
    const int64_t n = plan->n, E = plan->E;
    const int d = plan->d;
    const int kb = plan->key_bits > 0 ? plan->key_bits : 1;
    const int shift = kb > 15 ? kb - 15 : 0;
    if (((int64_t)1 << shift) > SF_MAX_CELLS) return GHN_ERR_UNSUPPORTED;
    const int nb = (int)(((E - 1) >> shift) + 1);
    const int nb1 = ((nb - 1) >> SF_L2_BITS) + 1;
    int32_t *bcount = (int32_t *)(ws + fast_bcur_off(plan));          // nb + 1: final bucket bases
    int32_t *cur2 = bcount + align256((size_t)(nb + 1) * 4) / 4;      // nb: final bucket cursors
    int32_t *cur1 = cur2 + align256((size_t)nb * 4) / 4;              // nb1: level-1 cursors
    int32_t *dmax = cur1 + align256((size_t)SF_MAX_L1 * 4) / 4;
    int32_t *cpre = dmax + 64;                                         // nb1 + 1
    uint32_t *part1 = (uint32_t *)(ws + plan->fast_rec_off);
    uint32_t *part2 = (uint32_t *)(ws + fast_part_off(plan));
    GHN_CUDA_CHECK(cudaMemsetAsync(bcount, 0, (size_t)(nb + 1) * 4, s));
    GHN_CUDA_CHECK(cudaMemsetAsync(dmax, 0, 4, s));
    const size_t csmem = (size_t)nb * 4;
    const void *cfn = d == 2 ? (const void *)sf_count_kernel<T, 2> : (const void *)sf_count_kernel<T, 0>;
    GHN_CUDA_CHECK(cudaFuncSetAttribute(cfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    const unsigned cg = (unsigned)sm_count() * (csmem > 64 * 1024 ? 1 : 2);
    if (d == 2)
        sf_count_kernel<T, 2><<<cg, SF_COUNT_THREADS, csmem, s>>>(X, n, p, shift, nb, bcount);
    else
        sf_count_kernel<T, 0><<<cg, SF_COUNT_THREADS, csmem, s>>>(X, n, p, shift, nb, bcount);
    GHN_LAUNCH_CHECK("sf_count_kernel");
    int32_t rc = exclusive_scan_i32(bcount, bcount, nb + 1, sws, s);
    if (rc) return rc;
    max_count_kernel<<<grid_for(nb), FIT_THREADS, 0, s>>>(bcount, nb, dmax);
    GHN_LAUNCH_CHECK("max_count_kernel");
    int32_t hmax = 0;
    GHN_CUDA_CHECK(cudaMemcpyAsync(&hmax, dmax, 4, cudaMemcpyDeviceToHost, s));
    GHN_CUDA_CHECK(cudaStreamSynchronize(s));
    const int ncell = (int)((int64_t)1 << shift);
    const size_t lsmem = (size_t)hmax * (RWP * 4 + 6) + (size_t)ncell * 4 + 64;
    if (hmax > SF_MAX_POINTS || lsmem > 200 * 1024) return GHN_ERR_UNSUPPORTED;
    // cursors: final buckets from their bases, level-1 buckets from their first final bucket's base
    GHN_CUDA_CHECK(cudaMemcpyAsync(cur2, bcount, (size_t)nb * 4, cudaMemcpyDeviceToDevice, s));
    GHN_CUDA_CHECK(cudaMemcpy2DAsync(cur1, 4, bcount, (size_t)4 << SF_L2_BITS, 4, nb1, cudaMemcpyDeviceToDevice, s));
    constexpr int IT = RWP == 4 ? 8 : 4;
    constexpr int CH = IT * SF_PART_THREADS;
    sf_chunk_prefix_kernel<<<1, 32, 0, s>>>(bcount, nb, nb1, CH, cpre);
    GHN_LAUNCH_CHECK("sf_chunk_prefix_kernel");
    const size_t psmem = (size_t)CH * (RWP * 4 + 2);
    const unsigned gp = (unsigned)((n + CH - 1) / CH);
    const void *p1 = (const void *)sf_part_kernel<T, RWP, 1, IT>;
    const void *p2 = (const void *)sf_part_kernel<T, RWP, 2, IT>;
    const void *lf = (const void *)sf_local_kernel<T, RWP>;
    GHN_CUDA_CHECK(cudaFuncSetAttribute(p1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    GHN_CUDA_CHECK(cudaFuncSetAttribute(p2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    GHN_CUDA_CHECK(cudaFuncSetAttribute(lf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsmem));
    sf_part_kernel<T, RWP, 1, IT><<<gp, SF_PART_THREADS, psmem, s>>>(X, out->labels_in, nullptr, n, p, shift, bcount,
                                                                     cpre, nb, nb1, cur1, part1);
    GHN_LAUNCH_CHECK("sf_part_kernel<1>");
    sf_part_kernel<T, RWP, 2, IT><<<gp + nb1, SF_PART_THREADS, psmem, s>>>(X, nullptr, part1, n, p, shift, bcount,
                                                                           cpre, nb, nb1, cur2, part2);
    GHN_LAUNCH_CHECK("sf_part_kernel<2>");
    sf_local_kernel<T, RWP><<<nb, SF_LOCAL_THREADS, lsmem, s>>>(part2, bcount, shift, E, n, p, (T *)out->coords,
                                                                out->perm, out->labels_perm, out->pt_off);
    GHN_LAUNCH_CHECK("sf_local_kernel");
    sf_tail_kernel<<<1, 1, 0, s>>>(out->pt_off, E, n);
    GHN_LAUNCH_CHECK("sf_tail_kernel");
    ne_flag_kernel<<<grid_for(E + 1), FIT_THREADS, 0, s>>>(out->pt_off, E, out->ne_off);
    GHN_LAUNCH_CHECK("ne_flag_kernel");
    rc = exclusive_scan_i32(out->ne_off, out->ne_off, E + 1, sws, s);
    if (rc) return rc;
    cells_from_offsets_kernel<<<grid_for(E), FIT_THREADS, 0, s>>>(out->pt_off, out->ne_off, E, n, p, out->cell_start,
                                                                  out->cell_ids, out->n_cells);
    GHN_LAUNCH_CHECK("cells_from_offsets_kernel");
    return GHN_OK;
}

template <typename T>
int32_t fit_stream(const ghn_fit_plan *plan, const T *X, const ghn_fit_out *out, char *ws, char *sws,
                   const DimParams &p, cudaStream_t s) {
    if (part_words(plan->d, plan->dtype) == 4) return fit_stream_rw<T, 4>(plan, X, out, ws, sws, p, s);
    return fit_stream_rw<T, 8>(plan, X, out, ws, sws, p, s);
}

template <typename T>
int32_t fit_build_impl(const ghn_fit_plan *plan, const T *X, const ghn_fit_out *out, char *ws,
                       size_t ws_bytes, cudaStream_t s) {
    const int64_t n = plan->n;
    const int d = plan->d;
    DimParams p = make_dims(d, plan->widths, plan->lo, plan->ext);
    const size_t n4 = align256((size_t)n * 4);
    uint32_t *kA = (uint32_t *)ws;
    uint32_t *kB = (uint32_t *)(ws + n4);
    uint32_t *kC = (uint32_t *)(ws + 2 * n4);
    int32_t *vT = (int32_t *)(ws + 3 * n4);
    int32_t *vP = (int32_t *)(ws + 4 * n4);
    char *rws = ws + 5 * n4;
    const size_t rws_bytes = align256(radix_workspace_bytes(n));
    char *sws = rws + rws_bytes;
    const unsigned g = grid_for(n);
    int32_t rc;

    const int RW = record_words(d, plan->dtype);
    if (plan->layout == GHN_LAYOUT_DENSE && RW > 0 && knob("GHN_FIT_STREAM", 1) != 0) {
        rc = fit_stream(plan, X, out, ws, sws, p, s);
        if (rc != GHN_ERR_UNSUPPORTED) return rc;   // unsupported: a bucket too large, use the chain below
    }
    if (plan->layout == GHN_LAYOUT_DENSE && RW > 0) {
        // counting scatter: histogram into pt_off[0..E), scan in place (E+1)
        const int64_t E = plan->E;
        // 16-bit counters in the cursor region (dead until after the scan)
        uint32_t *packed = (uint32_t *)(ws + plan->fast_cursor_off);
        GHN_CUDA_CHECK(cudaMemsetAsync(packed, 0, (size_t)((E + 1) / 2) * 4, s));
        hist16_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, packed);
        GHN_LAUNCH_CHECK("hist16_kernel");
        unpack16_kernel<<<grid_for(E + 1), FIT_THREADS, 0, s>>>(packed, E, out->pt_off);
        GHN_LAUNCH_CHECK("unpack16_kernel");
        rc = exclusive_scan_i32(out->pt_off, out->pt_off, E + 1, sws, s);
        if (rc) return rc;
        int32_t *dmax = (int32_t *)kA;
        int32_t hres[2] = {0, 0};   // largest cell, points counted
        GHN_CUDA_CHECK(cudaMemsetAsync(dmax, 0, 4, s));
        max_count_kernel<<<grid_for(E), FIT_THREADS, 0, s>>>(out->pt_off, E, dmax);
        GHN_LAUNCH_CHECK("max_count_kernel");
        GHN_CUDA_CHECK(cudaMemcpyAsync(&hres[0], dmax, 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaMemcpyAsync(&hres[1], out->pt_off + E, 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        if ((int64_t)hres[1] != n) {   // a 16-bit counter overflowed: exact int32 histogram
            GHN_CUDA_CHECK(cudaMemsetAsync(out->pt_off, 0, (size_t)(E + 1) * 4, s));
            hist_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, out->pt_off);
            GHN_LAUNCH_CHECK("hist_kernel");
            rc = exclusive_scan_i32(out->pt_off, out->pt_off, E + 1, sws, s);
            if (rc) return rc;
            GHN_CUDA_CHECK(cudaMemsetAsync(dmax, 0, 4, s));
            max_count_kernel<<<grid_for(E), FIT_THREADS, 0, s>>>(out->pt_off, E, dmax);
            GHN_LAUNCH_CHECK("max_count_kernel");
            GHN_CUDA_CHECK(cudaMemcpyAsync(&hres[0], dmax, 4, cudaMemcpyDeviceToHost, s));
            GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        }
        const int32_t hmax = hres[0];
        if (hmax <= FAST_MAX_CELL) {
            int32_t *cursor = (int32_t *)(ws + plan->fast_cursor_off);
            uint32_t *rec = (uint32_t *)(ws + plan->fast_rec_off);
            GHN_CUDA_CHECK(cudaMemcpyAsync(cursor, out->pt_off, (size_t)E * 4, cudaMemcpyDeviceToDevice, s));
            // locality pass: partition by the top key bits, then scatter bucket by bucket
            const int kb = plan->key_bits > 0 ? plan->key_bits : 1;
            const int shift = kb > 10 ? kb - 10 : 0;
            const int nbuck = (int)(((E - 1) >> shift) + 1);
            uint32_t *part = (uint32_t *)(ws + fast_part_off(plan));
            int32_t *bcur = (int32_t *)(ws + fast_bcur_off(plan));
            bucket_start_kernel<<<(nbuck + 255) / 256, 256, 0, s>>>(out->pt_off, shift, nbuck, bcur);
            GHN_LAUNCH_CHECK("bucket_start_kernel");
            const unsigned gp = (unsigned)((n + PART_CHUNK - 1) / PART_CHUNK);
            const int RWP = part_words(d, plan->dtype);
            if (RWP == 4) {
                partition_kernel<T, 4><<<gp, PART_THREADS, 0, s>>>(X, n, p, shift, out->labels_in, bcur, part);
                GHN_LAUNCH_CHECK("partition_kernel");
                if (RW == 4)
                    scatter_part_kernel<T, 4, 4><<<g, FIT_THREADS, 0, s>>>(part, n, p, cursor, rec);
                else
                    scatter_part_kernel<T, 4, 8><<<g, FIT_THREADS, 0, s>>>(part, n, p, cursor, rec);
            } else {
                partition_kernel<T, 8><<<gp, PART_THREADS, 0, s>>>(X, n, p, shift, out->labels_in, bcur, part);
                GHN_LAUNCH_CHECK("partition_kernel");
                scatter_part_kernel<T, 8, 8><<<g, FIT_THREADS, 0, s>>>(part, n, p, cursor, rec);
            }
            GHN_LAUNCH_CHECK("scatter_part_kernel");
            if (RW == 4)
                fixup_records_kernel<T, 4><<<g, FIT_THREADS, 0, s>>>(rec, n, p, out->pt_off, (T *)out->coords,
                                                                      out->perm, out->labels_perm);
            else
                fixup_records_kernel<T, 8><<<g, FIT_THREADS, 0, s>>>(rec, n, p, out->pt_off, (T *)out->coords,
                                                                      out->perm, out->labels_perm);
            GHN_LAUNCH_CHECK("fixup_records_kernel");
            ne_flag_kernel<<<grid_for(E + 1), FIT_THREADS, 0, s>>>(out->pt_off, E, out->ne_off);
            GHN_LAUNCH_CHECK("ne_flag_kernel");
            rc = exclusive_scan_i32(out->ne_off, out->ne_off, E + 1, sws, s);
            if (rc) return rc;
            cells_from_offsets_kernel<<<grid_for(E), FIT_THREADS, 0, s>>>(
                out->pt_off, out->ne_off, E, n, p, out->cell_start, out->cell_ids, out->n_cells);
            GHN_LAUNCH_CHECK("cells_from_offsets_kernel");
            return GHN_OK;
        }
        // a fat cell: fall through to the stable radix sort
    }
    if (plan->layout == GHN_LAYOUT_DENSE) {
        linear_key_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, kA);
        GHN_LAUNCH_CHECK("linear_key_kernel");
        rc = radix_sort_pairs(kA, nullptr, kB, out->perm, kC, vT, n, plan->key_bits, rws, s);
        if (rc) return rc;
        // kB = sorted keys; out->perm = order.  flags -> kA (as int32), cidx -> vT
        int32_t *flags = (int32_t *)kA;
        dense_flags_kernel<<<g, FIT_THREADS, 0, s>>>(kB, n, flags);
        GHN_LAUNCH_CHECK("dense_flags_kernel");
        rc = exclusive_scan_i32(flags, (int32_t *)kC, n, sws, s);
        if (rc) return rc;
        excl_to_cidx_kernel<<<g, FIT_THREADS, 0, s>>>((int32_t *)kC, flags, vT, n);
        GHN_LAUNCH_CHECK("excl_to_cidx_kernel");
        // ne flags live in ne_off before the scan
        GHN_CUDA_CHECK(cudaMemsetAsync(out->ne_off, 0, (size_t)(plan->E + 1) * 4, s));
        dense_emit_kernel<<<g, FIT_THREADS, 0, s>>>(kB, n, vT, p, out->cell_start, out->cell_ids,
                                                   out->n_cells, out->ne_off);
        GHN_LAUNCH_CHECK("dense_emit_kernel");
        rc = exclusive_scan_i32(out->ne_off, out->ne_off, plan->E + 1, sws, s);
        if (rc) return rc;
        pt_off_kernel<<<grid_for(plan->E + 1), FIT_THREADS, 0, s>>>(out->ne_off, out->cell_start,
                                                                    out->pt_off, plan->E + 1);
        GHN_LAUNCH_CHECK("pt_off_kernel");
    } else {
        // LIST: stable sort by each dimension, least significant (last) first.
        int32_t *cur = nullptr;       // nullptr = identity
        int32_t *bufs[2] = {vP, out->perm};
        int which = 0;
        for (int j = d - 1; j >= 0; --j) {
            dim_key_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, j, cur, kA);
            GHN_LAUNCH_CHECK("dim_key_kernel");
            int32_t *dst = bufs[which];
            rc = radix_sort_pairs(kA, cur, kB, dst, kC, vT, n, bits_for((uint64_t)(plan->ext[j] - 1)), rws, s);
            if (rc) return rc;
            cur = dst;
            which ^= 1;
        }
        if (cur != out->perm) GHN_CUDA_CHECK(cudaMemcpyAsync(out->perm, cur, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
        int32_t *flags = (int32_t *)kA;
        list_flags_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, out->perm, flags);
        GHN_LAUNCH_CHECK("list_flags_kernel");
        rc = exclusive_scan_i32(flags, (int32_t *)kC, n, sws, s);
        if (rc) return rc;
        excl_to_cidx_kernel<<<g, FIT_THREADS, 0, s>>>((int32_t *)kC, flags, vT, n);
        GHN_LAUNCH_CHECK("excl_to_cidx_kernel");
        list_emit_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, p, out->perm, vT, out->cell_start,
                                                       out->cell_ids, out->n_cells);
        GHN_LAUNCH_CHECK("list_emit_kernel");
    }
    gather_coords_kernel<T><<<g, FIT_THREADS, 0, s>>>(X, n, d, out->perm, (T *)out->coords,
                                                       out->labels_in, out->labels_perm);
    GHN_LAUNCH_CHECK("gather_coords_kernel");
    (void)ws_bytes;
    return GHN_OK;
}

}  // namespace
}  // namespace ghn

using namespace ghn;

extern "C" int32_t ghn_fit_bounds(const void *X, int32_t dtype, int64_t n, int32_t d,
                                  const double *widths, int64_t *out_bounds, double *out_origin,
                                  int32_t *out_flags, void *stream) {
    if (n <= 0) {
        set_error("empty dataset");
        return GHN_ERR_VALUE;
    }
    if (d < 1 || d > GHN_MAX_DIM) {
        set_error("d=%d unsupported (1..%d)", d, GHN_MAX_DIM);
        return GHN_ERR_UNSUPPORTED;
    }
    for (int j = 0; j < d; ++j) {
        if (!(widths[j] > 0.0) || !isfinite(widths[j])) {
            set_error("all cell widths must be positive");
            return GHN_ERR_VALUE;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    DimParams p = make_dims(d, widths, nullptr, nullptr);
    // origin keys are staged in out_origin's bytes (same size as uint64)
    unsigned long long *okey = (unsigned long long *)out_origin;
    bounds_init_kernel<<<1, 32, 0, s>>>(out_bounds, okey, out_flags, d);
    GHN_LAUNCH_CHECK("bounds_init_kernel");
    int32_t rc = dtype == GHN_F32
                     ? bounds_launch<float>((const float *)X, n, d, p, out_bounds, okey, out_flags, s)
                     : bounds_launch<double>((const double *)X, n, d, p, out_bounds, okey, out_flags, s);
    if (rc) return rc;
    origin_decode_kernel<<<1, 32, 0, s>>>(okey, out_origin, out_bounds, p);
    GHN_LAUNCH_CHECK("origin_decode_kernel");
    return GHN_OK;
}

extern "C" int32_t ghn_fit_plan_init(ghn_fit_plan *plan, int64_t n, int32_t d, int32_t dtype,
                                     const double *widths, const int64_t *bounds_host,
                                     int64_t dense_limit) {
    memset(plan, 0, sizeof(*plan));
    if (n <= 0 || n > 0x7ffffffeLL) {
        set_error("n=%lld out of range", (long long)n);
        return n <= 0 ? GHN_ERR_VALUE : GHN_ERR_UNSUPPORTED;
    }
    if (d < 1 || d > GHN_MAX_DIM) {
        set_error("d=%d unsupported", d);
        return GHN_ERR_UNSUPPORTED;
    }
    plan->n = n;
    plan->d = d;
    plan->dtype = dtype;
    double Ed = 1.0;
    for (int j = 0; j < d; ++j) {
        plan->widths[j] = widths[j];
        plan->lo[j] = bounds_host[j];
        int64_t hi = bounds_host[d + j];
        if (hi < plan->lo[j]) {
            set_error("bounds not computed");
            return GHN_ERR_VALUE;
        }
        plan->ext[j] = hi - plan->lo[j] + 1;
        if (plan->ext[j] > 0x7fffffffLL || plan->ext[j] <= 0) {
            set_error("grid extent %lld along dim %d exceeds the int32 id range", (long long)plan->ext[j], j);
            return GHN_ERR_UNSUPPORTED;
        }
        Ed *= (double)plan->ext[j];
    }
    if (dense_limit > (1LL << 31)) dense_limit = 1LL << 31;
    if (Ed <= (double)dense_limit) {
        plan->layout = GHN_LAYOUT_DENSE;
        plan->E = (int64_t)Ed;
        plan->key_bits = bits_for((uint64_t)(plan->E - 1));
    } else {
        plan->layout = GHN_LAYOUT_LIST;
        plan->E = 0;
    }
    size_t n4 = align256((size_t)n * 4);
    size_t scan_len = (size_t)n + 1;
    if (plan->layout == GHN_LAYOUT_DENSE && (size_t)plan->E + 1 > scan_len) scan_len = plan->E + 1;
    plan->workspace_bytes = 5 * n4 + align256(radix_workspace_bytes(n)) + scan_workspace_bytes(scan_len) + 256;
    // counting-scatter fast path (DENSE): cursor (E+1) + records (n x RW words),
    // laid out after the scan workspace region used by both paths
    const int RW = record_words(d, dtype);
    if (plan->layout == GHN_LAYOUT_DENSE && RW > 0) {
        const size_t base = 5 * n4 + align256(radix_workspace_bytes(n)) + align256(scan_workspace_bytes(scan_len));
        plan->fast_cursor_off = base;
        plan->fast_rec_off = base + align256((size_t)(plan->E + 1) * 4);
        // bucket cursors (chain) / streaming-fit bucket counts, cursors, max
        const size_t need = fast_bcur_off(plan) + 4 * align256((size_t)(SF_MAX_BUCKETS + 1) * 4);
        if (need > plan->workspace_bytes) plan->workspace_bytes = need;
    }
    return GHN_OK;
}

extern "C" int32_t ghn_fit_build(const ghn_fit_plan *plan, const void *X, const ghn_fit_out *out,
                                 void *workspace, size_t workspace_bytes, void *stream) {
    if (workspace_bytes < plan->workspace_bytes) {
        set_error("workspace too small: %zu < %zu", workspace_bytes, plan->workspace_bytes);
        return GHN_ERR_VALUE;
    }
    if (plan->layout == GHN_LAYOUT_DENSE && (!out->pt_off || !out->ne_off)) {
        set_error("DENSE layout needs pt_off and ne_off");
        return GHN_ERR_VALUE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (plan->dtype == GHN_F32)
        return fit_build_impl<float>(plan, (const float *)X, out, (char *)workspace, workspace_bytes, s);
    return fit_build_impl<double>(plan, (const double *)X, out, (char *)workspace, workspace_bytes, s);
}
