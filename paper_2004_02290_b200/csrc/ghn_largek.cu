// ghn_largek.cu -- knn_query for k > 256 (explore.py:66-137 allows any
// 1 <= k <= n; baselines.brute_knn with k = n returns every point sorted).
//
// The warp-resident top-k of the generic kernel holds at most 256 entries.
// Past that, each query runs here, layer by layer, from the host:
//   gather   every candidate of block(l) (cells at Chebyshev distance <= l,
//            or all points in brute mode): fp64 key (numpy einsum order /
//            L1 / L-inf, core.py:72-86), point index, and whether its cell
//            lies on shell l; plus the shell's cell / point counts
//   sort     stable LSD radix passes by index, key low word, key high word
//            == np.lexsort((idx, key)) (explore.py:114); keys are >= +0, so
//            their IEEE bit patterns sort like the values
//   select   T_l = the first k; changed(l) <=> T_l holds a shell-l point
//            (the top-k after merging layer l = the top-k of block(l))
//   stop     on the host, exactly explore.py:119-130
//   epilogue one thread: distances / indices, the vote with the
//            (sqrt(key), index) tie-break, the numpy pairwise mean or the
//            median (predict.py:20-50)
// One device sync per layer: this path serves correctness at large k, not
// throughput.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "ghn_common.cuh"

namespace ghn {
namespace {

constexpr int LK_THREADS = 256;

struct LkArgs {
    ghn_index_view ix;
    double q[GHN_MAX_DIM];
    int64_t r[GHN_MAX_DIM];   // query cell relative to lo
    int64_t l;
    int32_t brute;
};

struct LkCounters {
    int32_t count;            // candidates gathered
    int32_t pad;
    unsigned long long cells; // non-empty cells on shell l
    unsigned long long points;
};

template <typename T>
__device__ __forceinline__ void lk_emit(const LkArgs &a, int64_t slot, bool shell, uint32_t *khi, uint32_t *klo,
                                        uint32_t *kidx, uint8_t *flag, LkCounters *cnt) {
    const int d = a.ix.d;
    const T *coords = (const T *)a.ix.coords;
    double df[GHN_MAX_DIM];
    for (int j = 0; j < d; ++j) df[j] = __dsub_rn(to_double(coords[(int64_t)j * a.ix.n + slot]), a.q[j]);
    const double key = metric_key_rt(df, d, a.ix.metric);
    const unsigned long long b = (unsigned long long)__double_as_longlong(key);
    const int pos = atomicAdd(&cnt->count, 1);
    khi[pos] = (uint32_t)(b >> 32);
    klo[pos] = (uint32_t)b;
    kidx[pos] = (uint32_t)a.ix.perm[slot];
    flag[pos] = shell ? 1 : 0;
}

// DENSE: one thread per row of block(l) over the first d-1 dimensions.
template <typename T>
__global__ void __launch_bounds__(LK_THREADS) lk_gather_dense_kernel(const LkArgs a, int64_t rows, uint32_t *khi,
                                                                    uint32_t *klo, uint32_t *kidx, uint8_t *flag,
                                                                    LkCounters *cnt) {
    const ghn_index_view &ix = a.ix;
    const int d = ix.d, jl = d - 1;
    int64_t lo_c[GHN_MAX_DIM], hi_c[GHN_MAX_DIM];
    for (int j = 0; j < d; ++j) {
        lo_c[j] = max((int64_t)0, a.r[j] - a.l);
        hi_c[j] = min(ix.ext[j] - 1, a.r[j] + a.l);
    }
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = t, rowlin = 0, mul = 1, cheb = 0;
        for (int j = jl - 1; j >= 0; --j) {
            const int64_t len = hi_c[j] - lo_c[j] + 1;
            const int64_t rj = lo_c[j] + rem % len;
            rem /= len;
            const int64_t v = rj > a.r[j] ? rj - a.r[j] : a.r[j] - rj;
            cheb = v > cheb ? v : cheb;
            rowlin += rj * mul;
            mul *= ix.ext[j];
        }
        const int64_t base = rowlin * ix.ext[jl];
        unsigned long long sc = 0, sp = 0;
        for (int64_t z = lo_c[jl]; z <= hi_c[jl]; ++z) {
            const int64_t vz = z > a.r[jl] ? z - a.r[jl] : a.r[jl] - z;
            const bool shell = (cheb > vz ? cheb : vz) == a.l;
            const int32_t s0 = ix.pt_off[base + z], s1 = ix.pt_off[base + z + 1];
            if (shell && s1 > s0) {
                ++sc;
                sp += (unsigned long long)(s1 - s0);
            }
            for (int32_t s = s0; s < s1; ++s) lk_emit<T>(a, s, shell, khi, klo, kidx, flag, cnt);
        }
        if (sc) {
            atomicAdd(&cnt->cells, sc);
            atomicAdd(&cnt->points, sp);
        }
    }
}

// LIST layout (and brute mode over every cell): one thread per non-empty cell.
template <typename T>
__global__ void __launch_bounds__(LK_THREADS) lk_gather_list_kernel(const LkArgs a, uint32_t *khi, uint32_t *klo,
                                                                   uint32_t *kidx, uint8_t *flag, LkCounters *cnt) {
    const ghn_index_view &ix = a.ix;
    const int d = ix.d;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ix.n_cells;
         c += (int64_t)gridDim.x * blockDim.x) {
        int64_t cheb = 0;
        for (int j = 0; j < d; ++j) {
            const int64_t v = (int64_t)ix.cell_ids[c * d + j] - a.r[j];
            const int64_t av = v < 0 ? -v : v;
            cheb = av > cheb ? av : cheb;
        }
        if (!a.brute && cheb > a.l) continue;
        const bool shell = !a.brute && cheb == a.l;
        const int32_t s0 = ix.cell_start[c], s1 = ix.cell_start[c + 1];
        if (shell) {
            atomicAdd(&cnt->cells, 1ull);
            atomicAdd(&cnt->points, (unsigned long long)(s1 - s0));
        }
        for (int32_t s = s0; s < s1; ++s) lk_emit<T>(a, s, shell, khi, klo, kidx, flag, cnt);
    }
}

__global__ void lk_gather_u32_kernel(const uint32_t *src, const int32_t *perm, int64_t m, uint32_t *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

struct LkLayer {
    int32_t count;
    int32_t changed;
    double kth;
};

// T_l: the first min(k, m) sorted candidates, changed flag, k-th key.
__global__ void lk_select_kernel(const uint32_t *khi, const uint32_t *klo, const uint32_t *kidx, const uint8_t *flag,
                                 const int32_t *order, int32_t m, int32_t k, double *tkey, int32_t *tidx,
                                 LkLayer *res) {
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    const int take = m < k ? m : k;
    int mine = 0;
    for (int t = threadIdx.x; t < take; t += blockDim.x) {
        const int p = order[t];
        tkey[t] = __longlong_as_double((long long)(((unsigned long long)khi[p] << 32) | klo[p]));
        tidx[t] = (int32_t)kidx[p];
        mine |= flag[p];
    }
    if (mine) atomicOr(&any, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        res->count = m;
        res->changed = any;
        res->kth = take >= k ? tkey[k - 1] : INFINITY;
    }
}

__device__ double lk_pairwise(const double *v, int64_t n) {
    // numpy pairwise_sum (add.reduce over contiguous doubles)
    if (n < 8) {
        double r = n > 0 ? v[0] : 0.0;
        for (int64_t i = 1; i < n; ++i) r = __dadd_rn(r, v[i]);
        return r;
    }
    if (n <= 128) {
        double acc[8];
        for (int t = 0; t < 8; ++t) acc[t] = v[t];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int t = 0; t < 8; ++t) acc[t] = __dadd_rn(acc[t], v[i + t]);
        double r = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                             __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
        for (; i < n; ++i) r = __dadd_rn(r, v[i]);
        return r;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(lk_pairwise(v, n2), lk_pairwise(v + n2, n - n2));
}

// One query's outputs from its final T (sorted by (key, index)).  lab /
// tvals are scratch of k entries; slab / sord: the labels of T sorted (by a
// radix pass on the host side) with their T positions.
__global__ void lk_epilogue_kernel(ghn_index_view ix, const double *tkey, const int32_t *tidx, int32_t k,
                                   int32_t task, int64_t qi, ghn_query_out o, const int64_t *stats3,
                                   const uint32_t *slab, const int32_t *sord, double *tvals) {
    if (threadIdx.x != 0) return;
    if (o.idx || o.dist)
        for (int t = 0; t < k; ++t) {
            if (o.idx) o.idx[qi * k + t] = tidx[t];
            if (o.dist) o.dist[qi * k + t] = key_to_dist(tkey[t], ix.metric);
        }
    if (o.stats)
        for (int j = 0; j < 3; ++j) o.stats[qi * 3 + j] = stats3[j];
    if (o.totals) {
        atomicAdd(&o.totals[0], (unsigned long long)stats3[0]);
        atomicAdd(&o.totals[1], (unsigned long long)stats3[1]);
        atomicAdd(&o.totals[2], (unsigned long long)stats3[2]);
        atomicAdd(&o.totals[3], 1ull);
    }
    if (task == GHN_TASK_CLASSIFY && ix.labels) {
        // counts per label from the sorted labels; ties -> nearest member by (sqrt key, index)
        int best = 0;
        for (int i = 0; i < k;) {
            int j = i;
            while (j < k && slab[j] == slab[i]) ++j;
            best = j - i > best ? j - i : best;
            i = j;
        }
        double bd = INFINITY;
        int32_t bi = 0x7fffffff, bl = 0;
        for (int i = 0; i < k;) {
            int j = i;
            while (j < k && slab[j] == slab[i]) ++j;
            if (j - i == best)
                for (int u = i; u < j; ++u) {
                    const int t = sord[u];
                    const double dd = key_to_dist(tkey[t], ix.metric);
                    if (pair_less(dd, tidx[t], bd, bi)) {
                        bd = dd;
                        bi = tidx[t];
                        bl = (int32_t)(slab[u] ^ 0x80000000u);
                    }
                }
            i = j;
        }
        if (o.label) o.label[qi] = bl;
        if (o.confidence) o.confidence[qi] = __ddiv_rn((double)best, (double)k);
    } else if ((task == GHN_TASK_REGRESS_MEAN || task == GHN_TASK_REGRESS_MEDIAN) && ix.targets) {
        for (int t = 0; t < k; ++t) tvals[t] = ix.targets[tidx[t]];
        if (task == GHN_TASK_REGRESS_MEAN) {
            if (o.value) o.value[qi] = __ddiv_rn(lk_pairwise(tvals, k), (double)k);
        } else {
            // tvals sorted in place (insertion sort would be O(k^2): heap sort)
            int64_t nn = k;
            auto sift = [&](int64_t i, int64_t end) {
                for (;;) {
                    int64_t c = 2 * i + 1;
                    if (c >= end) break;
                    if (c + 1 < end && tvals[c + 1] > tvals[c]) ++c;
                    if (!(tvals[c] > tvals[i])) break;
                    const double tmp = tvals[c];
                    tvals[c] = tvals[i];
                    tvals[i] = tmp;
                    i = c;
                }
            };
            for (int64_t i = nn / 2 - 1; i >= 0; --i) sift(i, nn);
            for (int64_t e = nn - 1; e > 0; --e) {
                const double tmp = tvals[0];
                tvals[0] = tvals[e];
                tvals[e] = tmp;
                sift(0, e);
            }
            const double m1 = tvals[(k - 1) / 2], m2 = tvals[k / 2];
            if (o.value) o.value[qi] = (k & 1) ? m1 : __ddiv_rn(__dadd_rn(m1, m2), 2.0);
        }
    }
}

__global__ void lk_labels_kernel(const int32_t *labels, const int32_t *tidx, int32_t k, uint32_t *lab) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k; t += gridDim.x * blockDim.x)
        lab[t] = (uint32_t)labels[tidx[t]] ^ 0x80000000u;   // signed order as unsigned
}

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

unsigned lk_grid(int64_t m) {
    int64_t g = (m + LK_THREADS - 1) / LK_THREADS;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

size_t largek_workspace_bytes(const ghn_index_view *ix, int32_t k) {
    const size_t n4 = a256((size_t)ix->n * 4);
    return 9 * n4 + a256((size_t)ix->n) + a256(radix_workspace_bytes(ix->n)) + 3 * a256((size_t)k * 8) + 1024;
}

int32_t largek_query(const ghn_index_view *ix, const void *Q, int32_t q_dtype, int64_t nq, int32_t k, int32_t mode,
                     int32_t task, const ghn_query_out *out, void *workspace, size_t workspace_bytes,
                     cudaStream_t s) {
    if (!workspace || workspace_bytes < largek_workspace_bytes(ix, k)) {
        set_error("query workspace too small for k=%d", k);
        return GHN_ERR_VALUE;
    }
    const int64_t n = ix->n;
    const int d = ix->d;
    char *ws = (char *)workspace;
    const size_t n4 = a256((size_t)n * 4);
    uint32_t *khi = (uint32_t *)ws, *klo = (uint32_t *)(ws + n4), *kidx = (uint32_t *)(ws + 2 * n4);
    uint32_t *ka = (uint32_t *)(ws + 3 * n4), *kb = (uint32_t *)(ws + 4 * n4), *kt = (uint32_t *)(ws + 5 * n4);
    int32_t *p0 = (int32_t *)(ws + 6 * n4), *p1 = (int32_t *)(ws + 7 * n4), *pt = (int32_t *)(ws + 8 * n4);
    uint8_t *flag = (uint8_t *)(ws + 9 * n4);
    char *rws = ws + 9 * n4 + a256((size_t)n);
    char *tail = rws + a256(radix_workspace_bytes(n));
    double *tkey = (double *)tail;
    int32_t *tidx = (int32_t *)(tail + a256((size_t)k * 8));
    double *tvals = (double *)(tail + 2 * a256((size_t)k * 8));
    char *small = tail + 3 * a256((size_t)k * 8);
    LkCounters *cnt = (LkCounters *)small;
    LkLayer *res = (LkLayer *)(small + 256);
    int64_t *stats3 = (int64_t *)(small + 512);
    // queries on the host (the layer loop runs here)
    std::vector<double> qh((size_t)nq * d);
    if (q_dtype == GHN_F32) {
        std::vector<float> qf((size_t)nq * d);
        GHN_CUDA_CHECK(cudaMemcpyAsync(qf.data(), Q, qf.size() * 4, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
        for (size_t i = 0; i < qf.size(); ++i) qh[i] = (double)qf[i];
    } else {
        GHN_CUDA_CHECK(cudaMemcpyAsync(qh.data(), Q, qh.size() * 8, cudaMemcpyDeviceToHost, s));
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    LkArgs a;
    memset(&a, 0, sizeof(a));
    a.ix = *ix;
    a.brute = mode == GHN_MODE_BRUTE;
    for (int64_t qi = 0; qi < nq; ++qi) {
        int64_t lmin = 0, lmax = 0;
        for (int j = 0; j < d; ++j) {
            const double x = qh[(size_t)qi * d + j];
            double inv = 0.0;
            const double t = is_pow2_width(ix->widths[j], &inv) ? x * inv : x / ix->widths[j];
            double f = floor(t);
            f = fmin(fmax(f, -4.6116860184273879e18), 4.6116860184273879e18);
            a.q[j] = x;
            a.r[j] = (int64_t)f - ix->lo[j];
            const int64_t e1 = ix->ext[j] - 1;
            const int64_t outd = a.r[j] < 0 ? -a.r[j] : (a.r[j] > e1 ? a.r[j] - e1 : 0);
            lmin = outd > lmin ? outd : lmin;
            const int64_t far = std::max(a.r[j] < 0 ? -a.r[j] : a.r[j], e1 - a.r[j] < 0 ? a.r[j] - e1 : e1 - a.r[j]);
            lmax = far > lmax ? far : lmax;
        }
        int64_t st[3] = {0, 0, 0};
        int32_t have = 0;   // entries in T (the buffer)
        for (int64_t l = lmin;; ++l) {
            a.l = l;
            GHN_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(LkCounters), s));
            if (a.brute || ix->layout == GHN_LAYOUT_LIST) {
                if (ix->dtype == GHN_F32)
                    lk_gather_list_kernel<float><<<lk_grid(ix->n_cells), LK_THREADS, 0, s>>>(a, khi, klo, kidx, flag, cnt);
                else
                    lk_gather_list_kernel<double><<<lk_grid(ix->n_cells), LK_THREADS, 0, s>>>(a, khi, klo, kidx, flag, cnt);
            } else {
                int64_t rows = 1;
                for (int j = 0; j + 1 < d; ++j)
                    rows *= std::min(ix->ext[j] - 1, a.r[j] + l) - std::max((int64_t)0, a.r[j] - l) + 1;
                if (ix->dtype == GHN_F32)
                    lk_gather_dense_kernel<float><<<lk_grid(rows), LK_THREADS, 0, s>>>(a, rows, khi, klo, kidx, flag, cnt);
                else
                    lk_gather_dense_kernel<double><<<lk_grid(rows), LK_THREADS, 0, s>>>(a, rows, khi, klo, kidx, flag, cnt);
            }
            GHN_LAUNCH_CHECK("lk_gather_kernel");
            LkCounters hc;
            GHN_CUDA_CHECK(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
            GHN_CUDA_CHECK(cudaStreamSynchronize(s));
            const int32_t m = hc.count;
            // stable sort by (key, index): index, then key low word, then key high word
            int32_t rc = radix_sort_pairs(kidx, nullptr, ka, p0, kt, pt, m, 31, rws, s);
            if (rc) return rc;
            lk_gather_u32_kernel<<<lk_grid(m), LK_THREADS, 0, s>>>(klo, p0, m, kb);
            GHN_LAUNCH_CHECK("lk_gather_u32_kernel");
            rc = radix_sort_pairs(kb, p0, ka, p1, kt, pt, m, 32, rws, s);
            if (rc) return rc;
            lk_gather_u32_kernel<<<lk_grid(m), LK_THREADS, 0, s>>>(khi, p1, m, kb);
            GHN_LAUNCH_CHECK("lk_gather_u32_kernel");
            rc = radix_sort_pairs(kb, p1, ka, p0, kt, pt, m, 32, rws, s);
            if (rc) return rc;
            lk_select_kernel<<<1, 1024, 0, s>>>(khi, klo, kidx, flag, p0, m, k, tkey, tidx, res);
            GHN_LAUNCH_CHECK("lk_select_kernel");
            LkLayer hl;
            GHN_CUDA_CHECK(cudaMemcpyAsync(&hl, res, sizeof(hl), cudaMemcpyDeviceToHost, s));
            GHN_CUDA_CHECK(cudaStreamSynchronize(s));
            have = m < k ? m : k;
            if (a.brute) {   // exact full scan: the generic kernel's brute stats
                st[0] = 0;
                st[1] = ix->n_cells;
                st[2] = ix->n;
                break;
            }
            st[0] = l;
            st[1] += (int64_t)hc.cells;
            st[2] += (int64_t)hc.points;
            const bool full = have >= k;
            if (full) {
                if (mode == GHN_MODE_HEURISTIC && !hl.changed) break;
                if (mode == GHN_MODE_GUARANTEED) {
                    const double b = (double)l * ix->min_width;
                    const double bk = ix->metric == GHN_METRIC_EUCLIDEAN ? b * b : b;
                    if (bk > hl.kth) break;
                }
            }
            if (l >= lmax) break;
        }
        (void)have;
        GHN_CUDA_CHECK(cudaMemcpyAsync(stats3, st, sizeof(st), cudaMemcpyHostToDevice, s));
        uint32_t *slab = nullptr;
        int32_t *sord = nullptr;
        if (task == GHN_TASK_CLASSIFY && ix->labels) {
            lk_labels_kernel<<<lk_grid(k), LK_THREADS, 0, s>>>(ix->labels, tidx, k, kb);
            GHN_LAUNCH_CHECK("lk_labels_kernel");
            int32_t rc = radix_sort_pairs(kb, nullptr, ka, p0, kt, pt, k, 32, rws, s);
            if (rc) return rc;
            slab = ka;
            sord = p0;
        }
        lk_epilogue_kernel<<<1, 32, 0, s>>>(*ix, tkey, tidx, k, task, qi, *out, stats3, slab, sord, tvals);
        GHN_LAUNCH_CHECK("lk_epilogue_kernel");
        GHN_CUDA_CHECK(cudaStreamSynchronize(s));   // stats3 (host memory) must outlive the copy
    }
    return GHN_OK;
}

}  // namespace ghn
