// ghn_query.cu -- batched GHN predict for sm_100a.
//
// One warp per query (queries visited in central-cell order, K8 binning, so
// warps resident on an SM share neighbourhoods in L1/L2).  Per query:
//   centre     floor(q / w) in fp64                         explore.py:91
//   layers     l = l_min .. : the Chebyshev shell of radius l, clipped to
//              the id bounding box, enumerated as row segments along the
//              last dimension (one contiguous CSR slot range per segment);
//              a shell with more rows than there are non-empty cells is
//              scanned from the cell list instead (explore.py:105)
//   keys       fp64 squared L2 in numpy einsum order        core.py:78-80
//   top-k      warp-distributed sorted (key, index) list, KS entries per
//              lane; candidates pass a k-th-key filter before the index
//              load                                          explore.py:112-118
//   stop       heuristic: full buffer and no insertion in the layer;
//              guaranteed: (l*min_w)^2 > k-th key; always at l >= max_layer
//                                                            explore.py:119-130
//   epilogue   vote with (sqrt key, index) tie-break / numpy pairwise mean
//                                                            predict.py:20-47
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "ghn_common.cuh"
#include "ghn_tile2d.cuh"

namespace ghn {
namespace {

constexpr int Q_THREADS = 256;
constexpr int Q_WARPS = Q_THREADS / 32;

struct QArgs {
    ghn_index_view ix;
    double inv_w[GHN_MAX_DIM];
    uint32_t pow2;
    const void *Q;
    int32_t q_dtype;
    int64_t nq;
    int32_t k;
    int32_t mode;
    int32_t task;
    const int32_t *qorder;
    const int32_t *nq_dev;   // device count (fallback list); overrides nq when set
    ghn_query_out out;
};

template <int D>
struct DimOf {
    static constexpr int v = D > 0 ? D : 1;
};

// Warp-wide top-k: slot t = s*32 + lane, sorted ascending by (key, idx).
template <int KS>
struct TopK {
    double key[KS];
    int32_t idx[KS];
    int filled;          // warp-uniform
    double thr_key;      // k-th entry once filled == k
    int32_t thr_idx;

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            key[s] = INFINITY;
            idx[s] = 0x7fffffff;
        }
        filled = 0;
        thr_key = INFINITY;
        thr_idx = 0x7fffffff;
    }

    // Insert a warp-uniform candidate known to belong in the top-k.
    __device__ __forceinline__ void insert(double ck, int32_t ci, int k) {
        const int lane = lane_id();
        int pos = 0;
#pragma unroll
        for (int s = 0; s < KS; ++s) pos += __popc(__ballot_sync(GHN_FULL, pair_less(key[s], idx[s], ck, ci)));
        double rk[KS];
        int32_t ri[KS];
        const int src = (lane + 31) & 31;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            rk[s] = shfl_d(key[s], src);
            ri[s] = __shfl_sync(GHN_FULL, idx[s], src);
        }
#pragma unroll
        for (int s = KS - 1; s >= 0; --s) {
            const int t = s * 32 + lane;
            double pk;
            int32_t pi;
            if (lane == 0) {
                pk = s > 0 ? rk[s > 0 ? s - 1 : 0] : INFINITY;
                pi = s > 0 ? ri[s > 0 ? s - 1 : 0] : 0x7fffffff;
            } else {
                pk = rk[s];
                pi = ri[s];
            }
            if (t < k) {
                if (t == pos) {
                    key[s] = ck;
                    idx[s] = ci;
                } else if (t > pos) {
                    key[s] = pk;
                    idx[s] = pi;
                }
            }
        }
        if (filled < k) ++filled;
        if (filled == k) {
            const int ts = (k - 1) >> 5, tl = (k - 1) & 31;
            double v = 0.0;
            int32_t vi = 0;
#pragma unroll
            for (int s = 0; s < KS; ++s)
                if (s == ts) {
                    v = key[s];
                    vi = idx[s];
                }
            thr_key = shfl_d(v, tl);
            thr_idx = __shfl_sync(GHN_FULL, vi, tl);
        }
    }
};

struct LayerAcc {
    bool changed;
    int64_t cells;
    int64_t points;
};

// Consume up to two slot ranges per lane: compute keys for every candidate,
// filter against the k-th entry, insert survivors in lane order.
template <typename T, int D, int KS>
__device__ __forceinline__ void consume(const QArgs &a, const double *qd, int d, int32_t s0,
                                        int32_t n0, int32_t s1, int32_t n1, TopK<KS> &tk,
                                        LayerAcc &acc) {
    const int lane = lane_id();
    const int cnt = n0 + n1;
    const int incl = warp_inclusive_scan(cnt);
    const int total = __shfl_sync(GHN_FULL, incl, 31);
    acc.points += total;
    if (total == 0) return;
    const int excl = incl - cnt;
    const T *__restrict__ coords = (const T *)a.ix.coords;
    const int64_t n = a.ix.n;
    const int k = a.k;
    for (int base = 0; base < total; base += 32) {
        const int m = base + lane;
        // owner lane L = #lanes with incl <= m
        int L = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            int v = __shfl_sync(GHN_FULL, incl, L + step - 1);
            if (v <= m) L += step;
        }
        if (L > 31) L = 31;
        const int exL = __shfl_sync(GHN_FULL, excl, L);
        const int n0L = __shfl_sync(GHN_FULL, n0, L);
        const int s0L = __shfl_sync(GHN_FULL, s0, L);
        const int s1L = __shfl_sync(GHN_FULL, s1, L);
        const bool act = m < total;
        const int off = m - exL;
        const int64_t slot = off < n0L ? (int64_t)s0L + off : (int64_t)s1L + (off - n0L);
        double key = INFINITY;
        if (act) {
            if (D > 0) {
                constexpr int DC = DimOf<D>::v;
                double df[DC];
#pragma unroll
                for (int j = 0; j < DC; ++j)
                    df[j] = __dsub_rn(to_double(coords[(int64_t)j * n + slot]), qd[j]);
                key = metric_key<DC>(df, a.ix.metric);
            } else {
                double df[GHN_MAX_DIM];
                for (int j = 0; j < d; ++j) df[j] = __dsub_rn(to_double(coords[(int64_t)j * n + slot]), qd[j]);
                key = metric_key_rt(df, d, a.ix.metric);
            }
        }
        bool pass = act && (tk.filled < k || key <= tk.thr_key);
        int32_t pidx = 0x7fffffff;
        if (pass) pidx = a.ix.perm[slot];
        unsigned sm = __ballot_sync(GHN_FULL, pass);
        while (sm) {
            const int src = __ffs(sm) - 1;
            sm &= sm - 1;
            const double ck = shfl_d(key, src);
            const int32_t ci = __shfl_sync(GHN_FULL, pidx, src);
            if (tk.filled >= k && !pair_less(ck, ci, tk.thr_key, tk.thr_idx)) continue;
            tk.insert(ck, ci, k);
            acc.changed = true;
        }
    }
}

__device__ __forceinline__ int64_t iabs64(int64_t v) { return v < 0 ? -v : v; }

// Visit the non-empty cells at Chebyshev distance exactly l.  Returns the
// next non-empty layer when it is known (cell-list scan), else l + 1.
template <typename T, int D, int KS>
__device__ __forceinline__ int64_t visit_layer(const QArgs &a, const double *qd, const int64_t *r, int d, int64_t l,
                               TopK<KS> &tk, LayerAcc &acc) {
    constexpr int DM = D > 0 ? D : GHN_MAX_DIM;
    const int lane = lane_id();
    const ghn_index_view &ix = a.ix;
    int32_t lo_c[DM], hi_c[DM];
    double rows = 1.0;
    bool empty = false;
#pragma unroll
    for (int j = 0; j < DM; ++j) {
        if (j >= d) break;
        int64_t x0 = r[j] - l, x1 = r[j] + l;
        int64_t e1 = ix.ext[j] - 1;
        x0 = x0 < 0 ? 0 : x0;
        x1 = x1 > e1 ? e1 : x1;
        if (x0 > x1) empty = true;
        lo_c[j] = (int32_t)x0;
        hi_c[j] = (int32_t)x1;
        if (j < d - 1) rows *= (double)(x1 - x0 + 1);
    }
    if (empty) return l + 1;
    if (ix.layout == GHN_LAYOUT_LIST || rows > (double)ix.n_cells) {
        // cell-list scan (explore.py:105), also finds the next non-empty layer
        int64_t next = INT64_MAX;
        for (int cb = 0; cb < ix.n_cells; cb += 32) {
            const int c = cb + lane;
            bool match = false;
            int32_t st = 0, cntp = 0;
            if (c < ix.n_cells) {
                int64_t ch = 0;
                for (int j = 0; j < d; ++j) {
                    int64_t v = iabs64((int64_t)ix.cell_ids[(int64_t)c * d + j] - r[j]);
                    ch = v > ch ? v : ch;
                }
                match = ch == l;
                if (ch > l && ch < next) next = ch;
                if (match) {
                    st = ix.cell_start[c];
                    cntp = ix.cell_start[c + 1] - st;
                }
            }
            acc.cells += __popc(__ballot_sync(GHN_FULL, match));
            if (__any_sync(GHN_FULL, match)) consume<T, D, KS>(a, qd, d, st, cntp, 0, 0, tk, acc);
        }
        return warp_min(next);
    }
    // dense row enumeration over the first d-1 dims
    const int jl = d - 1;
    const int64_t R = (int64_t)rows;
    const int64_t ext_last = ix.ext[jl];
    for (int64_t rb = 0; rb < R; rb += 32) {
        const int64_t t = rb + lane;
        int32_t s0 = 0, n0 = 0, s1 = 0, n1 = 0;
        int cells = 0;
        if (t < R) {
            // decode: last row dim fastest; rowlin is row-major over ext[0..d-2].
            // DENSE: E <= 2^30, so rows, ids and the linear cell index fit 32 bits.
            uint32_t rem = (uint32_t)t;
            int64_t cheb = 0;
            uint32_t rowlin = 0, mul = 1;
            for (int j = jl - 1; j >= 0; --j) {
                const uint32_t len = (uint32_t)(hi_c[j] - lo_c[j] + 1);
                uint32_t q = rem, rj = (uint32_t)lo_c[j];
                if (len != 1) {
                    q = rem / len;
                    rj += rem - q * len;
                }
                rem = q;
                const int64_t v = iabs64((int64_t)rj - r[j]);
                cheb = v > cheb ? v : cheb;
                rowlin += rj * mul;
                mul *= (uint32_t)ix.ext[j];
            }
            const int64_t rowbase = (int64_t)rowlin * ext_last;
            if (cheb == l) {
                const int64_t c0 = rowbase + lo_c[jl], c1 = rowbase + hi_c[jl] + 1;
                s0 = ix.pt_off[c0];
                n0 = ix.pt_off[c1] - s0;
                cells += ix.ne_off[c1] - ix.ne_off[c0];
            } else {
                const int64_t za = r[jl] - l, zb = r[jl] + l;
                if (za >= 0 && za < ext_last) {
                    s0 = ix.pt_off[rowbase + za];
                    n0 = ix.pt_off[rowbase + za + 1] - s0;
                    cells += n0 > 0;
                }
                if (zb >= 0 && zb < ext_last && zb != za) {
                    s1 = ix.pt_off[rowbase + zb];
                    n1 = ix.pt_off[rowbase + zb + 1] - s1;
                    cells += n1 > 0;
                }
            }
        }
        acc.cells += warp_sum(cells);
        consume<T, D, KS>(a, qd, d, s0, n0, s1, n1, tk, acc);
    }
    return l + 1;
}

// numpy pairwise summation over the k sorted targets held one per slot.
template <int KS>
__device__ __forceinline__ double slot_value(const double (&v)[KS], int t) {
    double r = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        double x = shfl_d(v[s], t & 31);
        if (s == (t >> 5)) r = x;
    }
    return r;
}

template <int KS>
__device__ double pairwise_slots(const double (&v)[KS], int a, int n) {
    if (n < 8) {
        double r = slot_value<KS>(v, a);
        for (int i = 1; i < n; ++i) r = __dadd_rn(r, slot_value<KS>(v, a + i));
        return r;
    }
    double acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = slot_value<KS>(v, a + t);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = __dadd_rn(acc[t], slot_value<KS>(v, a + i + t));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3])),
                           __dadd_rn(__dadd_rn(acc[4], acc[5]), __dadd_rn(acc[6], acc[7])));
    for (; i < n; ++i) res = __dadd_rn(res, slot_value<KS>(v, a + i));
    return res;
}

template <int KS>
__device__ double pairwise_mean(const double (&v)[KS], int k) {
    double s;
    if (k <= 128) {
        s = pairwise_slots<KS>(v, 0, k);
    } else {
        int n2 = k / 2;
        n2 -= n2 % 8;
        // both halves are <= 128 for k <= 256
        s = __dadd_rn(pairwise_slots<KS>(v, 0, n2), pairwise_slots<KS>(v, n2, k - n2));
    }
    return __ddiv_rn(s, (double)k);
}

template <typename T, int D, int KS>
__device__ __forceinline__ void query_one(const QArgs &a, int64_t w) {
    constexpr int DM = D > 0 ? D : GHN_MAX_DIM;
    const int lane = lane_id();
    const int64_t qi = a.qorder ? (int64_t)a.qorder[w] : w;
    const ghn_index_view &ix = a.ix;
    const int d = D > 0 ? D : ix.d;
    double qd[DM];
    int64_t r[DM];
    int64_t lmin = 0, lmax = 0;
#pragma unroll
    for (int j = 0; j < DM; ++j) {
        if (j >= d) break;
        qd[j] = a.q_dtype == GHN_F32 ? (double)((const float *)a.Q)[qi * d + j]
                                     : ((const double *)a.Q)[qi * d + j];
        const int64_t c = cell_id(qd[j], ix.widths[j], a.inv_w[j], (a.pow2 >> j) & 1u);
        r[j] = c - ix.lo[j];
        const int64_t e1 = ix.ext[j] - 1;
        const int64_t out = r[j] < 0 ? -r[j] : (r[j] > e1 ? r[j] - e1 : 0);
        lmin = out > lmin ? out : lmin;
        int64_t far = iabs64(r[j]);
        int64_t far2 = iabs64(e1 - r[j]);
        far = far2 > far ? far2 : far;
        lmax = far > lmax ? far : lmax;
    }
    const int k = a.k;
    TopK<KS> tk;
    tk.init();
    int64_t cells = 0, points = 0, layers = 0;
    int64_t l = lmin;
    if (a.mode == GHN_MODE_BRUTE) {
        // exact full scan (baselines.py:40-55): every slot, one flattened range
        LayerAcc acc{false, 0, 0};
        consume<T, D, KS>(a, qd, d, 0, lane == 0 ? (int32_t)ix.n : 0, 0, 0, tk, acc);
        cells = ix.n_cells;
        points = ix.n;
        l = lmax;
    }
    for (; a.mode != GHN_MODE_BRUTE;) {
        LayerAcc acc{false, 0, 0};
        const int64_t next = visit_layer<T, D, KS>(a, qd, r, d, l, tk, acc);
        cells += acc.cells;
        points += acc.points;
        layers = l;
        const bool full = tk.filled >= k;
        if (full) {
            if (a.mode == GHN_MODE_HEURISTIC && !acc.changed) break;
            if (a.mode == GHN_MODE_GUARANTEED) {
                if (bound_key(l, ix.min_width, ix.metric) > tk.thr_key) break;
            }
        }
        if (l >= lmax) break;
        if (next > l + 1) {
            // layers (l, next) hold no cell: only the stop rules can fire there
            if (full) {
                if (a.mode == GHN_MODE_HEURISTIC) {
                    layers = l + 1;
                    break;
                }
                if (!(tk.thr_key < INFINITY)) {   // no finite bound can exceed it
                    l = next;
                    continue;
                }
                // guaranteed: smallest l' in (l, next) with bound(l') > kth
                const double est =
                    floor((ix.metric == GHN_METRIC_EUCLIDEAN ? sqrt(tk.thr_key) : tk.thr_key) / ix.min_width) - 2.0;
                int64_t lp = l + 1;
                if (est > (double)lp && est < (double)next) lp = (int64_t)est;
                while (lp > l + 1) {
                    if (bound_key(lp - 1, ix.min_width, ix.metric) > tk.thr_key) --lp;
                    else break;
                }
                bool stop = false;
                for (; lp < next; ++lp) {
                    if (bound_key(lp, ix.min_width, ix.metric) > tk.thr_key) {
                        stop = true;
                        break;
                    }
                }
                if (stop) {
                    layers = lp;
                    break;
                }
            }
            l = next;
        } else {
            ++l;
        }
    }
    // ---------------------------------------------------------- epilogue
    const ghn_query_out &o = a.out;
    if (o.idx || o.dist) {
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int t = s * 32 + lane;
            if (t < k) {
                if (o.idx) o.idx[qi * k + t] = tk.idx[s];
                if (o.dist) o.dist[qi * k + t] = key_to_dist(tk.key[s], ix.metric);
            }
        }
    }
    if (o.stats && lane == 0) {
        o.stats[qi * 3 + 0] = layers;
        o.stats[qi * 3 + 1] = cells;
        o.stats[qi * 3 + 2] = points;
    }
    if (o.totals && lane == 0) {
        atomicAdd(&o.totals[0], (unsigned long long)layers);
        atomicAdd(&o.totals[1], (unsigned long long)cells);
        atomicAdd(&o.totals[2], (unsigned long long)points);
        atomicAdd(&o.totals[3], 1ull);
    }
    if (a.task == GHN_TASK_CLASSIFY && ix.labels) {
        int32_t lab[KS];
        int cnt[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int t = s * 32 + lane;
            lab[s] = t < k ? ix.labels[tk.idx[s]] : INT32_MIN;
            cnt[s] = 0;
        }
        if (KS == 1) {
            const unsigned valid = __ballot_sync(GHN_FULL, lane < k);
            if (lane < k) cnt[0] = __popc(__match_any_sync(valid, lab[0]));
        } else {
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                if (s * 32 >= k) break;
                for (int src = 0; src < 32; ++src) {
                    if (s * 32 + src >= k) break;
                    const int32_t lt = __shfl_sync(GHN_FULL, lab[s], src);
#pragma unroll
                    for (int s2 = 0; s2 < KS; ++s2) cnt[s2] += (lab[s2] == lt);
                }
            }
        }
        int top = 0;
#pragma unroll
        for (int s = 0; s < KS; ++s)
            if (s * 32 + lane < k) top = cnt[s] > top ? cnt[s] : top;
        top = warp_max(top);
        // nearest member of the tied labels by (sqrt(key), index)
        double bd = INFINITY;
        int32_t bi = 0x7fffffff, bl = 0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            if (s * 32 + lane < k && cnt[s] == top) {
                const double dd = key_to_dist(tk.key[s], ix.metric);
                if (pair_less(dd, tk.idx[s], bd, bi)) {
                    bd = dd;
                    bi = tk.idx[s];
                    bl = lab[s];
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double od = shfl_d(bd, lane ^ off);
            const int32_t oi = __shfl_sync(GHN_FULL, bi, lane ^ off);
            const int32_t ol = __shfl_sync(GHN_FULL, bl, lane ^ off);
            if (pair_less(od, oi, bd, bi)) {
                bd = od;
                bi = oi;
                bl = ol;
            }
        }
        if (lane == 0) {
            if (o.label) o.label[qi] = bl;
            if (o.confidence) o.confidence[qi] = __ddiv_rn((double)top, (double)k);
        }
    } else if (a.task == GHN_TASK_REGRESS_MEAN && ix.targets) {
        double v[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int t = s * 32 + lane;
            v[s] = t < k ? ix.targets[tk.idx[s]] : 0.0;
        }
        const double mean = pairwise_mean<KS>(v, k);
        if (lane == 0 && o.value) o.value[qi] = mean;
    } else if (a.task == GHN_TASK_REGRESS_MEDIAN && ix.targets) {
        // np.median (predict.py:46-47): the middle order statistic, or the
        // mean (a + b) / 2 of the two middle ones for even k
        double v[KS];
        int rank[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int t = s * 32 + lane;
            v[s] = t < k ? ix.targets[tk.idx[s]] : INFINITY;
            rank[s] = 0;
        }
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
            if (s2 * 32 >= k) break;
            for (int src = 0; src < 32; ++src) {
                const int t2 = s2 * 32 + src;
                if (t2 >= k) break;
                const double x = shfl_d(v[s2], src);
#pragma unroll
                for (int s = 0; s < KS; ++s) {
                    const int t = s * 32 + lane;
                    rank[s] += (x < v[s] || (x == v[s] && t2 < t)) ? 1 : 0;
                }
            }
        }
        const int r1 = (k - 1) / 2, r2 = k / 2;
        double m1 = 0.0, m2 = 0.0;
        bool h1 = false, h2 = false;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            if (s * 32 + lane < k) {
                if (rank[s] == r1) {
                    m1 = v[s];
                    h1 = true;
                }
                if (rank[s] == r2) {
                    m2 = v[s];
                    h2 = true;
                }
            }
        }
        const unsigned b1 = __ballot_sync(GHN_FULL, h1), b2 = __ballot_sync(GHN_FULL, h2);
        m1 = shfl_d(m1, __ffs(b1) - 1);
        m2 = shfl_d(m2, __ffs(b2) - 1);
        const double med = (k & 1) ? m1 : __ddiv_rn(__dadd_rn(m1, m2), 2.0);
        if (lane == 0 && o.value) o.value[qi] = med;
    }
}

template <typename T, int D, int KS>
__global__ void __launch_bounds__(Q_THREADS, KS <= 2 ? 5 : (KS == 4 ? 3 : 2)) query_kernel(const QArgs a) {
    const int64_t nqv = a.nq_dev ? (int64_t)*a.nq_dev : a.nq;
    for (int64_t w = (int64_t)blockIdx.x * Q_WARPS + (threadIdx.x >> 5); w < nqv;
         w += (int64_t)gridDim.x * Q_WARPS)
        query_one<T, D, KS>(a, w);
}

// ------------------------------------------------------------ query binning
struct BinConsts {
    double w[GHN_MAX_DIM], inv[GHN_MAX_DIM];
    int64_t lo[GHN_MAX_DIM], ext[GHN_MAX_DIM];
};

// The grid constants travel as a kernel parameter (512 B): no H2D copy, so
// binning never synchronises the stream with the host.
template <typename T>
__global__ void query_bin_key_kernel(const T *__restrict__ Q, int64_t nq, int d, const BinConsts bc,
                                     uint32_t pow2, int drop, uint32_t *keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = 0;
        for (int j = 0; j < d; ++j) {
            int64_t c = cell_id(to_double(Q[i * d + j]), bc.w[j], bc.inv[j], (pow2 >> j) & 1u) - bc.lo[j];
            c = c < 0 ? 0 : (c >= bc.ext[j] ? bc.ext[j] - 1 : c);
            key = key * (uint64_t)bc.ext[j] + (uint64_t)c;
        }
        keys[i] = (uint32_t)(key >> drop);
    }
}

static size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

static int bits_of(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

constexpr int64_t BIN_MIN_QUERIES = 2048;

template <typename T, int D>
int32_t launch_query_d(const QArgs &a, int ks, cudaStream_t s) {
    int64_t g = a.nq_dev ? (int64_t)sm_count() * 8 : (a.nq + Q_WARPS - 1) / Q_WARPS;
    if (g > 0x7fffffffLL) g = 0x7fffffffLL;
    const unsigned grid = (unsigned)g;
    switch (ks) {
        case 1: query_kernel<T, D, 1><<<grid, Q_THREADS, 0, s>>>(a); break;
        case 2: query_kernel<T, D, 2><<<grid, Q_THREADS, 0, s>>>(a); break;
        case 4: query_kernel<T, D, 4><<<grid, Q_THREADS, 0, s>>>(a); break;
        default: query_kernel<T, D, 8><<<grid, Q_THREADS, 0, s>>>(a); break;
    }
    GHN_LAUNCH_CHECK("query_kernel");
    return GHN_OK;
}

template <typename T>
int32_t launch_query(const QArgs &a, int ks, cudaStream_t s) {
    switch (a.ix.d) {
        case 1: return launch_query_d<T, 1>(a, ks, s);
        case 2: return launch_query_d<T, 2>(a, ks, s);
        case 3: return launch_query_d<T, 3>(a, ks, s);
        case 4: return launch_query_d<T, 4>(a, ks, s);
        case 5: return launch_query_d<T, 5>(a, ks, s);
        case 6: return launch_query_d<T, 6>(a, ks, s);
        default: return launch_query_d<T, 0>(a, ks, s);
    }
}

}  // namespace
}  // namespace ghn

using namespace ghn;

static size_t order_workspace_bytes(int64_t nq) {
    size_t q4 = a256((size_t)(nq > 0 ? nq : 1) * 4);
    return a256(sizeof(BinConsts)) + 5 * q4 + a256(radix_workspace_bytes(nq > 0 ? nq : 1)) + 256;
}

extern "C" size_t ghn_query_workspace_size(const ghn_index_view *ix, int64_t nq, int32_t k) {
    size_t b = order_workspace_bytes(nq);
    Tile2dPlan tp;
    if (tile2d_plan(ix, nq, k, GHN_TASK_CLASSIFY, false, &tp)) {
        size_t t = tile2d_workspace_bytes(&tp, nq);
        if (t > b) b = t;
    }
    return b;
}

static int32_t validate_query(const ghn_index_view *ix, int32_t k, int32_t mode) {
    if (mode != GHN_MODE_HEURISTIC && mode != GHN_MODE_GUARANTEED && mode != GHN_MODE_BRUTE) {
        set_error("unknown mode %d", mode);
        return GHN_ERR_VALUE;
    }
    if (k < 1 || k > ix->n) {
        set_error("k=%d out of range [1, %lld]", k, (long long)ix->n);
        return GHN_ERR_VALUE;
    }
    if (k > 256) {
        set_error("k=%d > 256 is not supported by the device top-k", k);
        return GHN_ERR_UNSUPPORTED;
    }
    if (ix->d < 1 || ix->d > GHN_MAX_DIM) {
        set_error("d=%d unsupported", ix->d);
        return GHN_ERR_UNSUPPORTED;
    }
    return GHN_OK;
}

static uint32_t pow2_mask(const ghn_index_view *ix, double *inv_w) {
    uint32_t m = 0;
    for (int j = 0; j < ix->d; ++j) {
        double inv = 0.0;
        if (is_pow2_width(ix->widths[j], &inv)) {
            m |= 1u << j;
            inv_w[j] = inv;
        }
    }
    return m;
}

extern "C" int32_t ghn_query_order(const ghn_index_view *ix, const void *Q, int32_t q_dtype,
                                   int64_t nq, int32_t *order_out, void *workspace,
                                   size_t workspace_bytes, void *stream) {
    if (ix->layout != GHN_LAYOUT_DENSE) {
        set_error("query binning needs the DENSE layout");
        return GHN_ERR_UNSUPPORTED;
    }
    if (nq <= 0) return GHN_OK;
    if (!workspace || workspace_bytes < order_workspace_bytes(nq)) {
        set_error("query workspace too small");
        return GHN_ERR_VALUE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    char *ws = (char *)workspace;
    BinConsts bc;
    memset(&bc, 0, sizeof(bc));
    const uint32_t pow2 = pow2_mask(ix, bc.inv);
    for (int j = 0; j < ix->d; ++j) {
        bc.w[j] = ix->widths[j];
        bc.lo[j] = ix->lo[j];
        bc.ext[j] = ix->ext[j];
    }
    const size_t q4 = a256((size_t)nq * 4);
    char *p = ws + a256(sizeof(BinConsts));
    uint32_t *kin = (uint32_t *)p;
    uint32_t *kout = (uint32_t *)(p + q4);
    uint32_t *ktmp = (uint32_t *)(p + 2 * q4);
    int32_t *vtmp = (int32_t *)(p + 3 * q4);
    char *rws = p + 5 * q4;
    const int kb = bits_of((uint64_t)(ix->E > 0 ? ix->E - 1 : 0));
    int keep = bits_of((uint64_t)nq) + 2;
    if (keep > 24) keep = 24;
    const int drop = kb > keep ? kb - keep : 0;
    unsigned g = (unsigned)((nq + 255) / 256);
    if (g > (unsigned)sm_count() * 16) g = (unsigned)sm_count() * 16;
    if (q_dtype == GHN_F32)
        query_bin_key_kernel<float><<<g, 256, 0, s>>>((const float *)Q, nq, ix->d, bc, pow2, drop, kin);
    else
        query_bin_key_kernel<double><<<g, 256, 0, s>>>((const double *)Q, nq, ix->d, bc, pow2, drop, kin);
    GHN_LAUNCH_CHECK("query_bin_key_kernel");
    return radix_sort_pairs(kin, nullptr, kout, order_out, ktmp, vtmp, nq, kb - drop, rws, s);
}

extern "C" int32_t ghn_query(const ghn_index_view *ix, const void *Q, int32_t q_dtype, int64_t nq,
                             int32_t k, int32_t mode, int32_t task, const int32_t *qorder,
                             const ghn_query_out *out, void *workspace, size_t workspace_bytes,
                             void *stream) {
    int32_t rc = validate_query(ix, k, mode);
    if (rc) return rc;
    if (nq <= 0) return GHN_OK;
    cudaStream_t s = (cudaStream_t)stream;
    QArgs a;
    memset(&a, 0, sizeof(a));
    a.ix = *ix;
    a.pow2 = pow2_mask(ix, a.inv_w);
    a.Q = Q;
    a.q_dtype = q_dtype;
    a.nq = nq;
    a.k = k;
    a.mode = mode;
    a.task = task;
    a.out = *out;
    a.qorder = qorder;
    a.nq_dev = nullptr;
    const int ks = k <= 32 ? 1 : (k <= 64 ? 2 : (k <= 128 ? 4 : 8));
    Tile2dPlan tp;
    const bool want_nb = out->dist != nullptr || out->idx != nullptr;
    if (mode != GHN_MODE_BRUTE && workspace && tile2d_plan(ix, nq, k, task, want_nb, &tp) &&
        workspace_bytes >= tile2d_workspace_bytes(&tp, nq)) {
        int32_t *fb_list = nullptr, *fb_count = nullptr;
        rc = tile2d_run(ix, &tp, Q, q_dtype, nq, k, mode, out, a.inv_w, a.pow2, workspace, &fb_list,
                        &fb_count, s);
        if (rc) return rc;
        a.qorder = fb_list;
        a.nq_dev = fb_count;
        if (ix->dtype == GHN_F32) return launch_query<float>(a, ks, s);
        return launch_query<double>(a, ks, s);
    }
    if (mode != GHN_MODE_BRUTE && !qorder && ix->layout == GHN_LAYOUT_DENSE && nq >= BIN_MIN_QUERIES &&
        workspace) {
        if (workspace_bytes < order_workspace_bytes(nq)) {
            set_error("query workspace too small");
            return GHN_ERR_VALUE;
        }
        int32_t *order = (int32_t *)((char *)workspace + a256(sizeof(BinConsts)) + 4 * a256((size_t)nq * 4));
        rc = ghn_query_order(ix, Q, q_dtype, nq, order, workspace, workspace_bytes, stream);
        if (rc) return rc;
        a.qorder = order;
    }
    if (ix->dtype == GHN_F32) return launch_query<float>(a, ks, s);
    return launch_query<double>(a, ks, s);
}

namespace ghn {
__global__ void gather_i32_kernel(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}
}  // namespace ghn

extern "C" int32_t ghn_gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst,
                                  void *stream) {
    if (n <= 0) return GHN_OK;
    unsigned g = (unsigned)((n + 255) / 256);
    if (g > (unsigned)sm_count() * 16) g = (unsigned)sm_count() * 16;
    gather_i32_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(src, idx, n, dst);
    GHN_LAUNCH_CHECK("gather_i32_kernel");
    return GHN_OK;
}
