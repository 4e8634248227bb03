// ghn_query_impl.cuh -- the generic batched GHN predict kernel (device code).
//
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
#pragma once

#include <math.h>

#include "ghn_query.cuh"

namespace ghn {
namespace {


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
    long long nkeys;     // candidate keys evaluated (work counter, totals[4])

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            key[s] = INFINITY;
            idx[s] = 0x7fffffff;
        }
        filled = 0;
        thr_key = INFINITY;
        thr_idx = 0x7fffffff;
        nkeys = 0;
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

// Where candidates come from: the main CSR (SoA stride n, slot -> index via
// perm) or the points of the nested sub-grids (stride n_subpts, sub_idx).
template <typename T>
struct Src {
    const T *coords;
    int64_t stride;
    const int32_t *idx;
};

// Consume up to two slot ranges per lane: compute keys for every candidate,
// filter against the k-th entry, insert survivors in lane order.
template <typename T, int D, int KS>
__device__ __forceinline__ void consume(const QArgs &a, const Src<T> &src, const double *qd, int d, int32_t s0,
                                        int32_t n0, int32_t s1, int32_t n1, TopK<KS> &tk, bool &changed) {
    const int lane = lane_id();
    const int cnt = n0 + n1;
    const int incl = warp_inclusive_scan(cnt);
    const int total = __shfl_sync(GHN_FULL, incl, 31);
    if (total == 0) return;
    tk.nkeys += total;
    const int excl = incl - cnt;
    const T *__restrict__ coords = src.coords;
    const int64_t n = src.stride;
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
        if (pass) pidx = src.idx[slot];
        unsigned sm = __ballot_sync(GHN_FULL, pass);
        while (sm) {
            const int src_l = __ffs(sm) - 1;
            sm &= sm - 1;
            const double ck = shfl_d(key, src_l);
            const int32_t ci = __shfl_sync(GHN_FULL, pidx, src_l);
            if (tk.filled >= k && !pair_less(ck, ci, tk.thr_key, tk.thr_idx)) continue;
            tk.insert(ck, ci, k);
            changed = true;
        }
    }
}

__device__ __forceinline__ int64_t iabs64(int64_t v) { return v < 0 ? -v : v; }

// ------------------------------------------------------------------ bounds
// Lower bounds on the ordering key of every point of a set of cells, used to
// skip candidates that provably cannot enter the top-k (key > k-th key; the
// (key, index) order lets a candidate with key == k-th key in, so equality
// never prunes).  A box [blo, bhi] per dimension contains every point of the
// cells; the per-dimension gap fl(blo - q) / fl(q - bhi) is <= |fl(x - q)| for
// every x in the box (IEEE rounding is monotone and odd), and the metric keys
// (core.py:72-86) are monotone in each |diff|, so key(gaps) <= key(x).
//
// Coarse cell ids come from floor(fl(x / w)), so a point lies in [i w, (i+1) w)
// up to rounding; the box is widened by 2^-40 relative to absorb it.
__device__ __forceinline__ double widen_lo(double a, double w) { return a - (fabs(a) + w) * 0x1p-40; }
__device__ __forceinline__ double widen_hi(double b, double w) { return b + (fabs(b) + w) * 0x1p-40; }

__device__ __forceinline__ double gap_of(double q, double blo, double bhi) {
    return q < blo ? __dsub_rn(blo, q) : (q > bhi ? __dsub_rn(q, bhi) : 0.0);
}

// Gap of q to the (relative) coarse cell ids [i0, i1] of dimension j.
__device__ __forceinline__ double cell_gap(const ghn_index_view &ix, int j, double q, int64_t i0, int64_t i1) {
    const double w = ix.widths[j];
    return gap_of(q, widen_lo(__dmul_rn((double)(ix.lo[j] + i0), w), w),
                  widen_hi(__dmul_rn((double)(ix.lo[j] + i1 + 1), w), w));
}

// Gap of q to sub-cells [t0, t1] of dimension j of a sub-grid.
__device__ __forceinline__ double sub_gap(const ghn_subgrid &g, int j, double q, int64_t t0, int64_t t1) {
    const double o = g.origin[j], h = g.h[j];
    return gap_of(q, widen_lo(o + (double)t0 * h, h), widen_hi(o + (double)(t1 + 1) * h, h));
}

template <int D>
__device__ __forceinline__ double gap_key(const double *gap, int d, int metric) {
    if (D > 0) {
        constexpr int DC = DimOf<D>::v;
        double g[DC];
#pragma unroll
        for (int j = 0; j < DC; ++j) g[j] = gap[j];
        return metric_key<DC>(g, metric);
    }
    return metric_key_rt(gap, d, metric);
}

// Key lower bound of a single-dimension escape distance (a point outside a
// block differs from q by at least `gap` in some dimension).
__device__ __forceinline__ double escape_key(double gap, int metric) {
    if (!(gap > 0.0)) return 0.0;
    return metric == GHN_METRIC_EUCLIDEAN ? __dmul_rn(gap, gap) : gap;
}

// ------------------------------------------------------------ sub-grid walk
// Nearest members of one overfull cell (its nested grid, ghn_subgrid.cu):
// rings of sub-cells around the query's (clamped) sub-cell, each sub-cell
// skipped when its lower bound exceeds the k-th key, the walk ended when the
// block walked so far provably encloses every point that could still enter.
// Every member that can enter the top-k is evaluated, so the top-k after the
// walk equals the top-k after scanning the whole cell (explore.py:110-118).
template <typename T, int D, int KS>
__device__ __forceinline__ void sub_walk(const QArgs &a, const double *qd, int d, int32_t gid, TopK<KS> &tk, bool &changed) {
    constexpr int DM = D > 0 ? D : GHN_MAX_DIM;
    const int lane = lane_id();
    const ghn_subgrid &g = a.ix.subs[gid];
    const int metric = a.ix.metric;
    const int k = a.k;
    const Src<T> src{(const T *)a.ix.sub_coords, a.ix.n_subpts, a.ix.sub_idx};
    int32_t c[DM], ext[DM];
    int64_t rmax = 0;
#pragma unroll
    for (int j = 0; j < DM; ++j) {
        if (j >= d) break;
        ext[j] = g.ext[j];
        double t = floor(__dmul_rn(__dsub_rn(qd[j], g.origin[j]), g.inv_h[j]));
        t = fmin(fmax(t, 0.0), (double)(ext[j] - 1));
        c[j] = (int32_t)t;
        const int64_t far = max(c[j], ext[j] - 1 - c[j]);
        rmax = far > rmax ? far : rmax;
    }
    const int jl = d - 1;
    for (int64_t r = 0; r <= rmax; ++r) {
        if (r > 0 && tk.filled >= k) {
            // every unvisited sub-cell lies outside block(r-1) in some dimension
            double esc = INFINITY;
            _Pragma("unroll") for (int j = 0; j < DM; ++j) {
                if (j >= d) break;
                if (c[j] - (r - 1) > 0) {
                    const double face = widen_hi(g.origin[j] + (double)(c[j] - r + 1) * g.h[j], g.h[j]);
                    esc = fmin(esc, __dsub_rn(qd[j], face));
                }
                if (c[j] + (r - 1) < ext[j] - 1) {
                    const double face = widen_lo(g.origin[j] + (double)(c[j] + r) * g.h[j], g.h[j]);
                    esc = fmin(esc, __dsub_rn(face, qd[j]));
                }
            }
            if (esc == INFINITY || escape_key(esc, metric) > tk.thr_key) break;
        }
        int32_t lo_c[DM], hi_c[DM];
        int64_t rows = 1;
        _Pragma("unroll") for (int j = 0; j < DM; ++j) {
                if (j >= d) break;
            lo_c[j] = (int32_t)max((int64_t)0, (int64_t)c[j] - r);
            hi_c[j] = (int32_t)min((int64_t)ext[j] - 1, (int64_t)c[j] + r);
            if (j < jl) rows *= hi_c[j] - lo_c[j] + 1;
        }
        for (int64_t rb = 0; rb < rows; rb += 32) {
            const int64_t t = rb + lane;
            int32_t s0 = 0, n0 = 0, s1 = 0, n1 = 0;
            if (t < rows) {
                double gap[DM];
                uint32_t rem = (uint32_t)t;
                int64_t cheb = 0, rowlin = 0, mul = 1;
                _Pragma("unroll") for (int j = DM - 2; j >= 0; --j) {
                    if (j >= jl) continue;
                    const uint32_t len = (uint32_t)(hi_c[j] - lo_c[j] + 1);
                    const uint32_t q = rem / len;
                    const int64_t rj = lo_c[j] + (int64_t)(rem - q * len);
                    rem = q;
                    cheb = max(cheb, iabs64(rj - c[j]));
                    rowlin += rj * mul;
                    mul *= ext[j];
                    gap[j] = sub_gap(g, j, qd[j], rj, rj);
                }
                const int64_t base = g.off + rowlin * ext[jl];
                const bool full = tk.filled >= k;
                if (cheb == r) {
                    const int64_t z0 = lo_c[jl], z1 = hi_c[jl];
                    gap[jl] = sub_gap(g, jl, qd[jl], z0, z1);
                    if (!full || gap_key<D>(gap, d, metric) <= tk.thr_key) {
                        s0 = a.ix.sub_off[base + z0];
                        n0 = a.ix.sub_off[base + z1 + 1] - s0;
                    }
                } else {
                    const int64_t za = (int64_t)c[jl] - r, zb = (int64_t)c[jl] + r;
                    if (za >= 0) {
                        gap[jl] = sub_gap(g, jl, qd[jl], za, za);
                        if (!full || gap_key<D>(gap, d, metric) <= tk.thr_key) {
                            s0 = a.ix.sub_off[base + za];
                            n0 = a.ix.sub_off[base + za + 1] - s0;
                        }
                    }
                    if (zb < ext[jl] && zb != za) {
                        gap[jl] = sub_gap(g, jl, qd[jl], zb, zb);
                        if (!full || gap_key<D>(gap, d, metric) <= tk.thr_key) {
                            s1 = a.ix.sub_off[base + zb];
                            n1 = a.ix.sub_off[base + zb + 1] - s1;
                        }
                    }
                }
            }
            consume<T, D, KS>(a, src, qd, d, s0, n0, s1, n1, tk, changed);
        }
    }
}

// Overfull cells (sub-grids) are walked one at a time by the whole warp.
template <typename T, int D, int KS>
__device__ __forceinline__ void drain_fat(const QArgs &a, const double *qd, int d, bool &fat, int32_t fat_gid,
                                          TopK<KS> &tk, bool &changed) {
    unsigned m = __ballot_sync(GHN_FULL, fat);
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int32_t gid = __shfl_sync(GHN_FULL, fat_gid, src);
        sub_walk<T, D, KS>(a, qd, d, gid, tk, changed);
    }
    fat = false;
}

// Visit the non-empty cells at Chebyshev distance exactly l.  Returns the
// next non-empty layer when it is known (cell-list scan), else l + 1.  SUB:
// the index has nested grids (overfull cells are walked by sub-cell rings);
// the other instantiation carries none of that code.
template <typename T, int D, int KS, bool SUB>
__device__ __forceinline__ int64_t visit_layer(const QArgs &a, const double *qd, const int64_t *r, int d, int64_t l,
                                               bool want_stats, TopK<KS> &tk, LayerAcc &acc) {
    constexpr int DM = D > 0 ? D : GHN_MAX_DIM;
    const int lane = lane_id();
    const ghn_index_view &ix = a.ix;
    const int metric = ix.metric;
    const int k = a.k;
    const Src<T> main_src{(const T *)ix.coords, ix.n, ix.perm};
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
    if (!want_stats && l >= 1 && tk.filled >= k) {
        // whole-shell test: every cell of the shell lies outside block(l-1)
        // in some dimension; if that escape distance already exceeds the
        // k-th key, no point of the shell can enter (changed stays false)
        double esc = INFINITY;
        _Pragma("unroll") for (int j = 0; j < DM; ++j) {
                if (j >= d) break;
            const double w = ix.widths[j];
            if (r[j] - (l - 1) > 0)
                esc = fmin(esc, __dsub_rn(qd[j], widen_hi(__dmul_rn((double)(ix.lo[j] + r[j] - l + 1), w), w)));
            if (r[j] + (l - 1) < ix.ext[j] - 1)
                esc = fmin(esc, __dsub_rn(widen_lo(__dmul_rn((double)(ix.lo[j] + r[j] + l), w), w), qd[j]));
        }
        if (esc != INFINITY && escape_key(esc, metric) > tk.thr_key) return l + 1;
    }
    constexpr bool subs = SUB;
    if (ix.layout == GHN_LAYOUT_LIST || rows > (double)ix.n_cells) {
        // cell-list scan (explore.py:105), also finds the next non-empty layer
        int64_t next = INT64_MAX;
        for (int cb = 0; cb < ix.n_cells; cb += 32) {
            const int c = cb + lane;
            bool match = false, fat = false;
            int32_t st = 0, cntp = 0, gid = -1;
            if (c < ix.n_cells) {
                int64_t ch = 0;
                _Pragma("unroll") for (int j = 0; j < DM; ++j) {
                if (j >= d) break;
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
            acc.points += warp_sum(cntp);
            if (match && tk.filled >= k) {
                double gap[DM];
                _Pragma("unroll") for (int j = 0; j < DM; ++j) {
                if (j >= d) break;
                    const int64_t id = ix.cell_ids[(int64_t)c * d + j];
                    gap[j] = cell_gap(ix, j, qd[j], id, id);
                }
                if (gap_key<D>(gap, d, metric) > tk.thr_key) cntp = 0;
            }
            if (SUB && cntp > ix.sub_min) {
                gid = ix.sub_of_cell[c];
                if (gid >= 0) {
                    fat = true;
                    cntp = 0;
                }
            }
            if (__any_sync(GHN_FULL, cntp > 0)) consume<T, D, KS>(a, main_src, qd, d, st, cntp, 0, 0, tk, acc.changed);
            if (SUB) drain_fat<T, D, KS>(a, qd, d, fat, gid, tk, acc.changed);
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
        int32_t rid[DM];
        int64_t rowbase = 0;
        // intervals of the last dimension this lane covers: [x0, x1] and [y0, y1]
        int64_t x0 = 1, x1 = 0, y0 = 1, y1 = 0;
        bool heavy = false;
        if (t < R) {
            // decode: last row dim fastest; rowlin is row-major over ext[0..d-2].
            // DENSE: E <= 2^30, so rows, ids and the linear cell index fit 32 bits.
            uint32_t rem = (uint32_t)t;
            int64_t cheb = 0;
            uint32_t rowlin = 0, mul = 1;
            _Pragma("unroll") for (int j = DM - 2; j >= 0; --j) {
                    if (j >= jl) continue;
                const uint32_t len = (uint32_t)(hi_c[j] - lo_c[j] + 1);
                uint32_t q = rem, rj = (uint32_t)lo_c[j];
                if (len != 1) {
                    q = rem / len;
                    rj += rem - q * len;
                }
                rem = q;
                rid[j] = (int32_t)rj;
                const int64_t v = iabs64((int64_t)rj - r[j]);
                cheb = v > cheb ? v : cheb;
                rowlin += rj * mul;
                mul *= (uint32_t)ix.ext[j];
            }
            rowbase = (int64_t)rowlin * ext_last;
            if (cheb == l) {
                x0 = lo_c[jl];
                x1 = hi_c[jl];
                s0 = ix.pt_off[rowbase + x0];
                n0 = ix.pt_off[rowbase + x1 + 1] - s0;
                cells += ix.ne_off[rowbase + x1 + 1] - ix.ne_off[rowbase + x0];
            } else {
                const int64_t za = r[jl] - l, zb = r[jl] + l;
                if (za >= 0 && za < ext_last) {
                    s0 = ix.pt_off[rowbase + za];
                    n0 = ix.pt_off[rowbase + za + 1] - s0;
                    cells += n0 > 0;
                    if (n0 > 0) x0 = x1 = za;
                }
                if (zb >= 0 && zb < ext_last && zb != za) {
                    s1 = ix.pt_off[rowbase + zb];
                    n1 = ix.pt_off[rowbase + zb + 1] - s1;
                    cells += n1 > 0;
                    if (n1 > 0) y0 = y1 = zb;
                }
            }
        }
        acc.cells += warp_sum(cells);
        acc.points += warp_sum(n0 + n1);
        if (t < R && tk.filled >= k && n0 + n1 > 0) {
            // whole-row / per-end-cell lower bounds against the k-th key
            double gap[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j)
                if (j < jl) gap[j] = cell_gap(ix, j, qd[j], rid[j], rid[j]);
            if (x0 <= x1) {
                gap[jl] = cell_gap(ix, jl, qd[jl], x0, x1);
                if (gap_key<D>(gap, d, metric) > tk.thr_key) {
                    n0 = 0;
                    x0 = 1, x1 = 0;
                }
            }
            if (y0 <= y1) {
                gap[jl] = cell_gap(ix, jl, qd[jl], y0, y1);
                if (gap_key<D>(gap, d, metric) > tk.thr_key) {
                    n1 = 0;
                    y0 = 1, y1 = 0;
                }
            }
        }
        if (SUB && n0 + n1 > ix.sub_min) {   // may hold an overfull cell: cell by cell below
            heavy = true;
            n0 = n1 = 0;
        }
        if (__any_sync(GHN_FULL, n0 + n1 > 0)) consume<T, D, KS>(a, main_src, qd, d, s0, n0, s1, n1, tk, acc.changed);
        if (!SUB) continue;
        unsigned hm = __ballot_sync(GHN_FULL, heavy);
        while (hm) {
            const int src = __ffs(hm) - 1;
            hm &= hm - 1;
            int32_t brid[DM];
            _Pragma("unroll") for (int j = 0; j < DM; ++j) if (j < jl) brid[j] = __shfl_sync(GHN_FULL, rid[j], src);
            const int64_t bbase = __shfl_sync(GHN_FULL, rowbase, src);
            const int64_t iv[4] = {__shfl_sync(GHN_FULL, x0, src), __shfl_sync(GHN_FULL, x1, src),
                                   __shfl_sync(GHN_FULL, y0, src), __shfl_sync(GHN_FULL, y1, src)};
            _Pragma("unroll") for (int h = 0; h < 2; ++h) {
                for (int64_t zb = iv[2 * h]; zb <= iv[2 * h + 1]; zb += 32) {
                    const int64_t z = zb + lane;
                    int32_t st = 0, cnt = 0, gid = -1;
                    bool fat = false;
                    if (z <= iv[2 * h + 1]) {
                        st = ix.pt_off[bbase + z];
                        cnt = ix.pt_off[bbase + z + 1] - st;
                        if (cnt > 0 && tk.filled >= k) {
                            double gap[DM];
                            _Pragma("unroll") for (int j = 0; j < DM; ++j) if (j < jl) gap[j] = cell_gap(ix, j, qd[j], brid[j], brid[j]);
                            gap[jl] = cell_gap(ix, jl, qd[jl], z, z);
                            if (gap_key<D>(gap, d, metric) > tk.thr_key) cnt = 0;
                        }
                        if (cnt > ix.sub_min) {
                            gid = ix.sub_of_cell[ix.ne_off[bbase + z]];
                            if (gid >= 0) {
                                fat = true;
                                cnt = 0;
                            }
                        }
                    }
                    if (__any_sync(GHN_FULL, cnt > 0)) consume<T, D, KS>(a, main_src, qd, d, st, cnt, 0, 0, tk, acc.changed);
                    drain_fat<T, D, KS>(a, qd, d, fat, gid, tk, acc.changed);
                }
            }
        }
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

template <typename T, int D, int KS, bool SUB>
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
    const bool want_stats = a.out.stats != nullptr || a.out.totals != nullptr;
    TopK<KS> tk;
    tk.init();
    int64_t cells = 0, points = 0, layers = 0;
    int64_t l = lmin;
    if (a.mode == GHN_MODE_BRUTE) {
        // exact full scan (baselines.py:40-55): every slot, one flattened range
        bool ch = false;
        const Src<T> main_src{(const T *)ix.coords, ix.n, ix.perm};
        consume<T, D, KS>(a, main_src, qd, d, 0, lane == 0 ? (int32_t)ix.n : 0, 0, 0, tk, ch);
        cells = ix.n_cells;
        points = ix.n;
        l = lmax;
    }
    for (; a.mode != GHN_MODE_BRUTE;) {
        LayerAcc acc{false, 0, 0};
        const int64_t next = visit_layer<T, D, KS, SUB>(a, qd, r, d, l, want_stats, tk, acc);
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
        atomicAdd(&o.totals[4], (unsigned long long)tk.nkeys);
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

template <typename T, int D, int KS, bool SUB>
__global__ void __launch_bounds__(Q_THREADS, KS <= 2 ? 4 : (KS == 4 ? 3 : 2)) query_kernel(const QArgs a) {
    const int64_t nqv = a.nq_dev ? (int64_t)*a.nq_dev : a.nq;
    if (a.nq_dev) {
        // the tiled path's fallback list: a few thousand queries of very
        // different cost -- warps draw them from a cursor (nq_dev[1], zeroed
        // with the count) instead of striding
        int32_t *cursor = const_cast<int32_t *>(a.nq_dev) + 1;
        for (;;) {
            int32_t w = 0;
            if ((threadIdx.x & 31) == 0) w = atomicAdd(cursor, 1);
            w = __shfl_sync(GHN_FULL, w, 0);
            if (w >= nqv) break;
            query_one<T, D, KS, SUB>(a, w);
        }
        return;
    }
    for (int64_t w = (int64_t)blockIdx.x * Q_WARPS + (threadIdx.x >> 5); w < nqv;
         w += (int64_t)gridDim.x * Q_WARPS)
        query_one<T, D, KS, SUB>(a, w);
}

// ------------------------------------------------------------ launch
// One (T, D, KS, SUB) instantiation (the nested-grid runtime-d kernels compile
// for minutes each: one translation unit per KS).
template <typename T, int D, int KS, bool SUB>
int32_t launch_query_one(const QArgs &a, cudaStream_t s) {
    int64_t g = a.nq_dev ? (int64_t)sm_count() * 4 : (a.nq + Q_WARPS - 1) / Q_WARPS;
    if (g > 0x7fffffffLL) g = 0x7fffffffLL;
    query_kernel<T, D, KS, SUB><<<(unsigned)g, Q_THREADS, 0, s>>>(a);
    GHN_LAUNCH_CHECK("query_kernel");
    return GHN_OK;
}

template <typename T, int D, bool SUB>
int32_t launch_query_d(const QArgs &a, int ks, cudaStream_t s) {
    int64_t g = a.nq_dev ? (int64_t)sm_count() * 4 : (a.nq + Q_WARPS - 1) / Q_WARPS;
    if (g > 0x7fffffffLL) g = 0x7fffffffLL;
    const unsigned grid = (unsigned)g;
    switch (ks) {
        case 1: query_kernel<T, D, 1, SUB><<<grid, Q_THREADS, 0, s>>>(a); break;
        case 2: query_kernel<T, D, 2, SUB><<<grid, Q_THREADS, 0, s>>>(a); break;
        case 4: query_kernel<T, D, 4, SUB><<<grid, Q_THREADS, 0, s>>>(a); break;
        default:
            // k > 128: runtime-d only
            query_kernel<T, 0, 8, SUB><<<grid, Q_THREADS, 0, s>>>(a);
            break;
    }
    GHN_LAUNCH_CHECK("query_kernel");
    return GHN_OK;
}

}  // namespace
}  // namespace ghn
