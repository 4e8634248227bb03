// ghn_tile2d_grp.cuh -- sub-warp variant of the tiled 2-D predict: G lanes
// (G = 8 or 16) answer one query, so 32/G queries share every warp
// instruction.  Same semantics and shortcuts as the warp-per-query code in
// ghn_tile2d.cu (k = 1 running minimum, T_0 skip, shell pruning, exact radix
// select fused with the vote); this file is included by ghn_tile2d.cu after
// the shared helpers (T2Args, Win, Kth, key2, lt_pair, push_fallback,
// shell_cannot_change) are defined.
//
// Groups of a warp may diverge (different queries take different paths), so
// every warp primitive is issued with the group's own lane mask and
// width G.  Candidates are walked range by range (a CSR row segment or the
// two side cells of a shell row), G points per iteration -- no owner search.
#pragma once

namespace ghn {
namespace {

template <int G>
struct Grp {
    int lane;        // 0..G-1
    int base;        // first warp lane of the group
    unsigned mask;   // the group's lanes (absolute)

    __device__ __forceinline__ Grp() {
        const int wl = threadIdx.x & 31;
        lane = wl & (G - 1);
        base = wl & ~(G - 1);
        mask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << base);
    }
    template <typename T>
    __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(mask, v, src, G); }
    template <typename T>
    __device__ __forceinline__ T shfl_xor(T v, int m) const { return __shfl_xor_sync(mask, v, m, G); }
    __device__ __forceinline__ unsigned ballot(bool p) const {
        return (__ballot_sync(mask, p) >> base) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
    }
    __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask, p); }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    __device__ __forceinline__ unsigned lt() const { return (1u << lane) - 1u; }
    __device__ __forceinline__ int sum(int v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v += shfl_xor(v, o);
        return v;
    }
    __device__ __forceinline__ int max(int v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v = ::max(v, shfl_xor(v, o));
        return v;
    }
    __device__ __forceinline__ int incl_scan(int v) const {
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            const int u = __shfl_up_sync(mask, v, o, G);
            if (lane >= o) v += u;
        }
        return v;
    }
};

constexpr int GB_CAP = 16;   // boundary candidates ranked exactly per group

struct GrpScratch {
    int hist[32];
    int lcnt[32];
    double bkey[GB_CAP];
    int32_t bidx[GB_CAP];
    int32_t bg[GB_CAP];
};

// Iterate the points of block(L): rows lr-L..lr+L, columns lc-L..lc+L.
// BODY sees p (staged index), row (window row), valid.
#define GRP_FOR_BLOCK(w, gr, lr, lc, L_, ...)                                              \
    do {                                                                                   \
        const int l_ = (L_);                                                               \
        const int ca_ = max((lc) - l_, 0), cb_ = min((lc) + l_, (w).W - 1) + 1;            \
        const int i0_ = max((lr) - l_, 0), i1_ = min((lr) + l_, (w).R - 1);                \
        for (int row = i0_; row <= i1_; ++row) {                                           \
            const int32_t *rp_ = (w).loc + row * (w).W1;                                   \
            const int s_ = rp_[ca_], e_ = rp_[cb_];                                        \
            for (int b_ = s_; b_ < e_; b_ += GS) {                                         \
                const int p = b_ + (gr).lane;                                              \
                const bool valid = p < e_;                                                 \
                __VA_ARGS__;                                                               \
            }                                                                              \
        }                                                                                  \
    } while (0)

// Iterate the points of shell(L), L >= 1 (full rows lr -+ L, side cells of
// the rows between, both side cells of a row in one range).
#define GRP_FOR_SHELL(w, gr, lr, lc, L_, ...)                                              \
    do {                                                                                   \
        const int l_ = (L_);                                                               \
        const int i0_ = max((lr) - l_, 0), i1_ = min((lr) + l_, (w).R - 1);                \
        for (int row = i0_; row <= i1_; ++row) {                                           \
            const int32_t *rp_ = (w).loc + row * (w).W1;                                   \
            int sa_, na_, sb_ = 0, nb_ = 0;                                                \
            if (row == (lr) - l_ || row == (lr) + l_) {                                    \
                sa_ = rp_[max((lc) - l_, 0)];                                              \
                na_ = rp_[min((lc) + l_, (w).W - 1) + 1] - sa_;                            \
            } else {                                                                       \
                sa_ = 0;                                                                   \
                na_ = 0;                                                                   \
                if ((lc) - l_ >= 0) {                                                      \
                    sa_ = rp_[(lc) - l_];                                                  \
                    na_ = rp_[(lc) - l_ + 1] - sa_;                                        \
                }                                                                          \
                if ((lc) + l_ < (w).W) {                                                   \
                    sb_ = rp_[(lc) + l_];                                                  \
                    nb_ = rp_[(lc) + l_ + 1] - sb_;                                        \
                }                                                                          \
            }                                                                              \
            for (int b_ = 0; b_ < na_ + nb_; b_ += GS) {                                   \
                const int m_ = b_ + (gr).lane;                                             \
                const int p = m_ < na_ ? sa_ + m_ : sb_ + (m_ - na_);                      \
                const bool valid = m_ < na_ + nb_;                                         \
                __VA_ARGS__;                                                               \
            }                                                                              \
        }                                                                                  \
    } while (0)

// Find the bucket holding rank r in a 32-bucket group histogram: returns the
// bucket (or -1), its count m, and the rank inside it (r - count below).
template <int G>
__device__ __forceinline__ int find_bucket(const Grp<G> &gr, const int *hist, int &r, int &m) {
    constexpr int PER = 32 / G;
    int c[PER], s = 0;
#pragma unroll
    for (int t = 0; t < PER; ++t) {
        c[t] = hist[gr.lane * PER + t];
        s += c[t];
    }
    const int incl = gr.incl_scan(s);
    const unsigned ge = gr.ballot(incl >= r);
    if (!ge) return -1;
    const int owner = __ffs(ge) - 1;
    int below = gr.shfl(incl - s, owner);
    int bucket = -1, cnt = 0, rr = r - below;
    if (gr.lane == owner) {
        int acc = 0;
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            if (bucket < 0) {
                if (acc + c[t] >= rr) {
                    bucket = gr.lane * PER + t;
                    cnt = c[t];
                    rr -= acc;
                } else {
                    acc += c[t];
                }
            }
        }
    }
    bucket = gr.shfl(bucket, owner);
    m = gr.shfl(cnt, owner);
    r = gr.shfl(rr, owner);
    return bucket;
}

// Radix select over block(L) with key in [lo, hi] (see select_vote_c), group
// edition; labels must be small codes (vote by shared counters).  og0/og1:
// report through *outside whether a member's global slot lies outside
// [og0, og1).  The vote ends in sc.lcnt.
template <int G>
__device__ __forceinline__ bool select_grp(const T2Args &a, const Win &w, GrpScratch &sc, const Grp<G> &gr,
                                           int lr, int lc, int L, double q0, double q1, int r, double lo,
                                           double hi, Kth &out, int32_t og0, int32_t og1,
                                           bool *outside) {
    constexpr int GS = G;
    const float flo = __double2float_rd(lo);
    const float fhi = __double2float_ru(hi);
    const float sc1 = fhi > flo ? fminf(32.0f * __frcp_rn(fhi - flo), 1e30f) : 0.0f;
#define GRP_B1(k32) min((int)(((k32) - flo) * sc1), 31)
#pragma unroll
    for (int t = 0; t < 32 / G; ++t) {
        sc.hist[gr.lane * (32 / G) + t] = 0;
        sc.lcnt[gr.lane * (32 / G) + t] = 0;
    }
    gr.sync();
    GRP_FOR_BLOCK(w, gr, lr, lc, L, {
        double key = 0.0;
        if (valid) key = key2(w, p, q0, q1);
        const bool in = valid && key >= lo && key <= hi;
        const int b = in ? GRP_B1(__double2float_rd(key)) : -1;
        const unsigned im = __ballot_sync(gr.mask, in);
        if (in) {
            const unsigned grp = __match_any_sync(im, b);
            if ((grp & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&sc.hist[b], __popc(grp));
        }
    });
    gr.sync();
    int m = 0;
    const int bs1 = find_bucket<G>(gr, sc.hist, r, m);
    if (bs1 < 0) return false;
    int bs2 = -1;
    float lo2 = 0.0f, sc2 = 0.0f;
    if (m > GB_CAP) {
        lo2 = flo + (float)bs1 / sc1;
        sc2 = fminf(sc1 * 32.0f, 1e30f);
#define GRP_B2(k32) max(0, min((int)(((k32) - lo2) * sc2), 31))
        gr.sync();
#pragma unroll
        for (int t = 0; t < 32 / G; ++t) sc.hist[gr.lane * (32 / G) + t] = 0;
        gr.sync();
        GRP_FOR_BLOCK(w, gr, lr, lc, L, {
            double key = 0.0;
            if (valid) key = key2(w, p, q0, q1);
            bool in = valid && key >= lo && key <= hi;
            int b = -1;
            if (in) {
                const float k32 = __double2float_rd(key);
                in = GRP_B1(k32) == bs1;
                b = GRP_B2(k32);
            }
            const unsigned im = __ballot_sync(gr.mask, in);
            if (in) {
                const unsigned grp = __match_any_sync(im, b);
                if ((grp & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&sc.hist[b], __popc(grp));
            }
        });
        gr.sync();
        bs2 = find_bucket<G>(gr, sc.hist, r, m);
        if (bs2 < 0 || m > GB_CAP) return false;
    }
    int nb = 0;
    bool outs = false;
    GRP_FOR_BLOCK(w, gr, lr, lc, L, {
        double key = 0.0;
        int side = 1;
        if (valid) {
            key = key2(w, p, q0, q1);
            if (key >= lo && key <= hi) {
                const float k32 = __double2float_rd(key);
                const int b1 = GRP_B1(k32);
                side = b1 < bs1 ? -1 : (b1 > bs1 ? 1 : 0);
                if (side == 0 && bs2 >= 0) {
                    const int b2 = GRP_B2(k32);
                    side = b2 < bs2 ? -1 : (b2 > bs2 ? 1 : 0);
                }
            }
        }
        const int32_t g = p + w.delta[row];
        const unsigned mem = __ballot_sync(gr.mask, side < 0);
        if (side < 0) {
            const int32_t Lb = a.labels_perm[g];
            const unsigned grp = __match_any_sync(mem, Lb);
            if ((grp & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&sc.lcnt[Lb], __popc(grp));
            outs |= g < og0 || g >= og1;
        }
        const unsigned bnd = gr.ballot(side == 0);
        if (side == 0) {
            const int pos = nb + __popc(bnd & gr.lt());
            sc.bkey[pos] = key;
            sc.bidx[pos] = a.perm[g];
            sc.bg[pos] = g;
        }
        nb += __popc(bnd);
    });
#undef GRP_B1
#undef GRP_B2
    gr.sync();
    // rank the nb (<= GB_CAP) boundary candidates exactly; entries e = lane, lane + G
    constexpr int PE = GB_CAP / G > 0 ? GB_CAP / G : 1;
    double mk[PE];
    int32_t mi[PE], mg[PE];
    int rank[PE];
#pragma unroll
    for (int t = 0; t < PE; ++t) {
        const int e = gr.lane + t * G;
        mk[t] = INFINITY;
        mi[t] = 0x7fffffff;
        mg[t] = 0;
        rank[t] = 0;
        if (e < nb) {
            mk[t] = sc.bkey[e];
            mi[t] = sc.bidx[e];
            mg[t] = sc.bg[e];
        }
    }
    for (int e = 0; e < nb; ++e) {
        const double tk = sc.bkey[e];
        const int32_t ti = sc.bidx[e];
#pragma unroll
        for (int t = 0; t < PE; ++t) rank[t] += lt_pair(tk, ti, mk[t], mi[t]) ? 1 : 0;
    }
    bool found = false;
#pragma unroll
    for (int t = 0; t < PE; ++t) {
        const int e = gr.lane + t * G;
        const bool memb = e < nb && rank[t] < r;
        if (memb) {
            atomicAdd(&sc.lcnt[a.labels_perm[mg[t]]], 1);
            outs |= mg[t] < og0 || mg[t] >= og1;
        }
        if (e < nb && rank[t] == r - 1) found = true;
    }
    // the k-th's (key, idx): recompute from the owner
    const unsigned fl = gr.ballot(found);
    if (!fl) return false;
    const int src = __ffs(fl) - 1;
    double kk = INFINITY;
    int32_t ki = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < PE; ++t)
        if (gr.lane + t * G < nb && rank[t] == r - 1) {
            kk = mk[t];
            ki = mi[t];
        }
    out.key = gr.shfl(kk, src);
    out.idx = gr.shfl(ki, src);
    if (outside) *outside = gr.any(outs);
    gr.sync();
    return true;
}

// One query, G lanes.  Mirrors process_query_w (ghn_tile2d.cu).
template <int G>
__device__ __forceinline__ void process_query_grp(const T2Args &a, const Win &w, GrpScratch &sc,
                                                  const Grp<G> &gr, int32_t qi, int t0, int t1, int r_lo,
                                                  int c_lo, bool want_stats) {
    constexpr int GS = G;
    double q0, q1;
    if (a.q_dtype == GHN_F32) {
        q0 = (double)((const float *)a.Q)[2 * (int64_t)qi];
        q1 = (double)((const float *)a.Q)[2 * (int64_t)qi + 1];
    } else {
        q0 = ((const double *)a.Q)[2 * (int64_t)qi];
        q1 = ((const double *)a.Q)[2 * (int64_t)qi + 1];
    }
    const int64_t cc0 = cell_id(q0, a.w0, a.inv0, a.pow2 & 1u) - a.lo0;
    const int64_t cc1 = cell_id(q1, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1;
    const int64_t tr0 = (int64_t)t0 * a.T, tc0 = (int64_t)t1 * a.T;
    if (cc0 < tr0 || cc0 >= tr0 + a.T || cc1 < tc0 || cc1 >= tc0 + a.T || cc0 >= a.ext0 ||
        cc1 >= a.ext1) {
        if (gr.lane == 0) push_fallback(a, qi);
        return;
    }
    const int lr = (int)(cc0 - r_lo), lc = (int)(cc1 - c_lo);
    const int lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
    const int k = a.k;
    int64_t points = 0;
    int layers = 0;
    int32_t win_label = 0;
    int top = 0;
    if (k == 1) {
        // running minimum (explore.py:112-119 with k = 1)
        double ck = INFINITY;
        int32_t ci = 0x7fffffff, cg = -1;
        bool have = false;
        const ShellBound sbd(a, q0, q1, cc0, cc1);
        for (int l = 0;; ++l) {
            if (l > a.A) {
                if (gr.lane == 0) push_fallback(a, qi);
                return;
            }
            if (have && l > 0 && sbd.cannot_change(a, l - 1, ck)) {
                if (want_stats) {
                    int n = 0;
                    const int ca = max(lc - l, 0), cb = min(lc + l, w.W - 1) + 1;
                    const int ca1 = max(lc - l + 1, 0), cb1 = min(lc + l - 1, w.W - 1) + 1;
                    for (int row = max(lr - l, 0); row <= min(lr + l, w.R - 1); ++row) {
                        const int32_t *rp = w.loc + row * w.W1;
                        n += rp[cb] - rp[ca];
                        if (row > lr - l && row < lr + l) n -= rp[cb1] - rp[ca1];
                    }
                    points += n;
                }
                layers = l;
                bool stop = a.mode == GHN_MODE_HEURISTIC;
                if (a.mode == GHN_MODE_GUARANTEED) {
                    const double b = __dmul_rn((double)l, a.min_w);
                    if (__dmul_rn(b, b) > ck) stop = true;
                }
                if (stop || l >= lmax) break;
                continue;
            }
            double mk = INFINITY;
            int32_t mg = -1, mi = 0x7fffffff;
            int npts = 0;
            auto visit = [&](int p, int row, bool valid) {
                npts += valid ? 1 : 0;
                if (!valid) return;
                const double key = key2(w, p, q0, q1);
                const int32_t g = p + w.delta[row];
                if (key < mk) {
                    mk = key;
                    mg = g;
                    mi = 0x7fffffff;
                } else if (key == mk) {
                    if (mi == 0x7fffffff) mi = a.perm[mg];
                    const int32_t ii = a.perm[g];
                    if (ii < mi) {
                        mi = ii;
                        mg = g;
                    }
                }
            };
            if (l == 0) {
                GRP_FOR_BLOCK(w, gr, lr, lc, 0, visit(p, row, valid));
            } else {
                GRP_FOR_SHELL(w, gr, lr, lc, l, visit(p, row, valid));
            }
            if (mg >= 0 && mi == 0x7fffffff) mi = a.perm[mg];
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const double ok = gr.shfl_xor(mk, off);
                const int32_t oi = gr.shfl_xor(mi, off);
                const int32_t og = gr.shfl_xor(mg, off);
                if (lt_pair(ok, oi, mk, mi)) {
                    mk = ok;
                    mi = oi;
                    mg = og;
                }
            }
            npts = gr.sum(npts);
            points += npts;
            layers = l;
            bool changed = false;
            if (npts > 0 && (!have || lt_pair(mk, mi, ck, ci))) {
                ck = mk;
                ci = mi;
                cg = mg;
                changed = true;
                have = true;
            }
            bool stop = false;
            if (have) {
                if (a.mode == GHN_MODE_HEURISTIC && !changed) stop = true;
                if (a.mode == GHN_MODE_GUARANTEED) {
                    const double b = __dmul_rn((double)l, a.min_w);
                    if (__dmul_rn(b, b) > ck) stop = true;
                }
            }
            if (stop || l >= lmax) break;
        }
        win_label = a.labels_perm[cg];
        top = 1;
    } else {
        // phase 1: whole layers enter while fewer than k points are buffered
        int l = 0, total = 0;
        for (;; ++l) {
            if (l > a.A) {
                if (gr.lane == 0) push_fallback(a, qi);
                return;
            }
            const int ca = max(lc - l, 0), cb = min(lc + l, w.W - 1) + 1;
            int n = 0;
            for (int row = max(lr - l, 0); row <= min(lr + l, w.R - 1); ++row) {
                const int32_t *rp = w.loc + row * w.W1;
                n += rp[cb] - rp[ca];
            }
            total = n;
            if (total >= k || l >= lmax) break;
        }
        if (total < k) {
            if (gr.lane == 0) push_fallback(a, qi);
            return;
        }
        Kth kth{INFINITY, 0x7fffffff};
        bool stop = false;
        int sel_l = l;
        const bool skip0 = l == 0 && lmax >= 1;   // T_0 never needed (see process_query_w)
        const int ls = skip0 ? 1 : l;
        {
            const double e0 = fmax(q0 - (double)(a.lo0 + cc0 - ls) * a.w0, (double)(a.lo0 + cc0 + ls + 1) * a.w0 - q0);
            const double e1 = fmax(q1 - (double)(a.lo1 + cc1 - ls) * a.w1, (double)(a.lo1 + cc1 + ls + 1) * a.w1 - q1);
            const double hi = (e0 * e0 + e1 * e1) * (1.0 + 1e-6) + 1e-300;
            const int32_t *rp = w.loc + lr * w.W1;
            const int32_t og0 = skip0 ? rp[lc] + w.delta[lr] : 0;
            const int32_t og1 = skip0 ? rp[lc + 1] + w.delta[lr] : 0x7fffffff;
            bool outside = false;
            if (!select_grp<G>(a, w, sc, gr, lr, lc, ls, q0, q1, k, 0.0, hi, kth, og0, og1, &outside)) {
                if (gr.lane == 0) push_fallback(a, qi);
                return;
            }
            l = ls;
            sel_l = ls;
            if (skip0 && a.mode == GHN_MODE_HEURISTIC && !outside) stop = true;
            if (a.mode == GHN_MODE_GUARANTEED) {
                const double b = __dmul_rn((double)l, a.min_w);
                if (__dmul_rn(b, b) > kth.key) stop = true;
            }
        }
        {
            const int ca = max(lc - l, 0), cb = min(lc + l, w.W - 1) + 1;
            int n = 0;
            for (int row = max(lr - l, 0); row <= min(lr + l, w.R - 1); ++row) {
                const int32_t *rp = w.loc + row * w.W1;
                n += rp[cb] - rp[ca];
            }
            points = n;
        }
        layers = l;
        while (!stop && l < lmax) {
            ++l;
            if (l > a.A) {
                if (gr.lane == 0) push_fallback(a, qi);
                return;
            }
            int below = 0, pts = 0;
            if (shell_cannot_change(a, q0, q1, cc0, cc1, l - 1, kth.key)) {
                const int ca = max(lc - l, 0), cb = min(lc + l, w.W - 1) + 1;
                const int ca1 = max(lc - l + 1, 0), cb1 = min(lc + l - 1, w.W - 1) + 1;
                for (int row = max(lr - l, 0); row <= min(lr + l, w.R - 1); ++row) {
                    const int32_t *rp = w.loc + row * w.W1;
                    pts += rp[cb] - rp[ca];
                    if (row > lr - l && row < lr + l) pts -= rp[cb1] - rp[ca1];
                }
            } else {
                GRP_FOR_SHELL(w, gr, lr, lc, l, {
                    bool ltk = false;
                    if (valid) {
                        const double key = key2(w, p, q0, q1);
                        ltk = key < kth.key || (key == kth.key && a.perm[p + w.delta[row]] < kth.idx);
                    }
                    below += __popc(gr.ballot(ltk));
                    pts += __popc(gr.ballot(valid));
                });
            }
            points += pts;
            layers = l;
            const bool changed = below > 0;
            if (changed) {
                sel_l = l;
                if (!select_grp<G>(a, w, sc, gr, lr, lc, l, q0, q1, k, 0.0, kth.key, kth, 0, 0x7fffffff,
                                   nullptr)) {
                    if (gr.lane == 0) push_fallback(a, qi);
                    return;
                }
            }
            if (a.mode == GHN_MODE_HEURISTIC && !changed) stop = true;
            if (a.mode == GHN_MODE_GUARANTEED) {
                const double b = __dmul_rn((double)l, a.min_w);
                if (__dmul_rn(b, b) > kth.key) stop = true;
            }
        }
        // winner: top count; ties -> nearest member by (sqrt(key), index)
        constexpr int PER = 32 / G;
        int lc_[PER];
        int mx = 0;
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            lc_[t] = sc.lcnt[gr.lane * PER + t];
            mx = max(mx, lc_[t]);
        }
        top = gr.max(mx);
        unsigned tiedbits = 0;
#pragma unroll
        for (int t = 0; t < PER; ++t)
            if (lc_[t] == top) tiedbits |= 1u << (gr.lane * PER + t);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) tiedbits |= gr.shfl_xor(tiedbits, o);
        if (__popc(tiedbits) == 1) {
            win_label = __ffs(tiedbits) - 1;
        } else {
            // nearest member of a tied label over block(sel_l)
            double bd = INFINITY;
            int32_t bi = 0x7fffffff, bl = 0;
            GRP_FOR_BLOCK(w, gr, lr, lc, sel_l, {
                if (valid) {
                    const double key = key2(w, p, q0, q1);
                    if (key <= kth.key) {
                        const int32_t g = p + w.delta[row];
                        const int32_t idx = a.perm[g];
                        if (key < kth.key || idx <= kth.idx) {
                            const int32_t Lb = a.labels_perm[g];
                            if ((tiedbits >> Lb) & 1u) {
                                const double dd = sqrt(key);
                                if (dd < bd || (dd == bd && idx < bi)) {
                                    bd = dd;
                                    bi = idx;
                                    bl = Lb;
                                }
                            }
                        }
                    }
                }
            });
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const double od = gr.shfl_xor(bd, off);
                const int32_t oi = gr.shfl_xor(bi, off);
                const int32_t ol = gr.shfl_xor(bl, off);
                if (od < bd || (od == bd && oi < bi)) {
                    bd = od;
                    bi = oi;
                    bl = ol;
                }
            }
            win_label = bl;
        }
    }
    int64_t cells = 0;
    if (want_stats) {
        const int side = 2 * layers + 1;
        int c = 0;
        for (int e = gr.lane; e < side * side; e += G) {
            const int i = lr - layers + e / side, j = lc - layers + e % side;
            if (i >= 0 && i < w.R && j >= 0 && j < w.W) {
                const int32_t *rp = w.loc + i * w.W1;
                c += rp[j + 1] > rp[j];
            }
        }
        cells = gr.sum(c);
    }
    if (gr.lane == 0) {
        if (a.out_label) a.out_label[qi] = win_label;
        if (a.out_conf) a.out_conf[qi] = __ddiv_rn((double)top, (double)k);
        if (a.out_stats) {
            a.out_stats[3 * (int64_t)qi + 0] = layers;
            a.out_stats[3 * (int64_t)qi + 1] = cells;
            a.out_stats[3 * (int64_t)qi + 2] = points;
        }
        if (a.totals) {
            atomicAdd(&a.totals[0], (unsigned long long)layers);
            atomicAdd(&a.totals[1], (unsigned long long)cells);
            atomicAdd(&a.totals[2], (unsigned long long)points);
            atomicAdd(&a.totals[3], 1ull);
        }
    }
}

}  // namespace
}  // namespace ghn
