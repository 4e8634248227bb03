// ghn_tile2d_thr.cuh -- thread-per-query variant of the tiled 2-D classify
// (explore.py:66-137 + predict.py:20-36), for k <= 255 and <= 8 label codes.
//
// Each thread answers one query over the staged window, keeping PACKED keys:
//
//   packed = bits[62..31] of the fp64 key (exponent + 21 mantissa bits; the
//            sign is 0), low bits replaced by the label code (and, where a
//            path skips ahead, a shell flag above it).
//
// Truncating the IEEE pattern of a non-negative double is monotone, so the
// "d-part" (packed without its low bits) is a non-decreasing function of the
// exact key: sorting candidates by exact (key, index) also sorts them by
// d-part.  Hence, with tau = the k-th smallest packed value and D(.) the
// d-part:
//   * the k smallest d-parts are exactly the d-parts of the exact top-k, and
//     D(tau) = D(exact k-th key);
//   * a shell point precedes the exact k-th iff D(p) < D(tau) when
//     D(p) != D(tau) (explore.py:117 `changed`);
//   * when the (k+1)-th d-part exceeds D(tau) the top-k SET is {candidates
//     with D <= D(tau)} and their labels are known, so the vote needs no
//     point index.
// Every case the d-parts cannot decide (equal d-parts across the k-th
// boundary, a guaranteed-stop bound inside the k-th key's d-part interval,
// a vote tie-break between members less than two d-units apart) sends the
// query to the generic exact kernel -- rare (keys must agree to ~2^-18
// relative) and always correct.
//
// Three shapes, chosen per k (tile2d_thr_kernel):
//   k <= 2      each lane walks its own layers; branch-free min/max bubble
//               into a list of k+1 (process_query_thr);
//   3 <= k <= 32  warp lock-step rounds: block(l*) in batches of 8 sorted by
//               a network and merged into the list (ghn_nets.cuh), later
//               shells compare-only; k = 3-4 skip ahead to block(1)
//               (run_rounds_thr);
//   k > 32      bucket select: a histogram pass and a vote + boundary-list
//               pass (run_rounds_sel).
// Included by ghn_tile2d.cu after the shared helpers (T2Args, ShellBound,
// push_fallback).
#pragma once

#include "ghn_nets.cuh"

namespace ghn {
namespace {

// Bounds checks of the shared-memory walks, tables and note buffers: device
// asserts in a -DGHN_ASSERTS build (compute-sanitizer is closed on this GPU
// pool; tools/asserts.sh runs the GPU parity tests on such a build).
#ifdef GHN_ASSERTS
#include <assert.h>
#define GHN_ASSERT(c) assert(c)
#else
#define GHN_ASSERT(c) ((void)0)
#endif

constexpr int TT_THREADS = 256;
#ifndef GHN_TT_NOSORT_KM
#define GHN_TT_NOSORT_KM 2   // list capacities up to this keep the tile's query order (no counting sort by work)
#endif
#ifndef GHN_TT_TAB
#define GHN_TT_TAB 1   // k <= 32: table-driven rounds (run_rounds_tab); 0: the round-1 rounds, for A/B builds
#endif
constexpr uint32_t TT_INF = 0xffffffffu;

struct ThrWin {
    const float2 *xy;      // staged coordinates
    const uint8_t *sl;     // staged label codes
    const int32_t *loc;    // (R, W+1) local slot of each cell start
    int R, W, W1;
    const int32_t *rstart; // (R+1) first staged slot of each window row
    const int32_t *delta;  // (R) global CSR slot = staged slot + delta[row]
};

// Range r of shell(l) (l = 0: the centre cell; l >= 1: 4l ranges -- the full
// rows lr -+ l, then the side cells lc -+ l of the rows in between), clipped
// to the window (which holds every in-grid cell within the apron).
__device__ __forceinline__ void thr_shell_range(const ThrWin &w, int lr, int lc, int l, int r, int &s, int &e) {
    int row, ca, cb;
    if (l == 0) {
        row = lr;
        ca = cb = lc;
    } else if (r < 2) {
        row = r == 0 ? lr - l : lr + l;
        ca = max(lc - l, 0);
        cb = min(lc + l, w.W - 1);
    } else {
        row = lr - l + 1 + ((r - 2) >> 1);
        ca = cb = ((r - 2) & 1) ? lc + l : lc - l;
    }
    s = e = 0;
    if (row >= 0 && row < w.R && ca >= 0 && cb < w.W && ca <= cb) {
        const int32_t *rp = w.loc + row * w.W1;
        s = rp[ca];
        e = rp[cb + 1];
    }
}

__device__ __forceinline__ int thr_shell_count(const ThrWin &w, int lr, int lc, int l) {
    const int nr = l == 0 ? 1 : 4 * l;
    int n = 0;
    for (int r = 0; r < nr; ++r) {
        int s, e;
        thr_shell_range(w, lr, lc, l, r, s, e);
        n += e - s;
    }
    return n;
}

__device__ __forceinline__ int thr_block_cells(const ThrWin &w, int lr, int lc, int l) {
    int cells = 0;
    for (int row = max(lr - l, 0); row <= min(lr + l, w.R - 1); ++row) {
        const int32_t *rp = w.loc + row * w.W1;
        for (int c = max(lc - l, 0); c <= min(lc + l, w.W - 1); ++c) cells += rp[c + 1] > rp[c];
    }
    return cells;
}

// Packed key of a staged point: numpy einsum order for d = 2 (core.py:80;
// SURVEY Appendix A.3): d0^2 + d1^2, separate roundings, no FMA.
__device__ __forceinline__ uint32_t thr_pack(float2 c, double q0, double q1, uint32_t lab, uint32_t lmask) {
    const double d0 = __dsub_rn((double)c.x, q0);
    const double d1 = __dsub_rn((double)c.y, q1);
    const double key = __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
    const uint32_t top = __funnelshift_l((uint32_t)__double2loint(key), (uint32_t)__double2hiint(key), 1);
    return (top & ~lmask) | lab;
}

// The exact key itself (the same operations as thr_pack).
__device__ __forceinline__ double thr_key(float2 c, double q0, double q1) {
    const double d0 = __dsub_rn((double)c.x, q0);
    const double d1 = __dsub_rn((double)c.y, q1);
    return __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
}

// Keys whose d-part is D (label bits cleared) lie in [lower, upper).
__device__ __forceinline__ double thr_lower(uint32_t dm) {
    return __longlong_as_double((long long)((uint64_t)dm << 31));
}
__device__ __forceinline__ double thr_upper(uint32_t dm, uint32_t lmask) {
    return __longlong_as_double((long long)(((uint64_t)dm + lmask + 1u) << 31));
}

template <int N>
__device__ __forceinline__ void thr_bubble(uint32_t (&L)[N], uint32_t v) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const uint32_t m = min(L[j], v);
        v = max(L[j], v);
        L[j] = m;
    }
}

template <int N>
__device__ __forceinline__ uint32_t thr_pick(const uint32_t (&L)[N], int j) {
    uint32_t v = L[0];
#pragma unroll
    for (int i = 1; i < N; ++i) v = i == j ? L[i] : v;
    return v;
}

struct ThrTotals {
    unsigned long long layers, cells, points, n;
};

// Vote over the list's first k entries (predict.py:29-36).  False = the
// tie-break needs exact keys (generic kernel).
template <int KM>
__device__ __forceinline__ bool thr_vote(const uint32_t (&L)[KM + 1], int k, uint32_t lmask, int &wl, int &top,
                                         uint32_t dmask = 0u) {
    uint64_t cn = 0;   // 8-bit counter per label code
#pragma unroll
    for (int j = 0; j < KM; ++j)
        if (j < k) cn += 1ull << (8 * (L[j] & lmask));
    int ntie = 0;
    top = 0;
    wl = 0;
    for (int lab = 0; lab <= (int)lmask; ++lab) {
        const int c = (int)((cn >> (8 * lab)) & 0xffu);
        if (c > top) {
            top = c;
            wl = lab;
            ntie = 1;
        } else if (c == top && c > 0) {
            ++ntie;
        }
    }
    if (ntie > 1) {
        // the tied label of the member minimising (sqrt(key), index): the
        // first tied entry of the list, provided the first tied entry of
        // another label is >= 2 d-units behind it (then its key, and its
        // sqrt, is strictly larger)
        uint32_t w1 = TT_INF, w2 = TT_INF;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const uint32_t lab = L[j] & lmask;
            const bool tied = j < k && (int)((cn >> (8 * lab)) & 0xffu) == top;
            if (tied && w1 == TT_INF) w1 = L[j];
            else if (tied && w2 == TT_INF && lab != (w1 & lmask)) w2 = L[j];
        }
        const int lb = __popc(dmask ? dmask : lmask);   // bits below the d-part
        if ((w2 >> lb) - (w1 >> lb) < 2u) return false;
        wl = (int)(w1 & lmask);
    }
    return true;
}

// One query on one thread, each lane on its own (no lock-step): the best
// shape for k <= 2, where the bubble is short and lanes that need more
// layers should not hold the warp (measured at k = 1: 2.4 ms against 3.6
// for the lock-step rounds below and 2.8 with their skip-ahead; at k = 4 the
// skip-ahead rounds win, 2.8 against 3.4).
template <int KM, bool STATS>
__device__ __forceinline__ void process_query_thr(const T2Args &a, const ThrWin &w, int32_t qi, int t0, int t1,
                                                  int r_lo, int c_lo, ThrTotals &tot) {
    double q0, q1;
    if (a.q_dtype == GHN_F32) {
        const float2 qf = ((const float2 *)a.Q)[qi];
        q0 = (double)qf.x;
        q1 = (double)qf.y;
    } else {
        q0 = ((const double *)a.Q)[2 * (int64_t)qi];
        q1 = ((const double *)a.Q)[2 * (int64_t)qi + 1];
    }
    const int64_t cc0 = cell_id(q0, a.w0, a.inv0, a.pow2 & 1u) - a.lo0;
    const int64_t cc1 = cell_id(q1, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1;
    const int64_t tr0 = (int64_t)t0 * a.T, tc0 = (int64_t)t1 * a.T;
    if (cc0 < tr0 || cc0 >= tr0 + a.T || cc1 < tc0 || cc1 >= tc0 + a.T || cc0 >= a.ext0 || cc1 >= a.ext1) {
        push_fallback(a, qi);   // centre outside the grid
        return;
    }
    const int lr = (int)(cc0 - r_lo), lc = (int)(cc1 - c_lo);
    const int lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
    const int k = a.k;
    const uint32_t lmask = (uint32_t)a.lmask;
    uint32_t L[KM + 1];
#pragma unroll
    for (int j = 0; j <= KM; ++j) L[j] = TT_INF;
    const ShellBound sb(a, q0, q1, cc0, cc1);
    int cnt = 0, layers = 0;
    int64_t points = 0;
    for (int l = 0;; ++l) {
        if (l > a.A) {
            push_fallback(a, qi);
            return;
        }
        const bool full_prev = cnt >= k;
        const uint32_t tm = full_prev ? (thr_pick(L, k - 1) & ~lmask) : 0u;
        bool changed;
        if (full_prev && sb.cannot_change(a, l - 1, thr_upper(tm, lmask))) {
            // shell(l) cannot hold a point preceding the k-th (counted, not scanned)
            if (STATS) points += thr_shell_count(w, lr, lc, l);
            changed = false;
        } else {
            const int nr = l == 0 ? 1 : 4 * l;
            int r = 0, p, e;
            thr_shell_range(w, lr, lc, l, 0, p, e);
            bool lt = false, eq = false;
            int ns = 0;
            for (;;) {
                while (p >= e) {
                    if (++r >= nr) break;
                    thr_shell_range(w, lr, lc, l, r, p, e);
                }
                if (p >= e) break;
                const uint32_t pk = thr_pack(w.xy[p], q0, q1, (uint32_t)w.sl[p], lmask);
                lt |= pk < tm;
                eq |= (uint32_t)(pk - tm) <= lmask;
                thr_bubble(L, pk);
                ++ns;
                ++p;
            }
            if (full_prev && eq) {   // a shell point shares the k-th key's d-part
                push_fallback(a, qi);
                return;
            }
            cnt += ns;
            if (STATS) points += ns;
            changed = full_prev ? lt : ns > 0;
        }
        layers = l;
        bool stop = false;
        if (cnt >= k) {
            if (a.mode == GHN_MODE_HEURISTIC && !changed) stop = true;
            if (a.mode == GHN_MODE_GUARANTEED) {
                const double b = __dmul_rn((double)l, a.min_w);
                const double b2 = __dmul_rn(b, b);
                const uint32_t tk = thr_pick(L, k - 1) & ~lmask;
                if (b2 >= thr_upper(tk, lmask)) stop = true;
                else if (b2 > thr_lower(tk)) {   // bound inside the k-th key's interval
                    push_fallback(a, qi);
                    return;
                }
            }
        }
        if (stop || l >= lmax) break;
    }
    // top-k set = the list's first k entries unless the (k+1)-th shares the k-th's d-part
    const uint32_t tau = thr_pick(L, k - 1), nx = thr_pick(L, k);
    if (nx != TT_INF && (nx & ~lmask) == (tau & ~lmask)) {
        push_fallback(a, qi);
        return;
    }
    // vote (predict.py:29-36): 8-bit counters per label code
    uint64_t cn = 0;
#pragma unroll
    for (int j = 0; j < KM; ++j)
        if (j < k) cn += 1ull << (8 * (L[j] & lmask));
    int top = 0, ntie = 0, wl = 0;
    for (int lab = 0; lab <= (int)lmask; ++lab) {
        const int c = (int)((cn >> (8 * lab)) & 0xffu);
        if (c > top) {
            top = c;
            wl = lab;
            ntie = 1;
        } else if (c == top && c > 0) {
            ++ntie;
        }
    }
    if (ntie > 1) {
        // the tied label of the member minimising (sqrt(key), index): the
        // first tied entry of the list, provided the first tied entry of
        // another label is >= 2 d-units behind it (then its key, and its
        // sqrt, is strictly larger)
        uint32_t w1 = TT_INF, w2 = TT_INF;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const uint32_t lab = L[j] & lmask;
            const bool tied = j < k && (int)((cn >> (8 * lab)) & 0xffu) == top;
            if (tied && w1 == TT_INF) w1 = L[j];
            else if (tied && w2 == TT_INF && lab != (w1 & lmask)) w2 = L[j];
        }
        const int lb = __popc(lmask);
        if ((w2 >> lb) - (w1 >> lb) < 2u) {
            push_fallback(a, qi);
            return;
        }
        wl = (int)(w1 & lmask);
    }
    if (a.out_label) a.out_label[qi] = wl;
    if (a.out_conf) a.out_conf[qi] = __ddiv_rn((double)top, (double)k);
    if (STATS) {
        const int cells = thr_block_cells(w, lr, lc, layers);
        if (a.out_stats) {
            a.out_stats[3 * (int64_t)qi + 0] = layers;
            a.out_stats[3 * (int64_t)qi + 1] = cells;
            a.out_stats[3 * (int64_t)qi + 2] = points;
        }
        tot.layers += layers;
        tot.cells += cells;
        tot.points += points;
        tot.n += 1;
    }
}

// Per-range lower bound: q's distance to its own cell's faces (lower / upper
// per axis) and the rounding margin of ShellBound.  A rectangle of cells at
// offsets [ra, rb] x [ca, cb] from q's cell cannot hold a point whose key
// precedes `upper` when its distance to q (less the margin per axis) says so.
struct RectBound {
    double fl0, fh0, fl1, fh1, margin;
    __device__ __forceinline__ RectBound() : fl0(0.0), fh0(0.0), fl1(0.0), fh1(0.0), margin(0.0) {}
    __device__ __forceinline__ RectBound(const T2Args &a, double q0, double q1, int64_t cc0, int64_t cc1) {
        fl0 = q0 - (double)(a.lo0 + cc0) * a.w0;
        fh0 = (double)(a.lo0 + cc0 + 1) * a.w0 - q0;
        fl1 = q1 - (double)(a.lo1 + cc1) * a.w1;
        fh1 = (double)(a.lo1 + cc1 + 1) * a.w1 - q1;
        margin = 1e-9 * fmax(a.w0, a.w1) + 1e-12 * (fabs(q0) + fabs(q1));
    }
    // no point of shell(l) can precede `upper` (the face of block(l - 1))
    __device__ __forceinline__ bool shell_beyond(const T2Args &a, int l, double upper) const {
        const double d = fmin(fmin(fl0, fh0) + (double)(l - 1) * a.w0, fmin(fl1, fh1) + (double)(l - 1) * a.w1) - margin;
        return d > 0.0 && d * d * (1.0 - 1e-9) > upper;
    }
    __device__ __forceinline__ bool beyond(const T2Args &a, int ra, int rb, int ca, int cb, double upper) const {
        double dx = ra > 0 ? fh0 + (double)(ra - 1) * a.w0 : (rb < 0 ? fl0 + (double)(-rb - 1) * a.w0 : 0.0);
        double dy = ca > 0 ? fh1 + (double)(ca - 1) * a.w1 : (cb < 0 ? fl1 + (double)(-cb - 1) * a.w1 : 0.0);
        dx = fmax(dx - margin, 0.0);
        dy = fmax(dy - margin, 0.0);
        return (dx * dx + dy * dy) * (1.0 - 1e-9) > upper;
    }
};

// Range r of shell(l), l >= 1, as offsets from q's cell: rows [ra, rb] x cols [ca, cb].
__device__ __forceinline__ void thr_shell_rect(int l, int r, int &ra, int &rb, int &ca, int &cb) {
    if (r < 2) {
        ra = rb = r == 0 ? -l : l;
        ca = -l;
        cb = l;
    } else {
        ra = rb = -l + 1 + ((r - 2) >> 1);
        ca = cb = ((r - 2) & 1) ? l : -l;
    }
}

// Staged slot range of the cells at offsets (row ra, cols [ca, cb]) from (lr, lc), clipped.
__device__ __forceinline__ void thr_rect_slots(const ThrWin &w, int lr, int lc, int ra, int ca, int cb, int &s, int &e) {
    const int row = lr + ra, c0 = max(lc + ca, 0), c1 = min(lc + cb, w.W - 1);
    s = e = 0;
    if (row >= 0 && row < w.R && c0 <= c1) {
        const int32_t *rp = w.loc + row * w.W1;
        s = rp[c0];
        e = rp[c1 + 1];
    }
}

// Lock-step rounds cost the warp's LARGEST candidate count, so the tile's
// queries are first ordered by their candidate count (the block the first
// select walks): warps then hold queries of similar work.  The ordering
// pass also does phase A of the select once per query (sel_prep) and leaves
// its result in shared memory for the lane that takes the query.
constexpr int TT_SORT = 1024;     // queries per chunk of the list rounds
constexpr int SB_SORT_N = 512;   // queries ordered per chunk (a tile holds ~256)

// Points of block(l) in the window (rows lr -+ l, columns lc -+ l, clipped).
__device__ __forceinline__ int sel_block_count(const ThrWin &w, int lr, int lc, int l) {
    const int c0 = max(lc - l, 0), c1 = min(lc + l, w.W - 1);
    int n = 0;
    for (int row = max(lr - l, 0); row <= min(lr + l, w.R - 1); ++row) {
        const int32_t *rp = w.loc + row * w.W1;
        n += rp[c1 + 1] - rp[c0];
    }
    return n;
}

// Phase A of the bucket select for one query: l* = the first layer whose
// block holds k points (explore.py: every earlier layer leaves the buffer
// short, so it `changed` and no stop rule applies -- T_l* = top-k of
// block(l*)), and the skip-ahead decision (run_rounds_sel).  Packed:
// candidates | l* << 14 | skip << 17 | live << 18; 0 = the query leaves the
// tile path (centre outside the grid, or l* beyond the apron).
constexpr uint32_t SEL_LIVE = 1u << 18, SEL_SKIP = 1u << 17;
__device__ __forceinline__ uint32_t sel_prep(const T2Args &a, const ThrWin &w, int32_t qi, int t0, int t1, int r_lo,
                                             int c_lo, bool allow_skip) {
    double q0, q1;
    if (a.q_dtype == GHN_F32) {
        const float2 qf = ((const float2 *)a.Q)[qi];
        q0 = (double)qf.x;
        q1 = (double)qf.y;
    } else {
        q0 = ((const double *)a.Q)[2 * (int64_t)qi];
        q1 = ((const double *)a.Q)[2 * (int64_t)qi + 1];
    }
    const int64_t cc0 = cell_id(q0, a.w0, a.inv0, a.pow2 & 1u) - a.lo0;
    const int64_t cc1 = cell_id(q1, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1;
    const int64_t tr0 = (int64_t)t0 * a.T, tc0 = (int64_t)t1 * a.T;
    if (cc0 < tr0 || cc0 >= tr0 + a.T || cc1 < tc0 || cc1 >= tc0 + a.T || cc0 >= a.ext0 || cc1 >= a.ext1) return 0u;
    const int lr = (int)(cc0 - r_lo), lc = (int)(cc1 - c_lo);
    const int lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
    int l = 0, cnt = 0;
    for (;; ++l) {
        if (l > a.A) return 0u;
        cnt = sel_block_count(w, lr, lc, l);
        if (cnt >= a.k || l >= lmax) break;
    }
    // Skip-ahead (heuristic mode, fp32 queries): when block(l*) is barely
    // full (expected k-th radius beyond 0.8 of the block's half-width)
    // shell(l*+1) will most likely change the top-k, so the select runs over
    // block(l*+1) at once and learns changed(l*+1) from its members.
    uint32_t skip = 0u;
    if (allow_skip && a.mode == GHN_MODE_HEURISTIC && a.q_dtype == GHN_F32 && l < lmax && l + 1 <= a.A && cnt > 0) {
        const double kc = (double)a.k * (2.0 * l + 1.0) * (2.0 * l + 1.0) / (3.14159265358979 * (double)cnt);
        const double fc = a.sb_skipf * ((double)l + 0.5);
        if (kc > fc * fc) {
            const int c2 = sel_block_count(w, lr, lc, l + 1);
            if (c2 <= a.sb_capn) {
                skip = SEL_SKIP;
                cnt = c2;
            }
        }
    }
    return (uint32_t)cnt | ((uint32_t)l << 14) | skip | SEL_LIVE;
}

// info[i] = sel_prep of query c0 + i; ord[0, c1 - c0) = the local indices
// sorted by (skip-ahead, candidate count 0..255, larger clamped): a counting sort.
__device__ __forceinline__ void sel_sort_chunk(const T2Args &a, const ThrWin &w, int c0, int c1, int t0, int t1,
                                               int r_lo, int c_lo, int *hcnt, uint16_t *kr, uint16_t *ord,
                                               uint32_t *info, bool allow_skip, bool order = true) {
    if (!order) {   // phase A only, queries in tile order (k <= GHN_TT_NOSORT_K: the sort costs more than it saves)
        for (int i = threadIdx.x; i < c1 - c0; i += TT_THREADS) {
            info[i] = sel_prep(a, w, a.qorder[c0 + i], t0, t1, r_lo, c_lo, allow_skip);
            ord[i] = (uint16_t)i;
        }
        __syncthreads();
        return;
    }
    for (int i = threadIdx.x; i < 512; i += TT_THREADS) hcnt[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < c1 - c0; i += TT_THREADS) {
        const uint32_t f = sel_prep(a, w, a.qorder[c0 + i], t0, t1, r_lo, c_lo, allow_skip);
        info[i] = f;
        // skip-ahead queries together (their pass 2 also tracks the shell), then by count
        const int key = a.sb_sort ? min((int)(f & 0x3fffu), 255) + ((f & SEL_SKIP) ? 256 : 0) : 0;
        const int rank = atomicAdd(&hcnt[key], 1);
        kr[2 * i] = (uint16_t)key;
        kr[2 * i + 1] = (uint16_t)rank;
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the 512 counters, 16 per lane
        int v[16], sum = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            v[j] = hcnt[threadIdx.x * 16 + j];
            sum += v[j];
        }
        const int incl = warp_inclusive_scan(sum);
        int run = incl - sum;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            hcnt[threadIdx.x * 16 + j] = run;
            run += v[j];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < c1 - c0; i += TT_THREADS) ord[hcnt[kr[2 * i]] + kr[2 * i + 1]] = (uint16_t)i;
    __syncthreads();
}

// The tile's queries in rounds of one query per thread.  Per round:
//  A  (per lane) load the query; l* = the first layer whose block holds k
//     points (explore.py: every earlier layer leaves the buffer short, so it
//     `changed` and no stop rule applies -- T_l* = top-k of block(l*));
//  B  (warp lock-step) all candidates of block(l*), row by row, into the
//     list: one candidate per lane per step (+inf pads the shorter lanes), so
//     the bubble is always issued for the whole warp;
//  C  (warp lock-step) later layers while some lane continues: each lane
//     scans its shell's ranges that are not provably beyond the k-th key
//     (compare only); a lane whose shell changed the top-k re-scans it into
//     the list;
//  D  the vote (predict.py:29-36) and the outputs.
template <int KM, bool STATS>
__device__ __forceinline__ void run_rounds_thr(const T2Args &a, const ThrWin &w, const uint16_t *ord, int *s_grp, int qb, int qe, int t0, int t1,
                                               int r_lo, int c_lo, ThrTotals &tot) {
    const int k = a.k;
    const uint32_t lmask = (uint32_t)a.lmask;
    constexpr bool SKIP_AHEAD = KM == 4;
    // label bits + the shell flag above them (skip-ahead only)
    const uint32_t fmask = SKIP_AHEAD ? 2u * lmask + 1u : lmask;
    const int64_t tr0 = (int64_t)t0 * a.T, tc0 = (int64_t)t1 * a.T;
    for (;;) {
        // the next group of 32 (sorted) queries for this warp: warps that
        // finish early take more groups instead of waiting at the barrier
        int g0 = 0;
        if ((threadIdx.x & 31) == 0) g0 = atomicAdd(s_grp, 32);
        g0 = __shfl_sync(GHN_FULL, g0, 0);
        if (g0 >= qe - qb) break;
        const int qr = qb + g0 + (int)(threadIdx.x & 31);
        bool live = qr < qe;   // this lane holds a query still being answered
        const int qq = live ? qb + ord[qr - qb] : 0;
        int32_t qi = 0;
        double q0 = 0.0, q1 = 0.0;
        int64_t cc0 = 0, cc1 = 0;
        int lr = 0, lc = 0, lmax = 0, l = 0, cnt = 0;
        if (live) {
            qi = a.qorder[qq];
            if (a.q_dtype == GHN_F32) {
                const float2 qf = ((const float2 *)a.Q)[qi];
                q0 = (double)qf.x;
                q1 = (double)qf.y;
            } else {
                q0 = ((const double *)a.Q)[2 * (int64_t)qi];
                q1 = ((const double *)a.Q)[2 * (int64_t)qi + 1];
            }
            cc0 = cell_id(q0, a.w0, a.inv0, a.pow2 & 1u) - a.lo0;
            cc1 = cell_id(q1, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1;
            if (cc0 < tr0 || cc0 >= tr0 + a.T || cc1 < tc0 || cc1 >= tc0 + a.T || cc0 >= a.ext0 ||
                cc1 >= a.ext1) {
                push_fallback(a, qi);   // centre outside the grid
                live = false;
            }
        }
        if (live) {
            lr = (int)(cc0 - r_lo);
            lc = (int)(cc1 - c_lo);
            lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
            // l*: block(l) = block(l-1) + shell(l)
            for (;;) {
                if (l > a.A) {
                    push_fallback(a, qi);
                    live = false;
                    break;
                }
                if (l == 0) {
                    int s, e;
                    thr_rect_slots(w, lr, lc, 0, 0, 0, s, e);
                    cnt = e - s;
                } else {
                    for (int r = 0; r < 4 * l; ++r) {
                        int ra, rb, ca, cb, s, e;
                        thr_shell_rect(l, r, ra, rb, ca, cb);
                        thr_rect_slots(w, lr, lc, ra, ca, cb, s, e);
                        cnt += e - s;
                    }
                }
                if (cnt >= k || l >= lmax) break;
                ++l;
            }
        }
        // Skip-ahead (heuristic mode): when block(l*) is barely full the next
        // shell will most likely change the top-k, so select over block(l*+1)
        // at once; changed(l*+1) is read off a flag on shell(l*+1)'s points.
        // Compiled for the 4-slot list only (k = 3, 4): at k = 16 the next
        // shell rarely changes and the extra registers cost a CTA per SM.
        bool skipm = false;
        if (SKIP_AHEAD && live && a.mode == GHN_MODE_HEURISTIC && l < lmax && l + 1 <= a.A) {
            const double kc = (double)k * (2.0 * l + 1.0) * (2.0 * l + 1.0) / (3.14159265358979 * (double)cnt);
            const double fc = a.tt_skipf * ((double)l + 0.5);
            if (kc > fc * fc) {
                int sc = 0;
                for (int r = 0; r < 4 * (l + 1); ++r) {
                    int ra, rb, ca, cb, s0, e0;
                    thr_shell_rect(l + 1, r, ra, rb, ca, cb);
                    thr_rect_slots(w, lr, lc, ra, ca, cb, s0, e0);
                    sc += e0 - s0;
                }
                skipm = true;
                ++l;
                cnt += sc;
            }
        }
        // ---- B: block(l) row by row, lock-step
        uint32_t L[KM + 1];
#pragma unroll
        for (int j = 0; j <= KM; ++j) L[j] = TT_INF;
        {
            const int n = live ? cnt : 0;
            const int steps = __reduce_max_sync(GHN_FULL, n);
            int ra = -l, p = 0, e = 0, pi0 = 0, pi1 = 0;
            if (live) {
                thr_rect_slots(w, lr, lc, ra, -l, l, p, e);
                if (SKIP_AHEAD) thr_rect_slots(w, lr, lc, ra, -(l - 1), l - 1, pi0, pi1);
            }
            // batches of 8 candidates per lane: sorted by a 19-comparator
            // network, then merged into the list (NetMerge8: 41 comparators
            // at k = 16) -- 15 min/max pairs per candidate instead of the
            // bubble's k + 1
            for (int it = 0; it < steps; it += 8) {
                uint32_t bt[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const bool have = it + u < n;
                    while (have && p >= e) {
                        ++ra;
                        thr_rect_slots(w, lr, lc, ra, -l, l, p, e);
                        if (SKIP_AHEAD) thr_rect_slots(w, lr, lc, ra, -(l - 1), l - 1, pi0, pi1);
                    }
                    const int pp = have ? p : 0;
                    const bool insh = SKIP_AHEAD && skipm && (ra == -l || ra == l || pp < pi0 || pp >= pi1);
                    const uint32_t pk =
                        thr_pack(w.xy[pp], q0, q1, (uint32_t)w.sl[pp] | (insh ? lmask + 1u : 0u), fmask);
                    bt[u] = have ? pk : TT_INF;
                    p += have ? 1 : 0;
                }
                if constexpr (KM <= 2) {   // a list of 2-3: the bubble is cheaper than sort + merge
#pragma unroll
                    for (int u = 0; u < 8; ++u) thr_bubble(L, bt[u]);
                } else {
                    net_sort8(bt);
                    NetMerge8<KM + 1>::run(L, bt);
                }
            }
        }
        int layers = l;
        int64_t points = cnt;
        if (SKIP_AHEAD && live && skipm) {
            // changed(l*+1) <=> a member of T_{l*+1} carries the shell flag;
            // membership needs a clean k-th boundary
            const uint32_t tau = thr_pick(L, k - 1), nx = thr_pick(L, k);
            bool chg = false;
#pragma unroll
            for (int j = 0; j < KM; ++j) chg |= j < k && (L[j] & (lmask + 1u)) != 0u;
            if (nx != TT_INF && (nx & ~fmask) == (tau & ~fmask)) {
                push_fallback(a, qi);
                live = false;
            } else if (!chg) {
                lmax = l;   // heuristic stop at l*+1
            }
        }
        // stop rules after layer l* (it filled the buffer: changed)
        if (live && cnt >= k && a.mode == GHN_MODE_GUARANTEED) {
            const double b = __dmul_rn((double)l, a.min_w);
            const double b2 = __dmul_rn(b, b);
            const uint32_t tk = thr_pick(L, k - 1) & ~fmask;
            if (b2 >= thr_upper(tk, fmask)) {
                lmax = l;   // stop
            } else if (b2 > thr_lower(tk)) {
                push_fallback(a, qi);
                live = false;
            }
        }
        bool more = live && l < lmax;   // continues with layer l + 1
        bool fin = live && !more;       // answered after layer l
        // ---- C: later layers
        const RectBound rb0 = more ? RectBound(a, q0, q1, cc0, cc1) : RectBound();
        while (__any_sync(GHN_FULL, more)) {
            uint32_t tm = 0;
            double upper = 0.0;
            if (more) {
                ++l;
                if (l > a.A) {
                    push_fallback(a, qi);
                    more = false;
                }
                tm = thr_pick(L, k - 1) & ~fmask;
                upper = thr_upper(tm, fmask);
            }
            // compare-only scan of the shell's ranges that may hold a point preceding the k-th
            bool lt = false, eq = false;
            int sc = 0;   // points of shell(l) (stats)
            {
                int r = 0, p = 0, e = 0;
                const int nr = 4 * l;
                // the whole shell first (one test); per range only if it may matter
                bool act = more && !rb0.shell_beyond(a, l, upper);
                if (STATS && more && !act) sc = thr_shell_count(w, lr, lc, l);
                for (;;) {
                    while (act && p >= e) {
                        if (r >= nr) {
                            act = false;
                            break;
                        }
                        int ra, rb, ca, cb;
                        thr_shell_rect(l, r, ra, rb, ca, cb);
                        ++r;
                        thr_rect_slots(w, lr, lc, ra, ca, cb, p, e);
                        if (STATS) sc += e - p;
                        if (rb0.beyond(a, ra, rb, ca, cb, upper)) e = p;
                    }
                    if (!__any_sync(GHN_FULL, act)) break;
                    const int pp = act ? p : 0;
                    const uint32_t pk = thr_pack(w.xy[pp], q0, q1, (uint32_t)w.sl[pp], fmask);
                    lt |= act && pk < tm;
                    eq |= act && (uint32_t)(pk - tm) <= fmask;
                    p += act ? 1 : 0;
                }
            }
            if (more && eq) {   // a shell point shares the k-th key's d-part
                push_fallback(a, qi);
                more = false;
            }
            // a lane whose shell changed the top-k brings the shell into the list
            bool redo = more && lt;
            if (__any_sync(GHN_FULL, redo)) {
                int r = 0, p = 0, e = 0;
                const int nr = 4 * l;
                for (;;) {
                    while (redo && p >= e) {
                        if (r >= nr) {
                            redo = false;
                            break;
                        }
                        int ra, rb, ca, cb;
                        thr_shell_rect(l, r, ra, rb, ca, cb);
                        ++r;
                        thr_rect_slots(w, lr, lc, ra, ca, cb, p, e);
                        if (rb0.beyond(a, ra, rb, ca, cb, upper)) e = p;
                    }
                    if (!__any_sync(GHN_FULL, redo)) break;
                    const int pp = redo ? p : 0;
                    uint32_t pk = thr_pack(w.xy[pp], q0, q1, (uint32_t)w.sl[pp], fmask);
                    pk = redo ? pk : TT_INF;
                    thr_bubble(L, pk);
                    p += redo ? 1 : 0;
                }
            }
            if (more) {
                layers = l;
                points += sc;
                bool stop = !lt && a.mode == GHN_MODE_HEURISTIC;
                if (a.mode == GHN_MODE_GUARANTEED) {
                    const double b = __dmul_rn((double)l, a.min_w);
                    const double b2 = __dmul_rn(b, b);
                    const uint32_t tk = thr_pick(L, k - 1) & ~fmask;
                    if (b2 >= thr_upper(tk, fmask)) {
                        stop = true;
                    } else if (b2 > thr_lower(tk)) {
                        push_fallback(a, qi);
                        more = false;
                    }
                }
                if (more && (stop || l >= lmax)) {
                    more = false;
                    fin = true;
                }
            }
        }
        // ---- D: vote and outputs
        if (fin) {
            const uint32_t tau = thr_pick(L, k - 1), nx = thr_pick(L, k);
            int wl, top;
            if ((nx != TT_INF && (nx & ~fmask) == (tau & ~fmask)) || !thr_vote<KM>(L, k, lmask, wl, top, fmask)) {
                push_fallback(a, qi);
            } else {
                if (a.out_label) a.out_label[qi] = wl;
                if (a.out_conf) a.out_conf[qi] = __ddiv_rn((double)top, (double)k);
                if (STATS) {
                    const int cells = thr_block_cells(w, lr, lc, layers);
                    if (a.out_stats) {
                        a.out_stats[3 * (int64_t)qi + 0] = layers;
                        a.out_stats[3 * (int64_t)qi + 1] = cells;
                        a.out_stats[3 * (int64_t)qi + 2] = points;
                    }
                    tot.layers += layers;
                    tot.cells += cells;
                    tot.points += points;
                    tot.n += 1;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- k > 32
// Bucket select (k in (32, 255]): the bubble's cost grows with k, so for
// large k block(l*) is passed over twice in lock-step, one candidate per lane
// per step, on fp32 keys; only the few candidates around the k-th get the
// exact fp64 key (numpy einsum order).
//   Pass 1 histograms fp32 keys into SB_NB buckets of 2^-SB_MB octave
//     (exponent and SB_MB mantissa bits -- bucket edges are d-part edges)
//     around the expected k-th key, in a per-lane byte histogram in shared
//     memory; the bucket bb where the count reaches k follows.
//   Pass 2 classifies every candidate by its fp32 key again: more than
//     `ulps` below bucket bb's lower edge it is a member (voted at once: one
//     shift and one add), more than `ulps` above the upper edge it is not,
//     and the candidates in between (bucket bb itself: ~1 % of them) have
//     their slot noted in the lane's (now free) histogram words.
//   The noted candidates are then re-keyed exactly, in lock-step over the
//     warp's largest count: below bb's lower edge (a d-part edge) they are
//     members, the others are bubbled into a list of SB_C + 1 -- the k-th is
//     its r-th entry (r = k - members below) and must lie inside bucket bb.
// The fp32 key (two subtractions, a product and an fma of fp32 values) is
// within 5 ulps of the exact one for fp32 queries, so both sure classes are
// exact with ulps = 8; for fp64 queries the fp32 key uses the rounded query
// and ulps grows with |q| / sqrt(key) (sel_ulps).  Pass 1 only proposes bb:
// every count that decides the result is taken from pass 2 and the exact
// re-keying.
// Both passes walk the block through a per-lane table of its non-empty rows
// (slot ranges, filled once per select) with a branch-free advance: the
// per-lane row changes cost no divergent code.
// Later shells are checked compare-only; a shell that changes the top-k makes
// its block the next select (for >= SB_REDO lanes of the warp; a lone one
// goes to the generic kernel), as does a boundary bucket holding the k-th
// beyond SB_C.
constexpr int SB_NB = 64;   // buckets (0 and SB_NB-1 catch the tails)
#ifndef SB_MB
#define SB_MB 5             // mantissa bits in a bucket index: 2^SB_MB buckets per octave (4: -2 %)
#endif
constexpr int SB_S = 21 - SB_MB;   // packed >> SB_S: exponent + SB_MB mantissa bits
constexpr int SB_C = 8;     // boundary list capacity
constexpr int SB_LMAX = 4;  // largest block half-width the row table holds
constexpr int SB_ROWS = 2 * SB_LMAX + 2;   // table words per lane: the rows + the closing sentinel
constexpr int SB_F32_S = 23 - SB_MB;       // fp32 bits >> SB_F32_S: exponent + SB_MB mantissa bits
constexpr int SB_F32_SHIFT = (1023 - 127) << SB_MB;   // fp64 bucket index = fp32 bucket index + this
constexpr int SB_NOTE = SB_NB / 4;         // candidates a lane can note for exact re-keying (one per histogram word)
constexpr uint32_t SB_SENT = 0xffff0000u;  // table sentinel: slots [0, 65535) -- never exhausted

// min(max(x, 0), hi) in one instruction (VIMNMX.RELU)
__device__ __forceinline__ int sb_clamp(int x, int hi) {
    int r;
    asm("min.relu.s32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(hi));
    return r;
}

// fp32 key bits of a staged point (identical in both passes)
__device__ __forceinline__ uint32_t sb_bits32(float dx, float dy) {
    return __float_as_uint(__fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// The hot loops address shared memory through 32-bit shared-space addresses
// (generic pointers cost 64-bit arithmetic per step).
__device__ __forceinline__ uint32_t sm_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

// Lock-step walk over a lane's row table (word j at tab[j * TT_THREADS] =
// first slot | end slot << 16 of its j-th non-empty row, closed by SB_SENT).
// Every lane consumes slot p each step; a lane whose row is exhausted moves
// to the prefetched next row (selects only).  A lane past its last row -- or
// an idle one -- walks the sentinel's slots 0, 1, ... (in bounds: steps <=
// staged points); the caller masks what it computes there.
struct SelWalk {
    uint32_t tp;   // shared address of the prefetched word
    uint32_t nx;
    int p, e;
    __device__ __forceinline__ void start(uint32_t tab, bool on) {
        const uint32_t w0 = on ? lds_u32(tab) : SB_SENT;
        p = (int)(w0 & 0xffffu);
        e = (int)(w0 >> 16);
        tp = tab + TT_THREADS * 4;
        nx = lds_u32(tp);
    }
    __device__ __forceinline__ void step() {
        p += 1;
        const bool adv = p >= e;
        p = adv ? (int)(nx & 0xffffu) : p;
        e = adv ? (int)(nx >> 16) : e;
        tp += adv ? TT_THREADS * 4 : 0;
        nx = lds_u32(tp);
    }
};

template <bool WIDE> struct SelCnt { typedef uint32_t type; };
template <> struct SelCnt<true> { typedef uint64_t type; };

__device__ __forceinline__ int sel_bytesum(uint32_t v) { return (int)__dp4a(v, 0x01010101u, 0u); }
__device__ __forceinline__ int sel_bytesum(uint64_t v) {
    return (int)__dp4a((uint32_t)v, 0x01010101u, __dp4a((uint32_t)(v >> 32), 0x01010101u, 0u));
}

// Skip-ahead lanes: is a candidate of block(ls) in shell(ls)?  From fp32
// coordinates: u = the candidate's Chebyshev distance from the centre of q's
// cell in units of block(ls-1)'s half-width; u > 1 + eps: surely in the
// shell, u < 1 - eps: surely inside block(ls-1), else the point's own cell
// decides (exact re-keying pass).  Other lanes carry s = 0: u = 0, always
// inside.
struct SelGeo {
    float s0, s1, o0, o1;
    __device__ __forceinline__ float u(float dx, float dy) const {
        return fmaxf(fabsf(__fmaf_rn(dx, s0, o0)), fabsf(__fmaf_rn(dy, s1, o1)));
    }
};
constexpr float SEL_GEO_LO = 1.0f - 3e-6f, SEL_GEO_HI = 1.0f + 3e-6f;   // fp32 rounding of u: < 1e-6

// Pass 2 for the whole warp.  Sure members are voted into cn; the slots of
// the candidates to re-key are noted at note[j * TT_THREADS] (low half);
// `noted` may exceed SB_NOTE (SKIP only): the caller gives up then.
// SKIP: geo != 0 iff a sure member lies in shell(ls).
template <bool SKIP, bool WIDE>
__device__ __forceinline__ void sel_pass2(uint32_t xy_s, uint32_t sl_s, uint32_t myr_s, uint32_t note_s, bool sel, int n,
                                          int steps, float q0f, float q1f, uint32_t tlo, uint32_t span,
                                          const SelGeo &g, typename SelCnt<WIDE>::type &cn_out, int &noted,
                                          uint32_t &geo_out) {
    typedef typename SelCnt<WIDE>::type cnt_t;
    cnt_t cn = 0;
    uint32_t geo = 0u;
    int nnote = 0;
    uint32_t np = note_s;
    SelWalk wk;
    wk.start(myr_s, sel);
    const int n2 = sel ? n : 0;
    for (int it = 0; it < steps; ++it) {
        const float2 c = lds_f2(xy_s + 8u * (uint32_t)wk.p);
        const uint32_t lab8 = lds_u8(sl_s + (uint32_t)wk.p);   // label code * 8
        const float dx = __fsub_rn(c.x, q0f), dy = __fsub_rn(c.y, q1f);
        const uint32_t bits = sb_bits32(dx, dy);
        const bool have = it < n2;
        const bool low = have && bits < tlo;
        const bool amb = have && (uint32_t)(bits - tlo) < span;
        bool vote = low, note = amb;
        if (SKIP) {
            // a sure member whose cell the fp32 coordinates cannot place (on a
            // cell boundary of block(ls-1), common for fp32 data on a power-of-two
            // grid) is noted too: the re-keying places it exactly
            const float u = g.u(dx, dy);
            const bool band = low && u > SEL_GEO_LO && !(u > SEL_GEO_HI);
            geo |= low && u > SEL_GEO_HI ? 1u : 0u;
            vote = low && !band;
            note = amb || band;
            nnote += note ? 1 : 0;
        }
        if (WIDE) {
            const uint64_t inc = 1ull << lab8;
            cn += vote ? (cnt_t)inc : (cnt_t)0;
        } else {
            const uint32_t inc = __funnelshift_l(0u, 1u, lab8);   // 1 << lab8, lab8 <= 24
            cn += vote ? (cnt_t)inc : (cnt_t)0;
        }
        GHN_ASSERT(wk.p >= 0 && wk.p < 65536 && (!note || np < note_s + (uint32_t)SB_NOTE * TT_THREADS * 4));
        if (note) asm volatile("st.shared.u16 [%0], %1;" ::"r"(np), "h"((uint16_t)wk.p) : "memory");
        np += note ? TT_THREADS * 4 : 0;
        // (SKIP: the histogram does not bound the boundary members; past the
        // lane's SB_NOTE words the last one is overwritten and the count tells)
        if (SKIP) np = min(np, note_s + (uint32_t)(SB_NOTE - 1) * TT_THREADS * 4);
        wk.step();
    }
    cn_out = cn;
    noted = SKIP ? nnote : (int)((np - note_s) / (TT_THREADS * 4));
    geo_out = geo;
}

// fp32 key bits this far from an edge of bucket bb may be on the other side
// in exact arithmetic.  fp32 queries: the fp32 key is within 5 ulps.  fp64
// queries: the fp32 key is computed from the rounded query, off by at most
// |q| 2^-24 per axis, i.e. 2^-23 (|q0| + |q1|) / sqrt(key) relative -- a
// multiple of the fp32 ulp (2^-23 .. 2^-24 relative) taken at the bucket's
// lower edge, doubled.  0 = the bucket cannot be classified in fp32.
__device__ __forceinline__ uint32_t sel_ulps(bool f32q, double q0, double q1, double edge_lo) {
    if (f32q) return 8u;
    if (!(edge_lo > 0.0)) return 0u;
    const double m = 4.0 * (fabs(q0) + fabs(q1)) * rsqrt(edge_lo) + 8.0;
    return m < (double)(1u << (SB_F32_S - 2)) ? (uint32_t)m : 0u;
}

template <bool STATS, bool WIDE>
__device__ __forceinline__ void run_rounds_sel(const T2Args &a, const ThrWin &w, uint32_t *hist, uint32_t *rtab,
                                               const uint16_t *ord, const uint32_t *info, int *s_grp, int qb, int qe,
                                               int t0, int t1, int r_lo, int c_lo, ThrTotals &tot) {
    typedef typename SelCnt<WIDE>::type cnt_t;
    const int k = a.k;
    const uint32_t lmask = (uint32_t)a.lmask;
    const uint32_t fmask = 2u * lmask + 1u;   // label bits + the shell flag above them
    const bool f32q = a.q_dtype == GHN_F32;
    uint32_t *myh = hist + threadIdx.x;       // word i of this lane at myh[i * TT_THREADS]
    uint32_t *myr = rtab + threadIdx.x;       // row-table word j at myr[j * TT_THREADS]
    const uint32_t myh_s = sm_addr(myh), myr_s = sm_addr(myr), xy_s = sm_addr(w.xy), sl_s = sm_addr(w.sl);
    for (;;) {
        int g0 = 0;   // the next group of 32 (sorted) queries for this warp
        if ((threadIdx.x & 31) == 0) g0 = atomicAdd(s_grp, 32);
        g0 = __shfl_sync(GHN_FULL, g0, 0);
        if (g0 >= qe - qb) break;
        const int qr = g0 + (int)(threadIdx.x & 31);
        bool live = qr < qe - qb;
        // heaviest groups first (ord is ascending in candidate count): the
        // CTA's tail is then a light group
        const int li = live ? (int)ord[qe - qb - 1 - qr] : 0;
        const uint32_t f = live ? info[li] : 0u;
        int32_t qi = 0;
        double q0 = 0.0, q1 = 0.0;
        float q0f = 0.0f, q1f = 0.0f;
        int64_t cc0 = 0, cc1 = 0;
        int lr = 0, lc = 0, lmax = 0, l = 0, cnt = 0;
        bool skipm = false;
        if (live) {
            qi = a.qorder[qb + li];
            if (a.q_dtype == GHN_F32) {
                const float2 qf = ((const float2 *)a.Q)[qi];
                q0 = (double)qf.x;
                q1 = (double)qf.y;
                q0f = qf.x;
                q1f = qf.y;
            } else {
                q0 = ((const double *)a.Q)[2 * (int64_t)qi];
                q1 = ((const double *)a.Q)[2 * (int64_t)qi + 1];
                q0f = (float)q0;
                q1f = (float)q1;
            }
            if (!(f & SEL_LIVE)) {   // centre outside the grid / l* beyond the apron (sel_prep)
                { FB_REASON(1); push_fallback(a, qi); }
                live = false;
            }
        }
        if (live) {
            cc0 = cell_id(q0, a.w0, a.inv0, a.pow2 & 1u) - a.lo0;
            cc1 = cell_id(q1, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1;
            lr = (int)(cc0 - r_lo);
            lc = (int)(cc1 - c_lo);
            lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
            l = (int)((f >> 14) & 7u);
            cnt = (int)(f & 0x3fffu);
            skipm = (f & SEL_SKIP) != 0u;
        }
        // Select over block(ls) (lock-step passes), then check the later
        // shells compare-only; a shell that changes the top-k makes its
        // block the next select (explore.py:104-130).
        int ls = l + (skipm ? 1 : 0), layers = l, cls = 0;
        bool need = live, fin = false, noprune = false;
        cnt_t cn = 0;
        uint32_t tau = 0, tm = 0;
        double upper = 0.0;
        while (__any_sync(GHN_FULL, need)) {
            if (need && ls > SB_LMAX) {   // beyond the row table
                { FB_REASON(2); push_fallback(a, qi); }
                need = false;
            }
            // expected k-th key from the block's density
            int bbase = 0;
            double r2 = 0.0;   // pruning radius (squared); 0: the whole block
            if (need) {
                const double side = (double)(2 * ls + 1);
                const double kest = (double)k * side * side * a.w0 * a.w1 / (3.14159265358979 * (double)max(cnt, 1));
                // the 62 inner buckets span 62 / 2^SB_MB octaves centred on kest
                const double klo = kest * exp2(-0.5 * (SB_NB - 2) / (double)(1 << SB_MB));
                const uint32_t top = __funnelshift_l((uint32_t)__double2loint(klo), (uint32_t)__double2hiint(klo), 1);
                bbase = (int)(top >> SB_S) - 1;
                // the k-th key exceeds this with probability ~1e-6 (5 sigma of the
                // count inside the radius); checked after the select
                if (!noprune) r2 = kest * (1.0 + 5.0 * rsqrt((double)k));
            }
            // ---- the block's non-empty rows -> this lane's table.  Each row is
            // clipped to the cells that can hold a point within sqrt(r2) of q
            // (fp32 arithmetic with margins far above its rounding: a superset).
            int n = 0;
            {
                const int nrows = need ? 2 * ls + 1 : 0;
                const int rmax = __reduce_max_sync(GHN_FULL, nrows);
                const bool prune = r2 > 0.0;
                // q's distance to the faces of its own cell
                const float w0f = (float)a.w0, w1f = (float)a.w1;
                const float fl0 = (float)(q0 - (double)(a.lo0 + cc0) * a.w0), fh0 = w0f - fl0;
                const float fl1 = (float)(q1 - (double)(a.lo1 + cc1) * a.w1), fh1 = w1f - fl1;
                const float iw1 = 1.0f / w1f, r2f = (float)r2 * 1.0001f;
                const float mg0 = 1e-4f * w0f, mg1 = 1e-4f * w1f;
                int jw = 0;
                for (int j = 0; j < rmax; ++j) {
                    const int ra = j - ls;
                    int ca = -ls, cb = ls;
                    bool rowon = j < nrows;
                    if (prune) {
                        const float dy = fmaxf((ra > 0 ? fh0 + (float)(ra - 1) * w0f : (ra < 0 ? fl0 + (float)(-ra - 1) * w0f : 0.0f)) - mg0, 0.0f);
                        const float rem = r2f - dy * dy;
                        rowon = rowon && rem > 0.0f;
                        const float dxm = sqrtf(fmaxf(rem, 0.0f)) * 1.0001f + mg1;
                        cb = min(ls, max((int)floorf((dxm - fh1) * iw1) + 1, 0));
                        ca = -min(ls, max((int)floorf((dxm - fl1) * iw1) + 1, 0));
                    }
                    int s = 0, e = 0;
                    if (rowon) thr_rect_slots(w, lr, lc, ra, ca, cb, s, e);
                    if (e > s) {
                        GHN_ASSERT(jw < SB_ROWS - 1 && e <= a.cap);
                        myr[jw * TT_THREADS] = (uint32_t)s | ((uint32_t)e << 16);
                        ++jw;
                        n += e - s;
                    }
                }
                myr[jw * TT_THREADS] = SB_SENT;
            }
#pragma unroll
            for (int i = 0; i < SB_NB / 4; ++i) myh[i * TT_THREADS] = 0u;
            const int steps = __reduce_max_sync(GHN_FULL, n);
            // ---- pass 1: histogram of fp32 keys (bucket b: byte b & 3 of word
            // b >> 2).  Branch-free: an idle lane adds 0 to its own word.
            {
                SelWalk wk;
                wk.start(myr_s, need);
                const int kb = SB_F32_SHIFT - bbase;
                for (int it = 0; it < steps; ++it) {
                    GHN_ASSERT(wk.p >= 0 && wk.p <= a.cap);
                    const float2 c = lds_f2(xy_s + 8u * (uint32_t)wk.p);
                    const uint32_t bits = sb_bits32(__fsub_rn(c.x, q0f), __fsub_rn(c.y, q1f));
                    const int b = sb_clamp((int)(bits >> SB_F32_S) + kb, SB_NB - 1);
                    const uint32_t inc = it < n ? __funnelshift_l(0u, 1u, (uint32_t)b << 3) : 0u;
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(myh_s + (((uint32_t)b & 0x3cu) << 8)), "r"(inc)
                                 : "memory");
                    wk.step();
                }
            }
            int bb = 0;
            bool sel = need, reprune = false;
            {   // the bucket where the running count reaches k (all lanes, unrolled: no divergence)
                int cum = 0, cums = 0, wi = -1;
                uint32_t ws = 0u, wprev = 0u, wnext = 0u, last = 0u;
#pragma unroll
                for (int i = 0; i < SB_NB / 4; ++i) {
                    const uint32_t wd = myh[i * TT_THREADS];
                    const int sum = sel_bytesum(wd);
                    const bool hit = wi < 0 && cum + sum >= k;
                    wnext = wi == i - 1 && i > 0 ? wd : wnext;
                    wprev = hit ? last : wprev;
                    wi = hit ? i : wi;
                    ws = hit ? wd : ws;
                    cums = hit ? cum : cums;
                    cum += sum;
                    last = wd;
                }
                // more than 255 candidates: a byte counter may have carried
                // into its neighbour (or out of the word); each carry loses
                // >= 255 from the decoded total, so the total is exact iff none did
                const bool wrap = n > 255 && cum != n;
                int j = 0;
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int c = (int)((ws >> (8 * u)) & 0xffu);
                    const bool past = j == u && cums + c < k;
                    cums += past ? c : 0;
                    j += past ? 1 : 0;
                }
                bb = 4 * max(wi, 0) + j;
                // candidates pass 2 may note: buckets bb - 1, bb, bb + 1 (the
                // margin reaches into the neighbours)
                const uint64_t w3 = ((uint64_t)wnext << 40) | ((uint64_t)ws << 8) | (uint64_t)(wprev >> 24);
                const uint32_t near3 = (uint32_t)(w3 >> (8 * j)) & 0xffffffu;
                const int nnear = sel_bytesum(near3);
                // wrapped counts, the k-th too deep in its bucket, or too many to note
                if (sel && wi < 0 && r2 > 0.0) {   // fewer than k candidates inside the radius: the whole block next
                    reprune = true;
                    sel = false;
                }
                if (sel && (wi < 0 || wrap || k - cums > SB_C || nnear > SB_NOTE)) {
                    { FB_REASON(3); push_fallback(a, qi); }
                    sel = false;
                }
            }
            // ---- pass 2: vote below bb, note the candidates around bucket bb
            uint32_t tlo = 0u, span = 0u, plo = 0u;
            {
                // bucket bb holds the fp32 key bits [x0 << S, (x0 + 1) << S), fp64 d-parts from plo
                const int x0 = bb + bbase - SB_F32_SHIFT;
                const bool inrange = x0 > (16 << SB_MB) && x0 < (240 << SB_MB);   // normal fp32 range
                plo = bb > 0 ? (uint32_t)(bb + bbase) << SB_S : 0u;
                const uint32_t ulps = sel && inrange ? sel_ulps(f32q, q0, q1, thr_lower(plo)) : 0u;
                const uint32_t lo_edge = bb > 0 ? ((uint32_t)x0 << SB_F32_S) - ulps : 0u;
                const uint32_t hi_edge = bb < SB_NB - 1 ? ((uint32_t)(x0 + 1) << SB_F32_S) + ulps : 0xffffffffu;
                if (sel && ulps == 0u) {   // keys outside the fp32 range / queries too far from the data
                    { FB_REASON(10); push_fallback(a, qi); }
                    sel = false;
                }
                tlo = lo_edge;
                span = hi_edge - lo_edge;
            }
            // skip-ahead lanes: block(ls-1) around the centre of q's cell
            SelGeo geo{0.0f, 0.0f, 0.0f, 0.0f};
            if (sel && skipm) {
                const double i0 = 1.0 / (((double)ls - 0.5) * a.w0), i1 = 1.0 / (((double)ls - 0.5) * a.w1);
                geo.s0 = (float)i0;
                geo.s1 = (float)i1;
                geo.o0 = (float)((q0 - ((double)(a.lo0 + cc0) + 0.5) * a.w0) * i0);
                geo.o1 = (float)((q1 - ((double)(a.lo1 + cc1) + 0.5) * a.w1) * i1);
            }
            cnt_t cnv = 0;
            int noted = 0;
            uint32_t geoc = 0u;
            const bool anyskip = __any_sync(GHN_FULL, sel && skipm);
            if (anyskip)
                sel_pass2<true, WIDE>(xy_s, sl_s, myr_s, myh_s, sel, n, steps, q0f, q1f, tlo, span, geo, cnv, noted, geoc);
            else
                sel_pass2<false, WIDE>(xy_s, sl_s, myr_s, myh_s, sel, n, steps, q0f, q1f, tlo, span, geo, cnv, noted, geoc);
            // ---- exact re-keying of the noted candidates (lock-step over the warp's largest count)
            uint32_t Lb[SB_C + 1];
#pragma unroll
            for (int j = 0; j <= SB_C; ++j) Lb[j] = TT_INF;
            cnt_t cnx = 0;
            int nlx = 0, nlist = 0;
            bool chg = geoc != 0u;
            if (sel && noted > SB_NOTE) {   // more boundary members than a lane can note
                { FB_REASON(9); push_fallback(a, qi); }
                sel = false;
            }
            {
                const int nn = sel ? noted : 0;
                const int nmax = __reduce_max_sync(GHN_FULL, nn);
                for (int j = 0; j < nmax; ++j) {
                    const bool on = j < nn;
                    GHN_ASSERT(j < SB_NOTE);
                    const int slot = on ? (int)(myh[j * TT_THREADS] & 0xffffu) : 0;
                    GHN_ASSERT(slot >= 0 && slot < a.cap);
                    const float2 c = w.xy[slot];
                    const uint32_t lab8 = (uint32_t)w.sl[slot];
                    bool insh = false, ingeo = false;
                    if (anyskip) {
                        const float u = geo.u(__fsub_rn(c.x, q0f), __fsub_rn(c.y, q1f));
                        insh = u > SEL_GEO_HI;
                        ingeo = on && skipm && u > SEL_GEO_LO && !insh;
                        if (__any_sync(GHN_FULL, ingeo)) {   // on a boundary of block(ls-1): the point's own cell decides
                            const int64_t e0 = cell_id((double)c.x, a.w0, a.inv0, a.pow2 & 1u) - a.lo0 - cc0;
                            const int64_t e1 = cell_id((double)c.y, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1 - cc1;
                            const int64_t ch = max(e0 < 0 ? -e0 : e0, e1 < 0 ? -e1 : e1);
                            insh = ingeo ? ch >= (int64_t)ls : insh;
                        }
                    }
                    const uint32_t pk = thr_pack(c, q0, q1, (lab8 >> 3) | (insh ? lmask + 1u : 0u), fmask);
                    const bool lowx = on && pk < plo;
                    const bool lst = on && !lowx;
                    cnx += lowx ? (cnt_t)1 << lab8 : (cnt_t)0;
                    nlx += lowx ? 1 : 0;
                    nlist += lst ? 1 : 0;
                    chg |= lowx && insh;
                    thr_bubble(Lb, lst ? pk : TT_INF);
                }
            }
            need = false;
            bool more = false;
            const int nlo = sel_bytesum(cnv) + nlx;
            const int r = k - nlo;
            if (reprune) {
                need = true;
                noprune = true;
            }
            if (sel && r2 > 0.0) {
                // the rows were clipped to the radius sqrt(r2): exact only when the
                // k-th key lies inside it.  Else select again over the whole block.
                const bool ok = nlo < k && r <= nlist && r <= SB_C;
                const uint32_t t0k = thr_pick(Lb, max(r - 1, 0)) & ~fmask;
                if (nlo < k && !(ok && thr_upper(t0k, fmask) < r2)) {
                    FB_REASON(11);   // (a redo, not yet a fallback)
                    sel = false;
                    need = true;
                    noprune = true;
                }
            }
            if (sel) {
                // sure members: at most the histogram's count below bb (< k <=
                // 255), so no byte of cnv carried; the re-keyed ones join only
                // when the total stays below k
                bool stop = false, bad = !(nlo < k && r <= nlist && r <= SB_C);
                cn = cnv + (bad ? (cnt_t)0 : cnx);
                tau = thr_pick(Lb, max(r - 1, 0));
                const uint32_t nx = r < min(nlist, SB_C + 1) ? thr_pick(Lb, r) : TT_INF;
                // the k-th must lie in bucket bb: every candidate pass 2 left
                // out has its exact key at or beyond bb's upper edge
                bad |= bb < SB_NB - 1 && (int)(tau >> SB_S) >= bb + bbase + 1;
                tm = tau & ~fmask;
                upper = thr_upper(tm, fmask);
#pragma unroll
                for (int j = 0; j < SB_C; ++j)
                    if (j < r) {
                        cn += (cnt_t)1 << (8 * (Lb[j] & lmask));
                        chg |= (Lb[j] & (lmask + 1u)) != 0u;
                    }
                l = layers = ls;
                cls = cnt;
                // layer ls filled / changed the buffer, or (skip mode) changed iff a shell member
                const bool changed = !skipm || chg;
                skipm = false;
                stop = !changed;
                // the next listed candidate shares the k-th's d-part: undecidable
                bad |= nx != TT_INF && (nx & ~fmask) == tm;
                if (!bad && a.mode == GHN_MODE_GUARANTEED) {   // layer ls changed: only the bound may stop
                    const double b = __dmul_rn((double)l, a.min_w);
                    const double b2 = __dmul_rn(b, b);
                    if (b2 >= upper) stop = true;
                    else if (b2 > thr_lower(tm)) bad = true;
                }
#ifdef GHN_FB_REASONS
                if (!(nlo < k)) FB_REASON(12);
                else if (!(r <= nlist)) FB_REASON(13);
                else if (!(r <= SB_C)) FB_REASON(14);
                else if (bb < SB_NB - 1 && (int)(tau >> SB_S) >= bb + bbase + 1) FB_REASON(15);
#endif
                if (bad) { FB_REASON(4); push_fallback(a, qi); }
                else if (stop || l >= lmax) fin = true;
                else more = true;
            }
            // ---- later layers, compare-only
            const RectBound rb0 = more ? RectBound(a, q0, q1, cc0, cc1) : RectBound();
            while (__any_sync(GHN_FULL, more)) {
                bool act = false;
                if (more) {
                    ++l;
                    // the whole shell first (one test, no data): beyond the k-th it
                    // cannot change the top-k, wherever the apron ends
                    act = !rb0.shell_beyond(a, l, upper);
                    if (l > a.A && (STATS || act)) {
                        { FB_REASON(5); push_fallback(a, qi); }
                        more = false;
                        act = false;
                    }
                }
                bool lt = false, eq = false;
                int sc = 0;   // all points of shell(l)
                {
                    int rr = 0, p = 0, e = 0;
                    const int nr = 4 * l;
                    if (STATS && more && !act) sc = thr_shell_count(w, lr, lc, l);
                    for (;;) {   // per range only if it may matter
                        while (act && p >= e) {
                            if (rr >= nr) {
                                act = false;
                                break;
                            }
                            int ra, rb, ca, cb;
                            thr_shell_rect(l, rr, ra, rb, ca, cb);
                            ++rr;
                            thr_rect_slots(w, lr, lc, ra, ca, cb, p, e);
                            sc += e - p;
                            if (rb0.beyond(a, ra, rb, ca, cb, upper)) e = p;
                        }
                        if (!__any_sync(GHN_FULL, act)) break;
                        const int pp = act ? p : 0;
                        const uint32_t pk = thr_pack(w.xy[pp], q0, q1, (uint32_t)w.sl[pp] >> 3, fmask);
                        lt |= act && pk < tm;
                        eq |= act && (uint32_t)(pk - tm) <= fmask;
                        p += act ? 1 : 0;
                    }
                }
                if (more && eq) {   // undecidable d-part
                    { FB_REASON(6); push_fallback(a, qi); }
                    more = false;
                }
                if (more) {
                    layers = l;
                    cnt += sc;
                    if (lt) {   // shell(l) changed the top-k: select over block(l)
                        more = false;
                        ls = l;
                        need = true;
                    }
                    if (!lt) {
                        bool stop = a.mode == GHN_MODE_HEURISTIC;
                        if (a.mode == GHN_MODE_GUARANTEED) {
                            const double b = __dmul_rn((double)l, a.min_w);
                            const double b2 = __dmul_rn(b, b);
                            if (b2 >= upper) {
                                stop = true;
                            } else if (b2 > thr_lower(tm)) {
                                { FB_REASON(7); push_fallback(a, qi); }
                                more = false;
                            }
                        }
                        if (more && (stop || l >= lmax)) {
                            more = false;
                            fin = true;
                        }
                    }
                }
            }
            // a lone re-select would hold the whole warp for a block's worth
            // of steps: below SB_REDO lanes the generic kernel is cheaper
            const int nredo = __popc(__ballot_sync(GHN_FULL, need));
            if (need && (nredo < a.sb_redo || cnt > a.sb_recap)) {
                { FB_REASON(8); push_fallback(a, qi); }
                need = false;
            }
        }
        const int64_t points = cnt;   // every layer up to `layers` counted in full
        // ---- vote: top count; a tie is resolved by a third lock-step pass
        int top = 0, ntie = 0, wl = 0;
        if (fin) {
            for (int lab = 0; lab <= (int)lmask; ++lab) {
                const int c = (int)((cn >> (8 * lab)) & 0xffu);
                if (c > top) {
                    top = c;
                    wl = lab;
                    ntie = 1;
                } else if (c == top && c > 0) {
                    ++ntie;
                }
            }
        }
        bool tie = fin && ntie > 1;
        if (__any_sync(GHN_FULL, tie)) {
            // smallest packed member per label (members: d-part <= the k-th's)
            uint32_t mn[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) mn[j] = TT_INF;
            int ra = -ls, p = 0, e = 0;
            if (tie) thr_rect_slots(w, lr, lc, ra, -ls, ls, p, e);
            const int n3 = tie ? cls : 0;
            const int steps3 = __reduce_max_sync(GHN_FULL, n3);
            for (int it = 0; it < steps3; ++it) {
                const bool have = it < n3;
                while (have && p >= e) {
                    ++ra;
                    thr_rect_slots(w, lr, lc, ra, -ls, ls, p, e);
                }
                const int pp = have ? p : 0;
                const uint32_t pk = thr_pack(w.xy[pp], q0, q1, (uint32_t)w.sl[pp] >> 3, fmask);
                const bool mem = have && (pk & ~fmask) <= tm;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (mem && (pk & lmask) == (uint32_t)j) mn[j] = min(mn[j], pk);
                p += have ? 1 : 0;
            }
            if (tie) {
                const uint64_t cn8 = cn;   // 8 label slots whatever the counter width
                uint32_t w1 = TT_INF, w2 = TT_INF;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((int)((cn8 >> (8 * j)) & 0xffu) == top && j <= (int)lmask) w1 = min(w1, mn[j]);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((int)((cn8 >> (8 * j)) & 0xffu) == top && j <= (int)lmask && (uint32_t)j != (w1 & lmask))
                        w2 = min(w2, mn[j]);
                const int lbits = __popc(fmask);
                if ((w2 >> lbits) - (w1 >> lbits) < 2u) {
                    { FB_REASON(9); push_fallback(a, qi); }
                    fin = false;
                } else {
                    wl = (int)(w1 & lmask);
                }
            }
        }
        if (fin) {
            if (a.out_label) a.out_label[qi] = wl;
            if (a.out_conf) a.out_conf[qi] = __ddiv_rn((double)top, (double)k);
            if (STATS) {
                const int cells = thr_block_cells(w, lr, lc, layers);
                if (a.out_stats) {
                    a.out_stats[3 * (int64_t)qi + 0] = layers;
                    a.out_stats[3 * (int64_t)qi + 1] = cells;
                    a.out_stats[3 * (int64_t)qi + 2] = points;
                }
                tot.layers += layers;
                tot.cells += cells;
                tot.points += points;
                tot.n += 1;
            }
        }
    }
}

// ---------------------------------------------------------------- k <= 32, table-driven
// The register-list rounds on the select's machinery: phase A once per query
// in the ordering pass (groups hold queries of similar candidate counts), the
// candidates of block(l*) and of every later shell walked through the lane's
// row table with the branch-free advance, and both clipped to the cells that
// can matter: block(l*) to the expected k-th radius + 5 sigma (verified), a
// later shell to the radius of the current k-th key (exact: a point outside
// it cannot precede the k-th nor share its d-part).
//  A  (per lane) the query and its phase-A word;
//  B  (warp lock-step) block(l*) in batches of 8 candidates per lane, sorted
//     by a network and merged into the list (k <= 2: bubbled);
//  C  (warp lock-step) later layers while some lane continues: the clipped
//     shell's candidates are bubbled into the list; the layer `changed` iff
//     one of them precedes the k-th key it met (explore.py:117);
//  D  the vote (predict.py:29-36) and the outputs.
struct SelClip {
    float fl0, fh0, fl1, fh1, w0f, w1f, iw1, mg0, mg1;
    __device__ __forceinline__ SelClip(const T2Args &a, double q0, double q1, int64_t cc0, int64_t cc1) {
        // q's distance to the faces of its own cell
        w0f = (float)a.w0;
        w1f = (float)a.w1;
        fl0 = (float)(q0 - (double)(a.lo0 + cc0) * a.w0);
        fh0 = w0f - fl0;
        fl1 = (float)(q1 - (double)(a.lo1 + cc1) * a.w1);
        fh1 = w1f - fl1;
        iw1 = 1.0f / w1f;
        mg0 = 1e-4f * w0f;
        mg1 = 1e-4f * w1f;
    }
    // No point of shell(l) can precede a k-th key whose d-part interval ends at
    // `upper`: the nearest face of block(l - 1) lies beyond it.  fp32 with the
    // margins on the safe side (a false "not beyond" only costs the walk).
    __device__ __forceinline__ bool shell_beyond(int l, double upper) const {
        const float d = fminf(fminf(fl0, fh0) + (float)(l - 1) * w0f - mg0, fminf(fl1, fh1) + (float)(l - 1) * w1f - mg1);
        return d > 0.0f && d * d * (1.0f - 1e-4f) > (float)upper * 1.0001f;
    }
    // Columns [ca, cb] (offsets from q's cell, within -+ls) of row offset ra
    // that can hold a point within sqrt(r2f) of q; false: none.  fp32 with
    // margins far above its rounding (r2f is passed inflated): a superset.
    __device__ __forceinline__ bool cols(int ra, int ls, float r2f, int &ca, int &cb) const {
        const float dy =
            fmaxf((ra > 0 ? fh0 + (float)(ra - 1) * w0f : (ra < 0 ? fl0 + (float)(-ra - 1) * w0f : 0.0f)) - mg0, 0.0f);
        const float rem = r2f - dy * dy;
        const float dxm = sqrtf(fmaxf(rem, 0.0f)) * 1.0001f + mg1;
        cb = min(ls, max((int)fminf(floorf((dxm - fh1) * iw1), 64.0f) + 1, 0));
        ca = -min(ls, max((int)fminf(floorf((dxm - fl1) * iw1), 64.0f) + 1, 0));
        return rem > 0.0f;
    }
};

// Packed key of a staged slot through shared-space addresses.
__device__ __forceinline__ uint32_t tab_pack(uint32_t xy_s, uint32_t sl_s, int p, double q0, double q1, uint32_t lmask) {
    return thr_pack(lds_f2(xy_s + 8u * (uint32_t)p), q0, q1, lds_u8(sl_s + (uint32_t)p), lmask);
}

constexpr uint32_t NB_CLOSE = 511u << 13;   // closing word of the neighbour walk's table (slots [0, 511), row 0)

template <int KM, bool STATS, bool NB>
__device__ __forceinline__ void run_rounds_tab(const T2Args &a, const ThrWin &w, uint32_t *rtab, int nrw,
                                               const uint16_t *ord, const uint32_t *info, int *s_grp, int qb, int qe,
                                               int r_lo, int c_lo, ThrTotals &tot) {
    const int k = a.k;
    const uint32_t lmask = NB ? 0u : (uint32_t)a.lmask;   // (neighbours: no label bits, the staged codes are zero)
    uint32_t *myr = rtab + threadIdx.x;   // row-table word j at myr[j * TT_THREADS]
    const uint32_t myr_s = sm_addr(myr), xy_s = sm_addr(w.xy), sl_s = sm_addr(w.sl);
    for (;;) {
        int g0 = 0;   // the next group of 32 (sorted) queries for this warp
        if ((threadIdx.x & 31) == 0) g0 = atomicAdd(s_grp, 32);
        g0 = __shfl_sync(GHN_FULL, g0, 0);
        if (g0 >= qe - qb) break;
        const int qr = g0 + (int)(threadIdx.x & 31);
        bool live = qr < qe - qb;
        const int li = live ? (int)ord[qe - qb - 1 - qr] : 0;   // heaviest groups first
        const uint32_t f = live ? info[li] : 0u;
        int32_t qi = 0;
        double q0 = 0.0, q1 = 0.0;
        int64_t cc0 = 0, cc1 = 0;
        int lr = 0, lc = 0, lmax = 0, l = 0, cnt = 0;
        if (live) {
            qi = a.qorder[qb + li];
            if (a.q_dtype == GHN_F32) {
                const float2 qf = ((const float2 *)a.Q)[qi];
                q0 = (double)qf.x;
                q1 = (double)qf.y;
            } else {
                q0 = ((const double *)a.Q)[2 * (int64_t)qi];
                q1 = ((const double *)a.Q)[2 * (int64_t)qi + 1];
            }
            if (!(f & SEL_LIVE)) {   // centre outside the grid / l* beyond the apron (sel_prep)
                push_fallback(a, qi);
                live = false;
            }
        }
        if (live) {
            cc0 = cell_id(q0, a.w0, a.inv0, a.pow2 & 1u) - a.lo0;
            cc1 = cell_id(q1, a.w1, a.inv1, (a.pow2 >> 1) & 1u) - a.lo1;
            lr = (int)(cc0 - r_lo);
            lc = (int)(cc1 - c_lo);
            lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
            l = (int)((f >> 14) & 7u);
            cnt = (int)(f & 0x3fffu);
            if (2 * l + 2 > nrw) {   // beyond the row table
                push_fallback(a, qi);
                live = false;
            }
        }
        const SelClip clip(a, q0, q1, cc0, cc1);
        // ---- B: block(l) into the list, lock-step
        uint32_t L[KM + 1];
#pragma unroll
        for (int j = 0; j <= KM; ++j) L[j] = TT_INF;
        bool need = live, noprune = false;
        while (__any_sync(GHN_FULL, need)) {
#pragma unroll
            for (int j = 0; j <= KM; ++j) L[j] = need ? TT_INF : L[j];   // (a lane that is done keeps its list)
            // clip block(l), l >= 1, to the expected k-th radius + 5 sigma of the
            // count inside it (checked below; the whole block otherwise)
            double r2 = 0.0;
            if (need && !noprune && l >= 1) {
                const double side = (double)(2 * l + 1);
                const double kest = (double)k * side * side * a.w0 * a.w1 / (3.14159265358979 * (double)max(cnt, 1));
                r2 = kest * (1.0 + 5.0 * rsqrt((double)k));
            }
            int n = 0;
            {
                const int nrows = need ? 2 * l + 1 : 0;
                const int rmax = __reduce_max_sync(GHN_FULL, nrows);
                const float r2f = (float)r2 * 1.0001f;
                int jw = 0;
                for (int j = 0; j < rmax; ++j) {
                    const int ra = j - l;
                    int ca = -l, cb = l;
                    bool rowon = j < nrows;
                    if (r2 > 0.0) rowon = clip.cols(ra, l, r2f, ca, cb) && rowon;
                    int s = 0, e = 0;
                    if (rowon) thr_rect_slots(w, lr, lc, ra, ca, cb, s, e);
                    if (e > s) {
                        GHN_ASSERT(jw < nrw - 1 && e <= a.cap);
                        myr[jw * TT_THREADS] = (uint32_t)s | ((uint32_t)e << 16);
                        ++jw;
                        n += e - s;
                    }
                }
                myr[jw * TT_THREADS] = SB_SENT;
            }
            const int steps = __reduce_max_sync(GHN_FULL, n);
            SelWalk wk;
            wk.start(myr_s, need);
            // batches of 8 candidates per lane: sorted by a 19-comparator network,
            // then merged into the list (NetMerge8: 41 comparators at k = 16)
            for (int it = 0; it < steps; it += 8) {
                uint32_t bt[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    GHN_ASSERT(wk.p >= 0 && wk.p <= a.cap);
                    const uint32_t pk = tab_pack(xy_s, sl_s, wk.p, q0, q1, lmask);
                    bt[u] = it + u < n ? pk : TT_INF;
                    wk.step();
                }
                if constexpr (KM <= 2) {   // a list of 2-3: the bubble is cheaper than sort + merge
#pragma unroll
                    for (int u = 0; u < 8; ++u) thr_bubble(L, bt[u]);
                } else {
                    net_sort8(bt);
                    NetMerge8<KM + 1>::run(L, bt);
                }
            }
            if (need && r2 > 0.0) {
                // clipped rows: exact only when the k-th key lies inside the radius
                const uint32_t tk = thr_pick(L, k - 1);
                need = !(tk != TT_INF && thr_upper(tk & ~lmask, lmask) < r2);
                noprune = true;
            } else {
                need = false;
            }
        }
        int layers = l;
        int64_t points = cnt;
        // stop rules after layer l* (it filled the buffer: changed)
        if (live && cnt >= k && a.mode == GHN_MODE_GUARANTEED) {
            const double b = __dmul_rn((double)l, a.min_w);
            const double b2 = __dmul_rn(b, b);
            const uint32_t tk = thr_pick(L, k - 1) & ~lmask;
            if (b2 >= thr_upper(tk, lmask)) {
                lmax = l;   // stop
            } else if (b2 > thr_lower(tk)) {
                push_fallback(a, qi);
                live = false;
            }
        }
        bool more = live && l < lmax;   // continues with layer l + 1
        bool fin = live && !more;       // answered after layer l
        // ---- C (tab): later layers
        while (__any_sync(GHN_FULL, more)) {
            uint32_t tm = 0;
            double upper = 0.0;
            bool act = false;
            if (more) {
                ++l;
                tm = thr_pick(L, k - 1) & ~lmask;
                upper = thr_upper(tm, lmask);
                // the whole shell first (one test, no data): beyond the k-th it
                // cannot change the top-k, wherever the apron ends
                act = !clip.shell_beyond(l, upper);
                if (l > a.A && (STATS || act)) {
                    push_fallback(a, qi);
                    more = false;
                    act = false;
                }
            }
            // the shell's ranges within sqrt(upper) of q -> the lane's table
            int n = 0;
            bool over = false;
            {
                const int nrows = act ? 2 * l + 1 : 0;
                const int rmax = __reduce_max_sync(GHN_FULL, nrows);
                const float r2f = (float)upper * 1.0001f;
                int jw = 0;
                for (int j = 0; j < rmax; ++j) {
                    const int ra = j - l;
                    int ca = -l, cb = l;
                    const bool rowon = clip.cols(ra, l, r2f, ca, cb) && j < nrows;
                    const bool edge = ra == -l || ra == l;
                    // an inner row contributes its end cells only
                    int s0 = 0, e0 = 0, s1 = 0, e1 = 0;
                    if (rowon && (edge || ca == -l)) thr_rect_slots(w, lr, lc, ra, ca, edge ? cb : ca, s0, e0);
                    if (rowon && !edge && cb == l) thr_rect_slots(w, lr, lc, ra, cb, cb, s1, e1);
                    if (e0 > s0) {
                        if (jw < nrw - 1) myr[jw * TT_THREADS] = (uint32_t)s0 | ((uint32_t)e0 << 16);
                        ++jw;
                        n += e0 - s0;
                    }
                    if (e1 > s1) {
                        if (jw < nrw - 1) myr[jw * TT_THREADS] = (uint32_t)s1 | ((uint32_t)e1 << 16);
                        ++jw;
                        n += e1 - s1;
                    }
                }
                over = jw > nrw - 1;
                myr[min(jw, nrw - 1) * TT_THREADS] = SB_SENT;
            }
            if (over) {   // more ranges than the table holds
                push_fallback(a, qi);
                more = false;
                act = false;
                n = 0;
            }
            bool lt = false, eq = false;
            {
                const int steps = __reduce_max_sync(GHN_FULL, n);
                SelWalk wk;
                wk.start(myr_s, act);
                uint32_t lk1 = thr_pick(L, k);   // a candidate at or beyond the (k+1)-th leaves L[0..k] alone
                for (int it = 0; it < steps; ++it) {
                    const bool have = it < n;
                    GHN_ASSERT(wk.p >= 0 && wk.p <= a.cap);
                    const uint32_t pk = tab_pack(xy_s, sl_s, wk.p, q0, q1, lmask);
                    lt |= have && pk < tm;
                    eq |= have && (uint32_t)(pk - tm) <= lmask;
                    const bool ins = have && pk < lk1;
                    if (__any_sync(GHN_FULL, ins)) {
                        thr_bubble(L, ins ? pk : TT_INF);
                        lk1 = thr_pick(L, k);
                    }
                    wk.step();
                }
            }
            if (more && eq) {   // a shell point shares the k-th key's d-part
                push_fallback(a, qi);
                more = false;
            }
            if (more) {
                layers = l;
                if (STATS) points += thr_shell_count(w, lr, lc, l);
                bool stop = !lt && a.mode == GHN_MODE_HEURISTIC;
                if (a.mode == GHN_MODE_GUARANTEED) {
                    const double b = __dmul_rn((double)l, a.min_w);
                    const double b2 = __dmul_rn(b, b);
                    const uint32_t tk = thr_pick(L, k - 1) & ~lmask;
                    if (b2 >= thr_upper(tk, lmask)) {
                        stop = true;
                    } else if (b2 > thr_lower(tk)) {
                        push_fallback(a, qi);
                        more = false;
                    }
                }
                if (more && (stop || l >= lmax)) {
                    more = false;
                    fin = true;
                }
            }
        }
        // ---- D (tab), neighbours (explore.py:132-137): the members are the
        // candidates of block(layers) whose d-part does not exceed the k-th's
        // (exactly k when the (k+1)-th has another d-part).  They are walked
        // once more -- rows clipped to the k-th radius -- and written with their
        // exact keys and CSR slots, unordered; nb_sort_kernel maps the slots to
        // point indices, orders each row by (key, index) and takes the square roots.
        if constexpr (NB) {
            const uint32_t tau = fin ? thr_pick(L, k - 1) : 0u, nx = fin ? thr_pick(L, k) : TT_INF;
            if (fin && nx != TT_INF && (nx & ~lmask) == (tau & ~lmask)) {
                push_fallback(a, qi);
                fin = false;
            }
            const uint32_t tm = tau & ~lmask;
            // The members lie in the layers whose data was read: a last layer beyond
            // the apron was only visited because it provably holds none.
            const int le = min(layers, a.A);
            // table words of this walk: first slot (13 bits) | length (9) | window row (7)
            int n = 0;
            {
                const int nrows = fin ? 2 * le + 1 : 0;
                const int rmax = __reduce_max_sync(GHN_FULL, nrows);
                const float r2f = (float)thr_upper(tm, lmask) * 1.0001f;
                int jw = 0;
                bool toolong = false;
                for (int j = 0; j < rmax; ++j) {
                    const int ra = j - le;
                    int ca = -le, cb = le;
                    const bool rowon = clip.cols(ra, le, r2f, ca, cb) && j < nrows;
                    int s0 = 0, e0 = 0;
                    if (rowon) thr_rect_slots(w, lr, lc, ra, ca, cb, s0, e0);
                    if (e0 > s0) {
                        GHN_ASSERT(jw < nrw - 1 && lr + ra >= 0 && lr + ra < 128);
                        toolong |= e0 - s0 > 511;
                        myr[jw * TT_THREADS] = (uint32_t)s0 | ((uint32_t)(e0 - s0) << 13) | ((uint32_t)(lr + ra) << 22);
                        ++jw;
                        n += e0 - s0;
                    }
                }
                myr[jw * TT_THREADS] = NB_CLOSE;   // closes the table: slots [0, 511) of row 0, entered again and again
                if (fin && toolong) {   // (a row of more than 511 candidates inside the k-th radius)
                    push_fallback(a, qi);
                    fin = false;
                    n = 0;
                }
            }
            const int steps = __reduce_max_sync(GHN_FULL, n);
            uint32_t tp = myr_s;
            uint32_t wd = fin ? lds_u32(tp) : NB_CLOSE;
            int p = (int)(wd & 0x1fffu), e = p + (int)((wd >> 13) & 0x1ffu), dlt = w.delta[wd >> 22];
            tp += wd != NB_CLOSE ? TT_THREADS * 4 : 0;   // (the prefetch never passes the closing word)
            uint32_t nxw = lds_u32(tp);
            int m = 0;   // members written
            for (int it = 0; it < steps; ++it) {
                GHN_ASSERT(p >= 0 && p <= a.cap);
                const float2 c = lds_f2(xy_s + 8u * (uint32_t)p);
                const uint32_t pk = thr_pack(c, q0, q1, 0u, lmask);
                const bool mem = it < n && pk <= tm;
                if (__any_sync(GHN_FULL, mem)) {
                    if (mem && m < k) {
                        // (the CSR slot; nb_sort_kernel turns it into the point index: a
                        // dependent global load here would stall the lock-step walk)
                        a.out_dist[(int64_t)qi * k + m] = thr_key(c, q0, q1);
                        a.out_idx[(int64_t)qi * k + m] = (int64_t)(p + dlt);
                    }
                    m += mem ? 1 : 0;
                }
                // the walk (SelWalk with this table's word format); a lane past its
                // rows idles over the closing word's slots
                p = min(p + 1, a.cap);
                const bool adv = p >= e;
                if (__any_sync(GHN_FULL, adv)) {
                    const uint32_t wn = adv ? nxw : wd;
                    wd = wn;
                    p = adv ? (int)(wn & 0x1fffu) : p;
                    e = adv ? p + (int)((wn >> 13) & 0x1ffu) : e;
                    dlt = adv ? w.delta[wn >> 22] : dlt;
                    tp += adv && wn != NB_CLOSE ? TT_THREADS * 4 : 0;
                    nxw = lds_u32(tp);
                }
            }
            if (fin && m != k) {   // (cannot happen with a clean k-th boundary; the generic kernel decides)
                push_fallback(a, qi);
                fin = false;
            }
            if (fin && STATS) {
                const int cells = thr_block_cells(w, lr, lc, layers);
                if (a.out_stats) {
                    a.out_stats[3 * (int64_t)qi + 0] = layers;
                    a.out_stats[3 * (int64_t)qi + 1] = cells;
                    a.out_stats[3 * (int64_t)qi + 2] = points;
                }
                tot.layers += layers;
                tot.cells += cells;
                tot.points += points;
                tot.n += 1;
            }
            fin = false;   // (nothing left for the vote below)
        }
        // ---- D (tab): vote and outputs
        if (fin) {
            const uint32_t tau = thr_pick(L, k - 1), nx = thr_pick(L, k);
            int wl, top;
            if ((nx != TT_INF && (nx & ~lmask) == (tau & ~lmask)) || !thr_vote<KM>(L, k, lmask, wl, top, lmask)) {
                push_fallback(a, qi);
            } else {
                if (a.out_label) a.out_label[qi] = wl;
                if (a.out_conf) a.out_conf[qi] = __ddiv_rn((double)top, (double)k);
                if (STATS) {
                    const int cells = thr_block_cells(w, lr, lc, layers);
                    if (a.out_stats) {
                        a.out_stats[3 * (int64_t)qi + 0] = layers;
                        a.out_stats[3 * (int64_t)qi + 1] = cells;
                        a.out_stats[3 * (int64_t)qi + 2] = points;
                    }
                    tot.layers += layers;
                    tot.cells += cells;
                    tot.points += points;
                    tot.n += 1;
                }
            }
        }
    }
}

template <int KM, bool STATS, bool NB = false>
__device__ __forceinline__ void tile2d_thr_body(const T2Args &a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int s_P;
    const int t = blockIdx.x;
    const int qb = a.tile_start[t], qe = a.tile_start[t + 1];
    if (qb == qe) return;
    const int t0 = t / a.nt1, t1 = t - (t / a.nt1) * a.nt1;
    const int r_lo = max(t0 * a.T - a.A, 0), r_hi = min(t0 * a.T + a.T - 1 + a.A, a.ext0 - 1);
    const int c_lo = max(t1 * a.T - a.A, 0), c_hi = min(t1 * a.T + a.T - 1 + a.A, a.ext1 - 1);
    const int R = r_hi - r_lo + 1, W = c_hi - c_lo + 1, W1 = W + 1;
    float2 *sxy = (float2 *)sm;
    uint8_t *sl = (uint8_t *)(sxy + a.cap);
    int32_t *loc = (int32_t *)(sl + a.cap);                        // [R][W+1]
    int32_t *delta = loc + a.win * (a.win + 1);                    // [R]
    int32_t *rstart = delta + a.win;                               // [R+1]
    for (int e = threadIdx.x; e < R * W1; e += blockDim.x) {
        const int i = e / W1, j = e - (e / W1) * W1;
        loc[e] = a.pt_off[(int64_t)(r_lo + i) * a.ext1 + c_lo + j];
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // row prefix by one warp, 32 rows at a time
        int carry = 0;
        for (int i0 = 0; i0 < R; i0 += 32) {
            const int i = i0 + (int)threadIdx.x;
            const int len = i < R ? loc[i * W1 + W] - loc[i * W1] : 0;
            const int inc = warp_inclusive_scan(len);
            if (i < R) {
                rstart[i] = carry + inc - len;
                delta[i] = loc[i * W1] - (carry + inc - len);
            }
            carry += __shfl_sync(GHN_FULL, inc, 31);
        }
        if (threadIdx.x == 0) {
            rstart[R] = carry;
            s_P = carry;
        }
    }
    __syncthreads();
    const int P = s_P;
    if (P > a.cap) {
        for (int qq = qb + threadIdx.x; qq < qe; qq += blockDim.x) push_fallback(a, a.qorder[qq]);
        return;
    }
    for (int e = threadIdx.x; e < R * W1; e += blockDim.x) loc[e] -= delta[e / W1];
    // (measured and not kept, cfg4 sweep 13.7 ms: coordinates by 4-byte cp.async
    // into the float2 slots with the labels four loads deep -- 14.1 ms; rows'
    // ends fetched and scanned by warp 0 beside the offset loads, one barrier
    // fewer -- 14.3 ms.  Rows start at arbitrary slots, so 16-byte bulk copies
    // do not apply without a 12-byte-per-point SoA staging that costs a CTA per SM.)
    for (int i = threadIdx.x >> 5; i < R; i += TT_THREADS / 32) {   // warp per row: coalesced copy
        const int p0 = rstart[i], p1 = rstart[i + 1], d = delta[i];
        for (int p = p0 + (int)(threadIdx.x & 31); p < p1; p += 32) {
            sxy[p] = make_float2(__ldg(a.c0 + p + d), __ldg(a.c1 + p + d));
            // the bucket select keeps label code * 8: its vote is one shift and one add
            sl[p] = NB ? (uint8_t)0 : (uint8_t)(KM == 0 ? __ldg(a.labels_perm + p + d) << 3 : __ldg(a.labels_perm + p + d));
        }
    }
    __syncthreads();
    const ThrWin w{sxy, sl, loc, R, W, W1, rstart, delta};
    ThrTotals tot{0, 0, 0, 0};
    if constexpr (KM > 0 && GHN_TT_TAB) {
        // table-driven rounds (run_rounds_tab): the sort's scratch lives in the row tables
        __shared__ uint16_t s_ord[SB_SORT_N];
        __shared__ uint32_t s_info[SB_SORT_N];
        __shared__ int s_grp;
        uint32_t *rtab = (uint32_t *)(rstart + a.win + 1);
        const int nrw = 2 * a.A + 2;
        for (int c0 = qb; c0 < qe; c0 += SB_SORT_N) {
            const int c1 = min(c0 + SB_SORT_N, qe);
            if (threadIdx.x == 0) s_grp = 0;
            sel_sort_chunk(a, w, c0, c1, t0, t1, r_lo, c_lo, (int *)rtab, (uint16_t *)(rtab + 512), s_ord, s_info, false,
                           KM > GHN_TT_NOSORT_KM);
            run_rounds_tab<KM == 0 ? 1 : KM, STATS, NB>(a, w, rtab, nrw, s_ord, s_info, &s_grp, c0, c1, r_lo, c_lo, tot);
            __syncthreads();
        }
    } else if constexpr (KM > 0 && KM <= 2) {   // k <= 2: each lane on its own loop
        for (int qq = qb + (int)threadIdx.x; qq < qe; qq += TT_THREADS)
            process_query_thr<KM, STATS>(a, w, a.qorder[qq], t0, t1, r_lo, c_lo, tot);
    } else if constexpr (KM == 0) {
        // the sort's counters and (key, rank) pairs live in the histogram area
        // (free until the rounds start); the order and the per-query phase-A
        // words stay beside it
        __shared__ uint16_t s_ord[SB_SORT_N];
        __shared__ uint32_t s_info[SB_SORT_N];
        __shared__ int s_grp;
        // (the row tables first: the walk's prefetch may read one word past a lane's table)
        uint32_t *rtab = (uint32_t *)(rstart + a.win + 1);
        uint32_t *hist = rtab + SB_ROWS * TT_THREADS;
        for (int c0 = qb; c0 < qe; c0 += SB_SORT_N) {
            const int c1 = min(c0 + SB_SORT_N, qe);
            if (threadIdx.x == 0) s_grp = 0;
            sel_sort_chunk(a, w, c0, c1, t0, t1, r_lo, c_lo, (int *)hist, (uint16_t *)(hist + 512), s_ord, s_info, true);
            if (a.lmask > 3)
                run_rounds_sel<STATS, true>(a, w, hist, rtab, s_ord, s_info, &s_grp, c0, c1, t0, t1, r_lo, c_lo, tot);
            else
                run_rounds_sel<STATS, false>(a, w, hist, rtab, s_ord, s_info, &s_grp, c0, c1, t0, t1, r_lo, c_lo, tot);
            __syncthreads();
        }
    } else {
        __shared__ uint16_t s_ord[TT_SORT];
        __shared__ int s_grp;
        for (int c0 = qb; c0 < qe; c0 += TT_SORT) {
            const int c1 = min(c0 + TT_SORT, qe);
            if (threadIdx.x == 0) s_grp = 0;
            for (int i = threadIdx.x; i < c1 - c0; i += TT_THREADS) s_ord[i] = (uint16_t)i;
            __syncthreads();
            run_rounds_thr<KM, STATS>(a, w, s_ord, &s_grp, c0, c1, t0, t1, r_lo, c_lo, tot);
            __syncthreads();
        }
    }
    if (STATS && a.totals) {
        const unsigned long long v0 = warp_sum(tot.layers), v1 = warp_sum(tot.cells), v2 = warp_sum(tot.points),
                                 v3 = warp_sum(tot.n);
        if ((threadIdx.x & 31) == 0 && v3) {
            atomicAdd(&a.totals[0], v0);
            atomicAdd(&a.totals[1], v1);
            atomicAdd(&a.totals[2], v2);
            atomicAdd(&a.totals[3], v3);
        }
    }
}

// k <= 32 (register list): four CTAs per SM up to k = 4, GHN_TT_MINB16 for
// k = 5-16, two for k = 17-32.
#ifndef GHN_TT_MINB16
#define GHN_TT_MINB16 3
#endif
template <int KM, bool STATS>
__global__ void __launch_bounds__(TT_THREADS, KM <= 4 ? 4 : (KM <= 16 ? GHN_TT_MINB16 : 2)) tile2d_thr_kernel(const T2Args a) {
    tile2d_thr_body<KM, STATS>(a);
}

// The same rounds returning the neighbours (knn_query_batch): unordered rows
// of (exact key, CSR slot), finished by nb_sort_kernel.
template <int KM, bool STATS>
__global__ void __launch_bounds__(TT_THREADS, KM <= 4 ? 4 : (KM <= 16 ? GHN_TT_MINB16 : 2)) tile2d_nb_kernel(const T2Args a) {
    tile2d_thr_body<KM, STATS, true>(a);
}

// One row of k (key, CSR slot) pairs per group of P = 2^ceil(log2 k) lanes:
// point index = perm[slot], then a bitonic sort by (key, index) -- the reference's lexsort order,
// explore.py:114 -- then distance = sqrt(key) (core.py:88-91).
__global__ void __launch_bounds__(256) nb_sort_kernel(double *__restrict__ dist, int64_t *__restrict__ idx, int64_t nq, int k,
                                                      int P, const int32_t *__restrict__ perm, int64_t n) {
    const int lane = (int)(threadIdx.x & 31), sub = lane & (P - 1);
    const int64_t per_warp = 32 / P;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t q = warp * per_warp + lane / P;
    const bool on = q < nq && sub < k;
    double key = on ? dist[q * k + sub] : __longlong_as_double(0x7ff0000000000000LL);
    long long id = on ? idx[q * k + sub] : 0x7fffffffffffffffLL;
    // CSR slot -> point index (rows the tile kernel left to the generic kernel hold anything)
    if (on && id >= 0 && id < n) id = (long long)__ldg(perm + id);
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const double ok = __shfl_xor_sync(GHN_FULL, key, stride);
            const long long oi = __shfl_xor_sync(GHN_FULL, id, stride);
            const bool up = (sub & size) == 0;            // ascending half
            const bool lower = (sub & stride) == 0;       // keeps the smaller of the pair when ascending
            const bool mine_first = key < ok || (key == ok && id < oi);
            const bool keep = (lower == up) ? mine_first : !mine_first;
            key = keep ? key : ok;
            id = keep ? id : oi;
        }
    if (on) {
        dist[q * k + sub] = __dsqrt_rn(key);
        idx[q * k + sub] = id;
    }
}

// k > 32 (bucket select): three CTAs per SM (<= 80 registers).
template <bool STATS>
__global__ void __launch_bounds__(TT_THREADS, 3) tile2d_sel_kernel(const T2Args a) {
    tile2d_thr_body<0, STATS>(a);
}

}  // namespace
}  // namespace ghn
