// ghn_tile2d.cu -- thread-per-query tiled predict for 2-D DENSE grids (sm_100a).
//
// The same results as query_kernel (explore.py:66-137 + predict.py:20-36),
// organised for throughput:
//   * queries are counting-sorted by a tile of T x T cells around their
//     central cell (K8 binning); one CTA per tile stages the tile plus an
//     apron of A layers -- coordinates (SoA fp32) and permuted labels -- in
//     shared memory with coalesced row copies (one CSR row = one contiguous
//     slot range);
//   * one THREAD per query walks the Chebyshev shells over the staged cells;
//   * the k-th (key, index) pair is found by a per-thread radix select over
//     fp64 keys (32-bucket histograms on the monotone fp32 round-down of the
//     key, re-bucketing until the boundary bucket holds <= 8 candidates,
//     which are then ordered exactly) -- counting passes instead of a
//     sorted insert per candidate;
//   * the heuristic stop tests "some layer-l point precedes the current
//     k-th" (equivalent to explore.py:117 `changed`), the guaranteed stop
//     compares (l * min_w)^2 with the k-th key (explore.py:124-127);
//   * the vote keeps per-label counts and the label's nearest member under
//     (sqrt(key), index) (predict.py:29-35).
// Queries whose centre is outside the grid, that need more than A layers,
// whose tile overflows shared memory, whose boundary bucket cannot be split
// (exact duplicate keys) or that meet more than T2_NL labels are appended to
// a fallback list and answered by the generic warp-per-query kernel.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "ghn_common.cuh"
#include "ghn_tile2d.cuh"

namespace ghn {
namespace {

constexpr int T2_THREADS = 256;
constexpr int T2_NB = 32;        // histogram buckets per select round
constexpr int T2_SMALL = 4;      // boundary candidates ordered exactly
constexpr int T2_NL = 4;         // distinct labels tracked by the vote
constexpr int T2_CAP = 4096;     // staged points per tile
constexpr int TT_KMAX = 255;     // thread-per-query kernel: largest k (8-bit vote counters)
constexpr int TT_LIST_KMAX = 32; // largest k on the register list; above: bucket select
constexpr double TT_Q = 256.0;   // thread-per-query kernel: queries per tile
constexpr double TT_CAP = 8192.0;
#ifndef T2_EXT_MAXK
#define T2_EXT_MAXK 16     // k at or below which phase-1 selects extract
#endif
#ifndef T2_MINB
#define T2_MINB 4
#endif

struct T2Args {
    int64_t n;
    int32_t ext0, ext1;
    int64_t lo0, lo1;
    double w0, w1, inv0, inv1, min_w;
    uint32_t pow2;
    const float *c0;
    const float *c1;
    const int32_t *pt_off;
    const int32_t *perm;
    const int32_t *labels_perm;
    const void *Q;
    int32_t q_dtype;
    int32_t k;
    int32_t mode;
    const int32_t *qorder;
    const int32_t *tile_start;
    int32_t T, A, nt0, nt1, win, cap;
    int32_t *out_label;
    double *out_conf;
    double *out_dist;    // neighbours (tile2d_nb_kernel): (nq, k) exact keys, then distances
    int64_t *out_idx;    //                                (nq, k) point indices
    int64_t *out_stats;
    unsigned long long *totals;
    int32_t *fb_list;
    int32_t *fb_count;
    int32_t dbg;
    int32_t small_labels;
    int32_t lmask;   // label-code mask of the thread kernel (2^LB - 1)
    int32_t sb_capn, sb_redo, sb_wmax, sb_sort, sb_recap;   // bucket-select lock-step knobs (see ghn_tile2d_thr.cuh)
    double tt_skipf;   // k = 3, 4 rounds: skip-ahead threshold (fraction of the block half-width)
    int32_t tt_tab;    // k <= 32: table-driven rounds (run_rounds_tab)
    double sb_skipf;   // bucket select: skip ahead when the expected k-th radius exceeds this fraction of the block half-width
};

struct Win {
    const float *sx;
    const float *sy;
    const int32_t *sp;      // staged point index (perm) -- tile2d_kernel only
    const uint8_t *sl;      // staged label code          -- tile2d_kernel only
    const int32_t *loc;     // (R, W+1) local slot of each cell start
    const int32_t *delta;   // global slot = local + delta[row]
    int R, W, W1;
};

// --------------------------------------------------------------- per warp
// One warp answers one query at a time; lanes cover candidates.  A query's
// candidate set is a short list of contiguous staged ranges (the rows of
// the block around its cell, or the row segments / side cells of a shell),
// held one range per lane and flattened by an inclusive scan.
struct Ranges {
    int s;      // this lane's range start (staged index)
    int n;      // its length
    int incl;   // inclusive prefix of lengths over lanes
    int total;  // warp-uniform
};

__device__ __forceinline__ void ranges_finish(Ranges &rg) {
    rg.incl = warp_inclusive_scan(rg.n);
    rg.total = __shfl_sync(GHN_FULL, rg.incl, 31);
}

// Block(l): rows lr-l..lr+l, columns lc-l..lc+l (clipped), one row per lane.
__device__ __forceinline__ Ranges block_ranges(const Win &w, int lr, int lc, int l) {
    const int lane = lane_id();
    Ranges rg{0, 0, 0, 0};
    const int i = lr - l + lane;
    if (lane <= 2 * l && i >= 0 && i < w.R) {
        const int a = max(lc - l, 0), b = min(lc + l, w.W - 1);
        const int32_t *rp = w.loc + i * w.W1;
        rg.s = rp[a];
        rg.n = rp[b + 1] - rg.s;
    }
    ranges_finish(rg);
    return rg;
}

// Shell(l), l >= 1: lanes 0/1 the full rows lr -+ l, lanes 2.. the side cells
// lc -+ l of the rows in between (4l ranges, <= 32 for l <= 8).
__device__ __forceinline__ Ranges shell_ranges(const Win &w, int lr, int lc, int l) {
    const int lane = lane_id();
    Ranges rg{0, 0, 0, 0};
    if (lane < 4 * l) {
        int row, a, b;
        if (lane < 2) {
            row = lane == 0 ? lr - l : lr + l;
            a = max(lc - l, 0);
            b = min(lc + l, w.W - 1);
        } else {
            row = lr - l + 1 + ((lane - 2) >> 1);
            a = b = ((lane - 2) & 1) ? lc + l : lc - l;
        }
        if (row >= 0 && row < w.R && a >= 0 && b < w.W && a <= b) {
            const int32_t *rp = w.loc + row * w.W1;
            rg.s = rp[a];
            rg.n = rp[b + 1] - rg.s;
        }
    }
    ranges_finish(rg);
    return rg;
}

// Candidate m = base + lane of the flattened ranges -> staged index.
__device__ __forceinline__ bool ranges_at(const Ranges &rg, int m, int &p) {
    int L = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        const int v = __shfl_sync(GHN_FULL, rg.incl, L + step - 1);
        if (v <= m) L += step;
    }
    L = L > 31 ? 31 : L;
    const int exL = __shfl_sync(GHN_FULL, rg.incl - rg.n, L);
    const int sL = __shfl_sync(GHN_FULL, rg.s, L);
    p = sL + (m - exL);
    return m < rg.total;
}

__device__ __forceinline__ double key2(const Win &w, int p, double q0, double q1) {
    // numpy einsum order for d = 2: lane0 = d0^2, lane1 = d1^2, key = lane0 + lane1
    const double d0 = __dsub_rn((double)w.sx[p], q0);
    const double d1 = __dsub_rn((double)w.sy[p], q1);
    return __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
}

struct Kth {
    double key;
    int32_t idx;
};

// Per-warp shared scratch.
struct WarpScratch {
    int hist[32];
    int lcnt[32];     // vote counters when every label code is in [0, 32)
    double bkey[32];
    int32_t bidx[32];
    int32_t bg[32];
};

// Warp vote table: lane j holds label j's count (labels in first-met order).
struct VoteW {
    int32_t lab;    // this lane's label (valid for lane < used)
    int32_t cnt;
    int32_t used;   // warp-uniform
    bool overflow;  // warp-uniform
};

// Add the member lanes (mask) with labels L to the table.
__device__ __forceinline__ void vote_lanes(VoteW &v, unsigned members, int32_t L) {
    const int lane = lane_id();
    while (members) {
        const int src = __ffs(members) - 1;
        const int32_t lab = __shfl_sync(GHN_FULL, L, src);
        const unsigned same = __ballot_sync(GHN_FULL, ((members >> lane) & 1u) && L == lab);
        members &= ~same;
        const int c = __popc(same);
        const unsigned hit = __ballot_sync(GHN_FULL, lane < v.used && v.lab == lab);
        if (hit) {
            if (lane == __ffs(hit) - 1) v.cnt += c;
        } else if (v.used < 32) {
            if (lane == v.used) {
                v.lab = lab;
                v.cnt = c;
            }
            ++v.used;
        } else {
            v.overflow = true;
        }
    }
}

__device__ __forceinline__ bool lt_pair(double ka, int32_t ia, double kb, int32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// A candidate set: the flattened ranges of a block; keys are recomputed
// from the staged coordinates on every pass (cheaper than holding them:
// this kernel is latency-bound and occupancy-limited).
struct Cands {
    const Win *w;
    const Ranges *rg;
    double q0, q1;
    int nch;   // warp-uniform number of 32-candidate chunks
    // candidate i*32 + lane: key and staged index (-1 = absent)
    __device__ __forceinline__ void at(int i, double &key, int32_t &g) const {
        int p;
        key = INFINITY;
        g = -1;
        if (ranges_at(*rg, i * 32 + lane_id(), p)) {
            key = key2(*w, p, q0, q1);
            g = p;
        }
    }
};

__device__ __forceinline__ Cands make_cands(const Win &w, const Ranges &rg, double q0, double q1) {
    Cands c;
    c.w = &w;
    c.rg = &rg;
    c.q0 = q0;
    c.q1 = q1;
    c.nch = (rg.total + 31) >> 5;
    return c;
}

// Count member lanes into the vote: shared counters when labels are small
// codes, else the general per-lane table.
__device__ __forceinline__ void vote_members(const Win &w, WarpScratch &sc, VoteW &v, bool small,
                                             bool member, int32_t g) {
    const unsigned mem = __ballot_sync(GHN_FULL, member);
    if (!mem) return;
    const int32_t L = member ? (int32_t)w.sl[g] : -1;
    if (small) {
        if (member) {
            const unsigned grp = __match_any_sync(mem, L);
            if ((grp & lanemask_lt()) == 0) atomicAdd(&sc.lcnt[L], __popc(grp));
        }
    } else {
        vote_lanes(v, mem, L);
    }
}

// Radix select over cached candidates with key in [lo, hi]: the r-th smallest
// (key, index) and the vote over the r members.  Level-1 buckets on the
// monotone fp32 round-down of the key (32 buckets, one per lane), a level-2
// split of the boundary bucket when it holds more than 32, then the boundary
// candidates are ranked exactly.  False = cannot resolve.
__device__ __forceinline__ bool select_vote_c(const T2Args &a, WarpScratch &sc, const Cands &c, int r,
                                              double lo, double hi, Kth &out, VoteW &v,
                                              int32_t og0 = 0, int32_t og1 = 0x7fffffff,
                                              bool *outside = nullptr) {
    const int lane = lane_id();
    const bool small = a.small_labels != 0;
    const float flo = __double2float_rd(lo);
    const float fhi = __double2float_ru(hi);
    const float sc1 = fhi > flo ? fminf(32.0f * __frcp_rn(fhi - flo), 1e30f) : 0.0f;
#define T2_B1(k32) min((int)(((k32) - flo) * sc1), 31)
    sc.hist[lane] = 0;
    sc.lcnt[lane] = 0;
    __syncwarp();
    for (int i = 0; i < c.nch; ++i) {
        {
            double ckey;
            int32_t cgs;
            c.at(i, ckey, cgs);
            const bool in = cgs >= 0 && ckey >= lo && ckey <= hi;
            const int b = in ? T2_B1(__double2float_rd(ckey)) : -1;
            const unsigned im = __ballot_sync(GHN_FULL, in);
            if (in) {
                const unsigned grp = __match_any_sync(im, b);
                if ((grp & lanemask_lt()) == 0) atomicAdd(&sc.hist[b], __popc(grp));
            }
        }
    }
    __syncwarp();
    int cnt = sc.hist[lane];
    int incl = warp_inclusive_scan(cnt);
    unsigned ge = __ballot_sync(GHN_FULL, incl >= r);
    if (!ge) return false;
    const int bs1 = __ffs(ge) - 1;
    int m = __shfl_sync(GHN_FULL, cnt, bs1);
    r -= __shfl_sync(GHN_FULL, incl - cnt, bs1);
    int bs2 = -1;
    float lo2 = 0.0f, sc2 = 0.0f;
    if (m > 32) {
        lo2 = flo + (float)bs1 / sc1;
        sc2 = fminf(sc1 * 32.0f, 1e30f);
#define T2_B2(k32) max(0, min((int)(((k32) - lo2) * sc2), 31))
        __syncwarp();
        sc.hist[lane] = 0;
        __syncwarp();
        for (int i = 0; i < c.nch; ++i) {
            {
                double ckey;
                int32_t cgs;
                c.at(i, ckey, cgs);
                bool in = cgs >= 0 && ckey >= lo && ckey <= hi;
                int b = -1;
                if (in) {
                    const float k32 = __double2float_rd(ckey);
                    in = T2_B1(k32) == bs1;
                    b = T2_B2(k32);
                }
                const unsigned im = __ballot_sync(GHN_FULL, in);
                if (in) {
                    const unsigned grp = __match_any_sync(im, b);
                    if ((grp & lanemask_lt()) == 0) atomicAdd(&sc.hist[b], __popc(grp));
                }
            }
        }
        __syncwarp();
        cnt = sc.hist[lane];
        incl = warp_inclusive_scan(cnt);
        ge = __ballot_sync(GHN_FULL, incl >= r);
        if (!ge) return false;
        bs2 = __ffs(ge) - 1;
        m = __shfl_sync(GHN_FULL, cnt, bs2);
        r -= __shfl_sync(GHN_FULL, incl - cnt, bs2);
        if (m > 32) return false;
    }
    // members below the boundary vote now; boundary candidates are compacted
    v.lab = 0;
    v.cnt = 0;
    v.used = 0;
    v.overflow = false;
    int nb = 0;
    for (int i = 0; i < c.nch; ++i) {
        {
            double ckey;
            int32_t cgs;
            c.at(i, ckey, cgs);
            int side = 1;
            if (cgs >= 0 && ckey >= lo && ckey <= hi) {
                const float k32 = __double2float_rd(ckey);
                const int b1 = T2_B1(k32);
                side = b1 < bs1 ? -1 : (b1 > bs1 ? 1 : 0);
                if (side == 0 && bs2 >= 0) {
                    const int b2 = T2_B2(k32);
                    side = b2 < bs2 ? -1 : (b2 > bs2 ? 1 : 0);
                }
            }
            vote_members(*c.w, sc, v, small, side < 0, cgs);
            if (outside && __any_sync(GHN_FULL, side < 0 && (cgs < og0 || cgs >= og1))) *outside = true;
            const unsigned bnd = __ballot_sync(GHN_FULL, side == 0);
            if (side == 0) {
                const int pos = nb + __popc(bnd & lanemask_lt());
                sc.bkey[pos] = ckey;
                sc.bidx[pos] = c.w->sp[cgs];
                sc.bg[pos] = cgs;
            }
            nb += __popc(bnd);
        }
    }
#undef T2_B1
#undef T2_B2
    __syncwarp();
    double mk = INFINITY;
    int32_t mi = 0x7fffffff, mg = 0;
    if (lane < nb) {
        mk = sc.bkey[lane];
        mi = sc.bidx[lane];
        mg = sc.bg[lane];
    }
    int rank = 0;
    for (int t = 0; t < nb; ++t) {
        const double tk = __shfl_sync(GHN_FULL, mk, t);
        const int32_t ti = __shfl_sync(GHN_FULL, mi, t);
        rank += lt_pair(tk, ti, mk, mi) ? 1 : 0;
    }
    vote_members(*c.w, sc, v, small, lane < nb && rank < r, mg);
    if (outside && __any_sync(GHN_FULL, lane < nb && rank < r && (mg < og0 || mg >= og1))) *outside = true;
    const unsigned kl = __ballot_sync(GHN_FULL, lane < nb && rank == r - 1);
    if (!kl) return false;
    const int src = __ffs(kl) - 1;
    out.key = __shfl_sync(GHN_FULL, mk, src);
    out.idx = __shfl_sync(GHN_FULL, mi, src);
    __syncwarp();
    if (small) {   // counters -> table: lane j holds label j
        v.lab = lane;
        v.cnt = sc.lcnt[lane];
        v.used = 32;
    }
    return !v.overflow;
}

// Exact r-th smallest (key, index) by repeated warp-minimum extraction over
// at most 32*NC candidates held in registers (block(1) at k <= 16: about 54).
// Each round takes the warp minimum (redux.sync) of the candidates' fp32
// round-down keys: the round-down is monotone, so a unique minimum is the
// exact next candidate; only when round-downs collide (several lanes or
// slots at the minimum) are the colliding candidates ranked by exact fp64
// (key, index).  The extracted r members then vote.  Cost ~ r rounds of a
// dozen instructions instead of the histogram passes of select_vote_c.
template <int NC>
__device__ __forceinline__ bool select_extract(const Win &w, WarpScratch &sc, const Ranges &rg, double q0,
                                               double q1, int r, int lbits, Kth &out, VoteW &v,
                                               int32_t og0, int32_t og1, bool *outside) {
    static_assert(NC == 2, "slots kept sorted pairwise");
    const int lane = lane_id();
    unsigned k32[NC];
    int pp[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        int p = 0;
        k32[c] = 0xffffffffu;
        if (ranges_at(rg, c * 32 + lane, p)) k32[c] = __float_as_uint(__double2float_rd(key2(w, p, q0, q1)));
        pp[c] = p;
    }
    // each lane's two slots in exact (key, index) order: slot 0 is its best
    bool swap = k32[1] < k32[0];
    if (k32[1] == k32[0] && k32[0] != 0xffffffffu)
        swap = lt_pair(key2(w, pp[1], q0, q1), w.sp[pp[1]], key2(w, pp[0], q0, q1), w.sp[pp[0]]);
    if (swap) {
        const unsigned tk = k32[0];
        k32[0] = k32[1];
        k32[1] = tk;
        const int tp = pp[0];
        pp[0] = pp[1];
        pp[1] = tp;
    }
    // lane state: lm = next candidate, nx = the one after; a consumed slot
    // becomes TAKEN (a NaN pattern above every real key, below absent)
    constexpr unsigned TAKEN = 0xfffffffeu;
    unsigned lm = k32[0];
    unsigned nx = k32[1];
    int lastit = 0;   // countdown value of the round this lane last won
    for (int it = r; it > 0; --it) {
        unsigned m;
        asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(m) : "r"(lm));
        bool mine = lm == m;
        const unsigned win = __ballot_sync(GHN_FULL, mine);
        if (__builtin_expect((win & (win - 1)) != 0, 0)) {
            // colliding round-downs in several lanes: exact minimum among them
            double rk = INFINITY;
            int32_t ri = 0x7fffffff, rl = lane;
            if (mine) {
                const int p = nx == TAKEN ? pp[1] : pp[0];
                rk = key2(w, p, q0, q1);
                ri = w.sp[p];
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ok = __shfl_xor_sync(GHN_FULL, rk, off);
                const int32_t oi = __shfl_xor_sync(GHN_FULL, ri, off);
                const int32_t ol = __shfl_xor_sync(GHN_FULL, rl, off);
                if (lt_pair(ok, oi, rk, ri)) {
                    rk = ok;
                    ri = oi;
                    rl = ol;
                }
            }
            mine = lane == rl;
        }
        // branch-free update of the winner lane
        lm = mine ? nx : lm;
        nx = mine ? TAKEN : nx;
        lastit = mine ? it : lastit;
    }
    const int ne = (nx == TAKEN ? 1 : 0) + (lm == TAKEN ? 1 : 0);   // slots taken, in order
    const int wl = __ffs(__ballot_sync(GHN_FULL, lastit == 1)) - 1;
    const int lastp = ne == 2 ? pp[1] : pp[0];   // meaningful on lane wl
    unsigned memb = ne == 0 ? 0u : (ne == 1 ? 1u : 3u);
    // the r-th member, exactly
    const double kk = key2(w, lastp, q0, q1);
    out.key = __shfl_sync(GHN_FULL, kk, wl);
    out.idx = __shfl_sync(GHN_FULL, w.sp[lastp], wl);
    v.lab = 0;
    v.cnt = 0;
    v.used = 0;
    v.overflow = false;
    sc.lcnt[lane] = 0;
    __syncwarp();
    bool outl = false;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const bool mem = (memb >> c) & 1u;
        vote_members(w, sc, v, lbits >= 0, mem, pp[c]);
        outl |= mem && (pp[c] < og0 || pp[c] >= og1);
    }
    if (outside && __any_sync(GHN_FULL, outl)) *outside = true;
    __syncwarp();
    if (lbits >= 0) {
        v.lab = lane;
        v.cnt = sc.lcnt[lane];
        v.used = 32;
    }
    return !v.overflow;
}

// Tie-break among the labels tied at the top count: the label of the member
// minimising (sqrt(key), index) (predict.py:30-35), over the cached members.
__device__ __forceinline__ int32_t vote_tiebreak_c(const T2Args &a, const Cands &c, const Kth &kth,
                                                   const VoteW &v, int top) {
    const int lane = lane_id();
    // tied labels, one per lane of the table
    const bool my_tied = lane < v.used && v.cnt == top;
    double bd = INFINITY;
    int32_t bi = 0x7fffffff, bl = 0;
    for (int i = 0; i < c.nch; ++i) {
        {
            double key;
            int32_t cgs;
            c.at(i, key, cgs);
            int32_t idx = 0x7fffffff, Lb = -1;
            bool member = false;
            if (cgs >= 0 && key <= kth.key) {
                idx = c.w->sp[cgs];
                member = key < kth.key || idx <= kth.idx;
                if (member) Lb = c.w->sl[cgs];
            }
            bool tied = false;
            for (int t = 0; t < v.used; ++t) {
                const int32_t tl = __shfl_sync(GHN_FULL, v.lab, t);
                const bool tt = __shfl_sync(GHN_FULL, my_tied, t);
                tied |= member && tt && tl == Lb;
            }
            if (tied) {
                const double dd = sqrt(key);
                if (dd < bd || (dd == bd && idx < bi)) {
                    bd = dd;
                    bi = idx;
                    bl = Lb;
                }
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double od = __shfl_xor_sync(GHN_FULL, bd, off);
        const int32_t oi = __shfl_xor_sync(GHN_FULL, bi, off);
        const int32_t ol = __shfl_xor_sync(GHN_FULL, bl, off);
        if (od < bd || (od == bd && oi < bi)) {
            bd = od;
            bi = oi;
            bl = ol;
        }
    }
    return bl;
}

// Diagnostics build (-DGHN_FB_REASONS): per-site counts of the thread
// kernel's bucket-select fallbacks, printed under GHN_DEBUG_FALLBACK.
#ifdef GHN_FB_REASONS
__device__ unsigned long long g_fb_reason[16];
#define FB_REASON(r) atomicAdd(&g_fb_reason[r], 1ull)
#else
#define FB_REASON(r) ((void)0)
#endif

__device__ __forceinline__ void push_fallback(const T2Args &a, int32_t qi) {
    const int32_t slot = atomicAdd(a.fb_count, 1);
    a.fb_list[slot] = qi;
}

// Non-empty cells of block(l) (QueryStats; only when stats are requested).
__device__ __forceinline__ int block_cells(const Win &w, int lr, int lc, int l) {
    const int lane = lane_id();
    const int side = 2 * l + 1;
    int cells = 0;
    for (int e = lane; e < side * side; e += 32) {
        const int i = lr - l + e / side, j = lc - l + e % side;
        if (i >= 0 && i < w.R && j >= 0 && j < w.W) {
            const int32_t *rp = w.loc + i * w.W1;
            cells += rp[j + 1] > rp[j];
        }
    }
    return warp_sum(cells);
}

// Every point of shell(l+1) lies outside block(l), so its distance to q is at
// least the distance from q to the nearest face of block(l).  When that bound
// (less a rounding margin far above fp64 error: cell assignment by floor(x/w)
// and the key's own rounding are both within a few ulps) exceeds the k-th
// key, no point of the shell can precede the k-th: the layer is visited
// (counted in QueryStats) but cannot change the top-k.
__device__ __forceinline__ bool shell_cannot_change(const T2Args &a, double q0, double q1, int64_t cc0,
                                                    int64_t cc1, int l, double kth_key) {
    const double f0 = fmin(q0 - (double)(a.lo0 + cc0 - l) * a.w0, (double)(a.lo0 + cc0 + l + 1) * a.w0 - q0);
    const double f1 = fmin(q1 - (double)(a.lo1 + cc1 - l) * a.w1, (double)(a.lo1 + cc1 + l + 1) * a.w1 - q1);
    const double margin = 1e-9 * fmax(a.w0, a.w1) + 1e-12 * (fabs(q0) + fabs(q1));
    const double d = fmin(f0, f1) - margin;
    if (!(d > 0.0)) return false;
    return d * d * (1.0 - 1e-9) > kth_key;
}

// The same bound with the per-query part hoisted: the face distance of
// block(l) is (q's distance to its own cell's nearest face) + l * w per axis.
struct ShellBound {
    double f0, f1, margin;
    __device__ __forceinline__ ShellBound() : f0(0.0), f1(0.0), margin(0.0) {}
    __device__ __forceinline__ ShellBound(const T2Args &a, double q0, double q1, int64_t cc0, int64_t cc1) {
        f0 = fmin(q0 - (double)(a.lo0 + cc0) * a.w0, (double)(a.lo0 + cc0 + 1) * a.w0 - q0);
        f1 = fmin(q1 - (double)(a.lo1 + cc1) * a.w1, (double)(a.lo1 + cc1 + 1) * a.w1 - q1);
        margin = 1e-9 * fmax(a.w0, a.w1) + 1e-12 * (fabs(q0) + fabs(q1));
    }
    // shell(l + 1) cannot hold a point preceding kth_key
    __device__ __forceinline__ bool cannot_change(const T2Args &a, int l, double kth_key) const {
        const double d = fmin(f0 + (double)l * a.w0, f1 + (double)l * a.w1) - margin;
        return d > 0.0 && d * d * (1.0 - 1e-9) > kth_key;
    }
};

// Points in block(l) (warp-uniform; one row per lane).
__device__ __forceinline__ int block_total(const Win &w, int lr, int lc, int l) {
    const int lane = lane_id();
    int n = 0;
    const int i = lr - l + lane;
    if (lane <= 2 * l && i >= 0 && i < w.R) {
        const int a = max(lc - l, 0), b = min(lc + l, w.W - 1);
        const int32_t *rp = w.loc + i * w.W1;
        n = rp[b + 1] - rp[a];
    }
    return warp_sum(n);
}

// k = 1: the top-1 is a running minimum; a layer `changed` iff its minimum
// (key, index) precedes the current one (explore.py:112-119 with k = 1).
__device__ __forceinline__ void process_query_k1(const T2Args &a, const Win &w, double q0, double q1,
                                                 int32_t qi, int64_t cc0, int64_t cc1, int lr, int lc,
                                                 int lmax, bool want_stats) {
    const int lane = lane_id();
    double ck = INFINITY;
    int32_t ci = 0x7fffffff, cg = -1;
    bool have = false;
    int64_t points = 0;
    int layers = 0;
    for (int l = 0;; ++l) {
        if (l > a.A) {
            if (lane == 0) push_fallback(a, qi);
            return;
        }
        if (have && l > 0 && shell_cannot_change(a, q0, q1, cc0, cc1, l - 1, ck)) {
            // shell(l) cannot hold a point preceding the current minimum
            points += block_total(w, lr, lc, l) - block_total(w, lr, lc, l - 1);
            layers = l;
            bool stop = a.mode == GHN_MODE_HEURISTIC;
            if (a.mode == GHN_MODE_GUARANTEED) {
                const double b = __dmul_rn((double)l, a.min_w);
                if (__dmul_rn(b, b) > ck) stop = true;
            }
            if (stop || l >= lmax) break;
            continue;
        }
        const Ranges rg = l == 0 ? block_ranges(w, lr, lc, 0) : shell_ranges(w, lr, lc, l);
        // per-lane minimum by key, index resolved for the lane's winner / ties
        double mk = INFINITY;
        int32_t mg = -1, mi = 0x7fffffff;
        for (int base = 0; base < rg.total; base += 32) {
            int p;
            if (ranges_at(rg, base + lane, p)) {
                const double key = key2(w, p, q0, q1);
                const int32_t g = p;
                if (key < mk) {
                    mk = key;
                    mg = g;
                    mi = 0x7fffffff;
                } else if (key == mk) {
                    if (mi == 0x7fffffff) mi = w.sp[mg];
                    const int32_t ii = w.sp[g];
                    if (ii < mi) {
                        mi = ii;
                        mg = g;
                    }
                }
            }
        }
        if (mg >= 0 && mi == 0x7fffffff) mi = w.sp[mg];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ok = __shfl_xor_sync(GHN_FULL, mk, off);
            const int32_t oi = __shfl_xor_sync(GHN_FULL, mi, off);
            const int32_t og = __shfl_xor_sync(GHN_FULL, mg, off);
            if (lt_pair(ok, oi, mk, mi)) {
                mk = ok;
                mi = oi;
                mg = og;
            }
        }
        points += rg.total;
        layers = l;
        bool changed = false;
        if (rg.total > 0 && (!have || lt_pair(mk, mi, ck, ci))) {
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
    const int64_t cells = want_stats ? block_cells(w, lr, lc, layers) : 0;
    if (lane == 0) {
        if (a.out_label) a.out_label[qi] = (int32_t)w.sl[cg];
        if (a.out_conf) a.out_conf[qi] = 1.0;
        if (want_stats) {
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
}

template <bool EXT>
__device__ __forceinline__ void process_query_w(const T2Args &a, const Win &w, WarpScratch &sc, int qq,
                                                int t0, int t1, int r_lo, int c_lo, bool want_stats) {
    const int lane = lane_id();
    const int32_t qi = a.qorder[qq];
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
        if (lane == 0) push_fallback(a, qi);   // centre outside the grid
        return;
    }
    const int lr = (int)(cc0 - r_lo), lc = (int)(cc1 - c_lo);
    const int lmax = max(max((int)cc0, a.ext0 - 1 - (int)cc0), max((int)cc1, a.ext1 - 1 - (int)cc1));
    const int k = a.k;
    if (!EXT && k == 1 && a.dbg == 0) {
        process_query_k1(a, w, q0, q1, qi, cc0, cc1, lr, lc, lmax, want_stats);
        return;
    }
    // phase 1: whole layers enter while fewer than k points are buffered
    int l = 0;
    Ranges blk;
    for (;; ++l) {
        if (l > a.A) {
            if (lane == 0) push_fallback(a, qi);
            return;
        }
        blk = block_ranges(w, lr, lc, l);
        if (blk.total >= k || l >= lmax) break;
    }
    if (a.dbg == 1) {
        if (lane == 0 && a.out_label) a.out_label[qi] = blk.total;
        return;
    }
    bool stop = a.dbg == 2;
    Kth kth{INFINITY, 0x7fffffff};
    VoteW v{0, 0, 0, false};
    // Layer 0 filled the buffer and always `changed`; neither stop rule can
    // fire at l = 0, so T_0 is never needed: select T_1 over block(1)
    // directly.  changed(1) <=> a member of T_1 lies outside the centre cell.
    const bool skip0 = l == 0 && lmax >= 1 && a.A >= 1 && a.dbg != 2;
    int32_t og0 = 0, og1 = 0x7fffffff;   // staged range of the centre cell (skip0)
    if (skip0) {
        const int32_t *rp = w.loc + lr * w.W1;
        og0 = rp[lc];
        og1 = rp[lc + 1];
        l = 1;
        blk = block_ranges(w, lr, lc, 1);
    }
    if (blk.total < k) {
        if (lane == 0) push_fallback(a, qi);
        return;
    }
    int64_t points = 0, cells = 0;
    int layers = l;
    const ShellBound sb(a, q0, q1, cc0, cc1);
    double hi = -1.0;   // select bucket range: < 0 = the block's own bound
    bool first = true;
    // One select site (code size): T_l over block(l) first, then again for
    // every later layer that changes the top-k.
    for (;;) {
        bool outside = false;
        bool ok;
        if (EXT && blk.total <= 64) {
            ok = select_extract<2>(w, sc, blk, q0, q1, k, a.small_labels - 1, kth, v, og0, og1, &outside);
        } else {
            double h = hi;
            if (h < 0.0) {
                const double e0 =
                    fmax(q0 - (double)(a.lo0 + cc0 - l) * a.w0, (double)(a.lo0 + cc0 + l + 1) * a.w0 - q0);
                const double e1 =
                    fmax(q1 - (double)(a.lo1 + cc1 - l) * a.w1, (double)(a.lo1 + cc1 + l + 1) * a.w1 - q1);
                h = (e0 * e0 + e1 * e1) * (1.0 + 1e-6) + 1e-300;
            }
            ok = select_vote_c(a, sc, make_cands(w, blk, q0, q1), k, 0.0, h, kth, v, og0, og1, &outside);
        }
        if (!ok) {
            if (lane == 0) push_fallback(a, qi);
            return;
        }
        if (first) {
            if (skip0 && a.mode == GHN_MODE_HEURISTIC && !outside) stop = true;
            points = blk.total;
            cells = want_stats ? block_cells(w, lr, lc, l) : 0;
            first = false;
        }
        // the layer that filled / changed the buffer `changed`; the guaranteed bound may stop
        if (a.mode == GHN_MODE_GUARANTEED) {
            const double b = __dmul_rn((double)l, a.min_w);
            if (__dmul_rn(b, b) > kth.key) stop = true;
        }
        // a later layer matters only if one of its points precedes the k-th
        bool changed = false;
        while (!stop && l < lmax) {
            ++l;
            if (l > a.A) {
                if (lane == 0) push_fallback(a, qi);
                return;
            }
            int below = 0;
            if (sb.cannot_change(a, l - 1, kth.key)) {
                if (want_stats) points += block_total(w, lr, lc, l) - block_total(w, lr, lc, l - 1);
            } else {
                const Ranges sh = shell_ranges(w, lr, lc, l);
                for (int base = 0; base < sh.total; base += 32) {
                    int p;
                    const bool act = ranges_at(sh, base + lane, p);
                    bool lt = false;
                    if (act) {
                        const double key = key2(w, p, q0, q1);
                        lt = key < kth.key || (key == kth.key && w.sp[p] < kth.idx);
                    }
                    below += __popc(__ballot_sync(GHN_FULL, lt));
                }
                points += sh.total;
            }
            layers = l;
            if (want_stats) cells = block_cells(w, lr, lc, l);
            if (below > 0) {
                changed = true;
                break;
            }
            if (a.mode == GHN_MODE_HEURISTIC) stop = true;
            if (a.mode == GHN_MODE_GUARANTEED) {
                const double b = __dmul_rn((double)l, a.min_w);
                if (__dmul_rn(b, b) > kth.key) stop = true;
            }
        }
        if (!changed) break;
        blk = block_ranges(w, lr, lc, l);
        hi = kth.key;
        og0 = 0;
        og1 = 0x7fffffff;
    }
    // winner: top count; ties -> nearest member by (sqrt(key), index)
    const int top = warp_max(lane < v.used ? v.cnt : 0);
    const unsigned tiedm = __ballot_sync(GHN_FULL, lane < v.used && v.cnt == top);
    int32_t wl = __shfl_sync(GHN_FULL, v.lab, __ffs(tiedm) - 1);
    if (__popc(tiedm) > 1) {
        // members are the candidates of the last selected block
        const Cands cd = make_cands(w, blk, q0, q1);
        wl = vote_tiebreak_c(a, cd, kth, v, top);
    }
    if (lane == 0) {
        if (a.out_label) a.out_label[qi] = wl;
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

// EXT: phase-1 selects over <= 64 candidates by extraction (small k)
template <bool EXT>
__global__ void __launch_bounds__(T2_THREADS, T2_MINB) tile2d_kernel(const T2Args a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int s_P;
    __shared__ WarpScratch s_scratch[T2_THREADS / 32];
    const int t = blockIdx.x;
    const int qb = a.tile_start[t], qe = a.tile_start[t + 1];
    if (qb == qe) return;
    const int t0 = t / a.nt1, t1 = t - (t / a.nt1) * a.nt1;
    const int r_lo = max(t0 * a.T - a.A, 0), r_hi = min(t0 * a.T + a.T - 1 + a.A, a.ext0 - 1);
    const int c_lo = max(t1 * a.T - a.A, 0), c_hi = min(t1 * a.T + a.T - 1 + a.A, a.ext1 - 1);
    const int R = r_hi - r_lo + 1, W = c_hi - c_lo + 1, W1 = W + 1;
    float *sx = (float *)sm;
    float *sy = sx + a.cap;
    int32_t *sp = (int32_t *)(sy + a.cap);
    uint8_t *sl = (uint8_t *)(sp + a.cap);
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
    for (int i = threadIdx.x >> 5; i < R; i += T2_THREADS / 32) {   // warp per row: coalesced copy
        const int p0 = rstart[i], p1 = rstart[i + 1], d = delta[i];
        for (int p = p0 + (int)(threadIdx.x & 31); p < p1; p += 32) {
            sx[p] = a.c0[p + d];
            sy[p] = a.c1[p + d];
            sp[p] = a.perm[p + d];
            sl[p] = (uint8_t)a.labels_perm[p + d];
        }
    }
    __syncthreads();
    Win w{sx, sy, sp, sl, loc, delta, R, W, W1};
    const int warp = threadIdx.x >> 5;
    const bool want_stats = a.out_stats != nullptr || a.totals != nullptr;
    for (int qq = qb + warp; qq < qe; qq += T2_THREADS / 32)
        process_query_w<EXT>(a, w, s_scratch[warp], qq, t0, t1, r_lo, c_lo, want_stats);
}

}  // namespace
}  // namespace ghn

#include "ghn_tile2d_grp.cuh"
#include "ghn_tile2d_thr.cuh"

namespace ghn {
namespace {

template <int G>
__global__ void __launch_bounds__(T2_THREADS) tile2d_grp_kernel(const T2Args a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ int s_P;
    __shared__ GrpScratch s_gs[T2_THREADS / G];
    const int t = blockIdx.x;
    const int qb = a.tile_start[t], qe = a.tile_start[t + 1];
    if (qb == qe) return;
    const int t0 = t / a.nt1, t1 = t - (t / a.nt1) * a.nt1;
    const int r_lo = max(t0 * a.T - a.A, 0), r_hi = min(t0 * a.T + a.T - 1 + a.A, a.ext0 - 1);
    const int c_lo = max(t1 * a.T - a.A, 0), c_hi = min(t1 * a.T + a.T - 1 + a.A, a.ext1 - 1);
    const int R = r_hi - r_lo + 1, W = c_hi - c_lo + 1, W1 = W + 1;
    float *sx = (float *)sm;
    float *sy = sx + a.cap;
    int32_t *loc = (int32_t *)(sy + a.cap);                        // [R][W+1]
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
    for (int i = threadIdx.x >> 5; i < R; i += T2_THREADS / 32) {   // warp per row: coalesced copy
        const int p0 = rstart[i], p1 = rstart[i + 1], d = delta[i];
        for (int p = p0 + (int)(threadIdx.x & 31); p < p1; p += 32) {
            sx[p] = a.c0[p + d];
            sy[p] = a.c1[p + d];
        }
    }
    __syncthreads();
    Win w{sx, sy, nullptr, nullptr, loc, delta, R, W, W1};
    const Grp<G> gr;
    const int gid = threadIdx.x / G;
    const bool want_stats = a.out_stats != nullptr || a.totals != nullptr;
    for (int qq = qb + gid; qq < qe; qq += T2_THREADS / G)
        process_query_grp<G>(a, w, s_gs[gid], gr, a.qorder[qq], t0, t1, r_lo, c_lo, want_stats);
}

}  // namespace
}  // namespace ghn

namespace ghn {
namespace {

// ------------------------------------------------------------------ binning
__global__ void tile_key_kernel(const void *Q, int32_t q_dtype, int64_t nq, double w0, double w1,
                                double inv0, double inv1, uint32_t pow2, int64_t lo0, int64_t lo1,
                                int32_t ext0, int32_t ext1, int32_t T, int32_t nt1, int32_t *keys,
                                int32_t *ranks, int32_t *counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        double q0, q1;
        if (q_dtype == GHN_F32) {
            q0 = ((const float *)Q)[2 * i];
            q1 = ((const float *)Q)[2 * i + 1];
        } else {
            q0 = ((const double *)Q)[2 * i];
            q1 = ((const double *)Q)[2 * i + 1];
        }
        int64_t c0 = cell_id(q0, w0, inv0, pow2 & 1u) - lo0;
        int64_t c1 = cell_id(q1, w1, inv1, (pow2 >> 1) & 1u) - lo1;
        c0 = c0 < 0 ? 0 : (c0 >= ext0 ? ext0 - 1 : c0);
        c1 = c1 < 0 ? 0 : (c1 >= ext1 ? ext1 - 1 : c1);
        const int32_t key = (int32_t)(c0 / T) * nt1 + (int32_t)(c1 / T);
        keys[i] = key;
        ranks[i] = atomicAdd(&counts[key], 1);   // the query's slot inside its tile
    }
}

// No atomics here: the slot inside the tile came with the count.
__global__ void tile_scatter_kernel(const int32_t *keys, const int32_t *ranks, int64_t nq,
                                    const int32_t *tile_start, int32_t *order) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x)
        order[tile_start[keys[i]] + ranks[i]] = (int32_t)i;
}

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

// Window density around evenly spaced CSR slots (ghn_window_density).
__global__ void window_density_kernel(const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_ids,
                                      int32_t n_cells, const int32_t *__restrict__ pt_off, int64_t n,
                                      int32_t ext0, int32_t ext1, int32_t radius, int32_t samples,
                                      float *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= samples) return;
    const int32_t slot = (int32_t)(((int64_t)i * n + n / 2) / samples);
    int lo = 0, hi = n_cells - 1;   // the non-empty cell holding the slot
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cell_start[mid] <= slot) lo = mid;
        else hi = mid - 1;
    }
    const int r = cell_ids[2 * lo], c = cell_ids[2 * lo + 1];
    const int r0 = max(r - radius, 0), r1 = min(r + radius, ext0 - 1);
    const int c0 = max(c - radius, 0), c1 = min(c + radius, ext1 - 1);
    int64_t cnt = 0;
    for (int row = r0; row <= r1; ++row)
        cnt += pt_off[(int64_t)row * ext1 + c1 + 1] - pt_off[(int64_t)row * ext1 + c0];
    out[i] = (float)((double)cnt / ((double)(r1 - r0 + 1) * (double)(c1 - c0 + 1)));
}

}  // namespace

// Largest k answered with the register list; larger k use the bucket select
// (GHN_TT_LISTMAX overrides, for measurements).
static int tt_tab_on() {
    return GHN_TT_TAB;
}

static int tt_list_kmax_nb() {
    return TT_LIST_KMAX;
}

static int tt_list_kmax() {
    return (int)knob("GHN_TT_LISTMAX", TT_LIST_KMAX);
}

bool tile2d_plan(const ghn_index_view *ix, int64_t nq, int32_t k, int32_t task, bool want_neighbors, bool want_stats,
                 Tile2dPlan *plan) {
    memset(plan, 0, sizeof(*plan));
    if (ix->layout != GHN_LAYOUT_DENSE || ix->d != 2 || ix->dtype != GHN_F32) return false;
    // the fused vote, or (list rounds, k <= 32) the neighbours alone
    const bool nb = task == GHN_TASK_NONE && want_neighbors && GHN_TT_TAB != 0 && k <= tt_list_kmax_nb();
    if (!nb && (task != GHN_TASK_CLASSIFY || want_neighbors || !ix->labels_perm)) return false;
    if (ix->metric != GHN_METRIC_EUCLIDEAN) return false;
    if (nq < 4096 || k < 1 || k > 256) return false;
    // points per cell to size tiles for: the mean, or the caller's local
    // density quantile (ghn_window_density) when the points are clustered
    double rho = (double)ix->n / (double)ix->E;
    if (ix->density_hint > rho) rho = ix->density_hint;
    int lf = 0;
    while (lf < 8 && (2.0 * lf + 1) * (2.0 * lf + 1) * rho < (double)k) ++lf;
    // sparse for this k: the typical query needs layers beyond any apron a tile
    // can stage (4), so nearly every query would end on the fallback list after
    // the staging was paid (0.5 points per cell at k = 64: lf = 6)
    if (lf + 1 > 4) return false;
    // apron: two layers beyond the layer that fills the buffer on average.  The
    // thread kernels without QueryStats need one: a shell beyond the apron that
    // provably cannot change the top-k is skipped without its data.
    const bool thr = nb || (k <= TT_KMAX && ix->n_labels > 0 && ix->n_labels <= 8);
    // (only when block(lf) almost surely fills the buffer: a query that needs
    // the next block looks two layers out)
    double p_short = 0.0;   // P(Poisson((2 lf + 1)^2 rho) < k)
    {
        const double m = (2.0 * lf + 1) * (2.0 * lf + 1) * rho;
        double term = exp(-m);
        for (int i = 0; i < k; ++i) {
            p_short += term;
            term *= m / (i + 1);
        }
    }
    const int extra = thr && (k > tt_list_kmax() || tt_tab_on()) && !want_stats && p_short < 1e-3 ? 1 : 2;
    const int A = (int)knob("GHN_TILE_A", lf + extra > 4 ? 4 : lf + extra);
    int T = (int)floor(sqrt(0.7 * T2_CAP / (rho > 1e-9 ? rho : 1e-9))) - 2 * A;
    const double Tmax = sqrt((double)ix->E / (sm_count() * 4.0));
    if (T > Tmax) T = (int)Tmax;
    if (T > 64) T = 64;
    if (T < 1) return false;
    plan->T = T;
    plan->A = A;
    plan->nt0 = (int32_t)((ix->ext[0] + T - 1) / T);
    plan->nt1 = (int32_t)((ix->ext[1] + T - 1) / T);
    plan->ntiles = (int64_t)plan->nt0 * plan->nt1;
    plan->win = T + 2 * A;
    // lanes per query: k = 1 (a per-layer running minimum, no select) runs 4
    // queries per warp; the radix select is faster warp-wide (measured: the
    // sub-warp select loses to divergence between the groups of a warp).
    // The group kernel votes with shared counters: label codes in [0, 32).
    plan->G = 32;
    if (k == 1 && ix->n_labels > 0 && ix->n_labels <= 32) plan->G = 8;
    // thread per query (packed-key register list): k <= 32, <= 8 label codes
    if (k <= TT_KMAX && ix->n_labels > 0 && ix->n_labels <= 8) plan->G = 1;
    plan->G = (int)knob("GHN_TILE_G", plan->G);
    if (nb) plan->G = 1;
    plan->nb = nb ? 1 : 0;
    if (plan->G == 1) {
        // ~TT_Q queries per tile (one or two per thread) within the staging capacity
        const double qd = (double)nq / (double)ix->E;
        // (the list rounds for k = 5-32 run best with two groups per warp:
        // cfg4 k = 8 / 16 / 32 at 450 against 256: 2.57 / 2.70 / 6.69 against
        // 2.92 / 2.91 / 7.10 ms; k <= 4 and the bucket select do not)
        const double tq = knob("GHN_TT_Q", k > 4 && k <= tt_list_kmax() ? 450.0 : TT_Q);
        int Tq = (int)floor(sqrt(tq / (qd > 1e-9 ? qd : 1e-9)));
        const int Tc = (int)floor(sqrt((TT_CAP - 64.0) / 1.1 / (rho > 1e-9 ? rho : 1e-9))) - 2 * A;
        if (Tq > Tc) Tq = Tc;
        if (Tq > Tmax) Tq = (int)Tmax;
        if (Tq > 64) Tq = 64;
        if (Tq < 1) return false;
        T = Tq;
        plan->T = T;
        plan->nt0 = (int32_t)((ix->ext[0] + T - 1) / T);
        plan->nt1 = (int32_t)((ix->ext[1] + T - 1) / T);
        plan->ntiles = (int64_t)plan->nt0 * plan->nt1;
        plan->win = T + 2 * A;
    }
    // staged-point capacity: the expected window plus margin (an overflowing
    // tile sends its queries to the generic kernel)
    auto cap_for = [&](int win) {
        const double expect = (double)win * win * rho;
        int cap = (int)(1.1 * expect + 64.0);   // Poisson window count: +10 % is > 5 sigma at cfg4
        cap = (cap + 127) & ~127;
        if (cap > 8192) cap = 8192;
        if (cap < 256) cap = 256;
        return cap;
    };
    int cap = cap_for(plan->win);
    plan->cap = cap;
    if (plan->G == 1) {   // float2 coordinates + u8 label code per staged point
        const bool select = k > tt_list_kmax();
        auto smem_for = [&](int win, int cap_) {
            size_t b = (size_t)cap_ * 9 + (size_t)win * (win + 1) * 4 + (size_t)win * 4 + (size_t)(win + 1) * 4 + 64;
            // bucket select: per-lane row tables + byte histograms
            if (select) b += (size_t)SB_ROWS * TT_THREADS * 4 + (size_t)SB_NB * TT_THREADS;
            // list rounds: per-lane row tables (+ the word the walk prefetches past the sentinel)
            else if (tt_tab_on()) b += (size_t)(2 * A + 3) * TT_THREADS * 4;
            return b;
        };
        plan->smem = smem_for(plan->win, cap);
        if (select) {
            // three CTAs per SM (the kernel's register budget): shrink the tile
            // until three windows fit in the SM's 227 KB (1 KB reserved per CTA)
            const size_t fit3 = (227 * 1024) / 3 - 1024 - 3200;   // static shared: order, phase-A words
            int T3 = plan->T;
            while (smem_for(T3 + 2 * A, cap_for(T3 + 2 * A)) > fit3 && T3 > (int)knob("GHN_SB_TMIN", 14)) --T3;
            if (T3 != plan->T && smem_for(T3 + 2 * A, cap_for(T3 + 2 * A)) <= fit3) {
                plan->T = T3;
                plan->nt0 = (int32_t)((ix->ext[0] + T3 - 1) / T3);
                plan->nt1 = (int32_t)((ix->ext[1] + T3 - 1) / T3);
                plan->ntiles = (int64_t)plan->nt0 * plan->nt1;
                plan->win = T3 + 2 * A;
                plan->cap = cap = cap_for(plan->win);
                plan->smem = smem_for(plan->win, cap);
            }
        }
        return plan->smem <= 200 * 1024;
    }
    // the warp kernel also stages each point's index (int32) and label code (u8)
    if (plan->G == 32 && !(ix->n_labels > 0 && ix->n_labels <= 256)) return false;
    plan->smem = (size_t)cap * (plan->G == 32 ? 13 : 8) +
                 (size_t)plan->win * (plan->win + 1) * 4 + (size_t)plan->win * 4 +
                 (size_t)(plan->win + 1) * 4 + 64;
    if (plan->smem > 200 * 1024) return false;
    return true;
}

size_t tile2d_workspace_bytes(const Tile2dPlan *p, int64_t nq) {
    const size_t q4 = a256((size_t)nq * 4);
    const size_t t4 = a256((size_t)(p->ntiles + 1) * 4);
    return 3 * q4 + 3 * t4 + scan_workspace_bytes(p->ntiles + 1) + 256;
}

int32_t tile2d_run(const ghn_index_view *ix, const Tile2dPlan *plan, const void *Q, int32_t q_dtype,
                   int64_t nq, int32_t k, int32_t mode, const ghn_query_out *out, const double *inv_w,
                   uint32_t pow2, void *workspace, int32_t **fb_list, int32_t **fb_count,
                   cudaStream_t s) {
    char *ws = (char *)workspace;
    const size_t q4 = a256((size_t)nq * 4);
    const size_t t4 = a256((size_t)(plan->ntiles + 1) * 4);
    int32_t *keys = (int32_t *)ws;
    int32_t *order = (int32_t *)(ws + q4);
    int32_t *fbl = (int32_t *)(ws + 2 * q4);
    int32_t *tstart = (int32_t *)(ws + 3 * q4);
    int32_t *ranks = fbl;   // the fallback list is written only by the predict kernel, later
    int32_t *fbc = (int32_t *)(ws + 3 * q4 + 2 * t4);
    char *sws = ws + 3 * q4 + 3 * t4;
    GHN_CUDA_CHECK(cudaMemsetAsync(tstart, 0, (size_t)(plan->ntiles + 1) * 4, s));
    GHN_CUDA_CHECK(cudaMemsetAsync(fbc, 0, 8, s));   // the fallback count and the generic kernel's cursor over the list
    unsigned g = (unsigned)((nq + 255) / 256);
    if (g > (unsigned)sm_count() * 16) g = (unsigned)sm_count() * 16;
    tile_key_kernel<<<g, 256, 0, s>>>(Q, q_dtype, nq, ix->widths[0], ix->widths[1], inv_w[0], inv_w[1],
                                      pow2, ix->lo[0], ix->lo[1], (int32_t)ix->ext[0],
                                      (int32_t)ix->ext[1], plan->T, plan->nt1, keys, ranks, tstart);
    GHN_LAUNCH_CHECK("tile_key_kernel");
    int32_t rc = exclusive_scan_i32(tstart, tstart, plan->ntiles + 1, sws, s);
    if (rc) return rc;
    tile_scatter_kernel<<<g, 256, 0, s>>>(keys, ranks, nq, tstart, order);
    GHN_LAUNCH_CHECK("tile_scatter_kernel");
    T2Args a;
    memset(&a, 0, sizeof(a));
    a.n = ix->n;
    a.ext0 = (int32_t)ix->ext[0];
    a.ext1 = (int32_t)ix->ext[1];
    a.lo0 = ix->lo[0];
    a.lo1 = ix->lo[1];
    a.w0 = ix->widths[0];
    a.w1 = ix->widths[1];
    a.inv0 = inv_w[0];
    a.inv1 = inv_w[1];
    a.pow2 = pow2;
    a.min_w = ix->min_width;
    a.c0 = (const float *)ix->coords;
    a.c1 = (const float *)ix->coords + ix->n;
    a.pt_off = ix->pt_off;
    a.perm = ix->perm;
    a.labels_perm = ix->labels_perm;
    a.Q = Q;
    a.q_dtype = q_dtype;
    a.k = k;
    a.mode = mode;
    a.qorder = order;
    a.tile_start = tstart;
    a.T = plan->T;
    a.A = plan->A;
    a.nt0 = plan->nt0;
    a.nt1 = plan->nt1;
    a.win = plan->win;
    a.cap = plan->cap;
    a.out_label = out->label;
    a.out_conf = out->confidence;
    a.out_dist = out->dist;
    a.out_idx = out->idx;
    a.out_stats = out->stats;
    a.totals = out->totals;
    a.fb_list = fbl;
    a.fb_count = fbc;
    a.dbg = (int)knob("GHN_DEBUG_MODE", 0);   // tuning builds only: 1/2 are diagnostics that overwrite labels
    a.small_labels = ix->n_labels > 0 && ix->n_labels <= 32;
    a.lmask = ix->n_labels <= 2 ? 1 : (ix->n_labels <= 4 ? 3 : 7);
    // block sizes (whole blocks; the rows the select walks are clipped to the
    // expected k-th radius): 400 against 255 saves 0.25 ms at cfg4 k=64
    a.sb_capn = (int)knob("GHN_SB_CAPN", 400);
    a.sb_redo = (int)knob("GHN_SB_REDO", 2);
    a.sb_recap = (int)knob("GHN_SB_RECAP", 400);
    a.sb_wmax = (int)knob("GHN_SB_WMAX", 0);
    a.sb_sort = (int)knob("GHN_SB_SORT", 1);
    a.tt_skipf = knob("GHN_TT_SKIPF", 0.4);
    a.tt_tab = tt_tab_on();
    a.sb_skipf = knob("GHN_SB_SKIPF", 0.8);
    const bool stats = out->stats != nullptr || out->totals != nullptr;
    // warp kernel: extraction select for small k (EXT), histogram select otherwise
    int ki = plan->G == 8 ? 1 : (plan->G == 16 ? 2 : (k >= 2 && k <= T2_EXT_MAXK ? 3 : 0));
    const void *fn = ki == 0   ? (const void *)tile2d_kernel<false>
                     : ki == 3 ? (const void *)tile2d_kernel<true>
                     : ki == 1 ? (const void *)tile2d_grp_kernel<8>
                               : (const void *)tile2d_grp_kernel<16>;
    if (plan->G == 1) {   // thread per query: list capacity KM = next power of two >= k; 0 = bucket select
        int lk = 0;
        while ((1 << lk) < k) ++lk;
        const int v = k > tt_list_kmax() ? 0 : lk + 1;
        ki = 4 + 2 * v + (stats ? 1 : 0);
        static const void *const thr_fns[14] = {
            (const void *)tile2d_sel_kernel<false>,     (const void *)tile2d_sel_kernel<true>,
            (const void *)tile2d_thr_kernel<1, false>,  (const void *)tile2d_thr_kernel<1, true>,
            (const void *)tile2d_thr_kernel<2, false>,  (const void *)tile2d_thr_kernel<2, true>,
            (const void *)tile2d_thr_kernel<4, false>,  (const void *)tile2d_thr_kernel<4, true>,
            (const void *)tile2d_thr_kernel<8, false>,  (const void *)tile2d_thr_kernel<8, true>,
            (const void *)tile2d_thr_kernel<16, false>, (const void *)tile2d_thr_kernel<16, true>,
            (const void *)tile2d_thr_kernel<32, false>, (const void *)tile2d_thr_kernel<32, true>};
        fn = thr_fns[ki - 4];
        if (plan->nb) {
            static const void *const nb_fns[12] = {
                (const void *)tile2d_nb_kernel<1, false>,  (const void *)tile2d_nb_kernel<1, true>,
                (const void *)tile2d_nb_kernel<2, false>,  (const void *)tile2d_nb_kernel<2, true>,
                (const void *)tile2d_nb_kernel<4, false>,  (const void *)tile2d_nb_kernel<4, true>,
                (const void *)tile2d_nb_kernel<8, false>,  (const void *)tile2d_nb_kernel<8, true>,
                (const void *)tile2d_nb_kernel<16, false>, (const void *)tile2d_nb_kernel<16, true>,
                (const void *)tile2d_nb_kernel<32, false>, (const void *)tile2d_nb_kernel<32, true>};
            fn = nb_fns[ki - 6];
            ki += 14;   // (its own slot in the shared-memory attribute table)
        }
    }
    // largest dynamic smem opted into, per device and kernel (function
    // attributes are per device; callers may run on several devices / threads)
    static std::mutex attr_mu;
    static size_t attr_smem[64][36] = {};
    int dev = 0;
    GHN_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> attr_lock(attr_mu);
    if (dev >= 0 && dev < 64 && plan->smem > attr_smem[dev][ki]) {
        GHN_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan->smem));
        GHN_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            (int)cudaSharedmemCarveoutMaxShared));
        attr_smem[dev][ki] = plan->smem;
    }
    const unsigned nb = (unsigned)plan->ntiles;
    if (ki >= 4) {
        void *args[] = {&a};
        GHN_CUDA_CHECK(cudaLaunchKernel(fn, dim3(nb), dim3(TT_THREADS), args, plan->smem, s));
    } else if (ki == 1)
        tile2d_grp_kernel<8><<<nb, T2_THREADS, plan->smem, s>>>(a);
    else if (ki == 2)
        tile2d_grp_kernel<16><<<nb, T2_THREADS, plan->smem, s>>>(a);
    else if (ki == 3)
        tile2d_kernel<true><<<nb, T2_THREADS, plan->smem, s>>>(a);
    else
        tile2d_kernel<false><<<nb, T2_THREADS, plan->smem, s>>>(a);
    GHN_LAUNCH_CHECK("tile2d_kernel");
    if (plan->nb) {   // order every row by (key, index), keys -> distances (fallback rows are rewritten later)
        int P = 1;
        while (P < k) P <<= 1;
        const int64_t warps = (nq + 32 / P - 1) / (32 / P);
        nb_sort_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(out->dist, out->idx, nq, k, P, ix->perm, ix->n);
        GHN_LAUNCH_CHECK("nb_sort_kernel");
    }
    if (knob("GHN_DEBUG_FALLBACK", 0) != 0) {   // diagnostics: queries sent to the generic kernel
        int32_t nfb = 0;
        cudaMemcpyAsync(&nfb, fbc, 4, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "[ghn] tile2d k=%d nq=%lld fallbacks=%d\n", k, (long long)nq, nfb);
#ifdef GHN_FB_REASONS
        unsigned long long r[16];
        cudaMemcpyFromSymbol(r, g_fb_reason, sizeof(r));
        fprintf(stderr, "[ghn] fallback sites (cumulative):");
        for (int i = 0; i < 16; ++i) if (r[i]) fprintf(stderr, " %d:%llu", i, r[i]);
        fprintf(stderr, "\n");
#endif
    }
    *fb_list = fbl;
    *fb_count = fbc;
    return GHN_OK;
}

}  // namespace ghn

extern "C" int32_t ghn_window_density(const ghn_index_view *ix, int32_t radius, int32_t samples,
                                      float *out_density, void *stream) {
    if (ix->layout != GHN_LAYOUT_DENSE || ix->d != 2) {
        ghn::set_error("window density needs a 2-D DENSE index");
        return GHN_ERR_UNSUPPORTED;
    }
    if (samples <= 0 || radius < 0 || ix->n_cells <= 0) {
        ghn::set_error("bad window density arguments");
        return GHN_ERR_VALUE;
    }
    ghn::window_density_kernel<<<(samples + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        ix->cell_start, ix->cell_ids, ix->n_cells, ix->pt_off, ix->n, (int32_t)ix->ext[0], (int32_t)ix->ext[1],
        radius, samples, out_density);
    GHN_LAUNCH_CHECK("window_density_kernel");
    return GHN_OK;
}
