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

#include "ghn_query.cuh"

namespace ghn {
namespace {

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

}  // namespace
}  // namespace ghn

using namespace ghn;

using namespace ghn;

static size_t order_workspace_bytes(int64_t nq) {
    size_t q4 = a256((size_t)(nq > 0 ? nq : 1) * 4);
    return a256(sizeof(BinConsts)) + 5 * q4 + a256(radix_workspace_bytes(nq > 0 ? nq : 1)) + 256;
}

extern "C" size_t ghn_query_workspace_size(const ghn_index_view *ix, int64_t nq, int32_t k) {
    size_t b = order_workspace_bytes(nq);
    if (k > 256) {
        const size_t lk = largek_workspace_bytes(ix, k);
        return lk > b ? lk : b;
    }
    Tile2dPlan tp;
    // the tiling depends on whether QueryStats are requested and on vote / neighbours
    for (int v = 0; v < 4; ++v)
        if (tile2d_plan(ix, nq, k, (v & 2) ? GHN_TASK_NONE : GHN_TASK_CLASSIFY, (v & 2) != 0, (v & 1) != 0, &tp)) {
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
    if (k > 256) return largek_query(ix, Q, q_dtype, nq, k, mode, task, out, workspace, workspace_bytes, s);
    const int ks = k <= 32 ? 1 : (k <= 64 ? 2 : (k <= 128 ? 4 : 8));
    Tile2dPlan tp;
    const bool want_nb = out->dist != nullptr || out->idx != nullptr;
    const bool want_stats = out->stats != nullptr || out->totals != nullptr;
    if (mode != GHN_MODE_BRUTE && workspace && tile2d_plan(ix, nq, k, task, want_nb, want_stats, &tp) &&
        workspace_bytes >= tile2d_workspace_bytes(&tp, nq)) {
        int32_t *fb_list = nullptr, *fb_count = nullptr;
        rc = tile2d_run(ix, &tp, Q, q_dtype, nq, k, mode, out, a.inv_w, a.pow2, workspace, &fb_list,
                        &fb_count, s);
        if (rc) return rc;
        a.qorder = fb_list;
        a.nq_dev = fb_count;
        if (ix->dtype == GHN_F32) return launch_query_f32(a, ks, s);
        return launch_query_f64(a, ks, s);
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
    if (ix->dtype == GHN_F32) return launch_query_f32(a, ks, s);
    return launch_query_f64(a, ks, s);
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
