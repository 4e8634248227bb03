// ghn_query.cuh -- arguments of the generic (warp-per-query) predict kernel,
// shared by the host entry point (ghn_query.cu) and the kernel translation
// units (ghn_query_f32.cu / ghn_query_f64.cu, one per coordinate type so
// they compile in parallel).
#pragma once

#include "ghn_common.cuh"

namespace ghn {

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
    const int32_t *nq_dev;   // device count (fallback list); overrides nq when set; nq_dev[1] = work cursor (zeroed)
    ghn_query_out out;
};

// Launch the generic kernel over a.nq queries (or *a.nq_dev, the tiled
// path's fallback list) with KS top-k entries per lane.
int32_t launch_query_f32(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f64(const QArgs &a, int ks, cudaStream_t s);

// k > 256 (ghn_largek.cu): exact, one query and one layer at a time.
size_t largek_workspace_bytes(const ghn_index_view *ix, int32_t k);
int32_t largek_query(const ghn_index_view *ix, const void *Q, int32_t q_dtype, int64_t nq, int32_t k, int32_t mode,
                     int32_t task, const ghn_query_out *out, void *workspace, size_t workspace_bytes,
                     cudaStream_t s);

}  // namespace ghn
