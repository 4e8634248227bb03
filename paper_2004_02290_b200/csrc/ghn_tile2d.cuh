// ghn_tile2d.cuh -- tiled thread-per-query predict for 2-D DENSE grids.
#pragma once

#include "ghn_common.cuh"

namespace ghn {

struct Tile2dPlan {
    int32_t T;        // tile side in cells
    int32_t A;        // apron (layers staged around the tile)
    int32_t nt0, nt1; // tiles per dimension
    int64_t ntiles;
    int32_t win;      // T + 2A
    int32_t G;        // lanes per query (32: warp kernel; 8/16: group kernel; 1: thread kernels)
    int32_t nb;       // neighbours instead of the vote (thread kernel, list rounds)
    int32_t cap;      // staged points per CTA
    size_t smem;      // dynamic shared memory per CTA
};

// Whether the tiled path applies (2-D, DENSE, fp32; the fused vote without
// neighbour output, or -- k <= 32 -- the neighbours alone) and its geometry
// for this k.
// want_stats: QueryStats / totals are requested (the bucket select then stages one more apron layer).
bool tile2d_plan(const ghn_index_view *ix, int64_t nq, int32_t k, int32_t task, bool want_neighbors, bool want_stats,
                 Tile2dPlan *plan);
size_t tile2d_workspace_bytes(const Tile2dPlan *p, int64_t nq);
// Bins the queries by tile and launches the tiled kernel; queries it cannot
// answer land in (*fb_list, *fb_count) for the generic kernel.
int32_t tile2d_run(const ghn_index_view *ix, const Tile2dPlan *plan, const void *Q, int32_t q_dtype,
                   int64_t nq, int32_t k, int32_t mode, const ghn_query_out *out, const double *inv_w,
                   uint32_t pow2, void *workspace, int32_t **fb_list, int32_t **fb_count,
                   cudaStream_t s);

}  // namespace ghn
