// ghn_subgrid.cu -- nested grids for overfull cells (fit side).
//
// The reference scans every point of every visited cell (explore.py:104-111);
// a cell holding most of the data (cfg3: 36M of 50M points in cell
// (0,0,0,0)) makes that a brute-force scan per query.
// Here such a cell gets its own uniform sub-grid over the bounding box of its
// points, with a CSR of sub-cells and an SoA copy of the points in sub-cell
// order, so the predict (ghn_query.cu) walks sub-cell rings around the query
// and skips sub-cells whose lower-bound key exceeds the current k-th key.  The
// candidate SET each layer contributes is unchanged, so results are too.
#include <string.h>

#include "ghn_common.cuh"

namespace ghn {
namespace {

constexpr int SG_THREADS = 256;

__global__ void subgrid_select_kernel(const int32_t *__restrict__ cell_start, int32_t n_cells, int32_t min_points,
                                      int32_t *cells_out, int32_t *n_out) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
         c += (int64_t)gridDim.x * blockDim.x) {
        if (cell_start[c + 1] - cell_start[c] > min_points) cells_out[atomicAdd(n_out, 1)] = (int32_t)c;
    }
}

__global__ void bounds_init_kernel(unsigned long long *bmin, unsigned long long *bmax, int64_t m) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        bmin[i] = ~0ull;
        bmax[i] = 0ull;
    }
}

__global__ void bounds_final_kernel(unsigned long long *bmin, unsigned long long *bmax, int64_t m) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = dbl_from_order_key(bmin[i]), b = dbl_from_order_key(bmax[i]);
        bmin[i] = (unsigned long long)__double_as_longlong(a);
        bmax[i] = (unsigned long long)__double_as_longlong(b);
    }
}

// blockIdx.y strides over the selected cells, blockIdx.x over each cell's points.
template <typename T>
__global__ void __launch_bounds__(SG_THREADS) subgrid_bounds_kernel(const T *__restrict__ coords, int64_t n, int d,
                                                                   const int32_t *__restrict__ cell_start,
                                                                   const int32_t *__restrict__ cells, int32_t n_sub,
                                                                   unsigned long long *bmin, unsigned long long *bmax) {
    for (int g = blockIdx.y; g < n_sub; g += gridDim.y) {
        const int32_t c = cells[g];
        const int32_t s0 = cell_start[c], s1 = cell_start[c + 1];
        for (int j = 0; j < d; ++j) {
            double mn = INFINITY, mx = -INFINITY;
            for (int64_t s = s0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < s1;
                 s += (int64_t)gridDim.x * blockDim.x) {
                const double v = to_double(coords[(int64_t)j * n + s]);
                mn = fmin(mn, v);
                mx = fmax(mx, v);
            }
            mn = warp_min(mn);
            mx = warp_max(mx);
            if ((threadIdx.x & 31) == 0 && mn <= mx) {
                atomicMin(&bmin[(int64_t)g * d + j], dbl_order_key(mn));
                atomicMax(&bmax[(int64_t)g * d + j], dbl_order_key(mx));
            }
        }
    }
}

// Sub-cell of a coordinate: floor((x - o) / h), clamped into the grid.  The
// query side only needs valid per-sub-cell bounding boxes (ghn_query.cu
// widens them by a relative slack), not this exact assignment.
__device__ __forceinline__ int32_t sub_coord(double x, double o, double inv_h, int32_t ext) {
    double t = floor(__dmul_rn(__dsub_rn(x, o), inv_h));
    t = fmin(fmax(t, 0.0), (double)(ext - 1));
    return (int32_t)t;
}

template <typename T>
__device__ __forceinline__ int64_t sub_key(const T *__restrict__ coords, int64_t n, int d, int64_t slot,
                                           const ghn_subgrid &g) {
    int64_t key = 0;
    for (int j = 0; j < d; ++j)
        key = key * g.ext[j] + sub_coord(to_double(coords[(int64_t)j * n + slot]), g.origin[j], g.inv_h[j], g.ext[j]);
    return g.off + key;
}

template <typename T>
__global__ void __launch_bounds__(SG_THREADS) subgrid_count_kernel(const T *__restrict__ coords, int64_t n, int d,
                                                                  const ghn_subgrid *__restrict__ subs, int32_t n_sub,
                                                                  int32_t *counts) {
    for (int gi = blockIdx.y; gi < n_sub; gi += gridDim.y) {
        const ghn_subgrid g = subs[gi];
        for (int64_t s = g.start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < (int64_t)g.start + g.count;
             s += (int64_t)gridDim.x * blockDim.x)
            atomicAdd(&counts[sub_key(coords, n, d, s, g)], 1);
    }
}

template <typename T>
__global__ void __launch_bounds__(SG_THREADS) subgrid_scatter_kernel(const T *__restrict__ coords, int64_t n, int d,
                                                                    const int32_t *__restrict__ perm,
                                                                    const ghn_subgrid *__restrict__ subs, int32_t n_sub,
                                                                    int32_t *cursor, T *sub_coords, int64_t F,
                                                                    int32_t *sub_idx) {
    for (int gi = blockIdx.y; gi < n_sub; gi += gridDim.y) {
        const ghn_subgrid g = subs[gi];
        for (int64_t s = g.start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < (int64_t)g.start + g.count;
             s += (int64_t)gridDim.x * blockDim.x) {
            const int32_t pos = atomicAdd(&cursor[sub_key(coords, n, d, s, g)], 1);
            for (int j = 0; j < d; ++j) sub_coords[(int64_t)j * F + pos] = coords[(int64_t)j * n + s];
            sub_idx[pos] = perm[s];
        }
    }
}

__global__ void subgrid_mark_kernel(const ghn_subgrid *__restrict__ subs, int32_t n_sub, int32_t *sub_of_cell) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n_sub; g += gridDim.x * blockDim.x)
        sub_of_cell[subs[g].cell] = g;
}

__global__ void fill_i32_kernel(int32_t *p, int64_t m, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

unsigned grid_for(int64_t m) {
    int64_t g = (m + SG_THREADS - 1) / SG_THREADS;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace
}  // namespace ghn

using namespace ghn;

extern "C" int32_t ghn_subgrid_select(const ghn_index_view *ix, int32_t min_points, int32_t *cells_out,
                                      int32_t *n_out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    GHN_CUDA_CHECK(cudaMemsetAsync(n_out, 0, 4, s));
    if (ix->n_cells <= 0) return GHN_OK;
    subgrid_select_kernel<<<grid_for(ix->n_cells), SG_THREADS, 0, s>>>(ix->cell_start, ix->n_cells, min_points,
                                                                        cells_out, n_out);
    GHN_LAUNCH_CHECK("subgrid_select_kernel");
    return GHN_OK;
}

extern "C" int32_t ghn_subgrid_bounds(const ghn_index_view *ix, const int32_t *cells, int32_t n_sub, double *bmin,
                                      double *bmax, void *stream) {
    if (n_sub <= 0) return GHN_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t m = (int64_t)n_sub * ix->d;
    unsigned long long *kmin = (unsigned long long *)bmin, *kmax = (unsigned long long *)bmax;
    bounds_init_kernel<<<grid_for(m), SG_THREADS, 0, s>>>(kmin, kmax, m);
    GHN_LAUNCH_CHECK("bounds_init_kernel");
    const dim3 grid(32, (unsigned)(n_sub < 4096 ? n_sub : 4096));
    if (ix->dtype == GHN_F32)
        subgrid_bounds_kernel<float><<<grid, SG_THREADS, 0, s>>>((const float *)ix->coords, ix->n, ix->d,
                                                                  ix->cell_start, cells, n_sub, kmin, kmax);
    else
        subgrid_bounds_kernel<double><<<grid, SG_THREADS, 0, s>>>((const double *)ix->coords, ix->n, ix->d,
                                                                   ix->cell_start, cells, n_sub, kmin, kmax);
    GHN_LAUNCH_CHECK("subgrid_bounds_kernel");
    bounds_final_kernel<<<grid_for(m), SG_THREADS, 0, s>>>(kmin, kmax, m);
    GHN_LAUNCH_CHECK("bounds_final_kernel");
    return GHN_OK;
}

extern "C" size_t ghn_subgrid_workspace_size(int64_t e_tot) {
    return a256((size_t)(e_tot + 1) * 4) + a256(scan_workspace_bytes(e_tot + 1)) + 256;
}

extern "C" int32_t ghn_subgrid_build(const ghn_index_view *ix, const ghn_subgrid *subs, int32_t n_sub,
                                     int64_t e_tot, int32_t *sub_off, void *sub_coords, int32_t *sub_idx,
                                     int64_t n_subpts, int32_t *sub_of_cell, void *workspace,
                                     size_t workspace_bytes, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ix->n_cells > 0) {
        fill_i32_kernel<<<grid_for(ix->n_cells), SG_THREADS, 0, s>>>(sub_of_cell, ix->n_cells, -1);
        GHN_LAUNCH_CHECK("fill_i32_kernel");
    }
    if (n_sub <= 0) return GHN_OK;
    if (e_tot <= 0 || e_tot >= 0x7fffffffLL || n_subpts >= 0x7fffffffLL) {
        set_error("sub-grid sizes out of range (E_tot=%lld, points=%lld)", (long long)e_tot, (long long)n_subpts);
        return GHN_ERR_VALUE;
    }
    if (!workspace || workspace_bytes < ghn_subgrid_workspace_size(e_tot)) {
        set_error("sub-grid workspace too small");
        return GHN_ERR_VALUE;
    }
    int32_t *cursor = (int32_t *)workspace;
    void *sws = (char *)workspace + a256((size_t)(e_tot + 1) * 4);
    GHN_CUDA_CHECK(cudaMemsetAsync(sub_off, 0, (size_t)(e_tot + 1) * 4, s));
    const dim3 grid(64, (unsigned)(n_sub < 4096 ? n_sub : 4096));
    if (ix->dtype == GHN_F32)
        subgrid_count_kernel<float><<<grid, SG_THREADS, 0, s>>>((const float *)ix->coords, ix->n, ix->d, subs, n_sub,
                                                                 sub_off);
    else
        subgrid_count_kernel<double><<<grid, SG_THREADS, 0, s>>>((const double *)ix->coords, ix->n, ix->d, subs,
                                                                  n_sub, sub_off);
    GHN_LAUNCH_CHECK("subgrid_count_kernel");
    int32_t rc = exclusive_scan_i32(sub_off, sub_off, e_tot + 1, sws, s);
    if (rc) return rc;
    GHN_CUDA_CHECK(cudaMemcpyAsync(cursor, sub_off, (size_t)e_tot * 4, cudaMemcpyDeviceToDevice, s));
    if (ix->dtype == GHN_F32)
        subgrid_scatter_kernel<float><<<grid, SG_THREADS, 0, s>>>((const float *)ix->coords, ix->n, ix->d, ix->perm,
                                                                   subs, n_sub, cursor, (float *)sub_coords,
                                                                   n_subpts, sub_idx);
    else
        subgrid_scatter_kernel<double><<<grid, SG_THREADS, 0, s>>>((const double *)ix->coords, ix->n, ix->d,
                                                                    ix->perm, subs, n_sub, cursor,
                                                                    (double *)sub_coords, n_subpts, sub_idx);
    GHN_LAUNCH_CHECK("subgrid_scatter_kernel");
    subgrid_mark_kernel<<<grid_for(n_sub), SG_THREADS, 0, s>>>(subs, n_sub, sub_of_cell);
    GHN_LAUNCH_CHECK("subgrid_mark_kernel");
    return GHN_OK;
}
