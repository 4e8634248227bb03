/*
 * ghn.h -- C ABI of the B200-native Grid Hashing Neighborhood (GHN) path.
 *
 * The reference (gridneighbors, pure Python/numpy) has no FFI: its boundary
 * is the Python API re-exported at pkg/src/gridneighbors/__init__.py:7-36.
 * This library is the native layer under the drop-in Python mirror
 * (paper_2004_02290_b200/), loaded with ctypes.  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *   - every array argument is a DEVICE pointer to caller-owned memory
 *     (PyTorch tensors in the Python layer) unless documented "host";
 *   - `stream` is a cudaStream_t (NULL = legacy default stream);
 *   - return value: GHN_OK or an error code; ghn_last_error() gives a
 *     thread-local message.  GHN_ERR_VALUE maps to the reference's
 *     ValueError, the others to RuntimeError;
 *   - no global mutable state: calls on different streams are independent.
 */
#ifndef GHN_H_
#define GHN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GHN_MAX_DIM 16

enum { GHN_F32 = 0, GHN_F64 = 1 };
enum { GHN_LAYOUT_DENSE = 0, GHN_LAYOUT_LIST = 1 };
enum { GHN_MODE_HEURISTIC = 0, GHN_MODE_GUARANTEED = 1 };           /* explore.py:21 */
/* exact full scan (baselines.brute_knn, baselines.py:40-55; the recall
   oracle of bench.run_bench, bench.py:160-161): every point, no grid walk */
enum { GHN_MODE_BRUTE = 2 };
enum { GHN_TASK_NONE = 0, GHN_TASK_CLASSIFY = 1, GHN_TASK_REGRESS_MEAN = 2, GHN_TASK_REGRESS_MEDIAN = 3 };
enum { GHN_METRIC_EUCLIDEAN = 0, GHN_METRIC_MANHATTAN = 1, GHN_METRIC_CHEBYSHEV = 2 };   /* core.py:16 */
enum { GHN_OK = 0, GHN_ERR_VALUE = 1, GHN_ERR_CUDA = 2, GHN_ERR_UNSUPPORTED = 3 };

/* Thread-local description of the last failure on this thread. */
const char *ghn_last_error(void);
/* ABI version (major*100 + minor). */
int32_t ghn_abi_version(void);
/* Build flags: bit 0 = measurement knobs read from GHN_* environment
 * variables (a -DGHN_TUNING_KNOBS build; the product build ignores the
 * environment), bit 1 = per-site fallback counters (-DGHN_FB_REASONS). */
int32_t ghn_build_flags(void);

/* ------------------------------------------------------------------ fit
 * Replaces grid.build (grid.py:165-195) together with _hash_all
 * (grid.py:124-125) and the finite check of LabeledPoint (core.py:35-36).
 *
 * Phase 1 -- ghn_fit_bounds: per-dimension cell-id bounds lo/hi of
 * floor(x / w) (IEEE fp64), origin = per-dimension minimum coordinate
 * (GridParams.origin, grid.py:109), and a non-finite flag.
 *   X          (n, d) row-major, dtype GHN_F32 or GHN_F64
 *   widths     host, d doubles > 0
 *   out_bounds int64[2*d]: lo[0..d), hi[0..d)
 *   out_origin double[d]
 *   out_flags  int32[1]: bit0 = a non-finite coordinate was seen
 */
int32_t ghn_fit_bounds(const void *X, int32_t dtype, int64_t n, int32_t d, const double *widths,
                       int64_t *out_bounds, double *out_origin, int32_t *out_flags, void *stream);

/* Host-only plan: chooses the cell-table layout from the bounds and sizes
 * the workspace.  DENSE = offsets over the whole id bounding box (E cells);
 * LIST = sorted non-empty cell list only (for huge, sparse boxes). */
typedef struct ghn_fit_plan {
    int64_t n;
    int32_t d;
    int32_t dtype;
    int32_t layout;
    int32_t key_bits;                 /* bits of the dense linear key (DENSE) */
    int64_t E;                        /* cells in the id bounding box (DENSE) */
    double widths[GHN_MAX_DIM];
    int64_t lo[GHN_MAX_DIM];
    int64_t ext[GHN_MAX_DIM];         /* hi - lo + 1 */
    size_t workspace_bytes;
    size_t fast_cursor_off;           /* counting-scatter path: workspace offsets */
    size_t fast_rec_off;
} ghn_fit_plan;

int32_t ghn_fit_plan_init(ghn_fit_plan *plan, int64_t n, int32_t d, int32_t dtype,
                          const double *widths, const int64_t *bounds_host, int64_t dense_limit);

/* Outputs of phase 2.  Capacities: perm n; coords d*n; cell_start n+1;
 * cell_ids n*d; pt_off / ne_off E+1 (DENSE only, else NULL). */
typedef struct ghn_fit_out {
    int32_t *perm;        /* CSR slot -> original point index (= concat(buckets)) */
    void *coords;         /* permuted coordinates, SoA: coords[j*n + slot], dtype */
    int32_t *cell_start;  /* non-empty cell c holds slots [cell_start[c], cell_start[c+1]) */
    int32_t *cell_ids;    /* (C_ne, d) ids relative to lo, lexicographic (= cell_array - lo) */
    int32_t *n_cells;     /* scalar C_ne */
    int32_t *pt_off;      /* DENSE: slots before linear cell key c (E+1) */
    int32_t *ne_off;      /* DENSE: non-empty cells before linear cell key c (E+1) */
    const int32_t *labels_in;  /* optional: label codes in input order */
    int32_t *labels_perm;      /* optional: labels_in gathered into CSR slot order */
} ghn_fit_out;

/* Phase 2: stable LSD radix sort by cell (ties keep input order, as the
 * lexsort of grid.py:188-189), CSR extraction, dense tables, SoA gather. */
int32_t ghn_fit_build(const ghn_fit_plan *plan, const void *X, const ghn_fit_out *out,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Max-splits width fit (grid.fit_cell_measurements, grid.py:94-109): per
 * dimension the largest split count s <= min(#distinct, ceil(2 span /
 * max gap), max_splits) whose s equal bins over [min, max] are all occupied.
 * X (n, d) device, row-major; widths / splits / origin are HOST arrays of d
 * (origin = per-dimension minimum).  max_splits <= 0 means no cap. */
size_t ghn_fit_widths_workspace_size(int64_t n);
int32_t ghn_fit_widths(const void *X, int32_t dtype, int64_t n, int32_t d, int64_t max_splits,
                       double *widths, int64_t *splits, double *origin, void *workspace,
                       size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- query
 * Replaces explore.knn_query (explore.py:66-137) with core.ordering_keys /
 * keys_to_distances (core.py:72-91), batched over nq queries, with the
 * predict.classify / predict.regress(agg="mean") epilogue (predict.py:20-47)
 * fused. */
/* Nested grid of one overfull cell (new; no reference counterpart).  A cell
 * holding more than `sub_min` points is subdivided into ext[0] x ... x
 * ext[d-1] sub-cells of width h over the bounding box of its points, so the
 * predict can find the cell's nearest members without scanning all of them.
 * This changes only which candidates are evaluated, never the result: every
 * skipped sub-cell is provably farther than the current k-th key. */
typedef struct ghn_subgrid {
    double origin[GHN_MAX_DIM];   /* per-dimension minimum of the cell's points */
    double h[GHN_MAX_DIM];        /* sub-cell width (> 0) */
    double inv_h[GHN_MAX_DIM];    /* 1 / h */
    int32_t ext[GHN_MAX_DIM];     /* sub-cells per dimension (>= 1) */
    int64_t off;                  /* first entry of this sub-grid in sub_off */
    int32_t cell;                 /* non-empty cell index (cell_start row) */
    int32_t start;                /* CSR slot range of the cell: [start, start + count) */
    int32_t count;
    int32_t pad;
} ghn_subgrid;

typedef struct ghn_index_view {
    int64_t n;
    int32_t d;
    int32_t dtype;
    int32_t layout;
    int32_t n_cells;
    int64_t E;
    double widths[GHN_MAX_DIM];
    double min_width;
    int64_t lo[GHN_MAX_DIM];
    int64_t ext[GHN_MAX_DIM];
    const void *coords;          /* SoA permuted, dtype */
    const int32_t *perm;
    const int32_t *cell_start;
    const int32_t *cell_ids;
    const int32_t *pt_off;       /* DENSE */
    const int32_t *ne_off;       /* DENSE */
    const int32_t *labels;       /* original point order; classify only */
    const double *targets;       /* original point order; regress only */
    const int32_t *labels_perm;  /* labels in CSR slot order (ghn_gather_i32), or NULL */
    int32_t n_labels;            /* label codes lie in [0, n_labels), or 0 if unknown */
    int32_t metric;              /* GHN_METRIC_*: ordering key and stop bound (core.py:72-91) */
    double density_hint;         /* points per cell the tiled predict sizes its tiles for
                                    (ghn_window_density); 0 = the mean n / E */
    /* nested grids of overfull cells (ghn_subgrid_*), or n_sub = 0 */
    int32_t n_sub;
    int32_t sub_min;             /* cells with more points than this have a sub-grid */
    const int32_t *sub_of_cell;  /* (n_cells) sub-grid id of non-empty cell c, or -1 */
    const ghn_subgrid *subs;     /* (n_sub) */
    const int32_t *sub_off;      /* sub-cell prefix: sub-cell t of grid g holds sub-slots
                                    [sub_off[off_g + t], sub_off[off_g + t + 1]) */
    const void *sub_coords;      /* SoA over n_subpts sub-slots, dtype */
    const int32_t *sub_idx;      /* sub-slot -> original point index */
    int64_t n_subpts;
} ghn_index_view;

typedef struct ghn_query_out {
    double *dist;                /* (nq, k) sqrt(key) fp64, or NULL */
    int64_t *idx;                /* (nq, k) original point index, or NULL */
    int32_t *label;              /* (nq) CLASSIFY: winning label code, or NULL */
    double *confidence;          /* (nq) CLASSIFY: count / k, or NULL */
    double *value;               /* (nq) REGRESS_MEAN / _MEDIAN: the aggregate, or NULL */
    int64_t *stats;              /* (nq, 3) layers_visited, cells_visited, points_scanned, or NULL */
    unsigned long long *totals;  /* [5] += sum layers, cells, points, queries, and candidate keys
                                    evaluated by the generic kernel (a work counter; the tiled
                                    kernels leave it), or NULL */
} ghn_query_out;

/* Workspace for ghn_query / ghn_query_order with nq queries and this k
 * (query binning, the tiled path's tile table and fallback list). */
size_t ghn_query_workspace_size(const ghn_index_view *ix, int64_t nq, int32_t k);

/* K8 query binning (new; the reference loops per query, bench.py:194):
 * order_out[t] = query visited t-th, sorted by central cell (DENSE layout;
 * returns GHN_ERR_UNSUPPORTED for LIST).  Any order gives identical
 * results; this one makes warps on an SM share neighbourhoods. */
int32_t ghn_query_order(const ghn_index_view *ix, const void *Q, int32_t q_dtype, int64_t nq,
                        int32_t *order_out, void *workspace, size_t workspace_bytes, void *stream);

/* Q is (nq, d) row-major, dtype q_dtype (GHN_F32 / GHN_F64, independent of
 * the index dtype: queries are upcast to fp64 like explore.py:83).
 * 1 <= k <= n and k <= 256.  qorder: visit order from ghn_query_order, or
 * NULL to bin internally (when nq is large enough to benefit). */
int32_t ghn_query(const ghn_index_view *ix, const void *Q, int32_t q_dtype, int64_t nq, int32_t k,
                  int32_t mode, int32_t task, const int32_t *qorder, const ghn_query_out *out,
                  void *workspace, size_t workspace_bytes, void *stream);

/* dst[i] = src[idx[i]] for i < n (labels into CSR slot order). */
int32_t ghn_gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst, void *stream);

/* Local point density for tile sizing (new; no reference counterpart): for
 * `samples` points taken at evenly spaced CSR slots (so dense regions are
 * sampled in proportion to their points), the number of points in the
 * (2*radius+1)^2 window of cells around the point's cell, divided by the
 * window's cell count, written to out_density[samples] (device, fp32).
 * 2-D DENSE indexes only (GHN_ERR_UNSUPPORTED otherwise); asynchronous. */
int32_t ghn_window_density(const ghn_index_view *ix, int32_t radius, int32_t samples, float *out_density,
                           void *stream);

/* ---------------------------------------------------------- nested grids
 * Sub-grids for cells holding more than min_points points (SURVEY Appendix B:
 * cfg3's cell (0,0,0,0) holds 36M of 50M points).  Three steps, all device
 * arrays caller-owned:
 *   1. ghn_subgrid_select: the non-empty cells with > min_points points, in
 *      cell order, into cells_out (capacity n / (min_points + 1) + 1), and
 *      their number into *n_out (device int32);
 *   2. ghn_subgrid_bounds: per selected cell the per-dimension min / max of
 *      its points' coordinates (bmin / bmax, n_sub * d doubles each);
 *   3. the caller chooses each grid's resolution and fills ghn_subgrid
 *      records (host logic, copied to the device as `subs`), then
 *      ghn_subgrid_build counts the points per
 *      sub-cell (sub_off, E_tot + 1 entries, E_tot = sum of the grids'
 *      sub-cell counts), scans and scatters them into sub_coords (SoA,
 *      n_subpts = sum of counts) / sub_idx, and marks sub_of_cell.
 * workspace: ghn_subgrid_workspace_size(E_tot) bytes. */
int32_t ghn_subgrid_select(const ghn_index_view *ix, int32_t min_points, int32_t *cells_out, int32_t *n_out,
                           void *stream);
int32_t ghn_subgrid_bounds(const ghn_index_view *ix, const int32_t *cells, int32_t n_sub, double *bmin,
                           double *bmax, void *stream);
size_t ghn_subgrid_workspace_size(int64_t e_tot);
int32_t ghn_subgrid_build(const ghn_index_view *ix, const ghn_subgrid *subs, int32_t n_sub, int64_t e_tot, int32_t *sub_off, void *sub_coords, int32_t *sub_idx,
                          int64_t n_subpts, int32_t *sub_of_cell, void *workspace, size_t workspace_bytes,
                          void *stream);

/* Number of kernels this library has launched in this process (evidence for
 * the bench's gpu_launches; monotone, thread-safe). */
uint64_t ghn_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* GHN_H_ */
