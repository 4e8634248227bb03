// ghn_query_f32.cu -- generic predict kernel dispatch for float indexes.
// Kernels are specialised for the dimensions the configs use (2, 3, 4, 6);
// everything else runs the runtime-d instantiation -- same arithmetic, loops
// not unrolled.  Indexes with nested grids run the SUB instantiations (d = 4
// specialised: cfg3).
#include "ghn_query.cuh"

namespace ghn {
int32_t launch_query_f32_d2(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f32_d3(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f32_d4(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f32_d6(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f32_d0(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f32_d4s(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f32_d0s_k1(const QArgs &a, cudaStream_t s);
int32_t launch_query_f32_d0s_k2(const QArgs &a, cudaStream_t s);
int32_t launch_query_f32_d0s_k4(const QArgs &a, cudaStream_t s);
int32_t launch_query_f32_d0s_k8(const QArgs &a, cudaStream_t s);

static int32_t launch_query_f32_d0s(const QArgs &a, int ks, cudaStream_t s) {
    switch (ks) {
        case 1: return launch_query_f32_d0s_k1(a, s);
        case 2: return launch_query_f32_d0s_k2(a, s);
        case 4: return launch_query_f32_d0s_k4(a, s);
        default: return launch_query_f32_d0s_k8(a, s);
    }
}

int32_t launch_query_f32(const QArgs &a, int ks, cudaStream_t s) {
    if (a.ix.n_sub > 0) return a.ix.d == 4 ? launch_query_f32_d4s(a, ks, s) : launch_query_f32_d0s(a, ks, s);
    switch (a.ix.d) {
        case 2: return launch_query_f32_d2(a, ks, s);
        case 3: return launch_query_f32_d3(a, ks, s);
        case 4: return launch_query_f32_d4(a, ks, s);
        case 6: return launch_query_f32_d6(a, ks, s);
        default: return launch_query_f32_d0(a, ks, s);
    }
}
}  // namespace ghn
