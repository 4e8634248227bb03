// ghn_query_f64.cu -- generic predict kernel dispatch for double indexes
// (runtime-d instantiations only).
#include "ghn_query.cuh"

namespace ghn {
int32_t launch_query_f64_d0(const QArgs &a, int ks, cudaStream_t s);
int32_t launch_query_f64_d0s_k1(const QArgs &a, cudaStream_t s);
int32_t launch_query_f64_d0s_k2(const QArgs &a, cudaStream_t s);
int32_t launch_query_f64_d0s_k4(const QArgs &a, cudaStream_t s);
int32_t launch_query_f64_d0s_k8(const QArgs &a, cudaStream_t s);

static int32_t launch_query_f64_d0s(const QArgs &a, int ks, cudaStream_t s) {
    switch (ks) {
        case 1: return launch_query_f64_d0s_k1(a, s);
        case 2: return launch_query_f64_d0s_k2(a, s);
        case 4: return launch_query_f64_d0s_k4(a, s);
        default: return launch_query_f64_d0s_k8(a, s);
    }
}

int32_t launch_query_f64(const QArgs &a, int ks, cudaStream_t s) {
    return a.ix.n_sub > 0 ? launch_query_f64_d0s(a, ks, s) : launch_query_f64_d0(a, ks, s);
}
}  // namespace ghn
