// ghn_query_f64.cu -- generic predict kernel instantiations for double indexes.
#include "ghn_query_impl.cuh"

namespace ghn {
int32_t launch_query_f64(const QArgs &a, int ks, cudaStream_t s) { return launch_query<double>(a, ks, s); }
}  // namespace ghn
