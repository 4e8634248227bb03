// ghn_query_f32.cu -- generic predict kernel instantiations for float indexes.
#include "ghn_query_impl.cuh"

namespace ghn {
int32_t launch_query_f32(const QArgs &a, int ks, cudaStream_t s) { return launch_query<float>(a, ks, s); }
}  // namespace ghn
