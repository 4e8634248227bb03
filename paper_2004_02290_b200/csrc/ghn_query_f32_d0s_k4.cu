// ghn_query_f32_d0s_k4.cu -- generic predict kernel, float index, runtime d, nested grids, 4 top-k entries per lane
// (one translation unit per instantiation: they compile in parallel).
#include "ghn_query_impl.cuh"

namespace ghn {
int32_t launch_query_f32_d0s_k4(const QArgs &a, cudaStream_t s) { return launch_query_one<float, 0, 4, true>(a, s); }
}  // namespace ghn
