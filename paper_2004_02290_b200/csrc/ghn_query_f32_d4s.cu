// ghn_query_f32_d4s.cu -- generic predict kernel, float index, d = 4, nested grids
// (one translation unit per instantiation family: they compile in parallel).
#include "ghn_query_impl.cuh"

namespace ghn {
int32_t launch_query_f32_d4s(const QArgs &a, int ks, cudaStream_t s) { return launch_query_d<float, 4, true>(a, ks, s); }
}  // namespace ghn
