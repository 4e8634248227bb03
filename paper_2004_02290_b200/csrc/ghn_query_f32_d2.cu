// ghn_query_f32_d2.cu -- generic predict kernel, float index, d = 2
// (one translation unit per instantiation family: they compile in parallel).
#include "ghn_query_impl.cuh"

namespace ghn {
int32_t launch_query_f32_d2(const QArgs &a, int ks, cudaStream_t s) { return launch_query_d<float, 2, false>(a, ks, s); }
}  // namespace ghn
