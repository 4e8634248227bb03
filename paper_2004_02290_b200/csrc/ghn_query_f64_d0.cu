// ghn_query_f64_d0.cu -- generic predict kernel, double index, d = runtime
// (one translation unit per instantiation family: they compile in parallel).
#include "ghn_query_impl.cuh"

namespace ghn {
int32_t launch_query_f64_d0(const QArgs &a, int ks, cudaStream_t s) { return launch_query_d<double, 0, false>(a, ks, s); }
}  // namespace ghn
