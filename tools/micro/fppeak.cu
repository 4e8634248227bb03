// Microbenchmark: FP64 / FP32 add and multiply issue throughput on sm_100a
// (the FP-pipe roofline denominators for the compute-bound predicts, cfg2 /
// cfg3).  Each thread runs 8 independent dependency chains of mul-then-add
// (no FMA, as in the ordering keys, core.py:78-80), so the pipes -- not the
// latency -- bound the loop.  Prints one JSON line; ops count each add and
// each multiply as one operation.
#include <cstdio>
#include <cuda_runtime.h>

template <typename F>
__global__ void chains(F *out, F a, F b, int iters) {
    F x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = (F)(threadIdx.x + c);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (sizeof(F) == 8) {
                x[c] = __dadd_rn(__dmul_rn((double)x[c], (double)a), (double)b);
            } else {
                x[c] = __fadd_rn(__fmul_rn((float)x[c], (float)a), (float)b);
            }
        }
    }
    F s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double rate(int sms) {
    F *out;
    cudaMalloc(&out, sizeof(F) * sms * 8 * 256);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<F><<<sms * 8, 256>>>(out, (F)0.999999, (F)1e-7, 64);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        chains<F><<<sms * 8, 256>>>(out, (F)0.999999, (F)1e-7, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * 8 * iters * (double)sms * 8 * 256;
        if (ops / (ms * 1e-3) > best) best = ops / (ms * 1e-3);
    }
    cudaFree(out);
    return best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double f64 = rate<double>(sms), f32 = rate<float>(sms);
    printf("{\"fp64_add_mul_gops\": %.1f, \"fp32_add_mul_gops\": %.1f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
           "\"how\": \"tools/micro/fppeak.cu: 8 independent mul->add chains per thread, no FMA, %d CTAs x 256, best of 5\"}\n",
           f64 / 1e9, f32 / 1e9, sms, clk / 1e3, sms * 8);
    return 0;
}
