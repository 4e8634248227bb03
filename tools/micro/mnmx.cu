// Microbenchmark: integer vs float min/max bubble throughput / latency on sm_100a.
#include <cstdio>
#include <cstdint>
template <int N, bool FLT>
__global__ void bub(const uint32_t *in, uint32_t *out, int iters, long long *cyc) {
    uint32_t L[N];
    for (int j = 0; j < N; ++j) L[j] = 0x7f7fffffu - j;
    uint32_t v = in[threadIdx.x + blockIdx.x * blockDim.x];
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t x = v ^ (uint32_t)it;
        x &= 0x3fffffffu;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (FLT) {
                float a = __uint_as_float(L[j]), b = __uint_as_float(x);
                L[j] = __float_as_uint(fminf(a, b));
                x = __float_as_uint(fmaxf(a, b));
            } else {
                uint32_t m = min(L[j], x);
                x = max(L[j], x);
                L[j] = m;
            }
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int j = 0; j < N; ++j) s += L[j];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int N, bool FLT>
void run(int blocks, int threads, uint32_t *in, uint32_t *out, long long *cyc) {
    int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    bub<N, FLT><<<blocks, threads>>>(in, out, 10, cyc);
    cudaEventRecord(e0);
    bub<N, FLT><<<blocks, threads>>>(in, out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = 2.0 * N * iters * (double)blocks * threads;   // min+max per slot
    printf("%s N=%d blocks=%d thr=%d: %.3f ms, %.1f Gop/s (%.1f lane-ops/clk/SM @1.965GHz), cycles/iter/warp(b0) %.1f\n",
           FLT ? "FMNMX" : "IMNMX", N, blocks, threads, ms, ops / ms / 1e6, ops / (ms * 1e-3) / 1.965e9 / 148, (double)c / iters);
}
int main() {
    uint32_t *in, *out; long long *cyc;
    cudaMalloc(&in, 1 << 24); cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    cudaMemset(in, 0, 1 << 24);
    run<17, false>(1, 32, in, out, cyc);
    run<17, true>(1, 32, in, out, cyc);
    run<17, false>(148 * 8, 256, in, out, cyc);
    run<17, true>(148 * 8, 256, in, out, cyc);
    run<65, false>(148 * 4, 256, in, out, cyc);
    run<65, true>(148 * 4, 256, in, out, cyc);
    run<65, false>(148 * 2, 128, in, out, cyc);
    run<17, false>(148 * 2, 128, in, out, cyc);
    return 0;
}
