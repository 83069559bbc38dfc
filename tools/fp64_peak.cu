// FP64 FMA throughput microbenchmark ("FP64 ... microbenchmark
// it").  Each thread runs U independent DFMA chains for ITER steps; grid =
// SMs x 4 CTAs of 256 threads.  flops = 2 x threads x U x ITER.  Timed with
// CUDA events after a warm-up launch; prints TFLOP/s and the per-SM rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void k_dfma(double* out, int iter, double a, double b) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = threadIdx.x * 1e-3 + u;
    for (int i = 0; i < iter; ++i) {
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = fma(x[u], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) s += x[u];
    if (s == 1234.5) out[0] = s;  // keep the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    constexpr int U = 8;
    const int iter = 1 << 16, tpb = 256;
    for (int per_sm : {1, 2, 4, 8}) {
        const int grid = sms * per_sm;
        k_dfma<U><<<grid, tpb>>>(out, 64, 0.999999, 1e-9);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_dfma<U><<<grid, tpb>>>(out, iter, 0.999999, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double flops = 2.0 * grid * tpb * (double)U * iter;
        const double tf = flops / (ms * 1e-3) / 1e12;
        printf("{\"ctas_per_sm\": %d, \"threads\": %d, \"ms\": %.3f, \"fp64_tflops\": %.3f, "
               "\"dfma_per_clk_per_sm\": %.2f, \"sm_count\": %d, \"clock_khz_attr\": %d}\n",
               per_sm, grid * tpb, ms, tf, flops / 2.0 / (ms * 1e-3) / sms / (clk * 1e3), sms, clk);
    }
    return 0;
}
