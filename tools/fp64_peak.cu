// fp64_peak.cu — DFMA throughput microbenchmark (the FP64 roofline denominator; MEASURED_PEAKS.json
// has none).  Every thread runs 8 independent DFMA chains; grid = 148 SMs x 8 CTAs x 256 threads.
// flops = 2 * (#DFMA thread-instructions); best of `reps` launches, CUDA events.
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void __launch_bounds__(256) dfma_loop(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1.2345) out[0] = s;   // keep the chains alive
}

// Returns best DFMA TFLOP/s over `reps` launches (negative on error).
extern "C" double fp64_peak_tflops(int sms, int reps, int iters, double *best_ms) {
    double *out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return -1.0;
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(out, iters / 4 + 1, 0.999999, 1e-7);   // warm-up
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return -2.0;
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    if (best_ms) *best_ms = best;
    return flops / (best * 1e-3) / 1e12;
}
