// fp64_mix.cu — FP64 pipe microbenchmarks: DFMA-only, DADD-only, DMUL-only, 1:1 mixes, and the
// effect of warps per SM and chain count.  Prints warp-instructions/cycle/SM achieved.
#include <cuda_runtime.h>
#include <stdio.h>

template <int MODE, int CH>
__global__ void kmix(double *out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (MODE == 0) x[c] = fma(x[c], a, b);
                if (MODE == 1) x[c] = x[c] + b;
                if (MODE == 2) x[c] = x[c] * a;
                if (MODE == 3) { x[c] = fma(x[c], a, b); x[c] = x[c] + b; }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345) out[0] = s;
}

template <int MODE, int CH>
void run(const char *name, int blocks_per_sm, int threads, int iters) {
    double *out;
    cudaMalloc(&out, 8);
    int sms = 148;
    kmix<MODE, CH><<<sms * blocks_per_sm, threads>>>(out, 10, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kmix<MODE, CH><<<sms * blocks_per_sm, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    double ninst = (double)iters * 8 * CH * (MODE == 3 ? 2 : 1) * sms * blocks_per_sm * (threads / 32);
    double cycles = best * 1e-3 * 1965e6;
    printf("%-10s ch=%d warps/SM=%3d : %.3f warp-inst/clk/SM (at 1965 MHz), %.2f ms\n", name, CH,
           blocks_per_sm * threads / 32, ninst / cycles / sms, best);
    cudaFree(out);
}

int main() {
    run<0, 8>("dfma", 8, 256, 2000);
    run<1, 8>("dadd", 8, 256, 2000);
    run<2, 8>("dmul", 8, 256, 2000);
    run<3, 8>("dfma+dadd", 8, 256, 1000);
    run<0, 1>("dfma", 8, 256, 2000);
    run<0, 2>("dfma", 8, 256, 2000);
    run<0, 4>("dfma", 4, 256, 2000);
    run<0, 1>("dfma", 4, 256, 4000);
    run<0, 2>("dfma", 4, 256, 4000);
    run<0, 2>("dfma", 3, 256, 4000);
    run<0, 1>("dfma", 3, 256, 4000);
    run<1, 1>("dadd", 4, 256, 4000);
    run<1, 2>("dadd", 3, 256, 4000);
    return 0;
}
