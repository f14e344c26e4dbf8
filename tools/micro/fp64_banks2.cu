// Development microbenchmark: FP64 issue rate vs number of distinct VECTOR register operands.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, double* out) {
    constexpr int K = 8;
    double x[K], y[K], a[K], b[K], c[K];
    const double t = threadIdx.x * 1e-6;
#pragma unroll
    for (int j = 0; j < K; j++) { x[j] = t + j; y[j] = t - j; a[j] = 1.0 - t * j; b[j] = 0.5 + t * j; c[j] = 0.25 + t; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < K; j++) {
            if (MODE == 0) { x[j] = fma(a[j], b[j], x[j]); y[j] = fma(a[j], c[j], y[j]); }   // 3 vec operands each
            if (MODE == 1) { x[j] = x[j] * a[j]; y[j] = y[j] * b[j]; }                        // DMUL 2 operands
            if (MODE == 2) { x[j] = fma(x[j], a[j], 1e-7); y[j] = fma(y[j], b[j], 1e-7); }    // DFMA 2 vec + imm
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < K; j++) s += x[j] + y[j] + a[j] + b[j] + c[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(int warps_per_smsp) {
    double* out;
    const int blocks = 148, threads = 128 * warps_per_smsp;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int iters = 20000;
    k<MODE><<<blocks, threads>>>(iters, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double instr = (double)iters * 16 * blocks * threads / 32.0;
    printf("mode=%d warps/SMSP=%d  FP64 rate = %.3f of 0.5/clk/SMSP at 1965 MHz\n", MODE, warps_per_smsp,
           instr / (ms * 1e-3) / (148.0 * 4 * 0.5 * 1.965e9));
    cudaFree(out);
}

int main() {
    for (int w : {1, 2, 3, 4, 6}) { run<0>(w); run<1>(w); run<2>(w); }
    return 0;
}
