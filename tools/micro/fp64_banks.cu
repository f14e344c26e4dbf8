// Development microbenchmark: does a DFMA with three distinct 64-bit register operands issue at the
// FP64 pipe rate on sm_100a?  (register-bank / operand-collector limits)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, const double* __restrict__ in, double* out) {
    constexpr int K = 8;
    double x[K], a[K], b[K];
#pragma unroll
    for (int j = 0; j < K; j++) { x[j] = in[j]; a[j] = in[8 + j]; b[j] = in[16 + j]; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < K; j++) {
            if (MODE == 0) x[j] = fma(x[j], a[0], b[0]);          // shared operands (reuse)
            if (MODE == 1) x[j] = fma(a[j], b[j], x[j]);          // 3 distinct operands
            if (MODE == 2) x[j] = x[j] * a[j];                    // DMUL, 2 distinct
            if (MODE == 3) x[j] = x[j] + a[j];                    // DADD, 2 distinct
        }
        // perturb a, b every iteration so nothing is loop-invariant (adds 2*K DADD per 8*? ...)
        if (MODE == 1 && (it & 15) == 15) {
#pragma unroll
            for (int j = 0; j < K; j++) { a[j] = a[j] * 0.5 + x[j] * 1e-30; }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < K; j++) s += x[j] + a[j] + b[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(int warps_per_smsp) {
    double *in, *out;
    cudaMalloc(&in, 64 * sizeof(double));
    double h[64];
    for (int i = 0; i < 64; i++) h[i] = 1.0 + 1e-3 * i;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const int blocks = 148, threads = 128 * warps_per_smsp;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int iters = 20000;
    k<MODE><<<blocks, threads>>>(iters, in, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(iters, in, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double extra = (MODE == 1) ? 8.0 * 2 / 16 : 0.0;   // perturbation DMUL+DFMA per 16 iters
    const double instr = (double)iters * (8 + extra) * blocks * threads / 32.0;
    printf("mode=%d warps/SMSP=%d  FP64 warp-instr rate = %.3f of 0.5/clk/SMSP at 1965 MHz\n", MODE, warps_per_smsp,
           instr / (ms * 1e-3) / (148.0 * 4 * 0.5 * 1.965e9));
}

int main() {
    for (int w : {1, 2, 4}) { run<0>(w); run<1>(w); run<2>(w); run<3>(w); }
    return 0;
}
