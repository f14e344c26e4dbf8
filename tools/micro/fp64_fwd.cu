// Development microbenchmark: FP64 issue rate of DFMA a*b+c by the AGE of its three vector operands
// (whether operands produced by a recent instruction escape the register-bank read limit).
// Many warps per SMSP hide the 8-cycle latency of the dependent chains.
//   mode 0: x = fma(a_k, b_k, x)  per chain; a_k, b_k old, x produced by the previous DFMA of the chain
//   mode 1: x = fma(x, a_k, y), y = fma(y, b_k, x)  two recent operands (x, y) + one old
//   mode 2: x_k = fma(a_k, b_k, x_k), K = 8 independent (all three old)
//   mode 3: x = fma(a_k, x, b_k) ... recent in slot B
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int C>
__global__ void k(int iters, double* out) {
    const double t = threadIdx.x * 1e-9 + blockIdx.x * 1e-12;
    double a[8], b[8], x[C], y[C];
#pragma unroll
    for (int j = 0; j < 8; j++) { a[j] = 1.0 - t * (j + 1); b[j] = 1e-3 + t * (j + 3); }
#pragma unroll
    for (int c = 0; c < C; c++) { x[c] = t + c; y[c] = t - c; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 8; j++)
#pragma unroll
            for (int c = 0; c < C; c++) {
                if (MODE == 0) x[c] = fma(a[j], b[(j + c) & 7], x[c]);
                if (MODE == 1) { const double nx = fma(x[c], a[j], y[c]); y[c] = fma(y[c], b[j], nx); x[c] = nx; }
                if (MODE == 3) x[c] = fma(a[j], x[c], b[(j + c) & 7]);
            }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; c++) s += x[c] + y[c];
#pragma unroll
    for (int j = 0; j < 8; j++) s += a[j] + b[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int C>
void run(int warps_per_smsp) {
    double* out;
    const int blocks = 148, threads = 128 * warps_per_smsp;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int iters = 4000;
    const int fp64 = 8 * C * (MODE == 1 ? 2 : 1);
    k<MODE, C><<<blocks, threads>>>(iters, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE, C><<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double instr = (double)iters * fp64 * blocks * threads / 32.0;
    printf("mode=%d C=%d warps/SMSP=%2d  FP64 issue = %.3f of 0.5/clk/SMSP @1965  %s\n", MODE, C, warps_per_smsp,
           instr / (ms * 1e-3) / (148.0 * 4 * 0.5 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    for (int w : {4, 8}) {
        run<0, 1>(w); run<0, 2>(w); run<0, 8>(w);
        run<1, 1>(w); run<1, 2>(w);
        run<3, 1>(w); run<3, 2>(w);
    }
    return 0;
}
