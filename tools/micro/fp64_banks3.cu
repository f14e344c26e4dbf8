// Development microbenchmark: is register-read bandwidth a shared per-SMSP budget?  Interleave
// 3-vector-operand DFMAs with DADDs whose second operand is uniform (UR) vs a vector register.
#include <cstdio>
#include <cuda_runtime.h>

struct U8 { double u[8]; };
template <int MODE>
__global__ void k(int iters, const __grid_constant__ U8 uni, double* out) {
    constexpr int K = 8;
    double x[K], y[K], a[K], b[K], v[K];
    const double t = threadIdx.x * 1e-6;
#pragma unroll
    for (int j = 0; j < K; j++) { x[j] = t + j; y[j] = t - j; a[j] = 1.0 - t * j; b[j] = 0.5 + t * j; v[j] = 1e-9 * (t + j); }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < K; j++) {
            x[j] = fma(a[j], b[j], x[j]);                       // 3 vector operands
            if (MODE == 0) y[j] = y[j] + uni.u[j];     // uniform operand (UR after LDCU/ULDC)
            if (MODE == 1) y[j] = y[j] + v[j];                  // vector operand
            if (MODE == 1 && j == 0) v[0] = v[0] * 0.999;       // keep v live/varying (1 extra DMUL)
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < K; j++) s += x[j] + y[j] + a[j] + b[j] + v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(int warps_per_smsp, const U8& uni) {
    double* out;
    const int blocks = 148, threads = 128 * warps_per_smsp;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int iters = 20000;
    k<MODE><<<blocks, threads>>>(iters, uni, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(iters, uni, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double instr = (double)iters * (16 + (MODE == 1 ? 1 : 0)) * blocks * threads / 32.0;
    printf("mode=%d warps/SMSP=%d  FP64 rate = %.3f of 0.5/clk/SMSP at 1965 MHz\n", MODE, warps_per_smsp,
           instr / (ms * 1e-3) / (148.0 * 4 * 0.5 * 1.965e9));
    cudaFree(out);
}

int main() {
    U8 uni;
    for (int i = 0; i < 8; i++) uni.u[i] = 1e-9 * (i + 1);
    for (int w : {2, 3, 4}) { run<0>(w, uni); run<1>(w, uni); }
    return 0;
}
