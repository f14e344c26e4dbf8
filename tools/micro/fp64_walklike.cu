// Development microbenchmark: FP64 pipe rate of walk-like instruction streams (distinct register
// operands per complex multiply, with and without row-sum updates) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cmul2(double& xr, double& xi, double yr, double yi) {
    const double t = xi * yi, u = xi * yr;
    const double nr = fma(xr, yr, -t);
    xi = fma(xr, yi, u);
    xr = nr;
}

template <int R, int K, bool UPD>
__global__ void walklike(int iters, double* out, long long* cyc) {
    double wr[R], wi[R];
#pragma unroll
    for (int i = 0; i < R; i++) { wr[i] = 1.0 + 1e-3 * (threadIdx.x + i); wi[i] = 1e-3 * i; }
    const double cr = 1e-9, ci = -1e-9;
    double ar = 0, ai = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int term = 0; term < 4; term++) {
            if (UPD) {
#pragma unroll
                for (int i = 0; i < R; i++) { wr[i] += (term & 1) ? cr : -cr; wi[i] += (term & 1) ? ci : -ci; }
            }
            double pr[K], pi[K];
#pragma unroll
            for (int k = 0; k < K; k++) { pr[k] = wr[k * (R / K)]; pi[k] = wi[k * (R / K)]; }
#pragma unroll
            for (int k = 0; k < K; k++)
#pragma unroll
                for (int i = k * (R / K) + 1; i < (k + 1) * (R / K); i++) cmul2(pr[k], pi[k], wr[i], wi[i]);
#pragma unroll
            for (int k = 1; k < K; k++) cmul2(pr[0], pi[0], pr[k], pi[k]);
            ar += pr[0];
            ai += pi[0];
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = ar + ai;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int R, int K, bool UPD>
void run(int blocks, int threads) {
    double* out; long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    const int iters = 2000;
    walklike<R, K, UPD><<<blocks, threads>>>(iters, out, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    walklike<R, K, UPD><<<blocks, threads>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    const double fp64_per_term = (UPD ? 2 * R : 0) + 4.0 * (R - 1) + 2;
    const double instr = (double)iters * 4 * fp64_per_term * blocks * threads / 32.0;   // warp instrs
    const double pipe = instr / (ms * 1e-3) / (148 * 4 * 0.5 * 1.965e9);                // vs 0.5/clk/SMSP @ max clock
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, walklike<R, K, UPD>);
    printf("R=%d K=%d upd=%d regs=%d warps/SMSP=%.1f  pipe=%.3f (at 1965 MHz)  %s\n", R, K, (int)UPD, fa.numRegs,
           blocks * threads / 32.0 / 148 / 4, pipe, cudaGetErrorString(err));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {1, 2, 3, 4}) {
        run<22, 2, false>(148, 128 * w);
        run<22, 2, true>(148, 128 * w);
        run<22, 4, true>(148, 128 * w);
        run<44, 2, true>(148, 128 * w);
        run<44, 4, true>(148, 128 * w);
    }
    return 0;
}
