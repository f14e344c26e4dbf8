// Development microbenchmark: FP64 latency / issue behaviour on sm_100a.
// Usage: fp64_lat   (prints one line per configuration)
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(int iters, double* out, long long* cyc) {
    double x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = threadIdx.x * 1e-3 + k;
    const double a = 0.9999999, b = 1e-7;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++)
#pragma unroll
            for (int k = 0; k < K; k++) x[k] = fma(x[k], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// complex multiply chain (the walk's product structure): K independent complex chains
template <int K>
__global__ void cchains(int iters, double* out, long long* cyc) {
    double xr[K], xi[K];
#pragma unroll
    for (int k = 0; k < K; k++) { xr[k] = threadIdx.x * 1e-3 + k; xi[k] = 0.5 - k * 1e-3; }
    const double yr = 0.6, yi = 0.8;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++)
#pragma unroll
            for (int k = 0; k < K; k++) {
                const double t = xi[k] * yi, v = xi[k] * yr;
                const double nr = fma(xr[k], yr, -t);
                xi[k] = fma(xr[k], yi, v);
                xr[k] = nr;
            }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s += xr[k] + xi[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <class F>
void run(const char* name, F kern, int K, int fp64_per_iter_per_thread, int blocks, int threads) {
    double* out; long long* cyc;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    const int iters = 4000;
    kern<<<blocks, threads>>>(iters, out, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    double instr_per_thread = (double)iters * fp64_per_iter_per_thread;
    double warps_per_smsp = (double)blocks * threads / 32.0 / 148.0 / 4.0;
    // FP64 warp-instructions per cycle per SMSP (block 0's clock): peak 0.5
    double ipc = instr_per_thread * warps_per_smsp / (double)c;
    printf("%-8s K=%d warps/SMSP=%.2f  cycles/dep-step=%.2f  fp64 warp-instr/clk/SMSP=%.3f  (%.2f TFLOP/s-equiv)\n",
           name, K, warps_per_smsp, (double)c / (iters * 8.0), ipc,
           instr_per_thread * blocks * threads * 2.0 / (ms * 1e-3) / 1e12);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    // latency: 1 warp per SM, 1 chain
    run("dfma", chains<1>, 1, 8 * 1, 148, 32);
    run("dfma", chains<2>, 2, 8 * 2, 148, 32);
    run("dfma", chains<4>, 4, 8 * 4, 148, 32);
    run("dfma", chains<8>, 8, 8 * 8, 148, 32);
    for (int w : {1, 2, 3, 4}) {
        run("dfma", chains<1>, 1, 8, 148, 128 * w);
        run("dfma", chains<2>, 2, 16, 148, 128 * w);
        run("dfma", chains<4>, 4, 32, 148, 128 * w);
    }
    run("cmul", cchains<1>, 1, 8 * 4, 148, 32);
    for (int w : {1, 2, 3, 4}) {
        run("cmul", cchains<1>, 1, 32, 148, 128 * w);
        run("cmul", cchains<2>, 2, 64, 148, 128 * w);
        run("cmul", cchains<4>, 4, 128, 148, 128 * w);
    }
    return 0;
}
