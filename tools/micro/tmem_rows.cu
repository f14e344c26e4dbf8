// Development microbenchmark: can TMEM hold part of a thread's row sums at walk-like rates?
// 3 CTAs x 128 threads per SM (12 warps, <= 168 registers).  Per iteration each thread loads R complex
// values (4R 32-bit columns) from its TMEM lane, adds a constant (DADD), stores them back, and does F
// independent DFMA of FP64 work (the product chains of the walk).  Compare mode 1 (TMEM round trip)
// with mode 0 (the same values kept in registers, only possible for small R).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int R, int F, int MODE>
__global__ void __launch_bounds__(128, 3) k(int iters, double* out) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (MODE == 1) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                         :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)), "n"(64));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    // lane field (bits 31:16) = this warp's 32-lane quadrant; columns in bits 15:0
    const uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16);
    double acc[F], x[F];
#pragma unroll
    for (int f = 0; f < F; f++) { acc[f] = threadIdx.x * 1e-9 + f; x[f] = 1.0 + 1e-12 * f; }
    double w[2 * R];
#pragma unroll
    for (int r = 0; r < 2 * R; r++) w[r] = r * 0.5;
    if (MODE == 1) {
#pragma unroll
        for (int c = 0; c < R; c += 2) {   // store 2 complex = 8 columns at a time
            uint32_t v[8];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const double d = w[2 * c + q];
                v[2 * q] = (uint32_t)__double_as_longlong(d);
                v[2 * q + 1] = (uint32_t)(__double_as_longlong(d) >> 32);
            }
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                         :: "r"(taddr + 4 * c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                            "r"(v[6]), "r"(v[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    for (int it = 0; it < iters; it++) {
        if (MODE == 1) {
#pragma unroll
            for (int c = 0; c < R; c += 2) {
                uint32_t v[8];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                               "=r"(v[7])
                             : "r"(taddr + 4 * c));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    double d = __longlong_as_double(((long long)v[2 * q + 1] << 32) | v[2 * q]);
                    d += 1e-9;
                    acc[q % F] = fma(acc[q % F], x[q % F], d);
                    v[2 * q] = (uint32_t)__double_as_longlong(d);
                    v[2 * q + 1] = (uint32_t)(__double_as_longlong(d) >> 32);
                }
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                             :: "r"(taddr + 4 * c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                                "r"(v[6]), "r"(v[7]));
            }
        } else {
#pragma unroll
            for (int r = 0; r < 2 * R; r++) {
                w[r] += 1e-9;
                acc[r % F] = fma(acc[r % F], x[r % F], w[r]);
            }
        }
#pragma unroll
        for (int rep = 0; rep < 8; rep++)
#pragma unroll
            for (int f = 0; f < F; f++) acc[f] = fma(acc[f], x[f], 1e-15);
    }
    double s = 0;
#pragma unroll
    for (int f = 0; f < F; f++) s += acc[f];
#pragma unroll
    for (int r = 0; r < 2 * R; r++) s += w[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (MODE == 1) {
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tbase), "n"(64));
    }
}

template <int R, int F, int MODE>
void run() {
    double* out;
    const int blocks = 148 * 3, threads = 128;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    const int iters = 4000;
    k<R, F, MODE><<<blocks, threads>>>(iters, out);
    cudaError_t e0e = cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<R, F, MODE><<<blocks, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<R, F, MODE>);
    // FP64 instructions per iteration: 2R DADD + 2R DFMA (updates) + 8F DFMA
    const double fp64 = (double)iters * (4.0 * R + 8.0 * F) * blocks * threads / 32.0;
    printf("R=%2d F=%d mode=%d regs=%d  FP64 pipe %.3f of 0.5/clk/SMSP @1965  %.3f ms  %s %s\n", R, F, MODE, fa.numRegs,
           fp64 / (ms * 1e-3) / (148.0 * 4 * 0.5 * 1.965e9), ms, cudaGetErrorString(e0e),
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<12, 8, 0>();
    run<12, 8, 1>();
    run<12, 16, 0>();
    run<12, 16, 1>();
    run<16, 16, 1>();
    return 0;
}
