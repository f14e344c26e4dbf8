// reduce.cu -- fixed-order double-double reduction of per-block partials and
// the FP64 peak probe.
//
// The partials of one walk launch are added by ONE block: thread t adds partials t, t+256, ...
// sequentially in dd, then a fixed binary tree over the 256 thread sums.  The order depends only on
// the partial count, so results are bit-reproducible and the paper's advice to keep the
// partial sums in an array and sum them compensated is followed.  For a whole permanent
// the factor 2(-1)^n of App. A permanent step 4 is applied here; it is exact in dd.
#include "internal.h"

namespace perm {

constexpr int kReduceThreads = 256;

__global__ void __launch_bounds__(kReduceThreads) reduce_kernel(const ddc* __restrict__ parts, int count,
                                                                int n_final, ddc* __restrict__ out_dd,
                                                                double2* __restrict__ out_c) {
    __shared__ ddc s[kReduceThreads];
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    for (int k = threadIdx.x; k < count; k += kReduceThreads) acc = ddc_add(acc, parts[k]);
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int off = kReduceThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) s[threadIdx.x] = ddc_add(s[threadIdx.x], s[threadIdx.x + off]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ddc r = s[0];
        if (n_final > 0) {
            const double f = (n_final & 1) ? -2.0 : 2.0;   // 2 (-1)^n, exact
            r.re.hi *= f; r.re.lo *= f; r.im.hi *= f; r.im.lo *= f;
        }
        if (out_dd) *out_dd = r;
        if (out_c) out_c[0] = make_double2(r.re.hi + r.re.lo, r.im.hi + r.im.lo);
    }
}

cudaError_t reduce_launch(const ddc* parts, int count, int n_final, ddc* out_dd, double2* out_c, cudaStream_t s) {
    reduce_kernel<<<1, kReduceThreads, 0, s>>>(parts, count, n_final, out_dd, out_c);
    return cudaGetLastError();
}

// FP64 peak probe: 8 independent DFMA chains per thread (enough ILP to cover the DFMA latency at
// moderate occupancy).  Flops = blocks * threads * iters * 8 * 2.
__global__ void fp64_probe_kernel(int iters, double* __restrict__ sink) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 0.1, x2 = x0 + 0.2, x3 = x0 + 0.3;
    double x4 = x0 + 0.4, x5 = x0 + 0.5, x6 = x0 + 0.6, x7 = x0 + 0.7;
    const double a = 0.9999999, b = 1e-7;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

cudaError_t fp64_probe_launch(int blocks, int threads, int iters, double* sink, cudaStream_t s) {
    // each loop iteration issues 4 x 8 = 32 DFMA per thread
    fp64_probe_kernel<<<blocks, threads, 0, s>>>(iters, sink);
    return cudaGetLastError();
}

}  // namespace perm
