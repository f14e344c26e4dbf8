// walk.cuh -- the Gray-walk kernel for one complex matrix.
//
// Method (App. A): the 2^{n-1} half-range Ryser/Glynn terms
//     term(r) = (-1)^{r+1} prod_i w_i(gray r),   w_i(x) = a_{i,n} - 1/2 sum_j a_ij + sum_{j<n, x_j=1} a_ij
// are cut into ALIGNED chunks of 2^e consecutive ranks (P:1077-1095 distributes contiguous ranges;
// we additionally align them, R5).  For an aligned chunk c (ranks c 2^e .. c 2^e + 2^e - 1):
//   * the seed is w(gray(c 2^e)), gray(c 2^e) = (gray(c) << e) | ((c & 1) << (e-1))   (steps 2, 5-8)
//   * step s -> s+1 flips Gray bit j = ctz(s+1) to 1 ^ bit_{j+1}(c 2^e + s + 1)        (nextset)
//   * the term sign is (-1)^{s+1} because c 2^e is even                               (steps 3, 11-12)
// so every step except the one at s+1 = 2^{e-1} is IDENTICAL for all chunks: the lanes of a warp walk
// 32 different chunks in lock-step and every column operand is warp-uniform (a broadcast LDS.128 with
// a uniform-register address).  Within a chunk a block of 2^U ranks is fully unrolled, so its flips
// (columns 0..U-1) use compile-time shared-memory offsets and compile-time signs; the flip at the
// block boundary (column j >= U, once per 2^U terms) uses a dynamic column and sign.
//
// Per term: 2n DADD/DFMA (row-sum update) + 4(n-2) DMUL/DFMA (product, split
// into K independent chains) + 4 DFMA (last multiply fused with the signed accumulation)
// = 6n-4 FP64 instructions for ~8n flops.  The n row sums live in registers (4n 32-bit registers).
// Column operands are loaded with ld.volatile.shared right before use: this keeps ptxas from
// hoisting/CSE-ing the (loop-invariant) columns into registers, which at n = 44 would need another
// 4n registers per column and spill.  Each 2^U-term block is summed in plain double and folded into
// a per-thread double-double accumulator (TwoSum), then reduced warp -> block -> per-block partial
// in HBM; reduce.cu adds the partials in a fixed order.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace perm {

template <int N>
struct WalkCfg {
    static constexpr int U = walk_inner_bits(N);
    static constexpr int NT = kWalkThreads;
#ifdef PERM_WALK_K
    static constexpr int K = N >= 16 ? PERM_WALK_K : (N >= 4 ? 2 : 1);
#else
    static constexpr int K = N >= 16 ? 2 : (N >= 4 ? 2 : 1);  // independent product chains
#endif
    static constexpr size_t smem_bytes = (size_t)(N * N + N) * sizeof(double2);
};

struct WalkParams {
    const double2* A;                      // device, row-major
    ddc* partials;                         // [gridDim.x]
    uint64_t seg_c0[kMaxSegments];
    uint64_t seg_pre[kMaxSegments + 1];    // prefix item counts
    int32_t seg_e[kMaxSegments];
    int32_t nseg;
};

// Broadcast load of one complex entry from shared memory (volatile: never hoisted or merged).
__device__ __forceinline__ double2 lds_c(uint32_t addr) {
    double2 v;
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

// (xr + i xi) *= (yr + i yi): 2 DMUL + 2 DFMA.
__device__ __forceinline__ void cmul2(double& xr, double& xi, double yr, double yi) {
    const double t = xi * yi;
    const double u = xi * yr;
    const double nr = fma(xr, yr, -t);
    xi = fma(xr, yi, u);
    xr = nr;
}

// Product of rows [B, E) into (pr, pi).
template <int B, int E, int N>
__device__ __forceinline__ void chain(const double (&wr)[N], const double (&wi)[N], double& pr, double& pi) {
    pr = wr[B];
    pi = wi[B];
#pragma unroll
    for (int i = B + 1; i < E; i++) cmul2(pr, pi, wr[i], wi[i]);
}

// acc += SIGN * prod_i w_i.   The last complex multiply is fused with the accumulation (4 DFMA).
template <int N, int SIGN>
__device__ __forceinline__ void term_acc(const double (&wr)[N], const double (&wi)[N], double& ar, double& ai) {
    constexpr int K = WalkCfg<N>::K;
    if constexpr (N == 1) {
        if (SIGN > 0) { ar += wr[0]; ai += wi[0]; } else { ar -= wr[0]; ai -= wi[0]; }
    } else {
        double xr, xi, yr, yi;
        if constexpr (K == 1) {
            chain<0, N - 1, N>(wr, wi, xr, xi);
            yr = wr[N - 1];
            yi = wi[N - 1];
        } else if constexpr (K == 2) {
            chain<0, N / 2, N>(wr, wi, xr, xi);
            chain<N / 2, N, N>(wr, wi, yr, yi);
        } else {
            constexpr int q = N / 4;
            double r0, i0, r1, i1, r2, i2, r3, i3;
            chain<0, q, N>(wr, wi, r0, i0);
            chain<q, 2 * q, N>(wr, wi, r1, i1);
            chain<2 * q, 3 * q, N>(wr, wi, r2, i2);
            chain<3 * q, N, N>(wr, wi, r3, i3);
            cmul2(r0, i0, r1, i1);
            cmul2(r2, i2, r3, i3);
            xr = r0; xi = i0; yr = r2; yi = i2;
        }
        if (SIGN > 0) {
            ar = fma(xr, yr, ar);
            ar = fma(-xi, yi, ar);
            ai = fma(xr, yi, ai);
            ai = fma(xi, yr, ai);
        } else {
            ar = fma(-xr, yr, ar);
            ar = fma(xi, yi, ar);
            ai = fma(-xr, yi, ai);
            ai = fma(-xi, yr, ai);
        }
    }
}

// w += z * column (column at shared address col), z = +-1 (or 0/1 when seeding) as a double.
template <int N>
__device__ __forceinline__ void flip_dyn(uint32_t col, double z, double (&wr)[N], double (&wi)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double2 a = lds_c(col + i * 16);
        wr[i] = fma(z, a.x, wr[i]);
        wi[i] = fma(z, a.y, wi[i]);
    }
}

// w += column J (PLUS) or w -= column J, compile-time column and sign.
template <int N, int J, bool PLUS>
__device__ __forceinline__ void flip_static(uint32_t sc, double (&wr)[N], double (&wi)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double2 a = lds_c(sc + (J * N + i) * 16);
        if (PLUS) { wr[i] += a.x; wi[i] += a.y; }
        else      { wr[i] -= a.x; wi[i] -= a.y; }
    }
}

// Inner block: ranks t = 0 .. 2^U - 1 of the current block (t = 0 already seeded/flipped).
template <int N, int U, int T>
struct InnerStep {
    static __device__ __forceinline__ void run(uint32_t sc, double (&wr)[N], double (&wi)[N], double zmid,
                                               double& ar, double& ai) {
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                // new bit = 1 ^ bit_U(rank): depends on the block (or chunk) parity -> signed by zmid
                flip_dyn<N>(sc + (uint32_t)(J * N) * 16u, zmid, wr, wi);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;  // new bit = 1 ^ bit_{J+1}(t)
                flip_static<N, J, PLUS>(sc, wr, wi);
            }
        }
        if constexpr (T & 1) term_acc<N, +1>(wr, wi, ar, ai);   // sign (-1)^{r+1}, r == t (mod 2)
        else                 term_acc<N, -1>(wr, wi, ar, ai);
        if constexpr (T + 1 < (1 << U)) InnerStep<N, U, T + 1>::run(sc, wr, wi, zmid, ar, ai);
    }
};

// Seed w = base + sum_{j in [j0, N-1), bit_j(x) = 1} column_j   (App. A steps 5-8; branch-free in j).
template <int N>
__device__ __forceinline__ void seed_rows(uint32_t sc, uint32_t sbase, uint64_t x, int j0, double (&wr)[N],
                                          double (&wi)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double2 b = lds_c(sbase + i * 16);
        wr[i] = b.x;
        wi[i] = b.y;
    }
    for (int j = j0; j < N - 1; j++) {
        const double f = (double)((x >> j) & 1ull);
        flip_dyn<N>(sc + (uint32_t)(j * N) * 16u, f, wr, wi);
    }
}

// One aligned chunk of 2^e ranks (e >= U >= 1).
template <int N>
__device__ __forceinline__ void walk_chunk(uint32_t sc, uint32_t sbase, uint64_t c, int e, ddc& acc) {
    constexpr int U = WalkCfg<N>::U;
    double wr[N], wi[N];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    seed_rows<N>(sc, sbase, x, e - 1, wr, wi);
    const uint64_t nblk = 1ull << (e - U);
    const uint64_t cpar = c & 1ull;
    for (uint64_t q = 0; q < nblk; q++) {
        if (q > 0) {
            // block boundary: Gray bit j = U + ctz(q) flips to 1 ^ bit_{j+1}(rank)
            const int j = U + __ffsll((long long)q) - 1;
            const uint64_t nb = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1ull) : cpar;
            flip_dyn<N>(sc + (uint32_t)(j * N) * 16u, nb ? -1.0 : 1.0, wr, wi);
        }
        const uint64_t nbm = (U < e) ? (q & 1ull) : cpar;   // bit_U(rank) for the mid-block flip
        const double zmid = nbm ? -1.0 : 1.0;
        double ar = 0.0, ai = 0.0;
        InnerStep<N, U, 0>::run(sc, wr, wi, zmid, ar, ai);
        acc.re = dd_add_d(acc.re, ar);
        acc.im = dd_add_d(acc.im, ai);
    }
}

// A single rank r, seeded from scratch.
template <int N>
__device__ __forceinline__ void single_term(uint32_t sc, uint32_t sbase, uint64_t r, ddc& acc) {
    double wr[N], wi[N];
    seed_rows<N>(sc, sbase, r ^ (r >> 1), 0, wr, wi);
    double ar = 0.0, ai = 0.0;
    if (r & 1ull) term_acc<N, +1>(wr, wi, ar, ai);
    else          term_acc<N, -1>(wr, wi, ar, ai);
    acc.re = dd_add_d(acc.re, ar);
    acc.im = dd_add_d(acc.im, ai);
}

// Stage A column-major into shared memory (sc[j*N + i] = a_ij) and compute the App. A step-5 base
// vector w_i(0) = a_{i,n} - 1/2 sum_j a_ij (summed in column order j = 0..n-1).
template <int N>
__device__ __forceinline__ void stage_matrix(const double2* __restrict__ A, double2* sc, double2* sbase) {
    for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
        const int i = k / N, j = k - i * N;
        sc[j * N + i] = A[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        double sr = 0.0, si = 0.0;
        for (int j = 0; j < N; j++) {
            sr += sc[j * N + i].x;
            si += sc[j * N + i].y;
        }
        sbase[i] = make_double2(sc[(N - 1) * N + i].x - 0.5 * sr, sc[(N - 1) * N + i].y - 0.5 * si);
    }
    __syncthreads();
}

template <int N>
__global__ void __launch_bounds__(WalkCfg<N>::NT) walk_kernel(const __grid_constant__ WalkParams P) {
    extern __shared__ double2 smem[];
    stage_matrix<N>(P.A, smem, smem + N * N);
    const uint32_t sc = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sbase = sc + (uint32_t)(N * N) * 16u;

    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t total = P.seg_pre[P.nseg];
    int s = 0;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += T) {
        while (g >= P.seg_pre[s + 1]) s++;
        const uint64_t c = P.seg_c0[s] + (g - P.seg_pre[s]);
        const int e = P.seg_e[s];
        if constexpr (WalkCfg<N>::U >= 1) {
            if (e == 0) single_term<N>(sc, sbase, c, acc);
            else        walk_chunk<N>(sc, sbase, c, e, acc);
        } else {
            single_term<N>(sc, sbase, c, acc);
        }
    }

    // warp -> block reduction of the dd partials, fixed order.
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
    __shared__ ddc swarp[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) swarp[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        ddc b = swarp[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) b = ddc_add(b, swarp[w]);
        P.partials[blockIdx.x] = b;
    }
}

// Diagnostic: w(ranks[k]) via the same seeding code (perm_c128_seed).
template <int N>
__global__ void seed_kernel(const double2* __restrict__ A, const uint64_t* __restrict__ ranks, int count,
                            double2* __restrict__ out) {
    extern __shared__ double2 smem[];
    stage_matrix<N>(A, smem, smem + N * N);
    const uint32_t sc = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sbase = sc + (uint32_t)(N * N) * 16u;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
        const uint64_t r = ranks[k];
        double wr[N], wi[N];
        seed_rows<N>(sc, sbase, r ^ (r >> 1), 0, wr, wi);
#pragma unroll
        for (int i = 0; i < N; i++) out[(size_t)k * N + i] = make_double2(wr[i], wi[i]);
    }
}

template <int N>
cudaError_t walk_launch(const WalkLaunch& L) {
    using C = WalkCfg<N>;
    WalkParams P;
    P.A = L.A_dev;
    P.partials = L.partials;
    uint64_t pre = 0;
    for (int s = 0; s < kMaxSegments; s++) {
        P.seg_pre[s] = pre;
        if (s < L.nseg) {
            P.seg_c0[s] = L.seg[s].c0;
            P.seg_e[s] = L.seg[s].e;
            pre += L.seg[s].count;
        } else {
            P.seg_c0[s] = 0;
            P.seg_e[s] = 0;
        }
    }
    P.seg_pre[kMaxSegments] = pre;
    P.nseg = L.nseg;
    cudaError_t err = cudaFuncSetAttribute(walk_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    walk_kernel<N><<<L.grid, C::NT, C::smem_bytes, L.stream>>>(P);
    return cudaGetLastError();
}

template <int N>
cudaError_t walk_occupancy(int* blocks_per_sm, int* threads_per_block) {
    using C = WalkCfg<N>;
    cudaError_t err = cudaFuncSetAttribute(walk_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    *threads_per_block = C::NT;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, walk_kernel<N>, C::NT, C::smem_bytes);
}

template <int N>
cudaError_t walk_seed_launch(const double2* A_dev, const uint64_t* ranks_dev, int count, double2* w_out,
                             cudaStream_t s) {
    using C = WalkCfg<N>;
    cudaError_t err = cudaFuncSetAttribute(seed_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    int grid = (count + 127) / 128;
    if (grid < 1) grid = 1;
    seed_kernel<N><<<grid, 128, C::smem_bytes, s>>>(A_dev, ranks_dev, count, w_out);
    return cudaGetLastError();
}

}  // namespace perm
