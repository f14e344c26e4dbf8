// walk_table.cuh -- the single-matrix Gray walk with EVERY row-sum update fed from the kernel-parameter
// constant bank (uniform-register operands), for the orders of walk_table_path(N).
//
// Same method and arithmetic as walk_kernel / walk_kernel_c (walk.cuh; App. A): aligned
// chunks of 2^e ranks, one lane per chunk, seeded from gray(c 2^e) (steps 2, 5-8), then one column add or
// subtract per step (nextset) and the signed product.  What changes is where the
// column operands come from.  The kernel parameters hold a signed column table
//     tab[s][j][i] = (-1)^s a_ij,   s in {0, 1}, j < E = walk_table_cols(N)
// so that every flip of the walk -- the static ones inside the unrolled 2^U block, the mid-block flip whose
// sign is bit_U(rank), and the block-boundary flip of column U + ctz(q) -- is
//     w_i += tab[s][j][i]                       (DADD R, R, UR: one vector register read)
// with (s, j) warp-uniform.  walk_kernel_c takes only the U inner columns from the constant bank; its
// mid-block flip is fma(z, a, w) (two vector reads) and its boundary flip an LDS + DADD with two vector
// reads, which together cost the product DFMAs 4n register reads per block.
//
// Uniform signs need one more thing: the boundary flip of column e-1 (once per chunk, at block
// q = 2^{e-U-1}) takes the sign 1 ^ bit_e(rank) = 1 ^ (c & 1), the chunk's parity (S-2).  The 32 lanes of a
// warp therefore walk 32 chunks of EQUAL parity: items are taken in groups of 64 and a warp pass covers
// the even or the odd half of a group, so c & 1 is warp-uniform (the planner sends a body whose chunk
// count is a multiple of 64).  The boundary flip is the first thing of a block, so that its constant loads
// overlap the first term's product; block 0 of a chunk adds a zero column (w + 0 = w exactly), so the block
// loop body has no branch but the fold.  Only chunk exponents e <= E are walked here (the planner caps b).
#pragma once
#include "walk.cuh"

namespace perm {

template <int N>
struct WalkParamsT {
    static constexpr int E = walk_table_cols(N);
    static constexpr int SG = E * N;          // sign stride (entries)
    double2 tab[2 * E * N + N];               // tab[s*SG + j*N + i] = (-1)^s a_ij; tab[2*SG + i] = 0
    const double2* A;                         // device, row-major (seeding from shared memory)
    ddc* partials;                            // [gridDim.x]
    uint64_t c0;                              // first body chunk
    uint64_t count;                           // body chunks, a multiple of 64
    int32_t eb;                               // log2 body chunk length, U < eb <= E
};
static_assert(sizeof(WalkParamsT<kConstMaxN>) <= 32764, "kernel parameter space");

// w += tab[off .. off + N) (off warp-uniform)
template <int N>
__device__ __forceinline__ void flip_tab(const WalkParamsT<N>& P, int off, double (&wr)[N], double (&wi)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double2 a = P.tab[off + i];
        wr[i] += a.x;
        wi[i] += a.y;
    }
}

template <class C, int T>
struct InnerStepT {
    static constexpr int N = C::N;
    static __device__ __forceinline__ void run(const WalkParamsT<N>& P, int z, int smid, int boff, double (&wr)[N],
                                               double (&wi)[N], double& ar, double& ai) {
        constexpr int U = C::U;
        constexpr int SG = WalkParamsT<N>::SG;
        if constexpr (T == 0) {
            // block-boundary flip into this block (the zero column for the chunk's first block), at the top
            // of the block so that its loads and adds overlap the first term's product
#ifndef PERM_TABLE_MIDFMA
#define PERM_TABLE_MIDFMA 0
#endif
#if PERM_TABLE_BSMEM
            flip_add<N>((uint32_t)boff, wr, wi);          // shared-memory address
#else
            flip_tab<N>(P, boff, wr, wi);
#endif
        } else {
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                // new bit = 1 ^ bit_U(rank): subtract iff bit_U(rank) = smid
#if PERM_TABLE_MIDFMA
                const double zm = smid ? -1.0 : 1.0;
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const double2 a = P.tab[J * N + z * (T + 1) + i];
                    wr[i] = fma(zm, a.x, wr[i]);
                    wi[i] = fma(zm, a.y, wi[i]);
                }
#else
                flip_tab<N>(P, smid * SG + J * N, wr, wi);
#endif
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;  // new bit = 1 ^ bit_{J+1}(t)
                // z * (T + 1) == 0: a distinct opaque offset per use keeps ptxas from hoisting the
                // loop-invariant column into vector registers
#if PERM_TABLE_MIDFMA
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const double2 a = P.tab[J * N + z * (T + 1) + i];
                    if (PLUS) { wr[i] += a.x; wi[i] += a.y; }
                    else      { wr[i] -= a.x; wi[i] -= a.y; }
                }
#else
                flip_tab<N>(P, (PLUS ? 0 : SG) + J * N + z * (T + 1), wr, wi);
#endif
            }
        }
        if constexpr (T & 1) term_acc<N, C::K, +1>(wr, wi, ar, ai);   // sign (-1)^{r+1}, r == t (mod 2)
        else                 term_acc<N, C::K, -1>(wr, wi, ar, ai);
        if constexpr (T + 1 < (1 << U)) InnerStepT<C, T + 1>::run(P, z, smid, boff, wr, wi, ar, ai);
    }
};

// One aligned chunk c of 2^e ranks (U < e <= E); cpar = c & 1 (warp-uniform).
template <class C>
__device__ __forceinline__ void walk_chunk_table(const WalkParamsT<C::N>& P, uint32_t lc, uint32_t lb, uint64_t c,
                                                 int cpar, ddc& acc) {
    constexpr int N = C::N, U = C::U;
    constexpr int SG = WalkParamsT<N>::SG;
    const int e = P.eb;
    double wr[N], wi[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double2 b = lds_c(lb + i * 16);
        wr[i] = b.x;
        wi[i] = b.y;
    }
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    for (int j = e - 1; j < N - 1; j++) {                 // seed, App. A steps 5-8 (shared memory)
        const double f = (double)((x >> j) & 1ull);
        flip_dyn<N>(lc + (uint32_t)(j * N) * 16u, f, wr, wi);
    }
    const int nblk = 1 << (e - U);
    constexpr int kFoldMask = (U >= kWalkFoldBits) ? 0 : ((1 << (kWalkFoldBits - U)) - 1);
    double ar = 0.0, ai = 0.0;
    for (int q = 0; q < nblk; q++) {
        const int z = q >> 30;                            // 0 (nblk <= 2^19); uniform, loop-variant
        // boundary flip into block q: Gray bit j = U + ctz(q) flips to 1 ^ bit_{j+1}(rank) (j = e - 1:
        // bit_e = chunk parity); block 0 adds the zero column
        const int j = U + __ffs(q) - 1;
        const int s = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1) : cpar;
#if PERM_TABLE_BSMEM
        const int boff = (int)lc + ((q == 0) ? 2 * N * N * 16 : (s * N * N + j * N) * 16);
#else
        const int boff = (q == 0) ? 2 * SG : s * SG + j * N;
#endif
        InnerStepT<C, 0>::run(P, z, q & 1, boff, wr, wi, ar, ai);   // bit_U(rank) = q & 1 (e > U)
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

// Register cap of walk_kernel_t for order N (0: uncapped).  ptxas keeps the per-use parameter loads on
// the uniform datapath only for some register allocations (tools/const_ldcu_scan.sh --table).
__host__ __device__ constexpr int walk_table_maxnreg(int n) {
#ifdef PERM_TABLE_MAXNREG_ALL
    return PERM_TABLE_MAXNREG_ALL;
#else
    return n == 44 ? 216 : 0;
#endif
}

template <int N>
__global__ void __launch_bounds__(kTableThreads) __maxnreg__(walk_table_maxnreg(N) > 0 ? walk_table_maxnreg(N) : 255)
    walk_kernel_t(const __grid_constant__ WalkParamsT<N> P) {
    using C = WCfg<N, 1>;
    extern __shared__ double2 smem[];
    double2* scol = smem;                                    // scol[j*N + i] = a_ij (seeding only)
#if PERM_TABLE_BSMEM
    double2* sbase = smem + 2 * N * N + N;                   // after -a_ij (+N*N) and a zero column (+2*N*N)
    for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
        const int i = k / N, j = k - i * N;
        const double2 a = P.A[k];
        scol[j * N + i] = a;
        scol[N * N + j * N + i] = make_double2(-a.x, -a.y);
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) scol[2 * N * N + i] = make_double2(0.0, 0.0);
#else
    double2* sbase = smem + N * N;
    for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
        const int i = k / N, j = k - i * N;
        scol[j * N + i] = P.A[k];
    }
#endif
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {     // App. A step 5, summed in column order
        double sr = 0.0, si = 0.0;
        for (int j = 0; j < N; j++) {
            sr += scol[j * N + i].x;
            si += scol[j * N + i].y;
        }
        sbase[i] = make_double2(scol[(N - 1) * N + i].x - 0.5 * sr, scol[(N - 1) * N + i].y - 0.5 * si);
    }
    __syncthreads();
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(scol);
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(sbase);
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    // warp pass over 32 items of one parity: items [g64, g64 + 64) of a group, lane l takes item
    // g64 + 2l + h (h = pass parity), i.e. chunk c0 + g64 + 2l + h, whose parity (c0 + h) & 1 is uniform
    const uint32_t ln = threadIdx.x & 31u;
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (uint64_t)__shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t base = wid * 32u; base < P.count; base += nw * 32u) {
        const uint64_t h = (base >> 5) & 1ull;
        const uint64_t c = P.c0 + (base & ~63ull) + 2u * ln + h;
        const int cpar = (int)((P.c0 + h) & 1ull);
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        walk_chunk_table<C>(P, lc, lb, c, cpar, part);
        acc = ddc_add(acc, part);
    }
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

template <int N>
constexpr size_t walk_table_smem() { return (size_t)(PERM_TABLE_BSMEM ? 2 * N * N + 2 * N : N * N + N) * sizeof(double2); }

template <int N>
cudaError_t walk_launch_table(const WalkLaunch& L) {
    const Segment& b = L.seg[L.body];
    WalkParamsT<N> P;
    constexpr int E = WalkParamsT<N>::E, SG = WalkParamsT<N>::SG;
    for (int j = 0; j < E; j++)
        for (int i = 0; i < N; i++) {
            const double2 a = L.A_host[(size_t)i * N + j];
            P.tab[j * N + i] = a;
            P.tab[SG + j * N + i] = make_double2(-a.x, -a.y);
        }
    for (int i = 0; i < N; i++) P.tab[2 * SG + i] = make_double2(0.0, 0.0);
    P.A = L.A_dev;
    P.partials = L.partials;
    P.c0 = b.c0;
    P.count = b.count;
    P.eb = b.e;
    walk_kernel_t<N><<<L.grid, kTableThreads, walk_table_smem<N>(), L.stream>>>(P);
    return cudaGetLastError();
}

template <int N>
cudaError_t walk_occupancy_table(int* blocks_per_sm) {
    cudaError_t err = cudaFuncSetAttribute(walk_kernel_t<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)walk_table_smem<N>());
    if (err != cudaSuccess) return err;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, walk_kernel_t<N>, kTableThreads,
                                                         walk_table_smem<N>());
}

}  // namespace perm
