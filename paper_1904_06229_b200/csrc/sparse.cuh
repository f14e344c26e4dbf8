// sparse.cuh -- restricted enumeration for sparse matrices (App. B,
// sparsepermanent P:1254-1266 with greedypartition P:1275-1293, Sec. II-D).
//
// With the column partition D = {S_1, ..., S_d, T} (S_l = the column support of a row, pairwise disjoint),
// every set J of Eq. (3) that misses some S_l leaves that row's sum exactly 0, so
//     per(A) = (-1)^n sum_{s_l subset S_l, s_l != {}} sum_{t subset T} (-1)^{|J|} prod_i sum_{j in J} a_ij,
//     J = s_1 u ... u s_d u t,
// over 2^|T| prod_l (2^|S_l| - 1) sets instead of 2^n.  Here the t-part is walked in Gray order with the
// machinery of walk.cuh: an item is (outer combination o, aligned chunk c of 2^e ranks of the T walk);
// the lanes of a warp take consecutive items, so they share o and walk aligned chunks of the same T
// columns in lock-step (warp-uniform column operands).  Each item seeds its row sums explicitly:
//     w = sum_l sum_{j in s_l(o)} a_{.j} + sum_{q in gray(c 2^e)} a_{.,T_q},
// and the walk accumulates sum_r (-1)^{r+1} prod w (walk_seeded); with |J| = |s| + |gray r| and
// |gray r| = r (mod 2) the item's contribution is -(-1)^{|s|} times that.  Partials: dd per thread ->
// warp -> block -> fixed-order reduction (reduce.cu) with the final factor (-1)^n.
#pragma once
#include <cstring>

#include "walk.cuh"

namespace perm {

struct SparseParams {   // kernel-parameter copy of SparseLaunch
    const double2* A;             // device, row-major n x n
    ddc* partials;                // [gridDim.x]
    uint64_t outer;               // prod_l (2^{|S_l|} - 1)
    uint64_t chunks;              // 2^{nt - e} T-walk chunks per outer combination
    int32_t e;                    // log2 chunk length (0: single terms)
    int32_t nt;                   // |T|
    int32_t d;                    // number of S sets
    int32_t col[64];              // permuted column order: T columns, then S_1, S_2, ...
    int32_t row[64];              // row order: position i holds row row[i] of A
    int32_t soff[kSparseMaxD];    // slot of S_l's first column (in the permuted order)
    int32_t ssz[kSparseMaxD];     // |S_l|
};

// Constant-bank variant (walk.cuh, walk_kernel_c): the T walk's inner U columns ride in the kernel
// parameters (slots 0..U-1 of the permuted order are T's first columns) and reach the row-sum updates as
// uniform-register operands.  Needs a warp-uniform item loop (every lane runs every iteration; lanes past
// the end walk a valid item and drop it) and e > U; the e <= U case keeps the shared-memory walk.
// Orders for which ptxas keeps those loads on the uniform datapath (LDCU -> DADD R, R, UR; scanned with
// PERM_SPARSE_CONST=2, guarded by tests/test_abi_cpu.py); n = 48: 4.96e10 -> 5.55e10 sets/s.
// (sparse_const_path: internal.h)

template <int N>
struct SparseParamsC {
    WalkParamsC<N> w;             // col[][]: inner T columns (w.A, w.partials, c0, count, eb unused)
    SparseParams s;
    // group walk: comb[b - 1][i] = sum_{k in b} a_{row[N-M+i], T slot k}, b = 1 .. 2^G - 1 (subsets of the thin columns)
    double2 comb[(1 << kSparseGroupMaxG) - 1][kSparseGroupRows];
};

// Shared-rows group walk (round 2).  In a sparse matrix most rows are zero in any one column.  The host puts
// G "thin" T columns c_0 .. c_{G-1} -- together nonzero in at most M = kSparseGroupRows rows -- at T slots
// 0 .. G-1 (the walk's lowest Gray bits; any order of the T columns enumerates the same sets) and orders the rows
// so that those rows are the last M positions (per(PA) = per(A)).  The row sums v never hold a thin column; an
// aligned block q of 2^G ranks enumerates every subset b of the thin columns once at fixed high Gray bits h, and
// the rows outside the last M give all 2^G terms the SAME factor:
//     sum over the block = (-1)^{q+1} Z sum_b (-1)^{|b|} prod_{i >= N-M} (v_i + c_b,i),   Z = prod_{i < N-M} v_i,
// (term sign (-1)^{r+1} = -(-1)^{|b|} (-1)^{|h|}; |h| = |gray(r >> G)| = parity of r >> G = q mod 2 in a chunk
// whose first rank is a multiple of 2^e, e > G; App. A).  c_b = the subset sums, from the kernel parameters.
// Per block: one column flip (2N DADD), Z (N - M - 1 complex multiplies), 2^G products of M rows, the signed sum:
// 2N + 4(N - M) + 2^G (4M - 2) + 2 + 4 - ... FP64 instructions for 2^G sets (n = 48, M = 4: 153 / 88 / 55 / 39 per
// set for G = 1 / 2 / 3 / 4 instead of 6N - 4 = 284).  The same sets and terms, summed as signed block sums.
template <class C, int G>
__device__ __forceinline__ void walk_seeded_group(const SparseParamsC<C::N>& PC, uint32_t lc, uint64_t c, int e,
                                                  double (&wr)[C::N], double (&wi)[C::N], ddc& acc) {
    constexpr int N = C::N, M = kSparseGroupRows, Z0 = N - M;
    static_assert(G >= 1 && G <= kSparseGroupMaxG && Z0 >= 4, "group walk");
    const int nblk = 1 << (e - G);                        // e > G: >= 2 blocks, the seed holds no thin column
    const uint64_t cpar = c & 1ull;
    constexpr int kFoldMask = (G >= kWalkFoldBits) ? 0 : ((1 << (kWalkFoldBits - G)) - 1);
    double ar = 0.0, ai = 0.0;
    for (int q = 0; q < nblk; q++) {
        const int z = q >> 30;                            // 0 (nblk <= 2^29); per-use parameter loads
        if (q > 0) {
            const int j = G + __ffs(q) - 1;
            const uint64_t nb = (j + 1 < e) ? (uint64_t)((q >> (j + 1 - G)) & 1) : cpar;
            flip_add<N>(lc + (uint32_t)(j * N) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        double xr, xi, yr, yi, dr, di;
        chain<0, Z0 / 2, N>(wr, wi, xr, xi);
        chain<Z0 / 2, Z0, N>(wr, wi, yr, yi);
        chain<Z0, N, N>(wr, wi, dr, di);                  // b = {}: + prod v
#pragma unroll
        for (int b = 1; b < (1 << G); b++) {
            const int bb = b - 1 + z * b;                 // == b - 1
            double pr = wr[Z0] + PC.comb[bb][0].x, pi = wi[Z0] + PC.comb[bb][0].y;
#pragma unroll
            for (int i = 1; i < M; i++) cmul2(pr, pi, wr[Z0 + i] + PC.comb[bb][i].x, wi[Z0 + i] + PC.comb[bb][i].y);
            if (__builtin_popcount((unsigned)b) & 1) { dr -= pr; di -= pi; }
            else                                      { dr += pr; di += pi; }
        }
        cmul2(yr, yi, dr, di);
        const uint32_t neg = (q & 1) ? 0u : 0x80000000u;  // (-1)^{q+1}, an integer sign flip
        fused_acc<+1>(xr, xi, flip_sign_if(yr, neg), flip_sign_if(yi, neg), ar, ai);
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

// The walk of one aligned chunk c of the T walk (2^e ranks, e > U) from seeded row sums, inner columns
// from the constant bank (as walk_chunk_const), block-boundary columns from shared memory.
template <class C>
__device__ __forceinline__ void walk_seeded_cbank(const WalkParamsC<C::N>& Pw, uint32_t lc, uint64_t c, int e,
                                                 double (&wr)[C::N], double (&wi)[C::N], ddc& acc) {
    constexpr int N = C::N, U = C::U;
    const int nblk = 1 << (e - U);
    const uint64_t cpar = c & 1ull;
    constexpr int kFoldMask = (U >= kWalkFoldBits) ? 0 : ((1 << (kWalkFoldBits - U)) - 1);
    double ar = 0.0, ai = 0.0;
    for (int q = 0; q < nblk; q++) {
        const int z = q >> 30;
        if (q > 0) {
            const int j = U + __ffs(q) - 1;
            const uint64_t nb = (j + 1 < e) ? (uint64_t)((q >> (j + 1 - U)) & 1) : cpar;
            flip_add<N>(lc + (uint32_t)(j * N) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        InnerStepC<C, 0>::run(Pw, z, wr, wi, (q & 1) ? -1.0 : 1.0, ar, ai);
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

template <int N, int G>
__global__ void __launch_bounds__(walk_block_threads(N)) sparse_kernel_c(const __grid_constant__ SparseParamsC<N> PC) {
    using C = WCfg<N, 1>;
    const SparseParams& P = PC.s;
    extern __shared__ double2 smem[];
    for (int k = threadIdx.x; k < N * C::P; k += blockDim.x) {
        const int slot = k / C::P, i = k - slot * C::P;
        const double2 a = (i < N) ? P.A[P.row[i] * N + P.col[slot]] : make_double2(0.0, 0.0);
        smem[k] = a;
        smem[N * C::P + k] = make_double2(-a.x, -a.y);
    }
    __syncthreads();
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem);
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    const uint64_t total = P.outer * P.chunks;
    const uint32_t ln = threadIdx.x & 31u;
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (uint64_t)__shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t base = wid * 32u; base < total; base += nw * 32u) {
        const uint64_t gg = base + ln;
        const bool valid = gg < total;
        const uint64_t g = valid ? gg : base;
        uint64_t o = g / P.chunks;
        const uint64_t c = g - o * P.chunks;
        double wr[N], wi[N];
#pragma unroll
        for (int i = 0; i < N; i++) { wr[i] = 0.0; wi[i] = 0.0; }
        int ssum = 0;
        for (int l = 0; l < P.d; l++) {
            const uint64_t r = (1ull << P.ssz[l]) - 1ull;
            const uint64_t m = o % r + 1ull;
            o /= r;
            for (int q = 0; q < P.ssz[l]; q++) {
                const double f = (double)((m >> q) & 1ull);
                flip_dyn<N>(lc + (uint32_t)((P.soff[l] + q) * C::P) * 16u, f, wr, wi);
            }
            ssum += __popcll(m);
        }
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        const int e = P.e;                                   // > U on this path (sparse_launch_t)
        const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
        for (int q = e - 1; q < P.nt; q++)
            flip_dyn<N>(lc + (uint32_t)(q * C::P) * 16u, (double)((x >> q) & 1ull), wr, wi);
        if constexpr (G > 0) walk_seeded_group<C, G>(PC, lc, c, e, wr, wi, part);
        else                walk_seeded_cbank<C>(PC.w, lc, c, e, wr, wi, part);
        if ((ssum & 1) == 0) {
            part.re.hi = -part.re.hi; part.re.lo = -part.re.lo;
            part.im.hi = -part.im.hi; part.im.lo = -part.im.lo;
        }
        if (valid) acc = ddc_add(acc, part);
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

// Shared-memory sparse walk.  Lanes per item S = walk_lanes_per_chunk(N) (two from n = 33, rows split
// between the lanes exactly as in walk_kernel): the 4n row-sum registers of one lane would not fit next to
// the shared-memory column operands without spilling.  The S lanes of a group walk the same item.
template <int N>
__global__ void __launch_bounds__(WalkCfg<N>::NT, WalkCfg<N>::MINB) sparse_kernel(const __grid_constant__ SparseParams P) {
    using C = WalkCfg<N>;
    constexpr int R = C::R, S = C::S;
    extern __shared__ double2 smem[];
    // stage the permuted columns (slot k = column P.col[k]) and their negations, walk layout
    for (int k = threadIdx.x; k < N * C::P; k += blockDim.x) {
        const int slot = k / C::P, i = k - slot * C::P;
        const double2 a = (i < N) ? P.A[P.row[i] * N + P.col[slot]] : make_double2(0.0, 0.0);
        smem[k] = a;
        smem[N * C::P + k] = make_double2(-a.x, -a.y);
    }
    __syncthreads();
    const uint32_t h = threadIdx.x % S;
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem) + h * (uint32_t)R * 16u;
    // the item's dd partial lives in shared memory (touched once per 2^kWalkFoldBits terms)
    __shared__ ddc spart_[C::NT];
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    const uint64_t total = P.outer * P.chunks;
    const uint64_t W = (uint64_t)gridDim.x * (blockDim.x / S);
    for (uint64_t g = (uint64_t)blockIdx.x * (blockDim.x / S) + threadIdx.x / S; g < total; g += W) {
        uint64_t o = g / P.chunks;
        const uint64_t c = g - o * P.chunks;
        double wr[R], wi[R];
#pragma unroll
        for (int i = 0; i < R; i++) {                      // padding rows (odd n, S = 2) are a neutral factor 1
            wr[i] = ((int)h * R + i < N) ? 0.0 : 1.0;
            wi[i] = 0.0;
        }
        // outer combination o -> non-empty s_l: mixed radix 2^{|S_l|} - 1, digit v -> sub-mask v + 1
        int ssum = 0;
        for (int l = 0; l < P.d; l++) {
            const uint64_t r = (1ull << P.ssz[l]) - 1ull;
            const uint64_t m = o % r + 1ull;
            o /= r;
            for (int q = 0; q < P.ssz[l]; q++) {
                const double f = (double)((m >> q) & 1ull);
                flip_dyn<R>(lc + (uint32_t)((P.soff[l] + q) * C::P) * 16u, f, wr, wi);
            }
            ssum += __popcll(m);
        }
        {
            volatile ddc& z = *(volatile ddc*)&spart_[threadIdx.x];
            z.re.hi = 0.0; z.re.lo = 0.0; z.im.hi = 0.0; z.im.lo = 0.0;
        }
        ddc& part = spart_[threadIdx.x];
        if (P.e == 0) {
            // a single rank r = c of the T walk (|T| < U, or no T at all)
            const uint64_t x = c ^ (c >> 1);
            for (int q = 0; q < P.nt; q++)
                flip_dyn<R>(lc + (uint32_t)(q * C::P) * 16u, (double)((x >> q) & 1ull), wr, wi);
            double ar = 0.0, ai = 0.0;
            if constexpr (S == 1) {
                if (c & 1ull) term_acc<R, C::K, +1>(wr, wi, ar, ai);
                else          term_acc<R, C::K, -1>(wr, wi, ar, ai);
            } else {
                double pr, pi;
                lane_product<R, C::K>(wr, wi, pr, pi);
#pragma unroll
                for (int k = 1; k < S; k <<= 1) {           // butterfly: every lane ends with the full product
                    const double qr = __shfl_xor_sync(group_mask<S>(), pr, k);
                    const double qi = __shfl_xor_sync(group_mask<S>(), pi, k);
                    cmul2(pr, pi, qr, qi);
                }
                if (h == 0) {
                    if (c & 1ull) { ar += pr; ai += pi; }
                    else          { ar -= pr; ai -= pi; }
                }
            }
            part.re = dd_add_d(part.re, ar);
            part.im = dd_add_d(part.im, ai);
        } else {
            const int e = P.e;
            const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
            for (int q = e - 1; q < P.nt; q++)
                flip_dyn<R>(lc + (uint32_t)(q * C::P) * 16u, (double)((x >> q) & 1ull), wr, wi);
            walk_seeded<C>(lc, h, c, e, wr, wi, part);
        }
        ddc pv = part;
        if constexpr (S > 1) {          // the S lanes of a group hold interleaved terms: fixed-order combine
#pragma unroll
            for (int off = S / 2; off > 0; off >>= 1) pv = ddc_add(pv, shfl_down_ddc(pv, off, group_mask<S>()));
        }
        // contribution -(-1)^{|s|} * part
        if ((ssum & 1) == 0) {
            pv.re.hi = -pv.re.hi; pv.re.lo = -pv.re.lo;
            pv.im.hi = -pv.im.hi; pv.im.lo = -pv.im.lo;
        }
        if (h == 0) acc = ddc_add(acc, pv);
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
cudaError_t sparse_launch_t(const SparseLaunch& L) {
    using C = WCfg<N, 1>;
    SparseParams P;
    P.A = L.A_dev;
    P.partials = L.partials;
    P.outer = L.outer;
    P.chunks = L.chunks;
    P.e = L.e;
    P.nt = L.nt;
    P.d = L.d;
    for (int k = 0; k < 64; k++) P.col[k] = k < N ? L.col[k] : 0;
    for (int k = 0; k < 64; k++) P.row[k] = k < N ? L.row[k] : 0;
    for (int l = 0; l < kSparseMaxD; l++) {
        P.soff[l] = l < L.d ? L.soff[l] : 0;
        P.ssz[l] = l < L.d ? L.ssz[l] : 0;
    }
    if constexpr (sparse_const_path(N) && C::U >= 1 && WalkParamsC<N>::MN == 0) {
        if (L.e > C::U) {
            SparseParamsC<N> PC;
            memset(&PC.w, 0, sizeof(PC.w));
            constexpr int NC = WalkParamsC<N>::NC;
            for (int j = 0; j < NC; j++)
                for (int i = 0; i < N; i++) PC.w.col[j][i] = L.A_host[(size_t)L.row[i] * N + L.col[j]];
            PC.s = P;
            memset(PC.comb, 0, sizeof(PC.comb));
            auto kern = sparse_kernel_c<N, 0>;
            if constexpr (sparse_group_path(N)) {
                constexpr int M = kSparseGroupRows;
                for (int b = 1; b < (1 << L.group); b++)
                    for (int i = 0; i < M; i++) {
                        double re = 0.0, im = 0.0;
                        for (int k = 0; k < L.group; k++)
                            if ((b >> k) & 1) {
                                const double2 a = L.A_host[(size_t)L.row[N - M + i] * N + L.col[k]];
                                re += a.x;
                                im += a.y;
                            }
                        PC.comb[b - 1][i] = make_double2(re, im);
                    }
                if (L.group == 1) kern = sparse_kernel_c<N, 1>;
                if (L.group == 2) kern = sparse_kernel_c<N, 2>;
                if (L.group == 3) kern = sparse_kernel_c<N, 3>;
                if (L.group == 4) kern = sparse_kernel_c<N, 4>;
            }
            cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)C::smem_bytes);
            if (err != cudaSuccess) return err;
            kern<<<L.grid, walk_block_threads(N), C::smem_bytes, L.stream>>>(PC);
            return cudaGetLastError();
        }
    }
    cudaError_t err = cudaFuncSetAttribute(sparse_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)WalkCfg<N>::smem_bytes);
    if (err != cudaSuccess) return err;
    sparse_kernel<N><<<L.grid, WalkCfg<N>::NT, WalkCfg<N>::smem_bytes, L.stream>>>(P);
    return cudaGetLastError();
}

// Occupancy of the kernel the launch normally uses: the constant-bank kernel on its orders (the planner sizes
// the grid and the T-walk chunk length from it), else the shared-memory kernel.
template <int N>
cudaError_t sparse_occupancy_t(int* blocks_per_sm) {
    if constexpr (sparse_const_path(N) && WCfg<N, 1>::U >= 1 && WalkParamsC<N>::MN == 0) {
        cudaError_t err = cudaFuncSetAttribute(sparse_kernel_c<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)WCfg<N, 1>::smem_bytes);
        if (err != cudaSuccess) return err;
        err = cudaFuncSetAttribute(sparse_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)WalkCfg<N>::smem_bytes);
        if (err != cudaSuccess) return err;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sparse_kernel_c<N, 0>, walk_block_threads(N),
                                                             WCfg<N, 1>::smem_bytes);
    }
    using C = WalkCfg<N>;
    cudaError_t err = cudaFuncSetAttribute(sparse_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sparse_kernel<N>, C::NT, C::smem_bytes);
}

}  // namespace perm
