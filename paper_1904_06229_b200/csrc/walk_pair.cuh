// walk_pair.cuh -- the single-matrix Gray walk with each chunk's rows split between a PAIR OF WARPS
// (lane l of warp 2p and lane l of warp 2p+1 walk the same chunk), for the orders whose 4n registers of
// row sums would otherwise leave only two warps per scheduler (n = 40..48).
//
// Same method and arithmetic as walk_kernel (walk.cuh; App. A).  Warp role h = warp & 1
// keeps rows [h R, h R + R) (R = n/2): its row-sum updates and its half of every product -- together the
// same FP64 instruction count per term as one lane walking all rows.  After every two terms the roles
// exchange one partial product through shared memory (one 64-thread named barrier per pair, double-
// buffered slots): role 0 finishes the even term, role 1 the odd one (the last multiply fused with the
// signed sum).  Unlike the two-lanes-per-chunk layout (WCfg<N, 2>) the role is warp-uniform, so it is a
// compile-time parameter -- no selects, no shuffles -- and each scheduler runs warps of one role only
// (warp w sits on scheduler w % 4).  Halving the row-sum registers gives three 128-thread CTAs per SM.
//
// Every lane of both warps must reach every barrier: the kernel walks only the aligned body segment
// (all chunks of one length 2^eb) with a warp-uniform item loop (lanes past the end walk chunk c0 and
// drop the result); the planner sends the unaligned head/tail to walk_kernel.
#pragma once
#include "walk.cuh"

namespace perm {

template <int N>
struct PCfg {
    using C = WCfg<N, 2>;                            // R = ceil(N/2) rows per role, P = 2R padded rows
    static constexpr int NT = 128;                   // 2 pairs of warps
    static constexpr int MINB = 3;
    // +/- columns and base vector (walk layout) + exchange slots [2 buffers][2 pairs][2 roles][32] double2
    static constexpr size_t smem_bytes = C::smem_bytes + (size_t)2 * 2 * 2 * 32 * sizeof(double2);
};

struct WalkParamsP {
    const double2* A;      // device, row-major
    ddc* partials;         // [gridDim.x]
    uint64_t c0;           // first body chunk
    uint64_t count;        // body chunks
    int32_t eb;            // log2 body chunk length (> U)
};

__device__ __forceinline__ void pair_barrier(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// Inner block of 2^U ranks for role H (rows [H R, H R + R)); pr/pi hold this role's partial products of
// the block's two most recent terms; every odd t exchanges and finishes one term.
template <class C, int T, int H>
struct InnerStepP {
    static constexpr int R = C::R;
    static __device__ __forceinline__ void run(uint32_t lc, uint32_t lmid, double (&wr)[R], double (&wi)[R],
                                               double& ar, double& ai, double (&pr)[2], double (&pi)[2],
                                               double2* ex, int bar, uint32_t& buf) {
        constexpr int U = C::U;
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                flip_add<R>(lmid, wr, wi);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
                flip_static<R, PLUS>(lc + (uint32_t)(J * C::P) * 16u, wr, wi);
            }
        }
        lane_product<R, C::K>(wr, wi, pr[T & 1], pi[T & 1]);
        if constexpr (T & 1) {
            // exchange: role 0 hands over its partial of the odd term, role 1 of the even term
            const int lane = threadIdx.x & 31;
            double2* mine = ex + buf * 64 + H * 32 + lane;
            double2* other = ex + buf * 64 + (1 - H) * 32 + lane;
            *mine = make_double2(pr[1 - H], pi[1 - H]);
            pair_barrier(bar);
            const double2 q = *other;
            buf ^= 1u;
            // term sign (-1)^{t+1}: the even term (role 0) is subtracted, the odd one (role 1) added
            if constexpr (H == 0) fused_acc<-1>(pr[0], pi[0], q.x, q.y, ar, ai);
            else                  fused_acc<+1>(pr[1], pi[1], q.x, q.y, ar, ai);
        }
        if constexpr (T + 1 < (1 << U)) InnerStepP<C, T + 1, H>::run(lc, lmid, wr, wi, ar, ai, pr, pi, ex, bar, buf);
    }
};

template <int N, int H>
__device__ __forceinline__ void walk_chunk_p(uint32_t lc, uint32_t lb, uint64_t c, int e, double2* ex, int bar,
                                             uint32_t& buf, ddc& acc) {
    using C = typename PCfg<N>::C;
    constexpr int U = C::U, R = C::R;
    double wr[R], wi[R];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    seed_rows<C>(lc, lb, x, e - 1, wr, wi);
    const int nblk = 1 << (e - U);
    const uint32_t cpar = (uint32_t)(c & 1ull);
    constexpr int kFoldMask = (U >= kWalkFoldBits) ? 0 : ((1 << (kWalkFoldBits - U)) - 1);
    double ar = 0.0, ai = 0.0, pr[2], pi[2];
    for (int q = 0; q < nblk; q++) {
        if (q > 0) {
            const int j = U + __ffs(q) - 1;
            const uint32_t nb = (j + 1 < e) ? (uint32_t)((q >> (j + 1 - U)) & 1) : cpar;
            flip_add<R>(lc + (uint32_t)(j * C::P) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        const uint32_t lmid = lc + (uint32_t)((U - 1) * C::P) * 16u + ((q & 1) ? C::NEG : 0u);   // e > U
        InnerStepP<C, 0, H>::run(lc, lmid, wr, wi, ar, ai, pr, pi, ex, bar, buf);
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

template <int N, int H>
__device__ __forceinline__ void walk_body_p(const WalkParamsP& P, uint32_t lc0, uint32_t lb0, double2* ex, int bar,
                                            ddc& acc) {
    using C = typename PCfg<N>::C;
    const uint32_t hoff = (uint32_t)H * (uint32_t)C::R * 16u;
    const uint32_t lc = lc0 + hoff, lb = lb0 + hoff;
    const int lane = threadIdx.x & 31, pair = threadIdx.x >> 6;
    const uint64_t wid = (uint64_t)blockIdx.x * 2 + (uint64_t)pair;       // pair index (32 walkers each)
    const uint64_t nw = (uint64_t)gridDim.x * 2;
    uint32_t buf = 0;
    for (uint64_t base = wid * 32u; base < P.count; base += nw * 32u) {   // uniform over the pair
        const uint64_t g = base + (uint64_t)lane;
        const bool valid = g < P.count;
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        walk_chunk_p<N, H>(lc, lb, P.c0 + (valid ? g : 0), P.eb, ex, bar, buf, part);
        if (valid) acc = ddc_add(acc, part);
    }
}

template <int N>
__global__ void __launch_bounds__(PCfg<N>::NT, PCfg<N>::MINB) walk_kernel_p(const __grid_constant__ WalkParamsP P) {
    using C = typename PCfg<N>::C;
    extern __shared__ double2 smem[];
    stage_matrix<C>(P.A, smem, smem + 2 * N * C::P);
    double2* ex = smem + 2 * N * C::P + C::P;
    const int warp = threadIdx.x >> 5, pair = warp >> 1;
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem + 2 * N * C::P);
    double2* exp_ = ex + pair * 128;                                        // [buf][role][lane] within the pair
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    if (warp & 1) walk_body_p<N, 1>(P, lc, lb, exp_, 1 + pair, acc);
    else          walk_body_p<N, 0>(P, lc, lb, exp_, 1 + pair, acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
    __shared__ ddc swarp[PCfg<N>::NT / 32];
    if ((threadIdx.x & 31) == 0) swarp[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        ddc b = swarp[0];
        for (int w = 1; w < PCfg<N>::NT / 32; w++) b = ddc_add(b, swarp[w]);
        P.partials[blockIdx.x] = b;
    }
}

// ---- constant-bank variant (PERM_PAIR_CONST, development): the inner columns ride in the kernel
// parameters (WalkParamsC<N>, as walk_kernel_c) and reach the row-sum DADDs as uniform-register operands;
// the role H is warp-uniform, so the rows [H R, H R + R) of a column are compile-time parameter offsets.
#ifndef PERM_PAIR_CONST
#define PERM_PAIR_CONST 0
#endif
#ifndef PERM_PAIR_MAXNREG
#define PERM_PAIR_MAXNREG 168
#endif

template <class C, int T, int H>
struct InnerStepPC {
    static constexpr int R = C::R, N = C::N;
    static __device__ __forceinline__ void run(const WalkParamsC<N>& P, int z, int smid, double (&wr)[R],
                                               double (&wi)[R], double& ar, double& ai, double (&pr)[2],
                                               double (&pi)[2], double2* ex, int bar, uint32_t& buf) {
        constexpr int U = C::U;
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            const int jj = J + z * (T + 1);          // == J; distinct expression per use (no CSE/hoist)
            if constexpr (J == U - 1 && WalkParamsC<N>::MN == 1) {
                const int jm = jj + smid;            // +a at col[U-1], -a at col[U]
#pragma unroll
                for (int i = 0; i < R; i++) {
                    const double2 a = P.col[jm][H * R + i];
                    wr[i] += a.x;
                    wi[i] += a.y;
                }
            } else if constexpr (J == U - 1) {
                const double zm = smid ? -1.0 : 1.0;
#pragma unroll
                for (int i = 0; i < R; i++) {
                    const double2 a = P.col[jj][H * R + i];
                    wr[i] = fma(zm, a.x, wr[i]);
                    wi[i] = fma(zm, a.y, wi[i]);
                }
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
#pragma unroll
                for (int i = 0; i < R; i++) {
                    const double2 a = P.col[jj][H * R + i];
                    if (PLUS) { wr[i] += a.x; wi[i] += a.y; }
                    else      { wr[i] -= a.x; wi[i] -= a.y; }
                }
            }
        }
        lane_product<R, C::K>(wr, wi, pr[T & 1], pi[T & 1]);
        if constexpr (T & 1) {
            const int lane = threadIdx.x & 31;
            double2* mine = ex + buf * 64 + H * 32 + lane;
            double2* other = ex + buf * 64 + (1 - H) * 32 + lane;
            *mine = make_double2(pr[1 - H], pi[1 - H]);
            pair_barrier(bar);
            const double2 q = *other;
            buf ^= 1u;
            if constexpr (H == 0) fused_acc<-1>(pr[0], pi[0], q.x, q.y, ar, ai);
            else                  fused_acc<+1>(pr[1], pi[1], q.x, q.y, ar, ai);
        }
        if constexpr (T + 1 < (1 << U)) InnerStepPC<C, T + 1, H>::run(P, z, smid, wr, wi, ar, ai, pr, pi, ex, bar, buf);
    }
};

template <int N, int H>
__device__ __forceinline__ void walk_chunk_pc(const WalkParamsC<N>& P, uint32_t lc, uint32_t lb, uint64_t c,
                                              double2* ex, int bar, uint32_t& buf, ddc& acc) {
    using C = typename PCfg<N>::C;
    constexpr int U = C::U, R = C::R;
    const int e = P.eb;
    double wr[R], wi[R];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    seed_rows<C>(lc, lb, x, e - 1, wr, wi);
    const int nblk = 1 << (e - U);
    const uint32_t cpar = (uint32_t)(c & 1ull);
    constexpr int kFoldMask = (U >= kWalkFoldBits) ? 0 : ((1 << (kWalkFoldBits - U)) - 1);
    double ar = 0.0, ai = 0.0, pr[2], pi[2];
    for (int q = 0; q < nblk; q++) {
        const int z = q >> 30;
        if (q > 0) {
            const int j = U + __ffs(q) - 1;
            const uint32_t nb = (j + 1 < e) ? (uint32_t)((q >> (j + 1 - U)) & 1) : cpar;
            flip_add<R>(lc + (uint32_t)(j * C::P) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        InnerStepPC<C, 0, H>::run(P, z, q & 1, wr, wi, ar, ai, pr, pi, ex, bar, buf);   // bit_U(rank) = q & 1
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

template <int N, int H>
__device__ __forceinline__ void walk_body_pc(const WalkParamsC<N>& P, uint32_t lc0, uint32_t lb0, double2* ex, int bar,
                                             ddc& acc) {
    using C = typename PCfg<N>::C;
    const uint32_t hoff = (uint32_t)H * (uint32_t)C::R * 16u;
    const uint32_t lc = lc0 + hoff, lb = lb0 + hoff;
    const int lane = threadIdx.x & 31, pair = threadIdx.x >> 6;
    const uint64_t wid = (uint64_t)blockIdx.x * 2 + (uint64_t)pair;
    const uint64_t nw = (uint64_t)gridDim.x * 2;
    uint32_t buf = 0;
    for (uint64_t base = wid * 32u; base < P.count; base += nw * 32u) {
        const uint64_t g = base + (uint64_t)lane;
        const bool valid = g < P.count;
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        walk_chunk_pc<N, H>(P, lc, lb, P.c0 + (valid ? g : 0), ex, bar, buf, part);
        if (valid) acc = ddc_add(acc, part);
    }
}

template <int N>
__global__ void __maxnreg__(PERM_PAIR_MAXNREG)
    walk_kernel_pc(const __grid_constant__ WalkParamsC<N> P) {
    using C = typename PCfg<N>::C;
    extern __shared__ double2 smem[];
    stage_matrix<C>(P.A, smem, smem + 2 * N * C::P);
    double2* ex = smem + 2 * N * C::P + C::P;
    const int warp = threadIdx.x >> 5, pair = warp >> 1;
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem + 2 * N * C::P);
    double2* exp_ = ex + pair * 128;
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    if (__shfl_sync(0xffffffffu, warp, 0) & 1) walk_body_pc<N, 1>(P, lc, lb, exp_, 1 + pair, acc);
    else                                       walk_body_pc<N, 0>(P, lc, lb, exp_, 1 + pair, acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
    __shared__ ddc swarp[PCfg<N>::NT / 32];
    if ((threadIdx.x & 31) == 0) swarp[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        ddc b = swarp[0];
        for (int w = 1; w < PCfg<N>::NT / 32; w++) b = ddc_add(b, swarp[w]);
        P.partials[blockIdx.x] = b;
    }
}

template <int N>
cudaError_t walk_launch_pair(const WalkLaunch& L) {
    if constexpr (walk_pair_path(N)) {
        using Q = PCfg<N>;
        const Segment& b = L.seg[L.body];
        cudaError_t err;
        if constexpr (PERM_PAIR_CONST && N % 2 == 0) {
            WalkParamsC<N> Pc;
            for (int j = 0; j < WalkParamsC<N>::NC; j++)
                for (int i = 0; i < N; i++) Pc.col[j][i] = L.A_host[(size_t)i * N + j];
            if constexpr (WalkParamsC<N>::MN == 1)
                for (int i = 0; i < N; i++) {
                    const double2 a = L.A_host[(size_t)i * N + WalkParamsC<N>::NC - 1];
                    Pc.col[WalkParamsC<N>::NC][i] = make_double2(-a.x, -a.y);
                }
            Pc.A = L.A_dev;
            Pc.partials = L.partials;
            Pc.c0 = b.c0;
            Pc.count = b.count;
            Pc.eb = b.e;
            err = cudaFuncSetAttribute(walk_kernel_pc<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Q::smem_bytes);
            if (err != cudaSuccess) return err;
            walk_kernel_pc<N><<<L.grid, Q::NT, Q::smem_bytes, L.stream>>>(Pc);
        } else {
        WalkParamsP P;
        P.A = L.A_dev;
        P.partials = L.partials;
        P.c0 = b.c0;
        P.count = b.count;
        P.eb = b.e;
        err = cudaFuncSetAttribute(walk_kernel_p<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)Q::smem_bytes);
        if (err != cudaSuccess) return err;
        walk_kernel_p<N><<<L.grid, Q::NT, Q::smem_bytes, L.stream>>>(P);
        }
        err = cudaGetLastError();
        if (err != cudaSuccess || L.grid_edge == 0) return err;
        Segment rest[kMaxSegments];
        int nr = 0;
        for (int s = 0; s < L.nseg; s++)
            if (s != L.body) rest[nr++] = L.seg[s];
        return walk_launch_smem<N>(L, rest, nr, L.partials + L.grid, L.grid_edge);
    }
    return cudaErrorInvalidValue;
}

template <int N>
cudaError_t walk_occupancy_pair(int* blocks_per_sm) {
    *blocks_per_sm = 0;
    if constexpr (walk_pair_path(N)) {
        using Q = PCfg<N>;
        const void* k = (PERM_PAIR_CONST && N % 2 == 0) ? (const void*)walk_kernel_pc<N> : (const void*)walk_kernel_p<N>;
        cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::smem_bytes);
        if (err != cudaSuccess) return err;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k, Q::NT, Q::smem_bytes);
    }
    return cudaSuccess;
}

}  // namespace perm
