// walk_tmem.cuh -- the single-matrix Gray walk with part of each lane's row sums parked in tensor memory
// (TMEM), for orders whose 4n registers of row sums leave only two warps per scheduler (n = 40..48).
//
// Same method and arithmetic as walk_kernel (walk.cuh; App. A): aligned chunks of 2^e
// ranks, explicit seeding, inner blocks of 2^U = 4 ranks, row-sum updates from +a / -a columns in
// shared memory, two product chains, the last multiply fused with the signed accumulation, double-double
// folds every 2^5 terms.  The difference is where rows RR .. n-1 (RT = n - RR of them) live: in this
// thread's TMEM lane (tcgen05.st / tcgen05.ld, 4 complex per 16-column access, double-buffered between
// consecutive terms so a term never reads what the previous term is still storing).  Freeing 4 RT
// registers lets three 128-thread CTAs (12 warps) reside per SM instead of 8 warps, which is what the
// FP64 pipe needs to cover the three-source DFMA register-read cycles.
//
// tcgen05.ld/st are warp-collective (.sync.aligned): every lane of a warp runs every chunk (lanes past
// the end of the chunk list walk chunk c0 and drop the result), so all TMEM accesses stay converged.
#pragma once
#include "walk.cuh"

namespace perm {

template <int N>
struct TCfg {
    static constexpr int RT = PERM_WALK_TMEM_ROWS;   // rows in TMEM (multiple of 4)
    static constexpr int RR = N - RT;                // rows in registers
    static constexpr int NCH = RT / 4;               // 16-column TMEM chunks (4 complex each)
    static constexpr int COLS = RT * 4;              // 32-bit TMEM columns per buffer
    static constexpr int ALLOC = 2 * COLS <= 32 ? 32 : (2 * COLS <= 64 ? 64 : (2 * COLS <= 128 ? 128 : 256));
    static constexpr int NT = 128;                   // 4 warps = the 4 TMEM lane quadrants
    static constexpr int U = 2;
    static constexpr int K = 2;
    // zero column (a flip by it is a no-op) after the +/- columns and the base vector
    static constexpr size_t smem_bytes = (size_t)(2 * N * N + N + N) * sizeof(double2);
};

struct WalkParamsT {
    const double2* A;      // device, row-major
    ddc* partials;         // [gridDim.x]
    uint64_t c0;           // first body chunk
    uint64_t count;        // body chunks
    int32_t eb;            // log2 body chunk length (> U)
};

__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) {
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}
__device__ __forceinline__ void d2u(double d, uint32_t& lo, uint32_t& hi) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    lo = (uint32_t)b;
    hi = (uint32_t)(b >> 32);
}

// One Gray term: flip by the column at shared address fa (+a or -a; the zero column for none), then
// acc += SIGN * prod_i w_i.  TMEM rows are read from buffer RB and the updated values written to 1-RB.
template <int N, int SIGN, int RB>
__device__ __forceinline__ void term_t(uint32_t fa, uint32_t taddr, double (&wr)[TCfg<N>::RR],
                                       double (&wi)[TCfg<N>::RR], double& ar, double& ai) {
    using T = TCfg<N>;
    constexpr int RR = T::RR, NCH = T::NCH;
    double xr = 1.0, xi = 0.0, yr = 1.0, yi = 0.0;
    tm_wait_st();                                                   // the previous term's stores are done
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        uint32_t v[16];
        tm_ld16(taddr + (uint32_t)(RB * T::COLS + 16 * c), v);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const double2 a = lds_c(fa + (uint32_t)(RR + 4 * c + k) * 16u);
            const double pr = u2d(v[4 * k], v[4 * k + 1]) + a.x;
            const double pi = u2d(v[4 * k + 2], v[4 * k + 3]) + a.y;
            d2u(pr, v[4 * k], v[4 * k + 1]);
            d2u(pi, v[4 * k + 2], v[4 * k + 3]);
            if (c < NCH / 2) {
                if (c == 0 && k == 0) { xr = pr; xi = pi; } else cmul2(xr, xi, pr, pi);
            } else {
                if (c == NCH / 2 && k == 0) { yr = pr; yi = pi; } else cmul2(yr, yi, pr, pi);
            }
        }
        tm_st16(taddr + (uint32_t)((1 - RB) * T::COLS + 16 * c), v);
    }
#pragma unroll
    for (int i = 0; i < RR; i++) {
        const double2 a = lds_c(fa + (uint32_t)i * 16u);
        wr[i] += a.x;
        wi[i] += a.y;
        if (i < RR / 2) cmul2(xr, xi, wr[i], wi[i]);
        else            cmul2(yr, yi, wr[i], wi[i]);
    }
    fused_acc<SIGN>(xr, xi, yr, yi, ar, ai);
}

template <int N>
__device__ __forceinline__ void walk_chunk_t(uint32_t lc, uint32_t lb, uint32_t lz, uint32_t taddr, uint64_t c,
                                             int e, ddc& acc) {
    using T = TCfg<N>;
    using C = WCfg<N, 1>;
    constexpr int RR = T::RR, U = T::U;
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    // seed (App. A steps 5-8): the register rows, then the TMEM rows four at a time into buffer 0
    double wr[RR], wi[RR];
#pragma unroll
    for (int i = 0; i < RR; i++) {
        const double2 b = lds_c(lb + i * 16);
        wr[i] = b.x;
        wi[i] = b.y;
    }
    for (int j = e - 1; j < N - 1; j++) {
        const double f = (double)((x >> j) & 1ull);
        flip_dyn<RR>(lc + (uint32_t)(j * C::P) * 16u, f, wr, wi);
    }
    tm_wait_st();
#pragma unroll
    for (int ch = 0; ch < T::NCH; ch++) {
        double sr[4], si[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const double2 b = lds_c(lb + (uint32_t)(RR + 4 * ch + k) * 16u);
            sr[k] = b.x;
            si[k] = b.y;
        }
        for (int j = e - 1; j < N - 1; j++) {
            const double f = (double)((x >> j) & 1ull);
            flip_dyn<4>(lc + (uint32_t)(j * C::P + RR + 4 * ch) * 16u, f, sr, si);
        }
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            d2u(sr[k], v[4 * k], v[4 * k + 1]);
            d2u(si[k], v[4 * k + 2], v[4 * k + 3]);
        }
        tm_st16(taddr + (uint32_t)(16 * ch), v);
    }
    const int nblk = 1 << (e - U);
    const uint32_t cpar = (uint32_t)(c & 1ull);
    constexpr int kFoldMask = (1 << (kWalkFoldBits - U)) - 1;
    double ar = 0.0, ai = 0.0;
    for (int q = 0; q < nblk; q++) {
        // block boundary: Gray bit j = U + ctz(q) flips to 1 ^ bit_{j+1}(rank); none before the first block
        uint32_t fb = lz;
        if (q > 0) {
            const int j = U + __ffs(q) - 1;
            const uint32_t nb = (j + 1 < e) ? (uint32_t)((q >> (j + 1 - U)) & 1) : cpar;
            fb = lc + (uint32_t)(j * C::P) * 16u + (nb ? C::NEG : 0u);
        }
        const uint32_t fmid = lc + (uint32_t)((U - 1) * C::P) * 16u + ((q & 1) ? C::NEG : 0u);   // e > U
        // ranks t = 0..3 of the block: flips none/boundary, column 0 (+), column 1 (mid), column 0 (-);
        // term sign (-1)^{t+1}
        term_t<N, -1, 0>(fb, taddr, wr, wi, ar, ai);
        term_t<N, +1, 1>(lc, taddr, wr, wi, ar, ai);
        term_t<N, -1, 0>(fmid, taddr, wr, wi, ar, ai);
        term_t<N, +1, 1>(lc + C::NEG, taddr, wr, wi, ar, ai);
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

template <int N>
__global__ void __launch_bounds__(TCfg<N>::NT, 3) walk_kernel_t(const __grid_constant__ WalkParamsT P) {
    using T = TCfg<N>;
    using C = WCfg<N, 1>;
    extern __shared__ double2 smem[];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)), "n"(T::ALLOC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    stage_matrix<C>(P.A, smem, smem + 2 * N * C::P);
    double2* zc = smem + 2 * N * C::P + C::P;
    for (int i = threadIdx.x; i < N; i += blockDim.x) zc[i] = make_double2(0.0, 0.0);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t taddr = tbase + ((uint32_t)((warp & 3) * 32) << 16);   // this warp's lane quadrant
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem + 2 * N * C::P);
    const uint32_t lz = (uint32_t)__cvta_generic_to_shared(zc);
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (uint64_t)warp;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t base = wid * 32u; base < P.count; base += nw * 32u) {   // warp-uniform loop
        const uint64_t g = base + (uint64_t)lane;
        const bool valid = g < P.count;
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        walk_chunk_t<N>(lc, lb, lz, taddr, P.c0 + (valid ? g : 0), P.eb, part);
        if (valid) acc = ddc_add(acc, part);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
    __shared__ ddc swarp[T::NT / 32];
    if (lane == 0) swarp[warp] = acc;
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(T::ALLOC));
    if (threadIdx.x == 0) {
        ddc b = swarp[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) b = ddc_add(b, swarp[w]);
        P.partials[blockIdx.x] = b;
    }
}

template <int N>
cudaError_t walk_launch_tmem(const WalkLaunch& L) {
    if constexpr (walk_tmem_path(N)) {
        using T = TCfg<N>;
        const Segment& b = L.seg[L.body];
        WalkParamsT P;
        P.A = L.A_dev;
        P.partials = L.partials;
        P.c0 = b.c0;
        P.count = b.count;
        P.eb = b.e;
        cudaError_t err = cudaFuncSetAttribute(walk_kernel_t<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)T::smem_bytes);
        if (err != cudaSuccess) return err;
        walk_kernel_t<N><<<L.grid, T::NT, T::smem_bytes, L.stream>>>(P);
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
cudaError_t walk_occupancy_tmem(int* blocks_per_sm) {
    *blocks_per_sm = 0;
    if constexpr (walk_tmem_path(N)) {
        using T = TCfg<N>;
        cudaError_t err = cudaFuncSetAttribute(walk_kernel_t<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)T::smem_bytes);
        if (err != cudaSuccess) return err;
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, walk_kernel_t<N>, T::NT, T::smem_bytes);
        // TMEM: at most 512 columns per SM
        if (err == cudaSuccess && *blocks_per_sm * T::ALLOC > 512) *blocks_per_sm = 512 / T::ALLOC;
        return err;
    }
    return cudaSuccess;
}

}  // namespace perm
