// tools/experiments/walk_split.cuh -- NOT BUILT, not part of the library.  Round-2 experiment, measured on B200 and not
// kept (profiles/round2_split44.txt): 6.78e10 terms/s against 7.06e10 for the shipped one-lane walk.
// To rebuild: copy next to csrc/walk.cuh; before the "Small whole permanents" section of walk.cuh add
//     }  // namespace perm
//     #include "walk_split.cuh"
//     namespace perm {
// and in walk_launch, before `if (unit) {`:
//     if (unit && N == 44) { if constexpr (N == 44) { unit0_attr(walk_kernel_split<N>, walk_split_smem<N>());
//         walk_kernel_split<N><<<L.grid, 256, walk_split_smem<N>(), L.stream>>>(P); } } else
// then PERM_VARIANT=split PERM_EXTRA_FLAGS="-DPERM_SPLIT44 -DPERM_SPLIT_K=1" python -m paper_1904_06229_b200.build.
// Row-split unit-column walk (n even, U = 2).
// A chunk is walked by the same lane of the two WARPS of a pair, warp ROLE holding the row sums of rows
// [ROLE n/2, (ROLE + 1) n/2): half the row-sum registers per thread (128 registers, four warps per scheduler),
// inner column operands still warp-uniform (constant bank).  Per block of four terms each warp forms its four half
// products (prod v, prod (v + 1) at the two states of the block), the pair exchanges two of them through shared
// memory (double buffered, one named barrier per block) and each warp finishes two terms: the joining multiply is
// the one the one-lane walk spends anyway.
#pragma once
#ifndef PERM_SPLIT_FLIP
#define PERM_SPLIT_FLIP 0
#endif
#ifndef PERM_SPLIT_K
#define PERM_SPLIT_K 2
#endif
namespace perm {

template <int R>
__device__ __forceinline__ void half_product(const double (&wr)[R], const double (&wi)[R], double& pr, double& pi) {
    if constexpr (PERM_SPLIT_K == 1) {
        chain<0, R, R>(wr, wi, pr, pi);
    } else {
        double yr, yi;
        two_factors<R, 2>(wr, wi, pr, pi, yr, yi);
        cmul2(pr, pi, yr, yi);
    }
}
template <int R>
__device__ __forceinline__ void half_product_shift1(const double (&wr)[R], const double (&wi)[R], double& pr, double& pi) {
    if constexpr (PERM_SPLIT_K == 1) {
        pr = wr[0] + 1.0;
        pi = wi[0];
#pragma unroll
        for (int i = 1; i < R; i++) cmul_shift1(pr, pi, wr[i], wi[i]);
    } else {
        double yr, yi;
        two_factors_shift1<R, 2>(wr, wi, pr, pi, yr, yi);
        cmul2(pr, pi, yr, yi);
    }
}
__device__ __forceinline__ void sts_c(uint32_t addr, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ double2 lds_v(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void pair_barrier(int id) {      // id 1..4, warp-uniform: immediate barrier names
    if (id == 1)      asm volatile("bar.sync 1, 64;" ::: "memory");
    else if (id == 2) asm volatile("bar.sync 2, 64;" ::: "memory");
    else if (id == 3) asm volatile("bar.sync 3, 64;" ::: "memory");
    else              asm volatile("bar.sync 4, 64;" ::: "memory");
}

// xb: shared address of this lane's slot 0 in the pair's exchange area, laid out [parity][role][slot][lane] x 16 B
template <int N, int ROLE>
__device__ __forceinline__ void walk_chunk_split(const WalkParamsC<N>& P, uint32_t lc, uint32_t lb, uint32_t xb,
                                                 int barid, uint64_t c, ddc& acc) {
    using C = WCfg<N, 1>;
    constexpr int H = N / 2, OFF = ROLE * H, U = C::U;
    static_assert(N % 2 == 0 && U == 2, "row-split walk: even order, blocks of four terms");
    const int e = P.eb;
    double wr[H], wi[H];
#pragma unroll
    for (int i = 0; i < H; i++) {
        const double2 b = lds_c(lb + (OFF + i) * 16);
        wr[i] = b.x;
        wi[i] = b.y;
    }
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    for (int j = N - 2; j >= e - 1; j--) {
        const double f = (double)((x >> j) & 1ull);
        flip_dyn<H>(lc + (uint32_t)(j * N + OFF) * 16u, f, wr, wi);
    }
    const int nblk = 1 << (e - U);
    const uint64_t cpar = c & 1ull;
    constexpr int kFoldMask = (U >= walk_fold_bits_const(N)) ? 0 : ((1 << (walk_fold_bits_const(N) - U)) - 1);
    double ar = 0.0, ai = 0.0;
    for (int q = 0; q < nblk; q++) {
        const int z = q >> 30;
        if (q > 0) {
            const int j = U + __ffs(q) - 1;
            const uint64_t nb = (j + 1 < e) ? (uint64_t)((q >> (j + 1 - U)) & 1) : cpar;
            flip_add<H>(lc + (uint32_t)(j * N + OFF) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        const uint32_t mine = xb + (uint32_t)(q & 1) * 2048u + (uint32_t)ROLE * 1024u;
        const uint32_t other = xb + (uint32_t)(q & 1) * 2048u + (uint32_t)(1 - ROLE) * 1024u;
        double p0r, p0i, s0r, s0i, p2r, p2i, s2r, s2i;
        half_product<H>(wr, wi, p0r, p0i);                 // terms 0, 1 of the block: -prod v + prod (v + 1)
        half_product_shift1<H>(wr, wi, s0r, s0i);
        if constexpr (ROLE == 1) {
            sts_c(mine, p0r, p0i);
            sts_c(mine + 512u, s0r, s0i);
        }
#if PERM_SPLIT_FLIP == 0
        {
            const int jm = 1 + z * 3 + ((q & 1) ? 1 : 0);  // column 1 with its sign by address (col[2] = -col[1])
#pragma unroll
            for (int i = 0; i < H; i++) {
                const double2 a = P.col[jm][OFF + i];
                wr[i] += a.x;
                wi[i] += a.y;
            }
        }
#elif PERM_SPLIT_FLIP == 1
        flip_add<H>(lc + (uint32_t)(1 * N + OFF) * 16u + ((q & 1) ? C::NEG : 0u), wr, wi);   // diagnostic: shared-memory column
#else
        (void)z;                                           // diagnostic: no inner flip (wrong values, timing only)
#endif
        half_product<H>(wr, wi, p2r, p2i);                 // terms 2, 3: +prod v - prod (v + 1)
        half_product_shift1<H>(wr, wi, s2r, s2i);
        if constexpr (ROLE == 0) {
            sts_c(mine, p2r, p2i);
            sts_c(mine + 512u, s2r, s2i);
        }
        pair_barrier(barid);
        const double2 o1 = lds_v(other), o2 = lds_v(other + 512u);
        if constexpr (ROLE == 0) {
            fused_acc<-1>(p0r, p0i, o1.x, o1.y, ar, ai);
            fused_acc<+1>(s0r, s0i, o2.x, o2.y, ar, ai);
        } else {
            fused_acc<+1>(p2r, p2i, o1.x, o1.y, ar, ai);
            fused_acc<-1>(s2r, s2i, o2.x, o2.y, ar, ai);
        }
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

template <int N>
__global__ void __launch_bounds__(256, 2) walk_kernel_split(const __grid_constant__ WalkParamsC<N> P) {
    extern __shared__ double2 smem[];
    double2* scol = smem;
    double2* sbase = smem + 2 * N * N;
    double2* sx = sbase + N;                                 // 4 pairs x 4 KB exchange area
    for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
        const int i = k / N, j = k - i * N;
        const double2 a = P.A[k];
        scol[j * N + i] = a;
        scol[N * N + j * N + i] = make_double2(-a.x, -a.y);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
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
    const uint32_t ln = threadIdx.x & 31u;
    const uint32_t w = (uint32_t)__shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);   // warp in block, uniform
    const uint32_t pair = w >> 1, role = w & 1u;
    const uint32_t xb = (uint32_t)__cvta_generic_to_shared(sx) + pair * 4096u + ln * 16u;
    const int barid = 1 + (int)pair;
    const uint64_t wid = (uint64_t)blockIdx.x * 4u + pair;
    const uint64_t nw = (uint64_t)gridDim.x * 4u;
    for (uint64_t base = wid * 32u; base < P.count; base += nw * 32u) {
        const uint64_t g = base + ln;
        const bool valid = g < P.count;
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        const uint64_t c = P.c0 + (valid ? g : 0);
        if (role == 0) walk_chunk_split<N, 0>(P, lc, lb, xb, barid, c, part);
        else           walk_chunk_split<N, 1>(P, lc, lb, xb, barid, c, part);
        // the two halves of the chunk partial: role 1 hands its double-double to role 0 (exchange area, parity 0)
        pair_barrier(barid);
        if (role == 1) {
            sts_c(xb, part.re.hi, part.re.lo);
            sts_c(xb + 512u, part.im.hi, part.im.lo);
        }
        pair_barrier(barid);
        if (role == 0) {
            const double2 r = lds_v(xb), m = lds_v(xb + 512u);
            ddc o;
            o.re.hi = r.x; o.re.lo = r.y; o.im.hi = m.x; o.im.lo = m.y;
            part = ddc_add(part, o);
            if (P.scaled) part = ddc_mul(part, P.scale);
            if (valid) P.items[P.item0 + g] = part;
        }
        pair_barrier(barid);
    }
}
template <int N>
constexpr size_t walk_split_smem() { return WCfg<N, 1>::smem_bytes + 4 * 4096; }

}  // namespace perm
