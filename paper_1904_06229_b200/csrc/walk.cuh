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
// different chunks in lock-step and every column index is warp-uniform.  Within a chunk a block of
// 2^U ranks is fully unrolled, so its flips (columns 0..U-1) use compile-time shared-memory offsets
// and compile-time signs; the flip at the block boundary (column j >= U, once per 2^U terms) uses a
// dynamic column and sign.
//
// Lanes per chunk S (1 or 2).  With S = 2 the two lanes of a pair walk the SAME chunk and split the
// rows: lane h keeps the row sums of rows [hR, hR+R), R = ceil(n/2) (an odd n is padded with a
// neutral row w = 1).  Each lane multiplies its R row sums; after every two terms the pair swaps one
// partial product with a single shuffle (lane 0 finishes the even term, lane 1 the odd one), so the
// FP64 work per term is unchanged (6n-4) while registers per thread halve (n > 48 only).
//
// Per term: 2n DADD/DFMA (row-sum update) + 4(n-2) DMUL/DFMA (product, split
// into K independent chains) + 4 DFMA (last multiply fused with the signed accumulation)
// = 6n-4 FP64 instructions for ~8n flops.  Column operands are loaded with ld.volatile.shared right
// before use: this keeps ptxas from hoisting/CSE-ing the (loop-invariant) columns into registers,
// which at n = 44 would spill.  Plain-double sums over 2^kWalkFoldBits terms are folded into a
// double-double accumulator (TwoSum) that starts at zero for every item (chunk or single term); each
// item's dd partial is written to HBM at its index in the launch's item order, and tree.cu combines the
// items by the canonical pairwise tree -- so an item's value, and the result, depend only on (A, n, b).
#pragma once
#include <cooperative_groups.h>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace perm {

template <int N_, int S_>
struct WCfg {
    static constexpr int N = N_;
    static constexpr int U = walk_inner_bits(N);
    static constexpr int S = S_;                             // lanes per chunk
    static constexpr int R = (N + S - 1) / S;                // rows per lane
    static constexpr int P = R * S;                          // padded rows per column in shared memory
    static constexpr int NT = walk_block_threads(N);
#ifdef PERM_WALK_K
    static constexpr int K = R >= 16 ? PERM_WALK_K : (R >= 4 ? 2 : 1);
#else
    // independent product chains per lane: four (rows dealt round-robin) for the n = 44 constant-bank walk,
    // where the shorter dependency chains measured +2.7% (6.16e10 -> 6.33e10 terms/s); two elsewhere (four
    // measured slower at n = 32, 43, 45..48 and in the batched kernel: profiles/round1_walk_chains.txt)
    static constexpr int K = (N == 44 && S == 1) ? 4 : (R >= 4 ? 2 : 1);
#endif
    // columns a_{.j} (j < N), then their negations -a_{.j}, then the step-5 base vector
    static constexpr uint32_t NEG = (uint32_t)(N * P) * 16u;   // byte offset of -a_{.j} from a_{.j}
    static constexpr size_t smem_bytes = (size_t)(2 * N * P + P) * sizeof(double2);
    // Register budget per thread for S > 1: the 4R row-sum registers plus working set; it sets the
    // minimum resident blocks in __launch_bounds__ so ptxas does not trade occupancy for scheduling
    // freedom.  S = 1 is left uncapped (4n + ~30 registers).
#ifdef PERM_WALK_REG_EXTRA
    static constexpr int REGS = ((4 * R + PERM_WALK_REG_EXTRA + 7) / 8) * 8;
#else
    // >= 224: below that ptxas spills the two-lane walk at n = 33..48 (tools/spills.py)
    static constexpr int REGS = (4 * R + 128) > 224 ? ((4 * R + 128 + 7) / 8) * 8 : 224;
#endif
    static constexpr int MINB_RAW = (S == 1) ? 1 : 65536 / (NT * (REGS < 255 ? REGS : 255));
    static constexpr int MINB = MINB_RAW < 1 ? 1 : MINB_RAW;
};

template <int N>
using WalkCfg = WCfg<N, walk_lanes_per_chunk(N)>;

struct WalkParams {
    const double2* A;                      // device, row-major
    ddc* items;                            // one dd partial per item, at seg_item0[s] + (index in segment)
    uint64_t nitems;                       // items of the whole launch plan (bounds of `items`)
    uint64_t seg_item0[kMaxSegments];
    uint64_t seg_c0[kMaxSegments];
    uint64_t seg_pre[kMaxSegments + 1];    // prefix item counts
    int32_t seg_e[kMaxSegments];
    int32_t nseg;
    int32_t scaled;                        // unit-column walk: multiply every item partial by `scale`
    ddc scale;
};

// Load of one complex entry from shared memory (volatile: never hoisted or merged).
__device__ __forceinline__ double2 lds_c(uint32_t addr) {
    double2 v;
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

// (xr + i xi) *= (yr + i yi): 4 FP64 instructions (2 DMUL + 2 DFMA).  Measured and not kept (round 1-2):
// products as fma(a, b, +0.0) so all four are DFMA, and alternating the roles of xr and xi along a chain.
__device__ __forceinline__ void cmul2(double& xr, double& xi, double yr, double yi) {
    const double t = xi * yi;
    const double u = xi * yr;
    const double nr = fma(xr, yr, -t);
    xi = fma(xr, yi, u);
    xr = nr;
}

// Product of rows [B, E) into (pr, pi).
template <int B, int E, int R>
__device__ __forceinline__ void chain(const double (&wr)[R], const double (&wi)[R], double& pr, double& pi) {
    pr = wr[B];
    pi = wi[B];
#pragma unroll
    for (int i = B + 1; i < E; i++) cmul2(pr, pi, wr[i], wi[i]);
}

// Split prod_i w_i into two factors X * Y (K chains).
template <int R, int K>
__device__ __forceinline__ void two_factors(const double (&wr)[R], const double (&wi)[R], double& xr, double& xi,
                                            double& yr, double& yi) {
    if constexpr (K == 1) {
        chain<0, R - 1, R>(wr, wi, xr, xi);
        yr = wr[R - 1];
        yi = wi[R - 1];
    } else if constexpr (K == 2) {
        chain<0, R / 2, R>(wr, wi, xr, xi);
        chain<R / 2, R, R>(wr, wi, yr, yi);
    } else if constexpr (K == 3) {
        constexpr int t = R / 3;
        double zr, zi;
        chain<0, t, R>(wr, wi, xr, xi);
        chain<t, 2 * t, R>(wr, wi, yr, yi);
        chain<2 * t, R, R>(wr, wi, zr, zi);
        cmul2(xr, xi, yr, yi);
        yr = zr;
        yi = zi;
    } else if constexpr (K == 8) {
        // eight chains of ~R/8 rows, combined as a tree: (01)(23) and (45)(67) -> two factors
        double cr[8], ci[8];
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int b = c * R / 8, e = (c + 1) * R / 8;
            cr[c] = wr[b];
            ci[c] = wi[b];
#pragma unroll
            for (int i = b + 1; i < e; i++) cmul2(cr[c], ci[c], wr[i], wi[i]);
        }
        cmul2(cr[0], ci[0], cr[1], ci[1]);
        cmul2(cr[2], ci[2], cr[3], ci[3]);
        cmul2(cr[4], ci[4], cr[5], ci[5]);
        cmul2(cr[6], ci[6], cr[7], ci[7]);
        cmul2(cr[0], ci[0], cr[2], ci[2]);
        cmul2(cr[4], ci[4], cr[6], ci[6]);
        xr = cr[0]; xi = ci[0];
        yr = cr[4]; yi = ci[4];
    } else if constexpr (K >= 5) {
        // K chains of ~R/K rows, folded into two factors (K - 2 extra multiplies, same total n - 1)
        double cr[K], ci[K];
#pragma unroll
        for (int c = 0; c < K; c++) {
            const int b = c * R / K, e = (c + 1) * R / K;
            cr[c] = wr[b];
            ci[c] = wi[b];
#pragma unroll
            for (int i = b + 1; i < e; i++) cmul2(cr[c], ci[c], wr[i], wi[i]);
        }
#pragma unroll
        for (int c = 2; c < K; c++) {
            if (c & 1) cmul2(cr[1], ci[1], cr[c], ci[c]);
            else       cmul2(cr[0], ci[0], cr[c], ci[c]);
        }
        xr = cr[0]; xi = ci[0];
        yr = cr[1]; yi = ci[1];
    } else {
        // rows dealt round-robin to the four chains (chain c: rows c, c+4, ...); the two products then
        // multiply each other in the fused accumulation
        double r0, i0, r1, i1, r2, i2, r3, i3;
        r0 = wr[0]; i0 = wi[0]; r1 = wr[1]; i1 = wi[1]; r2 = wr[2]; i2 = wi[2]; r3 = wr[3]; i3 = wi[3];
#pragma unroll
        for (int i = 4; i < R; i++) {
            if ((i & 3) == 0) cmul2(r0, i0, wr[i], wi[i]);
            else if ((i & 3) == 1) cmul2(r1, i1, wr[i], wi[i]);
            else if ((i & 3) == 2) cmul2(r2, i2, wr[i], wi[i]);
            else cmul2(r3, i3, wr[i], wi[i]);
        }
        cmul2(r0, i0, r1, i1);
        cmul2(r2, i2, r3, i3);
        xr = r0; xi = i0; yr = r2; yi = i2;
    }
}

// Full product of the lane's rows.
template <int R, int K>
__device__ __forceinline__ void lane_product(const double (&wr)[R], const double (&wi)[R], double& pr, double& pi) {
    if constexpr (R == 1) {
        pr = wr[0];
        pi = wi[0];
    } else {
        double yr, yi;
        two_factors<R, K>(wr, wi, pr, pi, yr, yi);
        cmul2(pr, pi, yr, yi);
    }
}

// acc += SIGN * X * Y as 4 DFMA (the last complex multiply fused with the accumulation).
template <int SIGN>
__device__ __forceinline__ void fused_acc(double xr, double xi, double yr, double yi, double& ar, double& ai) {
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

// S = 1: acc += SIGN * prod_i w_i.
template <int R, int K, int SIGN>
__device__ __forceinline__ void term_acc(const double (&wr)[R], const double (&wi)[R], double& ar, double& ai) {
    if constexpr (R == 1) {
        if (SIGN > 0) { ar += wr[0]; ai += wi[0]; } else { ar -= wr[0]; ai -= wi[0]; }
    } else {
        double xr, xi, yr, yi;
        two_factors<R, K>(wr, wi, xr, xi, yr, yi);
        fused_acc<SIGN>(xr, xi, yr, yi, ar, ai);
    }
}

// Unit-column walk (internal.h walk_unit0): x *= (y + 1) as 4 DFMA -- the "+1" of the unit bit-0 column rides in
// the FMAs' addends: re = xr (yr + 1) - xi yi = fma(-xi, yi, fma(xr, yr, xr)), im = fma(xr, yi, fma(xi, yr, xi)).
__device__ __forceinline__ void cmul_shift1(double& xr, double& xi, double yr, double yi) {
    const double t = fma(xr, yr, xr);
    const double u = fma(xi, yr, xi);
    const double nr = fma(-xi, yi, t);
    xi = fma(xr, yi, u);
    xr = nr;
}

// prod_i (w_i + 1) split into two factors X * Y (the two_factors chain layouts, K = 2 or 4)
template <int R, int K>
__device__ __forceinline__ void two_factors_shift1(const double (&wr)[R], const double (&wi)[R], double& xr, double& xi,
                                                   double& yr, double& yi) {
    static_assert(K == 2 || K == 4, "unit-column walk: two or four chains");
    if constexpr (K == 2) {
        xr = wr[0] + 1.0;
        xi = wi[0];
#pragma unroll
        for (int i = 1; i < R / 2; i++) cmul_shift1(xr, xi, wr[i], wi[i]);
        yr = wr[R / 2] + 1.0;
        yi = wi[R / 2];
#pragma unroll
        for (int i = R / 2 + 1; i < R; i++) cmul_shift1(yr, yi, wr[i], wi[i]);
    } else {
        double r0 = wr[0] + 1.0, i0 = wi[0], r1 = wr[1] + 1.0, i1 = wi[1];
        double r2 = wr[2] + 1.0, i2 = wi[2], r3 = wr[3] + 1.0, i3 = wi[3];
#pragma unroll
        for (int i = 4; i < R; i++) {
            if ((i & 3) == 0) cmul_shift1(r0, i0, wr[i], wi[i]);
            else if ((i & 3) == 1) cmul_shift1(r1, i1, wr[i], wi[i]);
            else if ((i & 3) == 2) cmul_shift1(r2, i2, wr[i], wi[i]);
            else cmul_shift1(r3, i3, wr[i], wi[i]);
        }
        cmul2(r0, i0, r1, i1);
        cmul2(r2, i2, r3, i3);
        xr = r0; xi = i0; yr = r2; yi = i2;
    }
}

// acc += SIGN * prod_i (w_i + 1)
template <int R, int K, int SIGN>
__device__ __forceinline__ void term_acc_shift1(const double (&wr)[R], const double (&wi)[R], double& ar, double& ai) {
    double xr, xi, yr, yi;
    two_factors_shift1<R, K>(wr, wi, xr, xi, yr, yi);
    fused_acc<SIGN>(xr, xi, yr, yi, ar, ai);
}

__device__ __forceinline__ double flip_sign_if(double v, uint32_t mask_hi) {
    // v with its sign bit XOR-ed by mask_hi (0 or 0x80000000): an integer op, not an FP64 instruction
    const long long b = __double_as_longlong(v) ^ ((long long)mask_hi << 32);
    return __longlong_as_double(b);
}

// Shuffle mask of this thread's lane group (S consecutive lanes).
template <int S>
__device__ __forceinline__ unsigned group_mask() {
    return (S >= 32) ? 0xffffffffu : (((1u << S) - 1u) << ((threadIdx.x & 31u) & ~(unsigned)(S - 1)));
}

// S > 1, after the last term of an aligned group of S terms: (vr, vi)[t] is this lane's partial product
// (its R rows) of term t of the group.  Recursive halving over the S lanes: at round k the lane keeps the
// terms whose bit k equals its own bit k, ships the others to lane ^ 2^k and multiplies what it receives
// into what it kept; after log2 S rounds lane h holds the full product of term h of the group and adds it
// with the term's sign (-1)^{h+1} (groups start at even ranks) -- the last multiply fused with the sum.
// FP64 work per term is exactly that of S = 1 (n-1 complex multiplies per term in total).
template <int S>
__device__ __forceinline__ void group_finish(double (&vr)[S], double (&vi)[S], uint32_t h, double& ar, double& ai) {
    const unsigned gm = group_mask<S>();
#pragma unroll
    for (int k = 0, cnt = S; cnt > 1; k++, cnt >>= 1) {
        const uint32_t hb = (h >> k) & 1u;
#pragma unroll
        for (int j = 0; j < cnt / 2; j++) {
            const double kr = hb ? vr[2 * j + 1] : vr[2 * j];
            const double ki = hb ? vi[2 * j + 1] : vi[2 * j];
            const double sr = hb ? vr[2 * j] : vr[2 * j + 1];
            const double si = hb ? vi[2 * j] : vi[2 * j + 1];
            const double qr = __shfl_xor_sync(gm, sr, 1 << k);
            const double qi = __shfl_xor_sync(gm, si, 1 << k);
            if (cnt > 2) {
                vr[j] = kr;
                vi[j] = ki;
                cmul2(vr[j], vi[j], qr, qi);
            } else {
                const uint32_t neg = (h & 1u) ? 0u : 0x80000000u;   // even term: sign -
                fused_acc<+1>(flip_sign_if(kr, neg), flip_sign_if(ki, neg), qr, qi, ar, ai);
            }
        }
    }
}

// w += z * column (lane's slice at shared address col), z = +-1 (or 0/1 when seeding).
template <int R>
__device__ __forceinline__ void flip_dyn(uint32_t col, double z, double (&wr)[R], double (&wi)[R]) {
#pragma unroll
    for (int i = 0; i < R; i++) {
        const double2 a = lds_c(col + i * 16);
        wr[i] = fma(z, a.x, wr[i]);
        wi[i] = fma(z, a.y, wi[i]);
    }
}

// w += column (PLUS) or w -= column, compile-time sign; col = lane's slice of the column.
template <int R, bool PLUS>
__device__ __forceinline__ void flip_static(uint32_t col, double (&wr)[R], double (&wi)[R]) {
#pragma unroll
    for (int i = 0; i < R; i++) {
        const double2 a = lds_c(col + i * 16);
        if (PLUS) { wr[i] += a.x; wi[i] += a.y; }
        else      { wr[i] -= a.x; wi[i] -= a.y; }
    }
}

// w += column at shared address col (the address of a_{.j} or of -a_{.j} selects the sign): 2R DADD
// with two vector operands each.  (fma(z, a, w) with a register sign z would read three vector register
// pairs and issue at 2/3 of the FP64 pipe rate on sm_100a; tools/micro/fp64_reuse.cu.)
template <int R>
__device__ __forceinline__ void flip_add(uint32_t col, double (&wr)[R], double (&wi)[R]) {
#pragma unroll
    for (int i = 0; i < R; i++) {
        const double2 a = lds_c(col + i * 16);
        wr[i] += a.x;
        wi[i] += a.y;
    }
}

// Inner block: ranks t = 0 .. 2^U - 1 of the current block (t = 0 already seeded/flipped).
// lc = this lane's address of row 0 of column 0 (columns are P rows apart).
template <class C, int T>
struct InnerStep {
    static constexpr int R = C::R;
    static __device__ __forceinline__ void run(uint32_t lc, uint32_t lmid, uint32_t h, double (&wr)[R],
                                               double (&wi)[R], double& ar, double& ai, double (&pr)[C::S],
                                               double (&pi)[C::S]) {
        constexpr int U = C::U;
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                // new bit = 1 ^ bit_U(rank): depends on the block (or chunk) parity; lmid is the address
                // of +a_{.,U-1} or -a_{.,U-1} accordingly
                flip_add<R>(lmid, wr, wi);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;  // new bit = 1 ^ bit_{J+1}(t)
                flip_static<R, PLUS>(lc + (uint32_t)(J * C::P) * 16u, wr, wi);
            }
        }
        if constexpr (C::S == 1) {
            if constexpr (T & 1) term_acc<R, C::K, +1>(wr, wi, ar, ai);   // sign (-1)^{r+1}, r == t (mod 2)
            else                 term_acc<R, C::K, -1>(wr, wi, ar, ai);
        } else {
            lane_product<R, C::K>(wr, wi, pr[T % C::S], pi[T % C::S]);
            if constexpr (T % C::S == C::S - 1) group_finish<C::S>(pr, pi, h, ar, ai);
        }
        if constexpr (T + 1 < (1 << U)) InnerStep<C, T + 1>::run(lc, lmid, h, wr, wi, ar, ai, pr, pi);
    }
};

// Seed w = base + sum_{j in [j0, N-1), bit_j(x) = 1} column_j   (App. A steps 5-8; branch-free in j).
// lc / lb = this lane's addresses of column 0 and of the base vector.
template <class C>
__device__ __forceinline__ void seed_rows(uint32_t lc, uint32_t lb, uint64_t x, int j0, double (&wr)[C::R],
                                          double (&wi)[C::R]) {
    constexpr int N = C::N, R = C::R, P = C::P;
#pragma unroll
    for (int i = 0; i < R; i++) {
        const double2 b = lds_c(lb + i * 16);
        wr[i] = b.x;
        wi[i] = b.y;
    }
    // columns in DESCENDING order (every walk seeds this way): for lanes walking consecutive chunks the high
    // columns come first and are warp-uniform, so the small-permanent kernel can share that prefix exactly
    for (int j = N - 2; j >= j0; j--) {
        const double f = (double)((x >> j) & 1ull);
        flip_dyn<R>(lc + (uint32_t)(j * P) * 16u, f, wr, wi);
    }
}

template <class C>
__device__ __forceinline__ void walk_seeded(uint32_t lc, uint32_t h, uint64_t c, int e, double (&wr)[C::R],
                                            double (&wi)[C::R], ddc& acc);

// One aligned chunk of 2^e ranks (e >= U >= 1), walked by the S lanes of a group (h = lane in group).
template <class C>
__device__ __forceinline__ void walk_chunk(uint32_t lc, uint32_t lb, uint32_t h, uint64_t c, int e, ddc& acc) {
    constexpr int R = C::R;
    double wr[R], wi[R];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    seed_rows<C>(lc, lb, x, e - 1, wr, wi);
    walk_seeded<C>(lc, h, c, e, wr, wi, acc);
}

// The walk of chunk c (2^e ranks, e >= U) from row sums already seeded at its first rank c 2^e:
// acc += sum_{r in chunk} (-1)^{r+1} prod_i w_i(gray r).
template <class C>
__device__ __forceinline__ void walk_seeded(uint32_t lc, uint32_t h, uint64_t c, int e, double (&wr)[C::R],
                                            double (&wi)[C::R], ddc& acc) {
    constexpr int U = C::U, R = C::R;
    const uint32_t nblk = 1u << (e - U);                 // e <= 30: 32-bit block counter (fewer registers)
    const uint32_t cpar = (uint32_t)(c & 1ull);
    constexpr uint32_t kFoldMask = (U >= kWalkFoldBits) ? 0u : ((1u << (kWalkFoldBits - U)) - 1u);
    double ar = 0.0, ai = 0.0, pr[C::S], pi[C::S];
    for (uint32_t q = 0; q < nblk; q++) {
        if (q > 0) {
            // block boundary: Gray bit j = U + ctz(q) flips to 1 ^ bit_{j+1}(rank)
            const int j = U + __ffs((int)q) - 1;
            const uint32_t nb = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1u) : cpar;
            flip_add<R>(lc + (uint32_t)(j * C::P) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        const uint32_t nbm = (U < e) ? (q & 1u) : cpar;     // bit_U(rank) for the mid-block flip
        const uint32_t lmid = lc + (uint32_t)((U - 1) * C::P) * 16u + (nbm ? C::NEG : 0u);
        InnerStep<C, 0>::run(lc, lmid, h, wr, wi, ar, ai, pr, pi);
        // fold the plain block sums into the dd accumulator every 2^kWalkFoldBits terms (and at the end)
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

// Unit-column walk on shared-memory columns (batched kernel; internal.h walk_unit0): column 0 of the staged matrix
// is all ones and never added -- the row sums v hold Gray bit 0 = 0 -- and the pair (T, T+1), T even, adds
// s_T (prod (v + 1) - prod v), s_T = +1 iff bit 1 of T is 0 (see InnerStepCU).  One lane per chunk.
template <class C, int T>
struct InnerStepU {
    static constexpr int R = C::R;
    static __device__ __forceinline__ void run(uint32_t lc, uint32_t lmid, double (&wr)[R], double (&wi)[R], double& ar,
                                               double& ai) {
        constexpr int U = C::U;
        static_assert(C::S == 1 && T % 2 == 0 && U >= 2, "unit-column walk: one lane per chunk, blocks of >= 4");
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);            // >= 1
            if constexpr (J == U - 1) {
                flip_add<R>(lmid, wr, wi);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
                flip_static<R, PLUS>(lc + (uint32_t)(J * C::P) * 16u, wr, wi);
            }
        }
        constexpr int SP = ((T >> 1) & 1) ? -1 : 1;
        term_acc<R, C::K, -SP>(wr, wi, ar, ai);
        term_acc_shift1<R, C::K, SP>(wr, wi, ar, ai);
        if constexpr (T + 2 < (1 << U)) InnerStepU<C, T + 2>::run(lc, lmid, wr, wi, ar, ai);
    }
};

// One aligned chunk of 2^e ranks (e >= U >= 2) on the unit-column walk: the seed never includes column 0 (its Gray
// bit is 0 at an aligned start with e >= 2), and the bit-0 flips are replaced by the pairs of InnerStepU.
template <class C>
__device__ __forceinline__ void walk_chunk_unit(uint32_t lc, uint32_t lb, uint64_t c, int e, ddc& acc) {
    constexpr int U = C::U, R = C::R;
    double wr[R], wi[R];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    seed_rows<C>(lc, lb, x, e - 1, wr, wi);
    const uint32_t nblk = 1u << (e - U);
    const uint32_t cpar = (uint32_t)(c & 1ull);
    constexpr uint32_t kFoldMask = (U >= kWalkFoldBits) ? 0u : ((1u << (kWalkFoldBits - U)) - 1u);
    double ar = 0.0, ai = 0.0;
    for (uint32_t q = 0; q < nblk; q++) {
        if (q > 0) {
            const int j = U + __ffs((int)q) - 1;
            const uint32_t nb = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1u) : cpar;
            flip_add<R>(lc + (uint32_t)(j * C::P) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        const uint32_t nbm = (U < e) ? (q & 1u) : cpar;
        const uint32_t lmid = lc + (uint32_t)((U - 1) * C::P) * 16u + (nbm ? C::NEG : 0u);
        InnerStepU<C, 0>::run(lc, lmid, wr, wi, ar, ai);
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

// A single rank r, seeded from scratch (all S lanes of the group call it; one accumulates).
template <class C>
__device__ __forceinline__ void single_term(uint32_t lc, uint32_t lb, uint32_t h, uint64_t r, ddc& acc) {
    constexpr int R = C::R;
    double wr[R], wi[R];
    seed_rows<C>(lc, lb, r ^ (r >> 1), 0, wr, wi);
    double ar = 0.0, ai = 0.0;
    if constexpr (C::S == 1) {
        if (r & 1ull) term_acc<R, C::K, +1>(wr, wi, ar, ai);
        else          term_acc<R, C::K, -1>(wr, wi, ar, ai);
    } else {
        double pr, pi;
        lane_product<R, C::K>(wr, wi, pr, pi);
        const unsigned gm = group_mask<C::S>();
#pragma unroll
        for (int k = 1; k < C::S; k <<= 1) {      // butterfly: every lane ends with the full product
            const double qr = __shfl_xor_sync(gm, pr, k);
            const double qi = __shfl_xor_sync(gm, pi, k);
            cmul2(pr, pi, qr, qi);
        }
        if (h == 0) {
            if (r & 1ull) { ar += pr; ai += pi; }
            else          { ar -= pr; ai -= pi; }
        }
    }
    acc.re = dd_add_d(acc.re, ar);
    acc.im = dd_add_d(acc.im, ai);
}

// Stage A column-major into shared memory, sc[j*P + i] = a_ij (rows i >= N zero), and compute the
// App. A step-5 base vector w_i(0) = a_{i,n} - 1/2 sum_j a_ij (summed in column order j = 0..n-1);
// padding rows get w = 1 (a neutral factor).
template <class C>
__device__ __forceinline__ void stage_matrix(const double2* __restrict__ A, double2* sc, double2* sbase) {
    constexpr int N = C::N, P = C::P;
    for (int k = threadIdx.x; k < N * P; k += blockDim.x) {
        const int j = k / P, i = k - j * P;
        const double2 a = (i < N) ? A[i * N + j] : make_double2(0.0, 0.0);
        sc[k] = a;
        sc[N * P + k] = make_double2(-a.x, -a.y);   // negated copy (exact)
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i >= N) {
            sbase[i] = make_double2(1.0, 0.0);
            continue;
        }
        double sr = 0.0, si = 0.0;
        for (int j = 0; j < N; j++) {
            sr += sc[j * P + i].x;
            si += sc[j * P + i].y;
        }
        sbase[i] = make_double2(sc[(N - 1) * P + i].x - 0.5 * sr, sc[(N - 1) * P + i].y - 0.5 * si);
    }
    __syncthreads();
}

template <int N>
__global__ void __launch_bounds__(WalkCfg<N>::NT, WalkCfg<N>::MINB) walk_kernel(const __grid_constant__ WalkParams P) {
    using C = WalkCfg<N>;
    extern __shared__ double2 smem[];
    stage_matrix<C>(P.A, smem, smem + 2 * N * C::P);
    const uint32_t h = threadIdx.x % C::S;
    const uint32_t hoff = h * (uint32_t)C::R * 16u;
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem) + hoff;
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem + 2 * N * C::P) + hoff;

    // static round-robin over the launch's items: walker w takes the global items g = w (mod W); per segment
    // that is i = (w - seg_pre[s]) mod W, i + W, ...  (only the 64-bit item index is live across a chunk)
    const uint32_t wpb = blockDim.x / C::S;
    const uint64_t w = (uint64_t)blockIdx.x * wpb + threadIdx.x / C::S;
    // the item's dd accumulator lives in shared memory (touched once per 2^kWalkFoldBits terms): at n >= 33
    // the 4n row-sum registers leave no room for it without spilling
    __shared__ ddc sacc_[C::NT];
    for (int s = 0; s < P.nseg; s++) {
        const uint64_t W = (uint64_t)gridDim.x * wpb;
        const uint64_t pre = P.seg_pre[s], cnt = P.seg_pre[s + 1] - pre;
        const uint64_t i0 = (w + W - pre % W) % W;
        for (uint64_t i = i0; i < cnt; i += (uint64_t)gridDim.x * wpb) {
            const int e = P.seg_e[s];
            {
                volatile ddc& z = *(volatile ddc*)&sacc_[threadIdx.x];
                z.re.hi = 0.0; z.re.lo = 0.0; z.im.hi = 0.0; z.im.lo = 0.0;
            }
            ddc& acc = sacc_[threadIdx.x];
            const uint64_t c = P.seg_c0[s] + i;
            if constexpr (C::U >= 1) {
                if (e == 0) single_term<C>(lc, lb, h, c, acc);
                else        walk_chunk<C>(lc, lb, h, c, e, acc);
            } else {
                single_term<C>(lc, lb, h, c, acc);
            }
            ddc v = acc;
            if constexpr (C::S > 1) {  // the S lanes of a group hold interleaved terms: fixed-order combine
#pragma unroll
                for (int off = C::S / 2; off > 0; off >>= 1) v = ddc_add(v, shfl_down_ddc(v, off, group_mask<C::S>()));
            }
            PERM_DCHECK(P.seg_item0[s] + i < P.nitems);
            if (P.scaled) v = ddc_mul(v, P.scale);             // unit-column walk: back to the units of A
            if (h == 0) P.items[P.seg_item0[s] + i] = v;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// Constant-bank path (one lane per chunk, n <= kConstMaxN): the whole matrix rides in the kernel
// parameters, so every column entry is a warp-uniform LDCU.64 into a uniform register and the row-sum
// update is DADD R, R, UR -- no shared-memory load, no vector register for the column, and one vector
// operand fewer per update.  Only the aligned body of a range (all chunks of length 2^eb) runs here;
// the few unaligned head/tail pieces go to walk_kernel.  ptxas keeps parameter loads as LDCU only for
// warp-uniform addresses, so the block loop counter is a 32-bit uniform value and each use of an
// inner column gets its own opaque zero offset (z * (T+1), z = q >> 31 == 0): without it the
// loop-invariant columns are hoisted into vector registers and the kernel spills.
// Orders whose constant-bank walk takes the mid-block column with its sign by address (+a and -a both in
// the parameters: DADD R, R, UR instead of fma(z, a, w), one vector register read fewer per update).
// Bit-identical either way; n = 44: 6.16e10 vs 6.14e10 terms/s (profiles/round1_walk_table_variants.txt).
// PERM_CONST_MIDNEG=1 enables it for every order (scans: the register caps of walk_const_maxnreg were
// found without it).
#ifndef PERM_CONST_MIDNEG
#define PERM_CONST_MIDNEG 0
#endif
__host__ __device__ constexpr int walk_const_midneg(int n) { return (PERM_CONST_MIDNEG || n == 42 || n == 44) ? 1 : 0; }
template <int N>
struct WalkParamsC {
    static constexpr int NC = walk_inner_bits(N);   // columns held in the constant bank (the inner flips)
    static constexpr int MN = walk_const_midneg(N);
    double2 col[NC + 1][N];                // col[j][i] = a_ij, j < U; col[U][i] = -a_{i,U-1} (used by MN = 1 and unit)
    const double2* A;                      // device, row-major (staged to shared memory)
    ddc* items;                            // item partials; body chunk c0 + g -> items[item0 + g]
    uint64_t item0;
#ifdef PERM_DEBUG_CHECKS
    uint64_t nitems;                       // (debug build: bounds of `items`)
#endif
    uint64_t c0;                           // first body chunk
    uint64_t count;                        // body chunks
    int32_t eb;                            // log2 body chunk length (>= U)
    int32_t scaled;                        // unit-column walk: multiply every item partial by `scale`
    ddc scale;
};

template <class C, int T>
struct InnerStepC {
    static constexpr int N = C::N;
    static __device__ __forceinline__ void run(const WalkParamsC<N>& P, int z, double (&wr)[N], double (&wi)[N],
                                               double zmid, double& ar, double& ai) {
        constexpr int U = C::U;
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            const int jj = J + z * (T + 1);          // == J; distinct expression per use (no CSE/hoist)
            if constexpr (J == U - 1) {
                // new bit = 1 ^ bit_U(rank): sign zmid = -+1
                if constexpr (WalkParamsC<N>::MN == 1) {
                    // the column's sign by address (+a at col[U-1], -a at col[U]): DADD R, R, UR
                    const int jm = jj + (zmid < 0.0 ? 1 : 0);
#pragma unroll
                    for (int i = 0; i < N; i++) {
                        const double2 a = P.col[jm][i];
                        wr[i] += a.x;
                        wi[i] += a.y;
                    }
                } else {
                    // the column is a uniform-register operand, so this DFMA reads two vector registers
#pragma unroll
                    for (int i = 0; i < N; i++) {
                        const double2 a = P.col[jj][i];
                        wr[i] = fma(zmid, a.x, wr[i]);
                        wi[i] = fma(zmid, a.y, wi[i]);
                    }
                }
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;  // new bit = 1 ^ bit_{J+1}(t)
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const double2 a = P.col[jj][i];
                    if (PLUS) { wr[i] += a.x; wi[i] += a.y; }
                    else      { wr[i] -= a.x; wi[i] -= a.y; }
                }
            }
        }
        if constexpr (T & 1) term_acc<N, C::K, +1>(wr, wi, ar, ai);
        else                 term_acc<N, C::K, -1>(wr, wi, ar, ai);
        if constexpr (T + 1 < (1 << U)) InnerStepC<C, T + 1>::run(P, z, wr, wi, zmid, ar, ai);
    }
};

// Unit-column walk over the pairs (T, T+1), T even, of the inner block: the row sums v hold Gray bit 0 = 0 (column 0
// is all ones and never added), term T + (bit 0) reads v + 1.  Gray bit 0 of rank T is bit 1 of T, so the pair is
// s_T (prod (v + 1) - prod v) with s_T = +1 if bit 1 of T is 0, else -1 (signs (-1)^{r+1}, App. A).
template <class C, int T>
struct InnerStepCU {
    static constexpr int N = C::N;
    static __device__ __forceinline__ void run(const WalkParamsC<N>& P, int z, double (&wr)[N], double (&wi)[N],
                                               double zmid, double& ar, double& ai) {
        constexpr int U = C::U;
        static_assert(T % 2 == 0 && U >= 2, "pairs of an aligned block of >= 4 ranks");
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);            // >= 1
            const int jj = J + z * (T + 1);
            if constexpr (J == U - 1) {
                // the mid-block column with its sign by address (+a at col[U-1], -a at col[U]): DADD R, R, UR
                const int jm = jj + (zmid < 0.0 ? 1 : 0);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const double2 a = P.col[jm][i];
                    wr[i] += a.x;
                    wi[i] += a.y;
                }
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
#pragma unroll
                for (int i = 0; i < N; i++) {
                    const double2 a = P.col[jj][i];
                    if (PLUS) { wr[i] += a.x; wi[i] += a.y; }
                    else      { wr[i] -= a.x; wi[i] -= a.y; }
                }
            }
        }
        constexpr int SP = ((T >> 1) & 1) ? -1 : 1;
        // the shifted product keeps the walk's K chains; the plain one two (n = 44: 0.6650 -> 0.6670; interleaving
        // the two products' chains lost the uniform-register columns, profiles/round2_unit_column_rates.txt)
        term_acc<N, (C::K < 2 ? C::K : 2), -SP>(wr, wi, ar, ai);
        term_acc_shift1<N, C::K, SP>(wr, wi, ar, ai);
        if constexpr (T + 2 < (1 << U)) InnerStepCU<C, T + 2>::run(P, z, wr, wi, zmid, ar, ai);
    }
};

template <class C, bool UNIT>
__device__ __forceinline__ void walk_chunk_const(const WalkParamsC<C::N>& P, uint32_t lc, uint32_t lb, uint64_t c,
                                                 ddc& acc) {
    constexpr int N = C::N, U = C::U;
    const int e = P.eb;                                   // warp-uniform (kernel parameter)
    double wr[N], wi[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
        const double2 b = lds_c(lb + i * 16);
        wr[i] = b.x;
        wi[i] = b.y;
    }
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    for (int j = N - 2; j >= e - 1; j--) {                // seed, App. A steps 5-8 (shared memory), descending
        const double f = (double)((x >> j) & 1ull);
        flip_dyn<N>(lc + (uint32_t)(j * N) * 16u, f, wr, wi);
    }
    const int nblk = 1 << (e - U);                        // >= 2: the planner sends only e > U here
    const uint64_t cpar = c & 1ull;
    constexpr int kFoldMask = (U >= walk_fold_bits_const(N)) ? 0 : ((1 << (walk_fold_bits_const(N) - U)) - 1);
    double ar = 0.0, ai = 0.0;
    for (int q = 0; q < nblk; q++) {
        const int z = q >> 30;                            // 0 (nblk <= 2^27); uniform, loop-variant
        if (q > 0) {
            const int j = U + __ffs(q) - 1;
            const uint64_t nb = (j + 1 < e) ? (uint64_t)((q >> (j + 1 - U)) & 1) : cpar;
            flip_add<N>(lc + (uint32_t)(j * N) * 16u + (nb ? C::NEG : 0u), wr, wi);
        }
        if constexpr (UNIT) InnerStepCU<C, 0>::run(P, z, wr, wi, (q & 1) ? -1.0 : 1.0, ar, ai);
        else                InnerStepC<C, 0>::run(P, z, wr, wi, (q & 1) ? -1.0 : 1.0, ar, ai);   // bit_U(rank) = q & 1 (e > U)
        if (((q + 1) & kFoldMask) == 0 || q + 1 == nblk) {
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            ar = 0.0;
            ai = 0.0;
        }
    }
}

// Register cap of the constant-bank walk for order N (0: the default __launch_bounds__ kernel).  Whether
// ptxas keeps the per-use parameter loads on the uniform datapath (LDCU -> DADD R, R, UR: one vector
// register read per update instead of two) depends on its register allocation; these caps are the ones
// measured to produce LDCU with 0 spill bytes (rescanned in round 2 for the per-chunk partial stores,
// profiles/round2_const_ldcu_scan.txt; n = 42 only with its mid-block sign by address), and
// tests/test_abi_cpu.py checks the built library still does.
#ifndef PERM_CAP44
#define PERM_CAP44 244
#endif
__host__ __device__ constexpr int walk_const_maxnreg(int n) {
#ifdef PERM_CONST_MAXNREG_ALL
    return PERM_CONST_MAXNREG_ALL;                  // scans only (tools/const_ldcu_scan.sh)
#else
    return n == 33 ? (PERM_U2_FROM33 ? 176 : 172) : n == 34 ? 192 : n == 35 ? 196
         : n == 36 ? (PERM_U2_FROM33 ? 196 : 188) : n == 37 ? 204 : n == 38 ? (PERM_U2_FROM33 ? 204 : 200)
         : n == 39 ? 212 : n == 40 ? 212 : n == 41 ? 212 : n == 42 ? 216 : n == 43 ? 204 : n == 44 ? PERM_CAP44
         : n == 45 ? 236 : n == 46 ? 240 : n == 47 ? 240 : n == 48 ? 244 : 0;
#endif
}

template <int N, bool UNIT>
__device__ __forceinline__ void walk_body_c(const WalkParamsC<N>& P);

template <int N, bool UNIT>
__global__ void __launch_bounds__(walk_block_threads(N)) walk_kernel_c(const __grid_constant__ WalkParamsC<N> P) {
    walk_body_c<N, UNIT>(P);
}

template <int N, bool UNIT>
__global__ void __maxnreg__(walk_const_maxnreg(N) > 0 ? walk_const_maxnreg(N) : 255)
    walk_kernel_cm(const __grid_constant__ WalkParamsC<N> P) {
    walk_body_c<N, UNIT>(P);
}

template <int N, bool UNIT>
__device__ __forceinline__ void walk_body_c(const WalkParamsC<N>& P) {
    using C = WCfg<N, 1>;
    extern __shared__ double2 smem[];
    double2* scol = smem;                                    // scol[j*N + i] = a_ij, then -a_ij at + N*N
    double2* sbase = smem + 2 * N * N;
    for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
        const int i = k / N, j = k - i * N;
        const double2 a = P.A[k];
        scol[j * N + i] = a;
        scol[N * N + j * N + i] = make_double2(-a.x, -a.y);
    }
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
    // warp-uniform item loop (every lane runs every iteration; lanes past the end walk a valid chunk
    // and drop the result), so all control flow and column addresses stay on the uniform datapath
    const uint32_t ln = threadIdx.x & 31u;
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (uint64_t)__shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t base = wid * 32u; base < P.count; base += nw * 32u) {
        const uint64_t g = base + ln;
        const bool valid = g < P.count;
        ddc part;
        part.re.hi = part.re.lo = part.im.hi = part.im.lo = 0.0;
        walk_chunk_const<C, UNIT>(P, lc, lb, P.c0 + (valid ? g : 0), part);
        if (P.scaled) part = ddc_mul(part, P.scale);          // unit-column walk: back to the units of A
#ifdef PERM_DEBUG_CHECKS
        PERM_DCHECK(!valid || P.item0 + g < P.nitems);
#endif
        if (valid) P.items[P.item0 + g] = part;
    }
}

// ------------------------------------------------------------------------------------------------
// Small whole permanents (2^{n-1-b} <= kSmallMaxChunks chunks, n <= 16): ONE launch of a thread-block
// cluster of up to 16 CTAs.  Thread t of CTA k walks chunk k T + t (one chunk each), the CTA reduces its T
// chunk partials by the canonical pairwise tree in shared memory (its T chunks are an aligned subtree),
// and after a cluster barrier CTA 0 gathers the CTA roots through distributed shared memory and finishes
// the tree -> per(A) = 2(-1)^n root.  Bit-identical to the multi-launch path (same chunks, same tree), but
// without the separate tree launches: the latency of a small permanent is one kernel.
template <int N>
__global__ void __launch_bounds__(kSmallMaxThreads) walk_small_kernel(const double2* __restrict__ A, int e,
                                                                     ddc* __restrict__ raw, ddc* __restrict__ out_dd,
                                                                     double2* __restrict__ out_c) {
    namespace cg = cooperative_groups;
    using C = WalkCfg<N>;
    static_assert(C::S == 1, "small path: one lane per chunk");
    extern __shared__ double2 smem[];
    __shared__ ddc tree[kSmallMaxThreads];
    cg::cluster_group cluster = cg::this_cluster();
    stage_matrix<C>(A, smem, smem + 2 * N * C::P);
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem + 2 * N * C::P);
    const int T = blockDim.x, t = threadIdx.x;
    const uint64_t c = (uint64_t)cluster.block_rank() * T + t;
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    // the chunk length of a whole permanent is a compile-time function of n: with it as a constant the
    // seeding loop and the block loop unroll (same operations in the same order as the generic walk)
    constexpr int E = walk_chunk_log2(N);
    (void)e;
    if constexpr (C::U >= 1 && E > 0) {
        // seed w(gray(c 2^E)) -- the same operations in the same order as seed_rows -- sharing the warp-uniform
        // high columns: with T a multiple of 32 the lanes' chunks differ only in their low 5 bits, so Gray bits
        // >= 5 of c, i.e. columns >= E + 5, are the same for the whole warp.  Lane i (< N) folds those columns
        // into row i once; the rows are broadcast; each lane adds its own low columns.
        constexpr int R = C::R;
        double wr[R], wi[R];
        const uint64_t x = ((c ^ (c >> 1)) << E) | ((c & 1ull) << (E - 1));
        int jlo = E - 1;                                 // lowest column folded by this lane alone
        if (T >= 32) {
            const int lane = t & 31;
            double pr = 0.0, pi = 0.0;
            if (lane < N) {
                const double2 b = lds_c(lb + (uint32_t)lane * 16u);
                pr = b.x;
                pi = b.y;
                for (int j = N - 2; j >= E + 5; j--) {
                    const double f = (double)((x >> j) & 1ull);
                    const double2 a = lds_c(lc + (uint32_t)(j * C::P + lane) * 16u);
                    pr = fma(f, a.x, pr);
                    pi = fma(f, a.y, pi);
                }
            }
#pragma unroll
            for (int i = 0; i < R; i++) {
                wr[i] = __shfl_sync(0xffffffffu, pr, i);
                wi[i] = __shfl_sync(0xffffffffu, pi, i);
            }
            for (int j = (E + 4 < N - 2 ? E + 4 : N - 2); j >= jlo; j--) {
                const double f = (double)((x >> j) & 1ull);
                flip_dyn<R>(lc + (uint32_t)(j * C::P) * 16u, f, wr, wi);
            }
        } else {
            seed_rows<C>(lc, lb, x, jlo, wr, wi);
        }
        walk_seeded<C>(lc, 0u, c, E, wr, wi, acc);
    } else {
        single_term<C>(lc, lb, 0u, c, acc);
    }
    // node (L+1, k) = node (L, 2k) + node (L, 2k+1): the first levels inside each warp by shuffles (lane l
    // combines with l + off when l is a multiple of 2 off), then the warp roots in shared memory
    const int wl = T < 32 ? T : 32;
    const unsigned wmask = T < 32 ? ((1u << T) - 1u) : 0xffffffffu;     // T is a power of two
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const ddc o = shfl_down_ddc(acc, off, wmask);
        if (off < wl && (t & (2 * off - 1)) == 0) acc = ddc_add(acc, o);
    }
    if ((t & 31) == 0) tree[t >> 5] = acc;
    __syncthreads();
    const int nw = (T + 31) >> 5;                        // warp roots: finished by warp 0 in shuffles
    if (nw > 1 && t < 32) {
        ddc r;
        r.re.hi = r.re.lo = r.im.hi = r.im.lo = 0.0;
        if (t < nw) r = tree[t];
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {          // nw <= kSmallMaxThreads / 32 = 8
            const ddc o = shfl_down_ddc(r, off);
            if (off < nw && (t & (2 * off - 1)) == 0) r = ddc_add(r, o);
        }
        if (t == 0) tree[0] = r;
    }
    // every CTA pushes its root into CTA 0's shared memory (distributed shared memory store), then ONE cluster
    // barrier (release/acquire): after it only CTA 0 reads, from its own shared memory, so the others may exit
    __shared__ ddc roots[16];
    __syncthreads();
    if (t == 0) *cluster.map_shared_rank(&roots[cluster.block_rank()], 0) = tree[0];
    cluster.sync();
    const int nb = (int)cluster.num_blocks();
    if (cluster.block_rank() == 0 && t < 32) {
        ddc r;
        r.re.hi = r.re.lo = r.im.hi = r.im.lo = 0.0;
        if (t < nb) r = roots[t];
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) {
            const ddc o = shfl_down_ddc(r, off, wmask);
            if (off < nb && (t & (2 * off - 1)) == 0) r = ddc_add(r, o);
        }
        if (t == 0) {
            if (raw) *raw = r;
            const double f = (N & 1) ? -2.0 : 2.0;       // 2 (-1)^n, exact
            r.re.hi *= f; r.re.lo *= f; r.im.hi *= f; r.im.lo *= f;
            if (out_dd) *out_dd = r;
            if (out_c) *out_c = make_double2(r.re.hi + r.re.lo, r.im.hi + r.im.lo);
        }
    }
}

template <int N>
cudaError_t walk_small_launch(const double2* A_dev, int e, uint64_t chunks, ddc* raw, ddc* out_dd, double2* out_c,
                              cudaStream_t s) {
    if constexpr (N > kSmallMaxN || WalkCfg<N>::S != 1) {
        return cudaErrorInvalidValue;
    } else {
        using C = WalkCfg<N>;
        if (chunks < 1 || chunks > (uint64_t)kSmallMaxChunks || (chunks & (chunks - 1))) return cudaErrorInvalidValue;
        if (e != walk_chunk_log2(N)) return cudaErrorInvalidValue;    // the kernel walks chunks of 2^b(n)
        int ncta = (int)(chunks / 64);
        ncta = ncta < 1 ? 1 : (ncta > 16 ? 16 : ncta);
        const int T = (int)(chunks / (uint64_t)ncta);
        // function attributes once per device (host latency matters here: this path is one small launch)
        int dev = 0;
        cudaError_t err = cudaGetDevice(&dev);
        if (err != cudaSuccess) return err;
        static std::once_flag once[64];
        static cudaError_t attr_err[64];
        if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
        std::call_once(once[dev], [] (int d) {
            cudaError_t e2 = cudaFuncSetAttribute(walk_small_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)C::smem_bytes);
            if (e2 == cudaSuccess)
                e2 = cudaFuncSetAttribute(walk_small_kernel<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            attr_err[d] = e2;
        }, dev);
        if (attr_err[dev] != cudaSuccess) return attr_err[dev];
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)ncta, 1, 1);
        cfg.blockDim = dim3((unsigned)T, 1, 1);
        cfg.dynamicSmemBytes = C::smem_bytes;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)ncta;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, walk_small_kernel<N>, A_dev, e, raw, out_dd, out_c);
    }
}

// Diagnostic: w(ranks[k]) via the same seeding code (perm_c128_seed); one lane group per rank.
template <int N>
__global__ void seed_kernel(const double2* __restrict__ A, const uint64_t* __restrict__ ranks, int count,
                            double2* __restrict__ out) {
    using C = WalkCfg<N>;
    extern __shared__ double2 smem[];
    stage_matrix<C>(A, smem, smem + 2 * N * C::P);
    const uint32_t h = threadIdx.x % C::S;
    const uint32_t hoff = h * (uint32_t)C::R * 16u;
    const uint32_t lc = (uint32_t)__cvta_generic_to_shared(smem) + hoff;
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(smem + 2 * N * C::P) + hoff;
    const int groups = (int)(gridDim.x * (blockDim.x / C::S));
    for (int k = (int)(blockIdx.x * (blockDim.x / C::S) + threadIdx.x / C::S); k < count; k += groups) {
        const uint64_t r = ranks[k];
        double wr[C::R], wi[C::R];
        seed_rows<C>(lc, lb, r ^ (r >> 1), 0, wr, wi);
#pragma unroll
        for (int i = 0; i < C::R; i++) {
            const int row = (int)h * C::R + i;
            if (row < N) out[(size_t)k * N + row] = make_double2(wr[i], wi[i]);
        }
    }
}

// seg[k] is segment seg_index[k] of the launch plan; item0[k] the global index of its first item.
template <int N>
cudaError_t walk_launch_smem(const WalkLaunch& L, const Segment* seg, const uint64_t* item0, int nseg, int grid) {
    using C = WalkCfg<N>;
    WalkParams P;
    P.A = L.A_dev;
    P.items = L.items;
    P.nitems = L.nitems;
    uint64_t pre = 0;
    for (int s = 0; s < kMaxSegments; s++) {
        P.seg_pre[s] = pre;
        if (s < nseg) {
            P.seg_c0[s] = seg[s].c0;
            P.seg_e[s] = seg[s].e;
            P.seg_item0[s] = item0[s];
            pre += seg[s].count;
        } else {
            P.seg_c0[s] = 0;
            P.seg_e[s] = 0;
            P.seg_item0[s] = 0;
        }
    }
    P.seg_pre[kMaxSegments] = pre;
    P.nseg = nseg;
    P.scaled = L.scaled;
    P.scale = L.scale;
    // the dynamic shared-memory attribute was set by walk_occupancy<N> (abi.cu geometry cache)
    walk_kernel<N><<<grid, C::NT, C::smem_bytes, L.stream>>>(P);
    return cudaGetLastError();
}

// Dynamic shared memory attribute of a unit-column walk kernel (set once per kernel and device; the non-unit kernel's
// is set by walk_occupancy_c).
template <class K>
cudaError_t unit0_attr(K* kern, size_t smem) {
    static std::once_flag once[64];
    static cudaError_t err[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::call_once(once[dev], [&] {
        err[dev] = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    return err[dev];
}

// Launches the walk over L.seg; item k of the plan (segments in order, chunks in rank order) writes its dd
// partial to L.items[k].  For the constant-bank orders the largest segment (the aligned body) runs in
// walk_kernel_c on L.grid blocks and the remaining segments, if any, in walk_kernel on L.grid_edge blocks.
template <int N>
cudaError_t walk_launch(const WalkLaunch& L) {
    uint64_t item0[kMaxSegments];
    uint64_t pre = 0;
    for (int s = 0; s < L.nseg; s++) {
        item0[s] = pre;
        pre += L.seg[s].count;
    }
    if constexpr (walk_const_path(N) && walk_inner_bits(N) >= 1) {
        if (L.use_const) {
            const Segment& b = L.seg[L.body];
            WalkParamsC<N> P;
            for (int j = 0; j < WalkParamsC<N>::NC; j++)
                for (int i = 0; i < N; i++) P.col[j][i] = L.A_host[(size_t)i * N + j];
            for (int i = 0; i < N; i++) {
                const double2 a = L.A_host[(size_t)i * N + WalkParamsC<N>::NC - 1];
                P.col[WalkParamsC<N>::NC][i] = make_double2(-a.x, -a.y);
            }
            P.A = L.A_dev;
            P.items = L.items;
            P.item0 = item0[L.body];
#ifdef PERM_DEBUG_CHECKS
            P.nitems = L.nitems;
#endif
            P.c0 = b.c0;
            P.count = b.count;
            P.eb = b.e;
            P.scaled = L.scaled;
            P.scale = L.scale;
            const bool unit = walk_unit0(N) && L.unit0;
            if constexpr (walk_unit0(N)) {
                if (unit) {
                    cudaError_t ea = cudaSuccess;
                    if constexpr (walk_const_maxnreg(N) > 0)
                        ea = unit0_attr(walk_kernel_cm<N, true>, WCfg<N, 1>::smem_bytes);
                    else
                        ea = unit0_attr(walk_kernel_c<N, true>, WCfg<N, 1>::smem_bytes);
                    if (ea != cudaSuccess) return ea;
                    if constexpr (walk_const_maxnreg(N) > 0)
                        walk_kernel_cm<N, true><<<L.grid, walk_block_threads(N), WCfg<N, 1>::smem_bytes, L.stream>>>(P);
                    else
                        walk_kernel_c<N, true><<<L.grid, walk_block_threads(N), WCfg<N, 1>::smem_bytes, L.stream>>>(P);
                }
            }
            if (!unit) {
                if constexpr (walk_const_maxnreg(N) > 0)
                    walk_kernel_cm<N, false><<<L.grid, walk_block_threads(N), WCfg<N, 1>::smem_bytes, L.stream>>>(P);
                else
                    walk_kernel_c<N, false><<<L.grid, walk_block_threads(N), WCfg<N, 1>::smem_bytes, L.stream>>>(P);
            }
            cudaError_t err = cudaGetLastError();
            if (err != cudaSuccess || L.grid_edge == 0) return err;
            Segment rest[kMaxSegments];
            uint64_t rest0[kMaxSegments];
            int nr = 0;
            for (int s = 0; s < L.nseg; s++)
                if (s != L.body) {
                    rest[nr] = L.seg[s];
                    rest0[nr++] = item0[s];
                }
            return walk_launch_smem<N>(L, rest, rest0, nr, L.grid_edge);
        }
    }
    return walk_launch_smem<N>(L, L.seg, item0, L.nseg, L.grid);
}

// Occupancy of walk_kernel_c (0 when the constant-bank path does not exist for this order).
template <int N>
cudaError_t walk_occupancy_c(int* blocks_per_sm) {
    *blocks_per_sm = 0;
    if constexpr (walk_const_path(N) && walk_inner_bits(N) >= 1) {
        const void* k;
        if constexpr (walk_const_maxnreg(N) > 0) k = (const void*)walk_kernel_cm<N, false>;
        else                                     k = (const void*)walk_kernel_c<N, false>;
        cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)WCfg<N, 1>::smem_bytes);
        if (err != cudaSuccess) return err;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k, walk_block_threads(N),
                                                             WCfg<N, 1>::smem_bytes);
    }
    return cudaSuccess;
}

// blocks_per_sm: occupancy; walkers_per_block: independent chunk walkers (lane groups) per block.
template <int N>
cudaError_t walk_occupancy(int* blocks_per_sm, int* walkers_per_block) {
    using C = WalkCfg<N>;
    cudaError_t err = cudaFuncSetAttribute(walk_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    *walkers_per_block = C::NT / C::S;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, walk_kernel<N>, C::NT, C::smem_bytes);
}

template <int N>
cudaError_t walk_seed_launch(const double2* A_dev, const uint64_t* ranks_dev, int count, double2* w_out,
                             cudaStream_t s) {
    using C = WalkCfg<N>;
    cudaError_t err = cudaFuncSetAttribute(seed_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    int grid = (count * C::S + 127) / 128;
    if (grid < 1) grid = 1;
    seed_kernel<N><<<grid, 128, C::smem_bytes, s>>>(A_dev, ranks_dev, count, w_out);
    return cudaGetLastError();
}

}  // namespace perm
