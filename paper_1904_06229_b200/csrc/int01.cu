// int01.cu -- exact permanents of 0-1 matrices (BASELINE config 3).
//
// Same Gray walk as the complex path (App. A), in integers: with g_i = 2 w_i,
//     g_i(x) = a_{i,n} - sum_{j<n} a_ij + 2 sum_{j<n, x_j=1} a_ij    in [-n, n]   (int32)
//     Sum = sum_r (-1)^{r+1} prod_i g_i(gray r)  =  2^n * P(0, 2^{n-1})
//     per = 2 (-1)^n P  =  (-1)^n Sum / 2^{n-1}.
// Products: rows in groups of 6 in int32 (n^6 < 2^31 for n <= 28), pairs of groups in int64,
// then 64x64 -> 128 (and a further 128x64 for n > 24) modulo 2^128; the signed sum is kept mod 2^128
// in unsigned __int128.  The result is exact when |Sum| = 2^{n-1} per <= 2^{n-1} n! < 2^127, i.e.
// n <= 28 (R10); the low n-1 bits of Sum must be zero (self-check, PERM_E_CHECK).  For
// 29 <= n <= 33 the same walk runs over all 2^n subsets of Eq. (3) (row sums a_ij, no pinned column),
// whose signed sum is -(-1)^n per itself -- exact in int128 while n! < 2^127.
//
// Mapping: grid (blocks_per_matrix, B); each block stages its matrix (validating 0/1 bytes) in shared
// memory as int32 column increments 2 a_ij; each thread walks aligned chunks of 2^E ranks with the
// unrolled inner block of 2^U steps (compile-time columns and signs, warp-uniform broadcast loads).
// Per-block partial sums (exact, order-free) go to the workspace; a final kernel adds them per
// matrix, checks divisibility and writes per as int128.
// n = 20..24 and (0-1 entries) n = 29..33 walk a row/column-permuted copy with consecutive term pairs factored
// over the rows a bit-0 flip leaves unchanged (see "pair-factored walk" below).
#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace perm {

typedef unsigned __int128 u128;

template <int N>
struct I01Cfg {
    static constexpr int U = walk_inner_bits(N);
    static constexpr int NT = 128;
    static constexpr int NP = (N + 3) & ~3;          // column stride (ints): 16-byte aligned columns
    // n <= 28: the half-range Glynn walk (2^{n-1} terms, Sum = 2^{n-1} per must stay below 2^127);
    // 29 <= n <= 33: the full-range Ryser walk of Eq. (3) (2^n terms, Sum = -(-1)^n per, |per| <= n! < 2^127)
    static constexpr bool FULL = N > kMaxGlynnInt01N;
    static constexpr int NB = FULL ? N : N - 1;      // Gray bits (columns walked)
};

// Flips whose sign is known only at run time (mid-block bit U-1, block boundary) can read +CM a or -CM a by address
// (IADD3, alu pipe) instead of computing z * CM a (IMAD, fma pipe): kZNeg for both in the pair-factored walk,
// kPNeg = 0 / 1 (mid-block) / 2 (both) in the plain walk -- a pipe-balance choice, bit-identical results.
#ifndef PERM_INT01_ZNEG
#define PERM_INT01_ZNEG 1
#endif
#ifndef PERM_INT01_PNEG
#define PERM_INT01_PNEG 2
#endif
constexpr bool kZNeg = PERM_INT01_ZNEG;
constexpr int kPNeg = PERM_INT01_PNEG;
template <int N>
constexpr uint32_t kZNegOff = 4u * (uint32_t)(N * ((N + 3) & ~3));   // byte offset of the negated columns

__device__ __forceinline__ int lds_i(uint32_t addr) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// Four consecutive rows of a column in one 16-byte load (broadcast: every lane reads the same column).
__device__ __forceinline__ int4 lds_i4(uint32_t addr) {
    int4 v;
    asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// g += z * column (z = +-1, or 0/1 when seeding); col = address of row 0 of the column.
template <int N>
__device__ __forceinline__ void int_flip(uint32_t col, int z, int (&g)[N]) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
        const int4 a = lds_i4(col + 4u * (uint32_t)i);
        g[i] += z * a.x;
        if (i + 1 < N) g[i + 1] += z * a.y;
        if (i + 2 < N) g[i + 2] += z * a.z;
        if (i + 3 < N) g[i + 3] += z * a.w;
    }
}

// g += column (PLUS) or g -= column, compile-time sign.
template <int N, bool PLUS>
__device__ __forceinline__ void int_flip_static(uint32_t col, int (&g)[N]) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
        const int4 a = lds_i4(col + 4u * (uint32_t)i);
        const int v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (i + k < N) g[i + k] = PLUS ? g[i + k] + v[k] : g[i + k] - v[k];
    }
}

// prod_i g_i mod 2^128.
template <int N>
__device__ __forceinline__ u128 int_product(const int (&g)[N]) {
    constexpr int NG = (N + 5) / 6;
    int p[NG];
#pragma unroll
    for (int k = 0; k < NG; k++) {
        p[k] = g[6 * k];
#pragma unroll
        for (int i = 6 * k + 1; i < 6 * k + 6 && i < N; i++) p[k] *= g[i];
    }
    if constexpr (NG == 1) {
        return (u128)(__int128)(long long)p[0];
    } else {
        constexpr int NQ = (NG + 1) / 2;
        long long q[NQ];
#pragma unroll
        for (int k = 0; k < NQ; k++)
            q[k] = (2 * k + 1 < NG) ? (long long)p[2 * k] * (long long)p[2 * k + 1] : (long long)p[2 * k];
        if constexpr (NQ == 1) {
            return (u128)(__int128)q[0];
        } else {
            // signed 64 x 64 -> 128: unsigned high part minus the two-complement corrections
            const unsigned long long a = (unsigned long long)q[0], b = (unsigned long long)q[1];
            unsigned long long lo = a * b;
            unsigned long long hi = __umul64hi(a, b) - ((unsigned long long)(q[0] >> 63) & b) -
                                    ((unsigned long long)(q[1] >> 63) & a);
#pragma unroll
            for (int k = 2; k < NQ; k++) {
                const unsigned long long yl = (unsigned long long)q[k];
                const unsigned long long nl = lo * yl;
                unsigned long long nh = __umul64hi(lo, yl) + hi * yl;
                if (q[k] < 0) nh -= lo;
                lo = nl;
                hi = nh;
            }
            return ((u128)hi << 64) | (u128)lo;
        }
    }
}

template <int N, int SIGN>
__device__ __forceinline__ void int_term(const int (&g)[N], u128& acc) {
    const u128 p = int_product<N>(g);
    if (SIGN > 0) acc += p; else acc -= p;
}

// n <= 24 (at most four int32 groups): the 128-bit product and the 128-bit accumulate are replaced by 28-bit
// limbs.  With u = p0 p1 = u1 2^28 + u0 and w = p2 p3 = w1 2^28 + w0 (0 <= u0, w0 < 2^28, |u1|, |w1| <=
// n^12 / 2^28 < 2^27.1), the term is u0 w0 + 2^28 (u0 w1 + u1 w0) + 2^56 u1 w1; each limb sum grows by
// < 2^56.1 per term and is kept in int64 (one IMAD.WIDE with accumulate per partial product), separately for
// the + and - terms, and folded into the exact int128 total every 64 terms (64 x 2^56.1 < 2^63).  Three
// groups: u0 p2 + 2^28 u1 p2; two: p0 p1 (< n^12 < 2^56); one: p0.
template <int N>
constexpr bool kLimb = ((N + 5) / 6) <= 4;
constexpr int kLimbFoldBlocks = 8;                // inner blocks of 2^U <= 8 terms between folds

struct Limbs {
    long long p0, p1, p2, m0, m1, m2;
};

// s += a b, signed 32 x 32 -> 64 with a 64-bit addend: one IMAD.WIDE (plain C makes ptxas widen first and
// multiply 64 x 64)
__device__ __forceinline__ void mad_wide(long long& s, int a, int b) {
    asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(s) : "r"(a), "r"(b));
}

template <int N, int SIGN>
__device__ __forceinline__ void int_term(const int (&g)[N], Limbs& L) {
    constexpr int NG = (N + 5) / 6;
    int p[NG];
#pragma unroll
    for (int k = 0; k < NG; k++) {
        p[k] = g[6 * k];
#pragma unroll
        for (int i = 6 * k + 1; i < 6 * k + 6 && i < N; i++) p[k] *= g[i];
    }
    long long& s0 = SIGN > 0 ? L.p0 : L.m0;
    long long& s1 = SIGN > 0 ? L.p1 : L.m1;
    long long& s2 = SIGN > 0 ? L.p2 : L.m2;
    if constexpr (NG == 1) {
        s0 += p[0];
    } else if constexpr (NG == 2) {
        mad_wide(s0, p[0], p[1]);
    } else {
        const long long u = (long long)p[0] * p[1];
        const int u0 = (int)((unsigned)u & 0x0FFFFFFFu), u1 = (int)(u >> 28);
        if constexpr (NG == 3) {
            mad_wide(s0, u0, p[2]);
            mad_wide(s1, u1, p[2]);
        } else {
            const long long w = (long long)p[2] * p[3];
            const int w0 = (int)((unsigned)w & 0x0FFFFFFFu), w1 = (int)(w >> 28);
            mad_wide(s0, u0, w0);
            mad_wide(s1, u0, w1);
            mad_wide(s1, u1, w0);
            mad_wide(s2, u1, w1);
        }
    }
}

__device__ __forceinline__ void limb_fold(Limbs& L, u128& acc) {
    const __int128 d0 = (__int128)(L.p0 - L.m0), d1 = (__int128)(L.p1 - L.m1), d2 = (__int128)(L.p2 - L.m2);
    acc += (u128)d0 + ((u128)d1 << 28) + ((u128)d2 << 56);
    L = Limbs{0, 0, 0, 0, 0, 0};
}

// ---- pair-factored walk (perm_int01 / perm_pm1, 20 <= n <= 24) ------------------------------------------------
// Consecutive ranks 2q, 2q+1 of an aligned block differ in Gray bit 0 only and carry opposite signs
// ((-1)^{r+1}, App. A), so their two terms sum to  prod_{i<Z} g_i * (prod_{i>=Z} g'_i - prod_{i>=Z} g_i)  when the
// Z rows i < Z have a_{i,0} = 0 (unchanged by the bit-0 flip).  The block stages A with the Gray column holding the
// most zeros moved to position 0 and those zero rows moved first (per(A) is invariant under row and column
// permutations, and the walk still visits every sign vector once), then walks with a compile-time Z from a short
// menu (the largest entry <= the zero count; Z < 12 keeps the plain walk).  Per pair of terms: rows [0, 12) form
// u = p0 p1 (two int32 groups of 6, |u| <= n^12 < 2^55.1); rows [12, n) form W = vB vA with vB over [12, n-6) and
// vA over [n-6, n) (int32 each, the constant rows' part computed once per pair); F = W' - W (|F| <= 2 n^{n-12} <
// 2^56.1) and the pair adds u F, exactly, in three int64 28-bit-limb sums (u0 F0, u0 F1 + u1 F0, u1 F1: < 2^56.6
// per pair) folded into the int128 total every kZFoldPairs pairs.  Against the plain walk this drops the
// unchanged rows' updates at every bit-0 flip and their products at every second term.
template <int N>
constexpr bool kZSplit = N >= 20 && N <= 24;
#ifndef PERM_INT01_ZU
#define PERM_INT01_ZU 4
#endif
constexpr int kZU = PERM_INT01_ZU;                 // inner Gray bits of the pair-factored walk (2^{U-1} pairs per block)
constexpr int kZFoldPairs = 64;                    // 64 x 2^56.6 < 2^63

// minimum resident blocks per SM asked of ptxas (register cap); 1 = no cap
#ifndef PERM_INT01_MINB
#define PERM_INT01_MINB 1
#endif
constexpr int kInt01MinBlocks = PERM_INT01_MINB;

template <int N>
constexpr bool kZSplitFull = N > kMaxGlynnInt01N && N <= kMaxInt01N;   // 0-1 only (row sums >= 0)

// full-range orders: Z = n - M for M = 12 (exact u64 W), 15, 18 varying rows
__device__ __forceinline__ int zsplit_menu_full(int z, int n) {
    return z >= n - 12 ? n - 12 : z >= n - 15 ? n - 15 : z >= n - 18 ? n - 18 : 0;
}

// largest menu entry <= z (and <= n - 2), 0 = plain walk
__device__ __forceinline__ int zsplit_menu(int z, int n) {
    const int zm = z < n - 2 ? z : n - 2;
    return zm >= 18 ? 18 : zm >= 16 ? 16 : zm >= 14 ? 14 : zm >= 12 ? 12 : 0;
}

// g += column (PLUS) or g -= column for rows [LO, N) only (the rows a bit-0 flip can change).
template <int N, int LO, bool PLUS>
__device__ __forceinline__ void int_flip_rows(uint32_t col, int (&g)[N]) {
#pragma unroll
    for (int i = LO & ~3; i < N; i += 4) {
        const int4 a = lds_i4(col + 4u * (uint32_t)i);
        const int v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (i + k >= LO && i + k < N) g[i + k] = PLUS ? g[i + k] + v[k] : g[i + k] - v[k];
    }
}

template <int N, int LO, int HI>
__device__ __forceinline__ int int_rowprod(const int (&g)[N], int init) {
    int p = init;
#pragma unroll
    for (int i = LO; i < HI; i++) p *= g[i];
    return p;
}

__device__ __forceinline__ long long mul_wide(int a, int b) {
    long long r;
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}

struct ZLimbs {
    long long s0, s1, s2;
};

// W = vB vA for the current row sums; cB / cA = the constant rows' part of each group (computed once per pair)
template <int N, int Z>
__device__ __forceinline__ long long zsplit_w(const int (&g)[N], int cB, int cA) {
    constexpr int BV = Z > 12 ? Z : 12;            // B = [12, N-6): constant [12, min(Z, N-6)), varying after
    constexpr int AV = Z > N - 6 ? Z : N - 6;      // A = [N-6, N):  constant [N-6, max(Z, N-6)), varying after
    const int vB = int_rowprod<N, (BV < N - 6 ? BV : N - 6), N - 6>(g, cB);
    const int vA = int_rowprod<N, AV, N>(g, cA);
    return mul_wide(vA, vB);
}

template <int N, int Z, int U, int T>
struct IntInnerZ {
    static __device__ __forceinline__ void run(uint32_t sc, int (&g)[N], int zmid, ZLimbs& L) {
        constexpr int NP = I01Cfg<N>::NP;
        if constexpr (T > 0) {                       // flip of Gray bit J >= 1 (all rows)
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                if constexpr (kZNeg) int_flip_static<N, true>(sc + (zmid < 0 ? kZNegOff<N> : 0u) + 4u * (uint32_t)(J * NP), g);
                else int_flip<N>(sc + 4u * (uint32_t)(J * NP), zmid, g);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
                int_flip_static<N, PLUS>(sc + 4u * (uint32_t)(J * NP), g);
            }
        }
        constexpr int CB = Z < N - 6 ? Z : N - 6;   // constant rows of group B: [12, CB); of group A: [N-6, Z)
        const int cB = int_rowprod<N, 12, CB>(g, 1);
        const int cA = int_rowprod<N, N - 6, (Z > N - 6 ? Z : N - 6)>(g, 1);
        const long long u = mul_wide(int_rowprod<N, 0, 6>(g, 1), int_rowprod<N, 6, 12>(g, 1));
        const long long w0 = zsplit_w<N, Z>(g, cB, cA);         // term T (sign -)
        int_flip_rows<N, Z, ((T >> 1) & 1) == 0>(sc, g);         // bit 0 -> term T + 1 (sign +)
        const long long w1 = zsplit_w<N, Z>(g, cB, cA);
        const long long F = w1 - w0;
        const int u0 = (int)((unsigned)u & 0x0FFFFFFFu), u1 = (int)(u >> 28);
        const int f0 = (int)((unsigned)F & 0x0FFFFFFFu), f1 = (int)(F >> 28);
        mad_wide(L.s0, u0, f0);
        mad_wide(L.s1, u0, f1);
        mad_wide(L.s1, u1, f0);
        mad_wide(L.s2, u1, f1);
        if constexpr (T + 2 < (1 << U)) IntInnerZ<N, Z, U, T + 2>::run(sc, g, zmid, L);
    }
};

__device__ __forceinline__ void zlimb_fold(ZLimbs& L, u128& acc) {
    acc += (u128)(__int128)L.s0 + ((u128)(__int128)L.s1 << 28) + ((u128)(__int128)L.s2 << 56);
    L = ZLimbs{0, 0, 0};
}

// 29 <= n <= 33 (full-range Ryser of Eq. (3), 0-1 entries: row sums r_i in [0, n], products mod 2^128): the same pair
// factoring, pair = C (W' - W) mod 2^128 with C = prod_{i<Z} r_i (int32 groups of 6 rows, 33^6 < 2^31; u64 pairs of
// groups, 33^12 < 2^61; then mod 2^128) once per pair and W = prod_{i>=Z} r_i per term -- an exact u64 when the
// M = n - Z varying rows number <= 12 (then D = W' - W is an int64), else mod 2^128.
__device__ __forceinline__ u128 mul_u128_u64(u128 a, unsigned long long y) {
    const unsigned long long lo = (unsigned long long)a, hi = (unsigned long long)(a >> 64);
    return ((u128)(hi * y + __umul64hi(lo, y)) << 64) | (u128)(lo * y);
}

template <int N, int LO, int HI>
__device__ __forceinline__ unsigned long long rows_u64(const int (&g)[N]) {    // exact: HI - LO <= 12 rows
    static_assert(HI - LO <= 12 && HI - LO >= 1, "u64 row product: at most 12 rows");
    constexpr int MID = (HI - LO) > 6 ? LO + 6 : HI;
    const unsigned a = (unsigned)int_rowprod<N, LO + 1, MID>(g, g[LO]);
    if constexpr (MID == HI) return (unsigned long long)a;
    else return (unsigned long long)a * (unsigned)int_rowprod<N, MID + 1, HI>(g, g[MID]);
}

template <int N, int LO, int HI>
__device__ __forceinline__ u128 rows_u128(const int (&g)[N]) {                 // mod 2^128
    if constexpr (HI - LO <= 12) {
        return (u128)rows_u64<N, LO, HI>(g);
    } else {
        constexpr int MID = HI - 12 < LO + 12 ? HI - 12 : LO + 12;
        const unsigned long long hi12 = rows_u64<N, MID, HI>(g);
        if constexpr (MID - LO <= 12) {
            const unsigned long long a = rows_u64<N, LO, MID>(g);
            return ((u128)__umul64hi(a, hi12) << 64) | (u128)(a * hi12);
        } else {
            return mul_u128_u64(rows_u128<N, LO, MID>(g), hi12);
        }
    }
}

template <int N, int Z, int U, int T>
struct IntInnerZF {
    static __device__ __forceinline__ void run(uint32_t sc, int (&g)[N], int zmid, u128& acc) {
        constexpr int NP = I01Cfg<N>::NP;
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                if constexpr (kZNeg) int_flip_static<N, true>(sc + (zmid < 0 ? kZNegOff<N> : 0u) + 4u * (uint32_t)(J * NP), g);
                else int_flip<N>(sc + 4u * (uint32_t)(J * NP), zmid, g);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
                int_flip_static<N, PLUS>(sc + 4u * (uint32_t)(J * NP), g);
            }
        }
        const u128 C = rows_u128<N, 0, Z>(g);
        if constexpr (N - Z <= 12) {
            const unsigned long long w0 = rows_u64<N, Z, N>(g);
            int_flip_rows<N, Z, ((T >> 1) & 1) == 0>(sc, g);
            const unsigned long long w1 = rows_u64<N, Z, N>(g);
            const long long D = (long long)(w1 - w0);                 // |D| < 2^61
            const unsigned long long clo = (unsigned long long)C, chi = (unsigned long long)(C >> 64);
            const unsigned long long du = (unsigned long long)D;
            unsigned long long hi = __umul64hi(clo, du) + chi * du;
            if (D < 0) hi -= clo;                                     // C * (du - 2^64) mod 2^128
            acc += ((u128)hi << 64) | (u128)(clo * du);
        } else {
            const u128 w0 = rows_u128<N, Z, N>(g);
            int_flip_rows<N, Z, ((T >> 1) & 1) == 0>(sc, g);
            const u128 w1 = rows_u128<N, Z, N>(g);
            acc += C * (w1 - w0);
        }
        if constexpr (T + 2 < (1 << U)) IntInnerZF<N, Z, U, T + 2>::run(sc, g, zmid, acc);
    }
};

template <int N, int U, int T>
struct IntInner {
    template <class Acc>
    static __device__ __forceinline__ void run(uint32_t sc, int (&g)[N], int zmid, Acc& acc) {
        if constexpr (T > 0) {
            constexpr int J = ctz_c((unsigned)T);
            constexpr int NP = I01Cfg<N>::NP;
            if constexpr (J == U - 1) {
                if constexpr (kPNeg >= 1) int_flip_static<N, true>(sc + (zmid < 0 ? kZNegOff<N> : 0u) + 4u * (uint32_t)(J * NP), g);
                else int_flip<N>(sc + 4u * (uint32_t)(J * NP), zmid, g);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
                int_flip_static<N, PLUS>(sc + 4u * (uint32_t)(J * NP), g);
            }
        }
        if constexpr (T & 1) int_term<N, +1>(g, acc);
        else                 int_term<N, -1>(g, acc);
        if constexpr (T + 1 < (1 << U)) IntInner<N, U, T + 1>::run(sc, g, zmid, acc);
    }
};

template <int N>
__device__ __forceinline__ void int_seed(uint32_t sc, uint32_t sbase, uint64_t x, int j0, int (&g)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++) g[i] = lds_i(sbase + 4 * i);
    for (int j = j0; j < I01Cfg<N>::NB; j++) {
        const int f = (int)((x >> j) & 1ull);
        int_flip<N>(sc + 4u * (uint32_t)(j * I01Cfg<N>::NP), f, g);
    }
}

template <int N>
__device__ __forceinline__ void int_chunk(uint32_t sc, uint32_t sbase, uint64_t c, int e, u128& acc) {
    constexpr int U = I01Cfg<N>::U;
    int g[N];
    if (e == 0) {
        int_seed<N>(sc, sbase, c ^ (c >> 1), 0, g);
        if (c & 1ull) int_term<N, +1>(g, acc); else int_term<N, -1>(g, acc);
        return;
    }
    if constexpr (U >= 1) {
        const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
        int_seed<N>(sc, sbase, x, e - 1, g);
        const uint64_t nblk = 1ull << (e - U);
        const uint64_t cpar = c & 1ull;
        [[maybe_unused]] Limbs L{0, 0, 0, 0, 0, 0};
        for (uint64_t q = 0; q < nblk; q++) {
            if (q > 0) {
                const int j = U + __ffsll((long long)q) - 1;
                const uint64_t nb = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1ull) : cpar;
                if constexpr (kPNeg >= 2) int_flip_static<N, true>(sc + (nb ? kZNegOff<N> : 0u) + 4u * (uint32_t)(j * I01Cfg<N>::NP), g);
                else int_flip<N>(sc + 4u * (uint32_t)(j * I01Cfg<N>::NP), nb ? -1 : 1, g);
            }
            const uint64_t nbm = (U < e) ? (q & 1ull) : cpar;
            if constexpr (kLimb<N>) {
                static_assert((kLimbFoldBlocks << U) <= 64, "limb sums must stay below 2^63");
                IntInner<N, U, 0>::run(sc, g, nbm ? -1 : 1, L);
                if ((q & (kLimbFoldBlocks - 1)) == kLimbFoldBlocks - 1 || q + 1 == nblk) limb_fold(L, acc);
            } else {
                IntInner<N, U, 0>::run(sc, g, nbm ? -1 : 1, acc);
            }
        }
    }
}

// ---- quad-factored walk (perm_pm1, 20 <= n <= 24, columns without zero entries) ------------------------------
// The four ranks of an aligned quad 4t .. 4t+3 run through the four sign pairs (delta_0, delta_1) of Gray bits 0 and
// 1 at fixed higher bits (App. A).  With the rows negated so that the bit-0 column is all +1 (per changes by the
// product of the row signs) and the bit-1 column negated if that balances the classes below, every row reads
// g_i = h_i + delta_0 + delta_1 a_i1 with h_i the part of the other columns: the rows with a_i1 = +1 (class P,
// rows [0, Z)) take the values h + {2, 0, -2} as delta_0 + delta_1 = 2, 0, -2, the rows with a_i1 = -1 (class M)
// as delta_0 - delta_1 does.  The term signs (-1)^{r+1} equal d delta_0 delta_1 over the quad with d = +1 iff
// bit 2 of r is set, so the quad sums to
//     d [ M(0) (P(2) + P(-2)) - P(0) (M(2) + M(-2)) ],   X(s) = prod_{i in X} (h_i + s),
// six products over about n/2 rows instead of four over n, and two row adds instead of four flips per row.  The
// walk carries h (Gray bits >= 2 only); |h_i + s| <= n, a class of <= 13 rows multiplies exactly in int64
// (24^13 < 2^60), the two class products exactly in int128.
template <int N, bool PM1>
constexpr bool kQuad = PM1 && N >= 20 && N <= 24;
constexpr int kQuadCode = 1000;                    // plan code kQuadCode + Z selects the quad walk with |P| = Z

template <int N, int LO, int HI, int OFF>
__device__ __forceinline__ long long quad_prod(const int (&h)[N]) {
    static_assert(HI - LO >= 1 && HI - LO <= 13, "quad class: 1..13 rows");
    constexpr int M1 = (HI - LO) > 6 ? LO + 6 : HI;
    int p0 = h[LO] + OFF;
#pragma unroll
    for (int i = LO + 1; i < M1; i++) p0 *= h[i] + OFF;
    if constexpr (M1 == HI) {
        return (long long)p0;
    } else {
        constexpr int M2 = (HI - M1) > 6 ? M1 + 6 : HI;
        int p1 = h[M1] + OFF;
#pragma unroll
        for (int i = M1 + 1; i < M2; i++) p1 *= h[i] + OFF;
        const long long q = mul_wide(p0, p1);
        if constexpr (M2 == HI) return q;
        else return q * (long long)(h[M2] + OFF);          // the 13th row
    }
}

template <int N, int Z, int U, int T>
struct IntInnerQ {
    static __device__ __forceinline__ void run(uint32_t sc, int (&h)[N], int zmid, u128& acc) {
        constexpr int NP = I01Cfg<N>::NP;
        static_assert(T % 4 == 0 && U >= 3, "quads of an aligned block of >= 8 ranks");
        if constexpr (T > 0) {                       // flip of Gray bit J >= 2 (bits 0 and 1 live in the quad formula)
            constexpr int J = ctz_c((unsigned)T);
            if constexpr (J == U - 1) {
                int_flip_static<N, true>(sc + (zmid < 0 ? kZNegOff<N> : 0u) + 4u * (uint32_t)(J * NP), h);
            } else {
                constexpr bool PLUS = ((T >> (J + 1)) & 1) == 0;
                int_flip_static<N, PLUS>(sc + 4u * (uint32_t)(J * NP), h);
            }
        }
        const long long P2 = quad_prod<N, 0, Z, 2>(h), P0 = quad_prod<N, 0, Z, 0>(h), Pm = quad_prod<N, 0, Z, -2>(h);
        const long long M2 = quad_prod<N, Z, N, 2>(h), M0 = quad_prod<N, Z, N, 0>(h), Mm = quad_prod<N, Z, N, -2>(h);
        const __int128 v = (__int128)M0 * (P2 + Pm) - (__int128)P0 * (M2 + Mm);
        if constexpr (((T >> 2) & 1) != 0) acc += (u128)v; else acc -= (u128)v;
        if constexpr (T + 4 < (1 << U)) IntInnerQ<N, Z, U, T + 4>::run(sc, h, zmid, acc);
    }
};

// one aligned chunk of 2^e ranks (e >= kZU) on the quad walk; hbase = the rows' base without columns 0 and 1
template <int N, int Z>
__device__ __forceinline__ void int_chunk_q(uint32_t sc, uint32_t hbase, uint64_t c, int e, u128& acc) {
    constexpr int U = kZU;
    int h[N];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    int_seed<N>(sc, hbase, x, e - 1, h);              // e - 1 >= 2: columns 0 and 1 are not seeded
    const uint64_t nblk = 1ull << (e - U);
    const uint64_t cpar = c & 1ull;
    for (uint64_t q = 0; q < nblk; q++) {
        if (q > 0) {
            const int j = U + __ffsll((long long)q) - 1;
            const uint64_t nb = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1ull) : cpar;
            int_flip_static<N, true>(sc + (nb ? kZNegOff<N> : 0u) + 4u * (uint32_t)(j * I01Cfg<N>::NP), h);
        }
        const uint64_t nbm = (U < e) ? (q & 1ull) : cpar;
        IntInnerQ<N, Z, U, 0>::run(sc, h, nbm ? -1 : 1, acc);
    }
}

template <int N, int Z>
__device__ __forceinline__ void int_walk_q(uint32_t sc, uint32_t hbase, int e, uint64_t chunks, uint64_t c0, u128& acc) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks; c += T)
        int_chunk_q<N, Z>(sc, hbase, c0 + c, e, acc);    // the plan selects the quad walk only when e >= kZU
}

template <int N, int Z>
__device__ __forceinline__ void int_chunk_z(uint32_t sc, uint32_t sbase, uint64_t c, int e, u128& acc) {
    constexpr int U = kZU;
    constexpr uint64_t kFoldBlocks = (uint64_t)kZFoldPairs >> (U - 1);
    static_assert(U >= 2 && kFoldBlocks >= 1, "pair-factored walk: U >= 2");
    int g[N];
    const uint64_t x = ((c ^ (c >> 1)) << e) | ((c & 1ull) << (e - 1));
    int_seed<N>(sc, sbase, x, e - 1, g);
    const uint64_t nblk = 1ull << (e - U);
    const uint64_t cpar = c & 1ull;
    [[maybe_unused]] ZLimbs L{0, 0, 0};
    for (uint64_t q = 0; q < nblk; q++) {
        if (q > 0) {
            const int j = U + __ffsll((long long)q) - 1;
            const uint64_t nb = (j + 1 < e) ? ((q >> (j + 1 - U)) & 1ull) : cpar;
            if constexpr (kZNeg) int_flip_static<N, true>(sc + (nb ? kZNegOff<N> : 0u) + 4u * (uint32_t)(j * I01Cfg<N>::NP), g);
            else int_flip<N>(sc + 4u * (uint32_t)(j * I01Cfg<N>::NP), nb ? -1 : 1, g);
        }
        const uint64_t nbm = (U < e) ? (q & 1ull) : cpar;
        if constexpr (I01Cfg<N>::FULL) {
            IntInnerZF<N, Z, U, 0>::run(sc, g, nbm ? -1 : 1, acc);
        } else {
            IntInnerZ<N, Z, U, 0>::run(sc, g, nbm ? -1 : 1, L);
            if ((q & (kFoldBlocks - 1)) == kFoldBlocks - 1 || q + 1 == nblk) zlimb_fold(L, acc);
        }
    }
}

// the chunks [c0, c0 + chunks) of this thread's stride, plain walk (Z = 0) or pair-factored (Z >= 12)
template <int N, int Z>
__device__ __forceinline__ void int_walk(uint32_t sc, uint32_t sbase, int e, uint64_t chunks, uint64_t c0, u128& acc) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks; c += T) {
        if constexpr (Z > 0) {
            if (e >= kZU) { int_chunk_z<N, Z>(sc, sbase, c0 + c, e, acc); continue; }
        }
        int_chunk<N>(sc, sbase, c0 + c, e, acc);       // chunk c0 + c: ranks [(c0+c) 2^e, (c0+c+1) 2^e)
    }
}

// ws layout: [int flag][pad to 16][u128 partials[B][nblk]]
// PM1 = false: entries are bytes 0/1 (perm_int01); PM1 = true: signed bytes in {-1, 0, 1} (perm_pm1, the
// Bernoulli +-1 ensemble of Sec. V).  Either way |g_i| <= n, so the product and exactness bounds hold.
template <int N, bool PM1>
__global__ void __launch_bounds__(I01Cfg<N>::NT, kInt01MinBlocks) int01_kernel(const uint8_t* __restrict__ A, int e,
                                                              uint64_t chunks, u128* __restrict__ partials,
                                                              int* __restrict__ flag, uint64_t c0, int accum,
                                                              int zsplit) {
    constexpr int NP = I01Cfg<N>::NP;
    constexpr bool FULL = I01Cfg<N>::FULL;
    constexpr int CM = FULL ? 1 : 2;               // column increment: 2 a_ij (Glynn) or a_ij (Ryser)
    constexpr bool ZS = (kZSplit<N> && !FULL) || (kZSplitFull<N> && !PM1);
    // s_col[j*NP + i] = CM a_ij (rows N..NP-1 zero), then its negation (flips whose sign is known only at run time
    // read -CM a by address); the pair-factored walk's permuted copy and its negation follow
    __shared__ __align__(16) int s_col[(ZS ? 4 : 2) * N * NP];
    __shared__ int s_base[(ZS ? 2 : 1) * N];      // Glynn: a_{i,n} - sum_{j<n} a_ij; Ryser: 0
    const int64_t m = blockIdx.y;
    const uint8_t* a = A + m * (N * N);
    for (int k = threadIdx.x; k < 2 * N * NP; k += blockDim.x) s_col[k] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
        const int v = PM1 ? (int)(int8_t)a[k] : (int)a[k];
        if (PM1 ? (v < -1 || v > 1) : (v > 1)) atomicOr(flag, 1);
        const int i = k / N, j = k - i * N;
        const int cv = PM1 ? CM * (v < -1 ? -1 : (v > 1 ? 1 : v)) : CM * (v & 1);
        s_col[j * NP + i] = cv;
        s_col[N * NP + j * NP + i] = -cv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        int s = 0;
        for (int j = 0; j < N - 1; j++) s += s_col[j * NP + i];
        s_base[i] = FULL ? 0 : s_col[(N - 1) * NP + i] / 2 - s / 2;
    }
    __syncthreads();
    uint32_t sc = (uint32_t)__cvta_generic_to_shared(s_col);
    uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_base);
    u128 acc = 0;
    int zsel = 0;
    [[maybe_unused]] int qsign = 1;
    if constexpr (ZS) {
        // plan of the pair-factored walk (block-uniform): the Gray column js with the most zero entries (lowest index
        // on ties) goes to position 0, its zero rows first (stable order)
        __shared__ int s_plan[5 + N];                 // [zsel, js, quad: c1, tau, sign, row order]
        if (zsplit && threadIdx.x < 32) {
            const int lane = threadIdx.x;
            int cnt = -1;
            if (lane < N - 1) {
                cnt = 0;
                for (int i = 0; i < N; i++) cnt += s_col[lane * NP + i] == 0;
            }
            int best = cnt, bj = lane;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const int ob = __shfl_xor_sync(0xffffffffu, best, off), oj = __shfl_xor_sync(0xffffffffu, bj, off);
                if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
            }
            if (lane == 0) {
                s_plan[0] = FULL ? zsplit_menu_full(best, N) : zsplit_menu(best, N);
                s_plan[1] = bj;
                int r = 0;
                for (int i = 0; i < N; i++) if (s_col[bj * NP + i] == 0) s_plan[5 + r++] = i;
                for (int i = 0; i < N; i++) if (s_col[bj * NP + i] != 0) s_plan[5 + r++] = i;
                if constexpr (kQuad<N, PM1>) {
                    // no useful zeros: the quad plan -- bit-0 column c0 and bit-1 column c1 without zero entries,
                    // class P (rows whose a_{i,c1} matches the sign of a_{i,c0}, times tau) of size N/2 - 1 or N/2
                    if (s_plan[0] == 0 && e >= kZU) {
                        int q0 = -1, q1 = -1, tau = 1, zq = 0;
                        for (int j = 0; j < N - 1 && q0 < 0; j++) {
                            bool nz = true;
                            for (int i = 0; i < N; i++) nz = nz && s_col[j * NP + i] != 0;
                            if (nz) q0 = j;
                        }
                        for (int j = 0; j < N - 1 && q0 >= 0 && q1 < 0; j++) {
                            if (j == q0) continue;
                            int z = 0;
                            bool nz = true;
                            for (int i = 0; i < N; i++) {
                                const int v = s_col[j * NP + i];
                                nz = nz && v != 0;
                                z += (v > 0) == (s_col[q0 * NP + i] > 0);
                            }
                            if (!nz) continue;
                            const int zz = z < N - z ? z : N - z;
                            if (zz == N / 2 || zz == N / 2 - 1) { q1 = j; tau = (z == zz) ? 1 : -1; zq = zz; }
                        }
                        if (q1 >= 0) {
                            int sgn = tau, r2 = 0;
                            for (int i = 0; i < N; i++) {
                                const int si = s_col[q0 * NP + i] > 0 ? 1 : -1;
                                sgn *= si;
                                if ((s_col[q1 * NP + i] > 0 ? 1 : -1) * si * tau > 0) s_plan[5 + r2++] = i;
                            }
                            for (int i = 0; i < N; i++) {
                                const int si = s_col[q0 * NP + i] > 0 ? 1 : -1;
                                if ((s_col[q1 * NP + i] > 0 ? 1 : -1) * si * tau < 0) s_plan[5 + r2++] = i;
                            }
                            s_plan[0] = kQuadCode + zq;
                            s_plan[1] = q0;
                            s_plan[2] = q1;
                            s_plan[3] = tau;
                            s_plan[4] = sgn;
                        }
                    }
                }
            }
        }
        __syncthreads();
        zsel = zsplit ? s_plan[0] : 0;
        if constexpr (kQuad<N, PM1>) {
            if (zsel >= kQuadCode) {
                qsign = s_plan[4];
                // the quad plan's matrix A' = D_sigma A Q: columns c0, c1 first (c1 times tau), rows negated to
                // make column c0 all +1, class P first; per(A) = sign * per(A')
                const int q0 = s_plan[1], q1 = s_plan[2], tau = s_plan[3];
                for (int k = threadIdx.x; k < N * NP; k += blockDim.x) {
                    const int jj = k / NP, r = k - jj * NP;
                    int src = jj;
                    if (jj == 0) src = q0;
                    else if (jj == 1) src = q1;
                    else {                                    // the other columns in order, skipping q0 and q1
                        int t = jj - 2;
                        for (src = 0;; src++) {
                            if (src == q0 || src == q1) continue;
                            if (t-- == 0) break;
                        }
                    }
                    int v = 0;
                    if (r < N) {
                        const int row = s_plan[5 + r];
                        const int si = s_col[q0 * NP + row] > 0 ? 1 : -1;
                        v = si * (jj == 1 ? tau : 1) * s_col[src * NP + row];
                    }
                    s_col[2 * N * NP + k] = v;
                    s_col[3 * N * NP + k] = -v;
                }
                __syncthreads();
                // h base of A' (Gray bits >= 2 only): g = base + sum_{x_j = 1} 2 a'_j minus delta_0 a'_0 + delta_1 a'_1,
                // i.e. base' + a'_0 + a'_1 with a'_0 = +1 and a'_1 = +1 (class P) or -1 (class M)
                for (int r = threadIdx.x; r < N; r += blockDim.x) {
                    int t = 0;
                    for (int j = 0; j < N - 1; j++) t += s_col[2 * N * NP + j * NP + r];
                    s_base[N + r] = s_col[2 * N * NP + (N - 1) * NP + r] / 2 - t / 2 + 1 +
                                    (s_col[2 * N * NP + NP + r] > 0 ? 1 : -1);
                }
                __syncthreads();
                sc += 8u * (uint32_t)(N * NP);
                sbase += 4u * (uint32_t)N;
            }
        }
        if (zsel && zsel < kQuadCode) {
            const int js = s_plan[1];
            for (int k = threadIdx.x; k < N * NP; k += blockDim.x) {
                const int jj = k / NP, r = k - jj * NP;
                const int src = jj == 0 ? js : (jj == js ? 0 : jj);
                const int v = r < N ? s_col[src * NP + s_plan[5 + r]] : 0;
                s_col[2 * N * NP + k] = v;
                s_col[3 * N * NP + k] = -v;
            }
            for (int r = threadIdx.x; r < N; r += blockDim.x) s_base[N + r] = s_base[s_plan[5 + r]];
            __syncthreads();
            sc += 8u * (uint32_t)(N * NP);
            sbase += 4u * (uint32_t)N;
        }
    }
    if constexpr (ZS && FULL) {
        if (zsel == N - 12)      int_walk<N, N - 12>(sc, sbase, e, chunks, c0, acc);
        else if (zsel == N - 15) int_walk<N, N - 15>(sc, sbase, e, chunks, c0, acc);
        else if (zsel == N - 18) int_walk<N, N - 18>(sc, sbase, e, chunks, c0, acc);
        else                     int_walk<N, 0>(sc, sbase, e, chunks, c0, acc);
    } else if constexpr (ZS) {
        if constexpr (kQuad<N, PM1>) {
            if (zsel == kQuadCode + N / 2)          { int_walk_q<N, N / 2>(sc, sbase, e, chunks, c0, acc); zsel = -1; }
            else if (zsel == kQuadCode + N / 2 - 1) { int_walk_q<N, N / 2 - 1>(sc, sbase, e, chunks, c0, acc); zsel = -1; }
        }
        switch (zsel) {
            case -1: break;
            case 18: int_walk<N, 18>(sc, sbase, e, chunks, c0, acc); break;
            case 16: int_walk<N, 16>(sc, sbase, e, chunks, c0, acc); break;
            case 14: int_walk<N, 14>(sc, sbase, e, chunks, c0, acc); break;
            case 12: int_walk<N, 12>(sc, sbase, e, chunks, c0, acc); break;
            default: int_walk<N, 0>(sc, sbase, e, chunks, c0, acc); break;
        }
    } else {
        int_walk<N, 0>(sc, sbase, e, chunks, c0, acc);
    }
    // block reduction (exact; order irrelevant)
    unsigned long long lo = (unsigned long long)acc, hi = (unsigned long long)(acc >> 64);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long olo = __shfl_down_sync(0xffffffffu, lo, off);
        const unsigned long long ohi = __shfl_down_sync(0xffffffffu, hi, off);
        const u128 s = (((u128)hi << 64) | lo) + (((u128)ohi << 64) | olo);
        lo = (unsigned long long)s;
        hi = (unsigned long long)(s >> 64);
    }
    __shared__ u128 s_w[I01Cfg<N>::NT / 32];
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = ((u128)hi << 64) | lo;
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 t = 0;
        for (int w = 0; w < I01Cfg<N>::NT / 32; w++) t += s_w[w];
        if constexpr (ZS && kQuad<N, PM1>) {
            if (qsign < 0) t = (u128)0 - t;             // per(A) = sign * per(A') (quad plan)
        }
        u128* slot = partials + m * gridDim.x + blockIdx.x;
        *slot = accum ? *slot + t : t;                  // accum: later segments of a range add in (exact)
    }
}

__global__ void int01_final_kernel(const u128* __restrict__ partials, int nblk, int64_t B, int n,
                                   unsigned long long* __restrict__ out, int* __restrict__ flag) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= B) return;
    u128 s = 0;
    for (int k = 0; k < nblk; k++) s += partials[m * nblk + k];
    __int128 v;
    if (n > kMaxGlynnInt01N) {                    // full-range Ryser: per = (-1)^{n+1} Sum
        v = (__int128)s;
        if (!(n & 1)) v = -v;
    } else {
        const u128 mask = (((u128)1) << (n - 1)) - 1;
        if (s & mask) atomicOr(flag, 2);
        v = (__int128)s >> (n - 1);               // arithmetic shift: Sum / 2^{n-1}
        if (n & 1) v = -v;                        // per = (-1)^n Sum / 2^{n-1}
    }
    out[2 * m] = (unsigned long long)v;
    out[2 * m + 1] = (unsigned long long)((u128)v >> 64);
}

// PERM_INT01_ZSPLIT=0 (environment, read once) turns the pair-factored walk off (development comparisons)
static const int kInt01ZSplit = [] {
    const char* v = getenv("PERM_INT01_ZSPLIT");
    return (v && v[0] == '0') ? 0 : 1;
}();

struct I01Plan {
    int e;
    int nblk;
    uint64_t chunks;
};

// Resident blocks of int01_kernel<n> on the current device (SMs x occupancy), computed once per device.
// Sizing the grid to it matters: a grid of 2.3 waves leaves the last wave 70% idle.
#define PERM_R8I(M, b) M(b + 1) M(b + 2) M(b + 3) M(b + 4) M(b + 5) M(b + 6) M(b + 7) M(b + 8)
static int int01_resident_blocks(int n) {
    static std::once_flag once[64][kMaxInt01N + 1];
    static int res[64][kMaxInt01N + 1];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || n < 1 || n > kMaxInt01N) return 148 * 4;
    std::call_once(once[dev][n], [&] {
        int sms = 148, bps = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaErrorInvalidValue;
        switch (n) {
#define PERM_CASE(N) case N: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, int01_kernel<N, false>, \
                                                                                 I01Cfg<N>::NT, 0); break;
            PERM_R8I(PERM_CASE, 0) PERM_R8I(PERM_CASE, 8) PERM_R8I(PERM_CASE, 16) PERM_R8I(PERM_CASE, 24)
            PERM_CASE(33)
#undef PERM_CASE
            default: break;
        }
        if (e != cudaSuccess || bps < 1) bps = 4;
        res[dev][n] = sms * bps;
    });
    return res[dev][n];
}

// B matrices: floor(R / B) blocks per matrix when the batch is smaller than R (two waves of resident blocks),
// else one block per matrix; the chunk length makes every thread walk ~4 chunks.
static I01Plan int01_plan(int n, int64_t B) {
    const int U = walk_inner_bits(n);
    const int nb = n > kMaxGlynnInt01N ? n : n - 1;           // Gray bits
    // measured on B200 (tools/int01_scan.py, profiles/round2_int01_plan_scan.txt): two waves of resident blocks,
    // four chunks per thread -- more rounds mean shorter chunks and more seeding
    int64_t R = 2 * int01_resident_blocks(n);
    uint64_t rounds = 4;
    // development overrides (plan scans): PERM_INT01_WAVES = resident-block waves, PERM_INT01_ROUNDS = chunks
    // per thread
    if (const char* w = getenv("PERM_INT01_WAVES")) R = (int64_t)(R * atof(w));
    if (const char* r = getenv("PERM_INT01_ROUNDS")) rounds = (uint64_t)atoi(r);
    int64_t nblk = (B > 0 && B < R) ? R / B : 1;
    const uint64_t want = (uint64_t)nblk * 128u * rounds;      // chunks per matrix
    int lg = 0;
    while ((1ull << lg) < want) lg++;
    int e = nb - lg;
    if (e < U) e = U;
    if (e > nb) e = nb;
    if (n == 1) e = 0;
    I01Plan p;
    p.e = e;
    p.chunks = 1ull << (nb - e);
    const uint64_t need = (p.chunks + 127) / 128;
    if ((uint64_t)nblk > need) nblk = (int64_t)need;
    if (nblk < 1) nblk = 1;
    p.nblk = (int)nblk;
    return p;
}

size_t int01_workspace_bytes(int n, int64_t B) {
    const I01Plan p = int01_plan(n, B);
    return 16 + (size_t)B * p.nblk * sizeof(u128);
}

template <int N>
cudaError_t int01_launch_t(const uint8_t* A, int64_t B, const I01Plan& p, u128* partials, int* flag, bool pm1,
                           cudaStream_t s) {
    dim3 grid((unsigned)p.nblk, (unsigned)B);
    if (pm1) int01_kernel<N, true><<<grid, I01Cfg<N>::NT, 0, s>>>(A, p.e, p.chunks, partials, flag, 0, 0, kInt01ZSplit);
    else     int01_kernel<N, false><<<grid, I01Cfg<N>::NT, 0, s>>>(A, p.e, p.chunks, partials, flag, 0, 0, kInt01ZSplit);
    return cudaGetLastError();
}

#define PERM_R8(M, b) M(b + 1) M(b + 2) M(b + 3) M(b + 4) M(b + 5) M(b + 6) M(b + 7) M(b + 8)

cudaError_t int01_launch(const uint8_t* A, int n, int64_t B, bool pm1, void* out, void* ws, size_t ws_bytes,
                         cudaStream_t s, int* flag_host_status, int* launches) {
    *launches = 0;
    *flag_host_status = 0;
    if (B == 0) return cudaSuccess;
    if (B > 65535) return cudaErrorInvalidValue;   // gridDim.y; the ABI layer splits larger batches
    const I01Plan p = int01_plan(n, B);
    int* flag = (int*)ws;
    u128* partials = (u128*)((char*)ws + 16);
    cudaError_t err = cudaMemsetAsync(flag, 0, sizeof(int), s);
    if (err != cudaSuccess) return err;
    switch (n) {
#define PERM_CASE(N) case N: err = int01_launch_t<N>(A, B, p, partials, flag, pm1, s); break;
        PERM_R8(PERM_CASE, 0) PERM_R8(PERM_CASE, 8) PERM_R8(PERM_CASE, 16) PERM_R8(PERM_CASE, 24)
        PERM_CASE(33)
#undef PERM_CASE
        default: return cudaErrorInvalidValue;
    }
    if (err != cudaSuccess) return err;
    const int threads = 128;
    int01_final_kernel<<<(unsigned)((B + threads - 1) / threads), threads, 0, s>>>(
        partials, p.nblk, B, n, (unsigned long long*)out, flag);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    *launches = 2;
    int hflag = 0;
    err = cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (err != cudaSuccess) return err;
    err = cudaStreamSynchronize(s);
    if (err != cudaSuccess) return err;
    *flag_host_status = hflag;
    (void)ws_bytes;
    return cudaSuccess;
}

// ---- one matrix, a span of ranks (perm_int01_range): the span is cut like the complex walk's plan into
// maximal aligned pieces of 2^e ranks (e <= b; pieces with 0 < e < U become single ranks), one launch per
// run of equal pieces, all into the same per-block partial slots (accumulated), then one summing kernel.
__global__ void int01_range_final_kernel(const u128* __restrict__ partials, int nblk, u128* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    u128 s = 0;
    for (int k = 0; k < nblk; k++) s += partials[k];
    *out = s;
}

template <int N>
cudaError_t int01_range_seg(const uint8_t* A, int e, uint64_t c0, uint64_t count, int nblk, u128* partials, int* flag,
                            int accum, cudaStream_t s) {
    int01_kernel<N, false><<<dim3((unsigned)nblk, 1), I01Cfg<N>::NT, 0, s>>>(A, e, count, partials, flag, c0, accum, kInt01ZSplit);
    return cudaGetLastError();
}

size_t int01_range_workspace_bytes() { return 16 + 16 + (size_t)kInt01RangeBlocks * sizeof(u128); }

cudaError_t int01_range_launch(const uint8_t* A, int n, uint64_t k0, uint64_t k1, void* ws, cudaStream_t s,
                               unsigned long long* raw_host, int* flag_host_status, int* launches) {
    *launches = 0;
    *flag_host_status = 0;
    raw_host[0] = raw_host[1] = 0;
    if (k1 <= k0) return cudaSuccess;
    const int U = walk_inner_bits(n);
    const int nblk = kInt01RangeBlocks;           // (one wave of resident blocks measured slower: 0.28 vs 0.34)
    int* flag = (int*)ws;
    u128* out = (u128*)((char*)ws + 16);
    u128* partials = (u128*)((char*)ws + 32);
    // chunk length 2^b: ~8 chunks per thread of the nblk x 128 grid (>= 2^U, <= 2^30)
    const uint64_t T = (uint64_t)nblk * 128u;
    int b = 0;
    while (b < 30 && ((k1 - k0) >> (b + 1)) >= T * 8u) b++;
    if (b < U) b = U;
    cudaError_t err = cudaMemsetAsync(flag, 0, sizeof(int), s);
    int accum = 0;
    uint64_t r = k0;
    while (err == cudaSuccess && r < k1) {
        int e = (r == 0) ? 63 : __builtin_ctzll(r);
        if (e > b) e = b;
        while (e > 0 && (k1 - r) < (1ull << e)) e--;
        if (e < U) e = 0;
        uint64_t cnt = 1;
        if (e == b && e > 0) cnt = (k1 - r) >> b;                       // a run of whole 2^b chunks
        switch (n) {
#define PERM_CASE(N) case N: err = int01_range_seg<N>(A, e, r >> e, cnt, nblk, partials, flag, accum, s); break;
            PERM_R8(PERM_CASE, 0) PERM_R8(PERM_CASE, 8) PERM_R8(PERM_CASE, 16) PERM_R8(PERM_CASE, 24)
            PERM_CASE(33)
#undef PERM_CASE
            default: return cudaErrorInvalidValue;
        }
        accum = 1;
        ++*launches;
        r += cnt << e;
    }
    if (err != cudaSuccess) return err;
    int01_range_final_kernel<<<1, 32, 0, s>>>(partials, nblk, out);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    ++*launches;
    int hflag = 0;
    err = cudaMemcpyAsync(raw_host, out, sizeof(u128), cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess) err = cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
    *flag_host_status = hflag;
    return err;
}

}  // namespace perm
