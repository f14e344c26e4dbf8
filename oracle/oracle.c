/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the permanent.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this
 * library.  It shares no code, header, table or constant with the CUDA path
 * under paper_1904_06229_b200/ and neither side includes the other.
 *
 * Arithmetic: __float128 (IEEE binary128) for complex matrices, unsigned
 * __int128 (arithmetic mod 2^128) for 0-1 matrices.  Inputs are the same
 * bytes the GPU reads: row-major n x n, entry (i,j) = A[2*(i*n+j)] + i*A[2*(i*n+j)+1].
 * Results are returned as (hi, lo) double pairs so that the ~113-bit quad
 * value survives the trip back to Python: value = hi + lo.
 *
 * Citations: "P:<line>" is a line of the paper text (PAPER.md, arXiv
 * 1904.06229, Lundow & Markstrom) together with the equation/algorithm it is in.
 *
 * Functions and what pins them:
 *   oracle_naive_c128     Eq. (1), P:56-59            brute force; pinned by hand values,
 *                                                       per(J_n)=n!, D_n, diag, P7/P8 identities
 *   oracle_ryser_c128     Eq. (3), P:121-130          pinned against naive (n<=9) and closed forms
 *   oracle_subpermanent   App. A subpermanent, P:1131-1151 (steps 2-15 for a given (r, l))
 *   oracle_permanent_hr   App. A permanent, P:1153-1163 (distribute + subpermanent + combine)
 *   oracle_range_c128     App. A terms recomputed from steps 5-8 per rank (no walk)
 *   oracle_seed_c128      App. A steps 2,5-8: w(r)
 *   oracle_naive_i01 / oracle_ryser_i01   Eq. (1) / Eq. (3) in exact integers
 *   oracle_distribute, oracle_gray        App. A distribute P:1077-1095, Gray unrank P:1097-1106
 *   oracle_ryser_i8       Eq. (3) in exact integers for entries in {-1,0,1} (Sec. V Bernoulli +-1)
 *   oracle_sparse_partition / oracle_sparse_c128  App. B greedypartition + sparsepermanent
 *                                (P:1254-1293), pinned against Eq. (3) and by the enumeration count
 *   oracle_band_c128      App. C bandpermanent, literal polynomial steps; pinned against
 *                         Eq. (3)/(1) on banded matrices, Fibonacci (tridiagonal), diagonal, k >= n-1
 *   oracle_ryser_weighted_c128  Eq. (4), P:137-158 (repeated columns); pinned against Eq. (3) on the
 *                                expanded matrix, R = 1 (n! prod c_i) and the Boson-sampling
 *                                normalisation with collisions
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>
#include <quadmath.h>

typedef __float128 quad;
typedef struct { quad re, im; } qc;            /* complex binary128 */
typedef unsigned __int128 u128;

static inline qc qc_add(qc a, qc b) { qc r = { a.re + b.re, a.im + b.im }; return r; }
static inline qc qc_sub(qc a, qc b) { qc r = { a.re - b.re, a.im - b.im }; return r; }
static inline qc qc_mul(qc a, qc b) {
    qc r = { a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re };
    return r;
}
static inline qc qc_scale(qc a, quad s) { qc r = { a.re * s, a.im * s }; return r; }
static inline qc entry(const double* A, int n, int i, int j) {
    qc r = { (quad)A[2 * ((size_t)i * n + j)], (quad)A[2 * ((size_t)i * n + j) + 1] };
    return r;
}
static void put_q(double* out, quad q) {           /* (hi, lo) with hi + lo == q to ~106 bits */
    double hi = (double)q;
    out[0] = hi;
    out[1] = (double)(q - (quad)hi);
}
static void put_qc(double* out, qc v) { put_q(out, v.re); put_q(out + 2, v.im); }

/* ---------------- App. A integer helpers ---------------- */

/* distribute(n, m, i, k, l): q = floor(n/m), r = n mod m,
 * k = i*q + min(i, r), l = q + I(i < r). */
void oracle_distribute(uint64_t n, uint64_t m, uint64_t i, uint64_t* k, uint64_t* l) {
    uint64_t q = n / m, r = n % m;
    *k = i * q + (i < r ? i : r);
    *l = q + (i < r ? 1 : 0);
}

/* x := xor(k, rshift(k)) */
uint64_t oracle_gray(uint64_t k) { return k ^ (k >> 1); }

/* ---------------- Eq. (1): the definition ---------------- */

/* Sum over all n! permutations (Heap's algorithm enumerates them), each term the
 * plain product prod_i a_{i,pi(i)}.  n <= 10. */
int oracle_naive_c128(const double* A, int n, double* out4) {
    if (n < 1 || n > 10) return 1;
    int perm[10], c[10];
    for (int i = 0; i < n; i++) { perm[i] = i; c[i] = 0; }
    qc total = { 0, 0 };
    for (;;) {
        qc p = { 1, 0 };
        for (int i = 0; i < n; i++) p = qc_mul(p, entry(A, n, i, perm[i]));
        total = qc_add(total, p);
        /* Heap's algorithm, iterative form: next permutation */
        int i = 1;
        while (i < n && c[i] >= i) { c[i] = 0; i++; }
        if (i >= n) break;
        int s = (i % 2 == 0) ? 0 : c[i];
        int tmp = perm[s]; perm[s] = perm[i]; perm[i] = tmp;
        c[i]++;
    }
    put_qc(out4, total);
    return 0;
}

/* Eq. (1) for a 0-1 (uint8) matrix in exact integers. */
int oracle_naive_i01(const uint8_t* A, int n, uint64_t* out2) {
    if (n < 1 || n > 12) return 1;
    int perm[12], c[12];
    for (int i = 0; i < n; i++) { perm[i] = i; c[i] = 0; }
    u128 total = 0;
    for (;;) {
        u128 p = 1;
        for (int i = 0; i < n; i++) p *= (u128)A[(size_t)i * n + perm[i]];
        total += p;
        int i = 1;
        while (i < n && c[i] >= i) { c[i] = 0; i++; }
        if (i >= n) break;
        int s = (i % 2 == 0) ? 0 : c[i];
        int tmp = perm[s]; perm[s] = perm[i]; perm[i] = tmp;
        c[i]++;
    }
    out2[0] = (uint64_t)total;
    out2[1] = (uint64_t)(total >> 64);
    return 0;
}

/* ---------------- Eq. (3): Ryser, full range ----------------
 * per(A) = (-1)^n sum_{J subset N} (-1)^{|J|} prod_i sum_{j in J} a_ij.
 * The subsets J are visited in Gray-code order: J(r) = gray(r),
 * r = 0 .. 2^n - 1, and the row sums are updated by the one column whose
 * membership changed.  The 2^n ranks are split into m contiguous parts with
 * distribute; each part seeds its row sums from the definition
 * sum_{j in J} a_ij and the m partial sums are added in index order. */
static qc ryser_part(const double* A, int n, uint64_t k0, uint64_t len) {
    qc rs[64];
    qc S = { 0, 0 };
    uint64_t x = oracle_gray(k0);
    for (int i = 0; i < n; i++) {
        rs[i].re = 0; rs[i].im = 0;
        for (int j = 0; j < n; j++)
            if ((x >> j) & 1) rs[i] = qc_add(rs[i], entry(A, n, i, j));
    }
    for (uint64_t r = k0; r < k0 + len; r++) {
        if (r != k0) {
            uint64_t xn = oracle_gray(r);
            int j = __builtin_ctzll(xn ^ x);
            for (int i = 0; i < n; i++)
                rs[i] = ((xn >> j) & 1) ? qc_add(rs[i], entry(A, n, i, j))
                                        : qc_sub(rs[i], entry(A, n, i, j));
            x = xn;
        }
        qc p = { 1, 0 };
        for (int i = 0; i < n; i++) p = qc_mul(p, rs[i]);
        if (__builtin_popcountll(x) & 1) S = qc_sub(S, p); else S = qc_add(S, p);
    }
    return S;
}

int oracle_ryser_c128(const double* A, int n, int m, double* out4) {
    if (n < 1 || n > 40) return 1;
    if (m < 1) m = 1;
    uint64_t total = (uint64_t)1 << n;
    if ((uint64_t)m > total) m = (int)total;
    qc* part = (qc*)calloc((size_t)m, sizeof(qc));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < m; k++) {
        uint64_t k0, len;
        oracle_distribute(total, (uint64_t)m, (uint64_t)k, &k0, &len);
        part[k] = ryser_part(A, n, k0, len);
    }
    qc S = { 0, 0 };
    for (int k = 0; k < m; k++) S = qc_add(S, part[k]);
    free(part);
    if (n & 1) S = qc_scale(S, -1);
    put_qc(out4, S);
    return 0;
}

/* Eq. (3) in exact integer arithmetic for 0-1 matrices.  Row sums are
 * non-negative integers; products and the signed sum are taken mod 2^128
 * (unsigned __int128, two's complement), which is exact as long as
 * |per| < 2^127, i.e. n <= 33 since per <= n!. */
static u128 ryser_i01_part(const uint8_t* A, int n, uint64_t k0, uint64_t len) {
    int64_t rs[64];
    u128 S = 0;
    uint64_t x = oracle_gray(k0);
    for (int i = 0; i < n; i++) {
        rs[i] = 0;
        for (int j = 0; j < n; j++)
            if ((x >> j) & 1) rs[i] += A[(size_t)i * n + j];
    }
    for (uint64_t r = k0; r < k0 + len; r++) {
        if (r != k0) {
            uint64_t xn = oracle_gray(r);
            int j = __builtin_ctzll(xn ^ x);
            for (int i = 0; i < n; i++)
                rs[i] += ((xn >> j) & 1) ? A[(size_t)i * n + j] : -(int64_t)A[(size_t)i * n + j];
            x = xn;
        }
        u128 p = 1;
        for (int i = 0; i < n; i++) p *= (u128)(uint64_t)rs[i];
        if (__builtin_popcountll(x) & 1) S -= p; else S += p;
    }
    return S;
}

int oracle_ryser_i01(const uint8_t* A, int n, int m, uint64_t* out2) {
    if (n < 1 || n > 33) return 1;
    if (m < 1) m = 1;
    uint64_t total = (uint64_t)1 << n;
    if ((uint64_t)m > total) m = (int)total;
    u128* part = (u128*)calloc((size_t)m, sizeof(u128));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < m; k++) {
        uint64_t k0, len;
        oracle_distribute(total, (uint64_t)m, (uint64_t)k, &k0, &len);
        part[k] = ryser_i01_part(A, n, k0, len);
    }
    u128 S = 0;
    for (int k = 0; k < m; k++) S += part[k];
    free(part);
    if (n & 1) S = (u128)0 - S;
    out2[0] = (uint64_t)S;
    out2[1] = (uint64_t)(S >> 64);
    return 0;
}

/* Eq. (3) in exact integers for matrices with entries in {-1, 0, 1} (the Bernoulli +-1 ensemble of
 * Sec. V, P:846-860, and 0-1 matrices): row sums are small signed integers, products and the signed
 * sum are taken mod 2^128 -- exact while |per| < 2^127, i.e. n <= 33 since |per| <= n!. */
static u128 ryser_i8_part(const int8_t* A, int n, uint64_t k0, uint64_t len) {
    int64_t rs[64];
    u128 S = 0;
    uint64_t x = oracle_gray(k0);
    for (int i = 0; i < n; i++) {
        rs[i] = 0;
        for (int j = 0; j < n; j++)
            if ((x >> j) & 1) rs[i] += A[(size_t)i * n + j];
    }
    for (uint64_t r = k0; r < k0 + len; r++) {
        if (r != k0) {
            uint64_t xn = oracle_gray(r);
            int j = __builtin_ctzll(xn ^ x);
            for (int i = 0; i < n; i++)
                rs[i] += ((xn >> j) & 1) ? A[(size_t)i * n + j] : -(int64_t)A[(size_t)i * n + j];
            x = xn;
        }
        u128 p = 1;
        for (int i = 0; i < n; i++) p *= (u128)(int64_t)rs[i];      /* sign-extended, mod 2^128 */
        if (__builtin_popcountll(x) & 1) S -= p; else S += p;
    }
    return S;
}

int oracle_ryser_i8(const int8_t* A, int n, int m, uint64_t* out2) {
    if (n < 1 || n > 33) return 1;
    for (size_t k = 0; k < (size_t)n * n; k++)
        if (A[k] < -1 || A[k] > 1) return 2;
    if (m < 1) m = 1;
    uint64_t total = (uint64_t)1 << n;
    if ((uint64_t)m > total) m = (int)total;
    u128* part = (u128*)calloc((size_t)m, sizeof(u128));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < m; k++) {
        uint64_t k0, len;
        oracle_distribute(total, (uint64_t)m, (uint64_t)k, &k0, &len);
        part[k] = ryser_i8_part(A, n, k0, len);
    }
    u128 S = 0;
    for (int k = 0; k < m; k++) S += part[k];
    free(part);
    if (n & 1) S = (u128)0 - S;
    out2[0] = (uint64_t)S;
    out2[1] = (uint64_t)(S >> 64);
    return 0;
}

/* Batch of B independent 0-1 matrices, one Eq. (3) evaluation each. */
int oracle_ryser_i01_batch(const uint8_t* A, int n, int64_t B, uint64_t* out2) {
    if (n < 1 || n > 33) return 1;
    int bad = 0;
    #pragma omp parallel for schedule(dynamic, 1) reduction(|:bad)
    for (int64_t b = 0; b < B; b++) {
        u128 S = ryser_i01_part(A + (size_t)b * n * n, n, 0, (uint64_t)1 << n);
        if (n & 1) S = (u128)0 - S;
        out2[2 * b] = (uint64_t)S;
        out2[2 * b + 1] = (uint64_t)(S >> 64);
    }
    return bad;
}

/* Batch of B independent complex matrices, one Eq. (3) evaluation each. */
int oracle_ryser_c128_batch(const double* A, int n, int64_t B, double* out4) {
    if (n < 1 || n > 40) return 1;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; b++) {
        qc S = ryser_part(A + (size_t)b * 2 * n * n, n, 0, (uint64_t)1 << n);
        if (n & 1) S = qc_scale(S, -1);
        put_qc(out4 + 4 * b, S);
    }
    return 0;
}

/* ---------------- App. A, literally ---------------- */

/* nextset(t, j, x).  x[1..n] (1-indexed as in the paper). */
static void nextset(int* t, int* j, unsigned char* x) {
    *j = 1;                                     /* [1] j := 1 */
    *t = -*t;                                   /* [2] t := -t */
    if (*t == 1) {                              /* [2] if t = 1 then */
        while (x[*j] == 0) *j = *j + 1;         /* [3-5] while x_j = 0 do j := j+1 */
        *j = *j + 1;                            /* [6] j := j+1 */
    }
    x[*j] = 1 - x[*j];                          /* [7] x_j := 1 - x_j */
}

/* subpermanent steps 2-15 for a given start rank r and length l
 * (step 1, distribute, is done by the caller).  Returns S (no 2(-1)^n factor). */
static qc subpermanent_rl(const double* A, int n, uint64_t r, uint64_t l) {
    unsigned char x[66];
    qc w[64];
    uint64_t g = oracle_gray(r);                                /* [2] */
    memset(x, 0, sizeof(x));
    for (int j = 1; j <= n; j++) x[j] = (unsigned char)((g >> (j - 1)) & 1);
    int t = (r & 1) ? -1 : 1;                                   /* [3] t := (-1)^r */
    qc S = { 0, 0 };                                            /* [4] */
    for (int i = 1; i <= n; i++) {                              /* [5] */
        qc rowsum = { 0, 0 };
        for (int j = 1; j <= n; j++) rowsum = qc_add(rowsum, entry(A, n, i - 1, j - 1));
        w[i - 1] = qc_sub(entry(A, n, i - 1, n - 1), qc_scale(rowsum, (quad)0.5));
    }
    for (int j = 1; j <= n - 1; j++)                            /* [6] */
        if (x[j] == 1)
            for (int i = 1; i <= n; i++) w[i - 1] = qc_add(w[i - 1], entry(A, n, i - 1, j - 1)); /* [7] */
    for (uint64_t it = 0; it < l; it++) {                       /* [9] do l times */
        qc p = { 1, 0 };
        for (int i = 0; i < n; i++) p = qc_mul(p, w[i]);        /* [10] */
        int j;
        nextset(&t, &j, x);                                     /* [11] */
        S = (t == 1) ? qc_add(S, p) : qc_sub(S, p);             /* [12] S := S + t*p */
        if (it + 1 == l) break;  /* the trailing update may address column n (C4); it is never used */
        quad z = (quad)(2 * x[j] - 1);                          /* [13] */
        for (int i = 0; i < n; i++)                             /* [14] */
            w[i] = qc_add(w[i], qc_scale(entry(A, n, i, j - 1), z));
    }
    return S;
}

int oracle_subpermanent(const double* A, int n, uint64_t r, uint64_t l, double* out4) {
    if (n < 1 || n > 64) return 1;
    put_qc(out4, subpermanent_rl(A, n, r, l));
    return 0;
}

/* Same, but the rank range [r, r+l) is cut into `parts` contiguous pieces with
 * distribute and the pieces run on host threads; partials added in order.
 * (This is App. A's permanent() loop restricted to a sub-range.) */
int oracle_subpermanent_par(const double* A, int n, uint64_t r, uint64_t l, int parts, double* out4) {
    if (n < 1 || n > 64 || parts < 1) return 1;
    qc* part = (qc*)calloc((size_t)parts, sizeof(qc));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < parts; k++) {
        uint64_t k0, len;
        oracle_distribute(l, (uint64_t)parts, (uint64_t)k, &k0, &len);
        if (len) part[k] = subpermanent_rl(A, n, r + k0, len);
    }
    qc S = { 0, 0 };
    for (int k = 0; k < parts; k++) S = qc_add(S, part[k]);
    free(part);
    put_qc(out4, S);
    return 0;
}

/* permanent(A, n, m, S): S = 2 (-1)^n sum_k S_k, with S_k from
 * subpermanent(A, n, m, k) and distribute(2^{n-1}, m, k). */
int oracle_permanent_hr(const double* A, int n, int m, double* out4) {
    if (n < 1 || n > 64 || m < 1) return 1;
    uint64_t total = (uint64_t)1 << (n - 1);
    qc* part = (qc*)calloc((size_t)m, sizeof(qc));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < m; k++) {
        uint64_t r, l;
        oracle_distribute(total, (uint64_t)m, (uint64_t)k, &r, &l);   /* [1] */
        if (l) part[k] = subpermanent_rl(A, n, r, l);
    }
    qc S = { 0, 0 };
    for (int k = 0; k < m; k++) S = qc_add(S, part[k]);
    free(part);
    S = qc_scale(S, (n & 1) ? (quad)-2 : (quad)2);                      /* [4] */
    put_qc(out4, S);
    return 0;
}

/* w(r): App. A steps 2, 5-8 evaluated at rank r.  out: n x (re_hi, re_lo, im_hi, im_lo). */
int oracle_seed_c128(const double* A, int n, uint64_t r, double* out) {
    if (n < 1 || n > 64) return 1;
    uint64_t x = oracle_gray(r);
    for (int i = 0; i < n; i++) {
        qc rowsum = { 0, 0 };
        for (int j = 0; j < n; j++) rowsum = qc_add(rowsum, entry(A, n, i, j));
        qc w = qc_sub(entry(A, n, i, n - 1), qc_scale(rowsum, (quad)0.5));
        for (int j = 0; j < n - 1; j++)
            if ((x >> j) & 1) w = qc_add(w, entry(A, n, i, j));
        put_qc(out + 4 * i, w);
    }
    return 0;
}

/* P(k0, k1) = sum_{r=k0}^{k1-1} (-1)^{r+1} prod_i w_i(gray(r)): every term is
 * re-derived from steps 2, 3, 5-8 and 10 of subpermanent (no incremental walk),
 * so it checks the GPU's seeding, stepping and term signs independently. */
int oracle_range_c128(const double* A, int n, uint64_t k0, uint64_t k1, double* out4) {
    if (n < 1 || n > 64 || k1 < k0) return 1;
    qc base[64];
    for (int i = 0; i < n; i++) {
        qc rowsum = { 0, 0 };
        for (int j = 0; j < n; j++) rowsum = qc_add(rowsum, entry(A, n, i, j));
        base[i] = qc_sub(entry(A, n, i, n - 1), qc_scale(rowsum, (quad)0.5));
    }
    int nt = omp_get_max_threads();
    qc* part = (qc*)calloc((size_t)nt, sizeof(qc));
    uint64_t len = k1 - k0;
    #pragma omp parallel num_threads(nt)
    {
        int k = omp_get_thread_num();
        uint64_t a, l;
        oracle_distribute(len, (uint64_t)nt, (uint64_t)k, &a, &l);
        qc S = { 0, 0 };
        for (uint64_t r = k0 + a; r < k0 + a + l; r++) {
            uint64_t x = oracle_gray(r);
            qc p = { 1, 0 };
            for (int i = 0; i < n; i++) {
                qc w = base[i];
                for (int j = 0; j < n - 1; j++)
                    if ((x >> j) & 1) w = qc_add(w, entry(A, n, i, j));
                p = qc_mul(p, w);
            }
            S = (r & 1) ? qc_add(S, p) : qc_sub(S, p);     /* (-1)^{r+1} */
        }
        part[k] = S;
    }
    qc S = { 0, 0 };
    for (int k = 0; k < nt; k++) S = qc_add(S, part[k]);
    free(part);
    put_qc(out4, S);
    return 0;
}

/* ---------------- Eq. (4): weighted Ryser for repeated columns ----------------
 * A has R distinct columns cbar_1..cbar_R, column cbar_k repeated m_k times (sum m_k = n).
 * per(A) = (-1)^n sum_{f in Omega} (-1)^{sum_t f_t} (prod_j C(m_j, f_j)) prod_{i=1}^n sum_{k=1}^R f_k cbar_i(k),
 * Omega = {f : 0 <= f_k <= m_k}.  Written out literally: Omega is enumerated in plain odometer
 * order (digit 0 fastest), every row sum is recomputed from its definition, binomials are exact
 * integers (Pascal's triangle in unsigned __int128), arithmetic is binary128.  The outermost digit's
 * values are split over OpenMP threads; the partial sums are added in digit order.
 * C is n x R row-major (cbar_i(k) = C[i][k]); out4 = value (hi,lo re, hi,lo im); out2 (optional) =
 * sum_f |term_f| as (hi, lo), the scale of the rounding error of any evaluation of the sum. */
static quad binom_q(int m, int f) {
    u128 c = 1;
    for (int t = 1; t <= f; t++) c = c * (u128)(m - f + t) / (u128)t;   /* exact at every step */
    return (quad)c;
}

int oracle_ryser_weighted_c128(const double* C, const int* mult, int n, int R, double* out4, double* out2) {
    if (n < 1 || n > 40 || R < 1 || R > n) return 1;
    int tot = 0;
    for (int k = 0; k < R; k++) {
        if (mult[k] < 0) return 1;
        tot += mult[k];
    }
    if (tot != n) return 1;
    const int top = R - 1;
    const int nt = mult[top] + 1;
    qc* part = (qc*)calloc((size_t)nt, sizeof(qc));
    quad* apart = (quad*)calloc((size_t)nt, sizeof(quad));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int ftop = 0; ftop < nt; ftop++) {
        int f[64];
        for (int k = 0; k < R; k++) f[k] = 0;
        f[top] = ftop;
        qc S = { 0, 0 };
        quad Sa = 0;
        for (;;) {
            quad W = 1;
            int fs = 0;
            for (int k = 0; k < R; k++) { W *= binom_q(mult[k], f[k]); fs += f[k]; }
            qc p = { 1, 0 };
            for (int i = 0; i < n; i++) {
                qc rs = { 0, 0 };
                for (int k = 0; k < R; k++) {
                    qc c = { (quad)C[2 * ((size_t)i * R + k)], (quad)C[2 * ((size_t)i * R + k) + 1] };
                    rs = qc_add(rs, qc_scale(c, (quad)f[k]));
                }
                p = qc_mul(p, rs);
            }
            p = qc_scale(p, W);
            if (fs & 1) S = qc_sub(S, p); else S = qc_add(S, p);
            quad ab = p.re * p.re + p.im * p.im;
            Sa += sqrtq(ab);
            /* odometer over digits 0 .. R-2 */
            int k = 0;
            while (k < top && f[k] == mult[k]) { f[k] = 0; k++; }
            if (k == top) break;
            f[k]++;
        }
        part[ftop] = S;
        apart[ftop] = Sa;
    }
    qc S = { 0, 0 };
    quad Sa = 0;
    for (int t = 0; t < nt; t++) { S = qc_add(S, part[t]); Sa += apart[t]; }
    free(part);
    free(apart);
    if (n & 1) S = qc_scale(S, -1);
    put_qc(out4, S);
    if (out2) put_q(out2, Sa);
    return 0;
}

/* ---------------- App. B: sparse restricted enumeration ----------------
 * greedypartition(A, D), literally: b_ij = [a_ij != 0]; delta_i = out-degree of row i;
 * V = all rows; while V is not empty: k = argmin_{i in V} delta_i (lowest index on ties), S_d = N_k =
 * {l : b_kl = 1}, V -= {k}, V -= {l in V : N_k and N_l intersect}; T = columns in no S.  Returns d and
 * fills masks[0..d-1] = S_1..S_d (column bit masks) and *tmask = T.  n <= 64. */
int oracle_sparse_partition(const double* A, int n, uint64_t* masks, uint64_t* tmask) {
    if (n < 1 || n > 64) return -1;
    uint64_t N[64];
    int deg[64];
    for (int i = 0; i < n; i++) {
        N[i] = 0;
        deg[i] = 0;
        for (int j = 0; j < n; j++) {
            const double re = A[2 * ((size_t)i * n + j)], im = A[2 * ((size_t)i * n + j) + 1];
            if (re != 0.0 || im != 0.0) { N[i] |= (uint64_t)1 << j; deg[i]++; }
        }
    }
    uint64_t V = (n == 64) ? ~(uint64_t)0 : (((uint64_t)1 << n) - 1);
    uint64_t used = 0;
    int d = 0;
    while (V) {
        int k = -1;
        for (int i = 0; i < n; i++)
            if (((V >> i) & 1) && (k < 0 || deg[i] < deg[k])) k = i;
        masks[d++] = N[k];
        used |= N[k];
        V &= ~((uint64_t)1 << k);
        for (int l = 0; l < n; l++)
            if (((V >> l) & 1) && (N[k] & N[l])) V &= ~((uint64_t)1 << l);
    }
    *tmask = ((n == 64) ? ~(uint64_t)0 : (((uint64_t)1 << n) - 1)) & ~used;
    return d;
}

/* sparsepermanent(A, D, p), literally: for every choice of non-empty s_l subset of S_l
 * (l = 1..d) and every t subset of T, J = s_1 u ... u s_d u t and p += (-1)^{|J|} prod_i sum_{j in J} a_ij;
 * p *= (-1)^n.  Row sums from the definition for every J, binary128.  The outermost enumeration (the
 * subsets of T, in index order) is split over OpenMP threads and summed in index order.
 * out2 = number of sets J enumerated (as a double pair hi, lo). */
int oracle_sparse_c128(const double* A, int n, double* out4, double* out_count) {
    if (n < 1 || n > 40) return 1;
    uint64_t S[64], T;
    const int d = oracle_sparse_partition(A, n, S, &T);
    for (int i = 0; i < n; i++) {                    /* a zero row makes every product zero */
        int nz = 0;
        for (int j = 0; j < n; j++) nz |= A[2 * ((size_t)i * n + j)] != 0.0 || A[2 * ((size_t)i * n + j) + 1] != 0.0;
        if (!nz) { qc z = { 0, 0 }; put_qc(out4, z); if (out_count) put_q(out_count, 0); return 0; }
    }
    int tcols[64], nt = 0;
    for (int j = 0; j < n; j++) if ((T >> j) & 1) tcols[nt++] = j;
    const uint64_t ntsub = (uint64_t)1 << nt;
    const int parts = 256;
    qc* part = (qc*)calloc(parts, sizeof(qc));
    quad* cnt = (quad*)calloc(parts, sizeof(quad));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int pi = 0; pi < parts; pi++) {
        uint64_t t0, tl;
        oracle_distribute(ntsub, parts, (uint64_t)pi, &t0, &tl);
        qc acc = { 0, 0 };
        quad c = 0;
        for (uint64_t tb = t0; tb < t0 + tl; tb++) {
            uint64_t tsel = 0;
            for (int q = 0; q < nt; q++) if ((tb >> q) & 1) tsel |= (uint64_t)1 << tcols[q];
            /* odometer over the non-empty subsets s_l of S_l: s_l runs through the sub-masks of S_l */
            uint64_t s[64];
            for (int l = 0; l < d; l++) s[l] = S[l] & (~S[l] + 1);   /* lowest non-empty sub-mask */
            if (d == 0) s[0] = 0;
            for (;;) {
                uint64_t J = tsel;
                for (int l = 0; l < d; l++) J |= s[l];
                qc p = { 1, 0 };
                for (int i = 0; i < n; i++) {
                    qc rs = { 0, 0 };
                    for (int j = 0; j < n; j++) if ((J >> j) & 1) rs = qc_add(rs, entry(A, n, i, j));
                    p = qc_mul(p, rs);
                }
                if (__builtin_popcountll(J) & 1) acc = qc_sub(acc, p); else acc = qc_add(acc, p);
                c += 1;
                int l = 0;                         /* next combination: sub-mask successor, carry */
                for (; l < d; l++) {
                    s[l] = (s[l] - S[l]) & S[l];   /* next sub-mask of S[l] in increasing order */
                    if (s[l] != 0) break;
                    s[l] = S[l] & (~S[l] + 1);
                }
                if (l == d) break;
            }
        }
        part[pi] = acc;
        cnt[pi] = c;
    }
    qc P = { 0, 0 };
    quad C = 0;
    for (int pi = 0; pi < parts; pi++) { P = qc_add(P, part[pi]); C += cnt[pi]; }
    free(part);
    free(cnt);
    if (n & 1) P = qc_scale(P, -1);
    put_qc(out4, P);
    if (out_count) put_q(out_count, C);
    return 0;
}

/* ---------------- App. C: matrices of limited bandwidth ----------------
 * bandpermanent(A, k, p) literally: C_i = sum_j a_ij x_j (the band |i-j| <= k of row i); p := 1; for
 * i = 1..n: p := p * C_i, then in p set x_{i-k-1} = 1 and x_j^2 = 0; finally set every x_i = 1.
 * p is stored as dense binary128 coefficients over the monomials of its live variables: after row i
 * (1-based) only x_{i-k} .. x_{i+k} can be live, so before multiplying by C_i the live window is
 * x_{i-k-1} .. x_{i+k-1} (2k+1 bits) and after it x_{i-k-1} .. x_{i+k} (2k+2 bits); "set x_{i-k-1} = 1"
 * merges each monomial with and without that variable (a shift of the window).  x_j^2 = 0 discards any
 * product that would repeat a live variable.  A is n x n row-major; entries outside the band are not
 * read.  k <= 10. */
int oracle_band_c128(const double* A, int n, int k, double* out4) {
    if (n < 1 || k < 0) return 1;
    if (k > n - 1) k = n - 1;
    if (k > 10) return 1;
    const int W = 2 * k + 1;                             /* live window before a row */
    const size_t SW = (size_t)1 << W, SQ = (size_t)1 << (W + 1);
    qc* p = (qc*)calloc(SW, sizeof(qc));
    qc* q = (qc*)calloc(SQ, sizeof(qc));
    p[0].re = 1;                                         /* p := 1 */
    for (int i = 0; i < n; i++) {                        /* 0-based row i; window base b = i - k - 1 */
        const int b = i - k - 1;
        for (size_t m = 0; m < SQ; m++) { q[m].re = 0; q[m].im = 0; }
        for (size_t m = 0; m < SW; m++) {
            if (p[m].re == 0 && p[m].im == 0) continue;
            for (int j = i - k; j <= i + k; j++) {       /* p * C_i */
                if (j < 0 || j >= n) continue;
                const int bit = j - b;                   /* 1 .. 2k+1 */
                if ((m >> bit) & 1) continue;            /* x_j^2 = 0 */
                q[m | ((size_t)1 << bit)] = qc_add(q[m | ((size_t)1 << bit)], qc_mul(p[m], entry(A, n, i, j)));
            }
        }
        for (size_t m = 0; m < SW; m++) { p[m].re = 0; p[m].im = 0; }
        for (size_t m = 0; m < SQ; m++)                  /* set x_{b} = 1: drop bit 0, shift the window */
            p[m >> 1] = qc_add(p[m >> 1], q[m]);
    }
    qc S = { 0, 0 };
    for (size_t m = 0; m < SW; m++) S = qc_add(S, p[m]); /* set every x = 1 */
    free(p);
    free(q);
    put_qc(out4, S);
    return 0;
}

int oracle_num_threads(void) { return omp_get_max_threads(); }
