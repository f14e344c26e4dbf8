// weighted.cu -- weighted Ryser formula for matrices with repeated columns (
// PAPER.md Eq. (4)), batched: Boson-sampling amplitudes of output patterns WITH collisions.
//
// A problem is an n x R matrix C of distinct columns cbar_k with multiplicities m_k (sum m_k = n); it
// stands for the n x n matrix in which cbar_k appears m_k times.  Eq. (4):
//     per(A) = (-1)^n sum_{f in Omega} (-1)^{|f|} (prod_k C(m_k, f_k)) prod_i sum_k f_k cbar_i(k),
//     Omega = { 0 <= f_k <= m_k },  |Omega| = prod_k (m_k + 1)  (<= 2^n).
// Omega is walked in reflected mixed-radix Gray order, so consecutive vectors f differ in one digit by
// +-1 and the row sums w_i = sum_k f_k cbar_i(k) change by +-cbar_k: the same update / product /
// signed-sum step as the Gray walk of walk.cuh, with the weight prod_k C(m_k, f_k) as an extra real
// factor (an exact integer < 2^n, exact in binary64 for n <= 32).
//
// Mapping: one warp per problem, persistent (each warp takes the next problem from an atomic counter).  The
// two digits with the largest multiplicities, s and s2, are the fastest digits: a "tile" walks their
// (m_s + 1)(m_s2 + 1) values at fixed outer digits -- f_s sweeps 0..m_s or back, f_s2 steps by one, f_s
// sweeps back, ... -- while the other digits, numbered in input order, follow the reflected Gray code of
// the tile index q.  Lane l takes the contiguous tiles [distribute(NT, 32, l)) (App. A distribute,
// P:1086-1093) and seeds its row sums, digits and weight explicitly from q (the "chunk seeding" of the
// walk), so all lanes step f_s and f_s2 in lock-step and read the same column (+-cbar_s, +-cbar_s2: all
// four are staged in shared memory, the address picks the sign).  Between tiles each lane changes one
// outer digit (lane-dependent column, fma with the direction) and its binomial weight.  Tiles amortise
// that per-tile work (successor search, exact weight update, double-double fold) over ~4x more terms
// than one-digit sweeps.
// Each lane sums its terms in double per tile and folds them into a double-double; the 32 lane
// partials are combined by a fixed shuffle tree; lane 0 applies (-1)^n and writes per and |per|^2.
#include "walk.cuh"

namespace perm {

// largest-first work order (wgt_order_kernel); 0: input order
#ifndef PERM_WGT_ORDERED
#define PERM_WGT_ORDERED 1
#endif
constexpr bool kWgtOrdered = PERM_WGT_ORDERED != 0;

// unit sweep column (normalised rows); 0: every problem walked as given
#ifndef PERM_WGT_UNIT
#define PERM_WGT_UNIT 1
#endif
constexpr bool kWgtUnit = PERM_WGT_UNIT != 0;

// unroll factor of the sweep loop (1: rolled)
#ifndef PERM_WGT_UNROLL
#define PERM_WGT_UNROLL 1
#endif
constexpr int kWgtUnroll = PERM_WGT_UNROLL;
// independent product chains per term (walk.cuh two_factors)
#ifndef PERM_WGT_K4_MIN
#define PERM_WGT_K4_MIN 99
#endif
template <int N>
constexpr int kWgtChains = N >= PERM_WGT_K4_MIN ? 4 : (N >= 4 ? 2 : 1);

template <int N>
struct WgtCfg {
    static constexpr int NT = 32;                    // one warp (one problem at a time) per block
#ifndef PERM_WGT_REG_EXTRA
    // working-set registers beyond the 4n row sums (0 spill bytes at every order, tools/spills.py, with the
    // unrolled sweeps of m_s <= kWgtSpecMax)
    static constexpr int EXTRA = ((N >= 14 && N <= 18) || N == 21 || N == 23 || N == 24) ? 160 : 128;
#else
    static constexpr int EXTRA = PERM_WGT_REG_EXTRA;
#endif
    static constexpr int REGS = ((4 * N + EXTRA + 7) / 8) * 8;
    static constexpr int MINB_RAW = 65536 / (NT * (REGS < 255 ? REGS : 255));
    static constexpr int MINB = MINB_RAW > 32 ? 32 : (MINB_RAW < 1 ? 1 : MINB_RAW);
};

// C(m, f) for 0 <= f <= m <= kMaxBatchedN, exact in double (< 2^53).
__device__ __forceinline__ double binom_d(int m, int f) {
    double c = 1.0;
    for (int t = 1; t <= f; t++) c = c * (double)(m - f + t) / (double)t;   // exact: integer at every step
    return c;
}

// Shared-memory slot (bytes) of one warp for R distinct columns of order N.
__host__ __device__ constexpr size_t wgt_slot_bytes(int N, int R) {
    // cbar (R N double2) and -cbar of the two sweep digits (2 N double2), binomial row of each digit
    // (R (N+1) doubles), the two sweep tables (2 (N+1) doubles), radices / multiplicities / digit order
    // (3 R ints), the lanes' outer digits and directions (2 R x 32 bytes)
    return ((size_t)(R + 2) * N * 16 + (size_t)(R + 2) * (N + 1) * 8 + (size_t)3 * R * 4 + (size_t)2 * R * 32 + 15) &
           ~(size_t)15;
}

// One sweep of the fastest digit f_s over its m_s + 1 values (terms j = 0..m_s): weight, product, signed sum,
// then the step to the next value (+-cbar_s by address).  MS >= 0: m_s known at compile time (unrolled).
#ifndef PERM_WGT_SPECIALISE
#define PERM_WGT_SPECIALISE 1
#endif
constexpr bool kWgtSpecialise = PERM_WGT_SPECIALISE != 0;
#ifndef PERM_WGT_SPEC_MAX
#define PERM_WGT_SPEC_MAX 2
#endif
constexpr int kWgtSpecMax = PERM_WGT_SPEC_MAX;   // largest m_s with an unrolled sweep
// UNIT: the sweep column was normalised to 1 (its flips change the real parts only: n DADD instead of 2n)
template <int N, int MS, bool UNIT>
__device__ __forceinline__ void wgt_sweep(int ms, double sc2, const double* tsw, int& f1, int d1, uint32_t step,
                                          double (&wr)[N], double (&wi)[N], double& ar, double& ai) {
    const int m = MS >= 0 ? MS : ms;
#pragma unroll (MS >= 0 ? MS + 1 : kWgtUnroll)
    for (int j = 0; j <= m; j++) {
        const double wt = sc2 * tsw[f1];
        double xr, xi, yr, yi;
        two_factors<N, kWgtChains<N>>(wr, wi, xr, xi, yr, yi);
        if constexpr (N == 1) { yr = 1.0; yi = 0.0; }
        xr *= wt;
        xi *= wt;
        fused_acc<+1>(xr, xi, yr, yi, ar, ai);
        if (j < m) {
            if constexpr (UNIT) {
                const double dz = (double)d1;
#pragma unroll
                for (int i = 0; i < N; i++) wr[i] += dz;
            } else {
                flip_add<N>(step, wr, wi);
            }
            f1 += d1;
        }
    }
}

// Work order of the persistent queue: problems largest first (longest-processing-time rule), so that the big
// patterns start early instead of running alone at the end (problem sizes prod_k (m_k + 1) vary ~10x; ncu of the
// input-order queue: SMs active 82% of the launch).  One block counting-sorts the problems by floor(8 log2 |Omega|)
// (eighth-octave classes) into `order` (descending class, index order inside a class) -- scheduling only: every
// problem's result is computed by one warp from its own data, so the outputs do not depend on it.
constexpr int kWgtBuckets = 256;                  // eighth-octave size classes, 2^0 .. 2^32
__global__ void __launch_bounds__(1024) wgt_order_kernel(const int32_t* __restrict__ mult, int R, int64_t B,
                                                         int64_t* __restrict__ order) {
    // stable counting sort by one block: warp w owns the contiguous problems [w B / 32, (w + 1) B / 32); per-warp
    // class counts, an exclusive scan over (class, warp), then every warp places its problems in index order
    __shared__ uint32_t cnt[32][kWgtBuckets];                // per-warp counts, then per-warp cursors
    __shared__ unsigned long long tot[kWgtBuckets];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    auto bucket = [&](int64_t b) {
        double sz = 1.0;
        for (int k = 0; k < R; k++) {
            const int m = mult[b * R + k];
            sz *= (double)((m > 0 ? m : 0) + 1);
        }
        int e = (int)(8.0 * log2(sz));                   // floor(8 log2 |Omega|)
        e = e < 0 ? 0 : (e >= kWgtBuckets ? kWgtBuckets - 1 : e);
        return kWgtBuckets - 1 - e;                       // largest first
    };
    for (int k = threadIdx.x; k < 32 * kWgtBuckets; k += blockDim.x) (&cnt[0][0])[k] = 0;
    __syncthreads();
    const int64_t b0 = B * w / 32, b1 = B * (w + 1) / 32;
    for (int64_t b = b0 + lane; b < b1; b += 32) atomicAdd(&cnt[w][bucket(b)], 1u);
    __syncthreads();
    for (int k = threadIdx.x; k < kWgtBuckets; k += blockDim.x) {
        unsigned long long t = 0;
        for (int v = 0; v < 32; v++) t += cnt[v][k];
        tot[k] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int k = 0; k < kWgtBuckets; k++) { const unsigned long long c = tot[k]; tot[k] = run; run += c; }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kWgtBuckets; k += blockDim.x) {
        unsigned long long run = tot[k];
        for (int v = 0; v < 32; v++) { const uint32_t c = cnt[v][k]; cnt[v][k] = (uint32_t)run; run += c; }
    }
    __syncthreads();
    // (32-bit cursors: the launch sorts fewer than 2^31 problems; larger batches keep the input order)
    for (int64_t c0 = b0; c0 < b1; c0 += 32) {
        const int64_t b = c0 + lane;
        const int key = b < b1 ? bucket(b) : -1 - lane;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int before = __popc(peers & ((1u << lane) - 1u));
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (b < b1 && lane == leader) base = cnt[w][key];
        base = __shfl_sync(0xffffffffu, base, leader);
        if (b < b1) order[base + before] = b;
        __syncwarp();
        if (b < b1 && lane == leader) cnt[w][key] = base + (uint32_t)__popc(peers);
        __syncwarp();
    }
}

__global__ void wgt_identity_order_kernel(int64_t B, int64_t* __restrict__ order) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) order[b] = b;
}

template <int N>
__global__ void __launch_bounds__(WgtCfg<N>::NT, WgtCfg<N>::MINB)
    weighted_kernel(const double2* __restrict__ C, const int32_t* __restrict__ mult, int R, int64_t B,
                    double2* __restrict__ per, double* __restrict__ abs2, unsigned long long* __restrict__ next) {
    extern __shared__ __align__(16) unsigned char wsm[];
    const int lane = threadIdx.x & 31;
    double2* col = (double2*)wsm;                                         // col[k*N + i] = cbar_i(k)
    double2* negs = col + (size_t)R * N;                                  // -cbar_s (fast sweep digit)
    double2* negs2 = negs + N;                                            // -cbar_s2 (second sweep digit)
    double* bin = (double*)(wsm + (size_t)(R + 2) * N * 16);              // bin[k*(N+1) + f] = C(m_k, f)
    double* tsw = bin + (size_t)R * (N + 1);                              // tsw[j] = (-1)^j C(m_s, j)
    double* tsw2 = tsw + (N + 1);                                         // tsw2[j] = (-1)^j C(m_s2, j)
    int* order = (int*)(tsw2 + (N + 1));                                  // order[0] = s, then the outer digits
    int* rad = order + R;                                                 // rad[p] = m_{order[p]} + 1
    int* mlt = rad + R;                                                   // mlt[p] = m_{order[p]}
    unsigned char* gdig = (unsigned char*)(mlt + R);                      // gdig[p*32 + lane]: outer digit p
    signed char* gdir = (signed char*)(gdig + R * 32);                    // its direction (+-1)
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(col);
    const uint32_t nbase = (uint32_t)__cvta_generic_to_shared(negs);
    const uint32_t nbase2 = (uint32_t)__cvta_generic_to_shared(negs2);

    for (;;) {                                                            // persistent: a shared work queue
        __syncwarp();
        unsigned long long bq = 0;
        if (lane == 0) {
            bq = atomicAdd(next, 1ull);
            // the queue position's problem: the largest-first order follows the counter (wgt_order_kernel)
            if (kWgtOrdered && bq < (unsigned long long)B) bq = (unsigned long long)((const int64_t*)(next + 2))[bq];
        }
        const int64_t b = (int64_t)__shfl_sync(0xffffffffu, bq, 0);
        if (b >= B) break;
        const int32_t* mb = mult + b * (int64_t)R;
        int msum = 0, mbad = 0, s = 0, ms = -1;
        for (int k = 0; k < R; k++) {                                     // warp-uniform scan
            const int m = mb[k];
            msum += m;
            mbad |= (m < 0) | (m > N);
            if (m > ms) { ms = m; s = k; }
        }
        // the second sweep digit: the largest other multiplicity >= 1 (none: m_s2 = 0, a one-row tile)
        int s2 = -1, ms2 = 0;
        for (int k = 0; k < R; k++)
            if (k != s && mb[k] > ms2) { ms2 = mb[k]; s2 = k; }
        // stage the columns, column-major, and the negated sweep column
        const double2* src = C + b * (int64_t)N * R;
        for (int k = lane; k < N * R; k += 32) {
            const int i = k / R, j = k - i * R;
            const double2 a = src[k];
            col[j * N + i] = a;
            if (j == s) negs[i] = make_double2(-a.x, -a.y);
            if (j == s2) negs2[i] = make_double2(-a.x, -a.y);
        }
        if (msum != N || mbad) {                                          // not a valid multiplicity vector
            if (lane == 0) {
                const double nan = __longlong_as_double(0x7ff8000000000000ll);
                if (per) per[b] = make_double2(nan, nan);
                if (abs2) abs2[b] = nan;
            }
            continue;
        }
        // unit sweep column: rows divided by their entry in the sweep column s (per(A) is multilinear in
        // the rows; scale = prod_i c_is in double-double, a fixed shuffle tree), so the fast flips change real parts
        // only; a problem with a zero (or relatively tiny) entry in column s is walked as given
        bool unit = false;
        __shared__ ddc s_uscale;
        if constexpr (kWgtUnit) {
            __syncwarp();
            ddc f;
            f.re = dd{1.0, 0.0};
            f.im = dd{0.0, 0.0};
            bool okl = true;
            if (lane < N) {
                const double2 a = col[s * N + lane];
                const double m = fmax(fabs(a.x), fabs(a.y));
                double rmax = 0.0;
                for (int k = 0; k < R; k++) rmax = fmax(rmax, fabs(col[k * N + lane].x) + fabs(col[k * N + lane].y));
                okl = m > 0.0 && rmax / m <= 1e100;
                f.re = dd{a.x, 0.0};
                f.im = dd{a.y, 0.0};
            }
            unit = __all_sync(0xffffffffu, okl);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) f = ddc_mul(f, shfl_down_ddc(f, off));
            if (lane == 0) s_uscale = f;
            if (unit) {
                for (int k = lane; k < N * R; k += 32) {                  // col[k] = a_{i, j}, k = j N + i
                    const int j = k / N, i = k - j * N;
                    if (j == s) continue;
                    const double2 a0 = col[s * N + i];
                    const double m = fmax(fabs(a0.x), fabs(a0.y));
                    const double sr = a0.x / m, si = a0.y / m, d2 = sr * sr + si * si;
                    const double ir = sr / (d2 * m), ii = -si / (d2 * m);
                    const double2 a = col[k];
                    col[k] = make_double2(a.x * ir - a.y * ii, a.x * ii + a.y * ir);
                }
                __syncwarp();
                for (int i = lane; i < N; i += 32) {
                    col[s * N + i] = make_double2(1.0, 0.0);
                    negs[i] = make_double2(-1.0, 0.0);
                    if (s2 >= 0) negs2[i] = make_double2(-col[s2 * N + i].x, -col[s2 * N + i].y);
                }
            }
            __syncwarp();
        }
        for (int k = lane; k < R * (N + 1); k += 32) {
            const int d = k / (N + 1), f = k - d * (N + 1);
            const int m = mb[d];
            bin[k] = (f <= m) ? binom_d(m, f) : 0.0;
        }
        for (int j = lane; j <= ms; j += 32) tsw[j] = (j & 1) ? -binom_d(ms, j) : binom_d(ms, j);
        for (int j = lane; j <= ms2; j += 32) tsw2[j] = (j & 1) ? -binom_d(ms2, j) : binom_d(ms2, j);
        int P = 0;                                                        // outer digits with m_k > 0
        if (lane == 0) {
            order[0] = s;
            rad[0] = ms + 1;
            mlt[0] = ms;
            for (int k = 0; k < R; k++)
                if (k != s && k != s2 && mb[k] > 0) { order[1 + P] = k; rad[1 + P] = mb[k] + 1; mlt[1 + P] = mb[k]; P++; }
        }
        __syncwarp();
        P = __shfl_sync(0xffffffffu, P, 0);

        // tiles: NS = prod of the outer radices (<= 2^31 for N <= 32); lane l takes [q0, q0 + nq).  A tile is
        // the (m_s + 1)(m_s2 + 1) terms of the two sweep digits at fixed outer digits, walked as the two
        // fastest digits of the reflected mixed-radix Gray code: f_s sweeps, f_s2 steps, f_s reverses ...
        uint32_t NS = 1;
        for (int p = 1; p <= P; p++) NS *= (uint32_t)rad[p];
        const uint32_t qb = NS / 32u, qr = NS % 32u;
        const uint32_t q0 = (uint32_t)lane * qb + ((uint32_t)lane < qr ? (uint32_t)lane : qr);
        const uint32_t nq = qb + ((uint32_t)lane < qr ? 1u : 0u);
        const uint32_t cs = base + (uint32_t)(s * N) * 16u;               // +cbar_s
        const uint32_t cs2 = base + (uint32_t)((s2 < 0 ? s : s2) * N) * 16u;   // +cbar_s2 (unused if none)

        ddc acc;
        acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
        if (nq > 0) {
            // seed at tile q0: f_s has completed q0 (m_s2 + 1) sweeps and f_s2 q0 sweeps (each runs forward
            // iff that count is even); outer digit p has ordinary value t_p and runs forward iff the number
            // formed by the digits above it is even; its Gray value is t_p forward, r_p - 1 - t_p backward
            double wr[N], wi[N];
            bool fwd1 = ((q0 * (uint32_t)(ms2 + 1)) & 1u) == 0;
            bool fwd2 = (q0 & 1u) == 0;
            int f1 = fwd1 ? 0 : ms, f2 = fwd2 ? 0 : ms2;
            int fsum = 0;
            double wout = 1.0;
#pragma unroll
            for (int i = 0; i < N; i++) { wr[i] = 0.0; wi[i] = 0.0; }
            flip_dyn<N>(cs, (double)f1, wr, wi);
            flip_dyn<N>(cs2, (double)f2, wr, wi);
            {
                uint32_t x = q0;
                for (int p = 1; p <= P; p++) {
                    const uint32_t r = (uint32_t)rad[p];
                    const uint32_t t = x % r, up = x / r;
                    const bool fwd = (up & 1u) == 0;
                    const int g = (int)(fwd ? t : r - 1 - t);
                    gdig[(p - 1) * 32 + lane] = (unsigned char)g;
                    gdir[(p - 1) * 32 + lane] = fwd ? 1 : -1;
                    fsum += g;
                    wout *= bin[order[p] * (N + 1) + g];
                    flip_dyn<N>(base + (uint32_t)(order[p] * N) * 16u, (double)g, wr, wi);
                    x = up;
                }
            }
            // outer factor (-1)^{sum of outer digits} prod C(m_p, g_p); each term multiplies in
            // tsw2[f2] tsw[f1] = (-1)^{f1 + f2} C(m_s, f1) C(m_s2, f2)   (all exact integers < 2^n)
            double scale = (fsum & 1) ? -wout : wout;
            for (uint32_t q = q0;; q++) {
                double ar = 0.0, ai = 0.0;
                for (int r = 0; r <= ms2; r++) {
                    const double sc2 = scale * tsw2[f2];
                    const uint32_t step = fwd1 ? cs : nbase;
                    const int d1 = fwd1 ? 1 : -1;
                    // the fast sweep, unrolled for the common small multiplicities (warp-uniform switch)
                    const int sw = (kWgtSpecialise && N <= 24 && ms <= kWgtSpecMax ? ms : -1) + (unit ? 16 : 0);
                    switch (sw) {
                        case 1: wgt_sweep<N, 1, false>(ms, sc2, tsw, f1, d1, step, wr, wi, ar, ai); break;
                        case 2: wgt_sweep<N, 2, false>(ms, sc2, tsw, f1, d1, step, wr, wi, ar, ai); break;
                        case 17: wgt_sweep<N, 1, true>(ms, sc2, tsw, f1, d1, step, wr, wi, ar, ai); break;
                        case 18: wgt_sweep<N, 2, true>(ms, sc2, tsw, f1, d1, step, wr, wi, ar, ai); break;
                        case 15: wgt_sweep<N, -1, true>(ms, sc2, tsw, f1, d1, step, wr, wi, ar, ai); break;
                        default: wgt_sweep<N, -1, false>(ms, sc2, tsw, f1, d1, step, wr, wi, ar, ai); break;
                    }
                    fwd1 = !fwd1;
                    if (r < ms2) {
                        flip_add<N>(fwd2 ? cs2 : nbase2, wr, wi);
                        f2 += fwd2 ? 1 : -1;
                    }
                }
                fwd2 = !fwd2;
                acc.re = dd_add_d(acc.re, ar);
                acc.im = dd_add_d(acc.im, ai);
                if (q + 1 >= q0 + nq) break;
                // next tile: the lowest outer digit that can move in its direction moves; the digits
                // below it (at an end) reverse direction -- the reflected Gray successor of q
                int p = 1;
                int g = 0, d = 0;
                for (;; p++) {
                    g = gdig[(p - 1) * 32 + lane];
                    d = gdir[(p - 1) * 32 + lane];
                    const int ng = g + d;
                    if (ng >= 0 && ng <= mlt[p]) break;
                    gdir[(p - 1) * 32 + lane] = (signed char)(-d);
                }
                gdig[(p - 1) * 32 + lane] = (unsigned char)(g + d);
                const double* bk = bin + order[p] * (N + 1);
                wout = __dmul_rn(__ddiv_rn(wout, bk[g]), bk[g + d]);      // exact: integer quotient
                flip_dyn<N>(base + (uint32_t)(order[p] * N) * 16u, (double)d, wr, wi);   // once per tile
                scale = scale < 0.0 ? wout : -wout;                       // one outer digit moved by +-1
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
        if (lane == 0) {
            if (unit) acc = ddc_mul(acc, s_uscale);                       // back to the units of the problem
            const double f = (N & 1) ? -1.0 : 1.0;
            const double re = (acc.re.hi + acc.re.lo) * f;
            const double im = (acc.im.hi + acc.im.lo) * f;
            if (per) per[b] = make_double2(re, im);
            if (abs2) abs2[b] = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
        }
    }
}

template <int N>
cudaError_t weighted_launch_t(const double2* C, const int32_t* mult, int R, int64_t B, double2* per, double* abs2,
                              cudaStream_t st, int* launches) {
    const size_t smem = wgt_slot_bytes(N, R);
    cudaError_t err = cudaFuncSetAttribute(weighted_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, bps = 0;
    err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, weighted_kernel<N>, WgtCfg<N>::NT, smem);
    if (err != cudaSuccess) return err;
    if (bps < 1) return cudaErrorInvalidConfiguration;       // R too large for shared memory
    const int64_t cap = (int64_t)sms * bps;
    const int64_t grid = B < cap ? B : cap;
    // the work-queue counter and (more than one resident wave of problems) the largest-first order, stream-ordered
    const bool ordered = kWgtOrdered;
    unsigned long long* next = nullptr;
    err = malloc_async((void**)&next, 16 + (ordered ? (size_t)B * sizeof(int64_t) : 0), st);
    if (err != cudaSuccess) return err;
    int64_t* order = (int64_t*)((char*)next + 16);
    err = cudaMemsetAsync(next, 0, sizeof(unsigned long long), st);
    if (err == cudaSuccess && ordered) {
        if (B < (1ll << 31)) wgt_order_kernel<<<1, 1024, 0, st>>>(mult, R, B, order);
        else                 wgt_identity_order_kernel<<<1024, 256, 0, st>>>(B, order);   // (32-bit cursors)
        err = cudaGetLastError();
    }
    if (err == cudaSuccess) {
        weighted_kernel<N><<<(unsigned)grid, WgtCfg<N>::NT, smem, st>>>(C, mult, R, B, per, abs2, next);
        err = cudaGetLastError();
    }
    *launches = ordered ? 2 : 1;
    const cudaError_t e2 = cudaFreeAsync(next, st);
    return err != cudaSuccess ? err : e2;
}

#define PERM_R8(M, b) M(b + 1) M(b + 2) M(b + 3) M(b + 4) M(b + 5) M(b + 6) M(b + 7) M(b + 8)

cudaError_t weighted_launch(const double2* C, const int32_t* mult, int n, int R, int64_t B, double2* per,
                            double* abs2, cudaStream_t s, int* launches) {
    *launches = 0;
    if (B == 0) return cudaSuccess;
#define PERM_CASE(N) case N: return weighted_launch_t<N>(C, mult, R, B, per, abs2, s, launches);
    switch (n) { PERM_R8(PERM_CASE, 0) PERM_R8(PERM_CASE, 8) PERM_R8(PERM_CASE, 16) PERM_R8(PERM_CASE, 24)
                 default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

}  // namespace perm
