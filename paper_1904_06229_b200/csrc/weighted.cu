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
// Mapping: one warp per problem.  The digit with the largest multiplicity, s, is the fastest digit:
// every "sweep" runs f_s through 0..m_s (even sweeps) or m_s..0 (odd sweeps) while the other digits,
// numbered in input order, follow the reflected Gray code of the sweep index q.  Lane l takes the
// contiguous sweeps [distribute(NS, 32, l)) (App. A distribute) and seeds its row sums,
// digits and weight explicitly from q (the "chunk seeding" of the walk), so all lanes step f_s in
// lock-step and read the same column (+cbar_s or -cbar_s: both are staged in shared memory, the
// address picks the sign).  Between sweeps each lane changes one outer digit (lane-dependent column).
// Each lane sums its terms in double per sweep and folds them into a double-double; the 32 lane
// partials are combined by a fixed shuffle tree; lane 0 applies (-1)^n and writes per and |per|^2.
#include "walk.cuh"

namespace perm {

struct WgtCfg {
    static constexpr int WARPS = 2;                  // warps (problems) per block
    static constexpr int NT = 32 * WARPS;
};

// C(m, f) for 0 <= f <= m <= kMaxBatchedN, exact in double (< 2^53).
__device__ __forceinline__ double binom_d(int m, int f) {
    double c = 1.0;
    for (int t = 1; t <= f; t++) c = c * (double)(m - f + t) / (double)t;   // exact: integer at every step
    return c;
}

// Per-warp shared-memory slot (bytes) for R distinct columns of order N.
__host__ __device__ constexpr size_t wgt_slot_bytes(int N, int R) {
    // +cbar and -cbar (2 R N double2), binomial row of each digit (R (N+1) doubles), radices / digit
    // order (2 R ints), the lanes' outer digits (R x 32 bytes)
    return ((size_t)2 * R * N * 16 + (size_t)R * (N + 1) * 8 + (size_t)2 * R * 4 + (size_t)R * 32 + 15) & ~(size_t)15;
}

template <int N>
__global__ void __launch_bounds__(WgtCfg::NT) weighted_kernel(const double2* __restrict__ C,
                                                              const int32_t* __restrict__ mult, int R,
                                                              int64_t B, double2* __restrict__ per,
                                                              double* __restrict__ abs2) {
    extern __shared__ __align__(16) unsigned char wsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * WgtCfg::WARPS + warp;
    if (b >= B) return;                                                   // warp-uniform
    unsigned char* slot = wsm + (size_t)warp * wgt_slot_bytes(N, R);
    double2* col = (double2*)slot;                                        // col[k*N + i] = cbar_i(k)
    double* bin = (double*)(slot + (size_t)2 * R * N * 16);               // bin[k*(N+1) + f] = C(m_k, f)
    int* order = (int*)(bin + (size_t)R * (N + 1));                       // order[0] = s, then the outer digits
    int* rad = order + R;                                                 // rad[p] = m_{order[p]} + 1
    unsigned char* gdig = (unsigned char*)(rad + R);                      // gdig[p*32 + lane]: outer digit p

    // stage the columns (and their negations) and the multiplicities
    const double2* src = C + b * (int64_t)N * R;
    for (int k = lane; k < N * R; k += 32) {
        const int i = k / R, j = k - i * R;
        const double2 a = src[k];
        col[j * N + i] = a;
        col[R * N + j * N + i] = make_double2(-a.x, -a.y);
    }
    const int32_t* mb = mult + b * (int64_t)R;
    int msum = 0, mbad = 0, s = 0, ms = -1;
    for (int k = 0; k < R; k++) {                                         // warp-uniform scan
        const int m = mb[k];
        msum += m;
        mbad |= (m < 0) | (m > N);
        if (m > ms) { ms = m; s = k; }
    }
    if (msum != N || mbad) {                                              // not a valid multiplicity vector
        if (lane == 0) {
            const double nan = __longlong_as_double(0x7ff8000000000000ll);
            if (per) per[b] = make_double2(nan, nan);
            if (abs2) abs2[b] = nan;
        }
        return;
    }
    for (int k = lane; k < R * (N + 1); k += 32) {
        const int d = k / (N + 1), f = k - d * (N + 1);
        const int m = mb[d];
        bin[k] = (f <= m) ? binom_d(m, f) : 0.0;
    }
    int P = 0;                                                            // outer digits with m_k > 0
    if (lane == 0) {
        order[0] = s;
        rad[0] = ms + 1;
        for (int k = 0; k < R; k++)
            if (k != s && mb[k] > 0) { order[1 + P] = k; rad[1 + P] = mb[k] + 1; P++; }
    }
    __syncwarp();
    P = __shfl_sync(0xffffffffu, P, 0);

    // sweeps: NS = prod of the outer radices; lane l takes [q0, q0 + nq)
    uint64_t NS = 1;
    for (int p = 1; p <= P; p++) NS *= (uint64_t)rad[p];
    const uint64_t qb = NS / 32, qr = NS % 32;
    const uint64_t q0 = (uint64_t)lane * qb + ((uint64_t)lane < qr ? (uint64_t)lane : qr);
    const uint64_t nq = qb + ((uint64_t)lane < qr ? 1ull : 0ull);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(col);
    const uint32_t NEG = (uint32_t)(R * N) * 16u;
    const uint32_t cs = base + (uint32_t)(s * N) * 16u;                  // +cbar_s

    double wr[N], wi[N];
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    if (nq > 0) {
        // seed at sweep q0: outer Gray digits of q0 (reflected mixed radix: digit p runs backwards when
        // the number formed by the digits above it is odd), f_s = 0 (q0 even) or m_s (q0 odd)
        int fsum = (q0 & 1ull) ? ms : 0;
        {
            uint64_t x = q0;
            for (int p = 1; p <= P; p++) {
                const uint64_t r = (uint64_t)rad[p];
                const uint64_t t = x % r, up = x / r;
                const int g = (int)((up & 1ull) ? r - 1 - t : t);
                gdig[(p - 1) * 32 + lane] = (unsigned char)g;
                fsum += g;
                x = up;
            }
        }
#pragma unroll
        for (int i = 0; i < N; i++) { wr[i] = 0.0; wi[i] = 0.0; }
        const double fs0 = (q0 & 1ull) ? (double)ms : 0.0;
        flip_dyn<N>(cs, fs0, wr, wi);
        for (int p = 1; p <= P; p++)
            flip_dyn<N>(base + (uint32_t)(order[p] * N) * 16u, (double)gdig[(p - 1) * 32 + lane], wr, wi);
        double sgn = (fsum & 1) ? -1.0 : 1.0;                             // (-1)^{|f|}
        const double* bs = bin + s * (N + 1);
        for (uint64_t q = q0; q < q0 + nq; q++) {
            double wout = 1.0;                                            // prod over outer digits
            for (int p = 1; p <= P; p++) wout *= bin[order[p] * (N + 1) + gdig[(p - 1) * 32 + lane]];
            const bool fwd = (q & 1ull) == 0;
            const uint32_t step = cs + (fwd ? 0u : NEG);
            double ar = 0.0, ai = 0.0;
            for (int j = 0; j <= ms; j++) {
                const int fsv = fwd ? j : ms - j;
                const double wt = sgn * wout * bs[fsv];                  // exact: +-integer < 2^n
                double xr, xi, yr, yi;
                two_factors<N, (N >= 4 ? 2 : 1)>(wr, wi, xr, xi, yr, yi);
                if constexpr (N == 1) { yr = 1.0; yi = 0.0; }
                xr *= wt;
                xi *= wt;
                fused_acc<+1>(xr, xi, yr, yi, ar, ai);
                if (j < ms) {
                    flip_add<N>(step, wr, wi);
                    sgn = -sgn;
                }
            }
            acc.re = dd_add_d(acc.re, ar);
            acc.im = dd_add_d(acc.im, ai);
            if (q + 1 < q0 + nq) {
                // q -> q+1 changes the lowest outer digit p whose ordinary digit is not at its top;
                // its Gray value moves +1 if the number above it is even, else -1
                uint64_t x = q;
                int p = 1;
                for (; p <= P; p++) {
                    const uint64_t r = (uint64_t)rad[p];
                    if (x % r != r - 1) break;
                    x /= r;
                }
                const bool up = ((x / (uint64_t)rad[p]) & 1ull) == 0;
                unsigned char* g = gdig + (p - 1) * 32 + lane;
                *g = (unsigned char)(*g + (up ? 1 : -1));
                flip_add<N>(base + (uint32_t)(order[p] * N) * 16u + (up ? 0u : NEG), wr, wi);
                sgn = -sgn;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
    if (lane == 0) {
        const double f = (N & 1) ? -1.0 : 1.0;
        const double re = (acc.re.hi + acc.re.lo) * f;
        const double im = (acc.im.hi + acc.im.lo) * f;
        if (per) per[b] = make_double2(re, im);
        if (abs2) abs2[b] = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
    }
}

template <int N>
cudaError_t weighted_launch_t(const double2* C, const int32_t* mult, int R, int64_t B, double2* per, double* abs2,
                              cudaStream_t st) {
    const size_t smem = WgtCfg::WARPS * wgt_slot_bytes(N, R);
    cudaError_t err = cudaFuncSetAttribute(weighted_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const int64_t grid = (B + WgtCfg::WARPS - 1) / WgtCfg::WARPS;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    weighted_kernel<N><<<(unsigned)grid, WgtCfg::NT, smem, st>>>(C, mult, R, B, per, abs2);
    return cudaGetLastError();
}

#define PERM_R8(M, b) M(b + 1) M(b + 2) M(b + 3) M(b + 4) M(b + 5) M(b + 6) M(b + 7) M(b + 8)

cudaError_t weighted_launch(const double2* C, const int32_t* mult, int n, int R, int64_t B, double2* per,
                            double* abs2, cudaStream_t s, int* launches) {
    *launches = 0;
    if (B == 0) return cudaSuccess;
    *launches = 1;
#define PERM_CASE(N) case N: return weighted_launch_t<N>(C, mult, R, B, per, abs2, s);
    switch (n) { PERM_R8(PERM_CASE, 0) PERM_R8(PERM_CASE, 8) PERM_R8(PERM_CASE, 16) PERM_R8(PERM_CASE, 24)
                 default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

}  // namespace perm
