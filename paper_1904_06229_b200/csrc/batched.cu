// batched.cu -- per(A_b) and |per(A_b)|^2 for a batch of small complex matrices (
// BASELINE config 2: Boson-sampling probabilities of n x n submatrices of a Haar unitary).
//
// Mapping: a group of L lanes walks one matrix; lane l of the group takes the aligned chunk
// [l 2^E, (l+1) 2^E) of the 2^{n-1} Gray ranks (E = n-1-log2 L), using the same walker as the
// single-matrix kernel (walk.cuh: seeding, unrolled inner blocks, dd accumulation).  For n >= 12 a
// whole warp walks one matrix, so every column read is a warp-uniform shared-memory broadcast; for
// small n (few terms per matrix) several matrices share a warp.  Each warp stages its matrices
// (coalesced global reads) column-major, with a negated copy, into its own shared-memory slice.  The group's dd partials
// are combined with a fixed shuffle tree; lane 0 applies 2(-1)^n (App. A permanent step 4)
// and writes per (rounded from dd), |per|^2 = re^2 + im^2 of that rounded value and, if asked, the
// ensemble statistic X = |per| / sqrt(n!) of Secs. IV-V: X = sqrt(|per|^2 / n!).
#include "walk.cuh"

namespace perm {

// unit-column walk in the batched kernel (development: PERM_BATCHED_UNIT=0 walks every matrix as given)
#ifndef PERM_BATCHED_UNIT
#define PERM_BATCHED_UNIT 1
#endif
constexpr bool kBatchedUnit = PERM_BATCHED_UNIT != 0;

template <int N>
struct BatCfg {
    static constexpr int LOG_L = (N - 1 - 5) < 0 ? 0 : ((N - 1 - 5) > 5 ? 5 : (N - 1 - 5));
    static constexpr int L = 1 << LOG_L;          // lanes per matrix
    static constexpr int G = 32 / L;              // matrices per warp
    static constexpr int E = N - 1 - LOG_L;       // log2 ranks per lane
    static constexpr int WARPS = 4;
    static constexpr int NT = 32 * WARPS;
    static constexpr int MAT = 2 * N * N + N;     // double2 per matrix slot (columns, negated columns, base)
    static constexpr int SLOT = MAT + 1;          // +1 double2 pad: consecutive slots start in different banks
    static constexpr size_t smem_bytes = (size_t)WARPS * G * SLOT * sizeof(double2);
};

template <int N>
__global__ void __launch_bounds__(BatCfg<N>::NT) batched_kernel(const double2* __restrict__ A, int64_t B,
                                                                double2* __restrict__ per,
                                                                double* __restrict__ abs2,
                                                                double* __restrict__ xs, double nfact) {
    using C = BatCfg<N>;
    extern __shared__ double2 smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2* wbase = smem + (size_t)warp * C::G * C::SLOT;
    const int64_t m0 = ((int64_t)blockIdx.x * C::WARPS + warp) * C::G;   // first matrix of this warp
    if (m0 >= B) return;                                                 // warp-uniform
    const int gcount = (B - m0) < C::G ? (int)(B - m0) : C::G;

    // stage: element k of the warp's matrices (row-major, contiguous in the batch) -> column-major slot
    const double2* src = A + m0 * (N * N);
    for (int k = lane; k < gcount * N * N; k += 32) {
        const int g = k / (N * N), r = k - g * (N * N);
        const int i = r / N, j = r - i * N;
        const double2 a = src[k];
        wbase[g * C::SLOT + j * N + i] = a;
        wbase[g * C::SLOT + N * N + j * N + i] = make_double2(-a.x, -a.y);
    }
    __syncwarp();
    // unit-column walk (walk.cuh InnerStepU) when a warp walks one matrix (n >= 11): rows divided by their column-0
    // entry, scale = prod_i a_i0 in double-double (a fixed shuffle tree over the rows' lanes); a matrix with a zero (or
    // relatively tiny) column-0 entry is walked as given
    constexpr bool UNIT = kBatchedUnit && N >= 14 && C::G == 1 && C::E >= WCfg<N, 1>::U && WCfg<N, 1>::K >= 2;
    [[maybe_unused]] bool unit = false;
    [[maybe_unused]] ddc scale;
    if constexpr (UNIT) {
        ddc f;
        f.re = dd{1.0, 0.0};
        f.im = dd{0.0, 0.0};
        bool okl = true;
        if (lane < N) {
            const double2 a = wbase[lane];                        // column 0, row `lane`
            const double m = fmax(fabs(a.x), fabs(a.y));
            double rmax = 0.0;
            for (int j = 1; j < N; j++) rmax = fmax(rmax, fabs(wbase[j * N + lane].x) + fabs(wbase[j * N + lane].y));
            okl = m > 0.0 && rmax / m <= 1e100;
            f.re = dd{a.x, 0.0};
            f.im = dd{a.y, 0.0};
        }
        unit = __all_sync(0xffffffffu, okl);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) f = ddc_mul(f, shfl_down_ddc(f, off));   // lane 0: the product
        scale = f;
        if (unit) {
            // a'_ij = a_ij / a_i0 (= a_ij conj(a_i0) / |a_i0|^2, scaled by max(|re|, |im|) against underflow)
            for (int r = lane; r < N * N; r += 32) {
                const int jc = r / N, i = r - jc * N;             // column-major: r = j N + i
                const double2 a0 = wbase[i];
                const double m = fmax(fabs(a0.x), fabs(a0.y));
                const double sr = a0.x / m, si = a0.y / m, d = sr * sr + si * si;
                const double ir = sr / (d * m), ii = -si / (d * m);
                const double2 a = wbase[r];
                const double2 v = jc == 0 ? make_double2(1.0, 0.0)
                                          : make_double2(a.x * ir - a.y * ii, a.x * ii + a.y * ir);
                wbase[N * N + r] = make_double2(-v.x, -v.y);
                if (jc != 0) wbase[r] = v;
            }
            __syncwarp();
            if (lane < N) wbase[lane] = make_double2(1.0, 0.0);  // column 0 last (the others read it)
            __syncwarp();
        }
    }
    for (int k = lane; k < gcount * N; k += 32) {
        const int g = k / N, i = k - g * N;
        const double2* sc = wbase + g * C::SLOT;
        double sr = 0.0, si = 0.0;
        for (int j = 0; j < N; j++) {
            sr += sc[j * N + i].x;
            si += sc[j * N + i].y;
        }
        wbase[g * C::SLOT + 2 * N * N + i] =
            make_double2(sc[(N - 1) * N + i].x - 0.5 * sr, sc[(N - 1) * N + i].y - 0.5 * si);
    }
    __syncwarp();

    const int g = lane / C::L, l = lane % C::L;
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    if (g < gcount) {
        using WC = WCfg<N, 1>;   // one lane per chunk; column stride N (no padding); -A at WC::NEG
        const uint32_t sc = (uint32_t)__cvta_generic_to_shared(wbase + g * C::SLOT);
        const uint32_t sbase = sc + (uint32_t)(2 * N * N) * 16u;
        if constexpr (C::E == 0) {
            single_term<WC>(sc, sbase, 0u, (uint64_t)l, acc);
        } else if constexpr (UNIT) {
            if (unit) walk_chunk_unit<WC>(sc, sbase, (uint64_t)l, C::E, acc);
            else      walk_chunk<WC>(sc, sbase, 0u, (uint64_t)l, C::E, acc);
        } else {
            walk_chunk<WC>(sc, sbase, 0u, (uint64_t)l, C::E, acc);
        }
    }
    // fixed-order tree over the L lanes of each group
#pragma unroll
    for (int off = C::L / 2; off > 0; off >>= 1) acc = ddc_add(acc, shfl_down_ddc(acc, off));
    if (l == 0 && g < gcount) {
        if constexpr (UNIT) {
            if (unit) acc = ddc_mul(acc, scale);                 // back to the units of A (lane 0 holds the scale)
        }
        const double f = (N & 1) ? -2.0 : 2.0;
        const double re = (acc.re.hi + acc.re.lo) * f;
        const double im = (acc.im.hi + acc.im.lo) * f;
        const int64_t m = m0 + g;
        PERM_DCHECK(m < B);
        if (per) per[m] = make_double2(re, im);
        const double a2 = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));   // no FMA: fl(fl(re^2) + fl(im^2))
        if (abs2) abs2[m] = a2;
        if (xs) xs[m] = __dsqrt_rn(__ddiv_rn(a2, nfact));
    }
}

template <int N>
cudaError_t batched_launch_t(const double2* A, int64_t B, double2* per, double* abs2, double* xs, cudaStream_t s) {
    using C = BatCfg<N>;
    static_assert(C::E >= WCfg<N, 1>::U || C::E == 0, "lane chunk shorter than the unrolled block");
    cudaError_t err = cudaFuncSetAttribute(batched_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem_bytes);
    if (err != cudaSuccess) return err;
    const int64_t per_block = (int64_t)C::WARPS * C::G;
    const int64_t grid = (B + per_block - 1) / per_block;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    double nfact = 1.0;                                   // n! rounded to binary64 (exact for n <= 22)
    for (int k = 2; k <= N; k++) nfact *= (double)k;
    batched_kernel<N><<<(unsigned)grid, C::NT, C::smem_bytes, s>>>(A, B, per, abs2, xs, nfact);
    return cudaGetLastError();
}

#define PERM_R8(M, b) M(b + 1) M(b + 2) M(b + 3) M(b + 4) M(b + 5) M(b + 6) M(b + 7) M(b + 8)

cudaError_t batched_launch(const double2* A, int n, int64_t B, double2* per, double* abs2, double* xs,
                           cudaStream_t s, int* launches) {
    *launches = 0;
    if (B == 0) return cudaSuccess;
    *launches = 1;
#define PERM_CASE(N) case N: return batched_launch_t<N>(A, B, per, abs2, xs, s);
    switch (n) { PERM_R8(PERM_CASE, 0) PERM_R8(PERM_CASE, 8) PERM_R8(PERM_CASE, 16) PERM_R8(PERM_CASE, 24)
                 default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

}  // namespace perm
