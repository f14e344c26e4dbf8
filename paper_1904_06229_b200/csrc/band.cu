// band.cu -- permanents of matrices of limited bandwidth k (App. C
// bandpermanent, Sec. II-D), batched.
//
// App. C multiplies the row forms C_i = sum_j a_ij x_j with x_j^2 = 0, setting each x_j to 1 once no
// later row can reach column j.  Every surviving monomial is an injective row -> column assignment
// inside the band, so the coefficient bookkeeping is a transfer matrix over "which columns of the
// current window are already used".  The monomials that can still complete are exactly those in which
// every column left of the window is used, so before row i (0-based) the state is the set M of used
// columns among the 2k columns i-k .. i+k-1 and |M| = k (i columns used, the i-k left of the window
// all of them; virtual columns < 0 count as used).  Row i picks a free column j in i-k .. i+k (bit p,
// j = i-k+p); the column i-k leaves the window and must be used, so the new state is
// (M | 1<<p) >> 1, again with k bits.  After row n-1 the answer is the coefficient of the state
// "columns n-k .. n-1 used" (virtual columns >= n unused), i.e. the all-low-bits state, rank 0.
//
// C(2k, k) states (k = 6: 924), at most k+1 predecessors each.  One warp per matrix (persistent, matrices
// round-robin over the resident warps): lane l owns the states l, l+32, ... and keeps their predecessor
// ranks (combinatorial number system) in registers; the row's 2k+1 entries are prefetched one row
// ahead and broadcast from shared memory; coefficients are double-buffered in shared memory.
#include <mutex>
#include <vector>

#include "internal.h"

namespace perm {

constexpr int kBandWarps = 2;

__host__ __device__ constexpr int band_states(int k) {
    int c = 1;
    for (int r = 1; r <= k; r++) c = c * (k + r) / r;     // C(2k, k), exact at every step
    return c;
}

__host__ __device__ constexpr int binom_i(int m, int r) {
    if (r < 0 || r > m) return 0;
    int c = 1;
    for (int t = 1; t <= r; t++) c = c * (m - r + t) / t;
    return c;
}

// rank of a k-subset (bit mask over 2k positions) in the combinatorial number system
__device__ __forceinline__ int band_rank(uint32_t m) {
    int r = 0, i = 1;
    while (m) {
        const int c = __ffs(m) - 1;
        r += binom_i(c, i);
        i++;
        m &= m - 1;
    }
    return r;
}

__device__ __forceinline__ uint32_t band_unrank(int r, int k, int width) {
    uint32_t m = 0;
    for (int i = k; i >= 1; i--) {
        int c = i - 1;
        while (c + 1 < width && binom_i(c + 1, i) <= r) c++;
        r -= binom_i(c, i);
        m |= 1u << c;
    }
    return m;
}

// Coefficient slots: state rank t lives at slot[t] of a (S rounded up to 8)-entry array.  The slots are
// chosen on the host (band_layout) so that the 16-byte gathers of a warp hit distinct bank groups as
// often as possible: a 128-bit shared load is served per quarter warp (8 lanes x 16 B = the 32 banks),
// and two lanes of a quarter reading different slots with equal slot mod 8 cost an extra wavefront.
__host__ __device__ constexpr int band_nslots(int k) { return (band_states(k) + 7) / 8 * 8; }
constexpr int kBandMaxStates = 924;                    // C(12, 6)
struct BandSlots {
    int16_t slot[kBandMaxStates];                      // rank -> slot
};

// per warp: 2 nslots double2 coefficients (double buffer) + the current row (2k+1 double2); for k = 6
// the predecessor table (S (k+1) ints) follows
constexpr size_t band_smem_bytes(int k) {
    return (size_t)kBandWarps * ((size_t)2 * band_nslots(k) + 2 * k + 1) * sizeof(double2) +
           (k >= 6 ? (size_t)band_states(k) * (k + 1) * sizeof(int) : 0);
}

__device__ __forceinline__ double2 lds_band(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

template <int K>
__global__ void __launch_bounds__(32 * kBandWarps) band_kernel(const double2* __restrict__ A, int n, int64_t B,
                                                               double2* __restrict__ per,
                                                               double* __restrict__ abs2,
                                                               const __grid_constant__ BandSlots L) {
    constexpr int S = band_states(K), W = 2 * K + 1, P1 = K + 1, NS = band_nslots(K);
    constexpr int SPL = (S + 31) / 32;                                     // states per lane
    extern __shared__ __align__(16) unsigned char bsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (K == 0) {
        // bandwidth 0: one state (the empty window), the transfer step multiplies by a_ii -- per = prod a_ii;
        // one lane per matrix
        for (int64_t b = ((int64_t)blockIdx.x * kBandWarps + warp) * 32 + lane; b < B;
             b += (int64_t)gridDim.x * kBandWarps * 32) {
            double vr = 1.0, vi = 0.0;
            for (int i = 0; i < n; i++) {
                const double2 a = A[b * (int64_t)n + i];
                const double t = vr * a.y;
                vr = fma(vr, a.x, -vi * a.y);
                vi = fma(vi, a.x, t);
            }
            if (per) per[b] = make_double2(vr, vi);
            if (abs2) abs2[b] = __dadd_rn(__dmul_rn(vr, vr), __dmul_rn(vi, vi));
        }
        (void)bsm;
        return;
    } else {
    double2* cur = (double2*)bsm + (size_t)warp * (2 * NS + W);
    double2* nxt = cur + NS;
    double2* row = cur + 2 * NS;
    // this lane's states t = lane + 32 u and their predecessors, packed (old state rank << 4 | window bit
    // p): new state t <- old state (t's mask << 1 | 1) without bit p, for each set bit p.  In registers
    // up to k = 5; for k = 6 (29 states per lane) in shared memory, built once per block.
    constexpr bool REG = SPL * P1 <= 64;
    int predr[REG ? SPL : 1][REG ? P1 : 1];
    int* preds = (int*)(cur + (size_t)(kBandWarps - warp) * (2 * NS + W));  // after the warps' slots
#pragma unroll
    for (int u = 0; u < (REG ? SPL : (S + 32 * kBandWarps - 1) / (32 * kBandWarps)); u++) {
        const int t = REG ? lane + 32 * u : (int)threadIdx.x + u * 32 * kBandWarps;
        const uint32_t nw = t < S ? ((band_unrank(t, K, 2 * K) << 1) | 1u) : 0u;
        int q = 0;
        int packed[P1];
#pragma unroll
        for (int x = 0; x < P1; x++) packed[x] = -1;
        for (int p = 0; p <= 2 * K; p++) {
            if (!((nw >> p) & 1u)) continue;
            const uint32_t m = nw & ~(1u << p);
            if (m >> (2 * K)) continue;                                    // must fit the 2k-bit window
#pragma unroll
            for (int x = 0; x < P1; x++)
                if (x == q) packed[x] = ((int)L.slot[band_rank(m)] << 4) | p;
            q++;
        }
        if constexpr (REG) {
#pragma unroll
            for (int x = 0; x < P1; x++) predr[u][x] = packed[x];
        } else if (t < S) {
#pragma unroll
            for (int x = 0; x < P1; x++) preds[t * P1 + x] = packed[x];
        }
    }
    int st[SPL];                                                           // this lane's store slots
#pragma unroll
    for (int u = 0; u < SPL; u++) st[u] = (lane + 32 * u < S) ? (int)L.slot[lane + 32 * u] : 0;
    if constexpr (!REG) __syncthreads();
    const int64_t nwarps = (int64_t)gridDim.x * kBandWarps;
    for (int64_t b = (int64_t)blockIdx.x * kBandWarps + warp; b < B; b += nwarps) {
        const double2* Ab = A + b * (int64_t)n * W;
        const int slot0 = L.slot[0];
        for (int s = lane; s < NS; s += 32) cur[s] = make_double2(s == slot0 ? 1.0 : 0.0, 0.0);
        double2 rnext = make_double2(0.0, 0.0);
        if (lane < W) rnext = (lane - K >= 0 && lane - K < n) ? Ab[lane] : make_double2(0.0, 0.0);
        for (int i = 0; i < n; i++) {
            __syncwarp();
            if (lane < W) row[lane] = rnext;
            if (lane < W && i + 1 < n) {                                   // prefetch the next row
                const int j = i + 1 - K + lane;
                rnext = (j >= 0 && j < n) ? Ab[(int64_t)(i + 1) * W + lane] : make_double2(0.0, 0.0);
            }
            __syncwarp();
            const uint32_t cb = (uint32_t)__cvta_generic_to_shared(cur);
            const uint32_t rb = (uint32_t)__cvta_generic_to_shared(row);
#pragma unroll
            for (int u = 0; u < SPL; u++) {
                const int t = lane + 32 * u;
                if (t < S) {
                    // ranks < S/2 have no state bit 2k-1 set: k+1 predecessors; the others exactly one
                    const int np = (t < S / 2) ? P1 : 1;
                    double vr = 0.0, vi = 0.0;
#pragma unroll
                    for (int x = 0; x < P1; x++) {
                        if (x >= np) break;
                        const int e = REG ? predr[REG ? u : 0][REG ? x : 0] : preds[t * P1 + x];
                        const double2 c = lds_band(cb + (uint32_t)(e >> 4) * 16u);
                        const double2 a = lds_band(rb + (uint32_t)(e & 15) * 16u);
                        vr = fma(c.x, a.x, vr);
                        vr = fma(-c.y, a.y, vr);
                        vi = fma(c.x, a.y, vi);
                        vi = fma(c.y, a.x, vi);
                    }
                    nxt[st[u]] = make_double2(vr, vi);
                }
            }
            double2* tmp = cur;
            cur = nxt;
            nxt = tmp;
        }
        __syncwarp();
        if (lane == 0) {
            const double2 r = cur[L.slot[0]];
            if (per) per[b] = r;
            if (abs2) abs2[b] = __dadd_rn(__dmul_rn(r.x, r.x), __dmul_rn(r.y, r.y));
        }
    }
    }
}

// ---- host: the slot layout (computed once per k) --------------------------------------------------
static uint32_t h_unrank(int r, int k, int width) {
    uint32_t m = 0;
    for (int i = k; i >= 1; i--) {
        int c = i - 1;
        while (c + 1 < width && binom_i(c + 1, i) <= r) c++;
        r -= binom_i(c, i);
        m |= 1u << c;
    }
    return m;
}

static int h_rank(uint32_t m) {
    int r = 0, i = 1;
    for (int c = 0; m; c++, m >>= 1)
        if (m & 1u) r += binom_i(c, i++);
    return r;
}

// Colours (slot mod 8) by local search: start from slot = rank, swap the colours of two states when that
// does not increase the number of wavefronts of the gathers (every (state group u, predecessor x,
// quarter warp) of the kernel's loop) and of the coefficient stores; swaps keep the colour classes equal
// in size, so the slots fill 8 x ceil(S/8) entries.  Deterministic (fixed LCG).
static void band_layout_compute(int k, BandSlots& out) {
    const int S = band_states(k), P1 = k + 1, SPL = (S + 31) / 32;
    std::vector<int> np(S), pr((size_t)S * P1, -1);
    for (int t = 0; t < S; t++) {
        const uint32_t nw = (h_unrank(t, k, 2 * k) << 1) | 1u;
        int q = 0;
        for (int p = 0; p <= 2 * k; p++) {
            if (!((nw >> p) & 1u)) continue;
            const uint32_t m = nw & ~(1u << p);
            if (m >> (2 * k)) continue;
            pr[(size_t)t * P1 + q++] = h_rank(m);
        }
        np[t] = q;
    }
    std::vector<std::vector<int>> groups;                 // distinct states read / written together
    for (int u = 0; u < SPL; u++)
        for (int x = 0; x <= P1; x++)                     // x == P1: the stores nxt[slot[t]]
            for (int ph = 0; ph < 4; ph++) {
                std::vector<int> g;
                for (int l = 8 * ph; l < 8 * ph + 8; l++) {
                    const int t = l + 32 * u;
                    if (t >= S) continue;
                    const int v = x == P1 ? t : (x < np[t] ? pr[(size_t)t * P1 + x] : -1);
                    if (v < 0) continue;
                    bool dup = false;
                    for (int w : g) dup |= (w == v);
                    if (!dup) g.push_back(v);
                }
                if (g.size() > 1) groups.push_back(g);
            }
    std::vector<std::vector<int>> member(S);
    for (int gi = 0; gi < (int)groups.size(); gi++)
        for (int v : groups[gi]) member[v].push_back(gi);
    std::vector<int> col(S);
    for (int t = 0; t < S; t++) col[t] = t % 8;
    auto gcost = [&](int gi) {
        int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mx = 0;
        for (int v : groups[gi]) mx = std::max(mx, ++cnt[col[v]]);
        return mx;
    };
    uint64_t rng = 0x9e3779b97f4a7c15ull + (uint64_t)k;
    auto next = [&]() { rng = rng * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(rng >> 33); };
    std::vector<int> touched;
    const int iters = (k <= 5 ? 1500 : 300) * S;       // one-time host cost: ~0.1 s at k = 5
    for (int it = 0; it < iters; it++) {
        const int a = (int)(next() % (uint32_t)S), b = (int)(next() % (uint32_t)S);
        if (col[a] == col[b]) continue;
        touched.clear();
        for (int gi : member[a]) touched.push_back(gi);
        for (int gi : member[b]) touched.push_back(gi);
        int before = 0, after = 0;
        for (int gi : touched) before += gcost(gi);
        std::swap(col[a], col[b]);
        for (int gi : touched) after += gcost(gi);
        if (after > before) std::swap(col[a], col[b]);    // (groups shared by a and b count twice: harmless)
    }
    int fill[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int t = 0; t < S; t++) out.slot[t] = (int16_t)(col[t] + 8 * fill[col[t]]++);
}

static const BandSlots& band_layout(int k) {
    static std::once_flag once[kMaxBandK + 1];
    static BandSlots lay[kMaxBandK + 1];
    std::call_once(once[k], [k] { band_layout_compute(k, lay[k]); });
    return lay[k];
}

template <int K>
cudaError_t band_launch_t(const double2* A, int n, int64_t B, double2* per, double* abs2, cudaStream_t s) {
    const size_t smem = band_smem_bytes(K);
    cudaError_t err = cudaFuncSetAttribute(band_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, bps = 0;
    err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, band_kernel<K>, 32 * kBandWarps, smem);
    if (err != cudaSuccess) return err;
    if (bps < 1) bps = 1;
    const int64_t need = (B + kBandWarps - 1) / kBandWarps;
    const int64_t grid = need < (int64_t)sms * bps ? need : (int64_t)sms * bps;
    band_kernel<K><<<(unsigned)grid, 32 * kBandWarps, smem, s>>>(A, n, B, per, abs2, band_layout(K));
    return cudaGetLastError();
}

cudaError_t band_launch(const double2* A, int n, int k, int64_t B, double2* per, double* abs2, cudaStream_t s,
                        int* launches) {
    *launches = 0;
    if (B == 0) return cudaSuccess;
    *launches = 1;
    switch (k) {
        case 0: return band_launch_t<0>(A, n, B, per, abs2, s);
        case 1: return band_launch_t<1>(A, n, B, per, abs2, s);
        case 2: return band_launch_t<2>(A, n, B, per, abs2, s);
        case 3: return band_launch_t<3>(A, n, B, per, abs2, s);
        case 4: return band_launch_t<4>(A, n, B, per, abs2, s);
        case 5: return band_launch_t<5>(A, n, B, per, abs2, s);
        case 6: return band_launch_t<6>(A, n, B, per, abs2, s);
        default: *launches = 0; return cudaErrorInvalidValue;
    }
}

}  // namespace perm
