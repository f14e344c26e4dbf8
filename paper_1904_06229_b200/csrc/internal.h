// internal.h -- host-side launch interfaces between the C-ABI layer (abi.cu) and the kernel
// translation units.  Not part of the public ABI (see include/perm.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace perm {

constexpr int kMaxN = 64;          // ranks are 64-bit words
constexpr int kMaxBatchedN = 32;   // perm_c128_batched
constexpr int kMaxGlynnInt01N = 28;   // exactness bound of the int128 Glynn sum (R10)
constexpr int kMaxInt01N = 33;        // full-range Ryser in int128 beyond it: |per| <= n! < 2^127
constexpr int kMaxSegments = 96;

// Inner unrolled Gray bits U(N) of the single-matrix walk: a block of 2^U consecutive ranks is
// fully unrolled, so the columns 0..U-1 it touches are compile-time operands.
#ifdef PERM_WALK_U
__host__ __device__ constexpr int walk_inner_bits(int n) { return (n - 1) < PERM_WALK_U ? (n - 1) : PERM_WALK_U; }
#else
// U = 3 (8-term blocks) up to n = 39 and U = 2 beyond (the 4n-register row sums leave ptxas less room
// to overlap an 8-term block); U = 2 also for the constant-bank orders 34, 35, 37, 39, whose register caps
// (walk.cuh: walk_const_maxnreg) were found for U = 2.
#ifndef PERM_U2_FROM33
#define PERM_U2_FROM33 1                                  // U = 2 for every n >= 33 (n = 33, 36, 38: +6..13%)
#endif
__host__ __device__ constexpr int walk_inner_bits(int n) {
    return (n == 34 || n == 35 || n == 37 || n == 39 || n >= 40 || (PERM_U2_FROM33 && n >= 33)) ? 2
                                                                                 : ((n - 1) < 3 ? (n - 1) : 3);
}
#endif
constexpr int kWalkThreads = 64;
// Lanes that share one chunk in the shared-memory walk (rows split between them).  The n
// complex row sums take 4n registers; from n = 33 one lane cannot hold them next to the shared-memory column
// operands without spilling, so two lanes split the rows.  For n <= 48 the aligned chunks of a walk run in
// the constant-bank kernel (one lane per chunk, uniform-register columns); this kernel then only walks
// unaligned edge pieces and chunks of 2^U ranks.
#ifndef PERM_WALK_S2_MIN
#define PERM_WALK_S2_MIN 33
#endif
#ifndef PERM_WALK_S4_MIN
#define PERM_WALK_S4_MIN 65
#endif
__host__ __device__ constexpr int walk_lanes_per_chunk(int n) {
    return n >= PERM_WALK_S4_MIN ? 4 : (n >= PERM_WALK_S2_MIN ? 2 : 1);
}
// Threads per block of the shared-memory walk.  Each block stages A and -A column-major plus the base
// vector, (2 n P + P) x 16 bytes (P = padded rows); at n = 44 that is 62.6 KB, so 64-thread blocks
// (4 per SM at 255 registers) would not fit the 228 KB of shared memory per SM -- larger orders get
// larger blocks instead of fewer warps.
__host__ __device__ constexpr int walk_block_threads(int n) {
    const int s = walk_lanes_per_chunk(n);
    const int p = ((n + s - 1) / s) * s;
    const long bytes = (2L * n * p + p) * 16L;
    return bytes * 4 <= 200L * 1024 ? kWalkThreads : (bytes * 2 <= 220L * 1024 ? 2 * kWalkThreads : 4 * kWalkThreads);
}
// Plain-double partial sums are folded into the per-thread double-double accumulator every
// 2^kWalkFoldBits terms (R7).
#ifndef PERM_WALK_FOLD
#define PERM_WALK_FOLD 5
#endif
constexpr int kWalkFoldBits = PERM_WALK_FOLD;
// The n = 44 constant-bank walk folds every 2^7 terms: +0.3% (profiles/round1_walk_chains.txt); the plain
// partial over 128 terms of |prod w| ~ 1e23 carries ~1e9 absolute rounding, 1e-20 of the error floor.
#ifndef PERM_FOLD44
#define PERM_FOLD44 7
#endif
__host__ __device__ constexpr int walk_fold_bits_const(int n) { return n == 44 ? PERM_FOLD44 : kWalkFoldBits; }

// A run of `count` aligned chunks of 2^e ranks: chunk k covers ranks [(c0+k) 2^e, (c0+k+1) 2^e).
// e == 0 chunks are single terms (seeded from scratch).
struct Segment {
    uint64_t c0;
    uint64_t count;
    int e;
};

// Largest order whose whole matrix fits the 32 KB kernel-parameter space (walk_kernel_c).
constexpr int kConstMaxN = 48;
// Orders that use the constant-bank walk: the ones for which ptxas keeps the per-use parameter loads on
// the uniform datapath (LDCU -> DADD R, R, UR, one vector register read per update) -- n = 32 at its
// default allocation, 33..48 under the register caps of walk_const_maxnreg (walk.cuh).
// Measured on B200 (profiles/round1_const_table_rates.txt): +4..12% over the shared-memory walk (n = 44:
// 6.14e10 vs 5.49e10 terms/s).  PERM_CONST_ORDERS=0 enables the path for every n <= kConstMaxN (scans).
#ifndef PERM_CONST_ORDERS
#define PERM_CONST_ORDERS 32
#endif
#ifndef PERM_CONST_MIN
#define PERM_CONST_MIN 33                                 // (development: 99 = shared-memory walk above n = 32)
#endif
__host__ __device__ constexpr bool walk_const_path(int n) {
#if PERM_CONST_ORDERS == 0
    return n <= kConstMaxN;                               // scans only
#else
    return n == PERM_CONST_ORDERS || (n >= PERM_CONST_MIN && n <= kConstMaxN);
#endif
}

// Unit-column walk: for these constant-bank orders the library walks A' = D^{-1} A, each row
// divided by its entry in column 0 (the Gray bit-0 column), so that column is all ones; per(A) = prod_i a_i0 *
// per(A') term by term, and every item partial is multiplied by that product (in double-double) before it is
// written, so partials, tree nodes and results stay in the units of A.  With a unit bit-0 column the two terms of
// ranks 2q, 2q+1 are prod v and prod (v + 1) for one row-sum vector v: the bit-0 flips disappear and the "+1" fuses
// into the product's FMAs.  PERM_UNIT0_ORDERS=0: off; =1: every constant-bank order; else that order only.
#ifndef PERM_UNIT0_ORDERS
#define PERM_UNIT0_ORDERS 1
#endif
__host__ __device__ constexpr bool walk_unit0(int n) {
    return PERM_UNIT0_ORDERS == 1 ? walk_const_path(n) : (PERM_UNIT0_ORDERS != 0 && n == PERM_UNIT0_ORDERS);
}

// chunk walkers per block of the kernel that walks the aligned body (walk_kernel_c)
__host__ __device__ constexpr int walk_body_walkers(int n) { return walk_block_threads(n); }

// Chunk length 2^b of a WHOLE permanent (perm_c128) and of the chunk walk (perm_c128_chunks' default):
// a function of n alone, so the per-chunk partials -- and through the canonical tree (tree.cu) the
// result -- do not depend on the grid, the number of GPUs or how the chunks are sliced into launches.
// Chosen with a cost model for B200 (37,888 resident walkers): chunks = 2^{n-1-b} <= 2^25 for n <= 56
// (tail of the static round-robin <= 0.3% at 1 GPU, 0.3% at 8 GPUs for n >= 37), and b >= 10 where that
// leaves enough chunks (explicit seeding costs 2n(n-1-b) FP64 instructions per 2^b terms: < 1%).
__host__ __device__ constexpr int walk_chunk_log2(int n) {
    const int u = walk_inner_bits(n);
    const int a = n - 26, c = (n - 19) < 10 ? (n - 19) : 10;
    int b = a > c ? a : c;
    if (b < u) b = u;
    if (b > 30) b = 30;
    if (b > n - 1) b = n - 1;
    return b < 0 ? 0 : b;
}

struct WalkLaunch {
    const double2* A_dev;   // device, row-major n x n
    const double2* A_host;  // host, row-major n x n (walk_kernel_c takes the matrix as a kernel parameter)
    int n;
    int nseg;
    Segment seg[kMaxSegments];
    ddc* items;             // device: one dd partial per walked item (segment order, chunks in rank order)
    uint64_t nitems;        // items of the plan (the length of `items`)
    int grid;               // blocks of the main launch
    int use_const;          // run segment `body` in walk_kernel_c
    int body;               // index of the body segment (use_const)
    int grid_edge;          // blocks of the edge launch (use_const and nseg > 1), else 0
    int unit0;              // A_dev / A_host hold A' (column 0 all ones, walk_unit0): the body runs the unit-column walk
    int scaled;             // multiply every item partial by `scale` (= prod_i a_i0 when unit0)
    ddc scale;
    cudaStream_t stream;
};

// One-launch path of a small whole permanent (walk.cuh: walk_small_kernel, a cluster of <= 16 CTAs).
constexpr int kSmallMaxN = 16;
constexpr int kSmallMaxThreads = 256;
constexpr uint64_t kSmallMaxChunks = 16 * kSmallMaxThreads;
template <int N> cudaError_t walk_small_launch(const double2* A_dev, int e, uint64_t chunks, ddc* raw, ddc* out_dd,
                                               double2* out_c, cudaStream_t s);
cudaError_t walk_small_launch_n(int n, const double2* A_dev, int e, uint64_t chunks, ddc* raw, ddc* out_dd,
                                double2* out_c, cudaStream_t s);

// Defined in walk_inst.cu (explicit instantiations over N = 1..64).
template <int N> cudaError_t walk_launch(const WalkLaunch& L);
template <int N> cudaError_t walk_occupancy(int* blocks_per_sm, int* walkers_per_block);
template <int N> cudaError_t walk_occupancy_c(int* blocks_per_sm);
template <int N> cudaError_t walk_seed_launch(const double2* A_dev, const uint64_t* ranks_dev, int count,
                                              double2* w_out, cudaStream_t s);

cudaError_t walk_launch_n(int n, const WalkLaunch& L);
cudaError_t walk_occupancy_n(int n, int* blocks_per_sm, int* walkers_per_block);
cudaError_t walk_occupancy_c_n(int n, int* blocks_per_sm);
cudaError_t walk_seed_launch_n(int n, const double2* A_dev, const uint64_t* ranks_dev, int count,
                               double2* w_out, cudaStream_t s);

// tree.cu: the canonical pairwise tree over absolute leaf indices.  Leaf i of a
// span is node (0, a0 + i); node (L+1, k) = ddc_add(node (L, 2k), node (L, 2k+1)).  A span [a0, a0+count)
// reduces to its maximal complete nodes (at most two per level), so partials of disjoint spans -- other
// launches, other GPUs -- merge into exactly the value one launch over the union would give.
struct TreeNode {           // == perm_tree_node_t (48 bytes)
    uint32_t level;         // ~0u: unused slot
    uint32_t reserved;
    uint64_t index;         // covers leaves [index << level, (index + 1) << level)
    ddc v;
};
constexpr int kTreeMaxNodes = 128;
constexpr uint32_t kTreeUnused = 0xffffffffu;
size_t tree_workspace_bytes(uint64_t count);
// nodes_dev: kTreeMaxNodes slots, the maximal nodes sorted by position, the rest marked unused (may be
// NULL); raw_dev (may be NULL): their left-to-right dd sum; out_dd / out_c (may be NULL): raw * f in dd /
// rounded to double.
cudaError_t tree_launch(const ddc* leaves, uint64_t a0, uint64_t count, void* ws, TreeNode* nodes_dev, ddc* raw_dev,
                        ddc* out_dd, double2* out_c, double f, cudaStream_t s, int* launches);

// abi.cu: stream-ordered scratch allocation.  The first call per device raises the release threshold of the
// device's default memory pool so that freed scratch stays cached (otherwise every synchronisation hands it
// back to the driver and the next call pays a real allocation on its latency path).
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s);

// reduce.cu
cudaError_t reduce_launch(const ddc* parts, int count, int n_final, ddc* out_dd, double2* out_c,
                          cudaStream_t s);
cudaError_t fp64_probe_launch(int blocks, int threads, int iters, double* sink, cudaStream_t s);

// batched.cu
cudaError_t batched_launch(const double2* A, int n, int64_t B, double2* per, double* abs2, double* xs, cudaStream_t s,
                           int* launches);

// sparse.cuh / sparse_inst.cu (App. B restricted enumeration), n <= kMaxSparseN
constexpr int kMaxSparseN = 48;
constexpr int kSparseMaxD = 64;
// shared-rows group walk (sparse.cuh walk_seeded_group): up to kSparseGroupMaxG thin T columns, together nonzero
// in at most kSparseGroupRows rows
constexpr int kSparseGroupRows = 4;
constexpr int kSparseGroupMaxG = 4;
#ifndef PERM_SPARSE_CONST
#define PERM_SPARSE_CONST 1
#endif
// orders of the constant-bank sparse kernel (sparse.cuh sparse_kernel_c; PERM_SPARSE_CONST=2: every order)
__host__ __device__ constexpr bool sparse_const_path(int n) {
    return PERM_SPARSE_CONST == 2 ? true
         : PERM_SPARSE_CONST == 1 ? ((n >= 17 && n <= 33 && n != 24) || n == 47 || n == 48) : false;
}
// ... and of its shared-rows group walk (the product of n - kSparseGroupRows >= 8 rows in two chains)
__host__ __device__ constexpr bool sparse_group_path(int n) { return sparse_const_path(n) && n >= kSparseGroupRows + 8; }
struct SparseLaunch {
    const double2* A_dev;   // device, row-major n x n
    ddc* partials;          // device, grid entries
    uint64_t outer;         // prod_l (2^{|S_l|} - 1)
    uint64_t chunks;        // T-walk chunks per outer combination
    int e, nt, d, n, grid;
    int col[64];            // permuted column order: T columns, then S_1, S_2, ...
    int row[64];            // row order (position i holds row row[i] of A; the identity unless pair)
    int group;              // shared-rows group walk (sparse.cuh): G thin T columns at slots 0..G-1, their
                            // nonzero rows the last kSparseGroupRows positions (0: the plain T walk)
    int soff[kSparseMaxD];  // first slot of S_l
    int ssz[kSparseMaxD];   // |S_l|
    const double2* A_host;  // host, row-major n x n (inner T columns for the constant-bank walk)
    cudaStream_t stream;
};
template <int N> cudaError_t sparse_launch_t(const SparseLaunch& L);
template <int N> cudaError_t sparse_occupancy_t(int* blocks_per_sm);
cudaError_t sparse_launch(const SparseLaunch& L);
cudaError_t sparse_occupancy(int n, int* blocks_per_sm);

// band.cu (App. C bandwidth-limited matrices)
constexpr int kMaxBandK = 6;
cudaError_t band_launch(const double2* A, int n, int k, int64_t B, double2* per, double* abs2, cudaStream_t s,
                        int* launches);

// weighted.cu
constexpr int kMaxWeightedR = 64;
cudaError_t weighted_launch(const double2* C, const int32_t* mult, int n, int R, int64_t B, double2* per,
                            double* abs2, cudaStream_t s, int* launches);

// int01.cu
size_t int01_workspace_bytes(int n, int64_t B);
cudaError_t int01_launch(const uint8_t* A, int n, int64_t B, bool pm1, void* out, void* ws, size_t ws_bytes,
                         cudaStream_t s, int* flag_host_status, int* launches);
// one 0-1 matrix over ranks [k0, k1): raw Gray sum mod 2^128 -> raw_host[0] (lo), raw_host[1] (hi)
constexpr int kInt01RangeBlocks = 148 * 8;
size_t int01_range_workspace_bytes();
cudaError_t int01_range_launch(const uint8_t* A, int n, uint64_t k0, uint64_t k1, void* ws, cudaStream_t s,
                               unsigned long long* raw_host, int* flag_host_status, int* launches);

}  // namespace perm
