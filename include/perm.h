/*
 * perm.h -- C ABI of the B200 (sm_100a) Gray-code Ryser/Glynn permanent library (libperm.so).
 *
 * The operation is the permanent of an n x n matrix,
 *     per(A) = sum_{pi in S_n} prod_i a_{i,pi(i)}               (Eq. (1)),
 * evaluated by Ryser's inclusion-exclusion formula (Eq. (3)) in its half-range
 * (Nijenhuis-Wilf / Glynn) form walked in Gray-code order, exactly as the
 * paper's App. A subpermanent/permanent:
 *
 *     w_i(r) = a_{i,n} - 1/2 sum_j a_{i,j} + sum_{j<n, x_j = 1} a_{i,j},   x = gray(r) = r ^ (r >> 1)
 *     P(k0, k1) = sum_{r = k0}^{k1 - 1} (-1)^{r+1} prod_{i=1}^{n} w_i(r)         ("raw partial")
 *     per(A) = 2 (-1)^n P(0, 2^{n-1})
 *
 * Conventions (all calls):
 *   - Complex matrices are row-major n x n arrays of perm_c128_t = {re, im} (binary64), i.e. the
 *     memory layout of a contiguous numpy / torch complex128 array.  Entry (i, j) is A[i*n + j].
 *     Column index j is 0-based; the pinned column of App. A ("a_{i,n}") is column n-1, and Gray
 *     bit j (bit 0 = least significant) selects column j.
 *   - Every call returns a perm_status_t; PERM_OK == 0.  On PERM_E_CUDA the CUDA error text of
 *     the failing call is available from perm_last_error() (thread-local).
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream).  A call whose
 *     output is HOST memory synchronizes that stream before returning; a call whose outputs are all
 *     DEVICE memory returns after enqueueing (stream-ordered, no host sync).
 *   - Pointers documented "host or device" are classified with cudaPointerGetAttributes.
 *   - The caller owns every buffer.  The library keeps no mutable global state, so concurrent calls
 *     on distinct buffers (and streams) are safe.  When `workspace` is NULL the library allocates
 *     the scratch it needs stream-ordered (cudaMallocAsync / cudaFreeAsync) on `stream`.
 *   - Results are deterministic: bit-identical for the same inputs, n, range and device.
 *   - Floating point: IEEE-754 binary64, round-to-nearest, no fast-math; products in binary64
 *     (FMA-contracted), sums accumulated in double-double (hi + lo) per component, i.e. the
 *     paper's "double product, extended sum" mode.
 */
#ifndef PERM_H_
#define PERM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } perm_c128_t;                      /* == complex128 */
typedef struct { double hi_re, lo_re, hi_im, lo_im; } perm_dd_c128_t; /* value = (hi_re+lo_re) + i(hi_im+lo_im) */
typedef struct { uint64_t lo; int64_t hi; } perm_i128_t;             /* two's-complement int128 = hi*2^64 + lo */

typedef struct {
    uint64_t terms;        /* out: Gray-code terms evaluated (2^{n-1} for a whole permanent, C20) */
    uint32_t chunk_log2;   /* out: b, the walk's aligned chunk length is 2^b                      */
    uint32_t threads;      /* out: walker threads launched                                        */
    uint32_t blocks;       /* out: walker blocks launched                                         */
    uint32_t launches;     /* out: kernels launched by this call                                  */
    void* ev_walk_begin;   /* in, optional cudaEvent_t: recorded on `stream` just before the walk
                              kernel is launched (NULL = not recorded)                            */
    void* ev_walk_end;     /* in, optional cudaEvent_t: recorded just after the walk kernel        */
    uint64_t items;        /* out: walked items (aligned chunks + single-rank pieces), one dd partial each */
    uint32_t const_path;   /* out: 1 if the aligned body ran in the constant-bank walk (walk_kernel_c*) */
    uint32_t reserved;
} perm_stats_t;

/* One node of the canonical reduction tree (perm_c128_tree): the dd sum of the chunk partials
 * [index * 2^level, (index + 1) * 2^level), combined as node(L+1, k) = node(L, 2k) + node(L, 2k+1).
 * level == 0xffffffff marks an unused slot. */
typedef struct {
    uint32_t level;
    uint32_t reserved;
    uint64_t index;
    double hi_re, lo_re, hi_im, lo_im;
} perm_tree_node_t;
#define PERM_TREE_MAX_NODES 128

typedef enum {
    PERM_OK = 0,
    PERM_E_ARG = 1,        /* null required pointer, negative count, k_begin > k_end, bad workspace size */
    PERM_E_ORDER = 2,      /* n < 1, n > 64 (complex), n > 33 (int01, pm1), k_end > 2^{n-1}           */
    PERM_E_NONFINITE = 3,  /* a NaN/Inf matrix entry (perm_c128 / perm_c128_range)                       */
    PERM_E_NOT01 = 4,      /* a byte other than 0 or 1 (perm_int01)                                      */
    PERM_E_CUDA = 5,       /* a CUDA runtime call failed; see perm_last_error()                         */
    PERM_E_WORKSPACE = 6,  /* workspace smaller than perm_workspace_bytes()                             */
    PERM_E_CHECK = 7       /* int01 self-check failed: raw Glynn sum not divisible by 2^{n-1}           */
} perm_status_t;

/* ------------------------------------------------------------------------------------------
 * Single matrix (BASELINE configs 1, 4, 5).
 * ------------------------------------------------------------------------------------------ */

/* Scratch bytes needed by perm_c128 / perm_c128_range for order n and rank range [k_begin, k_end)
 * (one 32-byte dd partial per walked chunk plus the reduction tree: for a whole permanent
 * 2^{n-1-b} * 32 bytes, b = perm_chunk_log2(n) -- 1 GiB at n = 44). */
perm_status_t perm_workspace_bytes(int n, uint64_t k_begin, uint64_t k_end, size_t* bytes);

/* The chunk length 2^b a whole permanent of order n is walked in (perm_c128, and the default of the
 * chunk walk below): a function of n alone, so the result never depends on the grid, the number of GPUs
 * or the slicing.  -1 if n is outside 1..64. */
int perm_chunk_log2(int n);

/* per(A) of one n x n complex matrix, 1 <= n <= 64 (ranks are 64-bit words).
 *   A          host or device, n*n perm_c128_t, row-major, read only, all entries finite.
 *   out        host or device, one perm_c128_t: per(A) = 2(-1)^n P(0, 2^{n-1}) rounded from dd.
 *   out_dd     optional (may be NULL), host or device: the dd value of per(A) before rounding.
 *   workspace  device scratch of >= perm_workspace_bytes(n, 0, 2^{n-1}) bytes, or NULL.
 *   stats      optional host struct (may be NULL).
 * The 2^{n-1} ranks are walked as 2^{n-1-b} aligned chunks of 2^b ranks (b = perm_chunk_log2(n)), each
 * seeded explicitly (App. A steps 5-8); the chunks' dd partials are combined by the canonical
 * pairwise tree (perm_c128_tree), so the value is bit-identical to the chunk walk + tree + combine below
 * over ANY split of the chunks into launches or GPUs.
 * A non-finite entry: PERM_E_NONFINITE when `out` / `out_dd` are host memory; with device outputs (no host
 * synchronization) a device-resident A is checked by the kernel and the outputs become NaN.
 * Errors: PERM_E_ARG (A or out NULL), PERM_E_ORDER, PERM_E_NONFINITE, PERM_E_WORKSPACE, PERM_E_CUDA.
 * Cite: problem P:56-59; method App. A P:1126-1163 (subpermanent + permanent). */
perm_status_t perm_c128(const perm_c128_t* A, int n, perm_c128_t* out, perm_dd_c128_t* out_dd,
                        void* workspace, size_t workspace_bytes, void* stream, perm_stats_t* stats);

/* Raw partial P(k_begin, k_end) over the Gray ranks [k_begin, k_end) subset of [0, 2^{n-1}),
 * WITHOUT the 2(-1)^n factor: App. A subpermanent for the rank span that
 * distribute hands one worker.  Used to shard one permanent over GPUs/processes;
 * any split of [0, 2^{n-1}) into spans combined by perm_c128_finalize gives per(A) (up to rounding;
 * for bit-identity across splits use the chunk walk + tree above).  The span is cut into maximal aligned
 * pieces (chunks of 2^b ranks, b chosen from the span and the device, plus single ranks at unaligned
 * ends); their dd partials are combined by the canonical tree over the piece index.
 *   partial    host or device, one perm_dd_c128_t.  k_begin == k_end gives 0.
 * Errors: as perm_c128, plus PERM_E_ORDER if k_end > 2^{n-1}, PERM_E_ARG if k_begin > k_end. */
perm_status_t perm_c128_range(const perm_c128_t* A, int n, uint64_t k_begin, uint64_t k_end,
                              perm_dd_c128_t* partial, void* workspace, size_t workspace_bytes,
                              void* stream, perm_stats_t* stats);

/* ------------------------------------------------------------------------------------------
 * The chunk walk and its canonical reduction: one permanent split over launches / steps / GPUs
 * (App. A distribute P:1077-1095, subpermanent P:1133-1151, step 4 P:1162;
 * "partial sums ... stored in an array before the final summation").
 * ------------------------------------------------------------------------------------------ */

/* Walks the aligned chunks c in [c_begin, c_end) of 2^chunk_log2 ranks each (ranks [c 2^b, (c+1) 2^b))
 * and writes chunk c's raw dd partial sum_{r in chunk} (-1)^{r+1} prod_i w_i(gray r) to
 * partials_dev[c - c_begin].  A chunk's partial depends only on (A, n, b, c): the seed is recomputed from
 * gray(c 2^b) and the accumulator starts at zero.
 *   A            host or device, n*n perm_c128_t row-major (a device A is copied back once and checked).
 *   chunk_log2   b: 0 or U(n) <= b <= min(n-1, 30) (U(n) = 3 for 4 <= n <= 33, 2 for most larger n;
 *                perm_chunk_log2(n) always qualifies).
 *   partials_dev device, (c_end - c_begin) perm_dd_c128_t.  c_end <= 2^{n-1-b}.
 *   workspace    device, >= n*n*16 bytes when A is host memory (the H2D copy of A), else unused; NULL =
 *                allocated stream-ordered.
 * Stream-ordered when A is host memory (no synchronization); a device A is synchronized once.
 * Errors: PERM_E_ARG (NULL, c_begin > c_end, bad b, partials not device), PERM_E_ORDER, PERM_E_NONFINITE,
 *         PERM_E_WORKSPACE, PERM_E_CUDA. */
perm_status_t perm_c128_chunks(const perm_c128_t* A, int n, int chunk_log2, uint64_t c_begin, uint64_t c_end,
                               perm_dd_c128_t* partials_dev, void* workspace, size_t workspace_bytes, void* stream,
                               perm_stats_t* stats);

/* Chunk walkers one perm_c128_chunks launch of order n and chunk length 2^chunk_log2 keeps resident on
 * the current device (grid x walkers per block): a span of k * walkers chunks leaves no partial last round
 * of the static round-robin (bench.py slices one permanent into steps of whole rounds).
 * Errors: PERM_E_ARG (NULL), PERM_E_ORDER, PERM_E_CUDA. */
perm_status_t perm_chunk_walkers(int n, int chunk_log2, uint64_t* walkers);

/* Scratch bytes of perm_c128_tree for `count` partials. */
perm_status_t perm_tree_workspace_bytes(uint64_t count, size_t* bytes);

/* Reduces the chunk partials of [c_begin, c_end) (partials_dev[i] = chunk c_begin + i) by the canonical
 * binary tree over ABSOLUTE chunk indices to the span's maximal complete nodes (at most two per level),
 * sorted by position, in `nodes` (PERM_TREE_MAX_NODES slots, unused ones marked level = 0xffffffff), and
 * optionally their left-to-right dd sum in `raw` (the span's raw partial).  nodes / raw: host or device
 * (either may be NULL, not both).  Synchronizes if an output is host memory.
 * Errors: PERM_E_ARG, PERM_E_WORKSPACE, PERM_E_CUDA. */
perm_status_t perm_c128_tree(const perm_dd_c128_t* partials_dev, uint64_t c_begin, uint64_t c_end,
                             perm_tree_node_t* nodes, perm_dd_c128_t* raw, void* workspace, size_t workspace_bytes,
                             void* stream);

/* Host only: merges the nodes of disjoint spans (e.g. every GPU's perm_c128_tree output, in any order;
 * unused slots are skipped): sibling nodes combine left + right until none remain, the rest are summed
 * left to right.  raw receives the result; *root_level (optional) the level L if the nodes merged into
 * the single node covering chunks [0, 2^L), else -1.  With the chunks of a whole permanent
 * (L = n-1-b) raw is bit-identical to perm_c128's, and perm_c128_finalize(raw, 1, n) gives per(A).
 * Errors: PERM_E_ARG (NULL raw, count < 0, overlapping or invalid nodes). */
perm_status_t perm_c128_tree_combine(const perm_tree_node_t* nodes, int count, perm_dd_c128_t* raw, int* root_level);

/* Host-only: out = 2(-1)^n * sum_{k=0}^{count-1} partials[k], summed in index order in double-double
 * (App. A permanent step 4; "stored in an array before the final ... summation").
 *   partials   host, count perm_dd_c128_t.   out   host.   out_dd optional host.
 * Errors: PERM_E_ARG (NULL, count < 0), PERM_E_ORDER (n outside 1..64). */
perm_status_t perm_c128_finalize(const perm_dd_c128_t* partials, int count, int n, perm_c128_t* out,
                                 perm_dd_c128_t* out_dd);

/* ------------------------------------------------------------------------------------------
 * Batch of small complex matrices (BASELINE config 2: Boson-sampling probabilities).
 * ------------------------------------------------------------------------------------------ */

/* per and |per|^2 of B independent n x n complex matrices, 1 <= n <= 32.
 *   A_dev      device, B*n*n perm_c128_t, matrix b at A_dev + b*n*n (row-major).
 *   per_dev    device, B perm_c128_t, or NULL.       abs2_dev   device, B doubles |per|^2, or NULL.
 * Stream-ordered: returns after enqueueing.  B == 0 is a no-op.  Non-finite entries are not
 * checked; they propagate to NaN/Inf in that matrix's outputs only.
 * Errors: PERM_E_ARG (A_dev NULL, B < 0, both outputs NULL), PERM_E_ORDER, PERM_E_CUDA.
 * Cite: P:954-958 (submatrices of a Haar unitary), P:1126-1163 (method per matrix). */
perm_status_t perm_c128_batched(const perm_c128_t* A_dev, int n, int64_t B, perm_c128_t* per_dev,
                                double* abs2_dev, void* stream);

/* The same, plus the ensemble statistic of Secs. IV-V, X_b = |per(A_b)| / sqrt(n!), for
 * streaming random-matrix ensembles (Ginibre, circular, Haar minors: E[X^2] = 1 for Ginibre and circular):
 *   x_dev      device, B doubles X_b = sqrt(|per_b|^2 / n!) (n! rounded to binary64), or NULL.
 * At least one of per_dev, abs2_dev, x_dev must be non-NULL.  Otherwise as perm_c128_batched. */
perm_status_t perm_c128_batched_x(const perm_c128_t* A_dev, int n, int64_t B, perm_c128_t* per_dev,
                                  double* abs2_dev, double* x_dev, void* stream);

/* ------------------------------------------------------------------------------------------
 * Sparse matrices: restricted enumeration (App. B; Sec. II-D; NEXT-3).
 * ------------------------------------------------------------------------------------------ */

/* The column partition D = {S_1, ..., S_d, T} of greedypartition (repeatedly take the
 * remaining row k of least out-degree, the lowest index on ties; S = the columns where row k is
 * nonzero; drop the remaining rows whose supports meet S), and the enumeration size
 * sets = 2^{|T|} prod_l (2^{|S_l|} - 1). */
typedef struct {
    uint32_t d;          /* number of S sets */
    uint32_t nt;         /* |T| */
    uint64_t tmask;      /* columns of T (bit j = column j) */
    uint64_t smask[64];  /* columns of S_1 .. S_d */
    double sets;         /* sets J enumerated (0 when a zero row or column makes per = 0) */
    int32_t chunk_log2;  /* T-walk chunk length used by perm_c128_sparse (-1: not launched) */
    int32_t group_cols;  /* perm_c128_sparse: 0 = the plain T walk; G > 0 = the shared-rows group walk: G T
                            columns nonzero in <= 4 rows together are the walk's lowest Gray bits, and each
                            block of 2^G sets shares the product of the other rows */
} perm_sparse_info_t;

/* Host only: the partition and enumeration size for A (host, row-major n x n, 1 <= n <= 64).
 * Errors: PERM_E_ARG (NULL), PERM_E_ORDER, PERM_E_NONFINITE. */
perm_status_t perm_sparse_plan(const perm_c128_t* A_host, int n, perm_sparse_info_t* info);

/* per(A) by sparsepermanent over the partition of perm_sparse_plan: every set J that
 * meets each S_l, t-part walked in Gray order on the GPU, signed sum in double-double, (-1)^n applied.
 * Exactly Eq. (3) (every skipped J has a zero row sum).  A is host or device (row-major), 1 <= n <= 48;
 * out_host host; info optional; scratch is allocated stream-ordered.  Synchronizes `stream`.
 * Errors: PERM_E_ARG, PERM_E_ORDER, PERM_E_NONFINITE, PERM_E_CUDA. */
perm_status_t perm_c128_sparse(const perm_c128_t* A, int n, perm_c128_t* out_host, perm_sparse_info_t* info,
                               void* stream);

/* ------------------------------------------------------------------------------------------
 * Matrices of limited bandwidth: App. C transfer method (NEXT-4).
 * ------------------------------------------------------------------------------------------ */

/* per and |per|^2 of B matrices of bandwidth k (a_ij = 0 for |i - j| > k) in O(n C(2k,k) (k+1)) work
 * each: App. C's polynomial bookkeeping (x_j^2 = 0, x_j := 1 once column j leaves the band) as a
 * transfer matrix over the used columns of the sliding window.
 *   A_dev      device, band storage B*n*(2k+1) perm_c128_t: A_dev[(b*n + i)*(2k+1) + d] = a_{i, i-k+d};
 *              entries whose column i-k+d lies outside 0..n-1 are not read.
 *   per_dev    device, B perm_c128_t, or NULL.       abs2_dev   device, B doubles, or NULL.
 * 1 <= n <= 2^20, 0 <= k <= min(6, n-1).  Stream-ordered; B == 0 is a no-op.
 * Errors: PERM_E_ARG (NULL input, B < 0, k out of range, both outputs NULL), PERM_E_ORDER, PERM_E_CUDA. */
perm_status_t perm_c128_band_batched(const perm_c128_t* A_dev, int n, int k, int64_t B, perm_c128_t* per_dev,
                                     double* abs2_dev, void* stream);

/* ------------------------------------------------------------------------------------------
 * Repeated columns: the weighted Ryser formula, Eq. (4).
 * ------------------------------------------------------------------------------------------ */

/* per and |per|^2 of B matrices with repeated columns, each given by its R distinct columns and their
 * multiplicities (Boson-sampling output patterns with collisions):
 *     per(A) = (-1)^n sum_{0<=f_k<=m_k} (-1)^{sum f} prod_k C(m_k, f_k) prod_i sum_k f_k cbar_i(k),
 * prod_k (m_k + 1) terms instead of 2^{n-1}, walked in reflected mixed-radix Gray order.
 *   C_dev      device, B*n*R perm_c128_t; problem b's distinct columns at C_dev + b*n*R, row-major
 *              n x R (entry (i, k) = cbar_i(k)).
 *   mult_dev   device, B*R int32 multiplicities m_k >= 0 with sum_k m_k == n (zeros allowed, so one R
 *              serves a batch of patterns with different numbers of distinct modes).
 *   per_dev    device, B perm_c128_t, or NULL.       abs2_dev   device, B doubles |per|^2, or NULL.
 * 1 <= n <= 32, 1 <= R <= 64.  Stream-ordered: returns after enqueueing.  B == 0 is a no-op.  A problem
 * whose multiplicities are invalid (negative, > n, or not summing to n) gets NaN outputs; non-finite
 * entries propagate to that problem's outputs only.
 * Errors: PERM_E_ARG (NULL input, B < 0, R outside 1..64, both outputs NULL), PERM_E_ORDER, PERM_E_CUDA. */
perm_status_t perm_c128_weighted_batched(const perm_c128_t* C_dev, const int32_t* mult_dev, int n, int R,
                                         int64_t B, perm_c128_t* per_dev, double* abs2_dev, void* stream);

/* ------------------------------------------------------------------------------------------
 * Exact permanents of 0-1 matrices (BASELINE config 3; #P-hard even for 0-1).
 * ------------------------------------------------------------------------------------------ */

/* Scratch bytes needed by perm_int01 for B matrices of order n. */
perm_status_t perm_int01_workspace_bytes(int n, int64_t B, size_t* bytes);

/* Exact per(A) of B 0-1 matrices, 1 <= n <= 33, as int128.  n <= 28: integer Glynn sums g_i = 2 w_i are
 * walked in Gray order; products and the signed sum are exact mod 2^128, per = (-1)^n Sum / 2^{n-1} is
 * exact (n! 2^{n-1} < 2^127), and the low n-1 bits of Sum are checked to be zero.  29 <= n <= 33: the
 * same walk over all 2^n subsets of Eq. (3), Sum = (-1)^{n+1} per, exact while n! < 2^127.
 * 20 <= n <= 24: each matrix is walked with the Gray column holding the most zeros first and its zero rows
 * first (per is invariant under row/column permutations), consecutive term pairs factored over those rows
 * (DESIGN.md 5.3); the result is the same exact integer.
 *   A_dev     device, B*n*n bytes, each 0 or 1, row-major.
 *   out_dev   device, B perm_i128_t.
 * Synchronizes `stream` (to report PERM_E_NOT01 / PERM_E_CHECK).
 * Errors: PERM_E_ARG, PERM_E_ORDER, PERM_E_NOT01 (outputs unspecified), PERM_E_CHECK, PERM_E_WORKSPACE,
 *         PERM_E_CUDA. */
perm_status_t perm_int01(const uint8_t* A_dev, int n, int64_t B, perm_i128_t* out_dev,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Exact per(A) of B matrices with entries in {-1, 0, 1} -- the Bernoulli +-1 ensemble of Sec. V
 * -- by the same integer walks as perm_int01 (|g_i| <= n, so the
 * same n <= 33 range).  Same workspace (perm_int01_workspace_bytes), outputs and errors as
 * perm_int01; PERM_E_NOT01 here means an entry outside {-1, 0, 1}.
 *   A_dev     device, B*n*n signed bytes, row-major. */
perm_status_t perm_pm1(const int8_t* A_dev, int n, int64_t B, perm_i128_t* out_dev,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Sharding ONE exact 0-1 permanent (App. A partition): the
 * raw signed integer Gray sum over the ranks [k_begin, k_end) of the Gray walk of A AS GIVEN (Gray bit j =
 * column j; perm_int01 itself may walk a row- and column-permuted copy, DESIGN.md 5.3 -- same total),
 *     n <= 28:       P = sum_{r} (-1)^{r+1} prod_i g_i(gray r)   (half range, ranks < 2^{n-1})
 *     29 <= n <= 33: P = sum_{r} (-1)^{|gray r|} prod_i r_i(gray r)   (Eq. (3), ranks < 2^n)
 * modulo 2^128 (the exact value's two's-complement bits).  Partials of disjoint spans add exactly (mod
 * 2^128, in any order); perm_int01_finalize turns their sum into per(A).
 *   A_dev     device, n*n bytes, each 0 or 1, row-major.
 *   partial   host, one perm_i128_t (raw bits mod 2^128).
 * Synchronizes `stream`.  Workspace is allocated internally (stream-ordered).
 * Errors: PERM_E_ARG (null pointer, k_begin > k_end), PERM_E_ORDER (n outside 1..33, k_end beyond the
 *         rank space), PERM_E_NOT01, PERM_E_CUDA.  k_begin == k_end gives 0. */
perm_status_t perm_int01_range(const uint8_t* A_dev, int n, uint64_t k_begin, uint64_t k_end,
                               perm_i128_t* partial, void* stream);

/* per(A) from the partials of spans covering the whole rank space exactly once (host only): their sum
 * mod 2^128 is Sum; n <= 28: per = (-1)^n Sum / 2^{n-1} after checking the low n-1 bits are zero
 * (PERM_E_CHECK otherwise); 29 <= n <= 33: per = (-1)^{n+1} Sum.
 *   partials  host, count perm_i128_t;  out  host, one perm_i128_t.
 * Errors: PERM_E_ARG (null pointer, count < 0), PERM_E_ORDER, PERM_E_CHECK. */
perm_status_t perm_int01_finalize(const perm_i128_t* partials, int count, int n, perm_i128_t* out);

/* ------------------------------------------------------------------------------------------
 * Diagnostics.
 * ------------------------------------------------------------------------------------------ */

/* w(r) of App. A steps 2, 5-8 for ranks r_k = chunk-aligned starts, computed by the
 * device seeding code: w_out (host or device) receives count*n perm_c128_t, w(ranks[k]) at
 * w_out + k*n.  ranks: host array of count uint64 ranks < 2^{n-1}.  Synchronizes if w_out is host. */
perm_status_t perm_c128_seed(const perm_c128_t* A, int n, const uint64_t* ranks, int count,
                             perm_c128_t* w_out, void* stream);

/* FP64 peak probe: each of blocks x threads threads runs `iters` iterations of 32 DFMA
 * (8 independent dependent chains), i.e. 64 * iters flops per thread.  Writes a checksum to sink_dev
 * (device, blocks*threads doubles).  Stream-ordered. */
perm_status_t perm_fp64_probe(int blocks, int threads, int iters, double* sink_dev, void* stream);

/* Number of kernels enqueued by this thread's last successful call (for launch accounting). */
uint32_t perm_last_launches(void);

const char* perm_status_string(perm_status_t status);
const char* perm_last_error(void);
int perm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PERM_H_ */
