"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO permanent arithmetic.  It is the one module that both the
CUDA path's callers (bench.py, tests) and the oracle's callers draw inputs from,
so that both sides read identical bytes.  Recipe:

* complex Gaussian entries (g1 + i g2)/sqrt(2), g ~ N(0,1): re, im ~ N(0, 1/2)
  (Ginibre ensemble);
* Haar unitary U(m): QR of a complex Gaussian matrix, then U = Q * diag(r_ii/|r_ii|)
  (P:944-952);
* Boson-sampling submatrices: distinct rows and distinct columns drawn uniformly,
  sorted (P:954-958 with m = n^2, i.e. a = 2 of Sec. VI);
* Bernoulli(1/2) 0-1 matrices.

numpy's PCG64 (default_rng) with the seeds of SURVEY.md 8(d).
"""
from __future__ import annotations

import numpy as np

SEEDS = {"cfg1": 16, "cfg2_u": 2000, "cfg2_idx": 3000, "cfg3": 24, "cfg4": 1024, "cfg5": 44, "cfgw": 2424, "cfgpm": 2425, "cfgsp": 4848, "cfgbd": 1005,
         "cfgens_g": 2024, "cfgens_c": 3024}


def complex_gaussian(shape, seed: int | np.random.Generator) -> np.ndarray:
    """(g1 + i g2)/sqrt(2): real block drawn first, then imaginary block."""
    rng = np.random.default_rng(seed) if not isinstance(seed, np.random.Generator) else seed
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return np.ascontiguousarray((re + 1j * im) / np.sqrt(2.0))


def haar_unitary(m: int, seed: int | np.random.Generator) -> np.ndarray:
    """Haar-random m x m unitary: Q R = Z, U = Q diag(r_ii / |r_ii|)."""
    Z = complex_gaussian((m, m), seed)
    # single-threaded LAPACK: the bits of Q must not depend on the process's thread count (torchrun sets
    # OMP_NUM_THREADS=1, a plain run does not) -- bench results are compared bitwise across launches
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        Q, R = np.linalg.qr(Z)
    d = np.diag(R)
    return np.ascontiguousarray(Q * (d / np.abs(d))[None, :])


def submatrix_indices(m: int, n: int, count: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """count pairs (rows, cols) of n distinct sorted indices in [0, m), in sample order."""
    rng = np.random.default_rng(seed)
    rows = np.empty((count, n), dtype=np.int64)
    cols = np.empty((count, n), dtype=np.int64)
    for s in range(count):
        rows[s] = np.sort(rng.choice(m, n, replace=False))
        cols[s] = np.sort(rng.choice(m, n, replace=False))
    return rows, cols


def gather_submatrices(U: np.ndarray, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """(count, n, n) complex128 with out[s] = U[rows[s]][:, cols[s]]."""
    return np.ascontiguousarray(U[rows[:, :, None], cols[:, None, :]])


def bernoulli01(shape, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.integers(0, 2, size=shape, dtype=np.uint8))


def zero_column01(n: int, z: int, seed: int, p_one: float = 0.7, col: int | None = None) -> np.ndarray:
    """An n x n 0-1 matrix (Bernoulli(p_one) entries) whose column `col` (default: a seeded choice among the
    first n-1) holds exactly z zeros and every other column fewer than z -- test inputs that fix the largest
    zero count of a column (the int01 pair-factored walk's plan)."""
    rng = np.random.default_rng(seed)
    A = (rng.random((n, n)) < p_one).astype(np.uint8)
    if col is None:
        col = int(rng.integers(0, max(1, n - 1)))
    A[:, col] = 1
    A[rng.choice(n, z, replace=False), col] = 0
    for j in range(n):
        if j == col:
            continue
        zr = np.flatnonzero(A[:, j] == 0)
        if len(zr) >= z:
            A[rng.choice(zr, len(zr) - z + 1, replace=False), j] = 1
    return np.ascontiguousarray(A)


# ---------------------------------------------------------------- the 5 configs

def cfg1() -> np.ndarray:
    """Single 16x16 complex Gaussian (BASELINE.json configs[0])."""
    return complex_gaussian((16, 16), SEEDS["cfg1"])


def cfg2(n: int, count: int = 100_000) -> np.ndarray:
    """(count, n, n) submatrices of an n^2 x n^2 Haar unitary (configs[1])."""
    m = n * n
    U = haar_unitary(m, SEEDS["cfg2_u"] + n)
    rows, cols = submatrix_indices(m, n, count, SEEDS["cfg2_idx"] + n)
    return gather_submatrices(U, rows, cols)


def cfg3(batch: int = 64, n: int = 24) -> np.ndarray:
    """(64, 24, 24) Bernoulli(1/2) 0-1 matrices (configs[2])."""
    return bernoulli01((batch, n, n), SEEDS["cfg3"])


def cfg4() -> np.ndarray:
    """Leading 32x32 block of a 1024x1024 Haar unitary (configs[3])."""
    U = haar_unitary(1024, SEEDS["cfg4"])
    return np.ascontiguousarray(U[:32, :32])


def cfg5() -> np.ndarray:
    """Single 44x44 complex Gaussian (configs[4])."""
    return complex_gaussian((44, 44), SEEDS["cfg5"])


# ---------------------------------------------------------------- structured inputs

def block_diag_scrambled(B1: np.ndarray, B2: np.ndarray, seed: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """P (B1 (+) B2) Q with random permutations P, Q.  Returns (M, row_perm, col_perm)."""
    n1, n2 = B1.shape[0], B2.shape[0]
    n = n1 + n2
    M = np.zeros((n, n), dtype=np.complex128)
    M[:n1, :n1] = B1
    M[n1:, n1:] = B2
    rng = np.random.default_rng(seed)
    rp = rng.permutation(n)
    cp = rng.permutation(n)
    return np.ascontiguousarray(M[rp][:, cp]), rp, cp


def ones(n: int) -> np.ndarray:
    return np.ones((n, n), dtype=np.complex128)


# ---------------------------------------------------------------- repeated columns (Eq. (4), NEXT-1)

def collision_patterns(n: int, m: int, count: int, seed: int, R: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Boson-sampling output patterns WITH collisions: n photons enter the first n modes of an m-mode
    Haar unitary U (seed); each pattern sends them to n output modes drawn uniformly WITH replacement
    (sorted).  Returns C (count, n, R) complex128 -- the distinct output columns U[:n, mode] in
    increasing mode order, zero-padded -- and mult (count, R) int32 -- their multiplicities, zero-padded;
    R defaults to n.  Rows = input modes, columns = output modes."""
    R = n if R is None else R
    rng = np.random.default_rng(seed)
    U = haar_unitary(m, rng)
    C = np.zeros((count, n, R), dtype=np.complex128)
    mult = np.zeros((count, R), dtype=np.int32)
    for s in range(count):
        modes, counts = np.unique(rng.integers(0, m, size=n), return_counts=True)
        C[s, :, :len(modes)] = U[:n, modes]
        mult[s, :len(modes)] = counts
    return C, mult


def cfgw(count: int = 10_000) -> tuple[np.ndarray, np.ndarray]:
    """Weighted-Ryser workload (not a BASELINE config): 20 photons into the 20 modes
    of a Haar unitary, output modes drawn uniformly with replacement -- collision-rich patterns
    (about 13 distinct modes each).  C (count, 20, 20), mult (count, 20)."""
    return collision_patterns(20, 20, count, SEEDS["cfgw"])


# ---------------------------------------------------------------- ensembles of Secs. III-VI (NEXT-2)

def bernoulli_pm1(shape, seed: int) -> np.ndarray:
    """Bernoulli +-1 entries, Pr(+1) = Pr(-1) = 1/2 (Sec. V), as int8."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray((2 * rng.integers(0, 2, size=shape) - 1).astype(np.int8))


def circular(shape, seed: int | np.random.Generator) -> np.ndarray:
    """Complex circular entries exp(i theta), theta uniform on [0, 2 pi) (Sec. IV)."""
    rng = np.random.default_rng(seed)
    theta = rng.uniform(0.0, 2.0 * np.pi, size=shape)
    return np.ascontiguousarray(np.exp(1j * theta))


def cfgens(count: int = 10_000, n: int = 24) -> tuple[np.ndarray, np.ndarray]:
    """The ensemble workload: `count` Ginibre matrices and `count` circular matrices of
    order n (Secs. III-IV collect 10^7 of each for n <= 30; this is a bounded batch of the same shape)."""
    return (complex_gaussian((count, n, n), SEEDS["cfgens_g"]), circular((count, n, n), SEEDS["cfgens_c"]))


def haar_minors(n: int, a: float, count: int, seed: int) -> np.ndarray:
    """(count, n, n) submatrices with distinct sorted rows and columns of an m x m Haar unitary,
    m = round(n^a) (the minors S(n^a, n) of Sec. VI; a = 2 is config 2)."""
    m = int(round(n ** a))
    rng = np.random.default_rng(seed)
    U = haar_unitary(m, rng)
    rows = np.empty((count, n), dtype=np.int64)
    cols = np.empty((count, n), dtype=np.int64)
    for s in range(count):
        rows[s] = np.sort(rng.choice(m, n, replace=False))
        cols[s] = np.sort(rng.choice(m, n, replace=False))
    return gather_submatrices(U, rows, cols)


# ---------------------------------------------------------------- sparse matrices (App. B, NEXT-3)

def sparse_gaussian(n: int, density: float, seed: int) -> np.ndarray:
    """Sparse complex Gaussian matrix: each entry nonzero with probability `density`, plus a random
    perfect matching (so no row or column is empty and per != 0 generically) -- the low-depth
    Boson-sampling shape of Sec. II-D.  Nonzero entries (g1 + i g2)/sqrt(2)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    M = mask * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2.0)
    M[np.arange(n), rng.permutation(n)] += (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2.0)
    return np.ascontiguousarray(M)


def cfgsp() -> np.ndarray:
    """Sparse workload (not a BASELINE config): n = 48, density 4% + a matching
    (about 2.8 nonzeros per row; the paper's sparse code stops gaining above ~5%):
    1.8e11 restricted sets instead of 2^47 = 1.4e14 Gray terms."""
    return sparse_gaussian(48, 0.04, SEEDS["cfgsp"])


# ---------------------------------------------------------------- bandwidth-limited matrices (App. C, NEXT-4)

def band_gaussian(shape, k: int, seed: int) -> np.ndarray:
    """(B, n) -> (B, n, n) complex Gaussian matrices of bandwidth k (a_ij = 0 for |i - j| > k), the
    band-limited Boson-sampling shape of Sec. II-D."""
    B, n = shape
    A = complex_gaussian((B, n, n), seed)
    i, j = np.indices((n, n))
    A[:, np.abs(i - j) > k] = 0
    return np.ascontiguousarray(A)


def cfgbd(count: int = 10_000) -> np.ndarray:
    """Band-limited workload (not a BASELINE config): count complex Gaussian matrices of
    order 100 and bandwidth 5 (the largest case of the paper's App. C timing figure)."""
    return band_gaussian((count, 100), 5, SEEDS["cfgbd"])
