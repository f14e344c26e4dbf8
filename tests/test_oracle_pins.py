"""Pins for the CPU oracle (oracle/oracle.c): each check ties an oracle function to
something other than itself -- brute force, closed forms, the App. A hand trace,
or an algebraic identity of the permanent.  CPU only."""
from __future__ import annotations

import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_1904_06229_b200 import inputs
from tests import pins

COMPLEX_FNS = {
    "naive": lambda A: oracle.naive(A).value,
    "ryser": lambda A: oracle.ryser(A).value,
    "permanent_hr": lambda A: oracle.permanent_hr(A).value,
    "permanent_hr_m1": lambda A: oracle.permanent_hr(A, m=1).value,
}


def _close(a, b, tol=1e-13, scale=None):
    s = max(abs(b), 1e-300) if scale is None else scale
    return abs(a - b) <= tol * s


# ------------------------------------------------------------------ integer helpers

def test_distribute_examples():
    # SPEC examples, App. A distribute P:1086-1093
    assert oracle.distribute(10, 3, 0) == (0, 4)
    assert oracle.distribute(10, 3, 2) == (7, 3)
    assert oracle.distribute(5, 1, 0) == (0, 5)


@pytest.mark.parametrize("total,m", [(10, 3), (7, 7), (3, 5), (1 << 20, 148 * 7), (1000003, 64), (0, 4)])
def test_distribute_partition(total, m):
    spans = [oracle.distribute(total, m, i) for i in range(m)]
    pos = 0
    for k, l in spans:
        assert k == pos
        pos += l
    assert pos == total
    ls = [l for _, l in spans]
    assert max(ls) - min(ls) <= 1


def test_gray_examples():
    assert oracle.gray(0) == 0
    assert oracle.gray(5) == 7
    assert oracle.gray(4) == 6
    for r in range(1, 1 << 12):
        d = oracle.gray(r) ^ oracle.gray(r - 1)
        assert d & (d - 1) == 0 and d != 0          # one bit flips per step
    assert sorted(oracle.gray(r) for r in range(1 << 10)) == list(range(1 << 10))


# ------------------------------------------------------------------ naive (Eq. 1) pins

def test_naive_hand_values():
    assert oracle.naive([[1, 2], [3, 4]]).value == 10
    assert oracle.naive(np.eye(3)).value == 1
    assert oracle.naive(np.ones((4, 4))).value == 24
    assert oracle.naive([[5 + 1j]]).value == 5 + 1j           # n = 1
    a, b, c, d = 1.5 + 2j, -0.25 + 1j, 3 - 1j, 0.5 + 0.5j
    assert oracle.naive([[a, b], [c, d]]).value == a * d + b * c


def test_naive_brute_force_python():
    # brute force written out with itertools.permutations + Fraction (exact) on a small integer matrix
    rng = np.random.default_rng(1)
    for n in range(1, 7):
        A = rng.integers(-5, 6, size=(n, n))
        ref = sum(math.prod(int(A[i, p[i]]) for i in range(n)) for p in itertools.permutations(range(n)))
        assert oracle.naive(A.astype(np.complex128)).value == ref


# ------------------------------------------------------------------ shared pins for every complex oracle

@pytest.mark.parametrize("fn", list(COMPLEX_FNS))
def test_all_ones_factorial(fn):
    nmax = 8 if fn == "naive" else 18
    for n in range(1, nmax + 1):
        assert COMPLEX_FNS[fn](np.ones((n, n))) == math.factorial(n), n


@pytest.mark.parametrize("fn", list(COMPLEX_FNS))
def test_identity_diag_derangement(fn):
    nmax = 8 if fn == "naive" else 16
    rng = np.random.default_rng(7)
    for n in range(1, nmax + 1):
        assert COMPLEX_FNS[fn](np.eye(n)) == 1
        d = (rng.integers(1, 5, size=n) + 1j * rng.integers(-3, 4, size=n)).astype(np.complex128)
        assert COMPLEX_FNS[fn](np.diag(d)) == np.prod(d)
        assert COMPLEX_FNS[fn](pins.j_minus_i(n).astype(np.complex128)) == pins.derangements(n)


@pytest.mark.parametrize("fn", ["ryser", "permanent_hr", "permanent_hr_m1"])
def test_against_naive_random_complex(fn):
    for n in range(1, 9):
        A = inputs.complex_gaussian((n, n), 100 + n)
        ref = oracle.naive(A).value
        got = COMPLEX_FNS[fn](A)
        assert _close(got, ref, 1e-14, scale=max(abs(ref), pins.scaled_floor(A))), (n, got, ref)


@pytest.mark.parametrize("fn", ["ryser", "permanent_hr"])
def test_closed_forms_01_as_complex(fn):
    for n in range(3, 13):
        assert COMPLEX_FNS[fn](pins.tridiagonal_ones(n).astype(np.complex128)) == pins.fibonacci(n + 1)
        assert COMPLEX_FNS[fn](pins.hessenberg_ones(n).astype(np.complex128)) == 2 ** (n - 1)
        assert COMPLEX_FNS[fn](pins.identity_plus_shift(n).astype(np.complex128)) == 2
        assert COMPLEX_FNS[fn](pins.menage_matrix(n).astype(np.complex128)) == pins.menage(n)


@pytest.mark.parametrize("fn", ["ryser", "permanent_hr"])
def test_invariances_and_multilinearity(fn):
    f = COMPLEX_FNS[fn]
    rng = np.random.default_rng(3)
    for n in (5, 9, 12):
        A = inputs.complex_gaussian((n, n), 200 + n)
        p = f(A)
        sc = max(abs(p), pins.scaled_floor(A))
        assert _close(f(A.T.copy()), p, 1e-13, sc)
        P, Q = rng.permutation(n), rng.permutation(n)
        assert _close(f(A[P][:, Q].copy()), p, 1e-13, sc)
        # multilinearity in row i: per(row_i = alpha u + beta v) = alpha per(A_u) + beta per(A_v)
        i = int(rng.integers(n))
        u, v = inputs.complex_gaussian((2, n), 300 + n)
        al, be = 0.75 - 0.5j, -1.25 + 2j
        Au, Av, Aw = A.copy(), A.copy(), A.copy()
        Au[i], Av[i], Aw[i] = u, v, al * u + be * v
        lhs = f(Aw)
        rhs = al * f(Au) + be * f(Av)
        assert _close(lhs, rhs, 1e-12, max(abs(rhs), pins.scaled_floor(Aw)))


@pytest.mark.parametrize("fn", ["ryser", "permanent_hr"])
def test_rank_one_and_block_diag(fn):
    f = COMPLEX_FNS[fn]
    for n in (4, 7, 11):
        u = inputs.complex_gaussian((n,), 400 + n)
        v = inputs.complex_gaussian((n,), 500 + n)
        ref = math.factorial(n) * np.prod(u) * np.prod(v)        # per(u v^T) = n! prod u prod v
        assert _close(f(np.outer(u, v)), ref, 1e-12)
    B1 = inputs.complex_gaussian((5, 5), 11)
    B2 = inputs.complex_gaussian((6, 6), 12)
    M, _, _ = inputs.block_diag_scrambled(B1, B2, 13)
    ref = oracle.naive(B1).value * oracle.naive(B2).value
    assert _close(f(M), ref, 1e-13)
    # a zero row makes every product vanish exactly
    Z = inputs.complex_gaussian((9, 9), 14)
    Z[4] = 0
    assert f(Z) == 0


# ------------------------------------------------------------------ App. A hand trace (golden)

def test_app_a_trace(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "app_a_trace_n3.json")))
    A = np.array(g["A"], dtype=np.complex128)
    assert oracle.naive(A).value == g["per"]
    assert oracle.ryser(A).value == g["per"]
    assert oracle.permanent_hr(A, m=1).value == g["per"]
    assert oracle.permanent_hr(A, m=4).value == g["per"]
    for r, (seed, term) in enumerate(zip(g["seeds_num_den"], g["terms_num_den"])):
        w = oracle.seed(A, r)
        assert list(w) == [float(Fraction(a, b)) for a, b in seed]
        t = float(Fraction(*term))
        assert oracle.subpermanent(A, r, 1).value == t
        assert oracle.range_sum(A, r, r + 1).value == t
    S = float(Fraction(*g["S_num_den"]))
    assert oracle.subpermanent(A, 0, 4).value == S
    assert oracle.range_sum(A, 0, 4).value == S
    for k0 in range(5):
        for k1 in range(k0, 5):
            ref = sum(Fraction(*g["terms_num_den"][r]) for r in range(k0, k1))
            assert oracle.range_sum(A, k0, k1).value == float(ref)
            assert oracle.subpermanent(A, k0, k1 - k0).value == float(ref)


def test_subpermanent_par_pins(golden_dir):
    """oracle_subpermanent_par -- App. A's permanent loop restricted to a sub-range [r, r+l):
    the span cut by distribute into `parts` pieces walked on host threads, partials added in order.  Pinned
    (1) exactly on the dyadic n = 3 hand trace for every split of every span, (2) on random spans against
    range_sum, whose terms are re-derived from the definition per rank (no walk, no split), and the serial
    walk, for part counts that leave empty, single-rank and unaligned pieces."""
    g = json.load(open(os.path.join(golden_dir, "app_a_trace_n3.json")))
    A = np.array(g["A"], dtype=np.complex128)
    for parts in (1, 2, 3, 4, 7):
        for k0 in range(5):
            for k1 in range(k0, 5):
                ref = sum(Fraction(*g["terms_num_den"][r]) for r in range(k0, k1))
                assert oracle.subpermanent(A, k0, k1 - k0, parts=parts).value == float(ref), (parts, k0, k1)
    rng = np.random.default_rng(77)
    for n in (9, 20, 33):
        A = inputs.complex_gaussian((n, n), 700 + n)
        N = 1 << (n - 1)
        for _ in range(2):
            k0 = int(rng.integers(0, max(1, N - 2500)))
            k1 = min(N, k0 + int(rng.integers(1, 2500)))
            ref = oracle.range_sum(A, k0, k1).value
            ser = oracle.subpermanent(A, k0, k1 - k0).value
            for parts in (2, 3, 5, 16, 64, 4096):
                par = oracle.subpermanent(A, k0, k1 - k0, parts=parts).value
                assert _close(par, ref, 1e-20, scale=max(abs(ref), 1.0) * 1e3), (n, k0, k1, parts)
                assert _close(par, ser, 1e-20, scale=max(abs(ser), 1.0) * 1e3), (n, k0, k1, parts)


def test_n2_closed_form():
    # App. A at n = 2: S = (ad + bc)/2, per = ad + bc
    a, b, c, d = 1 + 2j, 3 - 1j, -2 + 0.5j, 0.25 + 4j
    A = np.array([[a, b], [c, d]])
    assert oracle.subpermanent(A, 0, 2).value == (a * d + b * c) / 2
    assert oracle.permanent_hr(A, m=1).value == a * d + b * c


# ------------------------------------------------------------------ range / seed / subpermanent consistency

def test_range_vs_walk_random_spans():
    rng = np.random.default_rng(5)
    for n in (6, 13, 20, 33):
        A = inputs.complex_gaussian((n, n), 600 + n)
        N = 1 << (n - 1)
        for _ in range(3):
            k0 = int(rng.integers(0, max(1, N - 3000)))
            k1 = min(N, k0 + int(rng.integers(1, 3000)))
            a = oracle.range_sum(A, k0, k1).value
            b = oracle.subpermanent(A, k0, k1 - k0).value
            assert _close(a, b, 1e-20, scale=max(abs(a), 1.0) * 1e3), (n, k0, k1)


def test_seed_matches_column_sums():
    # w(r) - w(0) = sum of the columns j < n-1 whose Gray bit is set
    A = inputs.complex_gaussian((7, 7), 9)
    w0 = oracle.seed(A, 0)
    assert np.allclose(w0, A[:, -1] - 0.5 * A.sum(axis=1), rtol=0, atol=1e-15)
    for r in (1, 5, 17, 63):
        x = oracle.gray(r)
        expect = w0 + sum(A[:, j] for j in range(6) if (x >> j) & 1)
        assert np.allclose(oracle.seed(A, r), expect, rtol=0, atol=1e-14)


def test_partition_invariance():
    A = inputs.complex_gaussian((15, 15), 15)
    ref = oracle.ryser(A).value
    sc = max(abs(ref), pins.scaled_floor(A))
    for m in (1, 2, 3, 7, 16, 1 << 14):
        assert _close(oracle.permanent_hr(A, m=m).value, ref, 1e-20, sc), m


def test_boson_sampling_normalization():
    # P13: for a unitary U (m x m) and fixed input rows S, |S| = n,
    # sum over output multisets T of |per(U_{S,T})|^2 / prod_j t_j! = 1.
    for (m, n) in ((4, 2), (9, 3)):
        U = inputs.haar_unitary(m, 77 + m)
        S = np.arange(n)
        mats, w = [], []
        for T in itertools.combinations_with_replacement(range(m), n):
            mats.append(U[np.ix_(S, list(T))])
            mult = np.bincount(np.array(T), minlength=m)
            w.append(1.0 / np.prod([math.factorial(int(k)) for k in mult]))
        per = oracle.ryser_batch(np.array(mats))
        assert abs(np.sum(np.abs(per) ** 2 * np.array(w)) - 1.0) < 1e-13


def test_gaussian_second_moment_statistical():
    # P15: E|per|^2 = n! for i.i.d. complex Gaussian entries with E|a|^2 = 1
    n, B = 5, 4000
    A = inputs.complex_gaussian((B, n, n), 4242)
    per = oracle.ryser_batch(A)
    m2 = np.mean(np.abs(per) ** 2)
    se = np.std(np.abs(per) ** 2) / np.sqrt(B)
    assert abs(m2 - math.factorial(n)) < 5 * se


# ------------------------------------------------------------------ integer oracle pins

def test_int_naive_vs_python_bruteforce():
    rng = np.random.default_rng(2)
    for n in range(1, 8):
        A = rng.integers(0, 2, size=(n, n), dtype=np.uint8)
        ref = sum(math.prod(int(A[i, p[i]]) for i in range(n)) for p in itertools.permutations(range(n)))
        assert oracle.naive_i01(A) == ref
        assert oracle.ryser_i01(A) == ref


def test_int_ryser_vs_naive_random():
    for n in range(1, 11):
        A = inputs.bernoulli01((n, n), 50 + n)
        assert oracle.ryser_i01(A) == oracle.naive_i01(A)


@pytest.mark.parametrize("n", [3, 8, 13, 20, 24])
def test_int_closed_forms(n):
    assert oracle.ryser_i01(np.ones((n, n), dtype=np.uint8)) == math.factorial(n)
    assert oracle.ryser_i01(np.eye(n, dtype=np.uint8)) == 1
    assert oracle.ryser_i01(pins.j_minus_i(n)) == pins.derangements(n)
    assert oracle.ryser_i01(pins.tridiagonal_ones(n)) == pins.fibonacci(n + 1)
    assert oracle.ryser_i01(pins.hessenberg_ones(n)) == 2 ** (n - 1)
    assert oracle.ryser_i01(pins.identity_plus_shift(n)) == 2
    assert oracle.ryser_i01(pins.menage_matrix(n)) == pins.menage(n)


def test_int_known_big_values():
    # D_24 and 24! (recurrence values)
    assert pins.derangements(24) == 228250211305338670494289
    assert math.factorial(24) == 620448401733239439360000
    assert pins.menage(7) == 579 and pins.menage(3) == 1


def test_int_block_diag_and_batch():
    A1 = inputs.bernoulli01((7, 7), 1)
    A2 = inputs.bernoulli01((6, 6), 2)
    M = np.zeros((13, 13), dtype=np.uint8)
    M[:7, :7], M[7:, 7:] = A1, A2
    rng = np.random.default_rng(0)
    M = M[rng.permutation(13)][:, rng.permutation(13)]
    assert oracle.ryser_i01(M) == oracle.naive_i01(A1) * oracle.naive_i01(A2)
    batch = inputs.bernoulli01((6, 9, 9), 3)
    assert oracle.ryser_i01_batch(batch) == [oracle.naive_i01(b) for b in batch]


def test_ryser_batch_matches_single():
    A = inputs.complex_gaussian((5, 6, 6), 31)
    got = oracle.ryser_batch(A)
    for b in range(5):
        ref = oracle.naive(A[b]).value
        assert _close(got[b], ref, 1e-14, max(abs(ref), pins.scaled_floor(A[b])))


# ------------------------------------------------------------------ Eq. (4) weighted Ryser pins (NEXT-1)

def _expand(C, mult):
    return np.repeat(np.asarray(C), np.asarray(mult), axis=1)


@pytest.mark.parametrize("mult", [(1, 1, 1, 1, 1), (2, 1, 1), (3, 2, 2), (1, 4), (2, 2, 2, 2), (5, 0, 2, 1)])
def test_weighted_matches_eq3_on_expanded_matrix(mult):
    # Eq. (4) against Eq. (3) / Eq. (1) of the matrix with the columns repeated: different formulas
    # (2^n subsets vs prod (m_k+1) multiplicity vectors), same permanent
    n = sum(mult)
    rng = np.random.default_rng(400 + n + len(mult))
    C = (rng.standard_normal((n, len(mult))) + 1j * rng.standard_normal((n, len(mult)))) / np.sqrt(2)
    val, asum = oracle.ryser_weighted(C, mult)
    A = _expand(C, mult)
    ref = oracle.naive(A).value if n <= 9 else oracle.ryser(A).value
    assert abs(val.value - ref) <= 1e-25 * asum + 1e-28


def test_weighted_all_distinct_is_eq3():
    # all m_k = 1: every weight is 1 and Omega = subsets, i.e. Eq. (4) is Eq. (3) term by term
    rng = np.random.default_rng(9)
    for n in (1, 2, 5, 10):
        C = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        val, asum = oracle.ryser_weighted(C, [1] * n)
        assert abs(val.value - oracle.ryser(C).value) <= 1e-25 * asum


def test_weighted_single_column_factorial():
    # R = 1: per of n copies of one column = n! prod_i c_i (every permutation gives the same product);
    # Eq. (4) then reads (-1)^n sum_f (-1)^f C(n,f) f^n prod c_i, a Stirling-number identity
    for n in (1, 2, 3, 7, 12, 20):
        val, _ = oracle.ryser_weighted(np.ones((n, 1)), [n])
        assert val.value == complex(math.factorial(n))
        c = np.arange(1, n + 1, dtype=float) * (1 - 0.5j)
        val, asum = oracle.ryser_weighted(c[:, None], [n])
        ref = math.factorial(n) * np.prod(c.astype(np.complex128))
        assert abs(val.value - ref) <= 1e-25 * asum + 1e-14 * abs(ref)


def test_weighted_integer_brute_force():
    # small integer columns: exact brute force over all n! permutations in Python integers
    rng = np.random.default_rng(5)
    for mult in ((2, 1), (1, 2, 1), (3, 1, 1), (2, 2, 1)):
        n = sum(mult)
        C = rng.integers(-3, 4, size=(n, len(mult)))
        A = _expand(C, mult)
        ref = sum(math.prod(int(A[i, p[i]]) for i in range(n)) for p in itertools.permutations(range(n)))
        val, _ = oracle.ryser_weighted(C.astype(np.complex128), mult)
        assert val.value == complex(ref)


def test_weighted_boson_sampling_normalization_with_collisions():
    # P13 with repeated output modes computed directly by Eq. (4): for a Haar unitary U (m x m) and
    # input rows S, sum over output multisets T of |per(U_{S,T})|^2 / prod_j t_j! = 1, where each
    # per(U_{S,T}) is evaluated from the DISTINCT columns of T and their multiplicities
    for (m, n) in ((4, 2), (5, 3), (6, 4)):
        U = inputs.haar_unitary(m, 177 + m)
        S = np.arange(n)
        tot = 0.0
        for T in itertools.combinations_with_replacement(range(m), n):
            modes, counts = np.unique(np.array(T), return_counts=True)
            val, _ = oracle.ryser_weighted(U[np.ix_(S, modes)], counts)
            tot += abs(val.value) ** 2 / math.prod(math.factorial(int(c)) for c in counts)
        assert abs(tot - 1.0) < 1e-13


# ------------------------------------------------------------------ entries in {-1, 0, 1} (NEXT-2, Sec. V)

def test_i8_brute_force_python():
    rng = np.random.default_rng(31)
    for n in range(1, 8):
        A = rng.integers(-1, 2, size=(n, n)).astype(np.int8)
        ref = sum(math.prod(int(A[i, p[i]]) for i in range(n)) for p in itertools.permutations(range(n)))
        assert oracle.ryser_i8(A) == ref


def test_i8_against_binary128_complex_oracle():
    # an independent evaluation: Eq. (3) in binary128 complex arithmetic (exact for these magnitudes)
    rng = np.random.default_rng(32)
    for n in (8, 12, 16):
        A = (2 * rng.integers(0, 2, size=(n, n)) - 1).astype(np.int8)
        q = oracle.ryser(A.astype(np.complex128))
        assert oracle.ryser_i8(A) == int(q.re_hi) + int(q.re_lo) and q.im_hi == 0.0


def test_i8_sign_identities_and_01_agreement():
    rng = np.random.default_rng(33)
    n = 14
    A = (2 * rng.integers(0, 2, size=(n, n)) - 1).astype(np.int8)
    p = oracle.ryser_i8(A)
    assert oracle.ryser_i8(-A) == (-1) ** n * p                        # per(-A) = (-1)^n per(A)
    B = A.copy()
    B[3] *= -1
    assert oracle.ryser_i8(B) == -p                                     # one row negated
    assert oracle.ryser_i8(np.ones((n, n), np.int8)) == math.factorial(n)
    Z = rng.integers(0, 2, size=(n, n)).astype(np.uint8)                # 0-1 special case
    assert oracle.ryser_i8(Z.astype(np.int8)) == oracle.ryser_i01(Z)
    with pytest.raises(ValueError):
        oracle.ryser_i8(np.full((3, 3), 2, np.int8))


# ------------------------------------------------------------------ App. B sparse enumeration (NEXT-3)

def _sparse_matrix(n, density, seed, complex_=True):
    rng = np.random.default_rng(seed)
    M = (rng.random((n, n)) < density).astype(float)
    M[np.arange(n), rng.permutation(n)] = 1.0                   # no zero rows / columns, per != 0 generically
    if complex_:
        M = M * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return M


def _partition_ok(A, S, T):
    n = A.shape[0]
    supp = [sum(1 << j for j in range(n) if A[i, j] != 0) for i in range(n)]
    used = 0
    for s in S:
        assert s in supp and (used & s) == 0                        # a row's support, pairwise disjoint
        used |= s
    assert T == ((1 << n) - 1) & ~used


@pytest.mark.parametrize("n,density,seed", [(6, 0.3, 1), (10, 0.2, 2), (14, 0.15, 3), (16, 0.1, 4), (12, 0.5, 5)])
def test_sparse_matches_eq3_and_counts(n, density, seed):
    # App. B restricts Eq. (3) to sets J meeting every S_l; every skipped J leaves some row sum exactly 0,
    # so the restricted sum equals Eq. (3)/(1).  The enumeration count is 2^|T| prod (2^|S_l| - 1).
    A = _sparse_matrix(n, density, seed)
    S, T = oracle.sparse_partition(A)
    _partition_ok(A, S, T)
    val, cnt = oracle.sparse(A)
    ref = oracle.naive(A).value if n <= 9 else oracle.ryser(A).value
    scale = max(abs(ref), 1e-30)
    assert abs(val.value - ref) <= 1e-25 * max(scale, float(np.prod(np.abs(A).sum(axis=1))))
    assert cnt == 2 ** bin(T).count("1") * math.prod(2 ** bin(s).count("1") - 1 for s in S)
    assert cnt <= 2 ** n


def test_sparse_structured_closed_forms():
    # permutation matrix -> 1; tridiagonal all-ones -> Fibonacci F_{n+1}; zero row -> 0;
    # diagonal -> product of the diagonal; block diagonal -> product of the blocks
    n = 12
    P = np.eye(n)[np.random.default_rng(7).permutation(n)]
    assert oracle.sparse(P)[0].value == 1.0
    assert oracle.sparse(pins.tridiagonal_ones(n).astype(float))[0].value == pins.fibonacci(n + 1)
    Z = _sparse_matrix(8, 0.3, 9)
    Z[3] = 0
    assert oracle.sparse(Z)[0].value == 0.0
    d = np.arange(1, n + 1) * (0.5 + 0.25j)
    assert abs(oracle.sparse(np.diag(d))[0].value - np.prod(d)) <= 1e-14 * abs(np.prod(d))
    B1, B2 = _sparse_matrix(5, 0.5, 10), _sparse_matrix(6, 0.4, 11)
    M = np.zeros((11, 11), complex)
    M[:5, :5], M[5:, 5:] = B1, B2
    ref = oracle.naive(B1).value * oracle.naive(B2).value
    assert abs(oracle.sparse(M)[0].value - ref) <= 1e-13 * abs(ref)


# ------------------------------------------------------------------ App. C band-limited (NEXT-4)

def _banded(n, k, seed):
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    i, j = np.indices((n, n))
    A[np.abs(i - j) > k] = 0
    return A


@pytest.mark.parametrize("n,k", [(1, 0), (2, 1), (5, 1), (7, 2), (9, 3), (12, 2), (14, 4), (16, 5), (18, 7)])
def test_band_matches_eq3(n, k):
    # App. C's transfer polynomial against Eq. (3)/(1) on matrices that vanish outside the band
    A = _banded(n, k, 100 * n + k)
    ref = oracle.naive(A).value if n <= 9 else oracle.ryser(A).value
    got = oracle.band(A, k).value
    scale = oracle.band(np.abs(A).astype(complex), k).value.real        # per(|A|): sum of |path products|
    assert abs(got - ref) <= 1e-25 * scale


def test_band_closed_forms():
    for n in (1, 2, 10, 40, 90):
        q = oracle.band(pins.tridiagonal_ones(n).astype(complex), 1)       # binary128: exact to 2^113
        assert int(q.re_hi) + int(q.re_lo) == pins.fibonacci(n + 1) and q.im_hi == 0.0
    d = np.arange(1, 13) * (1 - 0.5j)
    assert abs(oracle.band(np.diag(d), 0).value - np.prod(d)) <= 1e-14 * abs(np.prod(d))
    A = inputs.complex_gaussian((8, 8), 88)
    assert abs(oracle.band(A, 7).value - oracle.naive(A).value) <= 1e-25 * float(np.prod(np.abs(A).sum(1)))
    assert abs(oracle.band(A, 20).value - oracle.naive(A).value) <= 1e-25 * float(np.prod(np.abs(A).sum(1)))
    # entries outside the band are never read
    B = _banded(10, 2, 5)
    C = B + np.triu(np.ones((10, 10)), 3) * 7.0
    assert oracle.band(C, 2).value == oracle.band(B, 2).value
