"""CPU pins of the two regroupings the exact integer walk uses, derived here from the definition
of the Glynn sum in exact Python integers on small matrices -- independent of the CUDA code and of oracle/:

* pair identity (0-1 entries): the terms of ranks 2q, 2q+1 (Gray bit 0 flipped, opposite signs) sum to
  C (W' - W), C the product over the rows whose bit-0 entry is zero;
* quad identity (+-1 entries): after negating rows so that the bit-0 column is all +1, the terms of an aligned quad
  of ranks sum to d [M(0) (P(2) + P(-2)) - P(0) (M(2) + M(-2))] over the classes of the bit-1 column, d = +1 iff
  bit 2 of the rank is set; and per(D A Q) = sign * per(A) for the row negations D and the column negation Q
  (sign = the product of the negations);
* unit-column identities (complex entries, exact Gaussian rationals): per(A) = prod_i a_i0 per(A') for
  A' = D^{-1} A, and on A' the terms of ranks 2q, 2q+1 sum to s_q (prod (v + 1) - prod v) with v the row sums at
  Gray bit 0 = 0 -- the algebra of the unit-column walk.

The Glynn sum of App. A / SURVEY S-1: Sum = sum_r (-1)^{r+1} prod_i g_i(gray r), g_i = a_{i,n-1} + sum_{j<n-1}
delta_j a_ij with delta_j = +1 iff bit j of gray r is set; per = (-1)^n Sum / 2^{n-1}.
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest


def gray(r: int) -> int:
    return r ^ (r >> 1)


def g_vec(A, r):
    n = A.shape[0]
    x = gray(r)
    return [int(A[i, n - 1]) + sum((1 if (x >> j) & 1 else -1) * int(A[i, j]) for j in range(n - 1)) for i in range(n)]


def glynn_sum(A) -> int:
    n = A.shape[0]
    return sum((-1) ** (r + 1) * math.prod(g_vec(A, r)) for r in range(1 << (n - 1)))


def per_brute(A) -> int:
    n = A.shape[0]
    return sum(math.prod(int(A[i, s[i]]) for i in range(n)) for s in itertools.permutations(range(n)))


@pytest.mark.parametrize("n,seed", [(5, 1), (6, 2), (7, 3), (8, 4)])
def test_glynn_sum_is_the_permanent(n, seed):
    A = np.random.default_rng(seed).integers(0, 2, size=(n, n))
    assert (-1) ** n * glynn_sum(A) == per_brute(A) * 2 ** (n - 1)


@pytest.mark.parametrize("n,seed", [(6, 11), (7, 12), (8, 13), (9, 14)])
def test_pair_identity_01(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(0, 2, size=(n, n))
    A[rng.choice(n, n // 2, replace=False), 0] = 0               # some zero rows in the bit-0 column
    Z = [i for i in range(n) if A[i, 0] == 0]
    V = [i for i in range(n) if A[i, 0] != 0]
    total = 0
    for q in range(1 << (n - 2)):
        g0, g1 = g_vec(A, 2 * q), g_vec(A, 2 * q + 1)
        assert all(g0[i] == g1[i] for i in Z)                   # the bit-0 flip leaves the zero rows unchanged
        C = math.prod(g0[i] for i in Z)
        pair = C * (math.prod(g1[i] for i in V) - math.prod(g0[i] for i in V))
        assert pair == -math.prod(g0) + math.prod(g1)           # signs (-1)^{r+1}: rank 2q -, rank 2q+1 +
        total += pair
    assert total == glynn_sum(A)


@pytest.mark.parametrize("n,seed", [(6, 21), (7, 22), (8, 23), (9, 24)])
def test_quad_identity_pm1(n, seed):
    rng = np.random.default_rng(seed)
    A0 = 2 * rng.integers(0, 2, size=(n, n)) - 1
    # normalise: rows negated so that column 0 is all +1; column 1 negated (tau) -- the plan's transformation
    sigma = A0[:, 0].copy()
    tau = -1 if seed % 2 else 1
    A = A0 * sigma[:, None]
    A[:, 1] *= tau
    sign = int(np.prod(sigma)) * tau
    assert per_brute(A) == sign * per_brute(A0)
    P = [i for i in range(n) if A[i, 1] == 1]
    M = [i for i in range(n) if A[i, 1] == -1]
    total = 0
    for t in range(1 << (n - 3)):
        r0 = 4 * t
        g = g_vec(A, r0)
        x = gray(r0)
        d0, d1 = (1 if x & 1 else -1), (1 if (x >> 1) & 1 else -1)
        h = [g[i] - d0 * int(A[i, 0]) - d1 * int(A[i, 1]) for i in range(n)]   # the part of Gray bits >= 2

        def X(rows, s):
            return math.prod(h[i] + s for i in rows)

        d = 1 if (r0 >> 2) & 1 else -1
        quad = d * (X(M, 0) * (X(P, 2) + X(P, -2)) - X(P, 0) * (X(M, 2) + X(M, -2)))
        direct = sum((-1) ** (r + 1) * math.prod(g_vec(A, r)) for r in range(r0, r0 + 4))
        assert quad == direct
        total += quad
    assert (-1) ** n * total == per_brute(A) * 2 ** (n - 1)


# ---- the unit-column walk, in exact Gaussian rationals

from fractions import Fraction  # noqa: E402


class GQ:
    """Exact complex rational a + bi."""
    __slots__ = ("a", "b")

    def __init__(self, a, b=0):
        self.a, self.b = Fraction(a), Fraction(b)

    def __add__(self, o):
        return GQ(self.a + o.a, self.b + o.b)

    def __sub__(self, o):
        return GQ(self.a - o.a, self.b - o.b)

    def __mul__(self, o):
        return GQ(self.a * o.a - self.b * o.b, self.a * o.b + self.b * o.a)

    def __truediv__(self, o):
        d = o.a * o.a + o.b * o.b
        return GQ((self.a * o.a + self.b * o.b) / d, (self.b * o.a - self.a * o.b) / d)

    def __eq__(self, o):
        return self.a == o.a and self.b == o.b


def gq_prod(xs):
    p = GQ(1)
    for x in xs:
        p = p * x
    return p


def gq_per(M):
    n = len(M)
    tot = GQ(0)
    for s in itertools.permutations(range(n)):
        tot = tot + gq_prod(M[i][s[i]] for i in range(n))
    return tot


def gq_w(M, r):
    """App. A row sums w_i(gray r) = a_{i,n-1} - 1/2 sum_j a_ij + sum_{j<n-1, x_j=1} a_ij."""
    n = len(M)
    x = gray(r)
    out = []
    for i in range(n):
        w = M[i][n - 1]
        for j in range(n):
            w = w - M[i][j] * GQ(Fraction(1, 2))
        for j in range(n - 1):
            if (x >> j) & 1:
                w = w + M[i][j]
        out.append(w)
    return out


@pytest.mark.parametrize("n,seed", [(4, 31), (5, 32), (6, 33)])
def test_unit_column_identities(n, seed):
    rng = np.random.default_rng(seed)
    A = [[GQ(int(rng.integers(-3, 4)), int(rng.integers(-3, 4))) for _ in range(n)] for _ in range(n)]
    for i in range(n):
        if A[i][0] == GQ(0):
            A[i][0] = GQ(1, 1)
    # A' = D^-1 A: column 0 all ones; per(A) = prod_i a_i0 * per(A')
    Ap = [[A[i][j] / A[i][0] for j in range(n)] for i in range(n)]
    assert all(Ap[i][0] == GQ(1) for i in range(n))
    assert gq_per(A) == gq_prod(A[i][0] for i in range(n)) * gq_per(Ap)
    # the pairs of the walk: ranks 2q, 2q+1 read v (Gray bit 0 = 0) and v + 1, signs (-1)^{r+1}
    S_terms, S_pairs = GQ(0), GQ(0)
    for r in range(1 << (n - 1)):
        t = gq_prod(gq_w(Ap, r))
        S_terms = S_terms + t if r & 1 else S_terms - t
    for q in range(1 << (n - 2)):
        r = 2 * q
        v = gq_w(Ap, r) if gray(r) & 1 == 0 else [w - GQ(1) for w in gq_w(Ap, r)]
        sp = 1 if ((r >> 1) & 1) == 0 else -1
        d = gq_prod(w + GQ(1) for w in v) - gq_prod(v)
        S_pairs = S_pairs + d if sp > 0 else S_pairs - d
    assert S_pairs == S_terms
    # App. A: per = 2 (-1)^n S
    assert gq_per(Ap) == GQ(2 * (-1) ** n) * S_terms
