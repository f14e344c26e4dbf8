"""Closed forms and structured matrices used as pins (no permanent arithmetic).

Each value comes from combinatorics independent of any permanent algorithm:
derangement recurrence, Touchard's menage formula, Fibonacci numbers, powers
of two, factorials.  See DESIGN.md "Pins".
"""
from __future__ import annotations

import math

import numpy as np


def derangements(n: int) -> int:
    """D_0 = 1, D_1 = 0, D_n = (n-1)(D_{n-1} + D_{n-2})  ->  per(J - I)."""
    d0, d1 = 1, 0
    if n == 0:
        return 1
    for k in range(2, n + 1):
        d0, d1 = d1, (k - 1) * (d0 + d1)
    return d1


def menage(n: int) -> int:
    """Touchard: U_n = sum_k (-1)^k 2n/(2n-k) C(2n-k, k) (n-k)!  ->  per(J - I - shift), n >= 3."""
    tot = 0
    for k in range(n + 1):
        term = 2 * n * math.comb(2 * n - k, k) * math.factorial(n - k)
        assert term % (2 * n - k) == 0
        tot += (-1) ** k * (term // (2 * n - k))
    return tot


def fibonacci(k: int) -> int:
    a, b = 0, 1
    for _ in range(k):
        a, b = b, a + b
    return a


# ---------------- 0-1 structured matrices

def j_minus_i(n: int) -> np.ndarray:
    return (np.ones((n, n)) - np.eye(n)).astype(np.uint8)


def tridiagonal_ones(n: int) -> np.ndarray:
    """per = F_{n+1}."""
    A = np.zeros((n, n), dtype=np.uint8)
    for i in range(n):
        for j in range(max(0, i - 1), min(n, i + 2)):
            A[i, j] = 1
    return A


def hessenberg_ones(n: int) -> np.ndarray:
    """a_ij = 1 iff j >= i - 1; per = 2^{n-1}."""
    A = np.zeros((n, n), dtype=np.uint8)
    for i in range(n):
        for j in range(n):
            if j >= i - 1:
                A[i, j] = 1
    return A


def shift(n: int) -> np.ndarray:
    return np.roll(np.eye(n, dtype=np.uint8), 1, axis=1)


def identity_plus_shift(n: int) -> np.ndarray:
    """per = 2 for n >= 3."""
    return (np.eye(n, dtype=np.uint8) + shift(n)).astype(np.uint8)


def menage_matrix(n: int) -> np.ndarray:
    """J - I - shift; per = U_n (menage number) for n >= 3."""
    return (np.ones((n, n), dtype=np.int64) - np.eye(n, dtype=np.int64) - shift(n)).astype(np.uint8)


def scaled_error(got: complex, ref: complex, A: np.ndarray) -> float:
    """|got - ref| / max(|ref|, 2^{-n/2} prod_i ||a_i||_2)  (BASELINE.json north_star)."""
    n = A.shape[0]
    floor = 2.0 ** (-n / 2) * float(np.prod(np.linalg.norm(A, axis=1)))
    return abs(got - ref) / max(abs(ref), floor)


def scaled_floor(A: np.ndarray) -> float:
    n = A.shape[0]
    return 2.0 ** (-n / 2) * float(np.prod(np.linalg.norm(A, axis=1)))


def range_scale(A: np.ndarray, length: int) -> float:
    """Typical magnitude of a sum of `length` Gray terms: sqrt(length) * 2^{-n} prod_i ||a_i||_2
    (each |w_i| ~ ||a_i||/2, random signs)."""
    n = A.shape[0]
    return float(np.sqrt(max(length, 1))) * 2.0 ** (-n) * float(np.prod(np.linalg.norm(A, axis=1)))
