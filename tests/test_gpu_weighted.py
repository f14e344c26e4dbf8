"""GPU parity of perm_c128_weighted_batched (Eq. (4)) against the CPU
oracle's literal Eq. (4) (oracle.ryser_weighted, pinned in test_oracle_pins.py)."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

import oracle
import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs

pytestmark = pytest.mark.gpu
# |per_gpu - per_oracle| <= REL * sum_f |term_f|: the rounding scale of any evaluation of the Eq. (4)
# sum of prod(m_k+1) terms, each a product of n row sums (error <= ~(3n + log2 terms) eps relative to
# the term), reading R16
REL = 1e-12


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _run(torch, C, mult):
    per, abs2 = pb.perm_c128_weighted_batched(torch.from_numpy(C).cuda(), torch.from_numpy(mult).cuda())
    torch.cuda.synchronize()
    return per.cpu().numpy(), abs2.cpu().numpy()


def _check(torch, C, mult):
    per, abs2 = _run(torch, C, mult)
    for b in range(C.shape[0]):
        R = int(np.count_nonzero(mult[b] >= 0))
        ref, asum = oracle.ryser_weighted(C[b][:, :R], mult[b][:R])
        assert abs(per[b] - ref.value) <= REL * asum + 1e-300, (b, mult[b], per[b], ref.value, asum)
        assert abs2[b] == per[b].real * per[b].real + per[b].imag * per[b].imag


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 11, 12, 16])
def test_random_multiplicities(torch, n):
    # ragged batches of random multiplicity vectors (zeros, one big digit, all ones), R = n
    rng = np.random.default_rng(700 + n)
    B = 13
    C = inputs.complex_gaussian((B, n, n), 800 + n)
    mult = np.zeros((B, n), dtype=np.int32)
    for b in range(B):
        if b == 0:
            mult[b, :] = 1                        # no repeats: Eq. (4) = Eq. (3)
        elif b == 1:
            mult[b, 0] = n                        # one column n times
        else:
            for _ in range(n):
                mult[b, rng.integers(0, n)] += 1
    _check(torch, C, mult)


def test_all_distinct_matches_batched_glynn(torch):
    # m = 1 everywhere: the weighted kernel (full-range Ryser) and the Glynn batched kernel agree
    n, B = 10, 20
    A = inputs.cfg2(n, B)
    per_w, _ = _run(torch, A, np.ones((B, n), dtype=np.int32))
    per_g, _ = pb.perm_c128_batched(torch.from_numpy(A).cuda())
    per_g = per_g.cpu().numpy()
    floor = 2.0 ** (-n / 2) * np.prod(np.linalg.norm(A, axis=2), axis=1)
    assert np.all(np.abs(per_w - per_g) <= 1e-9 * np.maximum(np.abs(per_g), floor))


def test_single_column_factorial(torch):
    # R = 1: n copies of one column, per = n! prod_i c_i.  For the all-ones column every term
    # (-1)^f C(n,f) f^n is an integer; up to n = 13 they are below 2^53, the double sum is exact and so
    # is per = n!; beyond, the terms (~n^n) cancel down to n! and the error is bounded by REL * sum|term|
    for n in (1, 5, 13, 20, 32):
        C = np.ones((1, n, 1), dtype=np.complex128)
        per, _ = _run(torch, C, np.array([[n]], dtype=np.int32))
        if n <= 13:
            assert per[0] == complex(math.factorial(n))
        else:
            asum = sum(math.comb(n, f) * f ** n for f in range(n + 1))
            assert abs(per[0] - math.factorial(n)) <= REL * asum


def test_max_order_vs_oracle(torch):
    # the largest order (n = 32): 8 distinct columns four times each (5^8 terms, two-digit tiles of 25),
    # and a ragged vector over 6 columns whose second sweep digit is small
    n = 32
    C = inputs.complex_gaussian((2, n, 8), 932)
    mult = np.array([[4] * 8, [9, 7, 6, 5, 3, 2, 0, 0]], dtype=np.int32)
    assert np.all(mult.sum(axis=1) == n)
    per, _ = _run(torch, C, mult)
    for b in range(2):
        R = int(np.count_nonzero(mult[b]))
        ref, asum = oracle.ryser_weighted(C[b][:, :R], mult[b][:R])
        assert abs(per[b] - ref.value) <= REL * asum + 1e-300, (b, per[b], ref.value, asum)


def test_collision_patterns_vs_oracle(torch):
    # Boson-sampling output patterns with collisions (n = 12 photons in m = 36 modes, some n = 16)
    for (n, m, cnt, seed) in ((12, 36, 24, 5), (16, 64, 6, 6)):
        C, mult = inputs.collision_patterns(n, m, cnt, seed)
        _check(torch, C, mult)


def test_boson_sampling_normalization_with_collisions(torch):
    # P13 on the GPU outputs: sum over all output multisets T of |per(U_{S,T})|^2 / prod t_j! = 1
    for (m, n) in ((5, 3), (7, 4)):
        U = inputs.haar_unitary(m, 277 + m)
        Cs, Ms, W = [], [], []
        for T in itertools.combinations_with_replacement(range(m), n):
            modes, counts = np.unique(np.array(T), return_counts=True)
            C = np.zeros((n, n), dtype=np.complex128)
            C[:, :len(modes)] = U[:n][:, modes]
            M = np.zeros(n, dtype=np.int32)
            M[:len(modes)] = counts
            Cs.append(C)
            Ms.append(M)
            W.append(1.0 / math.prod(math.factorial(int(c)) for c in counts))
        _, abs2 = _run(torch, np.array(Cs), np.array(Ms))
        assert abs(float(np.dot(abs2, W)) - 1.0) < 1e-12


def test_invalid_multiplicities_give_nan_and_empty_batch(torch):
    C = inputs.complex_gaussian((3, 4, 4), 1)
    mult = np.array([[1, 1, 1, 1], [2, 1, 0, 0], [5, -1, 0, 0]], dtype=np.int32)   # ok, sum 3, negative
    per, abs2 = _run(torch, C, mult)
    assert np.isfinite(per[0]) and np.isnan(per[1]) and np.isnan(per[2]) and np.isnan(abs2[2])
    e, a = pb.perm_c128_weighted_batched(torch.zeros((0, 4, 4), dtype=torch.complex128, device="cuda"),
                                         torch.zeros((0, 4), dtype=torch.int32, device="cuda"))
    assert e.shape[0] == 0 and a.shape[0] == 0


def test_argument_errors(torch):
    C = torch.zeros((2, 4, 70), dtype=torch.complex128, device="cuda")
    m = torch.zeros((2, 70), dtype=torch.int32, device="cuda")
    with pytest.raises(pb.PermError):
        pb.perm_c128_weighted_batched(C, m)                  # R > 64
    C = torch.zeros((2, 33, 4), dtype=torch.complex128, device="cuda")
    m = torch.zeros((2, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(pb.PermError):
        pb.perm_c128_weighted_batched(C, m)                  # n > 32
