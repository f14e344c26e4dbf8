"""GPU parity of perm_pm1 (entries in {-1, 0, 1}: the Bernoulli +-1 ensemble of Sec. V, P:846-860;
SURVEY 8(f) NEXT-2) against the exact int128 oracle -- bit-exact -- and of the batched kernel on the
Haar minors S(n^a, n) of Sec. VI with a = 3."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 17, 20])
def test_pm1_bit_exact(torch, n):
    A = inputs.bernoulli_pm1((9, n, n), 900 + n)
    got = pb.perm_pm1(torch.from_numpy(A).cuda())
    assert got == [oracle.ryser_i8(A[b]) for b in range(A.shape[0])]


def test_pm1_mixed_entries_and_identities(torch):
    rng = np.random.default_rng(91)
    n = 16
    A = rng.integers(-1, 2, size=(4, n, n)).astype(np.int8)         # zeros allowed
    A[1] = 1                                                          # J: n!
    A[2] = -A[0]                                                      # per(-A) = per(A) (n even)
    got = pb.perm_pm1(torch.from_numpy(A).cuda())
    assert got[0] == oracle.ryser_i8(A[0]) and got[1] == math.factorial(n) and got[2] == got[0]
    assert got[3] == oracle.ryser_i8(A[3])


def test_pm1_n24_ensemble_sample(torch):
    # the Sec. V workload shape at n = 24: exact, compared with the int128 oracle on a few samples
    A = inputs.bernoulli_pm1((4, 24, 24), 2424)
    assert pb.perm_pm1(torch.from_numpy(A).cuda()) == [oracle.ryser_i8(A[b]) for b in range(4)]


def test_pm1_rejects_out_of_range(torch):
    A = np.ones((2, 6, 6), np.int8)
    A[1, 2, 3] = 2
    with pytest.raises(pb.PermError):
        pb.perm_pm1(torch.from_numpy(A).cuda())
    A[1, 2, 3] = -2
    with pytest.raises(pb.PermError):
        pb.perm_pm1(torch.from_numpy(A).cuda())


def test_haar_minors_a3_expectation(torch):
    # E|per(U_{S,T})|^2 = n!(m-1)!/(m+n-1)! for Haar U(m) (Schur on Sym^n), m = n^3
    n, B = 4, 100000
    A = inputs.haar_minors(n, 3, B, 4343)
    _, abs2 = pb.perm_c128_batched(torch.from_numpy(A).cuda())
    abs2 = abs2.cpu().numpy()
    m = n ** 3
    expect = math.factorial(n) * math.factorial(m - 1) / math.factorial(m + n - 1)
    se = abs2.std() / math.sqrt(B)
    assert abs(abs2.mean() - expect) < 5 * se
    ref = oracle.ryser_batch(A[:64])
    assert np.allclose(abs2[:64], np.abs(ref) ** 2, rtol=1e-9, atol=0)


# ---- the quad-factored walk: +-1 columns, rows sign-normalised on the bit-0 column, classes by the
# bit-1 column; each order 20..24, both class sizes of the menu and the column-negation case, plus the fall-backs

@pytest.mark.parametrize("n", [20, 21, 22, 23, 24])
def test_pm1_quad_vs_oracle(torch, n):
    A = inputs.bernoulli_pm1((6, n, n), 2000 + n)
    assert pb.perm_pm1(torch.from_numpy(A).cuda()) == [oracle.ryser_i8(A[b]) for b in range(A.shape[0])]


def test_pm1_quad_class_sizes_and_negation(torch):
    # column 1's agreement with column 0 forced to z rows, z = 11, 12, 13 (13: the plan negates the column)
    n = 24
    rng = np.random.default_rng(2411)
    mats = []
    for z in (11, 12, 13, 7):
        A = inputs.bernoulli_pm1((n, n), 5000 + z)
        agree = np.zeros(n, bool)
        agree[rng.choice(n, z, replace=False)] = True
        A[:, 1] = np.where(agree, A[:, 0], -A[:, 0])
        mats.append(A)
    A = np.stack(mats)
    assert pb.perm_pm1(torch.from_numpy(A).cuda()) == [oracle.ryser_i8(A[b]) for b in range(A.shape[0])]


def test_pm1_quad_fallbacks(torch):
    # zeros in every column (plain walk), zeros in a few columns only (quad plan on the others), and many zeros in
    # one column (the zero-row plan)
    n = 22
    rng = np.random.default_rng(2212)
    A = inputs.bernoulli_pm1((3, n, n), 2213)
    A[0, rng.integers(0, n, n), np.arange(n)] = 0
    A[1, 3, 0] = 0
    A[1, 5, 1] = 0
    A[2, rng.choice(n, 16, replace=False), 4] = 0
    assert pb.perm_pm1(torch.from_numpy(A).cuda()) == [oracle.ryser_i8(A[b]) for b in range(A.shape[0])]
