"""GPU parity of perm_c128_batched (BASELINE config 2) against the CPU oracle."""
from __future__ import annotations

import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs
from tests import pins

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _check_batch(torch, A, ref):
    per, abs2 = pb.perm_c128_batched(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    per = per.cpu().numpy()
    abs2 = abs2.cpu().numpy()
    for b in range(A.shape[0]):
        assert pins.scaled_error(per[b], ref[b], A[b]) <= TOL, (b, per[b], ref[b])
        assert abs2[b] == per[b].real * per[b].real + per[b].imag * per[b].imag


@pytest.mark.parametrize("n", list(range(1, 15)))
def test_random_small_batches(torch, n):
    B = 37 if n <= 10 else 9          # ragged: not a multiple of matrices-per-warp
    A = inputs.complex_gaussian((B, n, n), 500 + n)
    _check_batch(torch, A, oracle.ryser_batch(A))


@pytest.mark.parametrize("n", [16, 20, 24])
def test_larger_orders(torch, n):
    A = inputs.complex_gaussian((3, n, n), 600 + n)
    ref = np.array([oracle.permanent_hr(A[b]).value for b in range(3)])
    _check_batch(torch, A, ref)


@pytest.mark.parametrize("n", [28, 32])
def test_max_orders_block_diagonal(torch, n):
    # up to the kernel's largest order (32): P (B1 + B2) Q (direct sum, scrambled rows and columns) has
    # per = per(B1) per(B2), each block's permanent from the oracle's Eq. (3)
    h = n // 2
    rng = np.random.default_rng(900 + n)
    A = np.zeros((2, n, n), dtype=np.complex128)
    ref = []
    for b in range(2):
        B1 = inputs.complex_gaussian((h, h), 910 + n + b)
        B2 = inputs.complex_gaussian((n - h, n - h), 930 + n + b)
        M = np.zeros((n, n), dtype=np.complex128)
        M[:h, :h] = B1
        M[h:, h:] = B2
        A[b] = M[rng.permutation(n)][:, rng.permutation(n)]
        ref.append(oracle.ryser(B1).value * oracle.ryser(B2).value)
    _check_batch(torch, A, np.array(ref))


def test_empty_batch_and_errors(torch):
    A = torch.zeros((0, 8, 8), dtype=torch.complex128, device="cuda")
    per, abs2 = pb.perm_c128_batched(A)
    assert per.numel() == 0
    with pytest.raises(pb.PermError):
        pb.perm_c128_batched(torch.zeros((1, 33, 33), dtype=torch.complex128, device="cuda"))


def test_identity_and_ones(torch):
    for n in (1, 4, 8, 12, 16):
        A = np.stack([np.eye(n), np.ones((n, n))]).astype(np.complex128)
        per, _ = pb.perm_c128_batched(torch.from_numpy(A).cuda())
        per = per.cpu().numpy()
        assert per[0] == 1
        assert abs(per[1] - math.factorial(n)) <= 1e-13 * math.factorial(n)


@pytest.mark.parametrize("m,n", [(9, 3), (16, 4), (25, 5)])
def test_boson_sampling_normalization(torch, m, n):
    """P13: sum_T |per(U_{S,T})|^2 / prod t_j! = 1 over all output multisets T (unitarity)."""
    U = inputs.haar_unitary(m, 900 + m)
    S = np.arange(n)
    mats, w = [], []
    for T in itertools.combinations_with_replacement(range(m), n):
        mats.append(U[np.ix_(S, list(T))])
        cnt = np.bincount(np.array(T), minlength=m)
        w.append(1.0 / float(np.prod([math.factorial(int(k)) for k in cnt])))
    A = torch.from_numpy(np.ascontiguousarray(np.array(mats))).cuda()
    _, abs2 = pb.perm_c128_batched(A, want_per=False)
    total = float(np.sum(abs2.cpu().numpy() * np.array(w)))
    assert abs(total - 1.0) < 1e-12, total


@pytest.mark.parametrize("n,count", [(8, 100000), (12, 10000)])
def test_cfg2_full_batch_every_output(torch, n, count):
    """Config 2 at full size (the bench launch, 10^5 submatrices): every output for n = 8 and a seeded
    10^4 subset for n = 12 against the oracle's Eq. (3), computed here (SURVEY 8(c) parity plan)."""
    A = inputs.cfg2(n)
    per, _ = pb.perm_c128_batched(torch.from_numpy(A).cuda())
    per = per.cpu().numpy()
    idx = np.arange(A.shape[0]) if count >= A.shape[0] else \
        np.sort(np.random.default_rng(9100 + n).choice(A.shape[0], count, replace=False))
    ref = oracle.ryser_batch(np.ascontiguousarray(A[idx]))
    floor = 2.0 ** (-n / 2) * np.prod(np.linalg.norm(A[idx], axis=2), axis=1)
    err = np.abs(per[idx] - ref) / np.maximum(np.abs(ref), floor)
    assert err.max() <= TOL, (n, int(idx[np.argmax(err)]), err.max())


@pytest.mark.parametrize("n", [8, 12, 16, 20])
def test_cfg2_full_batch_samples(torch, golden_dir, n):
    """Config 2 at full size (10^5 submatrices, the bench launch): sampled outputs vs the oracle,
    plus the Haar expectation E|per|^2 = n!(m-1)!/(m+n-1)! (P14) as a statistical check."""
    A = inputs.cfg2(n)
    per, abs2 = pb.perm_c128_batched(torch.from_numpy(A).cuda())
    per = per.cpu().numpy()
    abs2 = abs2.cpu().numpy()
    p = os.path.join(golden_dir, "oracle_values.json")
    g = json.load(open(p)).get("cfg2", {}).get(str(n)) if os.path.exists(p) else None
    if g:
        idx = np.array(g["index"])
        ref = np.array(g["re"]) + 1j * np.array(g["im"])
    else:
        idx = np.sort(np.random.default_rng(9000 + n).choice(A.shape[0], 8, replace=False))
        ref = np.array([oracle.permanent_hr(A[i]).value for i in idx])
    for i, r in zip(idx, ref):
        assert pins.scaled_error(per[i], r, A[i]) <= TOL, (n, i)
    m = n * n
    expect = math.exp(math.lgamma(n + 1) + math.lgamma(m) - math.lgamma(m + n))
    se = np.std(abs2) / np.sqrt(len(abs2))
    assert abs(np.mean(abs2) - expect) < 6 * se, (np.mean(abs2), expect, se)


@pytest.mark.parametrize("n", [14, 16, 20])
def test_unit_column_walk_fallbacks(torch, n):
    # the unit-column walk normalises each matrix by its column 0; a matrix with a zero there, one
    # with a column-0 entry 1e-120 times its row's other entries, and one with a scaled row take the plain walk or
    # the normalised one -- all within the north-star bound of the oracle
    A = inputs.complex_gaussian((4, n, n), 900 + n)
    A[0, 3, 0] = 0.0
    A[1, 5, 0] = 1e-121 * A[1, 5, 0]
    A[2, 2, :] *= 1e30
    ref = np.array([oracle.permanent_hr(A[b]).value for b in range(4)])
    _check_batch(torch, A, ref)
