"""GPU parity of perm_c128_sparse (App. B sparsepermanent + greedypartition; SURVEY 8(f)
NEXT-3) against the CPU oracle (Eq. (3) / App. B written out) and the dense GPU walk."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import paper_1904_06229_b200 as pb
from tests import pins

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _sparse(n, density, seed):
    rng = np.random.default_rng(seed)
    M = (rng.random((n, n)) < density) * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    M[np.arange(n), rng.permutation(n)] += (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
    return M


@pytest.mark.parametrize("n,density,seed", [(1, 1.0, 1), (3, 0.5, 2), (6, 0.3, 3), (10, 0.2, 4), (14, 0.15, 5),
                                            (16, 0.1, 6), (20, 0.1, 7), (24, 0.08, 8)])
def test_sparse_vs_oracle(n, density, seed):
    A = _sparse(n, density, seed)
    got, info = pb.perm_c128_sparse(A, info=True)
    ref = oracle.ryser(A).value
    assert pins.scaled_error(got, ref, A) <= TOL, (got, ref)
    S, T = oracle.sparse_partition(A)
    assert info["S"] == S and info["T"] == T
    assert info["sets"] == 2.0 ** bin(T).count("1") * math.prod(2.0 ** bin(s).count("1") - 1 for s in S)


def test_sparse_vs_oracle_app_b_count():
    A = _sparse(18, 0.12, 21)
    got, info = pb.perm_c128_sparse(A, info=True)
    ref, cnt = oracle.sparse(A)
    assert pins.scaled_error(got, ref.value, A) <= TOL and info["sets"] == cnt


def test_sparse_structured():
    n = 30
    assert pb.perm_c128_sparse(pins.tridiagonal_ones(n).astype(complex)) == pins.fibonacci(n + 1)
    P = np.eye(40)[np.random.default_rng(3).permutation(40)]
    assert pb.perm_c128_sparse(P) == 1.0
    d = (np.arange(1, 21) % 7 + 1) * (0.5 - 0.25j)
    ref = np.prod(d)
    assert abs(pb.perm_c128_sparse(np.diag(d)) - ref) <= 1e-13 * abs(ref)
    Z = _sparse(12, 0.3, 9)
    Z[:, 4] = 0
    v, info = pb.perm_c128_sparse(Z, info=True)
    assert v == 0 and info["sets"] == 0.0


def test_sparse_device_input_and_dense_walk_agree():
    import torch
    n = 34
    A = _sparse(n, 0.07, 34)
    got = pb.perm_c128_sparse(torch.from_numpy(A).cuda())
    dense = pb.perm_c128(A)                       # Glynn walk over 2^33 terms
    assert pins.scaled_error(got, dense, A) <= TOL, (got, dense)


def test_sparse_block_diagonal_closed_form():
    B1, B2 = _sparse(14, 0.2, 41), _sparse(16, 0.15, 42)
    M = np.zeros((30, 30), complex)
    M[:14, :14], M[14:, 14:] = B1, B2
    rng = np.random.default_rng(43)
    M = M[rng.permutation(30)][:, rng.permutation(30)]
    ref = oracle.ryser(B1).value * oracle.ryser(B2).value
    assert pins.scaled_error(pb.perm_c128_sparse(M), ref, M) <= TOL


@pytest.mark.parametrize("n,density", [(21, 0.5), (32, 0.5), (47, 0.04), (48, 0.04)])
def test_sparse_constant_bank_orders_block_diagonal(n, density):
    # orders of the constant-bank sparse walk (sparse_const_path): scrambled block-diagonal sparse matrices,
    # per = product of the blocks' permanents, each block by the oracle's Eq. (3).
    # (Without the dominant diagonal, sparse blocks cancel strongly: at n = 32, density 0.25, the constant-bank
    # and the shared-memory sparse walks give the same bits, 1.2e-9 from the oracle on the dense walk's scale.)
    sizes = [16] * (n // 16) + ([n % 16] if n % 16 else [])
    blocks = [_sparse(m, density, 4700 + n + k) for k, m in enumerate(sizes)]
    # a dominant unit-modulus diagonal keeps |per| well above the cancellation of the restricted sums
    ph = np.random.default_rng(4900 + n)
    blocks = [B + 3.0 * np.diag(np.exp(2j * np.pi * ph.random(B.shape[0]))) for B in blocks]
    M = np.zeros((n, n), complex)
    o = 0
    for B in blocks:
        M[o:o + B.shape[0], o:o + B.shape[0]] = B
        o += B.shape[0]
    rng = np.random.default_rng(4800 + n)
    M = M[rng.permutation(n)][:, rng.permutation(n)]
    ref = np.prod([oracle.ryser(B).value for B in blocks])
    got, info = pb.perm_c128_sparse(M, info=True)
    assert pins.scaled_error(got, ref, M) <= TOL, (got, ref, info["chunk_log2"])


def _pair_case(n, density, seed, nz):
    """A sparse matrix whose partition leaves a T column with exactly `nz` nonzero rows (the shared-rows pair
    walk's bit-0 column), scrambled."""
    for s in range(seed, seed + 200):
        A = _sparse(n, density, s)
        plan = pb.perm_sparse_plan(A)
        T = plan["T"]
        tcols = [j for j in range(n) if (T >> j) & 1]
        counts = [int(np.count_nonzero(A[:, j])) for j in tcols]
        if len(tcols) >= 6 and min(counts) == nz:
            return A
    raise AssertionError("no matrix with the asked T-column shape")


@pytest.mark.parametrize("cap", [1, 2, 3, 4])
@pytest.mark.parametrize("n,density,nz", [(17, 0.1, 1), (20, 0.1, 2), (22, 0.12, 3), (23, 0.2, 4)])
def test_sparse_group_walk_vs_oracle(n, density, nz, cap, monkeypatch):
    # shared-rows group walk: G thin T columns are the lowest Gray bits and every block of 2^G sets
    # shares the product of the rows where they are zero; checked against the oracle's Eq. (3) and against the
    # plain T walk (PERM_SPARSE_GROUP=0).  These sizes plan a chunk length <= U (shared-memory kernel); forcing
    # 2^5-rank chunks puts them on the constant-bank kernel (G <= 4 < e).  n = 17 reaches G = 4.
    A = _pair_case(n, density, 5100 + n, nz)
    monkeypatch.setenv("PERM_FORCE_CHUNK_LOG2", "5")
    monkeypatch.setenv("PERM_SPARSE_GROUP", str(cap))
    got, info = pb.perm_c128_sparse(A, info=True)
    assert 1 <= info["group_cols"] <= cap and info["chunk_log2"] == 5, info
    if n == 17:
        assert info["group_cols"] == cap
    ref = oracle.ryser(A).value
    assert pins.scaled_error(got, ref, A) <= TOL, (got, ref, info)
    monkeypatch.setenv("PERM_SPARSE_GROUP", "0")
    plain, info0 = pb.perm_c128_sparse(A, info=True)
    assert info0["group_cols"] == 0
    assert pins.scaled_error(got, plain, A) <= TOL, (got, plain)


def test_sparse_group_walk_not_taken_for_thick_t_columns(monkeypatch):
    # every T column with more than 4 nonzero rows (density 0.4): the plain T walk
    B = _sparse(20, 0.4, 7800)
    T = pb.perm_sparse_plan(B)["T"]
    tc = [j for j in range(20) if (T >> j) & 1]
    assert len(tc) >= 5 and min(np.count_nonzero(B[:, j]) for j in tc) > 4
    monkeypatch.setenv("PERM_FORCE_CHUNK_LOG2", "4")
    got, info = pb.perm_c128_sparse(B, info=True)
    assert info["group_cols"] == 0 and info["chunk_log2"] == 4
    assert pins.scaled_error(got, oracle.ryser(B).value, B) <= TOL


@pytest.mark.parametrize("n", [32, 33, 47, 48])
def test_sparse_group_walk_block_diagonal(n, monkeypatch):
    # the group walk at the large constant-bank orders: scrambled block-diagonal matrices, per = product of the
    # blocks' permanents (oracle Eq. (3)); n = 47, 48 at the planned chunk length, n = 32, 33 forced to 2^5; the
    # plain T walk alongside
    sizes = [16] * (n // 16) + ([n % 16] if n % 16 else [])
    blocks = [_sparse(m, 0.05, 5300 + n + k) for k, m in enumerate(sizes)]
    ph = np.random.default_rng(5400 + n)
    blocks = [B + 3.0 * np.diag(np.exp(2j * np.pi * ph.random(B.shape[0]))) for B in blocks]
    M = np.zeros((n, n), complex)
    o = 0
    for B in blocks:
        M[o:o + B.shape[0], o:o + B.shape[0]] = B
        o += B.shape[0]
    rng = np.random.default_rng(5500 + n)
    M = M[rng.permutation(n)][:, rng.permutation(n)]
    if n <= 33:
        monkeypatch.setenv("PERM_FORCE_CHUNK_LOG2", "5")
    ref = np.prod([oracle.ryser(B).value for B in blocks])
    got, info = pb.perm_c128_sparse(M, info=True)
    assert info["group_cols"] >= 2, info
    assert pins.scaled_error(got, ref, M) <= TOL, (got, ref, info)
    monkeypatch.setenv("PERM_SPARSE_GROUP", "0")
    plain = pb.perm_c128_sparse(M)
    assert pins.scaled_error(got, plain, M) <= TOL, (got, plain)
