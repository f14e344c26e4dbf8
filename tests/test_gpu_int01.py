"""GPU parity of perm_int01 (BASELINE config 3): bit-exact against the CPU oracle."""
from __future__ import annotations

import hashlib
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


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _run(torch, A):
    return pb.perm_int01(torch.from_numpy(np.ascontiguousarray(A, dtype=np.uint8)).cuda())


@pytest.mark.parametrize("n", list(range(1, 15)))
def test_random_vs_oracle(torch, n):
    A = inputs.bernoulli01((13, n, n), 700 + n)
    assert _run(torch, A) == oracle.ryser_i01_batch(A)


def test_dense_and_sparse(torch):
    rng = np.random.default_rng(5)
    for p in (0.1, 0.5, 0.9):
        A = (rng.random((5, 12, 12)) < p).astype(np.uint8)
        assert _run(torch, A) == oracle.ryser_i01_batch(A)


@pytest.mark.parametrize("n", [20, 24, 26, 28, 29, 31, 33])
def test_closed_forms(torch, n):
    # n >= 29 runs the full-range Ryser walk (2^n subsets): the same closed forms, exact in int128
    mats = [np.ones((n, n), np.uint8), np.eye(n, dtype=np.uint8), pins.j_minus_i(n), pins.tridiagonal_ones(n),
            pins.hessenberg_ones(n), pins.identity_plus_shift(n), pins.menage_matrix(n),
            np.zeros((n, n), np.uint8)]
    expect = [math.factorial(n), 1, pins.derangements(n), pins.fibonacci(n + 1), 2 ** (n - 1), 2, pins.menage(n), 0]
    assert _run(torch, np.stack(mats)) == expect


def test_cfg3_bit_exact(torch, golden_dir):
    A = inputs.cfg3()
    p = os.path.join(golden_dir, "oracle_values.json")
    g = json.load(open(p)).get("cfg3") if os.path.exists(p) else None
    ref = [int(v) for v in g["values"]] if g else oracle.ryser_i01_batch(A)
    assert _run(torch, A) == ref


def test_not01_and_empty(torch):
    A = np.ones((2, 6, 6), np.uint8)
    A[1, 2, 3] = 2
    with pytest.raises(pb.PermError) as e:
        _run(torch, A)
    assert e.value.name == "PERM_E_NOT01"
    assert pb.perm_int01(torch.zeros((0, 5, 5), dtype=torch.uint8, device="cuda")) == []
    with pytest.raises(pb.PermError):
        _run(torch, np.ones((1, 34, 34), np.uint8))


def test_full_range_n29_vs_oracle(torch):
    # the Ryser (2^n subsets) branch against the int128 Eq. (3) oracle, 0-1 and +-1 entries
    A = inputs.bernoulli01((2, 29, 29), 2929)
    assert _run(torch, A) == oracle.ryser_i01_batch(A)
    P = inputs.bernoulli_pm1((1, 29, 29), 2930)
    assert pb.perm_pm1(torch.from_numpy(P).cuda()) == [oracle.ryser_i8(P[0])]


@pytest.mark.parametrize("n", [1, 2, 7, 12, 20, 24, 29])
def test_int01_range_partition_is_exact(torch, n):
    # one exact permanent from disjoint rank spans (perm_int01_range + perm_int01_finalize):
    # ragged and unaligned cuts, a single-rank span and an empty span, against the oracle's Eq. (3)
    from paper_1904_06229_b200 import shard
    A = inputs.bernoulli01((1, n, n), 3300 + n)
    ref = oracle.ryser_i01_batch(A)[0]
    Ad = torch.from_numpy(A[0]).cuda()
    N = shard.int01_rank_space(n)
    cuts = sorted({0, N, N // 3, N // 3 + 1, (N // 2) | 1, max(0, N - 5)})
    parts = [pb.perm_int01_range(Ad, cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
    parts.append(pb.perm_int01_range(Ad, N // 3, N // 3))              # empty span -> 0
    assert pb.perm_int01_finalize(parts, n) == ref
    assert pb.perm_int01_finalize([pb.perm_int01_range(Ad, 0, N)], n) == ref
    for G in (1, 3, 8):                                                  # distribute over G shards
        spans = [shard.rank_span(N, G, r) for r in range(G)]
        assert pb.perm_int01_finalize([pb.perm_int01_range(Ad, a, b) for a, b in spans], n) == ref


def test_int01_range_closed_forms_and_errors(torch):
    from paper_1904_06229_b200 import shard
    n = 26
    J = torch.ones((n, n), dtype=torch.uint8, device="cuda")
    N = shard.int01_rank_space(n)
    spans = [shard.rank_span(N, 5, r) for r in range(5)]
    assert pb.perm_int01_finalize([pb.perm_int01_range(J, a, b) for a, b in spans], n) == math.factorial(n)
    assert shard.sharded_int01(J) == math.factorial(n)                  # world = 1 path
    bad = J.clone()
    bad[3, 4] = 2
    with pytest.raises(pb.PermError) as e:
        pb.perm_int01_range(bad, 0, 1 << 10)
    assert e.value.name == "PERM_E_NOT01"
    with pytest.raises(pb.PermError) as e:
        pb.perm_int01_range(J, 0, N + 1)
    assert e.value.name == "PERM_E_ORDER"


# ---- the pair-factored walk: matrices whose largest column zero count z selects each menu entry
# (Glynn orders 20..24: Z = 18/16/14/12, below 12 the plain walk; full-range orders: n - 12 / n - 15 / n - 18)

@pytest.mark.parametrize("n,z", [(20, 18), (20, 19), (21, 16), (22, 14), (22, 15), (23, 12), (24, 13), (24, 11),
                                 (24, 17), (20, 20), (24, 24)])
def test_pair_factored_menu_vs_oracle(torch, n, z):
    A = np.stack([inputs.zero_column01(n, z, 5000 + 37 * n + z + k, col=k * (n - 2) // 2) for k in range(3)])
    assert _run(torch, A) == oracle.ryser_i01_batch(A)


@pytest.mark.parametrize("n", [20, 24])
def test_pair_factored_pm1_with_zeros(torch, n):
    # signed entries {-1, 0, 1}: the same plan (zero counts) on perm_pm1
    rng = np.random.default_rng(77 + n)
    P = rng.integers(-1, 2, size=(2, n, n)).astype(np.int8)
    P[0, rng.choice(n, 15, replace=False), 3] = 0
    got = pb.perm_pm1(torch.from_numpy(P).cuda())
    assert got == [oracle.ryser_i8(P[b]) for b in range(2)]


def test_pair_factored_full_range_goldens(torch, golden_dir):
    # 29 <= n <= 33 pair-factored walk at each menu entry, against oracle values written by make_oracle_values.py
    g = json.load(open(os.path.join(golden_dir, "oracle_values.json")))["int01_full"]
    for c in g["cases"]:
        A = inputs.zero_column01(c["n"], c["z"], c["seed"])
        assert hashlib.sha256(A.tobytes()).hexdigest() == c["sha256"], "generator changed: regenerate the golden"
        assert _run(torch, A[None]) == [int(c["value"])], c


def test_pair_factored_range_partition(torch):
    # perm_int01_range walks the same planned matrix: disjoint spans still finalize to per(A)
    from paper_1904_06229_b200 import shard
    A = inputs.zero_column01(22, 16, 2216)
    ref = oracle.ryser_i01_batch(A[None])[0]
    Ad = torch.from_numpy(A).cuda()
    N = shard.int01_rank_space(22)
    cuts = [0, 5, 1 << 10, (N // 3) | 1, N - 17, N]
    assert pb.perm_int01_finalize([pb.perm_int01_range(Ad, cuts[i], cuts[i + 1]) for i in range(5)], 22) == ref
