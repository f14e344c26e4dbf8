"""GPU parity of the single-matrix walk (perm_c128 / perm_c128_range / perm_c128_seed) against the
CPU oracle.  Tolerance: BASELINE north_star scaled error |gpu - oracle| / max(|oracle|,
2^{-n/2} prod_i ||a_i||_2) <= 1e-9; exact equality where the arithmetic is exact (dyadic inputs)."""
from __future__ import annotations

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


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pb.lib()


def _dd_val(d):
    return d.value


def _golden(golden_dir):
    p = os.path.join(golden_dir, "oracle_values.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def _q(v):
    return complex(v[0] + v[1], v[2] + v[3])


# ------------------------------------------------------------------ exact App. A trace (n = 3)

def test_app_a_trace_exact(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "app_a_trace_n3.json")))
    A = np.array(g["A"], dtype=np.complex128)
    assert pb.perm_c128(A) == g["per"]
    terms = [g["terms_num_den"][r][0] / g["terms_num_den"][r][1] for r in range(4)]
    for k0 in range(5):
        for k1 in range(k0, 5):
            assert pb.perm_c128_range(A, k0, k1).value == sum(terms[k0:k1]), (k0, k1)
    w = pb.perm_c128_seed(A, [0, 1, 2, 3])
    for r in range(4):
        assert list(w[r]) == [a / b for a, b in g["seeds_num_den"][r]]


def test_n1_n2():
    assert pb.perm_c128(np.array([[3 - 2j]])) == 3 - 2j
    a, b, c, d = 1.5 + 2j, -0.25 + 1j, 3 - 1j, 0.5 + 0.5j
    assert pb.perm_c128(np.array([[a, b], [c, d]])) == a * d + b * c


# ------------------------------------------------------------------ random complex vs oracle, n = 1..26

@pytest.mark.parametrize("n", list(range(1, 27)))
def test_gaussian_vs_oracle(n):
    A = inputs.complex_gaussian((n, n), 1000 + n)
    ref = oracle.naive(A).value if n <= 8 else (oracle.ryser(A).value if n <= 14 else oracle.permanent_hr(A).value)
    got = pb.perm_c128(A)
    assert pins.scaled_error(got, ref, A) <= TOL, (n, got, ref)


@pytest.mark.parametrize("n", [5, 12, 16, 21])
def test_haar_block_vs_oracle(n):
    U = inputs.haar_unitary(4 * n, 77 + n)
    A = np.ascontiguousarray(U[:n, :n])
    ref = oracle.permanent_hr(A).value
    assert pins.scaled_error(pb.perm_c128(A), ref, A) <= TOL


def test_device_input_and_device_output():
    import torch
    A = inputs.complex_gaussian((18, 18), 5)
    ref = oracle.permanent_hr(A).value
    At = torch.from_numpy(A).cuda()
    out = torch.zeros(1, dtype=torch.complex128, device="cuda")
    ws = pb.make_workspace(18)
    pb.perm_c128(At, workspace=ws, out=out)
    torch.cuda.synchronize()
    assert pins.scaled_error(complex(out.item()), ref, A) <= TOL
    assert pins.scaled_error(pb.perm_c128(At), ref, A) <= TOL


# ------------------------------------------------------------------ closed forms

@pytest.mark.parametrize("n", [1, 2, 5, 10, 16, 20, 24])
def test_identity_ones_derangement(n):
    assert pb.perm_c128(np.eye(n, dtype=np.complex128)) == 1
    d = (np.arange(1, n + 1) * (1 + 0.5j)).astype(np.complex128)
    ref = complex(np.prod(d))
    assert pins.scaled_error(pb.perm_c128(np.diag(d)), ref, np.diag(d)) <= 1e-14
    J = np.ones((n, n), dtype=np.complex128)
    got = pb.perm_c128(J)
    assert abs(got - math.factorial(n)) <= 1e-12 * math.factorial(n)
    D = pins.derangements(n)
    got = pb.perm_c128(pins.j_minus_i(n).astype(np.complex128))
    assert abs(got - D) <= 1e-12 * max(D, 1)


@pytest.mark.parametrize("n", [28, 32])
def test_ones_precision_curve(n):
    # P1: relative error on J_n; the paper's double-quad line is 10^{0.20 n - 18}
    got = pb.perm_c128(np.ones((n, n), dtype=np.complex128))
    rel = abs(got - math.factorial(n)) / math.factorial(n)
    assert rel <= max(1e-9, 10 ** (0.20 * n - 18))


def test_zero_row_and_invariances():
    A = inputs.complex_gaussian((20, 20), 99)
    Z = A.copy()
    Z[7] = 0
    assert pb.perm_c128(Z) == 0
    p = pb.perm_c128(A)
    rng = np.random.default_rng(1)
    for B in (A.T.copy(), A[rng.permutation(20)][:, rng.permutation(20)].copy()):
        assert pins.scaled_error(pb.perm_c128(B), p, A) <= 1e-11


def test_multilinearity_row():
    n = 22
    A = inputs.complex_gaussian((n, n), 3)
    u, v = inputs.complex_gaussian((2, n), 4)
    al, be = 0.5 - 1j, 2.0 + 0.25j
    Au, Av, Aw = A.copy(), A.copy(), A.copy()
    Au[3], Av[3], Aw[3] = u, v, al * u + be * v
    lhs = pb.perm_c128(Aw)
    rhs = al * pb.perm_c128(Au) + be * pb.perm_c128(Av)
    assert pins.scaled_error(lhs, rhs, Aw) <= 1e-10


def test_nonfinite_rejected():
    A = np.eye(4, dtype=np.complex128)
    A[1, 2] = np.nan
    with pytest.raises(pb.PermError) as e:
        pb.perm_c128(A)
    assert e.value.name == "PERM_E_NONFINITE"


# ------------------------------------------------------------------ range API

@pytest.mark.parametrize("n", [7, 20, 33, 44, 64])
def test_range_random_spans(n):
    A = inputs.complex_gaussian((n, n), 2000 + n)
    N = 1 << (n - 1)
    rng = np.random.default_rng(n)
    spans = [(0, min(N, 1000)), (N - min(N, 777), N)]
    for _ in range(4):
        k0 = int(rng.integers(0, N))
        k1 = min(N, k0 + int(rng.integers(0, 5000)))
        spans.append((k0, k1))
    for k0, k1 in spans:
        got = pb.perm_c128_range(A, k0, k1).value
        ref = oracle.subpermanent(A, k0, k1 - k0).value if k1 > k0 else 0
        scale = max(abs(ref), pins.range_scale(A, k1 - k0))
        assert abs(got - ref) <= 1e-12 * scale, (n, k0, k1, got, ref)


@pytest.mark.parametrize("n", [32, 34, 35, 37, 39, 42, 43, 44, 45])
def test_const_bank_walk_orders(n, monkeypatch):
    # the constant-bank kernels (uniform-register column operands) for every order that uses them:
    # PERM_FORCE_CHUNK_LOG2 = 3 makes a 2^16-term span an aligned body of 8-term chunks (e > U), which is
    # what the planner hands to walk_kernel_c; the head/tail pieces of the unaligned span go to walk_kernel
    monkeypatch.setenv("PERM_FORCE_CHUNK_LOG2", "3")
    A = inputs.complex_gaussian((n, n), 3000 + n)
    N = 1 << (n - 1)
    rng = np.random.default_rng(3000 + n)
    for k0 in (0, int(rng.integers(0, N - (1 << 17))) | 5):
        k1 = k0 + (1 << 16) + 3
        got = pb.perm_c128_range(A, k0, k1).value
        ref = oracle.subpermanent(A, k0, k1 - k0).value
        scale = max(abs(ref), pins.range_scale(A, k1 - k0))
        assert abs(got - ref) <= 1e-12 * scale, (n, k0, got, ref)


def test_range_empty_is_zero():
    A = inputs.complex_gaussian((10, 10), 1)
    assert pb.perm_c128_range(A, 17, 17).value == 0


def test_partition_additivity():
    n = 24
    A = inputs.complex_gaussian((n, n), 24)
    N = 1 << (n - 1)
    ref = pb.perm_c128(A)
    for G in (1, 2, 3, 4, 7, 8, 16):
        parts = [pb.perm_c128_range(A, *_span(N, G, i)) for i in range(G)]
        got = pb.perm_c128_finalize(parts, n)
        assert pins.scaled_error(got, ref, A) <= 1e-12, G


def _span(N, G, i):
    q, r = divmod(N, G)
    k = i * q + min(i, r)
    return k, k + q + (1 if i < r else 0)


def test_determinism():
    A = inputs.complex_gaussian((26, 26), 7)
    a = pb.perm_c128(A, return_dd=True)[1].astuple()
    b = pb.perm_c128(A, return_dd=True)[1].astuple()
    assert a == b


def test_seed_kernel_vs_oracle():
    for n in (3, 17, 44, 64):
        A = inputs.complex_gaussian((n, n), 300 + n)
        N = 1 << (n - 1)
        ranks = [0, 1, 2, N - 1, N // 2, N // 3, 12345 % N]
        w = pb.perm_c128_seed(A, ranks)
        for k, r in enumerate(ranks):
            ref = oracle.seed(A, r)
            assert np.max(np.abs(w[k] - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)) * n), (n, r)


# ------------------------------------------------------------------ BASELINE configs

def test_cfg1_vs_golden(golden_dir):
    g = _golden(golden_dir).get("cfg1")
    A = inputs.cfg1()
    ref = _q(g["value"]) if g else oracle.ryser(A).value
    assert pins.scaled_error(pb.perm_c128(A), ref, A) <= TOL


def test_cfg4_subranges(golden_dir):
    g = _golden(golden_dir).get("ranges32")
    if not g:
        pytest.skip("oracle_values.json has no ranges32 section")
    A = inputs.cfg4()
    for rr in g["ranges"]:
        got = pb.perm_c128_range(A, rr["k0"], rr["k1"]).value
        ref = _q(rr["value"])
        assert abs(got - ref) <= 1e-12 * max(abs(ref), pins.range_scale(A, rr["k1"] - rr["k0"]))


def test_cfg4_full_vs_golden(golden_dir):
    g = _golden(golden_dir).get("cfg4")
    if not g:
        pytest.skip("oracle_values.json has no cfg4 section yet")
    A = inputs.cfg4()
    assert pins.scaled_error(pb.perm_c128(A), _q(g["value"]), A) <= TOL


def test_cfg5_subranges(golden_dir):
    g = _golden(golden_dir).get("ranges44")
    if not g:
        pytest.skip("oracle_values.json has no ranges44 section")
    A = inputs.cfg5()
    for rr in g["ranges"]:
        got = pb.perm_c128_range(A, rr["k0"], rr["k1"]).value
        ref = _q(rr["value"])
        assert abs(got - ref) <= 1e-12 * max(abs(ref), pins.range_scale(A, rr["k1"] - rr["k0"]))

# The n = 44 block-diagonal full walk (P7) runs on the bench's path in tests/test_gpu_chunks.py.


@pytest.mark.parametrize("n", [32, 44])
def test_unit_column_walk_scale_and_fallback(n):
    # the unit-column walk: rows of very different scale (the normalisation's product of the column-0
    # entries spans 1e-200 .. 1e200) and a column-0 entry 1e-120 times its row (the plain walk) -- App. A span sums
    # against the oracle within the range bar
    A = inputs.complex_gaussian((n, n), 4400 + n)
    A[1, :] *= 1e-100
    A[2, :] *= 1e100
    B = A.copy()
    B[7, 0] = 1e-121 * B[7, 0]
    N = 1 << (n - 1)
    for M in (A, B):
        for k0 in (0, N // 3):
            k1 = k0 + (1 << 20)
            got = pb.perm_c128_range(M, k0, k1).value
            ref = oracle.subpermanent(M, k0, k1 - k0).value
            scale = max(abs(ref), pins.range_scale(M, k1 - k0))
            assert abs(got - ref) <= 1e-12 * scale, (n, k0, got, ref)
