"""GPU parity of perm_c128_band_batched (App. C bandpermanent) against
the oracle's literal App. C polynomial and Eq. (3)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs
from tests import pins

pytestmark = pytest.mark.gpu
REL = 1e-12      # |Δ| <= REL * per(|A|): the sum of the magnitudes of all band paths (R19)


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _run(torch, A, k):
    per, abs2 = pb.perm_c128_band_batched(torch.from_numpy(pb.band_storage(A, k)).cuda(), k)
    torch.cuda.synchronize()
    return per.cpu().numpy(), abs2.cpu().numpy()


@pytest.mark.parametrize("n,k", [(1, 0), (2, 1), (5, 0), (6, 2), (9, 3), (16, 4), (20, 5), (24, 6), (40, 3),
                                 (100, 5), (257, 2)])
def test_band_vs_oracle(torch, n, k):
    A = inputs.band_gaussian((5, n), k, 1000 * k + n)
    per, abs2 = _run(torch, A, k)
    for b in range(A.shape[0]):
        ref = oracle.band(A[b], k).value
        scale = oracle.band(np.abs(A[b]).astype(complex), k).value.real
        assert abs(per[b] - ref) <= REL * scale, (n, k, b, per[b], ref)
        assert abs2[b] == per[b].real ** 2 + per[b].imag ** 2
        if n <= 16:
            assert abs(per[b] - oracle.ryser(A[b]).value) <= 1e-11 * scale


def test_band_closed_forms(torch):
    for n in (1, 3, 30, 70):
        per, _ = _run(torch, pins.tridiagonal_ones(n).astype(complex)[None], min(1, n - 1))
        assert per[0] == pins.fibonacci(n + 1)                     # integers < 2^53: exact
    d = (np.arange(1, 31) % 5 + 1) * (1 - 0.5j)
    per, _ = _run(torch, np.diag(d)[None], 0)
    assert abs(per[0] - np.prod(d)) <= 1e-14 * abs(np.prod(d))


def test_band_errors_and_empty(torch):
    x = torch.zeros((2, 4, 15), dtype=torch.complex128, device="cuda")
    with pytest.raises(pb.PermError):
        pb.perm_c128_band_batched(x, 7)                            # k > 6
    y = torch.zeros((2, 3, 9), dtype=torch.complex128, device="cuda")
    with pytest.raises(pb.PermError):
        pb.perm_c128_band_batched(y, 4)                            # k > n - 1
    e, a = pb.perm_c128_band_batched(torch.zeros((0, 8, 5), dtype=torch.complex128, device="cuda"), 2)
    assert e.shape[0] == 0
