"""GPU: the Sec. III-IV ensembles through the batched kernel with the X = |per|/sqrt(n!) output (SURVEY 8(f)
NEXT-2; P:451-464 Ginibre, P:717-725 circular).  Parity of X against the oracle per matrix, and the exact
second moment E[X^2] = 1 (P:461-464 Ginibre; "again exactly 1", P:723 circular) plus E[X^4] = n + 1 for
Ginibre as 5-sigma statistical pins on large batches."""
from __future__ import annotations

import math

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


@pytest.mark.parametrize("gen,n", [("ginibre", 5), ("ginibre", 13), ("circular", 7), ("circular", 16),
                                   ("circular", 24)])
def test_x_output_vs_oracle(torch, gen, n):
    count = 40 if n < 20 else 6
    A = (inputs.complex_gaussian((count, n, n), 50 + n) if gen == "ginibre" else inputs.circular((count, n, n), 60 + n))
    per, abs2, x = pb.perm_c128_batched_x(torch.from_numpy(A).cuda(), want_per=True, want_abs2=True)
    per, abs2, x = per.cpu().numpy(), abs2.cpu().numpy(), x.cpu().numpy()
    ref = oracle.ryser_batch(A)
    for b in range(count):
        assert pins.scaled_error(per[b], ref[b], A[b]) <= 1e-9
        assert x[b] == math.sqrt(abs2[b] / float(math.factorial(n))) or \
            abs(x[b] - math.sqrt(abs2[b] / math.factorial(n))) <= 1e-15 * x[b]
        floor = pins.scaled_floor(A[b]) / math.sqrt(math.factorial(n))
        assert abs(x[b] - abs(ref[b]) / math.sqrt(math.factorial(n))) <= 1e-9 * max(x[b], floor)


def test_x_only_and_argument_errors(torch):
    A = torch.from_numpy(inputs.circular((3, 6, 6), 1)).cuda()
    per, abs2, x = pb.perm_c128_batched_x(A)
    assert per is None and abs2 is None and x.shape == (3,)
    L = pb.lib()
    assert L.perm_c128_batched_x(None, 6, 1, None, None, None, None) == 1
    assert L.perm_c128_batched_x(None, 33, 1, None, None, None, None) == 2
    assert L.perm_c128_batched_x(None, 6, 0, None, None, None, None) == 0


@pytest.mark.parametrize("gen", ["ginibre", "circular"])
def test_second_moment_is_one(torch, gen):
    n, count = 10, 200_000
    A = inputs.complex_gaussian((count, n, n), 7) if gen == "ginibre" else inputs.circular((count, n, n), 8)
    _, _, x = pb.perm_c128_batched_x(torch.from_numpy(A).cuda())
    X2 = x.cpu().numpy() ** 2
    m, sd = X2.mean(), X2.std() / math.sqrt(count)
    assert abs(m - 1.0) <= 5 * sd, (gen, m, sd)
    if gen == "ginibre":
        X4 = X2 ** 2
        m4, sd4 = X4.mean(), X4.std() / math.sqrt(count)
        assert abs(m4 - (n + 1)) <= 5 * sd4, (m4, sd4)
