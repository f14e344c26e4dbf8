"""Development tool: the block-diagonal sparse test matrices of tests/test_gpu_sparse.py through the
library named by $PERM_LIB (value, scaled error vs the oracle's block product, chunk length)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1904_06229_b200 as pb  # noqa: E402
from tests import pins  # noqa: E402
from tests.test_gpu_sparse import _sparse  # noqa: E402

tag = os.path.basename(os.environ.get("PERM_LIB", "libperm.so"))
for n in (21, 32, 47, 48):
    for dens in (0.25, 0.5):
        sizes = [16] * (n // 16) + ([n % 16] if n % 16 else [])
        blocks = [_sparse(m, dens, 4700 + n + k) for k, m in enumerate(sizes)]
        M = np.zeros((n, n), complex)
        o = 0
        for B in blocks:
            M[o:o + B.shape[0], o:o + B.shape[0]] = B
            o += B.shape[0]
        rng = np.random.default_rng(4800 + n)
        M = M[rng.permutation(n)][:, rng.permutation(n)]
        ref = np.prod([oracle.ryser(B).value for B in blocks])
        got, info = pb.perm_c128_sparse(M, info=True)
        print(tag, n, dens, repr(got), pins.scaled_error(got, ref, M), info["chunk_log2"], info["sets"], flush=True)
