"""Development tool: perm_c128_sparse rate (sets/s) with the shared-rows group walk capped at G = 4, 3, 2, 1, 0
(PERM_SPARSE_GROUP; 0 = the plain T walk)
for sparse Gaussian matrices of the constant-bank orders; the two values' scaled difference alongside."""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402
from tests import pins  # noqa: E402

cases = [(int(a.split(":")[0]), float(a.split(":")[1])) for a in sys.argv[1:]] or [(48, 0.04)]
for n, dens in cases:
    A = inputs.cfgsp() if (n, dens) == (48, 0.04) else inputs.sparse_gaussian(n, dens, 900 + n)
    res = {}
    for pair in ("4", "3", "2", "1", "0"):
        os.environ["PERM_SPARSE_GROUP"] = pair
        v, info = pb.perm_c128_sparse(A, info=True)                      # warm-up (and the plan)
        best = 1e30
        for _ in range(3):
            t0 = time.perf_counter()
            v = pb.perm_c128_sparse(A)
            best = min(best, time.perf_counter() - t0)
        res[pair] = v
        print(f"n={n} dens={dens} group_cols={info['group_cols']} e={info['chunk_log2']} sets={info['sets']:.3g} "
              f"{best * 1e3:.2f} ms {info['sets'] / best:.4g} sets/s value={v!r}", flush=True)
    for g in ("4", "3", "2", "1"):
        print(f"n={n} G<={g}: scaled |group - plain| = {pins.scaled_error(res[g], res['0'], A):.3g}", flush=True)
