"""Relative error of per(J_n) = n! (pin P1) computed by perm_c128 on the GPU, n = 10..40, against the paper's
fitted lines for log10 of the relative error (Fig. error caption): 0.37n - 17.8 (double, 1 core),
0.30n - 17.2 (double, multi-core/node), 0.20n - 18 (double-quadruple).  Output: one line per n."""
from __future__ import annotations

import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402

lo, hi = (int(x) for x in os.environ.get("JN_RANGE", "10,40").split(","))
print("n  per_gpu(re)  rel_err  log10(rel_err)  paper: double_1core double_multi double_quad")
for n in range(lo, hi + 1):
    v = pb.perm_c128(np.ones((n, n), dtype=np.complex128))
    f = math.factorial(n)
    rel = abs(v - f) / f
    lg = math.log10(rel) if rel > 0 else float("-inf")
    print(f"{n:2d} {v.real:.17e} {rel:.3e} {lg:7.2f}   {0.37 * n - 17.8:6.2f} {0.30 * n - 17.2:6.2f} "
          f"{0.20 * n - 18:6.2f}", flush=True)
