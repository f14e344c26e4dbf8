"""Development tool: perm_c128_range values and walk rates of the library named by $PERM_LIB on a few
n = 44 spans (aligned and unaligned), printed for comparison across library variants."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

tag = os.path.basename(os.environ.get("PERM_LIB", "libperm.so"))
n = int(os.environ.get("CMP_N", "44"))
A = inputs.cfg5() if n == 44 else inputs.complex_gaussian((n, n), n)
ws = pb.make_workspace(n)
spans = [(0, 1 << 30), (12345, (1 << 30) + 777), ((1 << 42) - (1 << 29), (1 << 42) + (1 << 29) + 5)]
for k0, k1 in spans:
    v = pb.perm_c128_range(A, k0, k1, workspace=ws)
    print(f"{tag} n={n} [{k0},{k1}) = {v!r}", flush=True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
span = int(os.environ.get("CMP_SPAN_LOG2", "37"))
for rep in range(3):
    s.record()
    pb.perm_c128_range(A, 0, 1 << span, workspace=ws)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    print(f"{tag} n={n} 2^{span} terms: {t:.4f} s  {(1 << span) / t:.4e} terms/s  "
          f"{(1 << span) / t * 8 * n / 37.22496e12:.4f} of FP64 peak", flush=True)
