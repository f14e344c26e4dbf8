"""Development tool: one walk launch at order n over a fixed span (for ncu captures)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 44
span = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 32
A = inputs.complex_gaussian((n, n), 44)
ws = pb.make_workspace(n)
d = pb.perm_c128_range(A, 0, span, workspace=ws)
print("partial", d.value)
