"""Development tool: one constant-bank sparse launch on the cfgsp matrix (n = 48), for ncu captures."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

print(pb.perm_c128_sparse(inputs.cfgsp()))
