"""Development tool: one bench-shaped step of the chunk walk at order n for ncu captures: `rounds` whole rounds
of the resident walkers (perm_c128_chunks) and the tree of the slice (perm_c128_tree).
    python tools/ncu_chunks.py [n=44] [rounds=1]"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 44
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A = inputs.cfg5() if n == 44 else inputs.complex_gaussian((n, n), 44)
W = pb.chunk_walkers(n)
cnt = min(1 << (n - 1 - pb.chunk_log2(n)), W * rounds)
parts = pb.perm_c128_chunks(A, 0, cnt)
nodes = pb.perm_c128_tree(parts, 0, cnt)
print("chunks", cnt, "nodes", len(pb.tree_nodes(nodes.cpu().numpy())))
