"""Debug: per-chunk partials of one launch over a chunk span vs. the same chunks walked in several launches
(slices / simulated ranks); reports the first chunks whose dd partials differ bitwise."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs, shard

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
A = inputs.cfg4() if n == 32 else inputs.complex_gaussian((n, n), 6000 + n)
b = pb.chunk_log2(n)
C = 1 << (n - 1 - b)
full = pb.perm_c128_chunks(A, 0, C).cpu().numpy()
v, d = pb.perm_c128(A, return_dd=True)
nodes = pb.perm_c128_tree(torch.from_numpy(full).cuda(), 0, C).cpu().numpy()
print("perm_c128", d.astuple(), "tree-of-full", pb.perm_c128_tree_combine(nodes))
for world, steps in ((2, 1), (3, 2), (2, 4)):
    allnodes = []
    for r in range(world):
        c0, c1 = shard.chunk_span(n, world, r, b)
        wave = pb.chunk_walkers(n, b)
        for s0, s1 in shard.step_slices(c0, c1, steps, wave):
            if s1 == s0:
                continue
            part = pb.perm_c128_chunks(A, s0, s1).cpu().numpy()
            diff = np.nonzero(np.any(part != full[s0:s1], axis=1))[0]
            if diff.size:
                print(f"world {world} steps {steps} slice [{s0},{s1}): {diff.size} chunks differ, first {diff[:5] + s0}",
                      part[diff[0]], full[s0 + diff[0]])
            allnodes.append(pb.perm_c128_tree(torch.from_numpy(part).cuda(), s0, s1).cpu().numpy())
    raw, lvl = pb.perm_c128_tree_combine(np.concatenate(allnodes))
    print(world, steps, raw.astuple(), lvl)
