"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Sizes are tiny so the instrumented run finishes in seconds; results are checked loosely (the parity
tests do the real checking)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs, shard  # noqa: E402

torch.cuda.set_device(0)
vals = []
for n in (3, 12, 16):                                   # walk_small_kernel (cluster, DSMEM)
    vals.append(pb.perm_c128(inputs.complex_gaussian((n, n), n)))
for n in (20, 33, 44):                                  # chunk walk (smem / constant bank) + tree
    A = inputs.complex_gaussian((n, n), n)
    b = pb.chunk_log2(n)
    c0 = 5
    c1 = c0 + 300
    parts = pb.perm_c128_chunks(A, c0, c1)
    nodes = pb.perm_c128_tree(parts, c0, c1)
    vals.append(shard.combine_nodes(nodes.cpu().numpy(), n, expect_root=False))
A = inputs.complex_gaussian((20, 20), 7)
vals.append(pb.perm_c128(A))                            # whole permanent through the multi-launch path
vals.append(pb.perm_c128_range(A, 1234, 99999).value)   # range API with edge pieces
Ab = torch.from_numpy(inputs.cfg2(8, 256)).cuda()
pb.perm_c128_batched(Ab)
pb.perm_c128_batched_x(torch.from_numpy(inputs.circular((64, 12, 12), 3)).cuda())
vals += pb.perm_int01(torch.from_numpy(inputs.bernoulli01((8, 12, 12), 4)).cuda())
vals += pb.perm_pm1(torch.from_numpy(inputs.bernoulli_pm1((8, 12, 12), 5)).cuda())
C, M = inputs.collision_patterns(10, 10, 16, 6)
pb.perm_c128_weighted_batched(torch.from_numpy(C).cuda(), torch.from_numpy(M).cuda())
Bd = inputs.band_gaussian((16, 40, 40), 3, 8)
pb.perm_c128_band_batched(torch.from_numpy(pb.band_storage(Bd, 3)).cuda(), 3)
vals.append(pb.perm_c128_sparse(inputs.sparse_gaussian(24, 0.1, 9)))
torch.cuda.synchronize()
print("sanitize cases ok:", len(vals), "values, finite:", all(np.isfinite(complex(v)) for v in vals))
