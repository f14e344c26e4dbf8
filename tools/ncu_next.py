"""Development tool: one launch of each §8(f) kernel in its bench configuration, for ncu captures."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

which = sys.argv[1:] or ["cfgw", "cfgpm", "cfgsp", "cfgbd"]
if "cfgw" in which:
    C, M = inputs.cfgw()
    pb.perm_c128_weighted_batched(torch.from_numpy(C).cuda(), torch.from_numpy(M).cuda())
if "cfgpm" in which:
    pb.perm_pm1(torch.from_numpy(inputs.bernoulli_pm1((1024, 24, 24), inputs.SEEDS["cfgpm"])).cuda())
if "cfgsp" in which:
    # a smaller instance of the cfgsp recipe (n = 40) so that ncu's replay stays short
    print(pb.perm_c128_sparse(inputs.sparse_gaussian(40, 0.04 * 48 / 40, inputs.SEEDS["cfgsp"])))
if "cfgbd" in which:
    pb.perm_c128_band_batched(torch.from_numpy(pb.band_storage(inputs.cfgbd(), 5)).cuda(), 5)
torch.cuda.synchronize()
