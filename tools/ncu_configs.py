"""Development tool: one launch of each bench configuration's dominant kernel, in the bench's launch
configuration, for `ncu --set full` captures (configs 1-4; config 5's 2^43-term launch is captured on a
2^34-term sub-range with tools/ncu_walk.py at the bench's chunk length, PERM_FORCE_CHUNK_LOG2=20)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

which = sys.argv[1:] or ["cfg1", "cfg4", "cfg2", "cfg3"]
if "cfg1" in which:
    print("cfg1", pb.perm_c128(inputs.cfg1()))
if "cfg4" in which:
    print("cfg4", pb.perm_c128(inputs.cfg4()))
if "cfg2" in which:
    for n in (8, 12, 16, 20):
        A = torch.from_numpy(inputs.cfg2(n, 100000)).cuda()
        per, abs2 = pb.perm_c128_batched(A)
        torch.cuda.synchronize()
        print("cfg2", n, float(abs2[0]))
if "cfg3" in which:
    print("cfg3", pb.perm_int01(torch.from_numpy(inputs.cfg3()).cuda())[0])
