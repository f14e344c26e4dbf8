"""Development tool: perm_c128_weighted_batched throughput on the cfgw workload for the library named by
$PERM_LIB; best of 5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

C, M = inputs.cfgw()
Cd, Md = torch.from_numpy(C).cuda(), torch.from_numpy(M).cuda()
per = torch.empty(C.shape[0], dtype=torch.complex128, device="cuda")
pb.perm_c128_weighted_batched(Cd, Md, per=per, want_abs2=False)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") == "1" else None
for _ in range(5):
    if flush is not None:
        flush.fill_(1)                     # evict L2 (as bench.py does between steps)
    s.record()
    pb.perm_c128_weighted_batched(Cd, Md, per=per, want_abs2=False)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
terms = float(np.sum(np.prod(M.astype(np.float64) + 1.0, axis=1)))
print(f"{os.path.basename(os.environ.get('PERM_LIB', 'libperm.so'))}: {best:.3f} ms  {C.shape[0] / best * 1e3:.4g} perms/s "
      f"frac={terms * 8 * 20 / (best * 1e-3) / 37.22e12:.4f}  per[0]={complex(per[0].item())}", flush=True)
