"""Development tool: walk throughput for the library named by $PERM_LIB (default libperm.so)."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402


def ev(fn, reps=3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


tag = os.path.basename(os.environ.get("PERM_LIB", "libperm.so"))
ORDERS = os.environ.get("WALK_RATE_N", "20,32,44")
for n, span in [(int(x), (1 << 36) if int(x) > 36 else None) for x in ORDERS.split(",") if x]:
    A = inputs.complex_gaussian((n, n), 44)
    ws = pb.make_workspace(n)
    terms = span or (1 << (n - 1))
    t = ev(lambda: pb.perm_c128_range(A, 0, terms, workspace=ws))
    print(f"{tag} n={n}: {terms / t:.4e} terms/s  {terms / t * 8 * n / 1e12:.2f} TF", flush=True)
if os.environ.get("WALK_RATE_BATCHED", "1") == "1":
    A = torch.from_numpy(inputs.cfg2(16, 100000)).cuda()
    t = ev(lambda: pb.perm_c128_batched(A))
    print(f"{tag} batched16: {1e5 / t:.4e} perms/s {1e5 * 2**15 * 128 / t / 1e12:.2f} TF", flush=True)
