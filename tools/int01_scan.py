"""Development tool: perm_int01 throughput on the config-3 batch (64 x n = 24) for the plan knobs in the
environment (PERM_INT01_WAVES, PERM_INT01_ROUNDS); best of 5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

A = torch.from_numpy(inputs.cfg3()).cuda()
B, n = A.shape[0], A.shape[1]
out = torch.empty((B, 2), dtype=torch.int64, device="cuda")
ws = torch.empty(pb.int01_workspace_bytes(n, B), dtype=torch.uint8, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pb.perm_int01(A, workspace=ws, out=out, as_int=False)
best = 1e9
for _ in range(5):
    s.record()
    pb.perm_int01(A, workspace=ws, out=out, as_int=False)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
ops = B * (1 << (n - 1)) * 2 * n
print(f"waves={os.environ.get('PERM_INT01_WAVES', '1')} rounds={os.environ.get('PERM_INT01_ROUNDS', '16')} "
      f"{best:.3f} ms  frac={ops / (best * 1e-3) / (148 * 128 * 1.965e9):.4f}", flush=True)
