"""Development tool: perm_int01 throughput on the config-3 batch (64 x n = 24), best of 5, for the build in PERM_LIB
and the knobs in the environment (PERM_INT01_WAVES, PERM_INT01_ROUNDS, PERM_INT01_ZSPLIT); checks the 64 values
against the oracle golden (tests/golden/oracle_values.json, written by make_oracle_values.py from oracle/ only)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
A = torch.from_numpy(inputs.cfg3() if which == "cfg3" else inputs.bernoulli_pm1((1024, 24, 24), 5)).cuda()
B, n = A.shape[0], A.shape[1]
ok = "unchecked"
if which == "cfg3":
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_values.json")))["cfg3"]["values"]
    ok = "exact" if pb.perm_int01(A) == [int(v) for v in gold] else "MISMATCH"
fn = pb.perm_int01 if which == "cfg3" else pb.perm_pm1
out = torch.empty((B, 2), dtype=torch.int64, device="cuda")
ws = torch.empty(pb.int01_workspace_bytes(n, B), dtype=torch.uint8, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fn(A, workspace=ws, out=out, as_int=False)
best = 1e9
for _ in range(5):
    s.record()
    fn(A, workspace=ws, out=out, as_int=False)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
ops = B * (1 << (n - 1)) * 2 * n
print(f"{which} lib={os.path.basename(os.environ.get('PERM_LIB', 'libperm.so'))} "
      f"zsplit={os.environ.get('PERM_INT01_ZSPLIT', '1')} waves={os.environ.get('PERM_INT01_WAVES', '-')} "
      f"rounds={os.environ.get('PERM_INT01_ROUNDS', '-')} {best:.3f} ms  frac={ops / (best * 1e-3) / (148 * 128 * 1.965e9):.4f} "
      f"{ok}", flush=True)
