"""Development tool: device time of one perm_c128 call replayed from a CUDA graph (device-resident matrix,
device output), per order n -- the latency of the small-permanent path."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

for n in [int(x) for x in os.environ.get("SMALL_N", "2,4,8,10,12,14,15,16,17,18,20").split(",")]:
    A = torch.from_numpy(inputs.complex_gaussian((n, n), 16)).cuda()
    out = torch.empty(1, dtype=torch.complex128, device="cuda")
    ws = pb.make_workspace(n)
    pb.perm_c128(A, workspace=ws, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pb.perm_c128(A, workspace=ws, out=out, stream=torch.cuda.current_stream())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    reps = 500
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    print(f"n={n:2d} chunks={1 << (n - 1 - pb.chunk_log2(n))} {s.elapsed_time(e) / reps * 1e3:.2f} us per call "
          f"(back-to-back replays)", flush=True)
