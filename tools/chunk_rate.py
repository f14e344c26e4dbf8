"""Development tool: chunk-walk throughput (the bench's path: perm_c128_chunks) per order for the library named
by $PERM_LIB (default libperm.so).  Orders from $RATE_N (default 32..48); each timed launch walks whole rounds
of the resident walkers (or the whole permanent) for >= ~0.3 s, best of 3."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

tag = os.path.basename(os.environ.get("PERM_LIB", "libperm.so"))
orders = [int(x) for x in os.environ.get("RATE_N", ",".join(map(str, range(32, 49)))).split(",") if x]
peak = 148 * 64 * 2 * 1965e6
for n in orders:
    A = inputs.complex_gaussian((n, n), 44)
    b = pb.chunk_log2(n)
    C = 1 << (n - 1 - b)
    W = pb.chunk_walkers(n, b)
    per_round = W << b
    rounds = max(1, int(0.3 * 6e10 / per_round))
    cnt = min(C, W * rounds)
    parts = torch.empty((cnt, 4), dtype=torch.float64, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pb.perm_c128_chunks(A, 0, cnt, partials=parts)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        s.record()
        _, st = pb.perm_c128_chunks(A, 0, cnt, partials=parts, stats=True)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    terms = cnt << b
    print(f"{tag} n={n} b={b} chunks={cnt} const={st['const_path']} {terms / best:.4e} terms/s "
          f"frac={terms / best * 8 * n / peak:.4f}", flush=True)
