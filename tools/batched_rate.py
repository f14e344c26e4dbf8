"""Development tool: perm_c128_batched throughput on the config-2 batches (10^5 submatrices of a Haar unitary per
n in $RATE_N, default 8,12,16,20) for the library in $PERM_LIB; best of 3 per n, and the whole config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1904_06229_b200 as pb  # noqa: E402
from paper_1904_06229_b200 import inputs  # noqa: E402

tag = os.path.basename(os.environ.get("PERM_LIB", "libperm.so"))
peak = 148 * 64 * 2 * 1965e6
tot_t = tot_f = 0.0
for n in [int(x) for x in os.environ.get("RATE_N", "8,12,16,20").split(",")]:
    A = torch.from_numpy(inputs.cfg2(n)).cuda()
    per, abs2 = pb.perm_c128_batched(A)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        s.record()
        pb.perm_c128_batched(A, per=per, abs2=abs2)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    flops = A.shape[0] * (1 << (n - 1)) * 8 * n
    tot_t += best
    tot_f += flops
    print(f"{tag} n={n} {best * 1e3:.3f} ms {A.shape[0] / best:.4g} perms/s frac={flops / best / peak:.4f} "
          f"per[0]={complex(per[0].item())}", flush=True)
print(f"{tag} all: {tot_t * 1e3:.3f} ms frac={tot_f / tot_t / peak:.4f}", flush=True)
