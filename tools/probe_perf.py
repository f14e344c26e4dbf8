"""Quick GPU throughput probe (development tool): FP64 peak probe, walk throughput at several n,
batched and int01 timings.  Prints one line per measurement."""
from __future__ import annotations

import sys
import time

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs


def ev_time(fn, reps=3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def main():
    dev = torch.cuda.get_device_properties(0)
    sms = dev.multi_processor_count
    print("device", dev.name, "SMs", sms, flush=True)
    sink = torch.empty(sms * 4 * 256, dtype=torch.float64, device="cuda")
    for blocks_per_sm, thr in ((4, 256), (8, 256), (2, 512)):
        iters = 20000
        t = ev_time(lambda: pb.perm_fp64_probe(sms * blocks_per_sm, thr, iters, sink))
        fl = sms * blocks_per_sm * thr * iters * 64
        print(f"fp64 probe {blocks_per_sm}x{thr}: {fl / t / 1e12:.2f} TFLOP/s", flush=True)
    for n, span in ((16, None), (24, None), (32, None), (44, 1 << 36)):
        A = inputs.complex_gaussian((n, n), 44)
        ws = pb.make_workspace(n)
        if span is None:
            f = lambda: pb.perm_c128(A, workspace=ws)
            terms = 1 << (n - 1)
        else:
            f = lambda: pb.perm_c128_range(A, 0, span, workspace=ws)
            terms = span
        t = ev_time(f, reps=3)
        _, st = (pb.perm_c128(A, workspace=ws, stats=True) if span is None else pb.perm_c128_range(A, 0, span, workspace=ws, stats=True))
        rate = terms / t
        print(f"walk n={n}: {t*1e3:.3f} ms  {rate:.3e} terms/s  {rate*8*n/1e12:.2f} TFLOP/s(8n)  stats={st}", flush=True)
    for n in (8, 12, 16, 20):
        A = torch.from_numpy(inputs.cfg2(n, 100000 if n < 20 else 20000)).cuda()
        t = ev_time(lambda: pb.perm_c128_batched(A), reps=3)
        B = A.shape[0]
        print(f"batched n={n} B={B}: {t*1e3:.3f} ms  {B/t:.3e} perms/s  {B*2**(n-1)*8*n/t/1e12:.2f} TFLOP/s", flush=True)
    A = torch.from_numpy(inputs.cfg3()).cuda()
    t = ev_time(lambda: pb.perm_int01(A, as_int=False), reps=3)
    print(f"int01 n=24 B=64: {t*1e3:.3f} ms  {64*2**23/t:.3e} terms/s", flush=True)


if __name__ == "__main__":
    main()
