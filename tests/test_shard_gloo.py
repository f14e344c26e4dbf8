"""Multi-process host logic of the sharded permanent (CPU, gloo, world_size 2 and 3): each rank takes
its App. A distribute span, produces the raw partial (here with the CPU oracle standing in for the GPU
walk), one all-gather exchanges the double-double partials and every rank combines them in rank order
with perm_c128_finalize.  Checks the result against the unsharded oracle on every rank."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1904_06229_b200 import inputs, shard
        A = inputs.complex_gaussian((n, n), 77)
        k0, k1 = shard.rank_span(1 << (n - 1), world, rank)
        qv = oracle.subpermanent(A, k0, k1 - k0)
        part = torch.tensor([qv.re_hi, qv.re_lo, qv.im_hi, qv.im_lo], dtype=torch.float64)
        gathered = [torch.zeros(4, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, part)
        val = shard.combine(torch.stack(gathered).numpy(), n)
        q.put((rank, val, k0, k1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_combine_matches_oracle(world):
    n = 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    from paper_1904_06229_b200 import inputs
    from tests import pins
    A = inputs.complex_gaussian((n, n), 77)
    ref = oracle.ryser(A).value
    vals = {r: v for r, v, _, _ in res}
    assert len(set(vals.values())) == 1                       # bit-identical on every rank
    assert pins.scaled_error(vals[0], ref, A) <= 1e-12
    spans = sorted((k0, k1) for _, _, k0, k1 in res)
    assert spans[0][0] == 0 and spans[-1][1] == 1 << (n - 1)
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_rank_span_matches_paper_distribute():
    import oracle
    from paper_1904_06229_b200 import shard
    for total, world in ((10, 3), (1 << 43, 8), (1 << 31, 7), (5, 8)):
        for r in range(world):
            k, l = oracle.distribute(total, world, r)
            assert shard.rank_span(total, world, r) == (k, k + l)
