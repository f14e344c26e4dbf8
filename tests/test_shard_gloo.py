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


def _int01_raw_partial(A, k0, k1):
    """Raw Gray sum of App. A in integers over ranks [k0, k1) (g_i = 2 w_i, term sign (-1)^{r+1}),
    straight from the definition -- stands in for the GPU's perm_int01_range in this CPU test."""
    n = A.shape[0]
    a = [[int(v) for v in row] for row in A]
    tot = 0
    for r in range(k0, k1):
        x = r ^ (r >> 1)
        prod = 1
        for i in range(n):
            g = a[i][n - 1] - sum(a[i][j] for j in range(n - 1)) + 2 * sum(a[i][j] for j in range(n - 1) if (x >> j) & 1)
            prod *= g
        tot += prod if (r & 1) else -prod
    return tot & ((1 << 128) - 1)


def _int01_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_06229_b200 import inputs, shard
        A = inputs.bernoulli01((1, n, n), 31)[0]
        k0, k1 = shard.rank_span(shard.int01_rank_space(n), world, rank)
        part = torch.from_numpy(shard.pack_i128(_int01_raw_partial(A, k0, k1)))
        gathered = torch.empty(2 * world, dtype=torch.int64)
        dist.all_gather_into_tensor(gathered, part)
        q.put((rank, shard.combine_int01(gathered.numpy(), n)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_int01_combine_is_exact(world):
    # one exact 0-1 permanent split over ranks: 16-byte raw partials, one all-gather, exact combine
    n = 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_int01_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    from paper_1904_06229_b200 import inputs
    A = inputs.bernoulli01((1, n, n), 31)
    ref = oracle.ryser_i01_batch(A)[0]
    assert all(v == ref for _, v in res), (res, ref)


def test_int01_finalize_host_logic():
    # the ABI's finalize (host only, no GPU): divisibility check, sign, exact wrap-around of partials
    from paper_1904_06229_b200 import shard, perm_int01_finalize, PermError
    import oracle
    from paper_1904_06229_b200 import inputs
    n = 9
    A = inputs.bernoulli01((1, n, n), 5)[0]
    N = shard.int01_rank_space(n)
    cuts = [0, 1, 100, 101, N]
    parts = [_int01_raw_partial(A, cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
    assert perm_int01_finalize(parts, n) == oracle.ryser_i01_batch(A[None])[0]
    assert perm_int01_finalize(parts[::-1], n) == oracle.ryser_i01_batch(A[None])[0]   # order-free
    with pytest.raises(PermError):
        perm_int01_finalize(parts[:2], n)          # an incomplete cover is not divisible by 2^{n-1}
