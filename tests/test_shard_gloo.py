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


def _span_nodes(leaves, a, b):
    """Maximal canonical tree nodes of the chunk span [a, b) as a node buffer: each node's value is the
    canonical merge of its leaves (the library's host merge, which is what the device tree computes)."""
    import paper_1904_06229_b200 as pb
    entries = []
    while a < b:
        lv = 0
        while a % (1 << (lv + 1)) == 0 and a + (1 << (lv + 1)) <= b:
            lv += 1
        k = a >> lv
        sub = [(0, c, leaves[c]) for c in range(k << lv, (k + 1) << lv)]
        raw, _ = pb.perm_c128_tree_combine(pb.make_tree_nodes(sub))
        entries.append((lv, k, raw.astuple()))
        a += 1 << lv
    buf = np.zeros((pb.TREE_MAX_NODES, 6), dtype=np.int64)
    raw = pb.make_tree_nodes(entries + [(pb.TREE_UNUSED, 0, (0, 0, 0, 0))] * (pb.TREE_MAX_NODES - len(entries)))
    buf.view(np.uint8).reshape(-1)[:] = raw
    return buf


def _chunk_leaves(n, b):
    """Oracle dd partials of every chunk of 2^b ranks (App. A subpermanent per chunk) -- stand-ins for
    perm_c128_chunks' output in this CPU test."""
    import oracle
    from paper_1904_06229_b200 import inputs
    A = inputs.complex_gaussian((n, n), 91)
    out = []
    for c in range(1 << (n - 1 - b)):
        q = oracle.subpermanent(A, c << b, 1 << b)
        out.append((float(q.re_hi), float(q.re_lo), float(q.im_hi), float(q.im_lo)))
    return A, out


def _tree_worker(rank, world, port, n, b, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1904_06229_b200 import shard
        _, leaves = _chunk_leaves(n, b)
        c0, c1 = shard.chunk_span(n, world, rank, b)
        collected = []
        for s0, s1 in shard.step_slices(c0, c1, steps, 3):        # a "wave" of 3 chunks
            nodes = torch.from_numpy(_span_nodes(leaves, s0, s1))
            gathered = torch.empty((world * nodes.shape[0], 6), dtype=torch.int64)
            dist.all_gather_into_tensor(gathered, nodes)
            collected.append(gathered.numpy().copy())
        v, d = shard.combine_nodes(np.concatenate(collected), n, return_dd=True)
        q.put((rank, d.astuple(), c0, c1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,steps", [(2, 1), (3, 2), (4, 3)])
def test_chunk_tree_sharding_is_bit_identical(world, steps):
    """The chunk path's host logic over gloo: whole-chunk spans per rank (distribute over chunks), each
    rank's span sliced into steps, one all-gather of the tree-node arrays per step, canonical merge --
    every rank gets the same double-double, bitwise equal to merging all chunk partials in one process,
    and equal to the oracle's permanent within the north-star bound."""
    import paper_1904_06229_b200 as pb
    from tests import pins
    import oracle
    n, b = 10, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tree_worker, args=(r, world, port, n, b, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, leaves = _chunk_leaves(n, b)
    raw, root = pb.perm_c128_tree_combine(pb.make_tree_nodes([(0, c, v) for c, v in enumerate(leaves)]))
    assert root == n - 1 - b
    _, ref_dd = pb.perm_c128_finalize([raw], n, return_dd=True)
    assert all(d == ref_dd.astuple() for _, d, _, _ in res), res
    spans = sorted((c0, c1) for _, _, c0, c1 in res)
    assert spans[0][0] == 0 and spans[-1][1] == 1 << (n - 1 - b)
    assert pins.scaled_error(ref_dd.value, oracle.ryser(A).value, A) <= 1e-12
