"""GPU parity of the chunk walk + canonical chunk tree -- the path bench.py times (perm_c128_chunks,
perm_c128_tree, perm_c128_tree_combine) -- against the CPU oracle, plus the bit-identity the tree
guarantees (any split of the chunk range over GPUs / steps gives perm_c128's exact double-double).

Tolerances: a chunk span's raw partial vs the oracle's App. A subpermanent over the same ranks,
|gpu - oracle| <= 1e-12 max(|oracle|, range_scale) (the range tests' bar); whole permanents: the north-star
scaled error <= 1e-9; self-consistency between two GPU walks of the same permanent: <= 1e-11 scaled."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import inputs, shard
from tests import pins

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pb.lib()


def _golden(golden_dir):
    p = os.path.join(golden_dir, "oracle_values.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def _q(v):
    return complex(v[0] + v[1], v[2] + v[3])


def _span_raw(A, c0, c1, b=None, stats=False):
    """Raw dd partial of the chunk span [c0, c1) by the GPU path: chunk walk -> tree -> combine."""
    parts, st = pb.perm_c128_chunks(A, c0, c1, chunk_log2_=b, stats=True)
    nodes = pb.perm_c128_tree(parts, c0, c1)
    raw, _ = pb.perm_c128_tree_combine(nodes.cpu().numpy())
    return (raw, st) if stats else raw


def _sharded(A, world, steps=1, b=None):
    """per(A) as `world` simulated GPUs, each slicing its span into `steps` launches: every launch's nodes
    are collected (what the all-gathers deliver) and merged on the host."""
    n = A.shape[0]
    b = pb.chunk_log2(n) if b is None else b
    allnodes = []
    for r in range(world):
        c0, c1 = shard.chunk_span(n, world, r, b)
        for s0, s1 in shard.step_slices(c0, c1, steps, 1 + (c1 - c0) // max(1, 2 * steps)):
            parts = pb.perm_c128_chunks(A, s0, s1, chunk_log2_=b)
            allnodes.append(pb.perm_c128_tree(parts, s0, s1).cpu().numpy())
    return shard.combine_nodes(np.concatenate(allnodes), n, return_dd=True)


# ------------------------------------------------------------------ per-chunk partials vs the oracle

@pytest.mark.parametrize("n,b", [(3, 0), (3, 2), (8, 3), (12, 3), (20, 3), (20, 7), (33, 3), (33, 10), (44, 2),
                                 (44, 12), (50, 2), (64, 3)])
def test_chunk_partials_vs_oracle(n, b):
    A = inputs.complex_gaussian((n, n), 5000 + n)
    C = 1 << (n - 1 - b)
    rng = np.random.default_rng(n * 64 + b)
    c0 = int(rng.integers(0, max(1, C - 40)))
    c1 = min(C, c0 + 37)
    parts, st = pb.perm_c128_chunks(A, c0, c1, chunk_log2_=b, stats=True)
    assert st["chunk_log2"] == b and st["items"] == c1 - c0 and st["terms"] == (c1 - c0) << b
    P = parts.cpu().numpy()
    for i in list(range(min(6, c1 - c0))) + [c1 - c0 - 1]:
        c = c0 + i
        ref = oracle.subpermanent(A, c << b, 1 << b).value
        got = complex(P[i, 0] + P[i, 1], P[i, 2] + P[i, 3])
        assert abs(got - ref) <= 1e-12 * max(abs(ref), pins.range_scale(A, 1 << b)), (n, b, c, got, ref)


def test_chunk_arguments():
    import torch
    A = inputs.complex_gaussian((10, 10), 1)
    P = torch.empty((4, 4), dtype=torch.float64, device="cuda")
    for bad_b in (1, 10, 31, -1):                           # 0 < b < U(10) = 3, b > n - 1
        with pytest.raises(pb.PermError):
            pb.perm_c128_chunks(A, 0, 1, partials=P, chunk_log2_=bad_b)
    with pytest.raises(pb.PermError):                       # beyond 2^{n-1-b} chunks
        pb.perm_c128_chunks(A, 60, 65, partials=P, chunk_log2_=3)
    with pytest.raises(pb.PermError):                       # host partials
        pb.perm_c128_chunks(A, 0, 1, partials=torch.empty((1, 4), dtype=torch.float64), chunk_log2_=3)
    Z = A.copy()
    Z[2, 3] = np.inf
    with pytest.raises(pb.PermError) as e:
        pb.perm_c128_chunks(torch.from_numpy(Z).cuda(), 0, 4, partials=P, chunk_log2_=3)
    assert e.value.name == "PERM_E_NONFINITE"
    pb.perm_c128_chunks(A, 5, 5, partials=P, chunk_log2_=3)         # empty span: nothing to do
    nodes = pb.perm_c128_tree(P, 5, 5)
    assert pb.tree_nodes(nodes.cpu().numpy()) == []


# ------------------------------------------------------------------ the tree on the device

@pytest.mark.parametrize("c0,c1", [(0, 1), (0, 256), (0, 1 << 16), (3, 700), (255, 257), (1000, 70000),
                                   ((1 << 20) - 5, (1 << 20) + 3), (12345, 12345 + (1 << 17) + 77)])
def test_device_tree_matches_host_merge(c0, c1):
    """Device tree nodes of a span == the host merge of its leaves (the same canonical tree), bitwise; the
    node set is the span's maximal aligned nodes."""
    import torch
    rng = np.random.default_rng(c0 + c1)
    cnt = c1 - c0
    leaves = rng.standard_normal((cnt, 4)) * 10.0 ** rng.integers(-6, 6, (cnt, 1))
    leaves[:, 1] *= 1e-17
    leaves[:, 3] *= 1e-17
    # normalise each leaf to a valid dd (hi = fl(hi + lo))
    leaves[:, 0], leaves[:, 1] = leaves[:, 0] + leaves[:, 1], 0.0
    leaves[:, 2], leaves[:, 3] = leaves[:, 2] + leaves[:, 3], 0.0
    nodes = pb.perm_c128_tree(torch.from_numpy(leaves).cuda(), c0, c1)
    dev = pb.tree_nodes(nodes.cpu().numpy())
    got_pos = [(lv, k) for lv, k, _ in dev]
    # maximal nodes of [c0, c1), left to right
    exp, a = [], c0
    while a < c1:
        lv = 0
        while a % (1 << (lv + 1)) == 0 and a + (1 << (lv + 1)) <= c1:
            lv += 1
        exp.append((lv, a >> lv))
        a += 1 << lv
    assert got_pos == exp
    if cnt <= 70000:
        host, _ = pb.perm_c128_tree_combine(pb.make_tree_nodes([(0, c0 + i, tuple(leaves[i])) for i in range(cnt)]))
        dev_raw, _ = pb.perm_c128_tree_combine(nodes.cpu().numpy())
        assert dev_raw.astuple() == host.astuple()


# ------------------------------------------------------------------ bit-identity across splits

@pytest.mark.parametrize("n", [5, 17, 24, 28, 33, 36])
def test_perm_c128_bit_identical_to_any_split(n):
    A = inputs.complex_gaussian((n, n), 6000 + n)
    v, d = pb.perm_c128(A, return_dd=True)
    for world, steps in ((1, 1), (2, 1), (3, 2), (8, 3), (5, 7)):
        v2, d2 = _sharded(A, world, steps)
        assert d2.astuple() == d.astuple() and v2 == v, (n, world, steps)
    ref = oracle.permanent_hr(A).value if n <= 24 else None
    if ref is not None:
        assert pins.scaled_error(v, ref, A) <= 1e-9
    # the range API (other pieces, other tree) agrees to rounding
    parts = [pb.perm_c128_range(A, *shard.rank_span(1 << (n - 1), 3, r)) for r in range(3)]
    assert pins.scaled_error(pb.perm_c128_finalize(parts, n), v, A) <= 1e-12


def test_sharded_permanent_single_process():
    A = inputs.complex_gaussian((30, 30), 30)
    assert shard.sharded_permanent(A, return_dd=True)[1].astuple() == pb.perm_c128(A, return_dd=True)[1].astuple()


def test_device_matrix_nonfinite_paths():
    import torch
    A = inputs.complex_gaussian((20, 20), 2)
    A[4, 5] = np.nan
    At = torch.from_numpy(A).cuda()
    with pytest.raises(pb.PermError) as e:                  # host output: the staging flag -> status
        pb.perm_c128(At)
    assert e.value.name == "PERM_E_NONFINITE"
    out = torch.zeros(1, dtype=torch.complex128, device="cuda")
    pb.perm_c128(At, out=out)                               # device output: no sync, NaN result
    torch.cuda.synchronize()
    assert np.isnan(complex(out.item()).real)
    with pytest.raises(pb.PermError):
        pb.perm_c128_range(At, 0, 1000)


# ------------------------------------------------------------------ BASELINE configs on the bench's path

def test_cfg5_chunk_spans_on_the_shipped_kernel(golden_dir):
    """Sub-spans of the actual config-5 matrix, 16 chunks (2^22 ranks) each at the bench's chunk length
    b = 18, walked by the constant-bank kernel walk_kernel_cm<44> exactly as in bench.py: first/last chunks,
    the chunk where 8 GPU shards meet (rank 2^40), an unaligned 3 * 2^40 crossing and a step boundary."""
    g = _golden(golden_dir).get("chunks44")
    if not g:
        pytest.skip("oracle_values.json has no chunks44 section")
    A = inputs.cfg5()
    b = g["chunk_log2"]
    assert pb.chunk_log2(44) == b
    for sp in g["spans"]:
        raw, st = _span_raw(A, sp["c0"], sp["c1"], b, stats=True)
        assert st["chunk_log2"] == b and st["const_path"] == 1, st
        ref = _q(sp["value"])
        got = raw.value
        scale = max(abs(ref), pins.range_scale(A, (sp["c1"] - sp["c0"]) << b))
        assert abs(got - ref) <= 1e-12 * scale, (sp["c0"], got, ref)


def test_cfg4_chunk_spans(golden_dir):
    g = _golden(golden_dir).get("chunks32")
    if not g:
        pytest.skip("oracle_values.json has no chunks32 section")
    A = inputs.cfg4()
    b = g["chunk_log2"]
    assert pb.chunk_log2(32) == b
    for sp in g["spans"]:
        raw, st = _span_raw(A, sp["c0"], sp["c1"], b, stats=True)
        assert st["chunk_log2"] == b and st["const_path"] == 1
        ref = _q(sp["value"])
        scale = max(abs(ref), pins.range_scale(A, (sp["c1"] - sp["c0"]) << b))
        assert abs(raw.value - ref) <= 1e-12 * scale, (sp["c0"], raw.value, ref)


def test_cfg4_full_sharded_vs_golden(golden_dir):
    g = _golden(golden_dir).get("cfg4")
    if not g:
        pytest.skip("oracle_values.json has no cfg4 section")
    A = inputs.cfg4()
    v8, d8 = _sharded(A, 8, 3)
    assert d8.astuple() == pb.perm_c128(A, return_dd=True)[1].astuple()
    assert pins.scaled_error(v8, _q(g["value"]), A) <= 1e-9


@pytest.mark.slow
def test_cfg5_blockdiag_full_walk_8_shards(golden_dir):
    """P7 at n = 44 on the bench's path: per(P (B1 (+) B2) Q) = per(B1) per(B2), the full 2^43-term walk as
    8 simulated GPU shards (chunk walk + tree per shard) merged by the canonical tree."""
    g = _golden(golden_dir).get("blockdiag44")
    if not g:
        pytest.skip("oracle_values.json has no blockdiag44 section")
    s1, s2, sp = g["seeds"]
    B1 = inputs.complex_gaussian((22, 22), s1)
    B2 = inputs.complex_gaussian((22, 22), s2)
    M, _, _ = inputs.block_diag_scrambled(B1, B2, sp)
    ref = _q(g["per_B1"]) * _q(g["per_B2"])
    got, _ = _sharded(M, 8, 1)
    assert pins.scaled_error(got, ref, M) <= 1e-9, (got, ref)


@pytest.mark.slow
def test_cfg5_self_consistency_transpose_and_permutation():
    """P4 at n = 44 on the config-5 matrix itself (its full value is out of the oracle's reach): per(A) as
    8 simulated shards against per(P A^T Q) in one launch -- two different matrices, walks and entry points
    that must agree to rounding (two full walks, about 250 s; the 3-shard / 2-step slicing of a third matrix
    is covered at n = 32 by test_gpu_bench_dist.py)."""
    A = inputs.cfg5()
    rng = np.random.default_rng(4444)
    PAtQ = np.ascontiguousarray(A.T[rng.permutation(44)][:, rng.permutation(44)])
    v_a, _ = _sharded(A, 8, 1)
    v_p = pb.perm_c128(PAtQ)
    assert pins.scaled_error(v_a, v_p, A) <= 1e-11, (v_a, v_p)


def test_unit_column_walk_device_and_host_matrix_bit_identical():
    """The unit-column walk normalises A on the host for every call: a device-resident matrix
    without a workspace (scratch allocated inside), with one, and the host matrix give the same bits; a matrix
    with a zero in column 0 takes the plain walk and still matches the oracle's App. A span."""
    import torch
    for n in (33, 44):
        A = inputs.complex_gaussian((n, n), 7700 + n)
        b = pb.chunk_log2(n)
        c0, c1 = 5, 5 + 300
        ref = pb.perm_c128_chunks(A, c0, c1).cpu().numpy()
        Ad = torch.from_numpy(A).cuda()
        assert np.array_equal(pb.perm_c128_chunks(Ad, c0, c1).cpu().numpy(), ref)
        ws = torch.empty(n * n * 16, dtype=torch.uint8, device="cuda")
        assert np.array_equal(pb.perm_c128_chunks(Ad, c0, c1, workspace=ws).cpu().numpy(), ref)
    n = 33
    A = inputs.complex_gaussian((n, n), 7733)
    A[4, 0] = 0.0
    raw = _span_raw(A, 0, 4, 10)
    ref = oracle.subpermanent(A, 0, 4 << 10)
    scale = max(abs(ref.value), pins.range_scale(A, 4 << 10))
    assert abs(raw.value - ref.value) <= 1e-12 * scale


def test_checkpointed_permanent_resumes_to_the_same_bits(tmp_path):
    """shard.checkpointed_permanent: a run interrupted after 2 of 5 slices and then after 2 more resumes from
    the checkpoint file to the bits of perm_c128(A) (the chunk tree does not depend on the slicing); the
    finished file answers without walking; two simulated GPUs checkpointing separately merge to the same bits."""
    A = inputs.complex_gaussian((30, 30), 3030)
    ref = pb.perm_c128(A, return_dd=True)
    path = str(tmp_path / "perm30.npz")
    assert shard.checkpointed_permanent(A, path, 5, max_steps=2) is None
    assert shard.checkpointed_permanent(A, path, 5, max_steps=2) is None
    with np.load(path) as f:
        assert f["nodes"].shape[0] == 4
    got = shard.checkpointed_permanent(A, path, 5, return_dd=True)
    assert got == ref, (got, ref)
    assert shard.checkpointed_permanent(A, path, 5, max_steps=0, return_dd=True) == ref   # nothing left to walk
    with pytest.raises(ValueError):
        shard.checkpointed_permanent(A + 1.0, path, 5)
    with pytest.raises(ValueError):
        shard.checkpointed_permanent(A, path, 4)
    nodes = [shard.checkpointed_permanent(A, str(tmp_path / f"r{r}.npz"), 3, world=2, rank=r) for r in range(2)]
    assert shard.combine_nodes(np.concatenate(nodes).reshape(-1, 6), 30, return_dd=True) == ref
