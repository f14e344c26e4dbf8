"""Host logic of the canonical chunk tree and of the chunk-level sharding/slicing (no GPU).

perm_c128_tree_combine (libperm.so, host-only) merges the maximal tree nodes of disjoint chunk spans; the
spans' maximal nodes are written here in plain Python from the definition (node (L, k) covers chunks
[k 2^L, (k+1) 2^L); a span's maximal nodes are the complete nodes whose parent is not complete).  With
integer leaf values every dd add is exact, so merged values must equal exact integer sums, and the
merge must reach the root exactly when the spans tile [0, 2^m).
"""
from __future__ import annotations

import random

import numpy as np
import pytest

import paper_1904_06229_b200 as pb
from paper_1904_06229_b200 import shard


def maximal_nodes(a: int, b: int) -> list[tuple[int, int]]:
    """Maximal aligned complete nodes (level, index) of the chunk span [a, b), left to right."""
    out = []
    while a < b:
        lv = 0
        while a % (1 << (lv + 1)) == 0 and a + (1 << (lv + 1)) <= b:
            lv += 1
        out.append((lv, a >> lv))
        a += 1 << lv
    return out


def span_entries(a, b, leaves):
    return [(lv, k, (float(sum(leaves[k << lv:(k + 1) << lv])), 0.0, 0.0, 0.0)) for lv, k in maximal_nodes(a, b)]


@pytest.mark.parametrize("m,parts", [(0, 1), (3, 2), (10, 3), (12, 7), (16, 1), (16, 8), (20, 5)])
def test_combine_of_random_tilings_reaches_the_root(m, parts):
    rng = random.Random(m * 100 + parts)
    leaves = [rng.randrange(-1000, 1000) for _ in range(1 << m)]
    cuts = sorted(rng.sample(range(1, 1 << m), min(parts - 1, (1 << m) - 1))) if m > 0 else []
    bounds = [0] + cuts + [1 << m]
    entries = []
    for a, b in zip(bounds, bounds[1:]):
        entries += span_entries(a, b, leaves)
    rng.shuffle(entries)                                     # order of ranks / steps is irrelevant
    raw, root = pb.perm_c128_tree_combine(pb.make_tree_nodes(entries))
    assert root == m
    assert raw.hi_re == float(sum(leaves)) and raw.lo_re == 0.0


def test_combine_partial_cover_and_unused_slots():
    leaves = list(range(1, 33))
    entries = span_entries(3, 19, leaves)
    buf = np.concatenate([pb.make_tree_nodes(entries),
                          pb.make_tree_nodes([(pb.TREE_UNUSED, 0, (9e99, 0, 0, 0))])])
    raw, root = pb.perm_c128_tree_combine(buf)
    assert root == -1 and raw.hi_re == float(sum(leaves[3:19]))
    # a single span starting at 0 of power-of-two length is a root of its own
    raw, root = pb.perm_c128_tree_combine(pb.make_tree_nodes(span_entries(0, 16, leaves)))
    assert root == 4 and raw.hi_re == float(sum(leaves[:16]))


def test_combine_rejects_overlap():
    e = [(2, 0, (1.0, 0, 0, 0)), (0, 3, (1.0, 0, 0, 0))]      # [0,4) and [3,4) overlap
    with pytest.raises(pb.PermError):
        pb.perm_c128_tree_combine(pb.make_tree_nodes(e))
    with pytest.raises(pb.PermError):
        pb.perm_c128_tree_combine(pb.make_tree_nodes([(64, 0, (1.0, 0, 0, 0))]))


def test_combine_is_the_canonical_dd_tree():
    # non-exact values: merging siblings in any grouping gives the canonical left+right tree, so the three
    # spans [0,3), [3,6), [6,8) merge to the same dd as the single span [0,8)
    rng = np.random.default_rng(5)
    vals = (rng.standard_normal(8) * 10.0 ** rng.integers(-8, 8, 8)).tolist()

    def node(lv, k):            # canonical node value by the library itself, from its leaves
        raw, _ = pb.perm_c128_tree_combine(pb.make_tree_nodes([(0, i, (vals[i], 0, 0, 0))
                                                                for i in range(k << lv, (k + 1) << lv)]))
        return raw.astuple()

    whole, root = pb.perm_c128_tree_combine(pb.make_tree_nodes([(0, i, (vals[i], 0, 0, 0)) for i in range(8)]))
    assert root == 3
    pieces = []
    for a, b in ((0, 3), (3, 6), (6, 8)):
        pieces += [(lv, k, node(lv, k)) for lv, k in maximal_nodes(a, b)]
    merged, root2 = pb.perm_c128_tree_combine(pb.make_tree_nodes(pieces[::-1]))
    assert root2 == 3 and merged.astuple() == whole.astuple()


def test_tree_nodes_roundtrip():
    e = [(3, 5, (1.5, 2.0 ** -60, -2.0, 0.0)), (0, 7, (0.25, 0.0, 0.0, 1e-30))]
    got = pb.tree_nodes(pb.make_tree_nodes(e))
    assert [(lv, k, d.astuple()) for lv, k, d in got] == [(lv, k, tuple(v)) for lv, k, v in e]


def test_chunk_log2_table():
    # a function of n alone; n = 44 walks 2^25 chunks of 2^18 ranks, n = 32 2^21 of 2^10
    assert pb.chunk_log2(44) == 18 and pb.chunk_log2(32) == 10 and pb.chunk_log2(16) == 3
    for n in range(1, 65):
        b = pb.chunk_log2(n)
        assert 0 <= b <= min(n - 1, 30)
        if n >= 4:
            assert b >= 2
    with pytest.raises(pb.PermError):
        pb.chunk_log2(0)


@pytest.mark.parametrize("n,world", [(44, 1), (44, 8), (44, 3), (32, 7), (16, 5), (20, 64)])
def test_chunk_spans_are_whole_chunks_and_tile(n, world):
    b = pb.chunk_log2(n)
    spans = [shard.chunk_span(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == 1 << (n - 1 - b)
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0
    sizes = [c1 - c0 for c0, c1 in spans]
    assert max(sizes) - min(sizes) <= 1                     # distribute: balanced +-1


@pytest.mark.parametrize("c0,c1,steps,wave", [(0, 1 << 25, 20, 37888), (5, 1000, 3, 64), (0, 10, 20, 4),
                                              (0, 4096, 7, 37888), (3, 3, 4, 8)])
def test_step_slices_whole_rounds(c0, c1, steps, wave):
    sl = shard.step_slices(c0, c1, steps, wave)
    assert len(sl) == steps and sl[0][0] == c0 and sl[-1][1] == c1
    for (a0, a1), (b0, b1) in zip(sl, sl[1:]):
        assert a1 == b0 and a0 <= a1
    # every slice but the one holding the span's end is a whole number of rounds
    for a0, a1 in sl:
        if a1 != c1:
            assert (a1 - a0) % wave == 0
    rounds = -(-(c1 - c0) // wave)
    per = [-(-(a1 - a0) // wave) for a0, a1 in sl]
    assert sum(per) == rounds and max(per) - min(per) <= 1


def test_checkpoint_of_another_matrix_or_slicing_is_refused_before_any_walk(tmp_path):
    """shard.checkpointed_permanent validates the file (matrix digest, slicing key) on the host before the
    first library call that needs a device."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((30, 30)) + 1j * rng.standard_normal((30, 30))
    b = pb.chunk_log2(30)
    c0, c1 = shard.chunk_span(30, 1, 0, b)
    key = np.array([30, b, c0, c1, 4, 1, 0, 4096], dtype=np.int64)
    path = str(tmp_path / "ck.npz")
    np.savez(path, digest=np.array("0" * 64), key=key, nodes=np.zeros((1, pb.TREE_MAX_NODES, 6), dtype=np.int64))
    with pytest.raises(ValueError, match="another matrix"):
        shard.checkpointed_permanent(A, path, 4, wave=4096)
    np.savez(path, digest=np.array(shard._matrix_digest(A)), key=key,
             nodes=np.zeros((1, pb.TREE_MAX_NODES, 6), dtype=np.int64))
    with pytest.raises(ValueError, match="another matrix or slicing"):
        shard.checkpointed_permanent(A, path, 3, wave=4096)
    with pytest.raises(ValueError, match="empty slice"):
        shard.checkpointed_permanent(A, str(tmp_path / "none.npz"), 4, wave=1 << 30)
