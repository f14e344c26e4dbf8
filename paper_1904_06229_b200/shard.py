"""Sharding one permanent over processes / GPUs (App. A distribute + permanent).

The 2^{n-1} Gray ranks form 2^{n-1-b} aligned chunks of 2^b ranks (b = chunk_log2(n), a function of n
alone).  The CHUNKS are split into contiguous spans with the paper's ``distribute``: rank
``i`` of ``G`` gets chunks ``[k, k+l)``, ``k = i q + min(i, r)``, ``l = q + [i < r]`` -- whole chunks, so
every GPU walks only aligned chunks.  Each process walks its span with
:func:`perm_c128_chunks` (one dd partial per chunk) and reduces it with :func:`perm_c128_tree` to the
span's maximal nodes of the canonical chunk tree; ONE collective -- an all-gather of every rank's node
array (128 x 48 bytes) over NCCL (NVLink/NVSwitch) -- and every rank merges the nodes with
:func:`perm_c128_tree_combine` and applies 2(-1)^n (:func:`perm_c128_finalize`; "partial sums ...
stored in an array before the final summation").  Because the tree is fixed by the chunk
indices, per(A) is bit-identical for every G, every slicing of the span into steps, and to
:func:`perm_c128` (S:172 determinism, strengthened).

The range API path (:func:`perm_c128_range` + ordered :func:`combine`) is kept for arbitrary rank spans.
Only host logic lives here; all arithmetic of the walk runs in libperm.so.
"""
from __future__ import annotations

import numpy as np

from . import (DD, TREE_MAX_NODES, chunk_log2, perm_c128_chunks, perm_c128_finalize, perm_c128_range,
               perm_c128_tree, perm_c128_tree_combine, perm_int01_finalize, perm_int01_range)


def rank_span(total: int, world: int, rank: int) -> tuple[int, int]:
    """App. A distribute(total, world, rank) -> [k0, k1)."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad distribute arguments")
    q, r = divmod(total, world)
    k0 = rank * q + min(rank, r)
    return k0, k0 + q + (1 if rank < r else 0)


def chunk_span(n: int, world: int, rank: int, b: int | None = None) -> tuple[int, int]:
    """Whole aligned chunks of 2^b ranks for rank ``rank`` of ``world``: distribute(2^{n-1-b}, world, rank)."""
    b = chunk_log2(n) if b is None else b
    return rank_span(1 << (n - 1 - b), world, rank)


def step_slices(c0: int, c1: int, steps: int, wave: int) -> list[tuple[int, int]]:
    """Cut the chunk span [c0, c1) into ``steps`` contiguous slices made of whole rounds of ``wave`` chunks
    (a wave = the chunk walkers one launch keeps resident): round counts per step by distribute, so only
    the very last round of the span can be partial.  Slices may be empty when steps > rounds."""
    if steps < 1 or wave < 1 or c1 < c0:
        raise ValueError("bad slicing arguments")
    rounds = -(-(c1 - c0) // wave)
    out, cur = [], c0
    for s in range(steps):
        r0, r1 = rank_span(rounds, steps, s)
        nxt = min(c1, c0 + r1 * wave)
        out.append((cur, nxt))
        cur = nxt
    return out


def combine_nodes(nodes, n: int, expect_root: bool = True, return_dd: bool = False):
    """per(A) from the tree nodes of disjoint chunk spans covering all 2^{n-1-b} chunks (any order; e.g. the
    all-gathered node arrays of every rank and step): canonical merge + 2(-1)^n."""
    raw, level = perm_c128_tree_combine(nodes)
    if expect_root and level < 0:
        raise ValueError("tree nodes do not cover the chunk range exactly")
    return perm_c128_finalize([raw], n, return_dd=return_dd)


def combine(gathered, n: int, return_dd: bool = False):
    """Ordered dd combine of a (G, 4) array of partials {hi_re, lo_re, hi_im, lo_im} -> per(A)."""
    arr = np.asarray(gathered, dtype=np.float64).reshape(-1, 4)
    return perm_c128_finalize([tuple(row) for row in arr], n, return_dd=return_dd)


def sharded_permanent(A, group=None, *, stream=None, return_dd: bool = False):
    """per(A) with the aligned chunks split over the ranks of a torch.distributed process group: chunk walk
    + canonical tree on each rank, one all-gather of the node arrays, canonical merge.  Bit-identical to
    perm_c128(A) for any group size.  A: host (numpy / pinned torch) or CUDA n x n complex128."""
    import torch
    import torch.distributed as dist

    n = A.shape[0]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    c0, c1 = chunk_span(n, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    parts = perm_c128_chunks(A, c0, c1, stream=stream)
    nodes = perm_c128_tree(parts, c0, c1, stream=stream)
    if world > 1:
        gathered = torch.empty((world * TREE_MAX_NODES, 6), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gathered, nodes, group=group)
    else:
        gathered = nodes
    return combine_nodes(gathered.cpu().numpy(), n, return_dd=return_dd)


def sharded_permanent_range(A, group=None, *, workspace=None, stream=None, partial_out=None, gathered_out=None,
                            events=None):
    """per(A) with the Gray RANK range split by distribute over the ranks of a process group (range API:
    perm_c128_range per rank + all-gather of the dd partials + ordered combine; equal to perm_c128 up to
    rounding, bit-identical run to run at fixed G).

    A: host (numpy / pinned torch) n x n complex128.  Every rank returns the same value.
    partial_out / gathered_out: optional preallocated CUDA float64 tensors of 4 and 4G elements."""
    import torch
    import torch.distributed as dist

    n = A.shape[0]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    k0, k1 = rank_span(1 << (n - 1), world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    part = partial_out if partial_out is not None else torch.empty(4, dtype=torch.float64, device=dev)
    perm_c128_range(A, k0, k1, workspace=workspace, stream=stream, out=part, events=events)
    if world > 1:
        gathered = gathered_out if gathered_out is not None else torch.empty(4 * world, dtype=torch.float64,
                                                                             device=dev)
        dist.all_gather_into_tensor(gathered, part, group=group)
    else:
        gathered = part
    return combine(gathered.cpu().numpy(), n)


def _matrix_digest(A) -> str:
    import hashlib
    a = A.detach().cpu().numpy() if hasattr(A, "detach") else np.asarray(A)
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.complex128).tobytes()).hexdigest()


def checkpointed_permanent(A, path: str, steps: int, *, world: int = 1, rank: int = 0, max_steps: int | None = None,
                           wave: int | None = None, stream=None, return_dd: bool = False):
    """per(A) of one long permanent walked as ``steps`` slices of this rank's chunk span, the tree nodes of every
    finished slice kept in the checkpoint file ``path`` ("per-chunk partials are naturally
    checkpointable"; P:202-206 stores the partial sums before the final summation).  A later call with the
    same matrix, steps, world and rank resumes after the last finished slice; a file written for another
    matrix or slicing is refused.  ``max_steps`` stops after that many slices of this call (returns None):
    the hook the tests use to interrupt a run; ``wave``: chunks per slicing round (default: the resident chunk
    walkers of one launch, so every slice is whole rounds; every slice must be non-empty).  With world = 1 the value returned after the last slice has
    the bits of perm_c128(A) (the chunk tree does not depend on the slicing); with world > 1 it returns this
    rank's node array (done, 128, 6) for the caller to gather and pass to combine_nodes.  Host logic only."""
    import os
    import torch

    n = A.shape[0]
    b = chunk_log2(n)
    c0, c1 = chunk_span(n, world, rank, b)
    if wave is None:
        from . import chunk_walkers
        wave = chunk_walkers(n, b)
    slices = step_slices(c0, c1, steps, wave)
    if any(s1 <= s0 for s0, s1 in slices):
        raise ValueError("more steps than rounds of chunks: an empty slice")
    key = np.array([n, b, c0, c1, steps, world, rank, wave], dtype=np.int64)
    digest = _matrix_digest(A)
    done = 0
    saved = np.zeros((0, TREE_MAX_NODES, 6), dtype=np.int64)
    if os.path.exists(path):
        with np.load(path) as f:
            if str(f["digest"]) != digest or not np.array_equal(f["key"], key):
                raise ValueError("checkpoint belongs to another matrix or slicing")
            saved = np.array(f["nodes"], dtype=np.int64).reshape(-1, TREE_MAX_NODES, 6)
            done = saved.shape[0]
            if done > steps:
                raise ValueError("checkpoint holds more slices than the run has")
    ran = 0
    for s in range(done, steps):
        if max_steps is not None and ran >= max_steps:
            return None
        s0, s1 = slices[s]
        parts = perm_c128_chunks(A, s0, s1, stream=stream)
        nodes = perm_c128_tree(parts, s0, s1, stream=stream)
        if stream is not None:
            stream.synchronize()
        saved = np.concatenate([saved, nodes.cpu().numpy().reshape(1, TREE_MAX_NODES, 6)])
        tmp = path + ".tmp.npz"
        np.savez(tmp, digest=np.array(digest), key=key, nodes=saved)
        os.replace(tmp, path)                       # a slice is either wholly in the file or not at all
        ran += 1
    if world > 1:
        return saved
    return combine_nodes(saved.reshape(-1, 6), n, return_dd=return_dd)


def int01_rank_space(n: int) -> int:
    """Ranks of perm_int01's walk: 2^{n-1} (half-range Glynn, n <= 28) or 2^n (Eq. (3), 29 <= n <= 33)."""
    return 1 << (n if n > 28 else n - 1)


def pack_i128(v: int) -> np.ndarray:
    """A raw partial (int mod 2^128) as two int64 {lo, hi} -- what the collective exchanges (exact)."""
    v = int(v) & ((1 << 128) - 1)
    lo, hi = v & ((1 << 64) - 1), v >> 64
    return np.array([lo - (1 << 64) if lo >= (1 << 63) else lo, hi - (1 << 64) if hi >= (1 << 63) else hi],
                    dtype=np.int64)


def combine_int01(gathered, n: int) -> int:
    """Exact per(A) from a (G, 2) int64 array of raw partials {lo, hi}: summed mod 2^128 in any order."""
    arr = np.asarray(gathered, dtype=np.int64).reshape(-1, 2)
    parts = [((int(hi) & ((1 << 64) - 1)) << 64) | (int(lo) & ((1 << 64) - 1)) for lo, hi in arr]
    return perm_int01_finalize(parts, n)


def sharded_int01(A, group=None, *, stream=None) -> int:
    """Exact per(A) of ONE 0-1 matrix (an (n, n) uint8 CUDA tensor) with its rank space split over the
    ranks of a process group: each rank walks its distribute span (perm_int01_range), one all-gather of
    the 16-byte raw partials, exact combine mod 2^128 on every rank ("sharding a single
    int01 permanent")."""
    import torch
    import torch.distributed as dist

    n = A.shape[-1]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    k0, k1 = rank_span(int01_rank_space(n), world, rank)
    part = torch.from_numpy(pack_i128(perm_int01_range(A, k0, k1, stream=stream))).to(A.device)
    if world > 1:
        gathered = torch.empty(2 * world, dtype=torch.int64, device=A.device)
        dist.all_gather_into_tensor(gathered, part, group=group)
    else:
        gathered = part
    return combine_int01(gathered.cpu().numpy(), n)


__all__ = ["rank_span", "chunk_span", "step_slices", "combine_nodes", "combine", "sharded_permanent",
           "sharded_permanent_range", "checkpointed_permanent", "int01_rank_space", "pack_i128", "combine_int01",
           "sharded_int01", "DD"]
