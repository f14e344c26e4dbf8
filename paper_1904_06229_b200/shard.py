"""Sharding one permanent over processes / GPUs (App. A distribute + permanent).

The 2^{n-1} Gray ranks are split into contiguous spans with the paper's ``distribute``:
rank ``i`` of ``G`` gets ``[k, k+l)``, ``k = i q + min(i, r)``, ``l = q + [i < r]``.  Each process
computes its raw partial with :func:`perm_c128_range` on its own GPU (no data-path communication),
then ONE collective -- an all-gather of the four float64 of each rank's double-double partial over
NCCL (NVLink/NVSwitch) -- and every rank combines the G partials in rank order with
:func:`perm_c128_finalize` (2(-1)^n * ordered dd sum; "partial sums ... stored in an array
before the final summation").  The ordered combine makes the result bit-identical on
every rank and run to run.

Only the host logic lives here; all arithmetic of the walk runs in libperm.so.
"""
from __future__ import annotations

import numpy as np

from . import DD, perm_c128_finalize, perm_c128_range


def rank_span(total: int, world: int, rank: int) -> tuple[int, int]:
    """App. A distribute(total, world, rank) -> [k0, k1)."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad distribute arguments")
    q, r = divmod(total, world)
    k0 = rank * q + min(rank, r)
    return k0, k0 + q + (1 if rank < r else 0)


def combine(gathered, n: int, return_dd: bool = False):
    """Ordered dd combine of a (G, 4) array of partials {hi_re, lo_re, hi_im, lo_im} -> per(A)."""
    arr = np.asarray(gathered, dtype=np.float64).reshape(-1, 4)
    return perm_c128_finalize([tuple(row) for row in arr], n, return_dd=return_dd)


def sharded_permanent(A, group=None, *, workspace=None, stream=None, partial_out=None, gathered_out=None,
                      events=None):
    """per(A) with the Gray range split over the ranks of a torch.distributed process group.

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


__all__ = ["rank_span", "combine", "sharded_permanent", "DD"]
