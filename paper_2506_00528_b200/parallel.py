"""G-GPU partition of the search (one process per GPU, torch.distributed).

The database is sharded into contiguous row ranges; each rank searches its
shard with ``id_base`` = the shard's first global row, then the per-rank [Q][k]
lists are exchanged with one NCCL ``all_gather_into_tensor`` (over NVLink /
NVSwitch) and merged by ``uq_merge_topk``.  Merging per-shard top-k lists under
the total order (Delta desc, id asc) is exact: the global top-k is a subset of
the union of the shard top-k's, so every rank ends with the unsharded result.

This module only orchestrates (sharding arithmetic + the collective); the
search and the merge are the C-ABI kernels.  ``search_fn`` / ``merge_fn`` exist
so the host logic can be exercised in multi-process CPU tests (gloo).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous shard [lo, hi) of n rows for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def allgather_lists(scores: torch.Tensor, ids: torch.Tensor, group=None):
    """[Q][k] per rank -> [G][Q][k] on every rank (one collective per tensor)."""
    world = dist.get_world_size(group)
    q, k = scores.shape
    # output as the rank-major concatenation [G*Q][k] (accepted by NCCL and gloo)
    sg = torch.empty((world * q, k), dtype=scores.dtype, device=scores.device)
    ig = torch.empty((world * q, k), dtype=ids.dtype, device=ids.device)
    dist.all_gather_into_tensor(sg, scores.contiguous(), group=group)
    dist.all_gather_into_tensor(ig, ids.contiguous(), group=group)
    return sg.view(world, q, k), ig.view(world, q, k)


def sharded_search(qcodes: torch.Tensor, db_shard: torch.Tensor, d: int, k: int, id_base: int,
                   group=None, search_fn: Optional[Callable] = None,
                   merge_fn: Optional[Callable] = None, **search_kw):
    """Local search on this rank's shard + allgather + merge.  Returns the global
    (scores [Q][k], ids [Q][k]) on every rank."""
    if search_fn is None or merge_fn is None:
        import paper_2506_00528_b200 as uq
        search_fn = search_fn or uq.search
        merge_fn = merge_fn or uq.merge_topk
    s, i = search_fn(qcodes, db_shard, d, k, id_base=id_base, **search_kw)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return s, i
    sg, ig = allgather_lists(s, i, group)
    return merge_fn(sg, ig, k)
