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


def result_digest(results) -> str:
    """SHA-256 over the bytes of the final [Q][k] (scores, ids) of every
    result in `results` (an iterable of (scores, ids) tensor pairs, in order).
    The search result is unique (total order (Delta desc, id asc)), so the
    digest must be identical for every GPU count G, engine and launch shape:
    bench.py prints it so the scaling runs can be checked for byte equality."""
    import hashlib
    h = hashlib.sha256()
    for s, i in results:
        h.update(s.detach().to("cpu", torch.int32).contiguous().numpy().tobytes())
        h.update(i.detach().to("cpu", torch.int64).contiguous().numpy().tobytes())
    return h.hexdigest()


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


class PeerExchange:
    """Exchange + merge as ONE kernel over peer memory (NVLink / NVSwitch).

    Each rank owns a symmetric-memory pair of [Q][k] buffers
    (``torch.distributed._symmetric_memory``); every rank maps all peers'
    buffers, so after a device-side barrier ``uq_merge_topk_ptrs`` reads every
    rank's lists directly and merges them -- no staging allgather.  A second
    barrier keeps a rank from overwriting its lists while peers still read them.
    """

    def __init__(self, nq: int, k: int, device, group=None):
        import torch.distributed._symmetric_memory as symm
        if group is None:
            group = dist.group.WORLD
        self.nq, self.k = nq, k
        self.s = symm.empty((nq, k), dtype=torch.int32, device=device)
        self.i = symm.empty((nq, k), dtype=torch.int64, device=device)
        self.hs = symm.rendezvous(self.s, group)
        self.hi = symm.rendezvous(self.i, group)
        world = self.hs.world_size
        sb = [self.hs.get_buffer(r, (nq, k), torch.int32) for r in range(world)]
        ib = [self.hi.get_buffer(r, (nq, k), torch.int64) for r in range(world)]
        self.world = world
        self.sptr = torch.tensor([t.data_ptr() for t in sb], dtype=torch.int64, device=device)
        self.iptr = torch.tensor([t.data_ptr() for t in ib], dtype=torch.int64, device=device)

    def merge(self, scores: torch.Tensor, ids: torch.Tensor):
        import paper_2506_00528_b200 as uq
        self.s.copy_(scores)
        self.i.copy_(ids)
        self.hs.barrier()          # every rank's lists are in its buffer
        out = uq.merge_topk_ptrs(self.sptr, self.iptr, self.nq, self.k)
        self.hs.barrier()          # every peer has finished reading
        return out


def sharded_search(qcodes: torch.Tensor, db_shard: torch.Tensor, d: int, k: int, id_base: int,
                   group=None, search_fn: Optional[Callable] = None,
                   merge_fn: Optional[Callable] = None, merge_out=None, exchange=None, **search_kw):
    """Local search on this rank's shard + allgather + merge.  Returns the global
    (scores [Q][k], ids [Q][k]) on every rank.  `merge_out` (optional) receives
    the merged result; `exchange` (optional, e.g. PeerExchange.merge) replaces
    the allgather + merge with one peer-memory merge."""
    if search_fn is None or merge_fn is None:
        import paper_2506_00528_b200 as uq
        search_fn = search_fn or uq.search
        merge_fn = merge_fn or uq.merge_topk
    s, i = search_fn(qcodes, db_shard, d, k, id_base=id_base, **search_kw)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return s, i
    if exchange is not None:
        return exchange(s, i)
    sg, ig = allgather_lists(s, i, group)
    return merge_fn(sg, ig, k) if merge_out is None else merge_fn(sg, ig, k, out=merge_out)
