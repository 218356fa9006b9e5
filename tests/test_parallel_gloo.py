"""Multi-process (world_size 2 and 3, gloo, CPU) test of the G-GPU host logic:
contiguous sharding, id_base offsets, the allgather of [Q][k] lists and the
final merge.  The per-rank kernels are stood in for by the oracle (CPU); the
orchestration code under test is paper_2506_00528_b200.parallel, unchanged."""
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


def _cpu_search(orc):
    def f(qcodes, db_shard, d, k, id_base=0):
        s, i = orc.knn(qcodes.numpy(), db_shard.numpy(), d, k, id_base=id_base)
        return torch.from_numpy(s), torch.from_numpy(i)
    return f


def _cpu_merge(sg, ig, k):
    sg, ig = sg.numpy(), ig.numpy()
    g, nq, _ = sg.shape
    out_s = np.full((nq, k), np.iinfo(np.int32).min, np.int32)
    out_i = np.full((nq, k), -1, np.int64)
    for q in range(nq):
        c = sorted(((int(sg[a, q, b]), int(ig[a, q, b])) for a in range(g) for b in range(k)
                    if ig[a, q, b] >= 0), key=lambda t: (-t[0], t[1]))[:k]
        out_s[q, :len(c)] = [t[0] for t in c]
        out_i[q, :len(c)] = [t[1] for t in c]
    return torch.from_numpy(out_s), torch.from_numpy(out_i)


def _worker(rank, world, port, n, k, ret):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as orc
    from paper_2506_00528_b200.parallel import shard_bounds, sharded_search
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    d, x, nq = 96, 48, 9
    u = rng.standard_normal((n + nq, d))
    u[n // 3] = u[2 * n // 3]                 # duplicate rows in different shards: tie by id
    codes = orc.pack(orc.encode(u, x))
    db, q = codes[:n], codes[n:]
    q[0] = db[2 * n // 3]
    lo, hi = shard_bounds(n, world, rank)
    s, i = sharded_search(torch.from_numpy(q), torch.from_numpy(db[lo:hi]), d, k, id_base=lo,
                          search_fn=_cpu_search(orc), merge_fn=_cpu_merge)
    ref_s, ref_i = orc.knn(q, db, d, k)
    ret[rank] = bool(np.array_equal(s.numpy(), ref_s) and np.array_equal(i.numpy(), ref_i))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k", [(2, 1000, 10), (3, 10, 5), (2, 3, 7)])
def test_sharded_search_gloo(world, n, k):
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), n, k, ret), nprocs=world,
                       start_method="spawn", join=True)
    assert dict(ret) == {r: True for r in range(world)}


def test_shard_bounds():
    from paper_2506_00528_b200.parallel import shard_bounds
    for n in (0, 1, 7, 100, 10**8):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(w - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def _digest_worker(rank, world, port, ret):
    """bench.py's strong-shard step on CPU stand-ins: shard_bounds -> local
    search with id_base -> sharded_search (allgather + merge) -> result_digest."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as orc
    from paper_2506_00528_b200.parallel import result_digest, shard_bounds, sharded_search
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    d, n, nq, k = 128, 5003, 17, 10
    u = rng.standard_normal((n + nq, d))
    u[100:140] = u[4000]                      # duplicates across shards: ties broken by id
    res = []
    for x in (32, 64, 96):                    # an x sweep, one digest over all of it
        codes = orc.pack(orc.encode(u, x))
        db, q = codes[:n], codes[n:]
        lo, hi = shard_bounds(n, world, rank)
        res.append(sharded_search(torch.from_numpy(q), torch.from_numpy(db[lo:hi]), d, k, id_base=lo,
                                  search_fn=_cpu_search(orc), merge_fn=_cpu_merge))
    ret[rank] = result_digest(res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_strong_shard_digest_equal_across_world(world):
    """The digest bench.py prints is the same for every GPU count: the merged
    result is unique (byte-identical across G)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as orc
    from paper_2506_00528_b200.parallel import result_digest
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    mp.start_processes(_digest_worker, args=(world, _free_port(), ret), nprocs=world,
                       start_method="spawn", join=True)
    rng = np.random.default_rng(11)
    d, n, nq, k = 128, 5003, 17, 10
    u = rng.standard_normal((n + nq, d))
    u[100:140] = u[4000]
    ref = []
    for x in (32, 64, 96):
        codes = orc.pack(orc.encode(u, x))
        s, i = orc.knn(codes[n:], codes[:n], d, k)
        ref.append((torch.from_numpy(s), torch.from_numpy(i)))
    want = result_digest(ref)
    assert dict(ret) == {r: want for r in range(world)}
