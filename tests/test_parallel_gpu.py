"""G-GPU orchestration with the real kernels: two processes (world_size 2,
gloo for the exchange) share the one GPU of the test box; each encodes and
searches its contiguous shard through the C ABI (id_base = shard start), the
per-rank [Q][k] lists are all-gathered (staged through host memory, since the
box has one GPU and NCCL refuses two ranks on one device) and merged by
uq_merge_topk on the GPU.  The result must equal the unsharded search byte for
byte (exactness of the merge under the total order, R8).  The ranks' kernels
never wait on each other; only the host-side collective couples them."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, algo_name):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import paper_2506_00528_b200 as uq
        from paper_2506_00528_b200.parallel import shard_bounds, sharded_search
        torch.cuda.set_device(0)
        algo = {"popc": uq.ALGO_POPC, "tc": uq.ALGO_TCGEN05, "f4": uq.ALGO_TC_FP4, "auto": uq.ALGO_AUTO}[algo_name]
        w = datagen.CONFIGS["c2"].scaled(n=150_000, nq=300)
        lo, hi = shard_bounds(w.n, world, rank)
        db = datagen.rows(w, "db", lo, hi - lo, "cuda")
        dbc = uq.encode(db, w.x)
        qc = uq.encode(datagen.queries(w, "cuda"), w.x)

        def search_fn(q, shard, d, k, id_base=0):
            s, i = uq.search(q, shard, d, k, id_base=id_base, algo=algo)
            return s.cpu(), i.cpu()          # gloo exchanges host tensors

        def merge_fn(sg, ig, k):
            return uq.merge_topk(sg.cuda(), ig.cuda(), k)

        s, i = sharded_search(qc, dbc, w.d, w.k, lo, search_fn=search_fn, merge_fn=merge_fn)
        np.save(os.path.join(out_dir, f"s{rank}.npy"), s.cpu().numpy())
        np.save(os.path.join(out_dir, f"i{rank}.npy"), i.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo", ["popc", "tc", "f4"])
def test_two_rank_sharded_search_real_kernels(tmp_path, algo):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    import datagen
    import paper_2506_00528_b200 as uq
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), algo), nprocs=2, join=True)
    w = datagen.CONFIGS["c2"].scaled(n=150_000, nq=300)
    dbc = uq.encode(datagen.db(w, "cuda"), w.x)
    qc = uq.encode(datagen.queries(w, "cuda"), w.x)
    algo_c = {"popc": uq.ALGO_POPC, "tc": uq.ALGO_TCGEN05, "f4": uq.ALGO_TC_FP4}[algo]
    s_ref, i_ref = uq.search(qc, dbc, w.d, w.k, algo=algo_c)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"s{r}.npy"), s_ref.cpu().numpy())
        assert np.array_equal(np.load(tmp_path / f"i{r}.npy"), i_ref.cpu().numpy())


def _peer_worker(rank, world, port, out_dir):
    """Two processes on the one GPU: each rank's [Q][k] lists live in symmetric
    memory; PeerExchange.merge reads both ranks' buffers through the mapped
    peer pointers in ONE merge kernel (uq_merge_topk_ptrs) between device-side
    barriers.  The result is saved for the parent to compare."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank % torch.cuda.device_count())   # distinct GPUs where the box has them
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    status = "ok"
    try:
        import paper_2506_00528_b200 as uq  # noqa: F401
        from paper_2506_00528_b200.parallel import PeerExchange
        rng = np.random.default_rng(100 + rank)
        nq, k = 33, 12
        s = torch.from_numpy(np.sort(rng.integers(-50, 50, size=(nq, k)), axis=1)[:, ::-1].astype(np.int32).copy()).to(dev)
        i = torch.from_numpy((rank * 1000 + np.stack([np.sort(rng.permutation(500)[:k]) for _ in range(nq)]))
                             .astype(np.int64)).to(dev)
        np.save(os.path.join(out_dir, f"in_s{rank}.npy"), s.cpu().numpy())
        np.save(os.path.join(out_dir, f"in_i{rank}.npy"), i.cpu().numpy())
        try:
            ex = PeerExchange(nq, k, dev)
        except Exception as e:   # symmetric memory refused (one GPU: both ranks' allocations overlap)
            status = f"skip: {type(e).__name__}: {e}"
        else:
            ms, mi = ex.merge(s, i)
            torch.cuda.synchronize()
            np.save(os.path.join(out_dir, f"out_s{rank}.npy"), ms.cpu().numpy())
            np.save(os.path.join(out_dir, f"out_i{rank}.npy"), mi.cpu().numpy())
    except Exception as e:
        status = f"error: {type(e).__name__}: {e}"
    finally:
        with open(os.path.join(out_dir, f"status{rank}.txt"), "w") as f:
            f.write(status)
        dist.destroy_process_group()


def test_two_rank_peer_exchange(tmp_path):
    """The fused exchange + merge over peer memory at world size 2 (one rank per
    GPU where the box has two; on a one-GPU box torch's symmetric-memory
    rendezvous refuses two ranks on one device and the test skips): every
    rank's merged lists equal uq_merge_topk of the two ranks' lists, byte for
    byte."""
    import paper_2506_00528_b200 as uq
    port = _free_port()
    mp.start_processes(_peer_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    st = [open(tmp_path / f"status{r}.txt").read() for r in range(2)]
    if any(x.startswith("skip") for x in st):
        pytest.skip(st[0] if st[0].startswith("skip") else st[1])
    assert st == ["ok", "ok"], st
    s = torch.from_numpy(np.stack([np.load(tmp_path / f"in_s{r}.npy") for r in range(2)])).cuda()
    i = torch.from_numpy(np.stack([np.load(tmp_path / f"in_i{r}.npy") for r in range(2)])).cuda()
    rs, ri = uq.merge_topk(s, i, s.shape[2])
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"out_s{r}.npy"), rs.cpu().numpy())
        assert np.array_equal(np.load(tmp_path / f"out_i{r}.npy"), ri.cpu().numpy())
