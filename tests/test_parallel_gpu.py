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
