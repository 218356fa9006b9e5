"""CUDA-graph-captured serving path (paper_2506_00528_b200.serving.CapturedSearch).

The captured chain (uq_encode + uq_search) replayed on new query batches must
give, byte for byte, what the direct calls give on the same batches -- and the
oracle's exhaustive kNN on a small database -- for every scan engine.
"""
import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def uq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2506_00528_b200 as m
    return m


def _db(uq, d, n, x, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.randn((n, d), generator=g, device="cuda")
    return uq.encode(u, x)


@pytest.mark.parametrize("engine", ["auto", "popc", "tc", "f4", "f4x"])
@pytest.mark.parametrize("nq", [1, 8, 130])
def test_graph_replay_matches_direct(uq, orc, engine, nq):
    from paper_2506_00528_b200.serving import CapturedSearch
    d, n, x, k = 256, 70_001, 128, 10
    dbc = _db(uq, d, n, x, 11)
    algo = {"auto": uq.ALGO_AUTO, "popc": uq.ALGO_POPC, "tc": uq.ALGO_TCGEN05,
            "f4": uq.ALGO_TC_FP4, "f4x": uq.ALGO_TC_FP4}[engine]
    f4 = uq.build_f4_index(dbc, d) if engine == "f4x" else None
    try:
        cs = CapturedSearch(dbc, d, x, k, nq, algo=algo, f4_index=f4, id_base=5)
    except uq.UQError:
        pytest.skip("engine does not take this shape")
    g = torch.Generator(device="cuda").manual_seed(100 + nq)
    db_h = dbc.cpu().numpy()
    for rep in range(3):
        q = torch.randn((nq, d), generator=g, device="cuda")
        s, i = cs(q)
        s, i = s.clone(), i.clone()
        qc = uq.encode(q, x)
        s2, i2 = uq.search(qc, dbc, d, k, id_base=5, algo=algo, f4_index=f4)
        assert torch.equal(s, s2) and torch.equal(i, i2), (engine, nq, rep)
        if rep == 0:
            qs = np.arange(min(nq, 4))
            o_q = orc.pack(orc.encode(q.cpu().numpy()[qs], x))
            s_ref, i_ref = orc.knn(o_q, db_h, d, k)
            assert np.array_equal(s.cpu().numpy()[qs], s_ref)
            assert np.array_equal(i.cpu().numpy()[qs] - 5, i_ref)


def test_graph_c2_shape_fp16(uq, orc):
    """c2's database (d=768, N=1e6, x=384, k=100) with Q=1 fp16 queries, replayed
    on three query batches; checked against direct calls and, on query 0, the oracle."""
    from paper_2506_00528_b200.serving import CapturedSearch
    w = datagen.CONFIGS["c2"]
    x = w.xs[0]
    u = datagen.rows(w, "db", 0, w.n, "cuda")
    dbc = uq.encode(u, x)
    del u
    qf = datagen.queries(w, "cuda").half()
    cs = CapturedSearch(dbc, w.d, x, w.k, 1, dtype=torch.float16)
    for r in range(3):
        s, i = cs(qf[r:r + 1])
        s2, i2 = uq.search(uq.encode(qf[r:r + 1], x), dbc, w.d, w.k)
        assert torch.equal(s, s2) and torch.equal(i, i2)
    o_q = orc.pack(orc.encode(qf[2:3].float().cpu().numpy(), x))
    s_ref, i_ref = orc.knn(o_q, dbc.cpu().numpy(), w.d, w.k)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)
