"""Full-size BASELINE configs 3-5 on the GPU, checked on sampled outputs.

Each test runs the workload at its BASELINE.json size in the launch shape
bench.py uses (the whole query batch in one uq_search call, AUTO engine) and
checks against the CPU oracle:
  * database codes: whole seeded 2^14-row chunks re-encoded by the oracle;
  * top-k: a few seeded queries, oracle exhaustive kNN (orc_knn) over ALL
    database codes the GPU produced (those codes verified on the chunks above
    and, for the smaller configs, by the encoder parity tests).
The float database is generated and encoded chunk by chunk, so configs whose
floats exceed HBM (c4: 614 GB fp32) never materialise them; the oracle gets the
exact float bytes the GPU encoded (generated on the device, copied to the host:
torch's CPU and CUDA generators differ).
"""
import numpy as np
import pytest
import torch

import datagen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GEN = 1 << 22  # rows generated + encoded per step


@pytest.fixture(scope="module")
def uq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2506_00528_b200 as m
    return m


def _encode_db(uq, w, x, out=None):
    cb = uq.code_bytes(w.d)
    if out is None:
        out = torch.empty((w.n, cb), dtype=torch.uint8, device="cuda")
    for s in range(0, w.n, GEN):
        c = min(GEN, w.n - s)
        u = datagen.rows(w, "db", s, c, "cuda")
        uq.encode(u, x, out=out[s:s + c])
        del u
    return out


def _check_chunks(uq, orc, w, x, dbc, rng, nchunks=2):
    last = (w.n - 1) // datagen.CHUNK
    picks = sorted({0, last, *rng.integers(0, last + 1, size=nchunks).tolist()})
    for c in picks:
        s = c * datagen.CHUNK
        cnt = min(datagen.CHUNK, w.n - s)
        u = datagen.rows(w, "db", s, cnt, "cuda").cpu().numpy()   # the bytes the GPU encoded
        ref = orc.pack(orc.encode(u, x))
        got = dbc[s:s + cnt].cpu().numpy()
        assert np.array_equal(got, ref), (w.name, x, c)


def _check_index_path(uq, qc, dbc, d, k, s, i):
    """The bench's launch configuration for the E2M1 engine reads the E2M1 index:
    its full result must equal the 2-bit path's byte for byte (all queries)."""
    s2, i2 = uq.search(qc, dbc, d, k, f4_index=uq.build_f4_index(dbc, d))
    assert torch.equal(s2, s) and torch.equal(i2, i)


def _check_queries(uq, orc, w, x, qc_gpu, s_gpu, i_gpu, dbc, rng, nsample):
    qs = np.sort(rng.choice(w.nq, size=nsample, replace=False))
    q = datagen.queries(w, "cuda").cpu().numpy()[qs]
    o_q = orc.pack(orc.encode(q, x))
    assert np.array_equal(qc_gpu.cpu().numpy()[qs], o_q)
    db_h = dbc.cpu().numpy()
    s_ref, i_ref = orc.knn(o_q, db_h, w.d, w.k)
    assert np.array_equal(s_gpu.cpu().numpy()[qs], s_ref), (w.name, x)
    assert np.array_equal(i_gpu.cpu().numpy()[qs], i_ref), (w.name, x)


def test_full_size_c3_sampled(uq, orc):
    """c3: d=1024, N=1e7, Q=1e4, k=10, x swept over {256, 512, 768}."""
    w = datagen.CONFIGS["c3"]
    rng = np.random.default_rng(3)
    dbc = None
    qf = datagen.queries(w, "cuda")
    for x in w.xs:
        dbc = _encode_db(uq, w, x, dbc)
        _check_chunks(uq, orc, w, x, dbc, rng)
        qc = uq.encode(qf, x)
        s, i = uq.search(qc, dbc, w.d, w.k)
        _check_queries(uq, orc, w, x, qc, s, i, dbc, rng, nsample=6)
        _check_index_path(uq, qc, dbc, w.d, w.k, s, i)


def test_full_size_c5_sampled(uq, orc):
    """c5: fp16 raw mixture, d=768, N=5e7 encoded on the GPU to x=384; Q=1 and
    Q=1024 batches, k=10."""
    w = datagen.CONFIGS["c5"]
    rng = np.random.default_rng(5)
    dbc = _encode_db(uq, w, w.x)
    _check_chunks(uq, orc, w, w.x, dbc, rng)
    qf = datagen.queries(w, "cuda")
    qc_all = uq.encode(qf, w.x)
    # Q = 1 (the HBM-bound case) and Q = 1024
    s1, i1 = uq.search(qc_all[:1], dbc, w.d, w.k)
    s, i = uq.search(qc_all, dbc, w.d, w.k)
    _check_index_path(uq, qc_all, dbc, w.d, w.k, s, i)
    db_h = dbc.cpu().numpy()
    qs = np.concatenate([[0], np.sort(rng.choice(np.arange(1, w.nq), size=3, replace=False))])
    o_q = orc.pack(orc.encode(qf.cpu().numpy()[qs], w.x))
    assert np.array_equal(qc_all.cpu().numpy()[qs], o_q)
    s_ref, i_ref = orc.knn(o_q, db_h, w.d, w.k)
    assert np.array_equal(s1.cpu().numpy()[0], s_ref[0])
    assert np.array_equal(i1.cpu().numpy()[0], i_ref[0])
    assert np.array_equal(s.cpu().numpy()[qs], s_ref)
    assert np.array_equal(i.cpu().numpy()[qs], i_ref)


def test_full_size_c4_shard_sampled(uq, orc):
    """c4: d=1536, N=1e8 sharded over 8 GPUs, Q=1e4, x=768, k=100: the per-GPU
    work of the 8-GPU configuration -- rank 5's shard, rows [5N/8, 6N/8)
    (12.5M rows, 4.8 GB of codes), searched with id_base = 5N/8 as bench.py's
    ranks do; the merge across shards is test_sharded_equals_unsharded."""
    w = datagen.CONFIGS["c4"]
    G, rank = 8, 5
    lo, hi = rank * w.n // G, (rank + 1) * w.n // G
    rng = np.random.default_rng(4)
    cb = uq.code_bytes(w.d)
    dbc = torch.empty((hi - lo, cb), dtype=torch.uint8, device="cuda")
    for s0 in range(lo, hi, GEN):
        c = min(GEN, hi - s0)
        uq.encode(datagen.rows(w, "db", s0, c, "cuda"), w.x, out=dbc[s0 - lo:s0 - lo + c])
    c0 = lo // datagen.CHUNK + 1          # a whole chunk inside the shard
    u = datagen.rows(w, "db", c0 * datagen.CHUNK, datagen.CHUNK, "cuda").cpu().numpy()
    off = c0 * datagen.CHUNK - lo
    assert np.array_equal(dbc[off:off + datagen.CHUNK].cpu().numpy(), orc.pack(orc.encode(u, w.x)))
    qf = datagen.queries(w, "cuda")
    qc = uq.encode(qf, w.x)
    s, i = uq.search(qc, dbc, w.d, w.k, id_base=lo)
    s2, i2 = uq.search(qc, dbc, w.d, w.k, id_base=lo, f4_index=uq.build_f4_index(dbc, w.d))
    assert torch.equal(s2, s) and torch.equal(i2, i)   # the bench's index-fed launch, all queries
    qs = np.sort(rng.choice(w.nq, size=3, replace=False))
    o_q = orc.pack(orc.encode(qf.cpu().numpy()[qs], w.x))
    assert np.array_equal(qc.cpu().numpy()[qs], o_q)
    s_ref, i_ref = orc.knn(o_q, dbc.cpu().numpy(), w.d, w.k, id_base=lo)
    assert np.array_equal(s.cpu().numpy()[qs], s_ref)
    assert np.array_equal(i.cpu().numpy()[qs], i_ref)
