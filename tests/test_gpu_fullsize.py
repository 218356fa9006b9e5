"""Full-size BASELINE configs 3-5 on the GPU, checked on sampled outputs.

Each test runs the workload at its BASELINE.json size in the launch shape
bench.py uses (the whole query batch in one uq_search call, AUTO engine, and
the E2M1-index launch the bench times) and checks against the CPU oracle:
  * database codes: the first and last 2^14-row chunks and 64 seeded ones
    (~2^20 rows per x) re-encoded by the oracle;
  * top-k: >= 32 seeded queries per x (c3, c5) and 2 queries at c4's full
    N = 1e8, oracle exhaustive kNN (orc_knn) over ALL database codes the GPU
    produced (those codes verified on the chunks above and, for the smaller
    configs, by the encoder parity tests);
  * sharding (c4): the full result equals, byte for byte, the merge of G = 2,
    4, 8 contiguous shards searched with their global id_base (bench.py
    --shard strong, run sequentially on one GPU).
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


def _encode_db(uq, w, x, out=None, lo=0, hi=None):
    hi = w.n if hi is None else hi
    cb = uq.code_bytes(w.d)
    if out is None:
        out = torch.empty((hi - lo, cb), dtype=torch.uint8, device="cuda")
    for s in range(lo, hi, GEN):
        c = min(GEN, hi - s)
        u = datagen.rows(w, "db", s, c, "cuda")
        uq.encode(u, x, out=out[s - lo:s - lo + c])
        del u
    return out


def _check_chunks(uq, orc, w, x, dbc, rng, nchunks=64):
    last = (w.n - 1) // datagen.CHUNK
    picks = sorted({0, last, *rng.integers(0, last + 1, size=nchunks).tolist()})
    for c in picks:
        s = c * datagen.CHUNK
        cnt = min(datagen.CHUNK, w.n - s)
        u = datagen.rows(w, "db", s, cnt, "cuda").cpu().numpy()   # the bytes the GPU encoded
        ref = orc.pack(orc.encode(u, x))
        got = dbc[s:s + cnt].cpu().numpy()
        assert np.array_equal(got, ref), (w.name, x, c)


def _index_search(uq, qc, dbc, d, k, id_base=0):
    """The bench's launch for the E2M1 engine: the search reads the E2M1 index."""
    return uq.search(qc, dbc, d, k, id_base=id_base, f4_index=uq.build_f4_index(dbc, d))


def _check_queries(orc, w, x, qf_host, qc_gpu, s_gpu, i_gpu, db_h, qs):
    o_q = orc.pack(orc.encode(qf_host[qs], x))
    assert np.array_equal(qc_gpu.cpu().numpy()[qs], o_q)
    s_ref, i_ref = orc.knn(o_q, db_h, w.d, w.k)
    s_g, i_g = s_gpu.cpu().numpy()[qs], i_gpu.cpu().numpy()[qs]
    assert np.array_equal(s_g, s_ref), (w.name, x, np.argwhere(s_g != s_ref)[:5])
    assert np.array_equal(i_g, i_ref), (w.name, x, np.argwhere(i_g != i_ref)[:5])


def test_full_size_c3_sampled(uq, orc):
    """c3: d=1024, N=1e7, Q=1e4, k=10, x swept over {256, 512, 768}: 32 seeded
    queries per x against the oracle; the index-fed launch equals the 2-bit one
    on all 10^4 queries."""
    w = datagen.CONFIGS["c3"]
    rng = np.random.default_rng(3)
    dbc = None
    qf = datagen.queries(w, "cuda")
    qf_h = qf.cpu().numpy()
    for x in w.xs:
        dbc = _encode_db(uq, w, x, dbc)
        _check_chunks(uq, orc, w, x, dbc, rng)
        qc = uq.encode(qf, x)
        s, i = _index_search(uq, qc, dbc, w.d, w.k)
        s2, i2 = uq.search(qc, dbc, w.d, w.k)
        assert torch.equal(s2, s) and torch.equal(i2, i)
        qs = np.sort(rng.choice(w.nq, size=32, replace=False))
        _check_queries(orc, w, x, qf_h, qc, s, i, dbc.cpu().numpy(), qs)


def test_full_size_c5_sampled(uq, orc):
    """c5: fp16 raw mixture, d=768, N=5e7 encoded on the GPU to x=384; Q=1 and
    Q=1024 batches, k=10: query 0 alone (the popcount engine) and 32 seeded
    queries of the 1024 batch (the index-fed E2M1 engine)."""
    w = datagen.CONFIGS["c5"]
    rng = np.random.default_rng(5)
    dbc = _encode_db(uq, w, w.x)
    _check_chunks(uq, orc, w, w.x, dbc, rng)
    qf = datagen.queries(w, "cuda")
    qf_h = qf.cpu().numpy()
    qc_all = uq.encode(qf, w.x)
    s1, i1 = uq.search(qc_all[:1], dbc, w.d, w.k)                 # Q = 1 (HBM-bound popcount scan)
    s, i = _index_search(uq, qc_all, dbc, w.d, w.k)               # Q = 1024
    s2, i2 = uq.search(qc_all, dbc, w.d, w.k)
    assert torch.equal(s2, s) and torch.equal(i2, i)
    assert torch.equal(s1[0], s[0]) and torch.equal(i1[0], i[0])
    qs = np.concatenate([[0], np.sort(rng.choice(np.arange(1, w.nq), size=32, replace=False))])
    _check_queries(orc, w, w.x, qf_h, qc_all, s, i, dbc.cpu().numpy(), qs)


def test_full_size_c4_g1_and_shards(uq, orc):
    """c4 at its BASELINE size on ONE GPU: d=1536, N=1e8 (38.4 GB of codes +
    a 76.8 GB E2M1 index), Q=1e4, x=768, k=100, the bench's index-fed launch;
    2 seeded queries checked against the oracle over all 10^8 codes; then the
    strong-shard plan of bench.py for G = 2, 4, 8 (shard_bounds, global
    id_base, uq_merge_topk) reproduces the G = 1 result byte for byte."""
    from paper_2506_00528_b200.parallel import result_digest, shard_bounds
    w = datagen.CONFIGS["c4"]
    rng = np.random.default_rng(4)
    dbc = _encode_db(uq, w, w.x)
    _check_chunks(uq, orc, w, w.x, dbc, rng)
    qf = datagen.queries(w, "cuda")
    qc = uq.encode(qf, w.x)
    s, i = _index_search(uq, qc, dbc, w.d, w.k)
    torch.cuda.empty_cache()
    want = result_digest([(s, i)])
    for G in (2, 4, 8):
        parts_s, parts_i = [], []
        for r in range(G):
            lo, hi = shard_bounds(w.n, G, r)
            ps, pi = uq.search(qc, dbc[lo:hi], w.d, w.k, id_base=lo)
            parts_s.append(ps)
            parts_i.append(pi)
        ms, mi = uq.merge_topk(torch.stack(parts_s), torch.stack(parts_i), w.k)
        assert result_digest([(ms, mi)]) == want, G
        del parts_s, parts_i
    qs = np.sort(rng.choice(w.nq, size=2, replace=False))
    _check_queries(orc, w, w.x, qf.cpu().numpy(), qc, s, i, dbc.cpu().numpy(), qs)
