"""Seeded random-shape sweep (GPU): every engine -- popcount, int8 and E2M1
tensor pairs, AUTO, single-operand int8 -- against the oracle on random
(n, nq, d, x, k, data mode) draws, bit-exact.  Sizes stay small enough for the
oracle; the draws cover ragged tiles, n < k, nq = 1, d not a multiple of 128,
duplicate rows and grid-valued (tie-heavy) inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def uq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2506_00528_b200 as m
    return m


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([1, 3, 31, 64, 100, 127, 128, 129, 255, 384, 500, 768, 1000, 1024]))
    x = int(rng.integers(1, d + 1))
    n = int(rng.choice([0, 1, 7, 100, 239, 240, 241, 1000, 3001, 9000]))
    nq = int(rng.choice([1, 2, 33, 129, 200, 257]))
    k = int(rng.choice([1, 5, 10, 64, 100, 300]))
    mode = str(rng.choice(["normal", "dup", "ties"]))
    return rng, d, x, n, nq, k, mode


def _data(rng, n, d, mode):
    if mode == "dup":
        base = rng.standard_normal((max(1, n // 5), d)).astype(np.float32)
        return base[rng.integers(0, base.shape[0], size=n)] if n else np.zeros((0, d), np.float32)
    if mode == "ties":
        return (rng.integers(-4, 5, size=(n, d)).astype(np.float32) / 4.0)
    return rng.standard_normal((n, d)).astype(np.float32)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("UQ_FUZZ_N", "160"))))
def test_fuzz_engines(uq, orc, seed):
    rng, d, x, n, nq, k, mode = _draw(seed)
    u_db = _data(rng, n, d, mode)
    u_q = _data(rng, nq, d, mode)
    o_db = orc.pack(orc.encode(u_db, x)) if n else np.zeros((0, 2 * orc.plane_bytes(d)), np.uint8)
    o_q = orc.pack(orc.encode(u_q, x))
    s_ref, i_ref = orc.knn(o_q, o_db, d, k, id_base=11)
    qg, dbg = torch.from_numpy(o_q).cuda(), torch.from_numpy(o_db).cuda()
    ran = 0
    for algo in (uq.ALGO_POPC, uq.ALGO_TCGEN05, uq.ALGO_TC_FP4, uq.ALGO_AUTO):
        try:
            uq.search_workspace(nq, n, d, k, algo)
        except uq.UQError:
            continue   # engine does not take this shape
        s, i = uq.search(qg, dbg, d, k, id_base=11, algo=algo)
        assert np.array_equal(s.cpu().numpy(), s_ref), (seed, algo, d, x, n, nq, k, mode)
        assert np.array_equal(i.cpu().numpy(), i_ref), (seed, algo, d, x, n, nq, k, mode)
        ran += 1
    assert ran >= 1
    try:
        uq.search_workspace(nq, n, d, k, uq.ALGO_TC_FP4)
        f4_ok = n > 0
    except uq.UQError:
        f4_ok = False
    if f4_ok:   # the E2M1 engine fed by the pre-expanded index
        s, i = uq.search(qg, dbg, d, k, id_base=11, f4_index=uq.build_f4_index(dbg, d))
        assert np.array_equal(s.cpu().numpy(), s_ref), (seed, "f4x", d, x, n, nq, k, mode)
        assert np.array_equal(i.cpu().numpy(), i_ref), (seed, "f4x", d, x, n, nq, k, mode)
    if d <= 1024:
        q8 = orc.quantize_i8(u_q)
        s, i = uq.search_asym(torch.from_numpy(q8).cuda(), dbg, d, k, id_base=11)
        s_ref, i_ref = orc.knn_asym(q8, o_db, d, k, id_base=11)
        assert np.array_equal(s.cpu().numpy(), s_ref), (seed, "asym", d, x, n, nq, k, mode)
        assert np.array_equal(i.cpu().numpy(), i_ref), (seed, "asym", d, x, n, nq, k, mode)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_seeded(uq, orc, seed):
    """Random shapes large enough for threshold seeding (n >= 2^16): optimistic
    histogram seeds, their verification and fallback, every engine."""
    rng = np.random.default_rng(5000 + seed)
    d = int(rng.choice([64, 128, 256, 384, 768]))
    x = int(rng.integers(1, d + 1))
    n = int(rng.choice([65536, 70001, 131072, 200003]))
    nq = int(rng.choice([9, 130, 257, 300]))
    k = int(rng.choice([1, 10, 100, 300]))
    mode = str(rng.choice(["normal", "dup", "ties"]))
    u_db, u_q = _data(rng, n, d, mode), _data(rng, nq, d, mode)
    o_db, o_q = orc.pack(orc.encode(u_db, x)), orc.pack(orc.encode(u_q, x))
    s_ref, i_ref = orc.knn(o_q, o_db, d, k)
    qg, dbg = torch.from_numpy(o_q).cuda(), torch.from_numpy(o_db).cuda()
    runs = [dict(algo=a) for a in (uq.ALGO_POPC, uq.ALGO_TCGEN05, uq.ALGO_TC_FP4, uq.ALGO_AUTO)]
    runs.append(dict(f4_index=uq.build_f4_index(dbg, d)))
    for kw in runs:
        try:
            uq.search_workspace(nq, n, d, k, kw.get("algo", uq.ALGO_TC_FP4))
        except uq.UQError:
            continue
        s, i = uq.search(qg, dbg, d, k, **kw)
        tag = (seed, tuple(kw), d, x, n, nq, k, mode)
        assert np.array_equal(s.cpu().numpy(), s_ref), tag
        assert np.array_equal(i.cpu().numpy(), i_ref), tag
