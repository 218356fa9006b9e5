"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element, on the same seeded inputs.  Integer / index outputs: bit-exact.

Sizes span several tiles plus ragged tails; full BASELINE sizes are checked on
sampled outputs (test_full_size_*).
"""
import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu

ALGOS = ("popc", "tc", "f4")


@pytest.fixture(scope="module")
def uq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2506_00528_b200 as m
    return m


def _algo(uq, name):
    return {"popc": uq.ALGO_POPC, "tc": uq.ALGO_TCGEN05, "f4": uq.ALGO_TC_FP4, "auto": uq.ALGO_AUTO}[name]


def _tc_supported(uq, nq, n, d, k, algo=None):
    try:
        uq.search_workspace(nq, n, d, k, uq.ALGO_TCGEN05 if algo is None else algo)
        return True
    except uq.UQError:
        return False


def _tie_heavy(rng, n, d, dtype=np.float32):
    """Values on a small grid: many exact |u| ties, zeros and -0.0 (encoder stress)."""
    u = rng.integers(-6, 7, size=(n, d)).astype(np.float32) / 8.0
    u[rng.random((n, d)) < 0.02] = -0.0
    return u.astype(dtype)


# --------------------------------------------------------------------------
# Encoder + pack
# --------------------------------------------------------------------------
@pytest.mark.parametrize("d", [1, 7, 10, 100, 128, 129, 300, 384, 768, 1000, 1024, 1536, 2048])
@pytest.mark.parametrize("dt", [torch.float32, torch.float16, torch.bfloat16])
def test_encode_parity_shapes(uq, orc, d, dt):
    rng = np.random.default_rng(d * 7 + 1)
    n = 777
    u = rng.standard_normal((n, d)).astype(np.float32)
    u[: n // 3] = _tie_heavy(rng, n // 3, d)
    ut = torch.from_numpy(u).to(dt)
    host = ut.float().numpy() if dt == torch.bfloat16 else ut.numpy()
    for x in sorted({1, max(1, d // 3), max(1, d // 2), max(1, (2 * d) // 3), d}):
        got = uq.encode(ut.cuda(), x).cpu().numpy()
        ref = orc.pack(orc.encode(host, x))
        assert np.array_equal(got, ref), (d, dt, x, np.argwhere((got != ref).any(1))[:5])


@pytest.mark.parametrize("dt", [torch.float32, torch.float16, torch.bfloat16])
def test_encode_extreme_distributions(uq, orc, dt):
    """Rows the search's probes mis-estimate: subnormal magnitudes, huge dynamic
    range, heavy tails, constants, all-zero rows, one-hot rows; interleaved so a
    warp's learned T*/RMS ratio is wrong for the next row (exactness must not
    depend on the probes)."""
    rng = np.random.default_rng(11)
    d, n = 768, 60000
    kinds = []
    base = rng.standard_normal((n, d)).astype(np.float32)
    tiny = 6e-8 if dt == torch.float16 else (1e-39 if dt == torch.float32 else 1e-38)
    for i in range(n):
        k = i % 7
        if k == 1:
            base[i] *= tiny                                   # subnormal range
        elif k == 2:
            base[i] *= np.float32(10.0) ** rng.integers(-4, 4, d)   # wide dynamic range
        elif k == 3:
            base[i] = rng.standard_cauchy(d).clip(-6e4, 6e4)  # heavy tails
        elif k == 4:
            base[i] = np.float32(rng.integers(-2, 3))         # constant (all ties or zeros)
        elif k == 5:
            base[i] = 0.0
            base[i, rng.integers(0, d)] = -1.0                # one non-zero
        elif k == 6:
            base[i] = np.abs(base[i]) + 1.0                   # all magnitudes in [1, ~5]
    ut = torch.from_numpy(base).to(dt)
    host = ut.float().numpy()
    for x in (1, 256, 384, 700, 768):
        got = uq.encode(ut.cuda(), x).cpu().numpy()
        ref = orc.pack(orc.encode(host if dt != torch.float16 else ut.numpy(), x))
        bad = np.argwhere((got != ref).any(1))[:5].ravel()
        assert bad.size == 0, (dt, x, bad, bad % 7)


@pytest.mark.parametrize("dt", [torch.float32, torch.float16])
def test_encode_threshold_boundaries(uq, orc, dt):
    """T* placed on the encoders' internal boundaries: row scales 2^k sweeping
    the whole exponent range (f32: the f16 coarse keys underflow / saturate and
    the FMA-pipe selection's S = 1/ulp(T-) leaves its range below 2^-104; f16:
    subnormal thresholds), magnitudes that are exact powers of two (T* on a
    binade edge, massive ties), values one f32 ulp apart inside one coarse value
    (the full-key phase), and values at / beyond the f16 maximum."""
    rng = np.random.default_rng(23)
    d = 768
    rows = []
    if dt == torch.float32:
        scales = [-149, -140, -130, -127, -126, -120, -110, -106, -105, -104, -103, -102, -100, -60, -24, -15,
                  -14, 0, 15, 16, 17, 40, 100, 120, 124]
    else:
        scales = [-24, -22, -20, -16, -15, -14, -13, -10, 0, 5, 10, 12, 13]
    for k in scales:
        for _ in range(3):
            rows.append(rng.standard_normal(d) * 2.0 ** k)
    for _ in range(12):
        rows.append(np.sign(rng.standard_normal(d)) * 2.0 ** rng.integers(-3, 4, d))      # binade edges, ties
    if dt == torch.float32:
        one = np.float32(1.0)
        for _ in range(12):                                   # one f32 ulp apart, one coarse value
            steps = rng.integers(0, 40, d).astype(np.float32)
            rows.append(np.sign(rng.standard_normal(d)) * (one + steps * np.float32(2.0 ** -23)))
        for _ in range(6):                                    # at / beyond the f16 maximum (coarse clamp)
            rows.append(np.sign(rng.standard_normal(d)) * (65504.0 + rng.integers(0, 64, d).astype(np.float64)))
    else:
        for _ in range(6):
            rows.append(np.sign(rng.standard_normal(d)) * (65504.0 - 32.0 * rng.integers(0, 4, d)))
    host = np.stack(rows).astype(np.float32)
    if dt == torch.float32:
        host = np.clip(host, -3.0e38, 3.0e38)
    ut = torch.from_numpy(host).to(dt)
    ref_in = ut.numpy() if dt == torch.float16 else ut.numpy()
    for x in (1, 2, 200, 384, 383, 767, 768):
        got = uq.encode(ut.cuda(), x).cpu().numpy()
        ref = orc.pack(orc.encode(ref_in, x))
        bad = np.argwhere((got != ref).any(1))[:5].ravel()
        assert bad.size == 0, (dt, x, bad)


def test_encode_strided_and_table3(uq, orc):
    import json, os
    t = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_p356.json")))
    u = torch.tensor([t["u1"], t["u2"]], dtype=torch.float32)
    got = uq.encode(u.cuda(), 5).cpu().numpy()
    assert np.array_equal(got, orc.pack(orc.encode(u.numpy(), 5)))
    assert got[0, 0] == 0x63 and got[0, 16] == 0x04          # v1+ / v1- of P:369-370
    # row stride > d (ld_elems), unaligned row starts -> scalar-load path
    rng = np.random.default_rng(0)
    big = torch.from_numpy(rng.standard_normal((300, 401)).astype(np.float32)).cuda()
    for view in (big[:, :384], big[:, 1:385], big[:, 3:300]):
        d = view.shape[1]
        got = uq.encode(view, d // 2).cpu().numpy()
        ref = orc.pack(orc.encode(view.cpu().numpy(), d // 2))
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("d", [128, 384, 768, 1024])
def test_encode_f16_row_pairs(uq, orc, d):
    """fp16 rows with d = 128k run two rows per warp (one per half-warp): odd
    and even row counts (the odd row out is duplicated, not stored), tiny n,
    and neighbouring rows of very different kinds so the two halves of a warp
    take different search paths (exact / ties / T* = 0 / extrapolation)."""
    rng = np.random.default_rng(d + 5)
    for n in (1, 2, 3, 17, 1000):
        u = rng.standard_normal((n, d)).astype(np.float32)
        u[1::4] = _tie_heavy(rng, len(u[1::4]), d)
        u[2::4] *= np.float32(1e-3) ** rng.integers(0, 3, (len(u[2::4]), 1))
        u[3::8] = 0.0
        u[3::8, ::5] = 1.0
        ut = torch.from_numpy(u).to(torch.float16)
        for x in sorted({1, d // 3, d // 2, d - 1, d}):
            got = uq.encode(ut.cuda(), x).cpu().numpy()
            ref = orc.pack(orc.encode(ut.numpy(), x))
            bad = np.argwhere((got != ref).any(1))[:5].ravel()
            assert bad.size == 0, (d, n, x, bad)


@pytest.mark.parametrize("d", [256, 512, 768, 1024])
def test_encode_f16_batched_rows(uq, orc, d):
    """Large-n fp16 encodes with d = 256k: the shape the batched kernel serves
    when the library is built with -DUQ_ENC16_BATCH=1 (8 or 4 rows per warp
    iteration staged in shared memory, lane r owning row r's search; measured
    slower and compiled out by default, DESIGN.md section 7 -- the default
    build runs the one-row-per-warp kernel here): a ragged row count (last batch partial, rows 1..7 of it), batches
    whose rows take different paths and different pass counts (exact at the
    probe / ties / T* = 0 / extrapolation far outside the learned ratio /
    subnormal and near-maximum scales / binade-edge ties), and a small-n call
    (one row per warp kernel) that must return the same bytes."""
    rng = np.random.default_rng(d + 77)
    n = 20011
    u = rng.standard_normal((n, d)).astype(np.float32)
    u[1::5] = _tie_heavy(rng, len(u[1::5]), d)
    u[2::7] *= np.float32(2.0) ** rng.integers(-22, 14, (len(u[2::7]), 1))
    u[3::11] = 0.0
    u[3::11, ::5] = 1.0
    u[4::13] = np.sign(u[4::13]) * np.float32(2.0) ** rng.integers(-3, 4, u[4::13].shape)
    u[6::17] = 0.0
    u[9::19] = np.float32(0.5)
    ut = torch.from_numpy(u).to(torch.float16)
    host = ut.numpy()
    for x in sorted({1, d // 4, d // 2, d - 1, d}):
        got = uq.encode(ut.cuda(), x).cpu().numpy()
        ref = orc.pack(orc.encode(host, x))
        bad = np.argwhere((got != ref).any(1))[:5].ravel()
        assert bad.size == 0, (d, x, bad)
        small = uq.encode(ut[:1003].cuda(), x).cpu().numpy()
        assert np.array_equal(small, ref[:1003]), (d, x)


def test_encode_c5_fp16_unnormalised(uq, orc):
    """Config 5 recipe (fp16, raw mixture values; ~10% of rows tie at the top-x boundary)."""
    w = datagen.CONFIGS["c5"].scaled(n=20000, nq=16)
    u = datagen.db(w, "cuda")
    got = uq.encode(u, w.x).cpu().numpy()
    ref = orc.pack(orc.encode(u.cpu().numpy(), w.x))
    assert np.array_equal(got, ref)


# --------------------------------------------------------------------------
# Dense Delta
# --------------------------------------------------------------------------
@pytest.mark.parametrize("d", [10, 384, 1000])
def test_scores_parity(uq, orc, d):
    rng = np.random.default_rng(d)
    u = rng.standard_normal((1100, d)).astype(np.float32)
    codes = uq.encode(torch.from_numpy(u).cuda(), max(1, d // 2))
    q, db = codes[:60], codes[60:]
    got = uq.scores(q, db, d).cpu().numpy()
    ref = orc.scores(q.cpu().numpy(), db.cpu().numpy(), d)
    assert np.array_equal(got, ref)


# --------------------------------------------------------------------------
# Search: scan + fused top-k + merge, every engine, ragged shapes, ties
# --------------------------------------------------------------------------
def _search_case(uq, orc, algo, d, x, n, nq, k, seed=0, mode="normal"):
    rng = np.random.default_rng(seed)
    if mode == "dup":
        base = rng.standard_normal((max(1, n // 7), d)).astype(np.float32)
        u_db = base[rng.integers(0, base.shape[0], size=n)]
    elif mode == "ties":
        u_db = _tie_heavy(rng, n, d)
    else:
        u_db = rng.standard_normal((n, d)).astype(np.float32)
    u_q = rng.standard_normal((nq, d)).astype(np.float32)
    if n > 0 and nq > 1:
        u_q[0] = u_db[n // 2]   # a stored vector as query: self-match first
    o_db = orc.pack(orc.encode(u_db, x)) if n else np.zeros((0, 2 * orc.plane_bytes(d)), np.uint8)
    o_q = orc.pack(orc.encode(u_q, x))
    a = _algo(uq, algo)
    if algo in ("tc", "f4") and not _tc_supported(uq, nq, n, d, k, a):
        pytest.skip("tcgen05 path does not support this shape")
    s, i = uq.search(torch.from_numpy(o_q).cuda(), torch.from_numpy(o_db).cuda(), d, k,
                     id_base=5, algo=a)
    s_ref, i_ref = orc.knn(o_q, o_db, d, k, id_base=5)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    assert np.array_equal(s, s_ref), (algo, d, n, nq, k, np.argwhere(s != s_ref)[:5])
    assert np.array_equal(i, i_ref), (algo, d, n, nq, k, np.argwhere(i != i_ref)[:5])


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("n,nq,k", [(0, 3, 4), (1, 2, 1), (9, 4, 10), (255, 1, 10), (257, 65, 10),
                                    (1000, 100, 100), (5000, 130, 10), (3000, 7, 1024),
                                    (20000, 200, 100), (70000, 3, 10)])
def test_search_parity_shapes(uq, orc, algo, n, nq, k):
    _search_case(uq, orc, algo, 384, 192, n, nq, k, seed=n + nq + k)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("d,x", [(10, 5), (100, 67), (768, 384), (1000, 667), (1024, 256),
                                 (1152, 576), (1536, 768), (2048, 1024), (129, 1)])
def test_search_parity_dims(uq, orc, algo, d, x):
    _search_case(uq, orc, algo, d, x, 6000, 150, 10, seed=d)


@pytest.mark.parametrize("algo", ["tc", "f4"])
def test_search_parity_large_k_pairs(uq, orc, algo):
    """Pair engines with k = 1000: counted candidate lists larger than the merge's
    shared-memory stage (its global-memory fallback) and many in-loop cuts."""
    _search_case(uq, orc, algo, 384, 192, 300_000, 200, 1000, seed=77, mode="dup")


@pytest.mark.parametrize("algo", ALGOS)
def test_search_parity_wide_d_seeded(uq, orc, algo):
    """d = 1536 (config 4's width: the one-CTA tensor engine with N = 64 tiles),
    several query tiles, a database large enough for threshold seeding."""
    _search_case(uq, orc, algo, 1536, 768, 70001, 300, 100, seed=1536, mode="dup")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("mode", ["dup", "ties"])
def test_search_parity_ties(uq, orc, algo, mode):
    """Duplicated rows / grid-valued inputs: massive Delta ties -> order decided by id."""
    _search_case(uq, orc, algo, 256, 128, 9000, 140, 50, seed=3, mode=mode)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("mode,n,k", [("dup", 131072, 100), ("ties", 100000, 10), ("normal", 70001, 1)])
def test_search_parity_seeded(uq, orc, algo, mode, n, k):
    """n >= 2^16 turns on threshold seeding (a strided-sample pre-scan); exactness must
    hold with massive ties at the seeded threshold."""
    _search_case(uq, orc, algo, 128, 64, n, 130, k, seed=11, mode=mode)


@pytest.mark.parametrize("algo", ALGOS)
def test_search_c1_full(uq, orc, algo):
    """BASELINE config 1 at full size (N=10,000, Q=100, d=384, x=192, k=10)."""
    w = datagen.CONFIGS["c1"]
    db = datagen.db(w, "cuda")
    q = datagen.queries(w, "cuda")
    dbc, qc = uq.encode(db, w.x), uq.encode(q, w.x)
    o_db = orc.pack(orc.encode(db.cpu().numpy(), w.x))
    o_q = orc.pack(orc.encode(q.cpu().numpy(), w.x))
    assert np.array_equal(dbc.cpu().numpy(), o_db) and np.array_equal(qc.cpu().numpy(), o_q)
    assert np.array_equal(uq.scores(qc, dbc, w.d).cpu().numpy(), orc.scores(o_q, o_db, w.d))
    if algo in ("tc", "f4") and not _tc_supported(uq, w.nq, w.n, w.d, w.k, _algo(uq, algo)):
        pytest.skip("tcgen05 path does not support this shape")
    s, i = uq.search(qc, dbc, w.d, w.k, algo=_algo(uq, algo))
    s_ref, i_ref = orc.knn(o_q, o_db, w.d, w.k)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)


def test_full_size_c2_all(uq, orc):
    """Config 2 at full size in the bench launch shape (N=1e6, Q=1000, k=100, AUTO
    and the E2M1-index launch the bench times): EVERY database code and EVERY
    query's top-k against the oracle (oracle-encoded rows, exhaustive kNN)."""
    w = datagen.CONFIGS["c2"]
    db = datagen.db(w, "cuda")
    q = datagen.queries(w, "cuda")
    dbc, qc = uq.encode(db, w.x), uq.encode(q, w.x)
    s, i = uq.search(qc, dbc, w.d, w.k)              # whole batch, AUTO engine
    # bench.py's launch: the E2M1 engine reading the E2M1 index -- all queries equal
    s2, i2 = uq.search(qc, dbc, w.d, w.k, f4_index=uq.build_f4_index(dbc, w.d))
    assert torch.equal(s2, s) and torch.equal(i2, i)
    db_h = db.cpu().numpy()
    del db
    o_db = orc.pack(orc.encode(db_h, w.x))
    assert np.array_equal(dbc.cpu().numpy(), o_db)
    o_q = orc.pack(orc.encode(q.cpu().numpy(), w.x))
    assert np.array_equal(qc.cpu().numpy(), o_q)
    s_ref, i_ref = orc.knn(o_q, o_db, w.d, w.k)
    assert np.array_equal(s.cpu().numpy(), s_ref)
    assert np.array_equal(i.cpu().numpy(), i_ref)


# --------------------------------------------------------------------------
# Merge (multi-GPU exchange step) and sharding invariance
# --------------------------------------------------------------------------
def test_merge_topk_parity(uq, orc):
    rng = np.random.default_rng(8)
    g, nq, k = 5, 33, 17
    sc = rng.integers(-20, 21, size=(g, nq, k)).astype(np.int32)
    ids = np.empty((g, nq, k), np.int64)
    for q in range(nq):
        ids[:, q, :] = rng.permutation(10 * g * k)[: g * k].reshape(g, k)
    ids[1, :, 10:] = -1                       # padding entries
    sc[1, :, 10:] = np.iinfo(np.int32).min
    s, i = uq.merge_topk(torch.from_numpy(sc).cuda(), torch.from_numpy(ids).cuda(), k)
    for q in range(nq):
        cand = [(int(sc[a, q, b]), int(ids[a, q, b])) for a in range(g) for b in range(k)
                if ids[a, q, b] >= 0]
        cand.sort(key=lambda t: (-t[0], t[1]))
        assert s[q].cpu().tolist() == [c[0] for c in cand[:k]]
        assert i[q].cpu().tolist() == [c[1] for c in cand[:k]]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_sharded_equals_unsharded(uq, orc, algo, G):
    """Shard -> local search with id_base -> merge == unsharded search (R8)."""
    rng = np.random.default_rng(G)
    d, x, n, nq, k = 768, 384, 20000, 96, 100
    u = torch.from_numpy(rng.standard_normal((n + nq, d)).astype(np.float32)).cuda()
    codes = uq.encode(u, x)
    db, q = codes[:n], codes[n:]
    a = _algo(uq, algo)
    if algo in ("tc", "f4") and not _tc_supported(uq, nq, n // G, d, k, a):
        pytest.skip("tcgen05 path does not support this shape")
    s0, i0 = uq.search(q, db, d, k, algo=a)
    bounds = np.linspace(0, n, G + 1).astype(int)
    parts = [uq.search(q, db[bounds[j]:bounds[j + 1]], d, k, id_base=int(bounds[j]), algo=a)
             for j in range(G)]
    s, i = uq.merge_topk(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]), k)
    assert torch.equal(s, s0) and torch.equal(i, i0)
    o = orc.knn(q.cpu().numpy(), db.cpu().numpy(), d, k)
    assert np.array_equal(s0.cpu().numpy(), o[0]) and np.array_equal(i0.cpu().numpy(), o[1])


def test_check_codes_parity(uq, orc):
    rng = np.random.default_rng(4)
    d = 300
    codes = uq.encode(torch.from_numpy(rng.standard_normal((500, d)).astype(np.float32)).cuda(), 100)
    assert uq.check_codes(codes, d) == 0
    h = codes.cpu().numpy()
    pb = h.shape[1] // 2
    h[3, 0] |= 1; h[3, pb] |= 1
    h[9, pb - 1] |= 0x80           # pos-plane pad bit 383 >= d
    h[10, 2 * pb - 2] |= 0x01      # neg-plane pad bit 368 >= d
    assert uq.check_codes(torch.from_numpy(h).cuda(), d) == orc.check_codes(h, d) == 3


def test_errors_are_loud(uq):
    with pytest.raises(uq.UQError):
        uq.encode(torch.zeros(4, 16, device="cuda"), 0)
    with pytest.raises(ValueError):
        uq.encode(torch.zeros(4, 16), 4)          # CPU tensor: no CPU path


@pytest.mark.parametrize("algo", ["tc", "f4"])
@pytest.mark.parametrize("opt,k", [("0", 100), ("3", 100), ("0.01", 500), ("0.01", 100)])
@pytest.mark.parametrize("mode", ["normal", "dup"])
def test_seed_optimistic_fallback(uq, orc, monkeypatch, algo, opt, k, mode):
    """Pair engines seed with an OPTIMISTIC bound (about c*k rows expected above
    it, c = UQ_SEED_OPT, default 3; 0 = exact bound).  A query with fewer than k
    rows above its bound is searched again without one; c = 0.01 forces that
    fallback (need = 8 sampled rows, ~128 expected above < k = 500).  Results
    stay bit-exact in every case."""
    monkeypatch.setenv("UQ_SEED_OPT", opt)
    _search_case(uq, orc, algo, 256, 128, 131072, 300, k, seed=5 + k, mode=mode)


# --------------------------------------------------------------------------
# Single-operand search: int8 queries x ternary DB, masked addition
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dt", [torch.float32, torch.float16, torch.bfloat16])
@pytest.mark.parametrize("d", [1, 10, 100, 384, 768, 1000, 1536])
def test_quantize_i8_parity(uq, orc, dt, d):
    rng = np.random.default_rng(d + 17)
    n = 333
    u = rng.standard_normal((n, d)).astype(np.float32)
    u[: n // 4] = _tie_heavy(rng, n // 4, d)       # exact .5 products -> round-half-even
    u[5] = 0.0                                      # zero row
    ut = torch.from_numpy(u).to(dt)
    host = ut.float().numpy()                       # exact widening of f16 / bf16
    got = uq.quantize_i8(ut.cuda()).cpu().numpy()
    assert np.array_equal(got, orc.quantize_i8(host))


def _asym_case(uq, orc, d, x, n, nq, k, seed=0, mode="normal"):
    rng = np.random.default_rng(seed)
    if mode == "dup":
        base = rng.standard_normal((max(1, n // 7), d)).astype(np.float32)
        u_db = base[rng.integers(0, base.shape[0], size=n)]
    elif mode == "ties":
        u_db = _tie_heavy(rng, n, d)
    else:
        u_db = rng.standard_normal((n, d)).astype(np.float32)
    u_q = rng.standard_normal((nq, d)).astype(np.float32)
    if mode == "ties":
        u_q = _tie_heavy(rng, nq, d)
    o_db = orc.pack(orc.encode(u_db, x)) if n else np.zeros((0, 2 * orc.plane_bytes(d)), np.uint8)
    q8 = orc.quantize_i8(u_q)
    s, i = uq.search_asym(torch.from_numpy(q8).cuda(), torch.from_numpy(o_db).cuda(), d, k, id_base=7)
    s_ref, i_ref = orc.knn_asym(q8, o_db, d, k, id_base=7)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    assert np.array_equal(s, s_ref), (d, n, nq, k, np.argwhere(s != s_ref)[:5])
    assert np.array_equal(i, i_ref), (d, n, nq, k, np.argwhere(i != i_ref)[:5])


@pytest.mark.parametrize("n,nq,k", [(0, 3, 4), (1, 2, 1), (9, 4, 10), (257, 1, 10), (5000, 130, 10),
                                    (3000, 7, 1024), (20000, 300, 100), (70001, 33, 10)])
def test_search_asym_parity_shapes(uq, orc, n, nq, k):
    _asym_case(uq, orc, 384, 192, n, nq, k, seed=n + nq + k)


@pytest.mark.parametrize("d,x", [(10, 5), (100, 67), (768, 384), (1000, 667), (1024, 256), (129, 1)])
def test_search_asym_parity_dims(uq, orc, d, x):
    _asym_case(uq, orc, d, x, 6000, 150, 10, seed=d)


@pytest.mark.parametrize("mode,n,k", [("dup", 131072, 100), ("ties", 100000, 10), ("normal", 70001, 1)])
def test_search_asym_parity_seeded(uq, orc, mode, n, k):
    """n >= 2^16: the exact 1/32-sample seed; massive score ties decided by id."""
    _asym_case(uq, orc, 128, 64, n, 260, k, seed=13, mode=mode)


def test_search_asym_full_size_c2_sampled(uq, orc):
    """c2 at full size (N = 10^6, Q = 1000, k = 100): int8 queries from the GPU
    quantiser (checked against the oracle's), top-k of 6 seeded queries against
    the oracle's exhaustive masked-addition kNN over all 10^6 oracle-encoded rows."""
    w = datagen.CONFIGS["c2"]
    db = datagen.db(w, "cuda")
    q = datagen.queries(w, "cuda")
    dbc = uq.encode(db, w.x)
    q8 = uq.quantize_i8(q)
    s, i = uq.search_asym(q8, dbc, w.d, w.k)
    db_h = db.cpu().numpy()
    del db
    o_db = orc.pack(orc.encode(db_h, w.x))
    o_q8 = orc.quantize_i8(q.cpu().numpy())
    assert np.array_equal(q8.cpu().numpy(), o_q8)
    rng = np.random.default_rng(4)
    qs = np.sort(rng.choice(w.nq, size=6, replace=False))
    s_ref, i_ref = orc.knn_asym(o_q8[qs], o_db, w.d, w.k)
    assert np.array_equal(s.cpu().numpy()[qs], s_ref)
    assert np.array_equal(i.cpu().numpy()[qs], i_ref)


@pytest.mark.parametrize("opt,k", [("0", 100), ("0.01", 500)])
def test_search_asym_seed_fallback(uq, orc, monkeypatch, opt, k):
    """Single-operand search with exact (0) and forced-failing (0.01) seeds."""
    monkeypatch.setenv("UQ_SEED_OPT", opt)
    _asym_case(uq, orc, 256, 128, 131072, 300, k, seed=21 + k)


@pytest.mark.parametrize("algo", ALGOS)
def test_one_bit_baseline_is_x_equals_d(uq, orc, algo):
    """1-bit quantisation (sign bits, Hamming distance) is the {d,d} EVP.
    With x = d the search ranks rows by d - 2 * Hamming(sign bits) -- checked here
    against a numpy popcount of the sign planes, independent of the oracle's kNN
    (zero coordinates are avoided so every code has x = d non-zeros)."""
    rng = np.random.default_rng(31)
    d, n, nq, k = 256, 20000, 140, 20
    u = rng.standard_normal((n + nq, d)).astype(np.float32)
    u[u == 0] = 1e-3
    codes = uq.encode(torch.from_numpy(u).cuda(), d)
    db, q = codes[:n], codes[n:]
    if algo in ("tc", "f4") and not _tc_supported(uq, nq, n, d, k, _algo(uq, algo)):
        pytest.skip("shape unsupported")
    s, i = uq.search(q, db, d, k, algo=_algo(uq, algo))
    sign = (u > 0)
    ham = (sign[n:, None, :] != sign[None, :n, :]).sum(-1)          # [nq][n]
    delta = d - 2 * ham
    for r in range(nq):
        order = np.lexsort((np.arange(n), -delta[r]))[:k]
        assert np.array_equal(i[r].cpu().numpy(), order)
        assert np.array_equal(s[r].cpu().numpy(), delta[r][order])


@pytest.mark.parametrize("d,x", [(1024, 512), (1000, 500)])
def test_search_asym_parity_wide_seeded(uq, orc, d, x):
    """Widest int8-query tiles (128 x 1024 B resident) with the seeding histogram
    in shared memory beside them: n >= 2^16 turns the seeding scan on."""
    _asym_case(uq, orc, d, x, 70001, 140, 10, seed=d + 1, mode="dup")


def test_merge_topk_ptrs_parity(uq, orc):
    """uq_merge_topk_ptrs (the peer-memory exchange's merge) over G separately
    allocated lists equals uq_merge_topk over the same lists stacked, and a
    Python brute force."""
    rng = np.random.default_rng(18)
    g, nq, k = 6, 41, 23
    lists_s, lists_i = [], []
    for r in range(g):
        sc = rng.integers(-30, 31, size=(nq, k)).astype(np.int32)
        ids = np.stack([rng.permutation(1000)[:k] + 1000 * r for _ in range(nq)]).astype(np.int64)
        if r == 2:
            ids[:, 15:] = -1
            sc[:, 15:] = np.iinfo(np.int32).min
        lists_s.append(torch.from_numpy(sc).cuda())
        lists_i.append(torch.from_numpy(ids).cuda())
    sp = torch.tensor([t.data_ptr() for t in lists_s], dtype=torch.int64, device="cuda")
    ip = torch.tensor([t.data_ptr() for t in lists_i], dtype=torch.int64, device="cuda")
    s, i = uq.merge_topk_ptrs(sp, ip, nq, k)
    s2, i2 = uq.merge_topk(torch.stack(lists_s), torch.stack(lists_i), k)
    assert torch.equal(s, s2) and torch.equal(i, i2)
    S = np.stack([t.cpu().numpy() for t in lists_s])
    I = np.stack([t.cpu().numpy() for t in lists_i])
    for q in range(nq):
        cand = sorted([(int(S[r, q, j]), int(I[r, q, j])) for r in range(g) for j in range(k) if I[r, q, j] >= 0],
                      key=lambda t: (-t[0], t[1]))[:k]
        assert s[q].cpu().tolist() == [c[0] for c in cand] and i[q].cpu().tolist() == [c[1] for c in cand]


def test_peer_exchange_world1(uq):
    """The symmetric-memory exchange path end to end on a one-rank group (the
    only topology a one-GPU test box has): rendezvous, barrier, merge over the
    mapped buffer equals the local lists."""
    import os
    import torch.distributed as dist
    from paper_2506_00528_b200.parallel import PeerExchange
    owned = not dist.is_initialized()
    if owned:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    rng = np.random.default_rng(5)
    nq, k = 17, 9
    s = torch.from_numpy(rng.integers(-9, 9, size=(nq, k)).astype(np.int32)).cuda()
    i = torch.from_numpy(np.stack([rng.permutation(100)[:k] for _ in range(nq)]).astype(np.int64)).cuda()
    try:
        ex = PeerExchange(nq, k, torch.device("cuda:0"))
    except Exception as e:   # symmetric memory unavailable in this build: nothing to exercise
        pytest.skip(f"symmetric memory unavailable: {e}")
    try:
        ms, mi = ex.merge(s, i)
        ref_s, ref_i = uq.merge_topk(s[None], i[None], k)
        assert torch.equal(ms, ref_s) and torch.equal(mi, ref_i)
    finally:
        if owned:
            torch.cuda.synchronize()
            dist.destroy_process_group()


@pytest.mark.parametrize("d,x,n,nq,k,mode", [(384, 192, 5000, 130, 10, "normal"), (768, 384, 20001, 300, 100, "dup"),
                                             (1024, 512, 131072, 260, 10, "normal"), (1536, 768, 70001, 140, 100, "dup"),
                                             (129, 40, 241, 3, 7, "ties"), (128, 64, 100000, 600, 1, "ties")])
def test_search_f4_index_parity(uq, orc, d, x, n, nq, k, mode):
    """E2M1 pair engine fed by the pre-expanded index (bulk-copy stages) equals
    the oracle, including seeded scans (n >= 2^16) and ragged tails."""
    rng = np.random.default_rng(d + n)
    if mode == "dup":
        base = rng.standard_normal((max(1, n // 7), d)).astype(np.float32)
        u_db = base[rng.integers(0, base.shape[0], size=n)]
    elif mode == "ties":
        u_db = _tie_heavy(rng, n, d)
    else:
        u_db = rng.standard_normal((n, d)).astype(np.float32)
    u_q = rng.standard_normal((nq, d)).astype(np.float32)
    o_db = orc.pack(orc.encode(u_db, x))
    o_q = orc.pack(orc.encode(u_q, x))
    dbc = torch.from_numpy(o_db).cuda()
    idx = uq.build_f4_index(dbc, d)
    s, i = uq.search(torch.from_numpy(o_q).cuda(), dbc, d, k, id_base=3, f4_index=idx)
    s_ref, i_ref = orc.knn(o_q, o_db, d, k, id_base=3)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)


@pytest.mark.parametrize("opt,k", [("0.01", 500), ("0", 100)])
def test_search_f4_index_seed_fallback(uq, orc, monkeypatch, opt, k):
    """Index-fed E2M1 engine with forced seed fallbacks (and exact seeds)."""
    monkeypatch.setenv("UQ_SEED_OPT", opt)
    rng = np.random.default_rng(40 + k)
    d, x, n, nq = 256, 128, 131072, 300
    u_db = rng.standard_normal((n, d)).astype(np.float32)
    u_q = rng.standard_normal((nq, d)).astype(np.float32)
    o_db, o_q = orc.pack(orc.encode(u_db, x)), orc.pack(orc.encode(u_q, x))
    dbc = torch.from_numpy(o_db).cuda()
    s, i = uq.search(torch.from_numpy(o_q).cuda(), dbc, d, k, f4_index=uq.build_f4_index(dbc, d))
    s_ref, i_ref = orc.knn(o_q, o_db, d, k)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)


@pytest.mark.parametrize("d,x,n,nq,k,mode", [(384, 192, 5000, 130, 10, "normal"), (768, 384, 20001, 300, 100, "dup"),
                                             (1024, 512, 131072, 260, 10, "normal"), (129, 40, 241, 3, 7, "ties")])
def test_search_asym_i8_index_parity(uq, orc, d, x, n, nq, k, mode):
    """Single-operand search fed by the int8 index (bulk-copy stages) equals the
    oracle's masked-addition kNN."""
    rng = np.random.default_rng(d + n + 1)
    if mode == "dup":
        base = rng.standard_normal((max(1, n // 7), d)).astype(np.float32)
        u_db = base[rng.integers(0, base.shape[0], size=n)]
    elif mode == "ties":
        u_db = _tie_heavy(rng, n, d)
    else:
        u_db = rng.standard_normal((n, d)).astype(np.float32)
    u_q = rng.standard_normal((nq, d)).astype(np.float32)
    o_db = orc.pack(orc.encode(u_db, x))
    q8 = orc.quantize_i8(u_q)
    dbc = torch.from_numpy(o_db).cuda()
    s, i = uq.search_asym(torch.from_numpy(q8).cuda(), dbc, d, k, id_base=2, i8_index=uq.build_i8_index(dbc, d))
    s_ref, i_ref = orc.knn_asym(q8, o_db, d, k, id_base=2)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)


@pytest.mark.parametrize("engine", ["f4x", "asym_x"])
@pytest.mark.parametrize("k", [2, 5, 8])
def test_index_seed_samples_spread_rows(uq, orc, engine, k):
    """Index-fed seeding scans (E2M1 / int8 index) must sample the same rows as
    the producer path: whole row blocks spread over the WHOLE database, each
    once (the bulk-copy path once sampled only the first rows, some
    several times).  k <= 8 gives exact seeds (need = k, no verification), so a
    row counted twice raises the bound above what the database supports and the
    search returns fewer than k rows.  Each of the first 16 queries gets k - 1
    planted copies (Delta = nnz, the maximum) at the start of sample block 1
    (row 3840 = 240 rows x stride 16; with the wrong mapping two chunks' items
    both read it); the remaining best rows are ordinary."""
    rng = np.random.default_rng(100 + k)
    d, x, n, nq = 128, 64, 1 << 20, 300
    u_db = rng.standard_normal((n, d)).astype(np.float32)
    u_q = rng.standard_normal((nq, d)).astype(np.float32)
    for j in range(16):
        for m in range(k - 1):
            u_db[3840 + j * (k - 1) + m] = u_q[j] * (1.0 + 0.001 * m)   # same code as the query
    for blk in (1, 2, 7):   # further planted copies at other block starts (2x-read rows under the old mapping)
        for m in range(k - 1):
            u_db[blk * 4096 + 7680 + m] = u_q[16] * (1.0 + 0.001 * m)
    o_db = orc.pack(orc.encode(u_db, x))
    dbc = torch.from_numpy(o_db).cuda()
    if engine == "f4x":
        o_q = orc.pack(orc.encode(u_q, x))
        s, i = uq.search(torch.from_numpy(o_q).cuda(), dbc, d, k, f4_index=uq.build_f4_index(dbc, d))
        s2, i2 = uq.search(torch.from_numpy(o_q).cuda(), dbc, d, k, algo=uq.ALGO_TC_FP4)
        s_ref, i_ref = orc.knn(o_q, o_db, d, k)
    else:
        q8 = orc.quantize_i8(u_q)
        s, i = uq.search_asym(torch.from_numpy(q8).cuda(), dbc, d, k, i8_index=uq.build_i8_index(dbc, d))
        s2, i2 = uq.search_asym(torch.from_numpy(q8).cuda(), dbc, d, k)
        s_ref, i_ref = orc.knn_asym(q8, o_db, d, k)
    assert (i.cpu().numpy() >= 0).all(), "padding returned: the seed bound was above the k-th best row"
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)
    assert torch.equal(s, s2) and torch.equal(i, i2)   # index-fed == producer-fed


@pytest.mark.parametrize("algo,nq,k", [("popc", 1, 100), ("popc", 3, 10), ("auto", 2, 1000), ("f4", 300, 10)])
def test_search_id_base_above_2_32(uq, orc, algo, nq, k):
    """ids = id_base + row for id_base + n > 2^32 (the two-level
    merge used for few queries once repacked id_base + row into 32 bits)."""
    rng = np.random.default_rng(7 + nq)
    d, x, n = 256, 128, 70001
    base = (1 << 33) + 12345
    o_db = orc.pack(orc.encode(rng.standard_normal((n, d)).astype(np.float32), x))
    o_q = orc.pack(orc.encode(rng.standard_normal((nq, d)).astype(np.float32), x))
    s, i = uq.search(torch.from_numpy(o_q).cuda(), torch.from_numpy(o_db).cuda(), d, k, id_base=base,
                     algo=_algo(uq, algo))
    s_ref, i_ref = orc.knn(o_q, o_db, d, k, id_base=base)
    assert np.array_equal(s.cpu().numpy(), s_ref) and np.array_equal(i.cpu().numpy(), i_ref)
