"""Pins for the CPU oracle (runs without a GPU).

Every oracle function is checked against something other than itself: values
the paper prints (Table 3, Fig. 2), brute-force enumeration of the vertex set,
closed forms, exact invariances, and independent numpy routes.  Citations:
P:NNN = PAPER.md line, R# = DESIGN.md reading.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _bits_to_bytes(bits, nbytes):
    out = np.zeros(nbytes, dtype=np.uint8)
    for i, b in enumerate(bits):
        if b:
            out[i // 8] |= 1 << (i % 8)
    return out


# --------------------------------------------------------------------------
# Table 3
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dt", [np.float64, np.float32, np.float16])
def test_table3_encode(orc, dt):
    t = _load("table3_p356.json")
    u = np.array([t["u1"], t["u2"]], dtype=dt)
    v = orc.encode(u, t["x"])
    assert v[0].tolist() == t["v1"]                       # printed v1
    rule_v2 = list(t["v2_printed"])
    rule_v2[8] = 1                                        # R13: u2[8] = +0.4 -> +1
    assert v[1].tolist() == rule_v2
    # with u2[8] negated, the rule reproduces the printed v2 exactly
    u2m = np.array(t["u2"], dtype=dt)
    u2m[8] = -u2m[8]
    assert orc.encode(u2m, t["x"])[0].tolist() == t["v2_printed"]


def test_table3_planes(orc):
    t = _load("table3_p356.json")
    pb = orc.plane_bytes(10)
    assert pb == 16                                       # R6: 128-bit plane granularity
    c1 = orc.pack(np.array(t["v1"], dtype=np.int8))[0]
    assert (c1[:pb] == _bits_to_bytes(t["v1_pos_bits"], pb)).all()
    assert (c1[pb:] == _bits_to_bytes(t["v1_neg_bits"], pb)).all()
    c2 = orc.pack(np.array(t["v2_printed"], dtype=np.int8))[0]
    assert (c2[:pb] == _bits_to_bytes(t["v2_pos_bits"], pb)).all()
    assert (c2[pb:] == _bits_to_bytes(t["v2_neg_bits"], pb)).all()
    assert c1[0] == 0x63 and c1[pb] == 0x04 and c2[0] == 0x0C and c2[pb] == 0x42 and c2[pb + 1] == 0x01


def test_table3_delta(orc):
    """Delta(v1,v2) from the printed rows (hand count: positions 1,2,6 give -1 each)."""
    t = _load("table3_p356.json")
    v1 = np.array(t["v1"], dtype=np.int8)
    for v2 in (t["v2_printed"], [0, -1, 1, 1, 0, 0, -1, 0, 1, 0]):
        v2 = np.array(v2, dtype=np.int8)
        assert orc.dot_naive(v1, v2) == -3
        assert orc.b2sp(orc.pack(v1)[0], orc.pack(v2)[0], 10) == -3
    # bsp(v1+, v2-) = 2: positions 1 and 6 (read off P:369 and P:372)
    assert orc.b2sp(orc.pack(v1)[0], orc.pack(v1)[0], 10) == 5     # self product = x


def test_table3_tie_pins(orc):
    """u2 has exact ties |u2[1]|=|u2[8]|=0.4 and |u2[2]|=|u2[6]|=0.38:
    sorted |u2| (desc) = 0.45@3, 0.4@1, 0.4@8, 0.38@2, 0.38@6, 0.35@9, 0.19@5, ...
    so lowest-index tie-breaking (R1) picks 1 over 8 at x=2 and 2 over 6 at x=4."""
    t = _load("table3_p356.json")
    for dt in (np.float64, np.float32, np.float16):
        u2 = np.array(t["u2"], dtype=dt)
        assert orc.encode(u2, 2)[0].tolist() == [0, -1, 0, 1, 0, 0, 0, 0, 0, 0]
        assert orc.encode(u2, 4)[0].tolist() == [0, -1, 1, 1, 0, 0, 0, 0, 1, 0]
        assert orc.encode(u2, 3)[0].tolist() == [0, -1, 0, 1, 0, 0, 0, 0, 1, 0]
        assert orc.encode(u2, 10)[0].tolist() == [int(np.sign(a)) for a in t["u2"]]


# --------------------------------------------------------------------------
# Fig. 2 and vertex count
# --------------------------------------------------------------------------
def test_fig2_vertices_and_count():
    f = _load("fig2_p159.json")
    assert sorted(bf.evp_vertices(2, 3)) == sorted(tuple(v) for v in f["vertices"])
    for d in range(1, 7):
        for x in range(1, d + 1):
            assert len(bf.evp_vertices(x, d)) == math.comb(d, x) * 2 ** x


# --------------------------------------------------------------------------
# Encoder vs brute force (the nearest vertex maximises the scalar product)
# --------------------------------------------------------------------------
def _tie_heavy(rng, d):
    # small integer grid -> many exact |u| ties, occasional zeros and -0.0
    u = rng.integers(-4, 5, size=d).astype(np.float64) / 4.0
    if rng.random() < 0.3:
        u[rng.integers(0, d)] = -0.0
    return u


def test_encode_bruteforce_optimal_and_lowest_index(orc):
    rng = np.random.default_rng(11)
    n_checked = 0
    for trial in range(160):
        d = int(rng.integers(1, 8))
        x = int(rng.integers(1, d + 1))
        u = _tie_heavy(rng, d) if trial % 2 else rng.standard_normal(d)
        v = orc.encode(u, x)[0]
        best, _ = bf.best_vertices(u, x)
        assert bf.exact_dot(u, v) == best, (u, x, v)
        sel = np.flatnonzero(v)
        # if x non-zero magnitudes exist, the code is a vertex (exactly x non-zeros)
        if np.count_nonzero(u) >= x:
            assert len(sel) == x
            # lowest-index rule: the support is the lexicographically first maximiser
            assert tuple(sel) == bf.first_max_support(u, x), (u, x)
        n_checked += 1
    assert n_checked == 160


def test_spec_style_examples(orc):
    # derivable by hand from P:192-196
    assert orc.encode(np.array([1.0, 0.0, 0.0]), 1)[0].tolist() == [1, 0, 0]
    assert orc.encode(np.array([0.1, -0.2, 0.3]), 2)[0].tolist() == [0, -1, 1]
    # a selected exact zero maps to 0 (R2); -0.0 has sign 0 (R3)
    assert orc.encode(np.array([0.5, -0.0, 0.0]), 3)[0].tolist() == [1, 0, 0]


def test_encode_closed_form_x_equals_d(orc):
    """x = d: the code is the sign vector (1-bit quantisation = {d,d} EVP)."""
    rng = np.random.default_rng(3)
    u = rng.standard_normal((50, 37)).astype(np.float32)
    v = orc.encode(u, 37)
    assert (v == np.sign(u).astype(np.int8)).all()


def test_encode_invariances(orc):
    rng = np.random.default_rng(5)
    u = rng.standard_normal((200, 96)).astype(np.float32)
    for x in (1, 17, 48, 95):
        v = orc.encode(u, x)
        assert (orc.encode(u * np.float32(8.0), x) == v).all()        # exact 2^k scaling
        assert (orc.encode(u * np.float32(0.125), x) == v).all()
        assert (orc.encode(-u, x) == -v).all()                         # sign symmetry
        perm = rng.permutation(96)
        assert (orc.encode(u[:, perm], x) == v[:, perm]).all()         # tie-free permutation
        assert (np.count_nonzero(v, axis=1) == x).all()                # exactly x non-zeros


# --------------------------------------------------------------------------
# Pack / unpack / code validity
# --------------------------------------------------------------------------
def _rand_ternary(rng, n, d, x=None):
    v = np.zeros((n, d), dtype=np.int8)
    for r in range(n):
        m = x if x is not None else int(rng.integers(0, d + 1))
        idx = rng.choice(d, size=m, replace=False)
        v[r, idx] = rng.choice([-1, 1], size=m)
    return v


@pytest.mark.parametrize("d", [1, 10, 100, 128, 129, 384, 1000])
def test_pack_roundtrip_and_layout(orc, d):
    rng = np.random.default_rng(d)
    v = _rand_ternary(rng, 40, d)
    c = orc.pack(v)
    pb = orc.plane_bytes(d)
    assert c.shape == (40, 2 * pb) and pb == 16 * math.ceil(d / 128)
    assert (orc.unpack(c, d) == v).all()
    # independent numpy route to the same bytes: bit i at byte i//8, bit i%8 (LSB first)
    padded = np.zeros((40, pb * 8), dtype=np.uint8)
    padded[:, :d] = (v == 1)
    assert (np.packbits(padded, axis=1, bitorder="little") == c[:, :pb]).all()
    padded[:, :d] = (v == -1)
    assert (np.packbits(padded, axis=1, bitorder="little") == c[:, pb:]).all()
    assert orc.check_codes(c, d) == 0


def test_check_codes_flags_corruption(orc):
    rng = np.random.default_rng(1)
    d = 100
    c = orc.pack(_rand_ternary(rng, 10, d))
    pb = orc.plane_bytes(d)
    c[3, 0] |= 1
    c[3, pb] |= 1            # position 0 in both planes
    c[7, pb + 13] |= 0x80    # neg-plane bit 111 >= d: a pad bit
    assert orc.check_codes(c, d) == 2


# --------------------------------------------------------------------------
# Delta: naive sum == literal 4-popcount b2sp == numpy
# --------------------------------------------------------------------------
@pytest.mark.parametrize("d", [10, 100, 384, 1000])
def test_delta_three_routes(orc, d):
    rng = np.random.default_rng(100 + d)
    a = _rand_ternary(rng, 48, d)
    b = _rand_ternary(rng, 64, d)
    ca, cb = orc.pack(a), orc.pack(b)
    s = orc.scores(ca, cb, d)
    ref = a.astype(np.int64) @ b.astype(np.int64).T        # exact integer matmul
    assert (s == ref).all()
    for i in range(0, 48, 7):
        for j in range(0, 64, 11):
            assert orc.dot_naive(a[i], b[j]) == s[i, j]
    # symmetry and |Delta| <= min(nnz)
    assert (orc.scores(cb, ca, d) == s.T).all()
    nz_a, nz_b = np.count_nonzero(a, 1), np.count_nonzero(b, 1)
    assert (np.abs(s) <= np.minimum(nz_a[:, None], nz_b[None, :])).all()


def test_delta_closed_forms(orc):
    rng = np.random.default_rng(9)
    d = 300
    v = _rand_ternary(rng, 20, d)
    c, cn = orc.pack(v), orc.pack(-v)
    nnz = np.count_nonzero(v, 1)
    s = orc.scores(c, c, d)
    assert (np.diag(s) == nnz).all()                        # Delta(v,v) = nnz
    assert (np.diag(orc.scores(c, cn, d)) == -nnz).all()    # Delta(v,-v) = -nnz
    # disjoint supports -> 0
    a = np.zeros((1, d), np.int8); a[0, :100] = 1
    b = np.zeros((1, d), np.int8); b[0, 100:] = -1
    assert orc.scores(orc.pack(a), orc.pack(b), d)[0, 0] == 0
    # x = d on zero-free inputs: Delta = d - 2 * Hamming(sign bits)
    u = rng.standard_normal((30, d))
    e = orc.encode(u, d)
    ham = (np.signbit(u)[:, None, :] != np.signbit(u)[None, :, :]).sum(-1)
    assert (orc.scores(orc.pack(e), orc.pack(e), d) == d - 2 * ham).all()


# --------------------------------------------------------------------------
# kNN: brute force over all rows, order (Delta desc, id asc)
# --------------------------------------------------------------------------
def _np_knn(s, k, id_base=0):
    nq, n = s.shape
    ids = np.arange(n)
    out_s = np.full((nq, k), np.iinfo(np.int32).min, dtype=np.int32)
    out_i = np.full((nq, k), -1, dtype=np.int64)
    for q in range(nq):
        order = np.lexsort((ids, -s[q].astype(np.int64)))[:k]
        out_s[q, :len(order)] = s[q, order]
        out_i[q, :len(order)] = order + id_base
    return out_s, out_i


@pytest.mark.parametrize("n,k", [(0, 5), (3, 5), (257, 10), (1000, 100), (64, 64)])
def test_knn_matches_bruteforce(orc, n, k):
    rng = np.random.default_rng(n + k)
    d, x = 200, 100
    u = rng.standard_normal((n + 30, d))
    codes = orc.pack(orc.encode(u, x))
    db, q = codes[:n], codes[n:]
    s, ids = orc.knn(q, db, d, k, id_base=77)
    ref_s, ref_i = _np_knn(orc.scores(q, db, d), k, id_base=77)
    ref_i[ref_i < 77] = -1
    assert (s == ref_s).all() and (ids == ref_i).all()


def test_knn_self_match_and_duplicates(orc):
    rng = np.random.default_rng(2)
    d, x = 128, 64
    codes = orc.pack(orc.encode(rng.standard_normal((50, d)), x))
    db = np.concatenate([codes, codes[10:11], codes[10:11]])   # rows 50, 51 duplicate row 10
    s, ids = orc.knn(codes[10:11], db, d, 3)
    assert s[0].tolist() == [x, x, x] and ids[0].tolist() == [10, 50, 51]
    # k = N: a full permutation
    s, ids = orc.knn(codes[:4], codes, d, 50)
    for q in range(4):
        assert sorted(ids[q].tolist()) == list(range(50))


def test_cosine_knn(orc):
    """fp64 cosine GT; on unit vectors l2^2 = 2 - 2 cos gives the same ranking."""
    rng = np.random.default_rng(4)
    db = rng.standard_normal((500, 64))
    q = rng.standard_normal((8, 64))
    s, ids = orc.cosine_knn(q, db, 10)
    qn = q / np.linalg.norm(q, axis=1, keepdims=True)
    dn = db / np.linalg.norm(db, axis=1, keepdims=True)
    l2 = ((qn[:, None, :] - dn[None, :, :]) ** 2).sum(-1)
    ref = np.argsort(l2, axis=1, kind="stable")[:, :10]
    assert (ids == ref).all()
    assert np.allclose(2 - 2 * s, np.take_along_axis(l2, ref, 1), atol=1e-12)
    s1, i1 = orc.cosine_knn(db[5:6] * 3.0, db, 1)
    assert i1[0, 0] == 5 and abs(s1[0, 0] - 1.0) < 1e-12


def test_rerank(orc):
    """k@n re-rank: with every row as a candidate it is exact cosine kNN
    (P:67-69 ranking pinned above); the candidate order does not matter; a
    candidate subset keeps the best k of that subset; invalid ids are skipped."""
    rng = np.random.default_rng(9)
    db = rng.standard_normal((300, 48))
    q = rng.standard_normal((6, 48))
    s0, i0 = orc.cosine_knn(q, db, 12)
    cand = np.stack([rng.permutation(300) for _ in range(6)])
    s1, i1 = orc.rerank(q, db, cand, 12)
    assert np.array_equal(i0, i1) and np.array_equal(s0, s1)
    # subset: brute force over the subset by explicit unit-vector dot products
    sub = cand[:, :40]
    s2, i2 = orc.rerank(q, db, sub, 5)
    for r in range(6):
        qn = q[r] / np.linalg.norm(q[r])
        sc = [(-float(qn @ (db[j] / np.linalg.norm(db[j]))), int(j)) for j in sub[r]]
        best = sorted(sc)[:5]
        assert [b[1] for b in best] == i2[r].tolist()
        assert np.allclose([-b[0] for b in best], s2[r], atol=1e-12)
    # padding / out-of-range ids are skipped; too few candidates pad with (-inf, -1)
    bad = np.array([[-1, 7, 300, 3]] * 6, dtype=np.int64)
    s3, i3 = orc.rerank(q, db, bad, 4)
    assert (i3[:, 2:] == -1).all() and np.isinf(s3[:, 2:]).all()
    assert all(set(i3[r, :2].tolist()) == {3, 7} for r in range(6))


def test_quantize_i8_closed_forms(orc):
    """R15 (P:507-509 names no scheme): per-vector scale 127/max|u| in fp32, round
    half to even.  Closed forms, the half-way ties, and exact invariances."""
    e = np.zeros((1, 9), np.float32)
    e[0, 4] = 3.7
    q = orc.quantize_i8(e)
    assert q[0, 4] == 127 and np.count_nonzero(q) == 1
    # 127 * 0.5 = 63.5 -> 64 (even), 127 * 0.25 = 31.75 -> 32, -63.5 -> -64
    q = orc.quantize_i8(np.array([[1.0, -1.0, 0.5, 0.25, -0.5, 0.0]], np.float32))
    assert q.tolist() == [[127, -127, 64, 32, -64, 0]]
    # 127/3 * 1.5 = 63.5 exactly?  not in fp32 -- check against an explicit fp32 recomputation
    rng = np.random.default_rng(3)
    u = rng.standard_normal((50, 37)).astype(np.float32)
    q = orc.quantize_i8(u)
    m = np.abs(u).max(axis=1, keepdims=True)
    scale = (np.float32(127.0) / m).astype(np.float32)
    ref = np.clip(np.rint((u * scale).astype(np.float32)), -127, 127).astype(np.int8)
    assert np.array_equal(q, ref)
    assert np.array_equal(orc.quantize_i8(-u), -q)                  # symmetric rounding
    assert np.array_equal(orc.quantize_i8(u * np.float32(8.0)), q)  # 2^k scaling is exact
    assert np.array_equal(orc.quantize_i8(np.zeros((2, 5), np.float32)), np.zeros((2, 5), np.int8))
    assert (np.abs(q).max(axis=1) == 127).all()


def test_knn_asym_masked_addition(orc):
    """Single-operand search by masked addition: (1) with a
    ternary query as the int8 operand it equals the paper's b2sp kNN exactly
    (Table 3 pins b2sp); (2) its scores equal an exact integer matmul with the
    unpacked codes; (3) its ranking equals a lexsort brute force."""
    rng = np.random.default_rng(12)
    d, n, nq, k = 200, 400, 7, 25
    u = rng.standard_normal((n + nq, d)).astype(np.float32)
    codes = orc.pack(orc.encode(u[:n], 67))
    qv = orc.encode(u[n:], 67)
    s_sym, i_sym = orc.knn(orc.pack(qv), codes, d, k, id_base=3)
    s_asym, i_asym = orc.knn_asym(qv.astype(np.int8), codes, d, k, id_base=3)
    assert np.array_equal(s_sym, s_asym) and np.array_equal(i_sym, i_asym)
    q8 = orc.quantize_i8(u[n:])
    s, ids = orc.knn_asym(q8, codes, d, n)
    full = q8.astype(np.int64) @ orc.unpack(codes, d).astype(np.int64).T
    for r in range(nq):
        order = np.lexsort((np.arange(n), -full[r]))
        assert np.array_equal(ids[r], order) and np.array_equal(s[r], full[r][order])
    s2, i2 = orc.knn_asym(q8, codes[:5], d, 8)   # n < k: padding
    assert (i2[:, 5:] == -1).all() and (s2[:, 5:] == np.iinfo(np.int32).min).all()


@pytest.mark.parametrize("threads", [1, 4])
def test_knn_row_parallel_path(orc, threads):
    """Few queries (nq < threads) take the row-parallel loop of orc_knn /
    orc_knn_asym (used by the full-size sampled checks); it must equal the
    lexsort brute force and the one-query-per-thread path exactly."""
    prev = orc.set_threads(threads)
    try:
        rng = np.random.default_rng(31)
        d, x, n, k = 160, 80, 5000, 20
        u = rng.standard_normal((n + 40, d))
        u[100:110] = u[4000]                        # ties broken by id
        codes = orc.pack(orc.encode(u, x))
        db, q = codes[:n], codes[n:]
        for nq in (1, 3):
            s, ids = orc.knn(q[:nq], db, d, k, id_base=9)
            ref_s, ref_i = _np_knn(orc.scores(q[:nq], db, d), k, id_base=9)
            assert (s == ref_s).all() and (ids == ref_i).all()
        s_all, i_all = orc.knn(q, db, d, k, id_base=9)   # 40 >= threads: query-parallel path
        s3, i3 = orc.knn(q[:3], db, d, k, id_base=9)
        assert (s_all[:3] == s3).all() and (i_all[:3] == i3).all()
        q8 = orc.quantize_i8(u[n:n + 2].astype(np.float32))
        sa, ia = orc.knn_asym(q8, db, d, k)
        full = q8.astype(np.int64) @ orc.unpack(db, d).astype(np.int64).T
        for r in range(2):
            order = np.lexsort((np.arange(n), -full[r]))[:k]
            assert np.array_equal(ia[r], order) and np.array_equal(sa[r], full[r][order])
    finally:
        orc.set_threads(prev)
