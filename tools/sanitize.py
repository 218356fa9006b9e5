"""Small (c1-sized) run of every kernel of libuq.so against the CHECKED build
(libuq_checked.so: device-side bounds asserts, UQ_ASSERT in csrc/common.cuh),
every result compared with the CPU oracle:

    python tools/sanitize.py            # builds + loads libuq_checked.so

compute-sanitizer is closed on this GPU pool (runs under it have left GPUs
needing a reset; profiles/r02/compute_sanitizer_closed.txt), so the checked
build's asserts + oracle comparison stand in for its memcheck.  The same
script runs under compute-sanitizer where that is allowed.

Engines: encode (f32 / f16 / bf16), scores, check_codes, the popcount scan (TMA
and LDG variants, seeded), the one-CTA int8 tcgen05 scan, the CTA-pair int8 and
E2M1 scans (2-bit codes and the E2M1 index, seeded), single-operand search (int8
index), merge_topk / merge_topk_ptrs, quantize_i8, rerank.  Every result is
checked against the CPU oracle, so a sanitizer run is also a parity run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("UQ_CHECKED_LIB", "1") == "1":
    os.environ["UQ_CHECKED_LIB"] = "1"
    import importlib.util as _ilu  # noqa: E402
    _spec = _ilu.spec_from_file_location("_uqb", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(
        __file__))), "paper_2506_00528_b200", "build.py"))
    _m = _ilu.module_from_spec(_spec)
    _spec.loader.exec_module(_m)
    _m.build(checked=True)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402


def check(name, got, want):
    g = [t.cpu().numpy() for t in got]
    ok = all(np.array_equal(a, b) for a, b in zip(g, want))
    print(f"{name:28s} {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    dev = torch.device("cuda")
    w = datagen.CONFIGS["c1"].scaled(n=70_001, nq=300)     # n >= 2^16: seeded scans run too
    db = datagen.db(w, dev)
    q = datagen.queries(w, dev)
    d, x, k = w.d, w.x, w.k
    o_db = oracle.pack(oracle.encode(db.cpu().numpy(), x))
    o_q = oracle.pack(oracle.encode(q.cpu().numpy(), x))
    for dt in (torch.float32, torch.float16, torch.bfloat16):
        u = q.to(dt)
        check(f"encode {str(dt)[6:]}", [uq.encode(u, x)], [oracle.pack(oracle.encode(u.float().cpu().numpy(), x))])
    dbc = uq.encode(db, x)
    qc = uq.encode(q, x)
    check("encode db", [dbc], [o_db])
    check("scores", [uq.scores(qc[:7], dbc[:500], d)], [oracle.scores(o_q[:7], o_db[:500], d)])
    assert uq.check_codes(dbc, d) == 0
    print(f"{'check_codes':28s} ok", flush=True)
    ref = {}

    def want(nq):
        if nq not in ref:
            ref[nq] = oracle.knn(o_q[:nq], o_db, d, k)
        return ref[nq]

    cases = [("popc tma q=1", qc[:1], uq.ALGO_POPC, None), ("popc tma q=70", qc[:70], uq.ALGO_POPC, None),
             ("tcgen05 one-CTA q=100", qc[:100], uq.ALGO_TCGEN05, None),
             ("tcgen05 pair int8 q=300", qc, uq.ALGO_TCGEN05, None),
             ("tcgen05 pair e2m1 q=300", qc, uq.ALGO_TC_FP4, None),
             ("tcgen05 pair e2m1 index", qc, uq.ALGO_TC_FP4, "f4x")]
    f4x = uq.build_f4_index(dbc, d)
    for name, qq, algo, idx in cases:
        if only and only not in name:
            continue
        s, i = uq.search(qq, dbc, d, k, algo=algo, f4_index=f4x if idx else None)
        check(name, [s, i], want(qq.shape[0]))
    q8 = uq.quantize_i8(q)
    o_q8 = oracle.quantize_i8(q.cpu().numpy())
    check("quantize_i8", [q8], [o_q8])
    ra = oracle.knn_asym(o_q8, o_db, d, k)
    check("asym", list(uq.search_asym(q8, dbc, d, k)), ra)
    check("asym int8 index", list(uq.search_asym(q8, dbc, d, k, i8_index=uq.build_i8_index(dbc, d))), ra)
    s1, i1 = uq.search(qc[:40], dbc[:35000], d, k, algo=uq.ALGO_POPC)
    s2, i2 = uq.search(qc[:40], dbc[35000:], d, k, id_base=35000, algo=uq.ALGO_POPC)
    check("merge_topk", list(uq.merge_topk(torch.stack([s1, s2]), torch.stack([i1, i2]), k)), want(40))
    sp = torch.tensor([s1.data_ptr(), s2.data_ptr()], dtype=torch.int64, device=dev)
    ip = torch.tensor([i1.data_ptr(), i2.data_ptr()], dtype=torch.int64, device=dev)
    check("merge_topk_ptrs", list(uq.merge_topk_ptrs(sp, ip, 40, k)), want(40))
    cand = torch.from_numpy(np.ascontiguousarray(want(300)[1])).to(dev)
    cos, ids = uq.rerank(q, db, cand, 5)
    o_cos, _ = oracle.rerank(q.double().cpu().numpy(), db.double().cpu().numpy(), want(300)[1], 5)
    assert np.abs(cos.double().cpu().numpy() - o_cos).max() <= 1e-5
    print(f"{'rerank':28s} ok", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE RUN DONE:", uq.lib_path(), flush=True)


if __name__ == "__main__":
    main()
