"""Quick tcgen05-path sanity check vs the oracle (small shapes); exits non-zero on mismatch."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2506_00528_b200 as uq
rng = np.random.default_rng(0)
ok = True
for (d, x, n, nq, k) in [(128, 64, 256, 128, 10), (384, 192, 3000, 100, 10), (768, 384, 20000, 300, 100),
                         (256, 128, 5000, 129, 10), (768, 384, 70000, 1000, 100)]:
    u = rng.standard_normal((n + nq, d)).astype(np.float32)
    c = oracle.pack(oracle.encode(u, x))
    db, q = c[:n], c[n:]
    t0 = time.time()
    s, i = uq.search(torch.from_numpy(q).cuda(), torch.from_numpy(db).cuda(), d, k, algo=uq.ALGO_TCGEN05)
    torch.cuda.synchronize()
    dt = time.time() - t0
    rs, ri = oracle.knn(q, db, d, k)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    good = np.array_equal(s, rs) and np.array_equal(i, ri)
    ok &= good
    print(d, n, nq, k, "OK" if good else "MISMATCH", f"{dt*1e3:.1f} ms", flush=True)
    if not good:
        bad = np.argwhere((s != rs).any(1))[:3, 0]
        for b in bad:
            print(" q", b, "got", s[b, :8], i[b, :8], "\n   ref", rs[b, :8], ri[b, :8])
        # raw score check via uq_scores
        full = uq.scores(torch.from_numpy(q).cuda(), torch.from_numpy(db).cuda(), d).cpu().numpy()
        print(" scores==oracle:", np.array_equal(full, oracle.scores(q, db, d)))
sys.exit(0 if ok else 1)
