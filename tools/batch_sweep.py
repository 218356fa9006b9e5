"""Batch-size sweep of the scan engines on c2 data (N = 10^6, d = 768, k = 100):
ms per query batch for the popcount engine (TMA-fed for <= 8 queries), the
E2M1 pair engine with its index, and AUTO -- the basis of AUTO's engine choice
(uq.search_resolve).  One JSON line per Q."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402

w = datagen.CONFIGS["c2"]
db = uq.encode(datagen.db(w, "cuda"), w.x)
f4x = uq.build_f4_index(db, w.d)
qall = uq.encode(datagen.rows(w, "q", 0, 4096, "cuda"), w.x)


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for q in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1000, 4096):
    qc = qall[:q]
    row = {"Q": q, "popc_ms": t(lambda: uq.search(qc, db, w.d, w.k, algo=uq.ALGO_POPC)),
           "auto_engine": {1: "popc", 2: "tcgen05", 3: "tcgen05-f4"}[uq.search_resolve(q, w.n, w.d, w.k)]}
    try:
        row["f4_index_ms"] = t(lambda: uq.search(qc, db, w.d, w.k, f4_index=f4x))
    except uq.UQError:
        row["f4_index_ms"] = None
    print(json.dumps(row), flush=True)
