"""One workload's encode + index + search, repeated (profiling driver for ncu):
python tools/search_one.py CFG [N] [NQ] [REPS]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402

cfg = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
nq = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
w = datagen.CONFIGS[cfg].scaled(n=n, nq=nq)
x = w.xs[0]
db = uq.encode(datagen.db(w, "cuda"), x)
q = uq.encode(datagen.queries(w, "cuda"), x)
idx = uq.build_f4_index(db, w.d)
ws = torch.empty(uq.search_workspace(w.nq, w.n, w.d, w.k, uq.ALGO_TC_FP4), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    s, i = uq.search(q, db, w.d, w.k, algo=uq.ALGO_TC_FP4, workspace=ws, f4_index=idx)
torch.cuda.synchronize()
print(cfg, w.n, w.nq, w.k, "ok", int(i[0, 0]))
