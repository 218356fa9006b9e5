"""c2 small-batch search (Q from argv, default 1): encode + search a few times;
run under `ncu --metrics gpu__time_duration.sum` for the per-launch chain."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = datagen.CONFIGS["c2"]
db = uq.encode(datagen.db(w, "cuda"), w.x)
qf = datagen.rows(w, "q", 0, q, "cuda")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measure")
for _ in range(3):
    qc = uq.encode(qf, w.x)
    uq.search(qc, db, w.d, w.k)
torch.cuda.synchronize()
