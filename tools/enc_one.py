"""One uq_encode workload for profiling (ncu): python tools/enc_one.py CFG DTYPE D X N [REPS]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402

cfg, dt, d, x, n = sys.argv[1], getattr(torch, sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
w = datagen.CONFIGS[cfg].scaled(n=n)
u = datagen.rows(w, "db", 0, n, "cuda").to(dt)
out = torch.empty((n, uq.code_bytes(d)), dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(reps):
    e0.record()
    uq.encode(u, x, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    by = n * (d * u.element_size() + uq.code_bytes(d))
    print(f"{cfg} {sys.argv[2]} d={d} x={x} n={n}: {ms:.3f} ms {by / ms / 1e6:.0f} GB/s", flush=True)
