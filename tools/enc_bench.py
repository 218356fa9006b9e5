"""uq_encode throughput on the BASELINE workloads' row shapes (measurement tool).
Prints one JSON line per (dtype, d, x, n): GB/s of algorithmic traffic
(d*sizeof(in) + code_bytes per row) and the fraction of MEASURED_PEAKS hbm_gbs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402

peak = 6534.0
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(p):
    peak = float(json.load(open(p))["hbm_gbs"])

cases = [("c2", torch.float32, 768, 384, 2_000_000), ("c5", torch.float16, 768, 384, 8_000_000),
         ("c3", torch.float32, 1024, 256, 2_000_000), ("c3", torch.float32, 1024, 768, 2_000_000),
         ("c4", torch.float32, 1536, 768, 1_000_000), ("c1", torch.float32, 384, 192, 4_000_000)]
for name, dt, d, x, n in cases:
    w = datagen.CONFIGS[name].scaled(n=n)
    u = datagen.rows(w, "db", 0, n, "cuda").to(dt)
    out = torch.empty((n, uq.code_bytes(d)), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        uq.encode(u, x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        uq.encode(u, x, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    by = n * (d * u.element_size() + uq.code_bytes(d))
    print(json.dumps({"cfg": name, "dtype": str(dt).replace("torch.", ""), "d": d, "x": x, "n": n,
                      "ms": ms, "rows_per_s": n / ms * 1e3, "GB_per_s": by / ms / 1e6,
                      "hbm_frac": by / ms / 1e6 / peak}), flush=True)
    del u, out
    torch.cuda.empty_cache()
