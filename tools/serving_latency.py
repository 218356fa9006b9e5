"""Small-batch serving latency on c2 (N = 10^6, d = 768, x = 384, k = 100):
query floats resident on the device -> encode -> search -> top-k on the device,
direct calls (binding + one launch chain per batch) against the same chain
replayed from a CUDA graph (serving.CapturedSearch).  Per Q, two numbers each:
  lat_ms  median over 50 isolated calls (host launch + device, sync after each;
          wall clock, since the host launch work is part of the latency);
  tput_ms back-to-back calls, device time per call (CUDA events over 50).
One JSON line per Q."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402
from paper_2506_00528_b200.serving import CapturedSearch  # noqa: E402

w = datagen.CONFIGS["c2"]
db = uq.encode(datagen.db(w, "cuda"), w.x)
qf = datagen.rows(w, "q", 0, 4096, "cuda")


def lat(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def tput(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for q in (1, 2, 4, 8, 16, 64, 256):
    qb = qf[:q].contiguous()
    ws = torch.empty(uq.search_workspace(q, w.n, w.d, w.k), dtype=torch.uint8, device="cuda")
    qc = torch.empty((q, uq.code_bytes(w.d)), dtype=torch.uint8, device="cuda")
    out = (torch.empty((q, w.k), dtype=torch.int32, device="cuda"),
           torch.empty((q, w.k), dtype=torch.int64, device="cuda"))

    def direct():
        uq.encode(qb, w.x, out=qc)
        uq.search(qc, db, w.d, w.k, workspace=ws, out=out)

    cs = CapturedSearch(db, w.d, w.x, w.k, q)
    graph = lambda: cs(qb)  # noqa: E731
    direct()
    s0, i0 = out[0].clone(), out[1].clone()
    s1, i1 = graph()
    assert torch.equal(s0, s1) and torch.equal(i0, i1)
    row = {"Q": q, "engine": {1: "popc", 2: "tcgen05", 3: "tcgen05-f4"}[uq.search_resolve(q, w.n, w.d, w.k)],
           "direct_lat_ms": round(lat(direct), 4), "graph_lat_ms": round(lat(graph), 4),
           "direct_tput_ms": round(tput(direct), 4), "graph_tput_ms": round(tput(graph), 4)}
    print(json.dumps(row), flush=True)
