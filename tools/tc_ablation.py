"""Timing ablation of scan_tc_kernel on c2-sized data (results are wrong in
ablated modes; timing only).  Mode via env UQ_TC_ABLATE read at first launch,
so each mode runs in its own process."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["UQ_PROFILE_LIB"] = "1"   # the profile build: ablations compiled in (libuq.so ignores UQ_TC_ABLATE)
import importlib.util as _ilu  # noqa: E402
_spec = _ilu.spec_from_file_location("_uqb", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_00528_b200", "build.py"))
_m = _ilu.module_from_spec(_spec); _spec.loader.exec_module(_m); _m.build(profile=True)  # noqa: E702
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, paper_2506_00528_b200 as uq
    d, x, n, nq, k = 768, 384, int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    db = uq.encode(torch.randn(n, d, device="cuda", generator=g), x)
    q = uq.encode(torch.randn(nq, d, device="cuda", generator=g), x)
    ws = torch.empty(uq.search_workspace(nq, n, d, k, uq.ALGO_TCGEN05), dtype=torch.uint8, device="cuda")
    for _ in range(3): uq.search(q, db, d, k, algo=uq.ALGO_TCGEN05, workspace=ws)
    uq.timing_enable(True)
    for _ in range(10): uq.search(q, db, d, k, algo=uq.ALGO_TCGEN05, workspace=ws)
    ms, cnt = uq.timing_collect()
    print(json.dumps({"mode": os.environ.get("UQ_TC_ABLATE", "0"), "scan_ms": ms / cnt,
                      "tflops": 2 * d * n * nq / (ms / cnt * 1e-3) / 1e12}))
else:
    n, nq, k = (sys.argv[1:4] if len(sys.argv) > 3 else ("1000000", "1000", "100"))
    n, nq, k = str(n), str(nq), str(k)
    for mode in sys.argv[4:] if len(sys.argv) > 4 else ("0", "2", "3", "7"):
        env = dict(os.environ, UQ_TC_ABLATE=mode, UQ_SEED_DIV="0")
        r = subprocess.run([sys.executable, __file__, "child", n, nq, k], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-500:], flush=True)
