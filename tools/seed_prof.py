import os, sys, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["UQ_PROFILE_LIB"] = "1"   # the profile build: ablations compiled in (libuq.so ignores UQ_TC_ABLATE)
import importlib.util as _ilu  # noqa: E402
_spec = _ilu.spec_from_file_location("_uqb", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_00528_b200", "build.py"))
_m = _ilu.module_from_spec(_spec); _spec.loader.exec_module(_m); _m.build(profile=True)  # noqa: E702
import torch, datagen, paper_2506_00528_b200 as uq
w = datagen.CONFIGS['c2']
db = uq.encode(datagen.db(w, 'cuda'), w.x); q = uq.encode(datagen.queries(w, 'cuda'), w.x)
ws = torch.empty(uq.search_workspace(w.nq, w.n, w.d, w.k), dtype=torch.uint8, device='cuda')
for _ in range(3): uq.search(q, db, w.d, w.k, workspace=ws)
uq.timing_enable(True)
for _ in range(10): uq.search(q, db, w.d, w.k, workspace=ws)
t = uq.timing_collect_ex()
L = uq._L; L.uq_debug_tc2_prof.argtypes=[ctypes.c_void_p]; buf=(ctypes.c_ulonglong*48)(); L.uq_debug_tc2_prof(buf)
print(json.dumps({"mode": os.environ.get("UQ_TC_ABLATE"), "seed_ms": t["seed"][0]/max(t["seed"][1],1), "main_ms": t["main"][0]/max(t["main"][1],1),
                  "flush_cycles_per_warp": buf[18]/max(buf[19],1)}))
