"""Cycle accounting of the CTA-pair tensor scan (measurement tool): runs
uq_search on the c2 workload with UQ_TC_ABLATE=8 (instrumented, results
unchanged) and prints where each warp role spends its cycles."""
import ctypes
import json
import os
import sys

os.environ["UQ_PROFILE_LIB"] = "1"   # the profile build: ablations compiled in (libuq.so ignores UQ_TC_ABLATE)
import importlib.util as _ilu  # noqa: E402
_spec = _ilu.spec_from_file_location("_uqb", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_00528_b200", "build.py"))
_m = _ilu.module_from_spec(_spec); _spec.loader.exec_module(_m); _m.build(profile=True)  # noqa: E702
os.environ["UQ_TC_ABLATE"] = str(int(os.environ.get("UQ_TC_ABLATE", "0")) | 8)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2506_00528_b200 as uq  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
nq = int(sys.argv[3]) if len(sys.argv) > 3 else None
w = datagen.CONFIGS[cfg].scaled(n=n, nq=nq)
if os.environ.get("UQ_PROF_K"):
    w = w.scaled(k=int(os.environ["UQ_PROF_K"]))
db = uq.encode(datagen.db(w, "cuda"), w.x)
q = uq.encode(datagen.queries(w, "cuda"), w.x)
MODE = os.environ.get("UQ_PROF_ALGO", "f4")   # f4 | tc | asym
ALGO = uq.ALGO_TC_FP4 if MODE == "f4" else uq.ALGO_TCGEN05
if MODE == "asym":
    q8 = uq.quantize_i8(datagen.queries(w, "cuda"))
    ws = torch.empty(uq.search_asym_workspace(w.nq, w.n, w.d, w.k), dtype=torch.uint8, device="cuda")
else:
    ws = torch.empty(uq.search_workspace(w.nq, w.n, w.d, w.k, ALGO), dtype=torch.uint8, device="cuda")


IDX = uq.build_f4_index(db, w.d) if (MODE == "f4" and os.environ.get("UQ_PROF_INDEX") == "1") else None


def run():
    if MODE == "asym":
        return uq.search_asym(q8, db, w.d, w.k, workspace=ws)
    return uq.search(q, db, w.d, w.k, algo=ALGO, workspace=ws, f4_index=IDX)
L = uq._L
L.uq_debug_tc2_prof.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 48)()
for _ in range(2):
    run()
torch.cuda.synchronize()
L.uq_debug_tc2_prof(buf)  # reset
reps = 5
for _ in range(reps):
    run()
torch.cuda.synchronize()
L.uq_debug_tc2_prof(buf)
c = list(buf)
out = {"algo": os.environ.get("UQ_PROF_ALGO", "f4") + ("+index" if IDX is not None else ""), "cfg": cfg, "n": w.n, "nq": w.nq, "k": w.k, "items": c[10],
       "mma_wait_tempty_frac": c[1] / max(c[0], 1), "mma_wait_full_frac": c[2] / max(c[0], 1),
       "prod_wait_empty_frac": c[4] / max(c[3], 1),
       "epi_wait_tfull_frac": c[6] / max(c[5], 1), "epi_filter_frac": c[7] / max(c[5], 1),
       "epi_rebuild_frac": c[8] / max(c[5], 1), "epi_publish_over_loop": c[9] / max(c[5], 1),
       "mma_loop_cycles_per_item": c[0] / max(c[10], 1),
       "cta_setup_cycles": c[11] / max(c[14], 1), "cta_items_cycles": c[12] / max(c[14], 1),
       "cta_teardown_cycles": c[13] / max(c[14], 1),
       "candidates_per_query": c[15] / max(w.nq * reps, 1), "inloop_cuts_per_query": c[16] / max(w.nq * reps, 1),
       "final_cuts_per_query": c[17] / max(w.nq * reps, 1),
       "hist": {"mma_loop_cycles_per_item": c[24] / max(c[34], 1), "mma_wait_tempty_frac": c[25] / max(c[24], 1),
                "mma_wait_full_frac": c[26] / max(c[24], 1), "prod_wait_empty_frac": c[28] / max(c[27], 1),
                "cta_setup_cycles": c[35] / max(c[38], 1), "cta_items_cycles": c[36] / max(c[38], 1),
                "cta_teardown_cycles": c[37] / max(c[38], 1), "items": c[34]},
       "raw": c}
print(json.dumps(out))
