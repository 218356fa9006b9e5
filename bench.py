#!/usr/bin/env python
"""Benchmark of the EVP ternary kNN hot path on B200 (BASELINE.json metric:
query x db Delta-evals/s and kNN QPS; % of roofline).

One step = one pass of the whole hot path over one query batch of the
workload: encode the Q query embeddings (uq_encode), scan all N database codes
with the fused per-query top-k (uq_search: scan kernel + merge kernel), and for
N GPUs the NCCL allgather of the [Q][k] lists + uq_merge_topk.  The database is
encoded once before timing (index build, "pre-processing of S before q
becomes available"); that encode is reported separately under "encode".

Default workload: BASELINE config 2 (d=768, N=1e6, Q=1000, x=384, k=100,
single GPU).  Multi-GPU (torchrun): weak scaling, each rank holds an N-row
shard of the global database (rows [r*N, (r+1)*N) of the same seeded stream).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--algo auto]
    python bench.py --impl reference ...   # the CPU oracle on the same workload
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import datagen  # noqa: E402

METRIC = "query x db Delta-evals/s (kNN over {x,d} EVP ternary codes)"
UNIT = "delta_evals/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


def _traffic(algo: str, workload: str, nq: int):
    """DRAM bytes per main-scan launch from a committed ncu capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t.get(f"{algo}/{workload}/{nq}")
        return (float(e["bytes"]), e["source"]) if e else (None, None)
    except Exception:
        return None, None


def _popc_peak():
    """POPC/clk/SM measured by tools/peaks.cu on a B200 (profiles/peaks_r01.json)."""
    p = os.path.join(ROOT, "profiles", "peaks_r01.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["popc_per_clk_sm_at_attr_clock"]), "measured (tools/peaks.cu)"
    return 16.0, "assumed 16/clk/SM (CUDA Programming Guide cc 7.x-9.0 value)"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)   # before NCCL binds this rank to a device
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return world, rank, local


def _barrier(world):
    if world > 1:
        dist.barrier()


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): the oracle as it stands
# ---------------------------------------------------------------------------
def _oracle_sample(w, target_s: float):
    """Time the oracle's encode(queries) + exhaustive kNN on a bounded sample of
    the workload: n_s database rows (oracle-encoded, untimed) x q_s queries."""
    import oracle
    n_s = min(w.n, 200_000)
    db = datagen.db(w, "cpu", 0, n_s).numpy()
    q_all = datagen.rows(w, "q", 0, min(w.nq, 1000), "cpu").numpy()
    o_db = oracle.pack(oracle.encode(db, w.x))

    def run(nq_s):
        t0 = time.perf_counter()
        o_q = oracle.pack(oracle.encode(q_all[:nq_s], w.x))
        oracle.knn(o_q, o_db, w.d, w.k)
        return time.perf_counter() - t0

    cores = os.cpu_count() or 1
    ncal = min(q_all.shape[0], cores)          # one query per thread: a full-width calibration
    tcal = run(ncal)
    nq_s = int(max(1, min(q_all.shape[0], ncal * target_s / max(tcal, 1e-6))))
    return n_s, nq_s, run, cores


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(w, target_s=10.0):
    """The oracle as it stands, on the host's cores: all threads, then 1 thread
    on a proportionally smaller query sample (BASELINE.md CPU plan)."""
    import oracle
    n_s, nq_s, run, cores = _oracle_sample(w, target_s)
    t = run(nq_s)
    prev = oracle.set_threads(1)
    nq1 = max(1, nq_s // max(cores, 1))
    t1 = run(nq1)
    oracle.set_threads(prev)
    return {"value": nq_s * n_s / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1thread": nq1 * n_s / t1, "cpu_model": _cpu_model(),
            "sample": f"{nq_s} queries (oracle encode + exhaustive kNN, k={w.k}) over the first "
                      f"{n_s} database rows of {w.name}; {t:.1f} s wall on {cores} host threads "
                      f"({nq1} queries, {t1:.1f} s on 1 thread)"}


# The paper's own speed numbers for this path (context only, other hardware):
PAPER_CONTEXT = {
    "b2sp_per_delta": "21.8 ns per Delta (10^6 comparisons in 21.75 ms median), d=384, Apple M3, "
                      "Rust BitVecSimd (P:463-476, Table 4): ~4.6e7 Delta-evals/s on one core",
    "exhaustive_1M": "Table 5 (P:485-496), unstated hardware: d=768 Laion {512,768} b2sp 35.7 ms per "
                     "~1M-row query (likelier reading: ~2.8e7 Delta-evals/s)",
    "note": "no GPU numbers in the paper; BASELINE.md"}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    w = datagen.CONFIGS[args.config]
    n_s, nq_s, run, cores = _oracle_sample(w, target_s=2.0)
    for _ in range(args.warmup):
        run(nq_s)
    times = [run(nq_s) for _ in range(args.steps)]
    tot = sum(times)
    value = args.steps * nq_s * n_s / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": _workload_desc(w), "sample": f"{nq_s} queries x {n_s} rows per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{nq_s} queries x first {n_s} rows of {w.name} per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _workload_desc(w):
    return (f"{w.name}: d={w.d}, N={w.n}, Q={w.nq}, x={w.x}, k={w.k}, {w.kind}"
            f"{' C=' + str(w.centres) if w.centres else ''}, {str(w.dtype).replace('torch.', '')}"
            f"{', l2-normalised' if w.normalise else ', raw'}")


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--algo", default="auto", choices=["auto", "popc", "tc", "f4", "asym"],
                    help="asym: single-operand search (P:507-509), int8 queries x ternary DB")
    ap.add_argument("--n", type=int, default=None, help="override DB rows per GPU")
    ap.add_argument("--nq", type=int, default=None, help="override query batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-f4-index", action="store_true",
                    help="E2M1 pair engine expands the 2-bit codes itself instead of reading the E2M1 index")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N>1: NCCL allgather + merge, or one merge kernel reading every rank's lists "
                         "from symmetric (peer-mapped) memory")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = _dist()
    if args.impl == "reference":
        rc = run_reference(args, world, rank)
        if world > 1:
            dist.destroy_process_group()
        return rc

    import paper_2506_00528_b200 as uq
    from paper_2506_00528_b200.parallel import PeerExchange, allgather_lists

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = datagen.CONFIGS[args.config].scaled(n=args.n, nq=args.nq)
    asym = args.algo == "asym"
    algo = {"auto": uq.ALGO_AUTO, "popc": uq.ALGO_POPC, "tc": uq.ALGO_TCGEN05, "f4": uq.ALGO_TC_FP4,
            "asym": uq.ALGO_TCGEN05}[args.algo]
    n_loc, nq, d, x, k = w.n, w.nq, w.d, w.x, w.k
    id_base = rank * n_loc

    # ---- data (seeded, synthetic; DB shard + replicated queries) ----
    u_db = datagen.rows(w, "db", id_base, n_loc, dev)
    u_q = datagen.queries(w, dev)
    u_q_host = u_q.cpu().pin_memory()
    torch.cuda.synchronize()

    # ---- index build: encode the DB shard once (timed separately) ----
    dbc = torch.empty((n_loc, uq.code_bytes(d)), dtype=torch.uint8, device=dev)
    uq.encode(u_db, x, out=dbc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    uq.encode(u_db, x, out=dbc)
    e1.record()
    torch.cuda.synchronize()
    enc_ms = e0.elapsed_time(e1)
    enc_bytes = n_loc * (d * u_db.element_size() + uq.code_bytes(d))
    del u_db
    torch.cuda.empty_cache()

    qc = torch.empty((nq, uq.code_bytes(d)), dtype=torch.uint8, device=dev)
    out = (torch.empty((nq, k), dtype=torch.int32, device=dev),
           torch.empty((nq, k), dtype=torch.int64, device=dev))
    # E2M1 index (uq_build_f4_index): when the search would run on the E2M1 pair
    # engine, its operand is expanded once at index build (outside the step,
    # like the encode) and every scan stage is one bulk copy
    i8x = uq.build_i8_index(dbc, d) if (asym and not args.no_f4_index and d <= 1024) else None
    f4x = None
    idx_ms = None
    if not args.no_f4_index and not asym and uq.search_resolve(nq, n_loc, d, k, algo) == uq.ALGO_TC_FP4:
        f4x = uq.build_f4_index(dbc, d)            # warm-up build
        ib0, ib1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ib0.record()
        f4x = uq.build_f4_index(dbc, d)
        ib1.record()
        torch.cuda.synchronize()
        idx_ms = ib0.elapsed_time(ib1)
    ws_bytes = uq.search_asym_workspace(nq, n_loc, d, k) if asym else uq.search_workspace(nq, n_loc, d, k, algo)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    q8 = torch.empty((nq, d), dtype=torch.int8, device=dev)
    launches = [0]

    peer = PeerExchange(nq, k, dev) if (world > 1 and args.exchange == "peer") else None

    def step(q_dev, o=None):
        o = out if o is None else o
        if asym:   # quantise the float queries to int8, masked-addition search
            uq.quantize_i8(q_dev, out=q8)
            launches[0] += uq.last_launches()
            s, i = uq.search_asym(q8, dbc, d, k, id_base=id_base, workspace=ws, out=o, i8_index=i8x)
        else:
            uq.encode(q_dev, x, out=qc)
            launches[0] += uq.last_launches()
            s, i = uq.search(qc, dbc, d, k, id_base=id_base, algo=algo, workspace=ws, out=o, f4_index=f4x)
        launches[0] += uq.last_launches()
        if world > 1 and peer is not None:
            s, i = peer.merge(s, i)
        elif world > 1:
            sg, ig = allgather_lists(s, i)
            s, i = uq.merge_topk(sg, ig, k)
            launches[0] += uq.last_launches()
        return s, i

    for _ in range(args.warmup):
        step(u_q)
    torch.cuda.synchronize()

    # ---- device-timed region ----
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches[0] = 0
    uq.timing_enable(True)
    _barrier(world)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    t0.record()
    marks[0].record()
    for st in range(args.steps):
        step(u_q)
        marks[st + 1].record()
    t1.record()
    torch.cuda.synchronize()
    _barrier(world)
    step_ms = sorted(marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps))
    uq.timing_enable(False)
    clk = clocks.stop()
    gpu_launches = launches[0]
    ms = t0.elapsed_time(t1)
    tim = uq.timing_collect_ex()
    main_ms, main_n, main_evals = tim["main"]
    seed_ms, seed_n, seed_evals = tim["seed"]
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # ---- end to end through the public API: pinned host queries in, results out ----
    # Every step copies its query floats host -> device and its (scores, ids)
    # device -> host inside the timed region.  Serving pipeline: the copies run
    # on their own streams, double-buffered, so step s+1's upload and step s's
    # download overlap step s's search (two query / result buffers, event
    # ordered); the region ends when the last results are in host memory.
    host_s = [torch.empty((nq, k), dtype=torch.int32).pin_memory() for _ in range(2)]
    host_i = [torch.empty((nq, k), dtype=torch.int64).pin_memory() for _ in range(2)]
    q_stage = [torch.empty_like(u_q) for _ in range(2)]
    outs = [(torch.empty((nq, k), dtype=torch.int32, device=dev), torch.empty((nq, k), dtype=torch.int64, device=dev))
            for _ in range(2)]
    ks = torch.cuda.current_stream()
    cs_in, cs_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    ev_start = torch.cuda.Event()
    _barrier(world)
    torch.cuda.synchronize()
    t2, t3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t2.record(ks)
    ev_start.record(ks)
    cs_in.wait_event(ev_start)
    for st in range(args.steps):
        b = st % 2
        with torch.cuda.stream(cs_in):
            if st >= 2:
                cs_in.wait_event(ev_done[b])      # the search of step st-2 has consumed q_stage[b]
            q_stage[b].copy_(u_q_host, non_blocking=True)
            ev_in[b].record(cs_in)
        ks.wait_event(ev_in[b])
        if st >= 2:
            ks.wait_event(ev_out[b])              # step st-2's results have left outs[b]
        s, i = step(q_stage[b], outs[b])
        ev_done[b].record(ks)
        with torch.cuda.stream(cs_out):
            cs_out.wait_event(ev_done[b])
            host_s[b].copy_(s, non_blocking=True)
            host_i[b].copy_(i, non_blocking=True)
            ev_out[b].record(cs_out)
    for b in range(min(2, args.steps)):
        ks.wait_event(ev_out[b])                  # every result is in host memory
    t3.record(ks)
    torch.cuda.synchronize()
    _barrier(world)
    e2e_ms = t2.elapsed_time(t3)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    evals_per_step = nq * n_loc * world
    value = evals_per_step * args.steps / (ms * 1e-3)
    e2e_value = evals_per_step * args.steps / (e2e_ms * 1e-3)

    # the timed run's result equals an untimed run's, byte for byte
    s_timed, i_timed = out[0].clone(), out[1].clone()
    s_chk, i_chk = step(u_q)
    checksum_ok = bool(torch.equal(s_chk, s_timed) and torch.equal(i_chk, i_timed))
    lb = (args.steps - 1) % 2           # the e2e run's last results, as they reached host memory
    e2e_ok = bool(torch.equal(host_s[lb], s_chk.cpu()) and torch.equal(host_i[lb], i_chk.cpu()))

    peaks, peaks_src = _peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    resolved = uq.search_resolve(nq, n_loc, d, k, algo)
    used_f4 = resolved == uq.ALGO_TC_FP4
    used_tc = resolved in (uq.ALGO_TCGEN05, uq.ALGO_TC_FP4)
    algo_name = "tcgen05-f4" if used_f4 else "tcgen05" if used_tc else "popc"
    if asym:
        used_f4, used_tc, algo_name = False, True, "tcgen05-asym-int8"
    if f4x is not None:
        algo_name = "tcgen05-f4-index"
    # dominant kernel = the main scan (every DB row); per launch: nq * n_loc Delta evaluations
    scan_avg_s = (main_ms / max(main_n, 1)) * 1e-3
    evals_per_launch = main_evals / max(main_n, 1)
    if used_f4:
        # E2M1 MACs: d per Delta (T_q . T_db^T with +-1 / 0 exact in E2M1), 2 ops per MAC
        ops = 2.0 * d * evals_per_launch
        peak = 4.0 * float(peaks["bf16_tflops"])   # dense fp4 = 4x bf16 (9 vs 2.25 PFLOP/s nominal)
        achieved = ops / scan_avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "scan_tc2_kernel<NB,0,1> (CTA-pair E2M1 tcgen05 kind::mxf4 Delta GEMM + fused top-k)",
                "peak_source": f"4 x bf16_tflops of {peaks_src} MEASURED_PEAKS.json (dense fp4 = 4x bf16 nominal)",
                "algorithmic": "2*d ops per Delta (d E2M1 MACs)",
                # the rule's peak (4 x measured cuBLAS bf16) is below what UTCOMMA.2CTA
                # sustains back to back (tools/fp4_probe.cu): both fractions reported
                "raw_mma_peak": 8592.0,
                "raw_mma_peak_source": "tools/fp4_probe.cu: back-to-back tcgen05.mma.cta_group::2.kind::mxf4 "
                                       "(M=256, N=256, K=64) on all 148 SMs",
                "frac_of_raw_mma_peak": achieved / 8592.0}
    elif used_tc:
        # int8 MACs: d per Delta (the int8 GEMM T_q . T_db^T), 2 ops per MAC
        ops = 2.0 * d * evals_per_launch
        peak = 2.0 * float(peaks["bf16_tflops"])   # int8 dense = 2x bf16 (guide's nominal ratio)
        achieved = ops / scan_avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": ("scan_tc2_kernel<NB,0,0> (CTA-pair int8 tcgen05, int8 queries as the A operand: "
                           "masked-addition scores + fused top-k)" if asym else
                           "scan_tc2_kernel (CTA-pair int8 tcgen05 Delta GEMM + fused top-k)"
                           if nq > 128 and d <= 1024 else
                           "scan_tc_kernel (int8 tcgen05 Delta GEMM + fused top-k)"),
                "peak_source": f"2 x bf16_tflops of {peaks_src} MEASURED_PEAKS.json (int8 = 2x bf16 nominal)",
                "algorithmic": "2*d ops per Delta (d int8 MACs)"}
    else:
        popc_clk, popc_src = _popc_peak()
        popc_per_delta = 2.0 * ((d + 31) // 32)   # identity: 2 POPC per 32-bit word
        popc_peak = popc_clk * sms * sm_mhz * 1e6 / 1e12
        # per launch the scan must stream every DB code once (d/4 B per row) plus the queries
        bytes_launch = (evals_per_launch / max(nq, 1)) * uq.code_bytes(d) + nq * uq.code_bytes(d)
        hbm_peak = float(peaks["hbm_gbs"])
        t_alu = popc_per_delta * evals_per_launch / (popc_peak * 1e12)
        t_hbm = bytes_launch / (hbm_peak * 1e9)
        if t_hbm >= t_alu:   # small query batches (Q <= ~3): the DB stream is the bound
            achieved = bytes_launch / scan_avg_s / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": None,
                    "kernel": "scan_popc_kernel (LOP3+POPC Delta scan + fused top-k)",
                    "peak_source": f"hbm_gbs of {peaks_src} MEASURED_PEAKS.json",
                    "algorithmic": "code_bytes(d) per DB row + the query codes, per launch",
                    "alu_frac": popc_per_delta * evals_per_launch / scan_avg_s / 1e12 / popc_peak}
        else:
            achieved = popc_per_delta * evals_per_launch / scan_avg_s / 1e12
            roof = {"bound": "alu", "achieved": achieved, "peak": popc_peak, "unit": "Tpopc/s",
                    "frac": achieved / popc_peak, "traffic": None,
                    "kernel": "scan_popc_kernel (LOP3+POPC Delta scan + fused top-k)",
                    "peak_source": f"{popc_clk:.2f} POPC/clk/SM {popc_src} x {sms} SMs x {sm_mhz:.0f} MHz",
                    "algorithmic": "2*ceil(d/32) POPC per Delta"}
    roof["traffic"], tsrc = _traffic(algo_name, w.name, nq)
    if tsrc:
        roof["traffic_source"] = tsrc
    roof["scan_ms_avg"] = scan_avg_s * 1e3
    roof["scan_share_of_step"] = (main_ms / max(ms, 1e-9)) if world == 1 else None
    roof["seed_scan"] = {"ms_avg": seed_ms / max(seed_n, 1), "launches": seed_n,
                         "delta_evals_per_launch": seed_evals / max(seed_n, 1),
                         "share_of_step": (seed_ms / max(ms, 1e-9)) if world == 1 else None,
                         "note": "threshold-seeding scan over a strided DB sample (exactness-preserving filter)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "e2m1" if used_f4 else "s8" if used_tc else "u32",
        "data": "synthetic",
        "config": {"workload": _workload_desc(w), "db_rows_per_gpu": n_loc, "global_db_rows": n_loc * world,
                   "queries": nq, "k": k, "algo": algo_name,
                   "parallelism": (f"db-shard x{world} + " + ("peer-memory merge" if peer is not None else
                                                               "NCCL allgather + merge")) if world > 1 else "single GPU",
                   "l2": f"inputs larger than L2: {n_loc * uq.code_bytes(d) / 1e6:.0f} MB of DB codes per GPU scanned per step"},
        "qps": nq * args.steps / (ms * 1e-3),
        "roofline": roof,
        "index": {"codes_bytes": n_loc * uq.code_bytes(d),
                  "f4_index_bytes": int(f4x.numel()) if f4x is not None else 0,
                  "i8_index_bytes": int(i8x.numel()) if i8x is not None else 0,
                  "f4_index_build_ms": idx_ms,
                  "note": "E2M1 operand image of the codes (4 bits per dim), built once with the index"
                          if f4x is not None else "2-bit codes only"},
        "encode": {"rows_per_s": n_loc / (enc_ms * 1e-3), "GB_per_s": enc_bytes / (enc_ms * 1e-3) / 1e9,
                   "hbm_frac": enc_bytes / (enc_ms * 1e-3) / 1e9 / float(peaks["hbm_gbs"]),
                   "ms": enc_ms, "note": "DB index build, outside the step"},
        "e2e": {"value": e2e_value, "unit": UNIT, "qps": nq * args.steps / (e2e_ms * 1e-3),
                "h2d_bytes_per_step": u_q.numel() * u_q.element_size(),
                "d2h_bytes_per_step": nq * k * (4 + 8),
                "pipeline": "H2D / D2H on copy streams, double-buffered, overlapping the previous / next search",
                "results_equal_untimed_run": e2e_ok},
        "gpu_launches": gpu_launches,
        "step_ms": {"median": statistics.median(step_ms), "min": step_ms[0], "max": step_ms[-1]},
        "checksum_equal_untimed_run": checksum_ok,
        "clocks": clk,
    }
    if world == 1:
        # recall@k of the ternary search vs exact fp32 cosine kNN on the
        # pre-quantisation vectors (untimed; a sample of the step's queries)
        from tools.recall import cosine_topk_fp32, recall_at_k
        ns = min(nq, 100)
        _, gt_i = cosine_topk_fp32(w, u_q[:ns], k, id_base=id_base, n=n_loc)
        line["recall"] = {"k": k, "recall_at_k": recall_at_k(out[1][:ns], gt_i), "queries": ns,
                          "ground_truth": "exact cosine, fp32 with TF32 off, on the float vectors "
                                          "(pinned to the fp64 oracle within 1e-5 relative in tests/test_recall.py)"}
        # k@n (uq_rerank): search n = 4k candidates, re-rank them by
        # cosine on the float vectors, keep k.  Untimed for the headline; the
        # re-rank kernel is timed on its own over the whole query batch.
        kn = min(4 * k, 1024)
        if n_loc >= kn and n_loc * d * 4 <= (40 << 30):
            ws_n = torch.empty(max(uq.search_workspace(nq, n_loc, d, kn, algo), 1), dtype=torch.uint8, device=dev)
            uq.encode(u_q, x, out=qc)
            _, cand = uq.search(qc, dbc, d, kn, id_base=0, algo=algo, workspace=ws_n)
            del ws_n
            u_db_f = datagen.rows(w, "db", id_base, n_loc, dev)
            uq.rerank(u_q, u_db_f, cand, k)                       # warm-up
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            r0.record()
            for _ in range(reps):
                rr_cos, rr_ids = uq.rerank(u_q, u_db_f, cand, k)
            r1.record()
            torch.cuda.synchronize()
            rr_ms = r0.elapsed_time(r1) / reps
            gathered = nq * kn * d * u_db_f.element_size()
            line["rerank"] = {"k": k, "n": kn, "recall_at_k_after_rerank":
                              recall_at_k((rr_ids[:ns] + id_base), gt_i), "queries": ns,
                              "kernel_ms": rr_ms, "candidates_per_s": nq * kn / (rr_ms * 1e-3),
                              "gather_GB_per_s": gathered / (rr_ms * 1e-3) / 1e9,
                              "note": "uq_rerank over the whole batch's n = 4k search candidates (float rows gathered "
                                      "from HBM); recall on the same query sample as `recall`"}
            del u_db_f
            torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    line["paper_context"] = PAPER_CONTEXT
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
