#!/usr/bin/env python
"""Benchmark of the EVP ternary kNN hot path on B200 (BASELINE.json metric:
query x db Delta-evals/s and kNN QPS at 1/2/4/8 B200; % of roofline).

One step = one pass of the whole hot path over one query batch of the
workload, for every x of the workload's sweep: encode the Q query embeddings
(uq_encode), scan all N database codes with the fused per-query
top-k (uq_search: seeding scan + main Delta scan + merge),
and for N GPUs the exchange of the per-shard [Q][k] lists + uq_merge_topk.
The database is encoded once before timing (S is pre-processed before q
is known); that encode is timed on its own and reported under "encode".

Default workload: BASELINE configs[2] = c3, the largest single-GPU config:
d=1024, N=1e7, Q=1e4, k=10, x swept over {256, 512, 768} -- one step runs all
three x.  The float database (41 GB fp32) is generated
and encoded chunk by chunk.  Extra keys (N=1, unless --no-extras) measure c2
(d=768, N=1e6, Q=1000, k=100) and c5 (N=5e7 fp16, Q=1 and Q=1024, plus the
end-to-end DB encode + batch) with the same code.

Multi-GPU (torchrun, one process per GPU): --shard strong (default) splits the
config's N rows into G contiguous shards (shard_bounds; BASELINE c4/c5: "N
sharded over 1/2/4/8 B200"), each rank searches its shard with its global
id_base, the lists are exchanged (NCCL allgather or the peer-memory merge
kernel) and merged; every rank ends with the unsharded result, whose SHA-256
("digest") must be identical for every G.  --shard weak gives every rank N rows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--algo auto]
    python bench.py --impl reference ...   # the CPU oracle on the same workload
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import re
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
GEN_BYTES = 4 << 30          # float rows generated + encoded per chunk (<= 4 GiB)
KEEP_FLOATS = 96 << 30       # keep the float DB resident (recall / re-rank / one-call encode) below this


def _log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print("[bench]", *a, file=sys.stderr, flush=True)


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


def _dist(backend: str = "nccl"):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        # before NCCL binds this rank to a device; the gloo test mode (below)
        # lets several ranks share the devices there are
        local = local % torch.cuda.device_count() if backend == "gloo" else local
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        if backend == "gloo":
            # test mode (tests/test_bench_dist.py): the bench's N > 1 code path
            # -- shards, global ids, exchange, merge, digest, max-over-ranks
            # timing -- on one GPU, the lists exchanged through host memory;
            # the ranks' kernels never wait on each other.  Not a scaling run.
            dist.init_process_group("gloo")
            return world, rank, local
        if torch.cuda.is_available() and "NCCL_DEBUG" not in os.environ:
            # NCCL's own record of the communicator (rank count, NVLS / NVLink
            # transport), read back into the JSON line; to a file, not stdout
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT,NVLS"
            os.environ["NCCL_DEBUG_FILE"] = f"/tmp/uq_nccl.{os.getpid()}.log"
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return world, rank, local


def _nccl_info():
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    out = {"backend": dist.get_backend() if dist.is_initialized() else None,
           "world_size": dist.get_world_size() if dist.is_initialized() else 1}
    try:
        out["nccl_version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        pass
    if not path:
        return out
    txt = ""
    for f in glob.glob(path.replace("%h", "*").replace("%p", "*")):
        try:
            with open(f, errors="replace") as fh:
                txt += fh.read()
        except OSError:
            pass
    m = re.findall(r"nRanks (\d+)", txt)
    if m:
        out["nccl_nranks"] = int(m[-1])
    nv = [ln.strip().split("NCCL INFO ", 1)[-1] for ln in txt.splitlines() if "NVLS" in ln][:3]
    if nv:
        out["nccl_nvls_lines"] = nv
    out["nccl_log"] = path
    return out


def _barrier(world):
    if world > 1:
        dist.barrier()


def _max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    t = torch.tensor([v], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): the oracle as it stands
# ---------------------------------------------------------------------------
def _oracle_sample(w, xs, target_s: float):
    """Time the oracle's encode(queries) + exhaustive kNN, for every x of the
    sweep, on a bounded sample of the workload: n_s database rows
    (oracle-encoded, untimed) x q_s queries."""
    import oracle
    n_s = min(w.n, 200_000 if w.d <= 768 else 100_000)
    db = datagen.db(w, "cpu", 0, n_s).numpy()
    q_all = datagen.rows(w, "q", 0, min(w.nq, 4000), "cpu").numpy()
    o_db = {x: oracle.pack(oracle.encode(db, x)) for x in xs}

    def run(nq_s):
        t0 = time.perf_counter()
        for x in xs:
            o_q = oracle.pack(oracle.encode(q_all[:nq_s], x))
            oracle.knn(o_q, o_db[x], w.d, w.k)
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


def cpu_baseline(w, xs, target_s=10.0):
    """The oracle as it stands, on the host's cores: all threads, then 1 thread
    on a proportionally smaller query sample (BASELINE.md CPU plan)."""
    import oracle
    n_s, nq_s, run, cores = _oracle_sample(w, xs, target_s)
    t = run(nq_s)
    prev = oracle.set_threads(1)
    nq1 = max(1, nq_s // max(cores, 1))
    t1 = run(nq1)
    oracle.set_threads(prev)
    nx = len(xs)
    return {"value": nx * nq_s * n_s / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1thread": nx * nq1 * n_s / t1, "cpu_model": _cpu_model(),
            "sample": f"{nq_s} queries x {nx} x in {list(xs)} (oracle encode + exhaustive kNN, k={w.k}) over the "
                      f"first {n_s} database rows of {w.name}; {t:.1f} s wall on {cores} host threads "
                      f"({nq1} queries, {t1:.1f} s on 1 thread)"}


# The paper's own speed numbers for this path (context only, other hardware):
PAPER_CONTEXT = {
    "b2sp_per_delta": "21.8 ns per Delta (10^6 comparisons in 21.75 ms median), d=384, Apple M3, "
                      "Rust BitVecSimd (P:463-476, Table 4): ~4.6e7 Delta-evals/s on one core",
    "exhaustive_1M": "Table 5 (P:485-496), unstated hardware: d=768 Laion {512,768} b2sp 35.7 ms per "
                     "~1M-row query (likelier reading: ~2.8e7 Delta-evals/s)",
    "note": "no GPU numbers in the paper; BASELINE.md"}


def _workload_desc(w, xs):
    xd = f"x={xs[0]}" if len(xs) == 1 else "x in {" + ",".join(str(x) for x in xs) + "}"
    return (f"{w.name}: d={w.d}, N={w.n}, Q={w.nq}, {xd}, k={w.k}, {w.kind}"
            f"{' C=' + str(w.centres) if w.centres else ''}, {str(w.dtype).replace('torch.', '')}"
            f"{', l2-normalised' if w.normalise else ', raw'}")


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    w = datagen.CONFIGS[args.config].scaled(n=args.db_rows, nq=args.nq)
    xs = _xs(args, w)
    n_s, nq_s, run, cores = _oracle_sample(w, xs, target_s=3.0)
    for _ in range(args.warmup):
        run(nq_s)
    times = [run(nq_s) for _ in range(args.steps)]
    tot = sum(times)
    value = args.steps * len(xs) * nq_s * n_s / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.shard == "strong" else "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": _workload_desc(w, xs),
                   "sample": f"{nq_s} queries x {len(xs)} x x {n_s} rows per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{nq_s} queries x first {n_s} rows of {w.name} for each x in {list(xs)}, "
                                   f"per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _xs(args, w):
    if args.x:
        return tuple(int(v) for v in args.x.split(","))
    return tuple(w.xs)


# ---------------------------------------------------------------------------
# GPU measurement of one workload
# ---------------------------------------------------------------------------
class Ctx:
    def __init__(self, args, world, rank, local):
        import paper_2506_00528_b200 as uq
        self.uq = uq
        self.args, self.world, self.rank = args, world, rank
        self.dev = torch.device("cuda", local)
        self.local = local


def build_db(c: Ctx, w, xs, lo: int, n_loc: int, keep_floats: bool):
    """Generate the float rows [lo, lo + n_loc) of the seeded DB stream chunk by
    chunk on the device and encode each chunk for every x (the float DB never
    needs to fit: c4 is 614 GB of fp32).  Returns (codes {x: [n][cb]},
    resident floats or None, encode ms {x: summed kernel time})."""
    uq, dev = c.uq, c.dev
    t_start = time.perf_counter()
    cb = uq.code_bytes(w.d)
    es = torch.tensor([], dtype=w.dtype).element_size()
    codes = {x: torch.empty((n_loc, cb), dtype=torch.uint8, device=dev) for x in xs}
    u_keep = torch.empty((n_loc, w.d), dtype=w.dtype, device=dev) if keep_floats else None
    gen = max(datagen.CHUNK, (GEN_BYTES // (w.d * es)) // datagen.CHUNK * datagen.CHUNK)
    enc_ms = {x: 0.0 for x in xs}
    evs = []
    for s in range(0, n_loc, gen):
        cnt = min(gen, n_loc - s)
        u = datagen.rows(w, "db", lo + s, cnt, dev, out=u_keep[s:s + cnt] if keep_floats else None)
        for x in xs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            uq.encode(u, x, out=codes[x][s:s + cnt])
            e1.record()
            evs.append((x, e0, e1))
        if not keep_floats:
            torch.cuda.synchronize()
            del u
    torch.cuda.synchronize()
    for x, e0, e1 in evs:
        enc_ms[x] += e0.elapsed_time(e1)
    return codes, u_keep, enc_ms, time.perf_counter() - t_start


def measure(c: Ctx, w, xs, steps: int, warmup: int, full: bool = True, prebuilt=None):
    """Time `steps` steps (each: for every x, encode the queries + sharded
    search + exchange) of workload w; returns the JSON fields.  `prebuilt`:
    a build_db() result of the same database (w.n, xs) to reuse."""
    uq, dev, world, rank, args = c.uq, c.dev, c.world, c.rank, c.args
    d, k, nq = w.d, w.k, w.nq
    gloo = world > 1 and dist.get_backend() == "gloo"
    if args.shard == "strong":
        from paper_2506_00528_b200.parallel import shard_bounds
        lo, hi = shard_bounds(w.n, world, rank)
        n_global = w.n
    else:
        lo, hi = rank * w.n, (rank + 1) * w.n
        n_global = w.n * world
    n_loc = hi - lo
    es = torch.tensor([], dtype=w.dtype).element_size()
    keep = full and world == 1 and n_loc * d * es <= KEEP_FLOATS
    if prebuilt is None:
        _log(f"{w.name}: generating + encoding {n_loc} rows (x={list(xs)}, keep floats={keep})")
        prebuilt = build_db(c, w, xs, lo, n_loc, keep)
    codes, u_db, enc_ms, t_gen = prebuilt
    u_q = datagen.queries(w, dev)
    u_q_host = u_q.cpu().pin_memory()

    # --algo asym: single-operand search -- int8-quantised float
    # queries (uq_quantize_i8, R15) x the ternary DB by masked addition
    # (uq_search_asym) on the int8 pair engine, fed by the int8 index
    asym = args.algo == "asym"
    algo = {"auto": uq.ALGO_AUTO, "popc": uq.ALGO_POPC, "tc": uq.ALGO_TCGEN05, "f4": uq.ALGO_TC_FP4,
            "asym": uq.ALGO_TCGEN05}[args.algo]
    resolved = uq.search_resolve(nq, n_loc, d, k, algo)
    use_x = (not args.no_f4_index) and resolved == uq.ALGO_TC_FP4 and not asym
    f4x, i8x, idx_ms = {}, {}, None
    if asym and not args.no_f4_index and d <= 1024:
        for x in xs:
            i8x[x] = uq.build_i8_index(codes[x], d)
    if use_x:
        for x in xs:
            f4x[x] = uq.build_f4_index(codes[x], d)
        ib0, ib1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ib0.record()
        uq.build_f4_index(codes[xs[0]], d, out=f4x[xs[0]])   # rebuilt in place (c4: 76.8 GB)
        ib1.record()
        torch.cuda.synchronize()
        idx_ms = ib0.elapsed_time(ib1)
    # one-call whole-DB encode timing (the floats are resident)
    enc_whole_ms = None
    if u_db is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        uq.encode(u_db, xs[0], out=codes[xs[0]])
        e1.record()
        torch.cuda.synchronize()
        enc_whole_ms = e0.elapsed_time(e1)

    ws = torch.empty(max(uq.search_asym_workspace(nq, n_loc, d, k) if asym else
                         uq.search_workspace(nq, n_loc, d, k, uq.ALGO_TC_FP4 if use_x else algo), 1),
                     dtype=torch.uint8, device=dev)
    q8 = torch.empty((nq, d), dtype=torch.int8, device=dev) if asym else None
    qc = torch.empty((nq, uq.code_bytes(d)), dtype=torch.uint8, device=dev)
    loc = (torch.empty((nq, k), dtype=torch.int32, device=dev), torch.empty((nq, k), dtype=torch.int64, device=dev))
    launches = [0]
    peer = None
    if world > 1 and args.exchange == "peer":
        from paper_2506_00528_b200.parallel import PeerExchange
        peer = PeerExchange(nq, k, dev)
    from paper_2506_00528_b200.parallel import sharded_search

    def new_outs():
        return {x: (torch.empty((nq, k), dtype=torch.int32, device=dev),
                    torch.empty((nq, k), dtype=torch.int64, device=dev)) for x in xs}

    outs_main = new_outs()

    def step(q_dev, outs, marks=None):
        for j, x in enumerate(xs):
            if marks is not None:
                marks[j].record()
            if asym:
                uq.quantize_i8(q_dev, out=q8)
            else:
                uq.encode(q_dev, x, out=qc)
            launches[0] += uq.last_launches()

            def search_fn(qq, db, dd, kk, id_base=0, **kw):
                if asym:
                    kw.pop("algo", None)
                    kw.pop("f4_index", None)
                    r = uq.search_asym(q8, db, dd, kk, id_base=id_base, i8_index=i8x.get(x), **kw)
                else:
                    r = uq.search(qq, db, dd, kk, id_base=id_base, **kw)
                launches[0] += uq.last_launches()
                return (r[0].cpu(), r[1].cpu()) if gloo else r   # gloo exchanges host tensors

            def merge_fn(sg, ig, kk, out=None):
                r = uq.merge_topk(sg.to(dev), ig.to(dev), kk, out=out)
                launches[0] += uq.last_launches()
                return r

            s, i = sharded_search(qc, codes[x], d, k, id_base=lo, search_fn=search_fn, merge_fn=merge_fn,
                                  merge_out=outs[x], exchange=peer.merge if peer is not None else None,
                                  algo=algo, workspace=ws, out=(outs[x] if world == 1 else loc),
                                  f4_index=f4x.get(x))
            if s.data_ptr() != outs[x][0].data_ptr():   # peer exchange returns fresh tensors
                outs[x][0].copy_(s)
                outs[x][1].copy_(i)
        return outs

    for _ in range(warmup):
        step(u_q, outs_main)
    torch.cuda.synchronize()

    # ---- device-timed region ----
    clocks = ClockSampler(c.local)
    clocks.start()
    time.sleep(0.3)
    launches[0] = 0
    uq.timing_enable(True)
    _barrier(world)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(len(xs))] for _ in range(steps)]
    t0.record()
    for st in range(steps):
        step(u_q, outs_main, marks[st])
    t1.record()
    torch.cuda.synchronize()
    _barrier(world)
    uq.timing_enable(False)
    clk = clocks.stop()
    gpu_launches = launches[0]
    ms = t0.elapsed_time(t1)
    # per-x segment times (the segment of x_j ends where x_{j+1}'s begins)
    seg = {x: [] for x in xs}
    for st in range(steps):
        for j, x in enumerate(xs):
            end = marks[st][j + 1] if j + 1 < len(xs) else (marks[st + 1][0] if st + 1 < steps else t1)
            seg[x].append(marks[st][j].elapsed_time(end))
    tim = uq.timing_collect_ex()
    main_ms, main_n, main_evals = tim["main"]
    seed_ms, seed_n, seed_evals = tim["seed"]
    ms = _max_over_ranks(ms, world, dev)

    # ---- end to end through the public API: pinned host queries in, results out ----
    # Every step copies its query floats host -> device and all its (scores,
    # ids) device -> host inside the timed region.  Serving pipeline: the
    # copies run on their own streams, double-buffered, so step s+1's upload
    # and step s's download overlap step s's search; the region ends when the
    # last results are in host memory.
    e2e_ms, e2e_ok = None, None
    h2d = u_q.numel() * u_q.element_size()
    d2h = len(xs) * nq * k * (4 + 8)
    if full:
        host = [{x: (torch.empty((nq, k), dtype=torch.int32).pin_memory(),
                     torch.empty((nq, k), dtype=torch.int64).pin_memory()) for x in xs} for _ in range(2)]
        q_stage = [torch.empty_like(u_q) for _ in range(2)]
        outs = [new_outs() for _ in range(2)]
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
        for st in range(steps):
            b = st % 2
            with torch.cuda.stream(cs_in):
                if st >= 2:
                    cs_in.wait_event(ev_done[b])      # the search of step st-2 has consumed q_stage[b]
                q_stage[b].copy_(u_q_host, non_blocking=True)
                ev_in[b].record(cs_in)
            ks.wait_event(ev_in[b])
            if st >= 2:
                ks.wait_event(ev_out[b])              # step st-2's results have left outs[b]
            step(q_stage[b], outs[b])
            ev_done[b].record(ks)
            with torch.cuda.stream(cs_out):
                cs_out.wait_event(ev_done[b])
                for x in xs:
                    host[b][x][0].copy_(outs[b][x][0], non_blocking=True)
                    host[b][x][1].copy_(outs[b][x][1], non_blocking=True)
                ev_out[b].record(cs_out)
        for b in range(min(2, steps)):
            ks.wait_event(ev_out[b])                  # every result is in host memory
        t3.record(ks)
        torch.cuda.synchronize()
        _barrier(world)
        e2e_ms = _max_over_ranks(t2.elapsed_time(t3), world, dev)
        lb = (steps - 1) % 2
        e2e_ok = all(torch.equal(host[lb][x][0], outs_main[x][0].cpu()) and
                     torch.equal(host[lb][x][1], outs_main[x][1].cpu()) for x in xs)
        del outs, q_stage

    # the timed run's results equal an untimed run's, byte for byte
    snap = {x: (outs_main[x][0].clone(), outs_main[x][1].clone()) for x in xs}
    chk = step(u_q, new_outs())
    checksum_ok = all(torch.equal(chk[x][0], snap[x][0]) and torch.equal(chk[x][1], snap[x][1]) for x in xs)
    from paper_2506_00528_b200.parallel import result_digest
    digest = {f"x={x}": result_digest([snap[x]]) for x in xs}
    digest["all"] = result_digest([snap[x] for x in xs])

    evals_step = len(xs) * nq * n_global
    value = evals_step * steps / (ms * 1e-3)
    peaks, peaks_src = _peaks()
    roof = _roofline(c, w, nq, n_loc, d, algo, use_x, main_ms, main_n, main_evals, seed_ms, seed_n, seed_evals,
                     ms, peaks, peaks_src, asym=asym, i8x=bool(i8x))
    res = {
        "value": value, "ms_per_step": ms / steps, "qps": len(xs) * nq * steps / (ms * 1e-3),
        "per_gpu": {"delta_evals_per_s": value / world, "qps": len(xs) * nq * steps / (ms * 1e-3) / world,
                    "db_rows": n_loc},
        "dtype": roof.pop("_dtype"),
        "roofline": roof,
        "per_x": {f"x={x}": {"ms_median": statistics.median(seg[x]),
                             "delta_evals_per_s": nq * n_global / (statistics.median(seg[x]) * 1e-3),
                             "qps": nq / (statistics.median(seg[x]) * 1e-3)} for x in xs},
        "db_rows_global": n_global, "db_rows_per_gpu": n_loc, "shard": args.shard,
        "index": {"codes_bytes": n_loc * uq.code_bytes(d) * len(xs),
                  "f4_index_bytes": sum(int(t.numel()) for t in f4x.values()),
                  "i8_index_bytes": sum(int(t.numel()) for t in i8x.values()),
                  "f4_index_build_ms": idx_ms,
                  "note": ("E2M1 operand image of the codes (4 bits per dim), one per x, built once with the "
                           "index" if f4x else "2-bit codes only")},
        "encode": _encode_stats(uq, w, xs, n_loc, enc_ms, enc_whole_ms, peaks, t_gen),
        "gpu_launches": gpu_launches,
        "checksum_equal_untimed_run": checksum_ok,
        "digest": digest,
        "clocks": clk,
    }
    if e2e_ms is not None:
        res["e2e"] = {"value": evals_step * steps / (e2e_ms * 1e-3), "unit": UNIT,
                      "qps": len(xs) * nq * steps / (e2e_ms * 1e-3),
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "pipeline": "H2D / D2H on copy streams, double-buffered, overlapping the previous / next search",
                      "results_equal_untimed_run": e2e_ok}
    if full and world == 1:
        res.update(_quality(c, w, xs, u_q, u_db, codes, snap, lo, n_loc, algo))
    del codes, f4x, ws, u_db, prebuilt
    torch.cuda.empty_cache()
    return res


def _encode_stats(uq, w, xs, n_loc, enc_ms, enc_whole_ms, peaks, t_gen):
    es = torch.tensor([], dtype=w.dtype).element_size()
    row_bytes = w.d * es + uq.code_bytes(w.d)
    ms = enc_ms[xs[0]] if enc_whole_ms is None else enc_whole_ms
    gbs = n_loc * row_bytes / (ms * 1e-3) / 1e9
    return {"rows_per_s": n_loc / (ms * 1e-3), "GB_per_s": gbs, "hbm_frac": gbs / float(peaks["hbm_gbs"]),
            "ms": ms, "bytes_per_row": row_bytes,
            "ms_per_x_chunked": {f"x={x}": v for x, v in enc_ms.items()},
            "timing": "one uq_encode call over the whole resident float DB" if enc_whole_ms is not None else
                      "sum of the per-chunk uq_encode kernels (floats generated chunk by chunk)",
            "datagen_s": t_gen, "note": "DB index build, outside the step"}


def _roofline(c, w, nq, n_loc, d, algo, use_x, main_ms, main_n, main_evals, seed_ms, seed_n, seed_evals, ms,
              peaks, peaks_src, asym=False, i8x=False):
    uq = c.uq
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(c.dev).multi_processor_count
    resolved = uq.search_resolve(nq, n_loc, d, w.k, algo)
    used_f4 = resolved == uq.ALGO_TC_FP4 and not asym
    used_tc = resolved in (uq.ALGO_TCGEN05, uq.ALGO_TC_FP4) or asym
    algo_name = ("tcgen05-asym-int8" + ("-index" if i8x else "")) if asym else \
        "tcgen05-f4-index" if use_x else "tcgen05-f4" if used_f4 else "tcgen05" if used_tc else "popc"
    scan_avg_s = (main_ms / max(main_n, 1)) * 1e-3
    evals_per_launch = main_evals / max(main_n, 1)
    if used_f4:
        ops = 2.0 * d * evals_per_launch
        peak = 4.0 * float(peaks["bf16_tflops"])   # dense fp4 = 4x bf16 (9 vs 2.25 PFLOP/s nominal)
        achieved = ops / scan_avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "scan_tc2_kernel<NB,0,1> (CTA-pair E2M1 tcgen05 kind::mxf4 Delta GEMM + fused top-k)",
                "peak_source": f"4 x bf16_tflops of {peaks_src} MEASURED_PEAKS.json (dense fp4 = 4x bf16 nominal)",
                "algorithmic": "2*d ops per Delta (d E2M1 MACs)",
                "raw_mma_peak": 8592.0,
                "raw_mma_peak_source": "tools/fp4_probe.cu: back-to-back tcgen05.mma.cta_group::2.kind::mxf4 "
                                       "(M=256, N=256, K=64) on all 148 SMs",
                "frac_of_raw_mma_peak": achieved / 8592.0, "_dtype": "e2m1"}
    elif used_tc:
        ops = 2.0 * d * evals_per_launch
        peak = 2.0 * float(peaks["bf16_tflops"])   # int8 dense = 2x bf16 (guide's nominal ratio)
        achieved = ops / scan_avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": ("scan_tc2_kernel<NB,0,0> (CTA-pair int8 tcgen05, int8 queries as the A operand: "
                           "masked-addition scores + fused top-k)" if asym else
                           "scan_tc2_kernel (CTA-pair int8 tcgen05 Delta GEMM + fused top-k)"
                           if nq > 128 and d <= 1024 else "scan_tc_kernel (int8 tcgen05 Delta GEMM + fused top-k)"),
                "peak_source": f"2 x bf16_tflops of {peaks_src} MEASURED_PEAKS.json (int8 = 2x bf16 nominal)",
                "algorithmic": "2*d ops per Delta (d int8 MACs)", "_dtype": "s8"}
    else:
        popc_clk, popc_src = _popc_peak()
        popc_per_delta = 2.0 * ((d + 31) // 32)   # identity: 2 POPC per 32-bit word
        popc_peak = popc_clk * sms * sm_mhz * 1e6 / 1e12
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
                    "alu_frac": popc_per_delta * evals_per_launch / scan_avg_s / 1e12 / popc_peak, "_dtype": "u32"}
        else:
            achieved = popc_per_delta * evals_per_launch / scan_avg_s / 1e12
            roof = {"bound": "alu", "achieved": achieved, "peak": popc_peak, "unit": "Tpopc/s",
                    "frac": achieved / popc_peak, "traffic": None,
                    "kernel": "scan_popc_kernel (LOP3+POPC Delta scan + fused top-k)",
                    "peak_source": f"{popc_clk:.2f} POPC/clk/SM {popc_src} x {sms} SMs x {sm_mhz:.0f} MHz",
                    "algorithmic": "2*ceil(d/32) POPC per Delta", "_dtype": "u32"}
    roof["traffic"], tsrc = _traffic(algo_name, w.name, nq)
    if tsrc:
        roof["traffic_source"] = tsrc
    roof["algo"] = algo_name
    roof["scan_ms_avg"] = scan_avg_s * 1e3
    roof["scan_launches"] = main_n
    roof["scan_share_of_step"] = (main_ms / max(ms, 1e-9)) if c.world == 1 else None
    roof["seed_scan"] = {"ms_avg": seed_ms / max(seed_n, 1), "launches": seed_n,
                         "delta_evals_per_launch": seed_evals / max(seed_n, 1),
                         "share_of_step": (seed_ms / max(ms, 1e-9)) if c.world == 1 else None,
                         "note": "threshold-seeding scan over a strided DB sample (exactness-preserving filter)"}
    return roof


def _quality(c, w, xs, u_q, u_db, codes, snap, lo, n_loc, algo):
    """recall@k of the ternary search against exact fp32 cosine kNN on the
    pre-quantisation vectors, and the paper's k@n re-rank, per x
    (untimed; a 100-query sample of the batch)."""
    uq, dev = c.uq, c.dev
    from tools.recall import cosine_topk_fp32, recall_at_k
    k = w.k
    ns = min(w.nq, 100)
    _, gt_i = cosine_topk_fp32(w, u_q[:ns], k, id_base=lo, n=n_loc, db_rows=u_db)
    out = {"recall": {"k": k, "queries": ns,
                      "ground_truth": "exact cosine, fp32 with TF32 off, on the float vectors (pinned to the fp64 "
                                      "oracle within 1e-5 relative in tests/test_recall.py)"}}
    for x in xs:
        out["recall"][f"x={x}"] = recall_at_k(snap[x][1][:ns], gt_i)
    kn = min(4 * k, 1024)
    if u_db is None or n_loc < kn:
        return out
    rr = {"k": k, "n": kn, "queries": ns}
    for x in xs:
        qc = uq.encode(u_q, x)
        _, cand = uq.search(qc, codes[x], w.d, kn, id_base=0, algo=algo)
        uq.rerank(u_q, u_db, cand, k)                       # warm-up
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        r0.record()
        for _ in range(reps):
            rr_cos, rr_ids = uq.rerank(u_q, u_db, cand, k)
        r1.record()
        torch.cuda.synchronize()
        rr_ms = r0.elapsed_time(r1) / reps
        gathered = w.nq * kn * w.d * u_db.element_size()
        rr[f"x={x}"] = {"recall_at_k_after_rerank": recall_at_k(rr_ids[:ns] + lo, gt_i), "kernel_ms": rr_ms,
                        "candidates_per_s": w.nq * kn / (rr_ms * 1e-3),
                        "gather_GB_per_s": gathered / (rr_ms * 1e-3) / 1e9}
    rr["note"] = ("uq_rerank over the whole batch's n = 4k search candidates (float rows gathered from HBM); "
                  "recall on the same query sample as `recall`")
    out["rerank"] = rr
    return out


def _extras(c: Ctx, args):
    """c2 and c5 at full size on this GPU (N=1): the other single-GPU
    workloads of BASELINE.json, measured with the same step; c5 adds the
    end-to-end number of its config (DB encode of 5e7 fp16 rows + one batch)."""
    ex = {}
    steps = max(3, min(args.steps, 10))
    w2 = datagen.CONFIGS["c2"]
    r = measure(c, w2, tuple(w2.xs), steps, 3, full=False)
    ex["c2"] = {"workload": _workload_desc(w2, w2.xs), "value": r["value"], "ms_per_step": r["ms_per_step"],
                "qps": r["qps"], "roofline": {kk: r["roofline"][kk] for kk in ("bound", "achieved", "peak", "unit",
                                                                                "frac", "scan_ms_avg", "algo")},
                "encode": {kk: r["encode"][kk] for kk in ("GB_per_s", "hbm_frac", "ms")}, "digest": r["digest"]["all"]}
    w5 = datagen.CONFIGS["c5"]
    _log(f"c5: generating + encoding {w5.n} rows")
    db5 = build_db(c, w5, tuple(w5.xs), 0, w5.n, False)
    for q in (1, w5.nq):
        wq = w5.scaled(nq=q)
        r = measure(c, wq, tuple(w5.xs), steps, 3, full=False, prebuilt=db5)
        key = f"c5_q{q}"
        ex[key] = {"workload": _workload_desc(wq, wq.xs), "value": r["value"], "ms_per_step": r["ms_per_step"],
                   "qps": r["qps"], "roofline": {kk: r["roofline"][kk] for kk in ("bound", "achieved", "peak", "unit",
                                                                                   "frac", "scan_ms_avg", "algo")},
                   "digest": r["digest"]["all"]}
        enc = r["encode"]
        ex[key]["encode"] = {kk: enc[kk] for kk in ("GB_per_s", "hbm_frac", "ms", "timing")}
        # end to end for the config: encode the whole fp16 DB, build the E2M1
        # index when the batch's engine reads one, then one batch
        idx_ms = (r.get("index") or {}).get("f4_index_build_ms") or 0.0
        ex[key]["f4_index_build_ms"] = idx_ms
        ex[key]["e2e_db_encode_plus_batch_ms"] = enc["ms"] + idx_ms + r["ms_per_step"]
    del db5
    torch.cuda.empty_cache()
    return ex


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--x", default=None, help="comma-separated x values (default: the config's sweep)")
    ap.add_argument("--algo", default="auto", choices=["auto", "popc", "tc", "f4", "asym"],
                    help="asym: single-operand search (P:507-509), int8 queries x ternary DB")
    ap.add_argument("--shard", default="strong", choices=["strong", "weak"],
                    help="strong: the config's N rows split over the G ranks; weak: N rows per rank")
    ap.add_argument("--db-rows", type=int, default=None, help="override DB rows N (global for --shard strong)")
    ap.add_argument("--queries", "--nq", dest="nq", type=int, default=None, help="override the query batch Q")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c2 / c5 extra measurements")
    ap.add_argument("--no-f4-index", action="store_true",
                    help="E2M1 pair engine expands the 2-bit codes itself instead of reading the E2M1 index")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test mode for the N>1 code path on one GPU (tests/test_bench_dist.py)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N>1: NCCL allgather + merge, or one merge kernel reading every rank's lists "
                         "from symmetric (peer-mapped) memory")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = _dist(args.dist_backend)
    if args.impl == "reference":
        rc = run_reference(args, world, rank)
        if world > 1:
            dist.destroy_process_group()
        return rc

    c = Ctx(args, world, rank, local)
    w = datagen.CONFIGS[args.config].scaled(n=args.db_rows, nq=args.nq)
    xs = _xs(args, w)
    r = measure(c, w, xs, args.steps, args.warmup, full=True)
    line = {
        "metric": METRIC, "value": r.pop("value"), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r.pop("ms_per_step"), "higher_is_better": True,
        "scaling": "strong" if args.shard == "strong" else "weak", "vs_baseline": None, "dtype": r.pop("dtype"),
        "data": "synthetic",
        "config": {"workload": _workload_desc(w, xs), "db_rows_global": r["db_rows_global"],
                   "db_rows_per_gpu": r["db_rows_per_gpu"], "queries": w.nq, "k": w.k, "x": list(xs),
                   "algo": r["roofline"]["algo"],
                   "parallelism": (f"db-shard x{world} ({args.shard}) + " +
                                   ("peer-memory merge" if args.exchange == "peer" else "NCCL allgather + merge"))
                   if world > 1 else "single GPU",
                   "l2": f"inputs larger than L2: {r['index']['codes_bytes'] / 1e6:.0f} MB of DB codes "
                         f"(+ {r['index']['f4_index_bytes'] / 1e6:.0f} MB E2M1 index) per GPU scanned per step"},
    }
    line.update(r)
    if world > 1:
        line["comm"] = _nccl_info()
    if rank == 0 and world == 1 and not args.no_extras and args.config == "c3" and args.db_rows is None:
        line["extras"] = _extras(c, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, xs)
    line["paper_context"] = PAPER_CONTEXT
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
