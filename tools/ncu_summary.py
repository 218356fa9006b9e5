"""Summarise ncu reports for profiles/: key raw metrics of every captured kernel
(`ncu -i X.ncu-rep --page raw --csv`) and, optionally, the per-source-line
instruction / stall hot spots (`--page source --print-source cuda,sass`).

    python tools/ncu_summary.py gpurun_out/prof_tc.ncu-rep [--lines 25] > profiles/...txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv   # launch-list CSV
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "Grid Size", "Block Size", "launch__registers_per_thread",
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
]


def ncu_csv(args):
    r = subprocess.run(["ncu", *args], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def raw(rep):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    if len(rows) < 3:
        print("(no raw data)")
        return
    h, u = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(h, row))
        print("-" * 78)
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]} {u[h.index(k)]}")
        def nz(k):
            try:
                return float(d[k].replace(",", "")) != 0.0
            except ValueError:
                return False
        extra = [k for k in h if ("tensor" in k or "tcgen" in k or "_tc_" in k) and "pct" in k and ".avg." in k
                 and k not in KEYS and nz(k)][:12]
        for k in extra:
            print(f"{k:70s} {d[k]} {u[h.index(k)]}")


def lines(rep, top):
    rows = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
    hdr, cur = None, None
    ie = collections.Counter()
    st = collections.defaultdict(collections.Counter)
    src = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] != "":
            key = f"{cur}:{r[0]}"
            src[key] = r[1][:70]
            try:
                ie[key] += int(r[hdr.index("Instructions Executed")] or 0)
            except (ValueError, IndexError):
                pass
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "(Not" not in h:
                    try:
                        st[key][h[6:]] += int(r[i] or 0)
                    except ValueError:
                        pass
    tot_i = sum(ie.values())
    tot_s = sum(sum(c.values()) for c in st.values())
    print(f"instructions executed {tot_i}  stall samples {tot_s}")
    keys = sorted(src, key=lambda k: -(ie[k] / max(tot_i, 1) + sum(st[k].values()) / max(tot_s, 1)))
    for k in keys[:top]:
        s = sum(st[k].values())
        print(f"{100*ie[k]/max(tot_i,1):5.1f}%i {100*s/max(tot_s,1):5.1f}%s {k:26s} "
              f"{dict(st[k].most_common(2))} | {src[k]}")


OURS = ("uq::", "tc2::", "encode_", "scan_", "merge_kernel", "rerank_", "quantize", "build_", "thr_from",
        "seed_verify", "check_codes", "scores_kernel")


def launches(path, ours=False):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                if d["Metric Unit"] in ("nsecond", "ns"):
                    v /= 1e3
                elif d["Metric Unit"] in ("msecond", "ms"):
                    v *= 1e3
                if ours and not any(t in d["Kernel Name"] for t in OURS):
                    continue   # data generation / recall ground truth (torch, cuBLAS)
                agg[(d["Kernel Name"][:70], d["Grid Size"])].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':70s} {'grid':>14s} {'n':>4s} {'mean_us':>10s} {'share':>6s}")
    for (k, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:70s} {g:>14s} {len(v):4d} {sum(v)/len(v):10.1f} {sum(v)/tot:6.1%}")


if __name__ == "__main__":
    a = sys.argv[1:]
    if a and a[0] == "--launches":
        launches(a[1], ours="--ours" in a)
    else:
        top = int(a[a.index("--lines") + 1]) if "--lines" in a else 0
        raw(a[0])
        if top:
            print("=" * 78)
            lines(a[0], top)
