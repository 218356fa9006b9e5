"""bench.py's N > 1 code path, run for real: two torchrun ranks share the test
box's one GPU with the gloo test backend (`--dist-backend gloo`: the per-rank
[Q][k] lists are exchanged through host memory, the ranks' kernels never wait
on each other).  Each rank generates, encodes and searches its strong shard
with its global id_base; the merged result's digest must equal the one-rank
run's (the byte-equality check the driver's scaling runs rely on, R17), and
the JSON line must report the rank count and whole-job throughput."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--config", "c2", "--db-rows", "120001", "--queries", "300", "--steps", "3", "--warmup", "3", "--no-extras",
        "--no-cpu-baseline"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out: str) -> dict:
    return json.loads([ln for ln in out.strip().splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("algo", ["auto", "popc"])
def test_bench_two_ranks_digest_equals_one_rank(algo):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, PYTHONPATH=ROOT)
    one = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *ARGS, "--algo", algo], env=env,
                         capture_output=True, text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-2000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                          os.path.join(ROOT, "bench.py"), *ARGS, "--algo", algo, "--gpus", "2",
                          "--dist-backend", "gloo"], env=env, capture_output=True, text=True, timeout=900)
    assert two.returncode == 0, two.stderr[-2000:]
    a, b = _line(one.stdout), _line(two.stdout)
    assert b["n_gpus"] == 2 and b["scaling"] == "strong" and b["comm"]["backend"] == "gloo"
    assert b["db_rows_global"] == a["db_rows_global"] == 120001 and b["db_rows_per_gpu"] in (60000, 60001)
    assert b["digest"] == a["digest"], (a["digest"], b["digest"])
    assert b["checksum_equal_untimed_run"] and b["e2e"]["results_equal_untimed_run"]
