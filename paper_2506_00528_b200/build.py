"""Build libuq.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libuq.so")
# Profile build (tools/ only): -DUQ_PROFILE compiles in the tensor scans'
# timing ablations and cycle accounting (UQ_TC_ABLATE); the product libuq.so
# never has them.
LIB_PROF = os.path.join(HERE, "libuq_prof.so")
# Checked build (tools/sanitize.py): -DUQ_CHECKED compiles in device-side
# bounds asserts (UQ_ASSERT, common.cuh) -- the stand-in for compute-sanitizer,
# which this GPU pool does not allow.
LIB_CHECKED = os.path.join(HERE, "libuq_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(HERE, "..", "include", "uq.h")])


def _variant_flags(profile: bool, checked: bool):
    return (["-DUQ_PROFILE"] if profile else []) + (["-DUQ_CHECKED"] if checked else [])


def _compile(src: str, verbose: bool, profile: bool = False, checked: bool = False) -> str:
    suffix = (".prof" if profile else "") + (".chk" if checked else "") + ".o"
    obj = os.path.join(OBJ, os.path.basename(src) + suffix)
    cmd = [NVCC, *ARCH, *FLAGS, *_variant_flags(profile, checked), "-c", src, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def _src_hash(profile: bool = False, checked: bool = False) -> str:
    import hashlib
    h = hashlib.sha256(" ".join(_variant_flags(profile, checked)).encode())
    for p in _deps():
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, profile: bool = False, checked: bool = False) -> str:
    """Compile if the library is missing or its recorded source hash differs
    (content-based: file mtimes do not survive the snapshot to the GPU box)."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    lib = LIB_PROF if profile else LIB_CHECKED if checked else LIB
    stamp = lib + ".srchash"
    digest = _src_hash(profile, checked)
    if not force and os.path.exists(lib) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == digest:
                return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, profile, checked), srcs))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    with open(stamp, "w") as f:
        f.write(digest + "\n")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv,
                checked="--checked" in sys.argv))
