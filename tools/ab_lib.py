"""Build an A/B variant of libuq.so with extra nvcc defines (measurement only):
python tools/ab_lib.py paper_2506_00528_b200/libuq_ab.so -DNAME=VALUE ...
Load it with UQ_LIB_AB=<path> (paper_2506_00528_b200/__init__.py)."""
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_00528_b200"))
import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
tmp = tempfile.mkdtemp()
import concurrent.futures as cf  # noqa: E402
import glob  # noqa: E402


def comp(src):
    obj = os.path.join(tmp, os.path.basename(src) + ".o")
    r = subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))))
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-Xcompiler", "-fPIC"], check=True)
print(out)
