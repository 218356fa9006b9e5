"""Per-kernel SASS opcode census of libuq.so (cuobjdump -sass): the
instructions that prove the sm_100a paths -- UTCOMMA / UTCIMMA (tcgen05.mma
kind::mxf4 / kind::i8), UTCBAR (tcgen05.commit), LDTM (tcgen05.ld), UBLKCP
(cp.async.bulk), UTMALDG (cp.async.bulk.tensor = TMA), UBLKPF (bulk L2
prefetch), SYNCS (mbarrier), POPC, HSET2.  Output: profiles/r02/sass_census.txt.

    python tools/sass_census.py [path/to/libuq.so]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2506_00528_b200", "libuq.so")
OPS = ["UTCOMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UBLKPF", "SYNCS",
       "POPC", "HSET2", "REDUX", "ATOMS"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, per = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)", line)
    if m:
        op = m.group(1)
        per[cur]["_total"] += 1
        for o in OPS:
            if op == o or op.startswith(o + "."):
                per[cur][o] += 1


def short(name):
    r = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return re.sub(r"\(.*", "", r).replace("uq::", "")[:70]


print(f"libuq.so SASS census ({lib}); counts are static instruction counts per kernel")
print(f"{'kernel':70s} {'total':>6s} " + " ".join(f"{o:>7s}" for o in OPS))
agg = collections.defaultdict(collections.Counter)
for f, c in per.items():
    agg[re.sub(r"<.*", "", short(f))].update(c)
for f, c in per.items():
    s = short(f)
    if any(c[o] for o in ("UTCOMMA", "UTCIMMA", "UTMALDG", "UBLKCP")) or "encode" in s or "merge" in s:
        if "<6," in s or "<8," in s or "<6>" in s or "<3," in s or "merge" in s or "encode_kernel<float, 8" in s:
            print(f"{s:70s} {c['_total']:6d} " + " ".join(f"{c[o]:7d}" for o in OPS))
print("\nper kernel family (all instantiations):")
for f, c in agg.items():
    print(f"{f:70s} {c['_total']:6d} " + " ".join(f"{c[o]:7d}" for o in OPS))
