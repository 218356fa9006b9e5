#!/bin/bash
# Negative control for tests/test_gpu_parity.py::test_index_seed_samples_spread_rows:
# rebuild the library with the round-1 index-seeding row map in a
# scratch copy and check that the test FAILS there (it passes on the fixed code).
set -u
rm -rf /tmp/bugrepo && cp -r "$(dirname "$0")/.." /tmp/bugrepo && cd /tmp/bugrepo || exit 2
python - <<'PY'
p = "paper_2506_00528_b200/csrc/scan_tc2.cu"
s = open(p).read()
a = "const int64_t sr = row0 + (int64_t)tile * BN + (int64_t)cr * BH;"
b = "        return row / BH;\n      };"
assert a in s and b in s
s = s.replace(a, "const int64_t sr = (int64_t)tile * BN + (int64_t)cr * BH;")
s = s.replace(b, "        return (row0 + row) / BH;\n      };")
open(p, "w").write(s)
PY
rm -f paper_2506_00528_b200/libuq.so paper_2506_00528_b200/libuq.so.srchash
python -m pytest tests/test_gpu_parity.py -q -k "spread_rows" 2>&1 | tail -15
