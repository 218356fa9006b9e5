"""Table 2 uniform rows reproduced through the CUDA path: Spearman
rho of true l2 distance vs the EVP / 1-bit proxy distance over 10^5 random
pairs of 2*10^4 uniform-sphere vectors (tests/test_table2_spearman.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_00528_b200 as uq  # noqa: E402
from tests.test_table2_spearman import spearman_uniform  # noqa: E402

PAPER = {100: {"evp": 0.80, "1bit": 0.70, "b1.58": 0.75}, 1000: {"evp": 0.79, "1bit": 0.64, "b1.58": 0.71}}
for d, x in ((100, 67), (1000, 667)):
    print(json.dumps({"d": d, "evp_x": x, "rho_evp": spearman_uniform(uq, d, x),
                      "rho_1bit": spearman_uniform(uq, d, d), "paper": PAPER[d],
                      "pairs": 100_000, "vectors": 20_000}), flush=True)
