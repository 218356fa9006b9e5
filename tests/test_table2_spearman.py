"""Table 2, the uniform rows: Spearman rho between the true
distance of random pairs and the EVP proxy distance, computed through the
CUDA path (uq_encode + uq_scores).  A statistical pin, not a bit-exact one:
the paper does not state its pair sample, so the check is |rho -
paper| <= 0.03 for EVP {67,100} / {667,1000} on uniform-on-the-sphere vectors
("uniformly distributed"; SURVEY.md section 4 reading), and the paper's
claim that EVP beats the 1-bit quantisation (the {d,d} EVP)
"without exception".  The 1-bit column itself does not reproduce
(measured ~0.62-0.63 vs the printed 0.70 / 0.64) and is
only reported, in tools/table2.py's output under profiles/."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def uq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2506_00528_b200 as m
    return m


def spearman_uniform(uq, d, x, n=20_000, pairs=100_000, seed=0):
    """Spearman rho between l2 distance (fp64, original vectors) and -Delta over
    `pairs` random pairs of n uniform-sphere vectors (codes from uq_encode, Delta
    from uq_scores)."""
    from scipy.stats import spearmanr
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.randn(n, d, device="cuda", generator=g, dtype=torch.float32)
    u = u / u.norm(dim=1, keepdim=True)
    codes = uq.encode(u, x)
    nq = 200
    delta = uq.scores(codes[:nq], codes[nq:], d).cpu().numpy().astype(np.float64)    # [nq][n - nq]
    rng = np.random.default_rng(seed)
    qi = rng.integers(0, nq, size=pairs)
    ri = rng.integers(0, n - nq, size=pairs)
    uh = u.double().cpu().numpy()
    dist = np.linalg.norm(uh[qi] - uh[nq + ri], axis=1)
    return float(spearmanr(dist, -delta[qi, ri]).statistic)


@pytest.mark.parametrize("d,x,paper", [(100, 67, 0.80), (1000, 667, 0.79)])
def test_table2_uniform_evp_spearman(uq, d, x, paper):
    rho = spearman_uniform(uq, d, x)
    rho_1bit = spearman_uniform(uq, d, d)
    assert abs(rho - paper) <= 0.03, (d, rho, paper)
    assert rho > rho_1bit + 0.05, (rho, rho_1bit)
