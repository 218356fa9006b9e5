"""Recall@k of the ternary (EVP) search against exact cosine kNN (evaluation,
not the hot path).

Ground truth (R12): cosine similarity on the
pre-quantisation vectors, top-k by (cos desc, id asc), computed on the GPU in
fp32 (TF32 off) over the database regenerated chunk by chunk from the same
seeded stream the index was encoded from.  recall@k = |ids_Delta ∩ ids_cos| / k
per query (the paper's k@n with n = k), averaged over the sampled
queries.  tests/test_recall.py pins the fp32 ground truth to the fp64 oracle
(orc_cosine_knn) within 1e-5 relative.
"""
from __future__ import annotations

import torch

import datagen


def cosine_topk_fp32(w, q_rows: torch.Tensor, k: int, id_base: int = 0, n: int | None = None,
                     chunk: int = 1 << 16, db_rows: torch.Tensor | None = None):
    """Exact cosine top-k of the float queries q_rows [Q][d] against database rows
    [id_base, id_base + n) of workload w: (cos [Q][k] fp32, ids [Q][k] int64).
    `db_rows` (optional): those rows already resident ([n][d]), else regenerated."""
    n = w.n if n is None else n
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        q = q_rows.float()
        q = q / q.norm(dim=1, keepdim=True)
        best_s = torch.full((q.shape[0], k), -float("inf"), device=q.device)
        best_i = torch.full((q.shape[0], k), -1, dtype=torch.int64, device=q.device)
        for s0 in range(0, n, chunk):
            c = min(chunk, n - s0)
            u = (db_rows[s0:s0 + c] if db_rows is not None else datagen.rows(w, "db", id_base + s0, c, q.device)).float()
            u = u / u.norm(dim=1, keepdim=True)
            sc = q @ u.T                                   # [Q][c] fp32
            ids = torch.arange(id_base + s0, id_base + s0 + c, device=q.device).expand(q.shape[0], c)
            cs = torch.cat([best_s, sc], dim=1)
            ci = torch.cat([best_i, ids], dim=1)
            # (cos desc, id asc): stable sort by id first, then by -cos
            o = torch.argsort(ci, dim=1, stable=True)
            cs, ci = torch.gather(cs, 1, o), torch.gather(ci, 1, o)
            o = torch.argsort(-cs, dim=1, stable=True)[:, :k]
            best_s, best_i = torch.gather(cs, 1, o), torch.gather(ci, 1, o)
        return best_s, best_i
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def recall_at_k(ids_delta: torch.Tensor, ids_cos: torch.Tensor) -> float:
    """Mean over queries of |ids_Delta ∩ ids_cos| / k."""
    k = ids_cos.shape[1]
    hit = (ids_delta.unsqueeze(2) == ids_cos.unsqueeze(1)).any(dim=2).sum(dim=1).float()
    return float((hit / k).mean())
