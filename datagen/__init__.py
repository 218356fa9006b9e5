"""Seeded synthetic workloads standing in for the paper's datasets.

This module holds NO arithmetic of the method (no encoding, no Delta, no
selection): it only draws the float embeddings that both the CUDA path and the
oracle consume.  Recipes:

* ``iid``: rows ~ N(0, I_d), then l2-normalised (BASELINE config 1; stands in
  for the paper's uniform-on-the-hypersphere sets).
* ``mixture``: C centres c_j ~ N(0, I_d) from their own stream, label j(r)
  uniform in [0, C), u = c_j + sigma * eps with eps ~ N(0, I_d); l2-normalised
  for configs 2-4, left raw (fp16) for config 5.  Stands in for GloVe-100 /
  PubMed-384 / CLIP-Laion-768, which are not available here.

Generation is chunk-addressable: rows [c*CHUNK, (c+1)*CHUNK) of a stream are a
pure function of (config seed, stream, c), so any shard / chunk can be
regenerated on any device and the data is identical for every GPU count.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional

import torch

CHUNK = 1 << 14
BASE_SEED = 250600528


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    d: int
    n: int              # database rows
    nq: int             # queries
    xs: tuple           # EVP non-zero counts x
    k: int
    kind: str           # "iid" | "mixture"
    centres: int = 0
    sigma: float = 0.3
    normalise: bool = True
    dtype: torch.dtype = torch.float32
    seed: int = BASE_SEED

    @property
    def x(self) -> int:
        return self.xs[0]

    def scaled(self, n: Optional[int] = None, nq: Optional[int] = None, **kw) -> "Workload":
        """Same recipe, fewer rows (same per-row distribution, same seeds)."""
        return dataclasses.replace(self, n=self.n if n is None else n,
                                   nq=self.nq if nq is None else nq, **kw)


# BASELINE.json "configs" (index 0..4)
CONFIGS = {
    "c1": Workload("c1", d=384, n=10_000, nq=100, xs=(192,), k=10, kind="iid", seed=BASE_SEED + 1),
    "c2": Workload("c2", d=768, n=1_000_000, nq=1_000, xs=(384,), k=100, kind="mixture",
                   centres=1_000, seed=BASE_SEED + 2),
    "c3": Workload("c3", d=1024, n=10_000_000, nq=10_000, xs=(256, 512, 768), k=10,
                   kind="mixture", centres=10_000, seed=BASE_SEED + 3),
    "c4": Workload("c4", d=1536, n=100_000_000, nq=10_000, xs=(768,), k=100, kind="mixture",
                   centres=100_000, seed=BASE_SEED + 4),
    "c5": Workload("c5", d=768, n=50_000_000, nq=1_024, xs=(384,), k=10, kind="mixture",
                   centres=10_000, normalise=False, dtype=torch.float16, seed=BASE_SEED + 5),
}


def _seed(*parts) -> int:
    h = hashlib.sha256(("/".join(str(p) for p in parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def _gen(device, *parts) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(_seed(*parts))
    return g


_centre_cache: dict = {}


def centres(w: Workload, device="cpu") -> torch.Tensor:
    key = (w.seed, w.d, w.centres, str(device))
    if key not in _centre_cache:
        g = _gen(device, w.seed, "centres")
        _centre_cache.clear()
        _centre_cache[key] = torch.randn(w.centres, w.d, generator=g, device=device,
                                         dtype=torch.float32)
    return _centre_cache[key]


def _chunk(w: Workload, stream: str, c: int, rows: int, device) -> torch.Tensor:
    g = _gen(device, w.seed, stream, c)
    eps = torch.randn(rows, w.d, generator=g, device=device, dtype=torch.float32)
    if w.kind == "iid":
        u = eps
    elif w.kind == "mixture":
        lab = torch.randint(0, w.centres, (rows,), generator=g, device=device)
        u = centres(w, device)[lab] + w.sigma * eps
    else:
        raise ValueError(w.kind)
    if w.normalise:
        u = u / torch.linalg.vector_norm(u, dim=1, keepdim=True)
    return u.to(w.dtype)


def rows(w: Workload, stream: str, start: int, count: int, device="cpu",
         out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Rows [start, start+count) of stream "db" or "q" as a [count][d] tensor."""
    if out is None:
        out = torch.empty(count, w.d, dtype=w.dtype, device=device)
    pos = 0
    while pos < count:
        r = start + pos
        c, off = divmod(r, CHUNK)
        take = min(CHUNK - off, count - pos)
        out[pos:pos + take] = _chunk(w, stream, c, CHUNK, device)[off:off + take]
        pos += take
    return out


def db(w: Workload, device="cpu", start: int = 0, count: Optional[int] = None) -> torch.Tensor:
    return rows(w, "db", start, w.n - start if count is None else count, device)


def queries(w: Workload, device="cpu") -> torch.Tensor:
    return rows(w, "q", 0, w.nq, device)
