"""CUDA-graph-captured query path for serving small batches.

A search over a fixed database is a short chain of launches (query encode,
threshold seeding scan, main scan, merge, seed verification, the normally-idle
fallback scan and merge); for one or a few queries their launch gaps are a
visible part of the latency (c2, Q = 1: ~0.1 ms per batch).  CapturedSearch
records the whole chain -- uq_encode of the query floats + uq_search -- once
into a torch.cuda.CUDAGraph for a fixed batch shape and replays it: the query
floats are copied into the graph's static input, the results are read from its
static outputs.  Every step still runs in libuq's kernels (the library
allocates nothing and makes no host round trip inside a search, so the chain
is capturable); this module only orchestrates.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch


class CapturedSearch:
    def __init__(self, dbcodes: torch.Tensor, d: int, x: int, k: int, nq: int, dtype=torch.float32,
                 algo: Optional[int] = None, f4_index: Optional[torch.Tensor] = None, id_base: int = 0):
        import paper_2506_00528_b200 as uq
        self.uq = uq
        dev = dbcodes.device
        algo = uq.ALGO_AUTO if algo is None else algo
        self.q = torch.zeros((nq, d), dtype=dtype, device=dev)            # static input (query floats)
        self.qc = torch.empty((nq, uq.code_bytes(d)), dtype=torch.uint8, device=dev)
        self.out = (torch.empty((nq, k), dtype=torch.int32, device=dev),
                    torch.empty((nq, k), dtype=torch.int64, device=dev))
        need = uq.search_workspace(nq, dbcodes.shape[0], d, k, uq.ALGO_TC_FP4 if f4_index is not None else algo)
        self.ws = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
        self.graph = torch.cuda.CUDAGraph()
        args = dict(d=d, x=x, k=k, algo=algo, f4_index=f4_index, id_base=id_base, db=dbcodes)
        self._args = args
        stream = torch.cuda.Stream(device=dev)
        stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(stream):
            self._run()                           # warm-up outside the capture (attributes, tensor maps)
        torch.cuda.current_stream(dev).wait_stream(stream)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(self.graph):
            self._run()

    def _run(self):
        a, uq = self._args, self.uq
        uq.encode(self.q, a["x"], out=self.qc)
        uq.search(self.qc, a["db"], a["d"], a["k"], id_base=a["id_base"], algo=a["algo"], workspace=self.ws,
                  out=self.out, f4_index=a["f4_index"])

    def __call__(self, q: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
        """Search the batch q ([nq][d], the captured shape and dtype): returns the
        graph's output tensors (overwritten by the next call)."""
        self.q.copy_(q, non_blocking=True)
        self.graph.replay()
        return self.out
