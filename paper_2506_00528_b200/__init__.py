"""uq -- B200-native brute-force kNN over {x,d} EVP ternary codes (arXiv 2506.00528).

Thin Python binding over the C ABI of ``libuq.so`` (``include/uq.h``): argument
marshalling only.  Every step of the path (encode, Delta scan, top-k, merge)
runs in the library's sm_100a kernels; PyTorch provides device memory, streams
and process groups.  There is no CPU fallback: importing this package without
the built library raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

__all__ = [
    "UQError", "lib_path", "code_bytes", "plane_bytes", "encode", "scores", "search",
    "search_workspace", "search_resolve", "merge_topk", "check_codes", "ALGO_AUTO", "ALGO_POPC", "ALGO_TCGEN05", "ALGO_TC_FP4",
    "last_launches", "version", "timing_enable", "timing_collect", "timing_collect_ex", "rerank",
    "quantize_i8", "search_asym", "search_asym_workspace", "merge_topk_ptrs", "build_f4_index", "build_i8_index",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# tools/ may load the profile build (timing ablations compiled in) with
# UQ_PROFILE_LIB=1, or the checked build (device bounds asserts) with
# UQ_CHECKED_LIB=1, set before import; everything else loads the product library.
_LIB_PATH = os.path.join(_HERE, "libuq_prof.so" if os.environ.get("UQ_PROFILE_LIB") == "1" else
                         "libuq_checked.so" if os.environ.get("UQ_CHECKED_LIB") == "1" else "libuq.so")
# A/B measurements of build variants (tools only): an explicit library path
_LIB_PATH = os.environ.get("UQ_LIB_AB") or _LIB_PATH

ALGO_AUTO, ALGO_POPC, ALGO_TCGEN05, ALGO_TC_FP4 = 0, 1, 2, 3
_DT = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}
_STATUS = {0: "UQ_OK", 1: "UQ_ERR_INVALID_ARG", 2: "UQ_ERR_UNSUPPORTED", 3: "UQ_ERR_CUDA",
           4: "UQ_ERR_WORKSPACE"}


class UQError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} failed: {_STATUS.get(status, status)}")
        self.status = status


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"libuq.so not found at {_LIB_PATH}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = ctypes.CDLL(_LIB_PATH)
    i32, i64, vp, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    L.uq_code_bytes.argtypes, L.uq_code_bytes.restype = [i32], sz
    L.uq_version.argtypes, L.uq_version.restype = [], ctypes.c_char_p
    L.uq_last_launches.argtypes, L.uq_last_launches.restype = [], i32
    L.uq_encode.argtypes = [vp, i32, i64, i32, i64, i32, vp, vp]
    L.uq_scores.argtypes = [vp, i64, vp, i64, i32, vp, vp]
    L.uq_search_workspace_ex.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz)]
    L.uq_search_ex.argtypes = [vp, i64, vp, i64, i32, i32, i64, vp, vp, vp, sz, i32, vp]
    L.uq_merge_topk.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp]
    L.uq_rerank.argtypes = [vp, i32, i64, i64, vp, i64, i64, i32, vp, i32, i32, vp, vp, vp]
    L.uq_check_codes.argtypes = [vp, i64, i32, vp, vp]
    L.uq_quantize_i8.argtypes = [vp, i32, i64, i32, i64, vp, i64, vp]
    L.uq_merge_topk_ptrs.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp]
    L.uq_f4_index_bytes.argtypes, L.uq_f4_index_bytes.restype = [i64, i32], sz
    L.uq_build_f4_index.argtypes = [vp, i64, i32, vp, vp]
    L.uq_search_f4x.argtypes = [vp, i64, vp, vp, sz, i64, i32, i32, i64, vp, vp, vp, sz, vp]
    L.uq_i8_index_bytes.argtypes, L.uq_i8_index_bytes.restype = [i64, i32], sz
    L.uq_build_i8_index.argtypes = [vp, i64, i32, vp, vp]
    L.uq_search_asym_x.argtypes = [vp, i64, i64, vp, vp, sz, i64, i32, i32, i64, vp, vp, vp, sz, vp]
    L.uq_search_asym_workspace.argtypes = [i64, i64, i32, i32, ctypes.POINTER(sz)]
    L.uq_search_asym.argtypes = [vp, i64, i64, vp, i64, i32, i32, i64, vp, vp, vp, sz, vp]
    L.uq_search_resolve.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(i32)]
    L.uq_timing_enable.argtypes = [i32]
    L.uq_timing_collect.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
    L.uq_timing_collect_ex.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64),
                                       ctypes.POINTER(ctypes.c_double)]
    for f in ("uq_search_resolve", "uq_timing_enable", "uq_timing_collect", "uq_timing_collect_ex", "uq_encode", "uq_scores", "uq_search_workspace_ex", "uq_search_ex", "uq_merge_topk",
              "uq_check_codes", "uq_rerank", "uq_quantize_i8", "uq_search_asym_workspace", "uq_search_asym",
              "uq_merge_topk_ptrs", "uq_build_f4_index", "uq_search_f4x", "uq_build_i8_index",
              "uq_search_asym_x"):
        getattr(L, f).restype = i32
    return L


_L = _load()


def lib_path() -> str:
    return _LIB_PATH


def version() -> str:
    return _L.uq_version().decode()


def last_launches() -> int:
    """Kernels enqueued by the most recent uq_* call on this thread."""
    return int(_L.uq_last_launches())


def timing_enable(on: bool = True) -> None:
    """Bracket every scan kernel launched from this thread with CUDA events."""
    _check("uq_timing_enable", _L.uq_timing_enable(1 if on else 0))


def timing_collect() -> Tuple[float, int]:
    """(summed scan-kernel milliseconds, number of timed launches) since last collect."""
    ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
    _check("uq_timing_collect", _L.uq_timing_collect(ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)


def timing_collect_ex() -> dict:
    """Scan-kernel timing split by kind: {"main": (ms, launches, delta_evals),
    "seed": (...)} since the last collect."""
    ms = (ctypes.c_double * 2)()
    n = (ctypes.c_int64 * 2)()
    ev = (ctypes.c_double * 2)()
    _check("uq_timing_collect_ex", _L.uq_timing_collect_ex(ms, n, ev))
    return {"main": (float(ms[0]), int(n[0]), float(ev[0])),
            "seed": (float(ms[1]), int(n[1]), float(ev[1]))}


def code_bytes(d: int) -> int:
    return int(_L.uq_code_bytes(d))


def plane_bytes(d: int) -> int:
    return code_bytes(d) // 2


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _empty(stream, *shape_args, **kw) -> torch.Tensor:
    """torch.empty allocated ON `stream` (the stream the kernels run on): the
    caching allocator then never hands the block to another stream's
    allocation while this call's kernels may still be using it."""
    if stream is None:
        return torch.empty(*shape_args, **kw)
    with torch.cuda.stream(stream):
        return torch.empty(*shape_args, **kw)


def _index_bytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() > 0 else 0)


def _check(fn: str, st: int):
    if st != 0:
        raise UQError(fn, st)


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")


def encode(u: torch.Tensor, x: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Nearest {x,d} EVP vertex codes of the rows of ``u`` ([n][d], row stride
    ``u.stride(0)``), packed [n][code_bytes(d)] uint8 (uq_encode)."""
    _dev(u, "u")
    if u.dim() != 2 or u.stride(1) != 1:
        raise ValueError("u must be 2-D with unit column stride")
    if u.dtype not in _DT:
        raise TypeError(f"unsupported dtype {u.dtype}")
    n, d = u.shape
    if out is None:
        out = _empty(stream, (n, code_bytes(d)), dtype=torch.uint8, device=u.device)
    _check("uq_encode", _L.uq_encode(_ptr(u), _DT[u.dtype], n, d, u.stride(0), x, _ptr(out),
                                     _stream(stream)))
    return out


def scores(qcodes: torch.Tensor, dbcodes: torch.Tensor, d: int, stream=None) -> torch.Tensor:
    """Dense Delta matrix [nq][n] int32 (uq_scores; test/debug)."""
    _dev(qcodes, "qcodes"); _dev(dbcodes, "dbcodes")
    nq, n = qcodes.shape[0], dbcodes.shape[0]
    out = _empty(stream, (nq, n), dtype=torch.int32, device=qcodes.device)
    _check("uq_scores", _L.uq_scores(_ptr(qcodes), nq, _ptr(dbcodes), n, d, _ptr(out),
                                     _stream(stream)))
    return out


def search_workspace(nq: int, n: int, d: int, k: int, algo: int = ALGO_AUTO) -> int:
    b = ctypes.c_size_t(0)
    _check("uq_search_workspace", _L.uq_search_workspace_ex(nq, n, d, k, algo, ctypes.byref(b)))
    return int(b.value)


def search_resolve(nq: int, n: int, d: int, k: int, algo: int = ALGO_AUTO) -> int:
    """Scan engine (ALGO_POPC / ALGO_TCGEN05 / ALGO_TC_FP4) that search(algo) runs for this shape."""
    r = ctypes.c_int32(0)
    _check("uq_search_resolve", _L.uq_search_resolve(nq, n, d, k, algo, ctypes.byref(r)))
    return int(r.value)


def build_f4_index(dbcodes: torch.Tensor, d: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """E2M1 index of the database codes for the pair engine (uq_build_f4_index)."""
    _dev(dbcodes, "dbcodes")
    n = dbcodes.shape[0]
    nb = max(int(_L.uq_f4_index_bytes(n, d)), 16)
    if out is None:
        out = _empty(stream, nb, dtype=torch.uint8, device=dbcodes.device)
    elif out.dtype != torch.uint8 or out.numel() != nb or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous uint8 tensor of {nb} bytes")
    _check("uq_build_f4_index", _L.uq_build_f4_index(_ptr(dbcodes), n, d, _ptr(out), _stream(stream)))
    return out


def build_i8_index(dbcodes: torch.Tensor, d: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """int8 index of the database codes for single-operand search (uq_build_i8_index)."""
    _dev(dbcodes, "dbcodes")
    n = dbcodes.shape[0]
    nb = max(int(_L.uq_i8_index_bytes(n, d)), 16)
    if out is None:
        out = _empty(stream, nb, dtype=torch.uint8, device=dbcodes.device)
    elif out.dtype != torch.uint8 or out.numel() != nb or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous uint8 tensor of {nb} bytes")
    _check("uq_build_i8_index", _L.uq_build_i8_index(_ptr(dbcodes), n, d, _ptr(out), _stream(stream)))
    return out


def search(qcodes: torch.Tensor, dbcodes: torch.Tensor, d: int, k: int, id_base: int = 0,
           algo: int = ALGO_AUTO, workspace: Optional[torch.Tensor] = None,
           out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None,
           stream=None, f4_index: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Exhaustive proxy-space kNN (uq_search): (scores [nq][k] int32, ids [nq][k] int64),
    best first under (Delta desc, id asc).  With ``f4_index`` (build_f4_index) the E2M1
    pair engine reads the pre-expanded index (uq_search_f4x)."""
    _dev(qcodes, "qcodes"); _dev(dbcodes, "dbcodes")
    nq, n = qcodes.shape[0], dbcodes.shape[0]
    dev = qcodes.device
    if out is None:
        out = (_empty(stream, (nq, k), dtype=torch.int32, device=dev),
               _empty(stream, (nq, k), dtype=torch.int64, device=dev))
    need = search_workspace(nq, n, d, k, ALGO_TC_FP4 if f4_index is not None else algo)
    if workspace is None or workspace.numel() < need:
        workspace = _empty(stream, max(need, 1), dtype=torch.uint8, device=dev)
    if f4_index is not None:
        _dev(f4_index, "f4_index")
        _check("uq_search_f4x", _L.uq_search_f4x(_ptr(qcodes), nq, _ptr(dbcodes), _ptr(f4_index), _index_bytes(f4_index), n, d, k, id_base,
                                                 _ptr(out[0]), _ptr(out[1]), _ptr(workspace), workspace.numel(),
                                                 _stream(stream)))
        return out
    _check("uq_search", _L.uq_search_ex(_ptr(qcodes), nq, _ptr(dbcodes), n, d, k, id_base,
                                        _ptr(out[0]), _ptr(out[1]), _ptr(workspace),
                                        workspace.numel(), algo, _stream(stream)))
    return out


def quantize_i8(u: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """int8 queries for single-operand search (uq_quantize_i8, R15): per row
    round-half-even(u * 127 / max|u|) in fp32 -> [n][d] int8."""
    _dev(u, "u")
    if u.dim() != 2 or u.stride(1) != 1 or u.dtype not in _DT:
        raise ValueError("u must be 2-D f32/f16/bf16 with unit column stride")
    n, d = u.shape
    if out is None:
        out = _empty(stream, (n, d), dtype=torch.int8, device=u.device)
    _check("uq_quantize_i8", _L.uq_quantize_i8(_ptr(u), _DT[u.dtype], n, d, u.stride(0), _ptr(out),
                                               out.stride(0), _stream(stream)))
    return out


def search_asym_workspace(nq: int, n: int, d: int, k: int) -> int:
    b = ctypes.c_size_t(0)
    _check("uq_search_asym_workspace", _L.uq_search_asym_workspace(nq, n, d, k, ctypes.byref(b)))
    return int(b.value)


def search_asym(q8: torch.Tensor, dbcodes: torch.Tensor, d: int, k: int, id_base: int = 0,
                workspace: Optional[torch.Tensor] = None,
                out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None,
                stream=None, i8_index: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Single-operand kNN (uq_search_asym): int8 queries q8 [nq][d]
    against ternary codes by masked addition; (scores int32, ids int64) [nq][k]."""
    _dev(q8, "q8"); _dev(dbcodes, "dbcodes")
    if q8.dtype != torch.int8 or q8.dim() != 2 or q8.stride(1) != 1:
        raise ValueError("q8 must be a 2-D int8 tensor with unit column stride")
    nq, n = q8.shape[0], dbcodes.shape[0]
    dev = q8.device
    if out is None:
        out = (_empty(stream, (nq, k), dtype=torch.int32, device=dev),
               _empty(stream, (nq, k), dtype=torch.int64, device=dev))
    need = search_asym_workspace(nq, n, d, k)
    if workspace is None or workspace.numel() < need:
        workspace = _empty(stream, max(need, 1), dtype=torch.uint8, device=dev)
    if i8_index is not None:
        _dev(i8_index, "i8_index")
        _check("uq_search_asym_x", _L.uq_search_asym_x(_ptr(q8), nq, q8.stride(0), _ptr(dbcodes), _ptr(i8_index), _index_bytes(i8_index), n,
                                                       d, k, id_base, _ptr(out[0]), _ptr(out[1]), _ptr(workspace),
                                                       workspace.numel(), _stream(stream)))
        return out
    _check("uq_search_asym", _L.uq_search_asym(_ptr(q8), nq, q8.stride(0), _ptr(dbcodes), n, d, k, id_base,
                                               _ptr(out[0]), _ptr(out[1]), _ptr(workspace),
                                               workspace.numel(), _stream(stream)))
    return out


def merge_topk(scores_g: torch.Tensor, ids_g: torch.Tensor, k: int,
               out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None,
               stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Merge [g][nq][k] candidate lists into the k best per query (uq_merge_topk)."""
    _dev(scores_g, "scores"); _dev(ids_g, "ids")
    g, nq, kin = scores_g.shape
    if kin != k:
        raise ValueError("lists must hold k entries per query")
    if out is None:
        out = (_empty(stream, (nq, k), dtype=torch.int32, device=scores_g.device),
               _empty(stream, (nq, k), dtype=torch.int64, device=scores_g.device))
    _check("uq_merge_topk", _L.uq_merge_topk(_ptr(scores_g), _ptr(ids_g), g, nq, k, _ptr(out[0]),
                                             _ptr(out[1]), _stream(stream)))
    return out


def merge_topk_ptrs(score_ptrs: torch.Tensor, id_ptrs: torch.Tensor, nq: int, k: int,
                    out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None,
                    stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """uq_merge_topk_ptrs: merge g lists given as DEVICE int64 tensors of base
    pointers (score_ptrs[r] -> int32 [nq][k], id_ptrs[r] -> int64 [nq][k]; peer-
    mapped buffers of other GPUs allowed) into the k best per query."""
    _dev(score_ptrs, "score_ptrs"); _dev(id_ptrs, "id_ptrs")
    if score_ptrs.dtype != torch.int64 or id_ptrs.dtype != torch.int64 or score_ptrs.numel() != id_ptrs.numel():
        raise ValueError("pointer arrays must be int64 device tensors of equal length")
    g = score_ptrs.numel()
    if out is None:
        out = (_empty(stream, (nq, k), dtype=torch.int32, device=score_ptrs.device),
               _empty(stream, (nq, k), dtype=torch.int64, device=score_ptrs.device))
    _check("uq_merge_topk_ptrs", _L.uq_merge_topk_ptrs(_ptr(score_ptrs), _ptr(id_ptrs), g, nq, k, _ptr(out[0]),
                                                       _ptr(out[1]), _stream(stream)))
    return out


def rerank(q: torch.Tensor, db: torch.Tensor, cand: torch.Tensor, k: int,
           out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None,
           stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """k@n (uq_rerank): re-rank each query's candidate ids cand [nq][n] by cosine on the
    float vectors q [nq][d] / db [N][d] (same dtype); (cos [nq][k] f32, ids [nq][k] int64)."""
    _dev(q, "q"); _dev(db, "db"); _dev(cand, "cand")
    if q.dtype != db.dtype or q.dtype not in _DT:
        raise TypeError("q and db must share a supported float dtype")
    if q.stride(1) != 1 or db.stride(1) != 1 or cand.dtype != torch.int64 or not cand.is_contiguous():
        raise ValueError("unit column stride vectors and contiguous int64 candidates expected")
    nq, d = q.shape
    n_cand = cand.shape[1]
    if out is None:
        out = (_empty(stream, (nq, k), dtype=torch.float32, device=q.device),
               _empty(stream, (nq, k), dtype=torch.int64, device=q.device))
    _check("uq_rerank", _L.uq_rerank(_ptr(q), _DT[q.dtype], nq, q.stride(0), _ptr(db), db.shape[0],
                                     db.stride(0), d, _ptr(cand), n_cand, k, _ptr(out[0]), _ptr(out[1]),
                                     _stream(stream)))
    return out


def check_codes(codes: torch.Tensor, d: int, stream=None) -> int:
    """Number of invalid code rows (uq_check_codes); synchronises to read the count."""
    _dev(codes, "codes")
    bad = _empty(stream, 1, dtype=torch.int64, device=codes.device)
    _check("uq_check_codes", _L.uq_check_codes(_ptr(codes), codes.shape[0], d, _ptr(bad),
                                               _stream(stream)))
    if stream is not None:
        stream.synchronize()
    return int(bad.item())
