"""CPU oracle for the EVP ternary search path of arXiv 2506.00528.

TEST INFRASTRUCTURE ONLY: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` are the only callers.
The product package ``paper_2506_00528_b200`` never imports this module and
shares no code with it ("Oracle").

The arithmetic lives in ``uq_oracle.c`` (plain C, one function per paper step,
each citing its passage); this module is numpy/ctypes marshalling plus the
tiny-d brute-force helpers in ``bruteforce.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "uq_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, hardware POPCNT for bsp, OpenMP over rows/queries)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-mpopcnt", "-fopenmp", "-shared", "-fPIC", "-std=c11", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        L.orc_plane_bytes.restype = i64
        L.orc_plane_bytes.argtypes = [i32]
        L.orc_code_bytes.restype = i64
        L.orc_code_bytes.argtypes = [i32]
        L.orc_encode.argtypes = [vp, i64, i32, i64, i32, vp]
        L.orc_encode.restype = None
        L.orc_pack.argtypes = [vp, i64, i32, vp]
        L.orc_pack.restype = None
        L.orc_unpack.argtypes = [vp, i64, i32, vp]
        L.orc_unpack.restype = None
        L.orc_dot_naive.argtypes = [vp, vp, i32]
        L.orc_dot_naive.restype = i32
        L.orc_b2sp.argtypes = [vp, vp, i32]
        L.orc_b2sp.restype = i32
        L.orc_scores.argtypes = [vp, i64, vp, i64, i32, vp]
        L.orc_scores.restype = None
        L.orc_knn.argtypes = [vp, i64, vp, i64, i32, i32, i64, vp, vp]
        L.orc_knn.restype = None
        L.orc_cosine_knn.argtypes = [vp, i64, vp, i64, i32, i32, vp, vp]
        L.orc_cosine_knn.restype = None
        L.orc_check_codes.argtypes = [vp, i64, i32]
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_rerank.argtypes = [vp, i64, vp, i64, i32, vp, i32, i32, vp, vp]
        L.orc_quantize_i8.argtypes = [vp, i64, i32, vp]
        L.orc_quantize_i8.restype = None
        L.orc_knn_asym.argtypes = [vp, i64, vp, i64, i32, i32, i64, vp, vp]
        L.orc_knn_asym.restype = None
        L.orc_rerank.restype = None
        L.orc_set_threads.restype = ctypes.c_int
        L.orc_check_codes.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def plane_bytes(d: int) -> int:
    return int(lib().orc_plane_bytes(d))


def code_bytes(d: int) -> int:
    return int(lib().orc_code_bytes(d))


def _as_f64_rows(u) -> np.ndarray:
    """Exact widening of f16/f32 inputs to f64 (order of |u| is preserved exactly)."""
    u = np.asarray(u)
    if u.dtype not in (np.float16, np.float32, np.float64):
        raise TypeError(f"unsupported dtype {u.dtype}")
    return np.ascontiguousarray(u.astype(np.float64))


def encode(u, x: int) -> np.ndarray:
    """Ternary nearest-vertex codes [n][d] int8."""
    u64 = _as_f64_rows(u)
    if u64.ndim == 1:
        u64 = u64[None, :]
    n, d = u64.shape
    if not (1 <= x <= d):
        raise ValueError("x must be in [1, d] (P:139)")
    v = np.zeros((n, d), dtype=np.int8)
    lib().orc_encode(_p(u64), n, d, d, x, _p(v))
    return v


def pack(v) -> np.ndarray:
    """Packed (pos | neg) planes [n][code_bytes] uint8."""
    v = np.ascontiguousarray(np.asarray(v, dtype=np.int8))
    if v.ndim == 1:
        v = v[None, :]
    n, d = v.shape
    out = np.zeros((n, code_bytes(d)), dtype=np.uint8)
    lib().orc_pack(_p(v), n, d, _p(out))
    return out


def unpack(codes, d: int) -> np.ndarray:
    codes = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
    if codes.ndim == 1:
        codes = codes[None, :]
    n = codes.shape[0]
    v = np.zeros((n, d), dtype=np.int8)
    lib().orc_unpack(_p(codes), n, d, _p(v))
    return v


def dot_naive(a, b) -> int:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int8))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.int8))
    assert a.shape == b.shape and a.ndim == 1
    return int(lib().orc_dot_naive(_p(a), _p(b), a.shape[0]))


def b2sp(ca, cb, d: int) -> int:
    ca = np.ascontiguousarray(np.asarray(ca, dtype=np.uint8))
    cb = np.ascontiguousarray(np.asarray(cb, dtype=np.uint8))
    return int(lib().orc_b2sp(_p(ca), _p(cb), d))


def scores(qcodes, dbcodes, d: int) -> np.ndarray:
    qc = np.ascontiguousarray(qcodes, dtype=np.uint8)
    dc = np.ascontiguousarray(dbcodes, dtype=np.uint8)
    nq, n = qc.shape[0], dc.shape[0]
    out = np.zeros((nq, n), dtype=np.int32)
    lib().orc_scores(_p(qc), nq, _p(dc), n, d, _p(out))
    return out


def knn(qcodes, dbcodes, d: int, k: int, id_base: int = 0):
    """Exhaustive proxy-space kNN: (scores[nq][k] int32, ids[nq][k] int64)."""
    qc = np.ascontiguousarray(qcodes, dtype=np.uint8)
    dc = np.ascontiguousarray(dbcodes, dtype=np.uint8)
    nq, n = qc.shape[0], dc.shape[0]
    s = np.zeros((nq, k), dtype=np.int32)
    ids = np.zeros((nq, k), dtype=np.int64)
    lib().orc_knn(_p(qc), nq, _p(dc), n, d, k, id_base, _p(s), _p(ids))
    return s, ids


def quantize_i8(u) -> np.ndarray:
    """Query quantisation to int8 (R15): per row, fp32 scale 127/max|u|,
    round half to even, fp32 arithmetic.  f16 / bf16 inputs widen exactly to f32."""
    u = np.asarray(u)
    if u.dtype not in (np.float16, np.float32):
        raise TypeError("quantize_i8 takes f16 / f32 rows (widened exactly to f32)")
    u32 = np.ascontiguousarray(u.astype(np.float32))
    if u32.ndim == 1:
        u32 = u32[None, :]
    n, d = u32.shape
    out = np.zeros((n, d), dtype=np.int8)
    lib().orc_quantize_i8(_p(u32), n, d, _p(out))
    return out


def knn_asym(q8, dbcodes, d: int, k: int, id_base: int = 0):
    """Single-operand kNN: int8 query x packed ternary rows by masked
    addition; (scores[nq][k] int32, ids[nq][k] int64), (score desc, id asc)."""
    q = np.ascontiguousarray(q8, dtype=np.int8)
    dc = np.ascontiguousarray(dbcodes, dtype=np.uint8)
    nq, n = q.shape[0], dc.shape[0]
    assert q.shape[1] == d
    s = np.zeros((nq, k), dtype=np.int32)
    ids = np.zeros((nq, k), dtype=np.int64)
    lib().orc_knn_asym(_p(q), nq, _p(dc), n, d, k, id_base, _p(s), _p(ids))
    return s, ids


def cosine_knn(qv, dv, k: int):
    """fp64 cosine ground truth: (cos[nq][k] f64, ids[nq][k] int64)."""
    q = _as_f64_rows(qv)
    db = _as_f64_rows(dv)
    nq, d = q.shape
    n = db.shape[0]
    s = np.zeros((nq, k), dtype=np.float64)
    ids = np.zeros((nq, k), dtype=np.int64)
    lib().orc_cosine_knn(_p(q), nq, _p(db), n, d, k, _p(s), _p(ids))
    return s, ids


def rerank(qv, dv, cand, k: int):
    """k@n re-rank in fp64: cosine of each candidate id, (cos desc, id asc),
    top k: (cos[nq][k] f64, ids[nq][k] int64)."""
    q = _as_f64_rows(qv)
    db = _as_f64_rows(dv)
    c = np.ascontiguousarray(cand, dtype=np.int64)
    nq, d = q.shape
    s = np.zeros((nq, k), dtype=np.float64)
    ids = np.zeros((nq, k), dtype=np.int64)
    lib().orc_rerank(_p(q), nq, _p(db), db.shape[0], d, _p(c), c.shape[1], k, _p(s), _p(ids))
    return s, ids


def check_codes(codes, d: int) -> int:
    c = np.ascontiguousarray(codes, dtype=np.uint8)
    return int(lib().orc_check_codes(_p(c), c.shape[0], d))


def set_threads(n: int) -> int:
    """Timing harness: worker threads of the oracle's OpenMP loops (returns the previous count)."""
    return int(lib().orc_set_threads(n))
