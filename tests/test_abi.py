"""C-ABI checks that need no GPU: libuq.so loads, exports every symbol that
include/uq.h declares, and rejects bad arguments synchronously (before any
CUDA call)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "uq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(uq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2506_00528_b200 as uq
    return ctypes.CDLL(uq.lib_path())


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert "uq_search" in names and "uq_encode" in names and "uq_merge_topk" in names
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/uq.h but not exported"


def test_host_side_contract(L):
    L.uq_code_bytes.restype = ctypes.c_size_t
    assert L.uq_code_bytes(384) == 96 and L.uq_code_bytes(768) == 192
    assert L.uq_code_bytes(1024) == 256 and L.uq_code_bytes(1536) == 384
    assert L.uq_code_bytes(10) == 32 and L.uq_code_bytes(129) == 64 and L.uq_code_bytes(0) == 0
    L.uq_status_str.restype = ctypes.c_char_p
    assert L.uq_status_str(4) == b"UQ_ERR_WORKSPACE"


def test_invalid_arguments_rejected_synchronously(L):
    i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    L.uq_encode.argtypes = [vp, i32, i64, i32, i64, i32, vp, vp]
    fake = vp(0x1000)  # never dereferenced: validation fails first
    assert L.uq_encode(fake, 0, 10, 384, 384, 0, fake, None) == 1      # x < 1
    assert L.uq_encode(fake, 0, 10, 384, 384, 385, fake, None) == 1    # x > d
    assert L.uq_encode(fake, 0, 10, 384, 383, 192, fake, None) == 1    # ld < d
    assert L.uq_encode(fake, 0, 10, 4096, 4096, 10, fake, None) == 2   # d > UQ_MAX_D
    assert L.uq_encode(fake, 0, 0, 384, 384, 192, None, None) == 0     # empty: no-op
    L.uq_search_ex.argtypes = [vp, i64, vp, i64, i32, i32, i64, vp, vp, vp, ctypes.c_size_t, i32, vp]
    assert L.uq_search_ex(fake, 4, fake, 10, 384, 0, 0, fake, fake, fake, 0, 0, None) == 1   # k < 1
    assert L.uq_search_ex(fake, 4, fake, 10, 384, 2000, 0, fake, fake, fake, 0, 0, None) == 2  # k > max
    assert L.uq_search_ex(vp(0x1001), 4, fake, 10, 384, 5, 0, fake, fake, fake, 0, 0, None) == 1  # misaligned
    assert L.uq_search_ex(fake, 0, fake, 10, 384, 5, 0, None, None, None, 0, 0, None) == 0   # nq = 0
    L.uq_search_workspace_ex.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(ctypes.c_size_t)]
    b = ctypes.c_size_t(0)
    assert L.uq_search_workspace_ex(100, 10000, 384, 10, 1, ctypes.byref(b)) == 0 and b.value > 0
    assert L.uq_search_ex(fake, 100, fake, 10000, 384, 10, 0, fake, fake, vp(0x100000), 16, 1, None) == 4
    L.uq_merge_topk.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp]
    assert L.uq_merge_topk(fake, fake, -1, 4, 5, fake, fake, None) == 1
    L.uq_check_codes.argtypes = [vp, i64, i32, vp, vp]
    assert L.uq_check_codes(fake, 10, 384, None, None) == 1


def test_index_size_checked_synchronously(L):
    """uq_search_f4x / uq_search_asym_x reject an index whose byte size does not
    match (n, d): a stale index fails before any launch instead of being read
    out of bounds."""
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
    fake = vp(0x1000)
    L.uq_f4_index_bytes.argtypes, L.uq_f4_index_bytes.restype = [i64, i32], sz
    L.uq_i8_index_bytes.argtypes, L.uq_i8_index_bytes.restype = [i64, i32], sz
    L.uq_search_f4x.argtypes = [vp, i64, vp, vp, sz, i64, i32, i32, i64, vp, vp, vp, sz, vp]
    L.uq_search_asym_x.argtypes = [vp, i64, i64, vp, vp, sz, i64, i32, i32, i64, vp, vp, vp, sz, vp]
    n, d = 100000, 768
    good = L.uq_f4_index_bytes(n, d)
    assert good == (n + 239) // 240 * 240 * 6 * 64
    stale = L.uq_f4_index_bytes(n - 1000, d)
    assert L.uq_search_f4x(fake, 300, fake, fake, stale, n, d, 10, 0, fake, fake, fake, 1 << 30, None) == 1
    assert L.uq_search_f4x(fake, 300, fake, fake, good + 64, n, d, 10, 0, fake, fake, fake, 1 << 30, None) == 1
    assert L.uq_search_f4x(fake, 300, fake, None, good, n, d, 10, 0, fake, fake, fake, 1 << 30, None) == 1
    gi = L.uq_i8_index_bytes(n, d)
    assert gi == (n + 255) // 256 * 256 * 6 * 128
    assert L.uq_search_asym_x(fake, 300, d, fake, fake, gi - 1, n, d, 10, 0, fake, fake, fake, 1 << 30, None) == 1
