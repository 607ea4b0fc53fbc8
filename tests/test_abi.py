"""C-ABI boundary checks that need no GPU (-m "not gpu").

The library must build for sm_100a, load, export every symbol include/ozaki.h
declares, and reject invalid BLAS arguments with xerbla-style codes BEFORE any
device work (so these calls are safe on a CPU-only box).
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2603_29975_b200 import _build, lib
    _build.build()
    return lib()


def _declared():
    with open(os.path.join(ROOT, "include", "ozaki.h")) as fh:
        src = fh.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ozaki_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(L):
    names = _declared()
    assert len(names) >= 14
    for nm in names:
        assert hasattr(L, nm), nm
    # and they are real dynamic symbols of the .so
    out = os.popen(f"nm -D --defined-only {L._name}").read()
    for nm in names:
        assert re.search(rf"\bT {nm}\b", out), nm


def test_sass_is_tcgen05(L):
    """The GEMM is tensor-core tcgen05 code (UTC*MMA), fed by bulk async copies."""
    out = os.popen(f"cuobjdump -sass {L._name}").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "UTCIMMA" in out
    assert "UBLKCP" in out
    assert "LDTM" in out


def _dg(L, ta=b"N", tb=b"N", m=4, n=4, k=4, lda=4, ldb=4, ldc=4, s=4):
    return L.ozaki_dgemm(ta, tb, m, n, k, 1.0, None, lda, None, ldb, 0.0, None, ldc, s)


def test_xerbla_codes_real(L):
    assert _dg(L, ta=b"X") == -1
    assert _dg(L, tb=b"Q") == -2
    assert _dg(L, m=-1) == -3
    assert _dg(L, n=-1) == -4
    assert _dg(L, k=-1) == -5
    assert _dg(L, lda=3) == -8            # 'N': lda >= m
    assert _dg(L, ta=b"T", m=4, k=6, lda=5) == -8   # 'T': lda >= k
    assert _dg(L, ldb=3) == -10
    assert _dg(L, ldc=3) == -13
    assert _dg(L, s=0) == -14
    assert _dg(L, s=17) == -14
    # quick returns need no device and write nothing
    assert _dg(L, m=0, lda=1, ldc=1) == 0
    assert _dg(L, n=0) == 0
    msg = L.ozaki_last_error()
    assert isinstance(msg, bytes)


def test_xerbla_codes_batched_and_complex(L):
    al = (ctypes.c_double * 2)(1.0, 0.0)
    rc = L.ozaki_zgemm_strided_batched(b"N", b"N", 4, 4, 4, al, None, 4, 16, None, 4, 16, al, None,
                                       4, 16, -1, 4)
    assert rc == -17
    rc = L.ozaki_zgemm_strided_batched(b"N", b"N", 4, 4, 4, al, None, 4, 16, None, 2, 16, al, None,
                                       4, 16, 2, 4)
    assert rc == -11
    rc = L.ozaki_zgemm_strided_batched(b"N", b"N", 4, 4, 4, al, None, 4, 16, None, 4, 16, al, None,
                                       4, 16, 2, 99)
    assert rc == -18
    rc = L.ozaki_zgemm(b"C", b"N", 4, 4, 4, al, None, 4, None, 4, al, None, 2, 4)
    assert rc == -13


def test_workspace_size_closed_form(L):
    from paper_2603_29975_b200 import workspace_size
    # real: s*(tiles_m*128 + tiles_n*BN)*round_up(k,32) + 4(m+n), each part 256-B aligned
    ws = workspace_size("d", 256, 128, 100, 1, 4)
    assert ws == 4 * 256 * 128 + 4 * 128 * 128 + 1024 + 512
    assert workspace_size("d", 1, 1, 1, 1, 0) == -1
    # s*k_eff beyond the INT32 level-sum bound (reading R8) is K-chunked, not refused
    assert workspace_size("d", 8, 8, 20000, 1, 8) > 0


def test_trsm_xerbla_codes_before_device_work():
    """ozaki_dtrsm / ozaki_ztrsm argument checks (BLAS parameter numbers) return before any
    device work (no GPU needed), and the block-size setter rejects nb < 1."""
    import ctypes
    import paper_2603_29975_b200 as oz
    L = oz.lib()
    buf = (ctypes.c_double * 64)()
    z = (ctypes.c_double * 2)(1.0, 0.0)
    p = ctypes.cast(buf, ctypes.c_void_p)
    d = lambda *a: L.ozaki_dtrsm(*a)  # noqa: E731
    assert d(b"X", b"L", b"N", b"N", 4, 4, 1.0, p, 4, p, 4, 7) == -1
    assert d(b"L", b"X", b"N", b"N", 4, 4, 1.0, p, 4, p, 4, 7) == -2
    assert d(b"L", b"L", b"X", b"N", 4, 4, 1.0, p, 4, p, 4, 7) == -3
    assert d(b"L", b"L", b"N", b"X", 4, 4, 1.0, p, 4, p, 4, 7) == -4
    assert d(b"L", b"L", b"N", b"N", -1, 4, 1.0, p, 4, p, 4, 7) == -5
    assert d(b"L", b"L", b"N", b"N", 4, -1, 1.0, p, 4, p, 4, 7) == -6
    assert d(b"L", b"L", b"N", b"N", 4, 2, 1.0, p, 3, p, 4, 7) == -9
    assert d(b"R", b"L", b"N", b"N", 4, 2, 1.0, p, 1, p, 4, 7) == -9
    assert d(b"L", b"L", b"N", b"N", 4, 2, 1.0, p, 4, p, 3, 7) == -11
    assert d(b"L", b"L", b"N", b"N", 4, 2, 1.0, p, 4, p, 4, 17) == -12
    assert L.ozaki_ztrsm(b"L", b"U", b"C", b"U", 4, 4, z, p, 4, p, 2, 7) == -11
    assert d(b"L", b"L", b"N", b"N", 0, 4, 1.0, p, 4, p, 4, 7) == 0      # quick return, no device
    assert L.ozaki_set_trsm_block(0) == -1
    assert L.ozaki_set_trsm_block(64) == 0 and L.ozaki_get_trsm_block() == 64
    L.ozaki_set_trsm_block(128)
