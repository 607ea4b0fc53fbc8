"""ozaki-b200: INT8 Ozaki-I emulation of FP64 DGEMM/ZGEMM on B200 (sm_100a).

Thin Python binding over the C ABI in ``include/ozaki.h`` (``libozaki.so``,
built in-tree by ``_build.py``).  The binding only marshals arguments: every
step of the method runs in the library's CUDA kernels.  There is no CPU
fallback -- importing this package on a machine without the built library, or
calling it on a non-sm_100 device, raises.

Matrix convention: BLAS column-major.  A torch tensor ``X`` of shape
(rows, cols) is passed as-is when ``X.stride(0) == 1`` (column-major, leading
dimension ``X.stride(1)``); use :func:`colmajor` to obtain such a tensor.
Batched tensors are (batch, rows, cols) with ``stride(1) == 1``.
"""
from __future__ import annotations

import ctypes
import os
import threading

__all__ = [
    "OzakiError", "lib", "dgemm", "zgemm", "zgemm3m", "dgemm_strided_batched",
    "zgemm_strided_batched", "zgemm3m_strided_batched", "set_stream", "get_stats",
    "reset_stats", "workspace_size", "debug_split", "debug_level_sums", "colmajor",
    "version", "pairs", "LIB_PATH", "profile_enable", "profile_read", "dtrsm", "ztrsm",
    "set_trsm_block", "get_trsm_block",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libozaki.so")
_lib = None


class OzakiError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: code {code}: {msg}")
        self.code = code


class Profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 4), ("launches", ctypes.c_uint64 * 4)]


PHASES = ("k1_exponent", "k1_slice", "k2_gemm", "other")


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "dgemm_calls", "zgemm_calls", "zgemm3m_calls", "batch_entries", "int8_gemm_equiv",
        "int8_macs", "k_chunks", "nonfinite_rows", "kernel_launches", "crt_calls")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def lib():
    """Load libozaki.so (build it first if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        try:
            from . import _build
            _build.build()
        except Exception as exc:  # noqa: BLE001
            raise ImportError(f"libozaki.so missing and could not be built: {exc}") from exc
    L = ctypes.CDLL(LIB_PATH)
    c, i64, i32, dbl, p = ctypes.c_char, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    dP = ctypes.POINTER(ctypes.c_double)
    L.ozaki_dgemm.argtypes = [c, c, i64, i64, i64, dbl, p, i64, p, i64, dbl, p, i64, i32]
    L.ozaki_zgemm.argtypes = [c, c, i64, i64, i64, dP, p, i64, p, i64, dP, p, i64, i32]
    L.ozaki_zgemm3m.argtypes = L.ozaki_zgemm.argtypes
    L.ozaki_dgemm_strided_batched.argtypes = [c, c, i64, i64, i64, dbl, p, i64, i64, p, i64, i64,
                                              dbl, p, i64, i64, i64, i32]
    L.ozaki_zgemm_strided_batched.argtypes = [c, c, i64, i64, i64, dP, p, i64, i64, p, i64, i64,
                                              dP, p, i64, i64, i64, i32]
    L.ozaki_zgemm3m_strided_batched.argtypes = L.ozaki_zgemm_strided_batched.argtypes
    L.ozaki_set_overlap.argtypes = [i32]
    L.ozaki_set_overlap.restype = i32
    L.ozaki_get_overlap.argtypes = []
    L.ozaki_get_overlap.restype = i32
    L.ozaki_set_exponent_block.argtypes = [i64]
    L.ozaki_set_exponent_block.restype = i32
    L.ozaki_get_exponent_block.argtypes = []
    L.ozaki_get_exponent_block.restype = i64
    if hasattr(L, "ozaki_dtrsm"):   # (a library built before round 2 lacks the TRSM entry points)
        L.ozaki_dtrsm.argtypes = [c, c, c, c, i64, i64, dbl, p, i64, p, i64, i32]
        L.ozaki_ztrsm.argtypes = [c, c, c, c, i64, i64, dP, p, i64, p, i64, i32]
        L.ozaki_set_trsm_block.argtypes = [i64]
        L.ozaki_set_trsm_block.restype = i32
        L.ozaki_get_trsm_block.argtypes = []
        L.ozaki_get_trsm_block.restype = i64
    L.ozaki_set_pair_set.argtypes = [i32]
    L.ozaki_set_pair_set.restype = i32
    L.ozaki_get_pair_set.argtypes = []
    L.ozaki_get_pair_set.restype = i32
    L.ozaki2_dgemm.argtypes = L.ozaki_dgemm.argtypes
    L.ozaki2_zgemm.argtypes = L.ozaki_zgemm.argtypes
    L.ozaki2_dgemm_strided_batched.argtypes = L.ozaki_dgemm_strided_batched.argtypes
    L.ozaki2_zgemm_strided_batched.argtypes = L.ozaki_zgemm_strided_batched.argtypes
    for fn in (L.ozaki2_dgemm, L.ozaki2_zgemm, L.ozaki2_dgemm_strided_batched, L.ozaki2_zgemm_strided_batched):
        fn.restype = i32
    for f in ("ozaki_dgemm", "ozaki_zgemm", "ozaki_zgemm3m", "ozaki_dgemm_strided_batched",
              "ozaki_zgemm_strided_batched", "ozaki_zgemm3m_strided_batched"):
        getattr(L, f).restype = i32
    L.ozaki_set_stream.argtypes = [p]
    L.ozaki_set_stream.restype = i32
    L.ozaki_get_stream.restype = p
    L.ozaki_get_stats.argtypes = [ctypes.POINTER(Stats)]
    L.ozaki_get_stats.restype = i32
    L.ozaki_reset_stats.restype = i32
    L.ozaki_workspace_size.argtypes = [c, i64, i64, i64, i64, i32]
    L.ozaki_workspace_size.restype = i64
    L.ozaki_last_error.restype = ctypes.c_char_p
    L.ozaki_version.restype = ctypes.c_char_p
    L.ozaki_profile_enable.argtypes = [i32]
    L.ozaki_profile_enable.restype = i32
    L.ozaki_profile_read.argtypes = [ctypes.POINTER(Profile)]
    L.ozaki_profile_read.restype = i32
    L.ozaki_debug_split.argtypes = [c, c, c, i64, i64, p, i64, i32, p, p, ctypes.POINTER(i64)]
    L.ozaki_debug_split.restype = i32
    L.ozaki_debug_level_sums.argtypes = [c, c, i64, i64, i64, p, i64, p, i64, i32, p]
    L.ozaki_debug_level_sums.restype = i32
    L.ozaki_debug_timing.argtypes = [i32, ctypes.POINTER(ctypes.c_uint64), i32]
    L.ozaki_debug_timing.restype = i32
    _lib = L
    return L


def version() -> str:
    return lib().ozaki_version().decode()


def pairs(s: int) -> int:
    return s * (s + 1) // 2


def _check(rc: int, where: str):
    if rc != 0:
        raise OzakiError(rc, where, lib().ozaki_last_error().decode())


def _ch(t: str) -> bytes:
    return t.encode()[:1]


# ------------------------------------------------------------------ plumbing
def colmajor(x):
    """Return a column-major (Fortran-order) copy/view of a 2-D or batched tensor."""
    import torch
    if x.dim() == 2:
        return x.t().contiguous().t() if x.stride(0) != 1 else x
    if x.dim() == 3:
        return x.transpose(1, 2).contiguous().transpose(1, 2) if x.stride(1) != 1 else x
    raise ValueError("expected a 2-D or 3-D tensor")


def _ld(x) -> int:
    rows, cols = x.shape[-2], x.shape[-1]
    if x.numel() == 0:
        return max(1, rows)
    if rows > 1 and x.stride(-2) != 1:
        raise ValueError("matrix must be column-major (stride(-2) == 1); use colmajor()")
    return max(1, x.stride(-1) if cols > 1 else rows)


def _cuda(x, dtype, name):
    """Operands are CUDA tensors, or CPU tensors (host offload: all of A, B, C)."""
    import torch
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if x.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {x.dtype}")
    return x


def _operands(dtype, A, B, C):
    """Type checks; resolves lazy conj / neg views of A and B (torch keeps them as a bit on the
    tensor, the library would read the unconjugated storage); C must be a plain tensor.  CUDA
    operands share one device (all-CPU operands take the host offload).  Returns (A, B, device)."""
    for x, nm in ((A, "A"), (B, "B"), (C, "C")):
        _cuda(x, dtype, nm)
    if C.is_conj() or C.is_neg():
        raise ValueError("C must not be a lazily conjugated / negated view (resolve it first)")
    # (resolving materialises a copy, which torch lays out row-major: make it column-major again)
    A = colmajor(A.resolve_conj().resolve_neg()) if (A.is_conj() or A.is_neg()) else A
    B = colmajor(B.resolve_conj().resolve_neg()) if (B.is_conj() or B.is_neg()) else B
    cuda = {x.device for x in (A, B, C) if x.device.type == "cuda"}
    if len(cuda) > 1:
        raise ValueError(f"A, B and C must live on one CUDA device, got {sorted(map(str, cuda))}")
    # host / device mixes are refused by the library itself (OZAKI_ERR_UNSUPPORTED)
    return A, B, (next(iter(cuda)) if cuda else C.device)


_NULLCTX = None
_bound = threading.local()      # last stream handle passed to ozaki_set_stream by this thread


def _on(device):
    """Device guard for one library call: the library works on the current CUDA device
    (no guard when the operands already live on it)."""
    global _NULLCTX
    import contextlib
    import torch
    if _NULLCTX is None:
        _NULLCTX = contextlib.nullcontext()
    if device is None or device.type != "cuda" or device.index is None or \
            device.index == torch.cuda.current_device():
        return _NULLCTX
    return torch.cuda.device(device)


_raw_stream = None   # torch's raw current-stream query (no Stream object per call), if present


def _current_stream_handle(device):
    import torch
    global _raw_stream
    if _raw_stream is None:
        _raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", False)
    idx = device.index if (device is not None and device.type == "cuda" and device.index is not None) \
        else torch.cuda.current_device()
    if _raw_stream:
        return int(_raw_stream(idx))
    return torch.cuda.current_stream(idx).cuda_stream


def _bind_stream(stream=None, device=None):
    import torch
    if stream is None and not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the Ozaki library has no CPU path")
    h = _current_stream_handle(device) if stream is None else stream.cuda_stream
    if getattr(_bound, "h", None) != h:      # the library's stream is thread-local too
        lib().ozaki_set_stream(ctypes.c_void_p(h))
        _bound.h = h


def _dims(transa, transb, A, B):
    ta, tb = transa.upper(), transb.upper()
    m, k = (A.shape[-2], A.shape[-1]) if ta == "N" else (A.shape[-1], A.shape[-2])
    kb, n = (B.shape[-2], B.shape[-1]) if tb == "N" else (B.shape[-1], B.shape[-2])
    if k != kb:
        raise ValueError(f"inner dimensions differ: op(A) is {m}x{k}, op(B) is {kb}x{n}")
    return m, n, k


_cpairs = {}


def _cpair(z):
    """(re, im) as a C double[2]; the arrays of recently used values are reused (read-only)."""
    import math
    z = complex(z)
    key = (z.real, z.imag, math.copysign(1.0, z.real), math.copysign(1.0, z.imag))   # -0.0 != +0.0
    a = _cpairs.get(key)
    if a is None:
        if len(_cpairs) > 64:
            _cpairs.clear()
        a = _cpairs[key] = (ctypes.c_double * 2)(z.real, z.imag)
    return a


# ------------------------------------------------------------------ GEMMs
def dgemm(transa, transb, alpha, A, B, beta, C, num_slices, stream=None):
    """C <- alpha op(A) op(B) + beta C, emulated with ``num_slices`` INT8 slices."""
    import torch
    A, B, dev = _operands(torch.float64, A, B, C)
    m, n, k = _dims(transa, transb, A, B)
    if tuple(C.shape) != (m, n):
        raise ValueError(f"C must be {m}x{n}")
    with _on(dev):
        _bind_stream(stream, dev)
        rc = lib().ozaki_dgemm(_ch(transa), _ch(transb), m, n, k, float(alpha), A.data_ptr(), _ld(A),
                               B.data_ptr(), _ld(B), float(beta), C.data_ptr(), _ld(C), int(num_slices))
    _check(rc, "ozaki_dgemm")
    return C


def _zgemm(fn, transa, transb, alpha, A, B, beta, C, num_slices, stream):
    import torch
    A, B, dev = _operands(torch.complex128, A, B, C)
    m, n, k = _dims(transa, transb, A, B)
    if tuple(C.shape) != (m, n):
        raise ValueError(f"C must be {m}x{n}")
    with _on(dev):
        _bind_stream(stream, dev)
        rc = fn(_ch(transa), _ch(transb), m, n, k, _cpair(alpha), A.data_ptr(), _ld(A), B.data_ptr(),
                _ld(B), _cpair(beta), C.data_ptr(), _ld(C), int(num_slices))
    _check(rc, fn.__name__)
    return C


def zgemm(transa, transb, alpha, A, B, beta, C, num_slices, stream=None):
    """Complex GEMM through the 4M real embedding (one INT8 GEMM of 2m x 2k x n)."""
    return _zgemm(lib().ozaki_zgemm, transa, transb, alpha, A, B, beta, C, num_slices, stream)


def zgemm3m(transa, transb, alpha, A, B, beta, C, num_slices, stream=None):
    """Complex GEMM through 3M (three emulated real products)."""
    return _zgemm(lib().ozaki_zgemm3m, transa, transb, alpha, A, B, beta, C, num_slices, stream)


def _batched(fn, dtype, transa, transb, alpha, A, B, beta, C, num_slices, stream, cplx):
    A, B, dev = _operands(dtype, A, B, C)
    for x, nm in ((A, "A"), (B, "B"), (C, "C")):
        if x.dim() != 3:
            raise ValueError(f"{nm} must be (batch, rows, cols)")
    batch = A.shape[0]
    if B.shape[0] != batch or C.shape[0] != batch:
        raise ValueError("batch sizes differ")
    m, n, k = _dims(transa, transb, A, B)
    if tuple(C.shape[1:]) != (m, n):
        raise ValueError(f"C entries must be {m}x{n}")
    al = _cpair(alpha) if cplx else float(alpha)
    be = _cpair(beta) if cplx else float(beta)
    sA = A.stride(0) if batch > 1 else 0
    sB = B.stride(0) if batch > 1 else 0
    sC = C.stride(0) if batch > 1 else 0
    with _on(dev):
        _bind_stream(stream, dev)
        rc = fn(_ch(transa), _ch(transb), m, n, k, al, A.data_ptr(), _ld(A), sA, B.data_ptr(), _ld(B),
                sB, be, C.data_ptr(), _ld(C), sC, batch, int(num_slices))
    _check(rc, fn.__name__)
    return C


def dgemm_strided_batched(transa, transb, alpha, A, B, beta, C, num_slices, stream=None):
    import torch
    return _batched(lib().ozaki_dgemm_strided_batched, torch.float64, transa, transb, alpha, A, B,
                    beta, C, num_slices, stream, False)


def zgemm_strided_batched(transa, transb, alpha, A, B, beta, C, num_slices, stream=None):
    import torch
    return _batched(lib().ozaki_zgemm_strided_batched, torch.complex128, transa, transb, alpha, A,
                    B, beta, C, num_slices, stream, True)


def zgemm3m_strided_batched(transa, transb, alpha, A, B, beta, C, num_slices, stream=None):
    import torch
    return _batched(lib().ozaki_zgemm3m_strided_batched, torch.complex128, transa, transb, alpha,
                    A, B, beta, C, num_slices, stream, True)


# ------------------------------------------------- Ozaki-II (CRT), NEXT-1
def ozaki2_dgemm(transa, transb, alpha, A, B, beta, C, num_moduli, stream=None):
    """C <- alpha op(A) op(B) + beta C via Ozaki-II with ``num_moduli`` moduli (R16..R20)."""
    import torch
    A, B, dev = _operands(torch.float64, A, B, C)
    m, n, k = _dims(transa, transb, A, B)
    if tuple(C.shape) != (m, n):
        raise ValueError(f"C must be {m}x{n}")
    with _on(dev):
        _bind_stream(stream, dev)
        rc = lib().ozaki2_dgemm(_ch(transa), _ch(transb), m, n, k, float(alpha), A.data_ptr(), _ld(A),
                                B.data_ptr(), _ld(B), float(beta), C.data_ptr(), _ld(C), int(num_moduli))
    _check(rc, "ozaki2_dgemm")
    return C


def ozaki2_zgemm(transa, transb, alpha, A, B, beta, C, num_moduli, stream=None):
    """Complex Ozaki-II through the 4M real embedding (k_eff = 2k)."""
    return _zgemm(lib().ozaki2_zgemm, transa, transb, alpha, A, B, beta, C, num_moduli, stream)


def ozaki2_dgemm_strided_batched(transa, transb, alpha, A, B, beta, C, num_moduli, stream=None):
    import torch
    return _batched(lib().ozaki2_dgemm_strided_batched, torch.float64, transa, transb, alpha, A, B,
                    beta, C, num_moduli, stream, False)


def ozaki2_zgemm_strided_batched(transa, transb, alpha, A, B, beta, C, num_moduli, stream=None):
    import torch
    return _batched(lib().ozaki2_zgemm_strided_batched, torch.complex128, transa, transb, alpha, A,
                    B, beta, C, num_moduli, stream, True)


# ------------------------------------------------- emulated TRSM (R23, NEXT-4c)
def _trsm(fn, dtype, side, uplo, transa, diag, alpha, A, B, num_slices, stream, cplx):
    import torch
    for x, nm in ((A, "A"), (B, "B")):
        _cuda(x, dtype, nm)
    if B.is_conj() or B.is_neg():
        raise ValueError("B must not be a lazily conjugated / negated view (resolve it first)")
    if A.is_conj() or A.is_neg():
        A = colmajor(A.resolve_conj().resolve_neg())
    if A.device != B.device and A.device.type == "cuda" and B.device.type == "cuda":
        raise ValueError("A and B must live on one CUDA device")
    m, n = B.shape
    dim = m if side.upper() == "L" else n
    if tuple(A.shape) != (dim, dim):
        raise ValueError(f"A must be {dim}x{dim}")
    dev = A.device if A.device.type == "cuda" else B.device
    with _on(dev):
        _bind_stream(stream, dev)
        al = _cpair(alpha) if cplx else float(alpha)
        rc = fn(_ch(side), _ch(uplo), _ch(transa), _ch(diag), m, n, al, A.data_ptr(), _ld(A), B.data_ptr(),
                _ld(B), int(num_slices))
    _check(rc, fn.__name__)
    return B


def dtrsm(side, uplo, transa, diag, alpha, A, B, num_slices, stream=None):
    """B <- X with op(A) X = alpha B (side 'L') or X op(A) = alpha B ('R'), emulated (R23)."""
    import torch
    return _trsm(lib().ozaki_dtrsm, torch.float64, side, uplo, transa, diag, alpha, A, B, num_slices,
                 stream, False)


def ztrsm(side, uplo, transa, diag, alpha, A, B, num_slices, stream=None):
    """Complex emulated TRSM (R23), updates through the 4M ZGEMM."""
    import torch
    return _trsm(lib().ozaki_ztrsm, torch.complex128, side, uplo, transa, diag, alpha, A, B, num_slices,
                 stream, True)


def set_trsm_block(nb: int) -> None:
    """Block size nb of the emulated TRSM for this thread (R23, default 128)."""
    _check(lib().ozaki_set_trsm_block(int(nb)), "ozaki_set_trsm_block")


def get_trsm_block() -> int:
    return int(lib().ozaki_get_trsm_block())


# ------------------------------------------------------------- utilities
def set_pair_set(kind: str) -> None:
    """Ozaki-I pair set for this thread: 'triangular' (R1, default) or 'full' (R21, NEXT-4)."""
    if kind not in ("triangular", "full"):
        raise ValueError(kind)
    lib().ozaki_set_pair_set(1 if kind == "full" else 0)


def get_pair_set() -> str:
    return "full" if lib().ozaki_get_pair_set() else "triangular"


def set_exponent_block(kb: int) -> None:
    """Per-block exponent alignment along K for this thread (R22, NEXT-4); 0 = per row/column."""
    _check(lib().ozaki_set_exponent_block(int(kb)), "ozaki_set_exponent_block")


def get_exponent_block() -> int:
    return int(lib().ozaki_get_exponent_block())


def set_overlap(on: bool) -> None:
    """ozaki_set_overlap: overlap consecutive Ozaki-I calls on one stream (include/ozaki.h)."""
    _check(lib().ozaki_set_overlap(1 if on else 0), "ozaki_set_overlap")


def get_overlap() -> bool:
    return bool(lib().ozaki_get_overlap())


def set_stream(stream) -> None:
    h = getattr(stream, "cuda_stream", stream) or 0
    lib().ozaki_set_stream(ctypes.c_void_p(h))
    _bound.h = h


def get_stats() -> dict:
    st = Stats()
    _check(lib().ozaki_get_stats(ctypes.byref(st)), "ozaki_get_stats")
    return st.as_dict()


def reset_stats() -> None:
    lib().ozaki_reset_stats()


def profile_enable(on: bool = True) -> None:
    """Bracket every library kernel with CUDA events (per-phase device time)."""
    lib().ozaki_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """Per-phase device ms and launch counts since the last read (synchronises)."""
    pr = Profile()
    _check(lib().ozaki_profile_read(ctypes.byref(pr)), "ozaki_profile_read")
    return {ph: {"ms": float(pr.ms[i]), "launches": int(pr.launches[i])} for i, ph in enumerate(PHASES)}


def workspace_size(kind: str, m: int, n: int, k: int, batch: int, num_slices: int) -> int:
    return int(lib().ozaki_workspace_size(_ch(kind), m, n, k, batch, num_slices))


def debug_split(side, kind, trans, X, num_slices, stream=None):
    """Run K1 on one operand; returns (slices[s][rows_out][kdepth] int8, exps int32).

    side 'A': rows of op(X); side 'B': columns of op(X).  kind 'd' real,
    'z' 4M embedding, 'r'/'i'/'s' 3M operands.  See include/ozaki.h."""
    import torch
    cplx = kind != "d"
    _cuda(X, torch.complex128 if cplx else torch.float64, "X")
    t = trans.upper()
    if side.upper() == "A":
        rows, cols = (X.shape[0], X.shape[1]) if t == "N" else (X.shape[1], X.shape[0])
    else:
        rows, cols = (X.shape[1], X.shape[0]) if t == "N" else (X.shape[0], X.shape[1])
    rows_out = 2 * rows if (kind == "z" and side.upper() == "B") else rows
    kdepth = cols if kind != "z" else 2 * ((cols + 31) // 32 * 32)
    s = int(num_slices)
    sl = torch.empty((s, rows_out, kdepth), dtype=torch.int8, device=X.device)
    ex = torch.empty((rows_out,), dtype=torch.int32, device=X.device)
    kd = ctypes.c_int64(0)
    if X.is_conj() or X.is_neg():
        X = colmajor(X.resolve_conj().resolve_neg())
    with _on(X.device):
        _bind_stream(stream, X.device)
        rc = lib().ozaki_debug_split(_ch(side), _ch(kind), _ch(trans), rows, cols, X.data_ptr(), _ld(X),
                                     s, sl.data_ptr(), ex.data_ptr(), ctypes.byref(kd))
    _check(rc, "ozaki_debug_split")
    assert kd.value == kdepth
    return sl, ex


TIMER_NAMES = ("prod_wait_empty", "mma_wait_full", "mma_wait_slot", "mma_total", "epi_wait_pass",
               "epi_drain", "epi_store", "cta_total", "mma_wait_slot_pass0", "epi_prefix",
               "epi_first_arrive", "mma_wait_full_first_kb", "mma_wait_full_pass0")


def debug_timing(enable: bool = True, read: bool = False) -> dict | None:
    """Per-role clock64 timers inside the GEMM kernel (summed over CTAs)."""
    buf = (ctypes.c_uint64 * len(TIMER_NAMES))()
    lib().ozaki_debug_timing(1 if enable else 0, buf if read else None, len(TIMER_NAMES))
    return {n: int(buf[i]) for i, n in enumerate(TIMER_NAMES)} if read else None


def debug_level_sums(transa, transb, A, B, num_slices, stream=None):
    """Exact INT32 level sums S[L-2] (m x n, torch row-major view) of a real product."""
    import torch
    _cuda(A, torch.float64, "A")
    _cuda(B, torch.float64, "B")
    m, n, k = _dims(transa, transb, A, B)
    s = int(num_slices)
    nlev = 2 * s - 1 if get_pair_set() == "full" else s
    S = torch.zeros((nlev, n, m), dtype=torch.int32, device=A.device)   # column-major per level
    with _on(A.device):
        _bind_stream(stream, A.device)
        rc = lib().ozaki_debug_level_sums(_ch(transa), _ch(transb), m, n, k, A.data_ptr(), _ld(A),
                                          B.data_ptr(), _ld(B), s, S.data_ptr())
    _check(rc, "ozaki_debug_level_sums")
    return S.transpose(1, 2)
