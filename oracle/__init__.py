"""CPU oracle for the INT8 Ozaki-I emulation of FP64 DGEMM / ZGEMM.

TEST INFRASTRUCTURE ONLY -- only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2603_29975_b200``) never imports it and
shares no code with it; the only common module is ``synth`` (seeded input
generators, no method arithmetic).

Layers:
  * step O1 (op(): transpose / conjugate, "ZGEMM", BLAS semantics)
    is done here in numpy;
  * steps O2..O7 run in plain C (``ozaki_oracle.c``, built with gcc
    -ffp-contract=off) -- see that file for the per-step citations;
  * ``exact_*`` is the TRUE FP64 product (long accumulator, one rounding);
  * ``fp64_*`` is the plain FP64 triple loop ("native FP64 GEMM").

Parity status: every function here is pinned by tests/test_oracle_*.py
(brute force with ``fractions.Fraction``, closed forms, invariants); see
DESIGN.md §4 for the pin of each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ozaki_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no CUDA involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, i32, dbl, p = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.orc_exponent.restype = i32
        L.orc_exponent.argtypes = [p, i64, p]
        L.orc_digits.restype = i32
        L.orc_digits.argtypes = [dbl, i32, i32, p]
        L.orc_split_rows.restype = i32
        L.orc_split_rows.argtypes = [i64, i64, p, i32, p, p, p]
        L.orc_level_sums.restype = None
        L.orc_level_sums.argtypes = [i64, i64, i64, i32, p, p, p]
        L.orc_combine.restype = None
        L.orc_combine.argtypes = [i64, i64, i32, p, p, p, p, p, p]
        L.orc_emulated_product.restype = i32
        L.orc_emulated_product.argtypes = [i64, i64, i64, i32, p, p, p]
        L.orc_apply_real.restype = None
        L.orc_apply_real.argtypes = [i64, dbl, p, dbl, p]
        L.orc_apply_complex.restype = None
        L.orc_apply_complex.argtypes = [i64, dbl, dbl, p, p, dbl, dbl, p, p]
        L.orc_combine_3m.restype = None
        L.orc_combine_3m.argtypes = [i64, p, p, p, p, p]
        L.orc_fp64_gemm.restype = None
        L.orc_fp64_gemm.argtypes = [i64, i64, i64, p, p, p]
        L.orc_exact_dot.restype = dbl
        L.orc_exact_dot.argtypes = [i64, p, p]
        L.orc_exact_gemm.restype = None
        L.orc_exact_gemm.argtypes = [i64, i64, i64, p, p, p]
        L.orc_num_threads.restype = i32
        L.orc_quick_real.restype = None
        L.orc_quick_real.argtypes = [i64, dbl, p]
        L.orc_level_sums_full.restype = None
        L.orc_level_sums_full.argtypes = [i64, i64, i64, i32, p, p, p]
        L.orc_combine_levels.restype = None
        L.orc_combine_levels.argtypes = [i64, i64, i32, p, p, p, p, p, p]
        L.orc_emulated_product_full.restype = i32
        L.orc_emulated_product_full.argtypes = [i64, i64, i64, i32, p, p, p]
        L.orc_quick_complex.restype = None
        L.orc_quick_complex.argtypes = [i64, dbl, dbl, p, p]
        L.orc_trsm_diag_real.restype = None
        L.orc_trsm_diag_real.argtypes = [i32, i32, i32, i64, p, i64, p]
        L.orc_trsm_diag_complex.restype = None
        L.orc_trsm_diag_complex.argtypes = [i32, i32, i32, i64, p, i64, p]
        _lib = L
    return _lib


def _cplx(re, im):
    """Assemble complex128 without arithmetic (1j*x would turn inf into NaN)."""
    out = np.empty(np.shape(re), dtype=np.complex128)
    out.real = re
    out.imag = im
    return out


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return lib().orc_num_threads()


# --------------------------------------------------------------------------- O1
def op(X, trans: str):
    """O1: materialise op(X) for BLAS trans in {'N','T','C'} ('C' == 'T' for real)."""
    t = trans.upper()
    if t == "N":
        return X
    if t == "T":
        return X.T
    if t == "C":
        return np.conj(X.T) if np.iscomplexobj(X) else X.T
    raise ValueError(trans)


# ----------------------------------------------------------------------- O2..O4
def exponent(row) -> tuple[int, bool]:
    r = _c(row, np.float64)
    nf = ctypes.c_int(0)
    e = lib().orc_exponent(_ptr(r), r.size, ctypes.byref(nf))
    return int(e), bool(nf.value)


def digits(x: float, e: int, s: int) -> np.ndarray:
    d = np.zeros(16, dtype=np.int8)
    rc = lib().orc_digits(float(x), int(e), int(s), _ptr(d))
    if rc != 0:
        raise ArithmeticError("top digit out of range")
    return d[:s].copy()


def split_rows(X, s: int):
    """Split every row of a real rows x k matrix.

    Returns (D[s][rows][k] int8 with D[t-1] = slice t, exps int32[rows],
    nonfinite bool[rows])."""
    X = _c(X, np.float64)
    rows, k = X.shape
    D = np.zeros((s, rows, k), dtype=np.int8)
    e = np.zeros(rows, dtype=np.int32)
    nf = np.zeros(rows, dtype=np.int32)
    rc = lib().orc_split_rows(rows, k, _ptr(X), s, _ptr(D), _ptr(e), _ptr(nf))
    if rc != 0:
        raise ArithmeticError("top digit out of range")
    return D, e, nf.astype(bool)


# --------------------------------------------------------------------------- O5
def level_sums(DA, DB, s: int) -> np.ndarray:
    """S[L-2][i][j] = sum_{t+u=L} dA_t[i,:] . dB_u[j,:]  (int64, exact)."""
    DA = _c(DA, np.int8)
    DB = _c(DB, np.int8)
    _, m, k = DA.shape
    _, n, k2 = DB.shape
    assert k == k2
    S = np.zeros((s, m, n), dtype=np.int64)
    lib().orc_level_sums(m, n, k, s, _ptr(DA), _ptr(DB), _ptr(S))
    return S


# --------------------------------------------------------------------------- O6
def combine(S, e, nfa, f, nfb, s: int) -> np.ndarray:
    S = _c(S, np.int64)
    _, m, n = S.shape
    e = _c(e, np.int32)
    f = _c(f, np.int32)
    nfa = _c(nfa, np.int32)
    nfb = _c(nfb, np.int32)
    P = np.zeros((m, n), dtype=np.float64)
    lib().orc_combine(m, n, s, _ptr(S), _ptr(e), _ptr(nfa), _ptr(f), _ptr(nfb), _ptr(P))
    return P


def level_sums_full(DA, DB, s: int) -> np.ndarray:
    """R21 (NEXT-4): all s^2 pairs, S[L-2] for L = 2..2s (int64, exact)."""
    DA = _c(DA, np.int8)
    DB = _c(DB, np.int8)
    _, m, k = DA.shape
    _, n, _ = DB.shape
    S = np.zeros((2 * s - 1, m, n), dtype=np.int64)
    lib().orc_level_sums_full(m, n, k, s, _ptr(DA), _ptr(DB), _ptr(S))
    return S


def emulated_product(A_op, B_op, s: int, pairs: str = "triangular") -> np.ndarray:
    """O2..O6: P = emulated A_op @ B_op for real matrices (returns m x n).
    pairs = 'triangular' (R1, t + u <= s + 1) or 'full' (R21, all s^2 products)."""
    A = _c(A_op, np.float64)
    Bt = _c(np.asarray(B_op).T, np.float64)
    m, k = A.shape
    n = Bt.shape[0]
    P = np.zeros((m, n), dtype=np.float64)
    fn = lib().orc_emulated_product_full if pairs == "full" else lib().orc_emulated_product
    rc = fn(m, n, k, s, _ptr(A), _ptr(Bt), _ptr(P))
    if rc != 0:
        raise ArithmeticError("oracle split failed")
    return P


# ------------------------------------------------------------------------ O1..O7
def _quick(beta, C):
    """BLAS quick return (reading R7): alpha == 0 or k == 0 -> C = beta*C;
    beta == 0 -> zeros without reading C.  Same FP64 op shapes as O7."""
    if np.iscomplexobj(C):
        Cr = _c(C.real, np.float64).copy()
        Ci = _c(C.imag, np.float64).copy()
        b = complex(beta)
        lib().orc_quick_complex(Cr.size, b.real, b.imag, _ptr(Cr), _ptr(Ci))
        return _cplx(Cr, Ci)
    out = _c(C, np.float64).copy()
    lib().orc_quick_real(out.size, float(beta), _ptr(out))
    return out


def blocked_product(A_op, B_op, s: int, kb: int, pairs: str = "triangular", cplx: bool = False,
                    method: str = "4m"):
    """R22 (NEXT-4 per-block exponent alignment): K in blocks of kb; each block's product is
    emulated with its OWN row / column exponents (O2..O6 on the sub-matrices), and the block
    products are summed in ascending block order in FP64 (one RNE per addition).  Real:
    returns P; complex (4M): returns (Pr, Pi)."""
    k = A_op.shape[1]
    acc = None
    for b0 in range(0, k, kb):
        Ab = A_op[:, b0:b0 + kb]
        Bb = B_op[b0:b0 + kb, :]
        Pb = zproduct(Ab, Bb, s, method, pairs) if cplx else emulated_product(Ab, Bb, s, pairs)
        if acc is None:
            acc = Pb
        elif cplx:
            acc = (acc[0] + Pb[0], acc[1] + Pb[1])       # numpy float64 '+' = one RNE each
        else:
            acc = acc + Pb
    return acc


def dgemm_blocked(transa, transb, alpha, A, B, beta, C, s: int, kb: int) -> np.ndarray:
    """R22 DGEMM: per-block exponents, then O7 alpha/beta on the summed P."""
    Aop = op(np.asarray(A, dtype=np.float64), transa)
    Bop = op(np.asarray(B, dtype=np.float64), transb)
    m, k = Aop.shape
    n = Bop.shape[1]
    C = np.zeros((m, n)) if C is None else np.asarray(C, dtype=np.float64)
    if m == 0 or n == 0:
        return C.copy()
    if alpha == 0 or k == 0:
        return _quick(beta, C)
    P = blocked_product(Aop, Bop, s, kb)
    out = _c(C, np.float64).copy()
    lib().orc_apply_real(m * n, float(alpha), _ptr(_c(P, np.float64)), float(beta), _ptr(out))
    return out


def zgemm_blocked(transa, transb, alpha, A, B, beta, C, s: int, kb: int, method: str = "4m") -> np.ndarray:
    """R22 ZGEMM (4M or 3M per block)."""
    Aop = op(np.asarray(A, dtype=np.complex128), transa)
    Bop = op(np.asarray(B, dtype=np.complex128), transb)
    m, k = Aop.shape
    n = Bop.shape[1]
    alpha = complex(alpha)
    beta = complex(beta)
    C = np.zeros((m, n), dtype=np.complex128) if C is None else np.asarray(C, dtype=np.complex128)
    if m == 0 or n == 0:
        return C.copy()
    if alpha == 0 or k == 0:
        return _quick(beta, C)
    Pr, Pi = blocked_product(Aop, Bop, s, kb, cplx=True, method=method)
    Cr = _c(C.real, np.float64).copy()
    Ci = _c(C.imag, np.float64).copy()
    lib().orc_apply_complex(m * n, alpha.real, alpha.imag, _ptr(_c(Pr, np.float64)),
                            _ptr(_c(Pi, np.float64)), beta.real, beta.imag, _ptr(Cr), _ptr(Ci))
    return _cplx(Cr, Ci)


def dgemm(transa, transb, alpha, A, B, beta, C, s: int, pairs: str = "triangular") -> np.ndarray:
    """Full emulated DGEMM: returns alpha*emul(op(A)op(B)) + beta*C (new array)."""
    Aop = op(np.asarray(A, dtype=np.float64), transa)
    Bop = op(np.asarray(B, dtype=np.float64), transb)
    m, k = Aop.shape
    n = Bop.shape[1]
    C = np.zeros((m, n)) if C is None else np.asarray(C, dtype=np.float64)
    if m == 0 or n == 0:
        return C.copy()
    if alpha == 0 or k == 0:
        return _quick(beta, C)
    P = emulated_product(Aop, Bop, s, pairs)
    out = _c(C, np.float64).copy()
    lib().orc_apply_real(m * n, float(alpha), _ptr(P), float(beta), _ptr(out))
    return out


def emb_4m(Aop, Bop):
    """Real embedding used by 4M (reading R9, N-side form):
    C = A B with A = Ar + i Ai, B = Br + i Bi is
        [Cr | Ci] = [Ar | Ai] @ [[Br, Bi], [-Bi, Br]]
    i.e. op(A)' = [Ar, Ai] (m x 2k) and op(B)' (2k x 2n); the -Bi block is
    split from the negated FP64 values.  Returns (A2, B2)."""
    Ar, Ai = Aop.real, Aop.imag
    Br, Bi = Bop.real, Bop.imag
    A2 = np.hstack([Ar, Ai])
    B2 = np.block([[Br, Bi], [-Bi, Br]])
    return A2, B2


def zproduct(Aop, Bop, s: int, method: str = "4m", pairs: str = "triangular"):
    """Emulated complex product P = Pr + i Pi (O2..O6, 4M or 3M)."""
    n = Bop.shape[1]
    if method == "4m":
        A2, B2 = emb_4m(Aop, Bop)
        P2 = emulated_product(A2, B2, s, pairs)
        return P2[:, :n].copy(), P2[:, n:].copy()
    if method == "3m":
        Ar, Ai = np.ascontiguousarray(Aop.real), np.ascontiguousarray(Aop.imag)
        Br, Bi = np.ascontiguousarray(Bop.real), np.ascontiguousarray(Bop.imag)
        T1 = emulated_product(Ar, Br, s, pairs)
        T2 = emulated_product(Ai, Bi, s, pairs)
        T3 = emulated_product(Ar + Ai, Br + Bi, s, pairs)  # fl(Ar+Ai), fl(Br+Bi) in FP64
        Pr = np.zeros_like(T1)
        Pi = np.zeros_like(T1)
        lib().orc_combine_3m(T1.size, _ptr(_c(T1, np.float64)), _ptr(_c(T2, np.float64)),
                             _ptr(_c(T3, np.float64)), _ptr(Pr), _ptr(Pi))
        return Pr, Pi
    raise ValueError(method)


def zgemm(transa, transb, alpha, A, B, beta, C, s: int, method: str = "4m",
          pairs: str = "triangular") -> np.ndarray:
    Aop = op(np.asarray(A, dtype=np.complex128), transa)
    Bop = op(np.asarray(B, dtype=np.complex128), transb)
    m, k = Aop.shape
    n = Bop.shape[1]
    alpha = complex(alpha)
    beta = complex(beta)
    C = np.zeros((m, n), dtype=np.complex128) if C is None else np.asarray(C, dtype=np.complex128)
    if m == 0 or n == 0:
        return C.copy()
    if alpha == 0 or k == 0:
        return _quick(beta, C)
    Pr, Pi = zproduct(Aop, Bop, s, method, pairs)
    Cr = _c(C.real, np.float64).copy()
    Ci = _c(C.imag, np.float64).copy()
    lib().orc_apply_complex(m * n, alpha.real, alpha.imag, _ptr(_c(Pr, np.float64)),
                            _ptr(_c(Pi, np.float64)), beta.real, beta.imag, _ptr(Cr), _ptr(Ci))
    return _cplx(Cr, Ci)


# ----------------------------------------------------------- truth / native FP64
def exact_product(A_op, B_op) -> np.ndarray:
    """TRUE product of real matrices: every entry rounded once (RNE)."""
    A = _c(A_op, np.float64)
    Bt = _c(np.asarray(B_op).T, np.float64)
    m, k = A.shape
    n = Bt.shape[0]
    T = np.zeros((m, n))
    lib().orc_exact_gemm(m, n, k, _ptr(A), _ptr(Bt), _ptr(T))
    return T


def exact_zproduct(A_op, B_op) -> np.ndarray:
    """TRUE complex product, re and im each rounded once."""
    A2, B2 = emb_4m(A_op, B_op)
    T2 = exact_product(A2, B2)
    n = B_op.shape[1]
    return _cplx(T2[:, :n], T2[:, n:])


def exact_dot(a, b) -> float:
    a = _c(a, np.float64)
    b = _c(b, np.float64)
    return lib().orc_exact_dot(a.size, _ptr(a), _ptr(b))


def fp64_product(A_op, B_op) -> np.ndarray:
    """Plain FP64 triple loop, ascending k with fma (the 'native' comparison)."""
    A = _c(A_op, np.float64)
    Bt = _c(np.asarray(B_op).T, np.float64)
    m, k = A.shape
    n = Bt.shape[0]
    T = np.zeros((m, n))
    lib().orc_fp64_gemm(m, n, k, _ptr(A), _ptr(Bt), _ptr(T))
    return T


def pairs(s: int) -> int:
    """Number of retained slice pairs t+u <= s+1 (reading R1)."""
    return s * (s + 1) // 2


# ------------------------------------------------------------ R23 emulated TRSM (NEXT-4c)
def trsm_diag(side, lower, unit, T, X):
    """Diagonal-block solve of R23 (orc_trsm_diag_*): side 'L' solves T x = b for every
    column of X, 'R' solves x T = b for every row; returns the solved copy of X."""
    T = np.asarray(T)
    kb = T.shape[0]
    cplx = np.iscomplexobj(T) or np.iscomplexobj(X)
    right = side.upper() == "R"
    vec = np.ascontiguousarray(X.T if not right else X)          # one vector per row
    if cplx:
        Tc = _c(np.asarray(T, dtype=np.complex128), np.complex128)
        v = _c(vec, np.complex128).copy()
        lib().orc_trsm_diag_complex(int(right), int(lower), int(unit), kb, _ptr(Tc), v.shape[0], _ptr(v))
    else:
        Tc = _c(T, np.float64)
        v = _c(vec, np.float64).copy()
        lib().orc_trsm_diag_real(int(right), int(lower), int(unit), kb, _ptr(Tc), v.shape[0], _ptr(v))
    return v.T if not right else v


def _scale_alpha(alpha, B, cplx):
    """B <- alpha B with R7's beta*C shapes (the BLAS quick return's: real alpha b, complex
    fma(ar, br, -(ai bi)) / fma(ar, bi, ai br); alpha == 0: zeros, B not read); alpha == 1
    leaves B unchanged."""
    if (complex(alpha) if cplx else float(alpha)) == 1:
        return np.array(B, copy=True)
    return _quick(complex(alpha) if cplx else float(alpha), B)


def trsm(side, uplo, transa, diag, alpha, A, B, s: int, nb: int = 128, method: str = "4m"):
    """R23 blocked TRSM: side 'L' solves op(A) X = alpha B, 'R' solves X op(A) = alpha B.
    B <- alpha B first; then over nb-blocks of the triangle (forward for lower op(A) on the
    left / upper on the right, backward otherwise): X_K = the R23 diagonal solve of
    T_KK, and the remaining rows (left) / columns (right) are updated by the EMULATED GEMM
    B_R <- -T_RK X_K + B_R (left) or B_R <- -X_K T_KR + B_R (right) with s slices (O1..O7).
    Only the uplo triangle of A is referenced (diag 'U': its diagonal is not either).
    Returns X (new array)."""
    cplx = np.iscomplexobj(A) or np.iscomplexobj(B)
    side, uplo, transa, diag = side.upper(), uplo.upper(), transa.upper(), diag.upper()
    A = np.asarray(A, dtype=np.complex128 if cplx else np.float64)
    dim = A.shape[0]
    tri = np.tril(A) if uplo == "L" else np.triu(A)
    T = op(tri, transa)                              # op(A), other triangle zero
    lower = (uplo == "L") == (transa == "N")         # op(A) lower triangular?
    unit = diag == "U"
    X = _scale_alpha(alpha, np.asarray(B, dtype=A.dtype), cplx)
    if X.size == 0 or complex(alpha) == 0:
        return X
    blocks = [(k0, min(dim, k0 + nb)) for k0 in range(0, dim, nb)]
    left = side == "L"
    forward = lower if left else not lower
    gemm = (lambda a_, b_, c_: zgemm("N", "N", -1.0, a_, b_, 1.0, c_, s, method)) if cplx else \
           (lambda a_, b_, c_: dgemm("N", "N", -1.0, a_, b_, 1.0, c_, s))
    for (a, b) in (blocks if forward else blocks[::-1]):
        Tkk = T[a:b, a:b]
        if left:
            X[a:b] = trsm_diag("L", lower, unit, Tkk, X[a:b])
            r0, r1 = (b, dim) if forward else (0, a)
            if r1 > r0:
                X[r0:r1] = gemm(T[r0:r1, a:b], X[a:b], X[r0:r1])
        else:
            X[:, a:b] = trsm_diag("R", lower, unit, Tkk, X[:, a:b])
            r0, r1 = (b, dim) if forward else (0, a)
            if r1 > r0:
                X[:, r0:r1] = gemm(X[:, a:b], T[a:b, r0:r1], X[:, r0:r1])
    return X
