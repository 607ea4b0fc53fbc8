"""CPU oracle for Ozaki-II (CRT) emulation of FP64 DGEMM / ZGEMM -- NEXT-1.

TEST INFRASTRUCTURE ONLY (same rule as ``oracle/__init__.py``): only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s oracle legs may import it.

What the paper fixes (§2.2): Ozaki-II "converts floating-point
matrices into integers, performs multiple matrix multiplications using smaller,
pairwise coprime moduli and uses the CRT to reconstruct the final result"; the
precision knob is the moduli count, 10..18 in the experiments (PAPER.md:109,
:119, :127).  Everything else is SPEC.md [MODULE] ozaki2 and the DESIGN.md
readings R16..R20:

  R16 choose_moduli(N): 256, then greedily the largest integers <= 256 coprime
      to all chosen (SPEC "greedily maximal").
  R17 quantize: nu = floor((log2 M - ceil(log2 k) - 1) / 2), M = prod moduli,
      capped at 62 (int64); per row of op(A) / column of op(B) e = frexp
      exponent of max|x|, bumped by one if RNE(max|x| 2^(nu-e)) reaches 2^nu;
      Q = RNE(x 2^(nu-e)), |Q| < 2^nu.  Complex (4M, R9 N side): k_eff = 2k.
  R18 residues: r = Q mod p centered (even p: [-p/2, p/2-1]; odd: symmetric).
  R19 residue GEMM: per modulus, (rA @ rB) mod p, centered.
  R20 CRT: Z = the unique integer in (-M/2, M/2] congruent to every residue
      (exact big-integer arithmetic); by the choice of nu, Z IS the exact
      integer product Q_A @ Q_B.  P = RNE(Z 2^(e_i + f_j - 2 nu)) rounded ONCE
      (Fraction -> float, correct for subnormals too); C = alpha P + beta C as
      in R7.  Non-finite rows / columns give NaN (R10).

Two independent routes to Z are provided -- the residue/CRT route the method
takes and the direct exact integer product -- and the tests pin them equal.
"""
from __future__ import annotations

import ctypes
import math
from fractions import Fraction

import numpy as np

from . import _c, _cplx, _ptr, _quick, emb_4m, lib as _lib1, op

NU_CAP = 62


def lib():
    L = _lib1()
    if not getattr(L, "_ozaki2_ready", False):
        i64, i32, p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.orc2_quantize_rows.restype = i32
        L.orc2_quantize_rows.argtypes = [i64, i64, p, i32, p, p, p]
        L.orc2_int_gemm.restype = None
        L.orc2_int_gemm.argtypes = [i64, i64, i64, p, p, p]
        L.orc2_residue_gemm.restype = None
        L.orc2_residue_gemm.argtypes = [i64, i64, i64, p, p, i32, p]
        L._ozaki2_ready = True
    return L


# ------------------------------------------------------------------------ R16
def choose_moduli(count: int) -> list[int]:
    """SPEC choose_moduli: 256, then the largest integers coprime to all chosen."""
    if not 1 <= count <= 24:
        raise ValueError("moduli count out of range [1, 24]")
    out = [256]
    c = 255
    while len(out) < count:
        if all(math.gcd(c, q) == 1 for q in out):
            out.append(c)
        c -= 1
    return out


def modulus_product(moduli) -> int:
    M = 1
    for q in moduli:
        M *= q
    return M


# ------------------------------------------------------------------------ R17
def nu_bits(count: int, k: int) -> int:
    """Largest nu with k_pow2 * 2^(2 nu + 1) <= M (= floor((log2 M - ceil(log2 k) - 1)/2)),
    capped at 62; raises if < 1 (SPEC ModuliBudgetTooSmall)."""
    M = modulus_product(choose_moduli(count))
    c = max(0, (int(k) - 1).bit_length())          # ceil(log2 k), k >= 1
    nu = 0
    while (1 << (2 * (nu + 1) + c + 1)) <= M:
        nu += 1
    nu = min(nu, NU_CAP)
    if nu < 1:
        raise ValueError("moduli budget too small for this k")
    return nu


def quantize_rows(X, nu: int):
    """R17 on every row of a real rows x k matrix -> (Q int64, e int32, nonfinite bool)."""
    X = _c(X, np.float64)
    rows, k = X.shape
    Q = np.zeros((rows, k), dtype=np.int64)
    e = np.zeros(rows, dtype=np.int32)
    nf = np.zeros(rows, dtype=np.int32)
    lib().orc2_quantize_rows(rows, k, _ptr(X), int(nu), _ptr(Q), _ptr(e), _ptr(nf))
    return Q, e, nf.astype(bool)


# ------------------------------------------------------------------------ R18
def residues(Q, p: int) -> np.ndarray:
    r = np.mod(np.asarray(Q, dtype=np.int64), p)
    r = np.where(r >= (p + 1) // 2, r - p, r)
    return r.astype(np.int8)


# ------------------------------------------------------------------------ R19
def residue_gemm(RA, RBt, p: int) -> np.ndarray:
    """(RA @ RBt^T) mod p, centered; RA m x k, RBt n x k int8 -> int32 m x n."""
    RA = _c(RA, np.int8)
    RBt = _c(RBt, np.int8)
    m, k = RA.shape
    n = RBt.shape[0]
    C = np.zeros((m, n), dtype=np.int32)
    lib().orc2_residue_gemm(m, n, k, _ptr(RA), _ptr(RBt), int(p), _ptr(C))
    return C


# ------------------------------------------------------------------------ R20
def crt(res, moduli) -> int:
    """Unique integer in (-M/2, M/2] congruent to res[i] mod moduli[i] (big integers)."""
    M = modulus_product(moduli)
    z = 0
    for r, p in zip(res, moduli):
        Mi = M // p
        z += int(r) * Mi * pow(Mi, -1, p)
    z %= M
    if 2 * z > M:
        z -= M
    return z


def int_product(QA, QBt) -> np.ndarray:
    """Exact Z = QA @ QBt^T as a numpy object array of Python ints (direct route)."""
    QA = _c(QA, np.int64)
    QBt = _c(QBt, np.int64)
    m, k = QA.shape
    n = QBt.shape[0]
    raw = np.zeros((m, n, 6), dtype=np.uint64)
    lib().orc2_int_gemm(m, n, k, _ptr(QA), _ptr(QBt), _ptr(raw))
    Z = np.empty((m, n), dtype=object)
    for i in range(m):
        for j in range(n):
            o = raw[i, j]
            parts = []
            for q in range(3):
                v = int(o[2 * q]) | (int(o[2 * q + 1]) << 64)
                if v >= 1 << 127:
                    v -= 1 << 128
                parts.append(v)
            Z[i, j] = (parts[0] << 64) + (parts[1] << 32) + parts[2]
    return Z


def crt_product(QA, QBt, count: int) -> np.ndarray:
    """The method's route: residues per modulus -> residue GEMMs -> CRT per entry."""
    moduli = choose_moduli(count)
    Cs = [residue_gemm(residues(QA, p), residues(QBt, p), p) for p in moduli]
    m, n = Cs[0].shape
    Z = np.empty((m, n), dtype=object)
    for i in range(m):
        for j in range(n):
            Z[i, j] = crt([C[i, j] for C in Cs], moduli)
    return Z


def round_scaled(Z, e, nfa, f, nfb, nu: int) -> np.ndarray:
    """P_ij = RNE(Z_ij 2^(e_i + f_j - 2 nu)), one rounding (Fraction -> float)."""
    m, n = Z.shape
    P = np.empty((m, n), dtype=np.float64)
    for i in range(m):
        for j in range(n):
            if nfa[i] or nfb[j]:
                P[i, j] = np.nan
                continue
            sh = int(e[i]) + int(f[j]) - 2 * nu
            v = Fraction(Z[i, j]) * (Fraction(2) ** sh)
            try:
                P[i, j] = float(v)
            except OverflowError:
                P[i, j] = math.copysign(math.inf, v)
    return P


def emulated_product(A_op, B_op, count: int, route: str = "crt") -> np.ndarray:
    """R17..R20: P = Ozaki-II emulated A_op @ B_op (real), route 'crt' or 'direct'."""
    A = _c(A_op, np.float64)
    Bt = _c(np.asarray(B_op).T, np.float64)
    k = A.shape[1]
    nu = nu_bits(count, max(k, 1))
    QA, e, nfa = quantize_rows(A, nu)
    QB, f, nfb = quantize_rows(Bt, nu)
    Z = crt_product(QA, QB, count) if route == "crt" else int_product(QA, QB)
    return round_scaled(Z, e, nfa, f, nfb, nu)


def dgemm(transa, transb, alpha, A, B, beta, C, count: int, route: str = "direct") -> np.ndarray:
    Aop = op(np.asarray(A, dtype=np.float64), transa)
    Bop = op(np.asarray(B, dtype=np.float64), transb)
    m, k = Aop.shape
    n = Bop.shape[1]
    C = np.zeros((m, n)) if C is None else np.asarray(C, dtype=np.float64)
    if m == 0 or n == 0:
        return C.copy()
    if alpha == 0 or k == 0:
        return _quick(beta, C)
    P = emulated_product(Aop, Bop, count, route)
    out = _c(C, np.float64).copy()
    _lib1().orc_apply_real(m * n, float(alpha), _ptr(_c(P, np.float64)), float(beta), _ptr(out))
    return out


def zgemm(transa, transb, alpha, A, B, beta, C, count: int, route: str = "direct") -> np.ndarray:
    """4M real embedding (R9, N side) of the complex product; k_eff = 2k in nu."""
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
    A2, B2 = emb_4m(Aop, Bop)
    P2 = emulated_product(A2, B2, count, route)
    Pr, Pi = P2[:, :n].copy(), P2[:, n:].copy()
    Cr = _c(C.real, np.float64).copy()
    Ci = _c(C.imag, np.float64).copy()
    _lib1().orc_apply_complex(m * n, alpha.real, alpha.imag, _ptr(_c(Pr, np.float64)),
                              _ptr(_c(Pi, np.float64)), beta.real, beta.imag, _ptr(Cr), _ptr(Ci))
    return _cplx(Cr, Ci)
