"""Pins for the oracle's emulated TRSM (reading R23, NEXT-4c; PAPER.md:115 names ZTRSM).

The R23 diagonal-block substitution is re-derived here by an independent route: the same
FP64 operation sequence evaluated with exact rationals and one correct rounding per fma /
division (Python's int true division rounds correctly).  The blocked TRSM is pinned by exact
integer systems (unit-triangular integer A, integer B: the solution is integer and every
emulated GEMM is exact), by the residual of the solve, by nb >= dim reducing to the plain
substitution, and by the real side-'R' / side-'L' transposition identity.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import synth


def _rnd(q: Fraction) -> float:
    return q.numerator / q.denominator      # correctly rounded (CPython int true division)


def fma(a, b, c):
    return _rnd(Fraction(a) * Fraction(b) + Fraction(c))


def div(a, b):
    return _rnd(Fraction(a) / Fraction(b))


def mul(a, b):
    return _rnd(Fraction(a) * Fraction(b))


def brute_diag(side, lower, unit, T, X):
    """R23 substitution, one vector at a time, every op rounded once (see oracle docstring)."""
    T = np.asarray(T)
    kb = T.shape[0]
    cplx = np.iscomplexobj(T) or np.iscomplexobj(X)
    right = side == "R"
    vecs = [list(X[v, :]) for v in range(X.shape[0])] if right else [list(X[:, v]) for v in range(X.shape[1])]
    fwd = (not lower) if right else lower
    for x in vecs:
        for s in range(kb):
            i = s if fwd else kb - 1 - s
            nb = range(0, i) if fwd else range(i + 1, kb)
            if cplx:
                ar, ai = float(np.real(x[i])), float(np.imag(x[i]))
                for r in nb:
                    t = T[r, i] if right else T[i, r]
                    tr, ti = float(t.real), float(t.imag)
                    xr, xi = float(np.real(x[r])), float(np.imag(x[r]))
                    ar = fma(-tr, xr, fma(ti, xi, ar))
                    ai = fma(-tr, xi, fma(-ti, xr, ai))
                if not unit:
                    tr, ti = float(T[i, i].real), float(T[i, i].imag)
                    d = fma(tr, tr, mul(ti, ti))
                    ar, ai = div(fma(ar, tr, mul(ai, ti)), d), div(fma(ai, tr, -mul(ar, ti)), d)
                x[i] = complex(ar, ai)
            else:
                a = float(x[i])
                for r in nb:
                    t = T[r, i] if right else T[i, r]
                    a = fma(-float(t), float(x[r]), a)
                x[i] = a if unit else div(a, float(T[i, i]))
    out = np.array(vecs, dtype=X.dtype)
    return out if right else out.T


@pytest.mark.parametrize("side,lower,unit,cplx", list(itertools.product("LR", (True, False), (False, True),
                                                                        (False, True))))
def test_diag_solve_vs_bruteforce(orc, side, lower, unit, cplx):
    kb, nv = 7, 3
    T = synth.uniform(kb, kb, 11, complex_=cplx) + 4.0 * np.eye(kb)
    T = np.tril(T) if lower else np.triu(T)
    X = synth.spread(nv, kb, 12, phi=1.0, complex_=cplx) if side == "R" else \
        synth.spread(kb, nv, 12, phi=1.0, complex_=cplx)
    got = orc.trsm_diag(side, lower, unit, T, X)
    want = brute_diag(side, lower, unit, T, X)
    assert got.shape == want.shape
    assert (got == want).all()


def _int_system(dim, nrhs, seed, side, uplo, transa, cplx=False):
    g = np.random.default_rng(seed)
    A = g.integers(-2, 3, (dim, dim)).astype(float)
    if cplx:
        A = A + 1j * g.integers(-2, 3, (dim, dim))
    A = np.tril(A, -1) if uplo == "L" else np.triu(A, 1)
    A = A + np.eye(dim) * 7.0                      # the diagonal is not referenced for diag 'U'
    shape = (dim, nrhs) if side == "L" else (nrhs, dim)
    B = g.integers(-3, 4, shape).astype(float)
    if cplx:
        B = B + 1j * g.integers(-3, 4, shape)
    return A, B


def _exact_solve(T, B):
    """Exact rational solve of the triangular T (as Fraction / complex pairs) by substitution."""
    dim = T.shape[0]
    cplx = np.iscomplexobj(T) or np.iscomplexobj(B)
    lower = np.allclose(np.triu(T, 1), 0)

    def fr(z):
        return (Fraction(float(np.real(z))), Fraction(float(np.imag(z)))) if cplx else Fraction(float(z))

    out = np.empty(B.shape, dtype=B.dtype)
    for v in range(B.shape[1]):
        x = [None] * dim
        order = range(dim) if lower else range(dim - 1, -1, -1)
        for i in order:
            acc = fr(B[i, v])
            for j in (range(i) if lower else range(i + 1, dim)):
                t = fr(T[i, j])
                if cplx:
                    acc = (acc[0] - (t[0] * x[j][0] - t[1] * x[j][1]), acc[1] - (t[0] * x[j][1] + t[1] * x[j][0]))
                else:
                    acc = acc - t * x[j]
            x[i] = acc                                            # unit diagonal
        for i in range(dim):
            out[i, v] = complex(float(x[i][0]), float(x[i][1])) if cplx else float(x[i])
    return out


@pytest.mark.parametrize("side,uplo,transa", list(itertools.product("LR", "LU", "NTC")))
@pytest.mark.parametrize("cplx", [False, True])
def test_trsm_integer_exact(orc, side, uplo, transa, cplx):
    """Unit-triangular integer A and integer B: X is integer and small, every block update is
    an exact emulated GEMM (integer operands, s = 8), so the blocked result equals the exact
    solution -- over several blocks (nb = 3, dim = 10, ragged last block)."""
    if transa == "C" and not cplx:
        pytest.skip("'C' == 'T' for real")
    dim, nrhs = 10, 4
    A, B = _int_system(dim, nrhs, 5 + ord(side) + ord(uplo) + ord(transa), side, uplo, transa, cplx)
    X = orc.trsm(side, uplo, transa, "U", 1.0, A, B, 8, nb=3)
    Au = (np.tril(A, -1) if uplo == "L" else np.triu(A, 1)) + np.eye(dim)
    T = Au if transa == "N" else (Au.T if transa == "T" else np.conj(Au.T))
    want = _exact_solve(T, B) if side == "L" else _exact_solve(T.T, B.T).T
    assert np.max(np.abs(want)) < 2.0 ** 20          # integers well inside the exact range
    assert (X == want).all()


@pytest.mark.parametrize("side,uplo,transa,diag", list(itertools.product("LR", "LU", "NTC", "NU")))
def test_trsm_residual_complex(orc, side, uplo, transa, diag):
    dim, nrhs, s = 13, 5, 8
    A = synth.uniform(dim, dim, 3, complex_=True) * 0.2 + np.eye(dim) * 2.0
    A = np.tril(A) if uplo == "L" else np.triu(A)
    B = synth.uniform(dim, nrhs, 4, complex_=True) if side == "L" else synth.uniform(nrhs, dim, 4, complex_=True)
    alpha = 0.75 - 0.5j
    X = orc.trsm(side, uplo, transa, diag, alpha, A, B, s, nb=4)
    Ad = A.copy()
    if diag == "U":
        np.fill_diagonal(Ad, 1.0)
    T = Ad if transa == "N" else (Ad.T if transa == "T" else np.conj(Ad.T))
    R = (T @ X if side == "L" else X @ T) - alpha * B
    assert np.max(np.abs(R)) < 1e-13


@pytest.mark.parametrize("side,uplo,transa", list(itertools.product("LR", "LU", "NT")))
def test_trsm_real_nb_ge_dim_is_substitution(orc, side, uplo, transa):
    dim = 9
    A = synth.spread(dim, dim, 7, phi=1.0) + np.eye(dim) * 3.0
    A = np.tril(A) if uplo == "L" else np.triu(A)
    B = synth.uniform(dim, 4, 8) if side == "L" else synth.uniform(4, dim, 8)
    X = orc.trsm(side, uplo, transa, "N", 1.0, A, B, 7, nb=64)
    T = A if transa == "N" else A.T
    lower = (uplo == "L") == (transa == "N")
    assert (X == brute_diag(side, lower, False, T, B.copy())).all()


@pytest.mark.parametrize("uplo,transa", list(itertools.product("LU", "NT")))
def test_trsm_real_right_equals_left_transposed(orc, uplo, transa):
    """X op(A) = B  <=>  op(A)^T X^T = B^T: for real operands the R23 right-side diagonal solve
    is the left-side one on T^T op for op, and a real emulated GEMM's transpose is the emulated
    GEMM of the transposed operands (same slice pairs per level), so the results are bitwise
    transposes of each other."""
    dim, nrhs = 11, 6
    A = synth.uniform(dim, dim, 1) * 0.3 + np.eye(dim) * 2.0
    A = np.tril(A) if uplo == "L" else np.triu(A)
    B = synth.spread(nrhs, dim, 2, phi=1.0)
    XR = orc.trsm("R", uplo, transa, "N", -1.5, A, B, 6, nb=4)
    tr2 = "T" if transa == "N" else "N"
    XL = orc.trsm("L", uplo, tr2, "N", -1.5, A, B.T.copy(), 6, nb=4)
    assert (XR == XL.T).all()


def test_trsm_alpha_zero_and_identity(orc):
    B = np.full((5, 3), np.nan)
    A = np.eye(5)
    assert (orc.trsm("L", "L", "N", "N", 0.0, A, B, 7) == 0).all()
    Bv = synth.uniform(5, 3, 1)
    assert (orc.trsm("L", "U", "T", "N", 1.0, A, Bv, 7, nb=2) == Bv).all()
