"""Seeded synthetic operand generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the method's arithmetic (no exponent scan, no slicing,
no products).  It only draws FP64 / complex128 matrices whose value
distribution mimics the workloads the paper talks about:

* ``uniform``  -- U[-1, 1) entries (benign data, SURVEY.md §8(d) family U).
* ``spread``   -- (U(0,1) - 1/2) * exp(phi * N(0,1)): a controllable exponent
  spread inside every row/column (family Phi(phi); "accuracy depends
  on ... the properties of the operator").
* ``kkr``      -- graded-channel KKR/tau-like blocks (family KKR(gamma)):
  block size 2(l_max+1)^2 = 32, angular channel l(r) = floor(sqrt(r mod 16)),
  x_ij = (2*delta_ij + g_ij) * 2^(-gamma*(l(i)+l(j))).  This mimics the
  angular-momentum scaling of the multiple-scattering matrices that LSMS
  inverts (§3.2, 33,750^2 double-complex at PAPER.md:151).
* ``integer``  -- integer-valued entries |x| < 2^bits (exactness pins).
* ``hamiltonian`` -- Hermitian test operator H = Q diag(lambda) Q^H with a seeded
  random unitary Q (SPEC.md [MODULE] workload build_test_hamiltonian: the
  synthetic stand-in for the Kohn-Sham operator of PAPER.md:113-117).

All matrices are returned in Fortran (column-major) order, the BLAS layout the
C ABI consumes; complex matrices are ``complex128`` (interleaved re, im).
"""
from __future__ import annotations

import numpy as np

__all__ = ["rng", "uniform", "spread", "kkr", "integer", "hamiltonian", "make", "FAMILIES"]


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _f(x):
    return np.asfortranarray(x)


def uniform(rows, cols, seed, complex_=False):
    g = rng(seed)
    re = g.uniform(-1.0, 1.0, size=(rows, cols))
    if not complex_:
        return _f(re)
    im = g.uniform(-1.0, 1.0, size=(rows, cols))
    return _f(re + 1j * im)


def spread(rows, cols, seed, phi=2.0, complex_=False):
    g = rng(seed)

    def one():
        return (g.uniform(0.0, 1.0, size=(rows, cols)) - 0.5) * np.exp(
            phi * g.standard_normal(size=(rows, cols)))

    re = one()
    if not complex_:
        return _f(re)
    return _f(re + 1j * one())


def _channel(idx):
    # angular channel l(r) = floor(sqrt(r mod 16)) for l_max = 3 (16 = (l_max+1)^2)
    return np.floor(np.sqrt(np.asarray(idx) % 16)).astype(np.int64)


def kkr(rows, cols, seed, gamma=1.0, complex_=True):
    g = rng(seed)
    li = _channel(np.arange(rows))[:, None]
    lj = _channel(np.arange(cols))[None, :]
    scale = np.exp2(-gamma * (li + lj).astype(np.float64))
    eye = np.zeros((rows, cols))
    d = min(rows, cols)
    eye[np.arange(d), np.arange(d)] = 2.0
    re = (eye + g.uniform(-1.0, 1.0, size=(rows, cols))) * scale
    if not complex_:
        return _f(re)
    im = g.uniform(-1.0, 1.0, size=(rows, cols)) * scale
    return _f(re + 1j * im)


def integer(rows, cols, seed, bits=7, complex_=False):
    g = rng(seed)
    hi = (1 << bits) - 1

    def one():
        return g.integers(-hi, hi + 1, size=(rows, cols)).astype(np.float64)

    re = one()
    if not complex_:
        return _f(re)
    return _f(re + 1j * one())


FAMILIES = {
    "uniform": uniform,
    "spread": spread,
    "kkr": kkr,
    "integer": integer,
}


def make(family, rows, cols, seed, complex_=False, **kw):
    """Dispatch by family name; ``kw`` carries phi / gamma / bits."""
    return FAMILIES[family](rows, cols, seed, complex_=complex_, **kw)


def hamiltonian(n, seed, eigs=None):
    """Hermitian n x n complex128 H = Q diag(eigs) Q^H (Fortran order) and its sorted
    eigenvalues.  Q: QR of a seeded complex Gaussian matrix (phase-fixed), eigs default
    U[-1, 1).  H is symmetrised exactly: H = (H + H^H) / 2 computed entrywise."""
    g = rng(seed)
    if eigs is None:
        eigs = np.sort(g.uniform(-1.0, 1.0, size=n))
    eigs = np.asarray(eigs, dtype=np.float64)
    Z = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))
    Q, R = np.linalg.qr(Z)
    Q = Q * (np.diag(R) / np.abs(np.diag(R)))          # unique unitary factor
    H = (Q * eigs) @ Q.conj().T
    H = 0.5 * (H + H.conj().T)
    return np.asfortranarray(H), np.sort(eigs)
