"""Pins of the NEXT-4 full-pair-set variant of the oracle (reading R21: all s^2 slice
products, levels L = 2..2s, same ascending FP64 combine) -- (-m "not gpu").

Pinned against ``oracle/brute.py`` (Fraction exponents / rounding / digits written
independently of the C oracle) and against closed forms: with every pair kept, the
level sums reconstruct the EXACT integer product of the integerised operands.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import brute
import synth


@pytest.mark.parametrize("s", [1, 2, 3, 5, 8])
def test_full_levels_reconstruct_integer_product(s):
    A = synth.spread(4, 7, seed=10 + s, phi=2.0)
    Bt = synth.spread(3, 7, seed=20 + s, phi=2.0)
    DA, e, _ = oracle.split_rows(A, s)
    DB, f, _ = oracle.split_rows(Bt, s)
    S = oracle.level_sums_full(DA, DB, s)
    assert S.shape[0] == 2 * s - 1
    St = oracle.level_sums(DA, DB, s)
    assert (S[:s] == St).all()                         # triangular levels are the first s of the full set
    eb = [brute.exponent_def(r) for r in A]
    fb = [brute.exponent_def(r) for r in Bt]
    assert list(e) == eb and list(f) == fb
    for i in range(4):
        for j in range(3):
            XA = [brute.integerise(x, eb[i], s) for x in A[i]]
            XB = [brute.integerise(x, fb[j], s) for x in Bt[j]]
            exact = sum(a * b for a, b in zip(XA, XB))
            assert sum(int(S[L - 2, i, j]) * 256 ** (2 * s - L) for L in range(2, 2 * s + 1)) == exact


@pytest.mark.parametrize("s", [2, 4, 6, 8])
def test_full_product_is_rounded_integer_product(s):
    """P_full = the ascending FP64 sum of the exact levels: within 2 ulp of RNE(X_A X_B 2^(e+f-2P))."""
    m, k, n = 6, 19, 5
    A = synth.spread(m, k, seed=30 + s, phi=1.5)
    B = synth.spread(k, n, seed=40 + s, phi=1.5)
    P = oracle.emulated_product(A, B, s, pairs="full")
    Pbits = 8 * s - 1
    for i in range(m):
        ei = brute.exponent_def(A[i])
        for j in range(n):
            fj = brute.exponent_def(B[:, j])
            z = sum(brute.integerise(A[i, t], ei, s) * brute.integerise(B[t, j], fj, s) for t in range(k))
            ref = float(Fraction(z) * Fraction(2) ** (ei + fj - 2 * Pbits))
            assert abs(P[i, j] - ref) <= 2 * math.ulp(ref) + 0.0, (s, i, j)


def test_full_pairs_integer_exact_and_bound():
    # integer inputs: every digit product is kept, so the result is exact (no T(e)+T(f) <= s+1 rule)
    A = synth.integer(12, 20, seed=1, bits=20)
    B = synth.integer(20, 9, seed=2, bits=20)
    assert (oracle.emulated_product(A, B, 4, pairs="full") == A @ B).all()
    assert not (oracle.emulated_product(A, B, 4) == A @ B).all()   # the triangular set drops pairs here
    # pure quantisation error: |P - AB| <= sum_k (|a| d_b + |b| d_a + d_a d_b) + 2 ulp, d = 2^(e-P-1)
    s = 4
    A = synth.spread(10, 40, seed=3, phi=2.0)
    B = synth.spread(40, 8, seed=4, phi=2.0)
    P = oracle.emulated_product(A, B, s, pairs="full")
    T = oracle.exact_product(A, B)
    Pb = 8 * s - 1
    for i in range(10):
        da = 2.0 ** (brute.exponent_def(A[i]) - Pb - 1)
        for j in range(8):
            db = 2.0 ** (brute.exponent_def(B[:, j]) - Pb - 1)
            bound = np.sum(np.abs(A[i]) * db + np.abs(B[:, j]) * da + da * db)
            assert abs(P[i, j] - T[i, j]) <= bound + 2 * math.ulp(T[i, j])


def test_full_pairs_more_accurate_than_triangular():
    A = synth.uniform(16, 64, seed=5)
    B = synth.uniform(64, 12, seed=6)
    T = oracle.exact_product(A, B)
    w = np.abs(A) @ np.abs(B)
    for s in (3, 4, 5):
        et = np.max(np.abs(oracle.emulated_product(A, B, s) - T) / w)
        ef = np.max(np.abs(oracle.emulated_product(A, B, s, pairs="full") - T) / w)
        assert ef <= et
