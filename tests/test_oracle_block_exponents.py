"""Pins of the NEXT-4 per-block exponent variant of the oracle (reading R22) (-m "not gpu").

R22: K in blocks of kb; every block is emulated with its own row/column exponents; the block
products are summed in ascending block order (one RNE per addition); then R7.  Pinned to: the
per-row result when kb >= k; a Fraction brute force of a whole 2-block product; exactness of
the block sum on integer data; the accuracy gain on block-graded rows (the reason for the
variant); per-block scale invariance.
"""
import math
from fractions import Fraction

import numpy as np

import oracle
from oracle import brute
import synth


def test_one_block_equals_per_row():
    A = synth.spread(9, 40, seed=1, phi=2.0)
    B = synth.spread(40, 7, seed=2, phi=2.0)
    for kb in (40, 64, 1000):
        assert (oracle.dgemm_blocked("N", "N", 1.0, A, B, 0.0, None, 5, kb) ==
                oracle.dgemm("N", "N", 1.0, A, B, 0.0, None, 5)).all()


def test_two_block_bruteforce():
    """Each block from oracle/brute.py's exact retained sum (rounded as O6 would), then the sum."""
    s, kb = 3, 4
    A = synth.spread(3, 8, seed=3, phi=2.0)
    B = synth.spread(8, 2, seed=4, phi=2.0)
    P = oracle.blocked_product(A, B, s, kb)
    for i in range(3):
        for j in range(2):
            parts = []
            for b0 in (0, 4):
                Ar = [list(A[i, b0:b0 + kb])]
                Bt = [list(B[b0:b0 + kb, j])]
                _, e, f, S, _, _ = brute.retained_exact(Ar, Bt, s)
                acc = 0.0
                for L in range(s + 1, 1, -1):          # O6 ascending, RNE per step
                    acc = acc + float(S[L - 2][0][0]) * 2.0 ** (-8 * (L - 2))
                parts.append(math.ldexp(acc, e[0] + f[0] - 14))
            assert P[i, j] == parts[0] + parts[1]


def test_block_graded_rows_more_accurate():
    """A block of A 2^40 smaller, paired with a block of B 2^40 larger: their products count
    fully, but per-row / per-column exponents are set by the other blocks and drop it at s <= 5
    (error ~0.2 of |A||B|); per-block exponents keep it (error ~1e-10 at s = 4)."""
    g = np.random.default_rng(5)
    m, k, n, kb = 16, 256, 12, 64
    A = g.uniform(-1, 1, (m, k))
    A[:, 64:128] *= 2.0 ** -40
    B = g.uniform(-1, 1, (k, n))
    B[64:128, :] *= 2.0 ** 40
    T = oracle.exact_product(A, B)
    w = np.abs(A) @ np.abs(B)
    e_row = np.max(np.abs(oracle.dgemm("N", "N", 1.0, A, B, 0.0, None, 4) - T) / w)
    e_blk = np.max(np.abs(oracle.dgemm_blocked("N", "N", 1.0, A, B, 0.0, None, 4, kb) - T) / w)
    assert e_row > 0.1 and e_blk < 1e-9


def test_integer_exact_and_block_scale_invariance():
    A = synth.integer(10, 96, seed=6, bits=7)
    B = synth.integer(96, 5, seed=7, bits=7)
    assert (oracle.dgemm_blocked("N", "N", 1.0, A, B, 0.0, None, 2, 32) == A @ B).all()
    # scaling one K block of A by 2^p scales that block's product exactly; with power-of-two
    # data the block products are exact, so the sum is exact as well
    A2 = A.copy()
    A2[:, 32:64] *= 2.0 ** 20
    P = oracle.blocked_product(A2, B, 2, 32)
    assert (P == A[:, :32] @ B[:32] + 2.0 ** 20 * (A[:, 32:64] @ B[32:64]) + A[:, 64:] @ B[64:]).all()


def test_complex_blocked_matches_blockwise_4m():
    A = synth.make("kkr", 6, 70, seed=8, complex_=True, gamma=1.0)
    B = synth.make("kkr", 70, 5, seed=9, complex_=True, gamma=1.0)
    C = oracle.zgemm_blocked("N", "N", 1.0, A, B, 0.0, None, 5, 32)
    P0 = oracle.zgemm("N", "N", 1.0, A[:, :32], B[:32], 0.0, None, 5)
    P1 = oracle.zgemm("N", "N", 1.0, A[:, 32:64], B[32:64], 0.0, None, 5)
    P2 = oracle.zgemm("N", "N", 1.0, A[:, 64:], B[64:], 0.0, None, 5)
    ref = (P0 + P1) + P2
    assert (C.real == ref.real).all() and (C.imag == ref.imag).all()
