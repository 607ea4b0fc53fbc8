"""Pins of the Ozaki-II (CRT) oracle, oracle/ozaki2.py (-m "not gpu").

NEXT-1 of SURVEY.md §8(f).  The oracle is pinned to things other than itself:
SPEC.md's worked examples (tests/golden/ozaki2_spec_examples.txt), brute force
over the CRT range, Fraction brute force of the whole product on tiny inputs,
the two independent routes to the integer product (residues + CRT vs the direct
exact integer GEMM), closed-form error bounds, exactness on integer inputs,
scale invariance and monotone refinement in the moduli count.
"""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import ozaki2 as o2
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ozaki2_spec_examples.txt")


def _gold():
    with open(GOLD) as fh:
        return [ln.split() for ln in fh if ln.strip() and not ln.startswith("#")]


# ----------------------------------------------------------------- R16 moduli
def test_spec_examples_golden():
    for rec in _gold():
        kind = rec[0]
        if kind == "moduli":
            assert o2.choose_moduli(int(rec[1])) == [int(x) for x in rec[2:]]
        elif kind == "product_bits_at_least":
            assert math.log2(o2.modulus_product(o2.choose_moduli(int(rec[1])))) >= float(rec[2])
        elif kind == "nu":
            assert o2.nu_bits(int(rec[1]), int(rec[2])) == int(rec[3])
        elif kind == "crt":
            mods = [int(x) for x in rec[1].split(",")]
            res = [int(x) for x in rec[2].split(",")]
            assert o2.crt([r % p for r, p in zip(res, mods)], mods) == int(rec[3])
        else:
            raise AssertionError(kind)


@pytest.mark.parametrize("count", [1, 2, 5, 10, 16, 18, 24])
def test_moduli_pairwise_coprime_greedy(count):
    mods = o2.choose_moduli(count)
    assert len(mods) == count and mods[0] == 256 and all(2 <= q <= 256 for q in mods)
    for a, b in itertools.combinations(mods, 2):
        assert math.gcd(a, b) == 1
    # greedy maximality: every skipped integer above the smallest chosen shares a
    # factor with a LARGER chosen modulus
    chosen = set(mods)
    for c in range(min(mods) + 1, 257):
        if c not in chosen:
            assert any(math.gcd(c, q) > 1 for q in mods if q > c), c
    with pytest.raises(ValueError):
        o2.choose_moduli(0)


@pytest.mark.parametrize("count,k", [(6, 8), (10, 256), (12, 100), (14, 1000), (16, 1024), (18, 4096)])
def test_nu_is_the_largest_safe_budget(count, k):
    """k 2^(2 nu) <= M/2 (the exact product fits the CRT range) and nu+1 would not."""
    M = o2.modulus_product(o2.choose_moduli(count))
    nu = o2.nu_bits(count, k)
    kp = 1 << max(0, (k - 1).bit_length())
    assert kp * (1 << (2 * nu)) * 2 <= M
    if nu < o2.NU_CAP:
        assert kp * (1 << (2 * (nu + 1))) * 2 > M
    with pytest.raises(ValueError):
        o2.nu_bits(1, 1 << 10)


# ----------------------------------------------------------------- R20 CRT
def test_crt_bruteforce_small_moduli():
    mods = [3, 5, 7]
    M = 105
    for z in range(-(M // 2), M // 2 + 1):
        assert o2.crt([z % p for p in mods], mods) == z
    mods = [4, 9, 5]
    M = 180
    for z in range(-M // 2 + 1, M // 2 + 1):
        assert o2.crt([z % p for p in mods], mods) == z


def test_crt_wide_values():
    mods = o2.choose_moduli(18)
    M = o2.modulus_product(mods)
    rng = np.random.default_rng(0)
    for _ in range(200):
        z = int(rng.integers(-2**62, 2**62)) * int(rng.integers(1, 2**62)) * int(rng.integers(1, 2**15))
        z = z % M
        if 2 * z > M:
            z -= M
        assert o2.crt([z % p for p in mods], mods) == z


# ----------------------------------------------------------------- R17 / R18
def test_quantize_bounds_and_bruteforce():
    X = synth.spread(9, 23, seed=5, phi=3.0)
    X[3] = 0.0
    nu = 20
    Q, e, nf = o2.quantize_rows(X, nu)
    assert not nf.any() and e[3] == 0 and (Q[3] == 0).all()
    assert (np.abs(Q) < 2**nu).all()
    for i in range(9):
        if i == 3:
            continue
        M = np.abs(X[i]).max()
        assert M < 2.0 ** e[i]
        for j in range(23):
            exact = Fraction(X[i, j]) * Fraction(2) ** (nu - int(e[i]))
            q = round(exact)                                   # Python: ties to even
            assert Q[i, j] == q
            assert abs(Fraction(X[i, j]) - Fraction(int(Q[i, j])) * Fraction(2) ** (int(e[i]) - nu)) \
                <= Fraction(2) ** (int(e[i]) - nu - 1)


def test_quantize_integers_exact_and_bump():
    # integer row within nu bits: exact, e = nu when max in [2^(nu-1), 2^nu)
    nu = 12
    x = np.array([[4000.0, -3.0, 17.0, 0.0]])
    Q, e, _ = o2.quantize_rows(x, nu)
    assert e[0] == 12 and (Q[0] == x[0]).all()
    # max just below 2^e but RNE reaches 2^nu -> exponent bumped
    x = np.array([[1.0 - 2.0**-30, 0.25]])
    Q, e, _ = o2.quantize_rows(x, 8)
    assert e[0] == 1 and Q[0, 0] == 128 and Q[0, 1] == 32
    x = np.array([[np.inf, 1.0]])
    _, _, nf = o2.quantize_rows(x, 8)
    assert nf[0]


def test_residues_centered_and_congruent():
    Q = np.arange(-600, 601, dtype=np.int64).reshape(1, -1)
    for p in (256, 255, 253, 7, 2):
        r = o2.residues(Q, p)
        assert ((Q - r.astype(np.int64)) % p == 0).all()
        lo = -(p // 2)
        hi = (p - 1) // 2
        assert r.min() >= lo and r.max() <= hi


# ----------------------------------------------------------------- R19 + R20
@pytest.mark.parametrize("count,k", [(8, 40), (12, 129), (16, 300)])
def test_two_routes_agree(count, k):
    """Residue GEMMs + CRT == the direct exact integer product (quantised inputs)."""
    A = synth.spread(7, k, seed=11, phi=2.0)
    Bt = synth.spread(5, k, seed=12, phi=2.0)
    nu = o2.nu_bits(count, k)
    QA, _, _ = o2.quantize_rows(A, nu)
    QB, _, _ = o2.quantize_rows(Bt, nu)
    Zd = o2.int_product(QA, QB)
    Zc = o2.crt_product(QA, QB, count)
    # the direct product also against Python integers (no int128 tricks)
    for i in range(7):
        for j in range(5):
            zz = sum(int(a) * int(b) for a, b in zip(QA[i], QB[j]))
            assert Zd[i, j] == zz == Zc[i, j]
    # every residue GEMM equals the exact product mod p, centered (commutes)
    for p in o2.choose_moduli(count):
        C = o2.residue_gemm(o2.residues(QA, p), o2.residues(QB, p), p)
        for i in range(7):
            for j in range(5):
                r = Zd[i, j] % p
                r = r - p if r >= (p + 1) // 2 else r
                assert C[i, j] == r


def test_product_fraction_bruteforce_tiny():
    """Whole Ozaki-II product on a 3x4x2 problem from first principles."""
    A = synth.spread(3, 4, seed=21, phi=1.5)
    B = synth.spread(4, 2, seed=22, phi=1.5)
    count = 6
    nu = o2.nu_bits(count, 4)
    P = o2.emulated_product(A, B, count, route="crt")
    for i in range(3):
        M = max(abs(Fraction(x)) for x in A[i])
        e = math.frexp(float(M))[1]
        if round(M * Fraction(2) ** (nu - e)) >= 2**nu:
            e += 1
        for j in range(2):
            N = max(abs(Fraction(x)) for x in B[:, j])
            f = math.frexp(float(N))[1]
            if round(N * Fraction(2) ** (nu - f)) >= 2**nu:
                f += 1
            z = sum(round(Fraction(A[i, t]) * Fraction(2) ** (nu - e)) *
                    round(Fraction(B[t, j]) * Fraction(2) ** (nu - f)) for t in range(4))
            assert P[i, j] == float(Fraction(z) * Fraction(2) ** (e + f - 2 * nu))


def test_error_is_pure_quantization_bound():
    """|P - AB| <= sum_k (|a| 2^(f-nu-1) + |b| 2^(e-nu-1) + 2^(e+f-2nu-2)) + ulp/2(P)."""
    m, k, n = 12, 64, 9
    A = synth.spread(m, k, seed=31, phi=2.0)
    B = synth.spread(k, n, seed=32, phi=2.0)
    count = 10
    nu = o2.nu_bits(count, k)
    P = o2.emulated_product(A, B, count, route="direct")
    _, e, _ = o2.quantize_rows(A, nu)
    _, f, _ = o2.quantize_rows(B.T, nu)
    T = oracle.exact_product(A, B)
    for i in range(m):
        for j in range(n):
            bound = sum(abs(A[i, t]) * 2.0 ** (f[j] - nu - 1) + abs(B[t, j]) * 2.0 ** (e[i] - nu - 1)
                        + 2.0 ** (e[i] + f[j] - 2 * nu - 2) for t in range(k))
            assert abs(P[i, j] - T[i, j]) <= bound * (1 + 1e-12) + np.spacing(abs(P[i, j]))


def test_integer_inputs_exact():
    A = synth.integer(20, 30, seed=41, bits=10)
    B = synth.integer(30, 11, seed=42, bits=10)
    P = o2.emulated_product(A, B, 8, route="direct")     # nu(8, 30) well above 10 bits
    assert (P == A @ B).all()


def test_scale_invariance_rows():
    A = synth.spread(6, 33, seed=51, phi=2.0)
    B = synth.spread(33, 7, seed=52, phi=2.0)
    P = o2.emulated_product(A, B, 12, route="direct")
    A2 = A.copy()
    A2[2] *= 2.0**37
    A2[4] *= 2.0**-300
    P2 = o2.emulated_product(A2, B, 12, route="direct")
    assert (P2[2] == P[2] * 2.0**37).all() and (P2[4] == P[4] * 2.0**-300).all()
    assert (np.delete(P2, [2, 4], 0) == np.delete(P, [2, 4], 0)).all()


def test_monotone_in_moduli_count():
    A = synth.uniform(24, 96, seed=61)
    B = synth.uniform(96, 20, seed=62)
    T = oracle.exact_product(A, B)
    prev = np.inf
    for count in (8, 10, 12, 14, 16):
        P = o2.emulated_product(A, B, count, route="direct")
        err = np.max(np.abs(P - T) / (np.abs(A) @ np.abs(B)))
        assert err <= prev
        if count <= 12:
            assert err < prev / 64 or prev == np.inf
        prev = err
    assert prev < 1e-15


def test_zgemm_identity_and_real_inputs():
    """a = i I gives C = i B (SURVEY §8(c) complex pins; B integer-valued so its
    quantisation is exact), real inputs give Im == 0."""
    n = 6
    B = synth.make("integer", n, 5, seed=71, complex_=True, bits=12)
    A = np.eye(n) * 1j
    C = o2.zgemm("N", "N", 1.0, A, B, 0.0, None, 12)
    assert (C.real == -B.imag).all() and (C.imag == B.real).all()
    Ar = synth.uniform(5, 7, seed=72).astype(np.complex128)
    Br = synth.uniform(7, 4, seed=73).astype(np.complex128)
    C = o2.zgemm("N", "N", 1.0, Ar, Br, 0.0, None, 12)
    assert (C.imag == 0).all()
