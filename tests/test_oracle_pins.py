"""Pins for the CPU oracle (-m "not gpu").

Every oracle function is checked against something other than itself:
hand-derived golden values (tests/golden/), exact rational brute force
(oracle/brute.py, written independently of the C code), closed forms and
invariants.  The readings R1..R15 referenced here are listed in DESIGN.md §3.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_lines(name):
    with open(os.path.join(GOLD, name)) as fh:
        return [ln.strip() for ln in fh if ln.strip() and not ln.startswith("#")]


# ------------------------------------------------------------------ golden pins
def test_hand_digits_golden(orc):
    """R3/R4 against hand derivations (tests/golden/hand_digits.txt)."""
    for ln in _golden_lines("hand_digits.txt"):
        row_s, s_s, e_s, d_s = [x.strip() for x in ln.split("|")]
        row = [float(x) for x in row_s.split()]
        s, e_exp = int(s_s), int(e_s)
        e, nf = orc.exponent(np.array(row))
        assert not nf and e == e_exp, ln
        want = [[int(v) for v in part.split()] for part in d_s.split(";")]
        for x, w in zip(row, want):
            assert list(orc.digits(x, e, s)) == w, (ln, x)


def test_spec_int8_example(orc):
    """SPEC.md:50 worked example used as one slice (s=1): S_2 = dA . dB^T."""
    g = {}
    for ln in _golden_lines("spec_int8_2x2.txt"):
        k, v = ln.split(":")
        g[k] = np.array([int(x) for x in v.split()]).reshape(2, 2)
    DA = g["A"].astype(np.int8)[None]
    DB = g["B"].T.copy().astype(np.int8)[None]  # columns of b as rows
    S = orc.level_sums(DA, DB, 1)
    assert (S[0] == g["S"]).all()


def test_paper_modes_golden(orc):
    """PAPER.md:119 mode labels <-> slice counts (reading R2: bits = 8s-1)."""
    rows = [tuple(int(x) for x in ln.split()) for ln in _golden_lines("paper_modes.txt")]
    for bits, s in rows:
        assert 8 * s - 1 == bits
        # one slice set of s slices can carry 8s-1 significant bits: the top
        # digit is in [-127,127] (7 bits + sign) and s-1 full bytes follow
        X_max = 127 * 256 ** (s - 1) + sum(127 * 256 ** j for j in range(s - 1))
        assert X_max < 2 ** bits
        assert orc.pairs(s) == s * (s + 1) // 2


# -------------------------------------------------------- O2 exponent (R3) pins
def _exp_cases():
    g = synth.rng(11)
    rows = [
        [0.0, 0.0],
        [1.0], [0.5], [2.0 ** -1074], [2.0 ** -1074 * 3], [2.0 ** -1022],
        [1.7976931348623157e308], [127.0], [127.0 * 2 ** -10], [127.5],
        [np.nextafter(127.0, 200.0)], [127.25 * 2 ** 40], [-128.0], [63.999],
        [1.984375], [np.nextafter(1.984375, 3.0)],
    ]
    for _ in range(200):
        n = int(g.integers(1, 6))
        rows.append(list(g.uniform(-1, 1, n) * np.exp(g.normal(0, 30, n))))
    return rows


def test_exponent_vs_definition(orc):
    for row in _exp_cases():
        e, nf = orc.exponent(np.array(row, dtype=np.float64))
        assert not nf
        assert e == brute.exponent_def(row), row


def test_exponent_nonfinite(orc):
    for bad in (np.inf, -np.inf, np.nan):
        e, nf = orc.exponent(np.array([1.0, bad, 3.0]))
        assert nf


# ------------------------------------------------------ O3/O4 digits (R4) pins
@pytest.mark.parametrize("s", list(range(1, 17)))
def test_digits_vs_bruteforce(orc, s):
    g = synth.rng(100 + s)
    for trial in range(60):
        n = int(g.integers(1, 5))
        row = list(g.uniform(-1, 1, n) * np.exp(g.normal(0, 8, n)))
        if trial % 7 == 0:
            row[0] = 2.0 ** -1074 * int(g.integers(1, 100))
        if trial % 11 == 0:
            row = [float(v) for v in g.integers(-127, 128, n)]
        e, _ = orc.exponent(np.array(row))
        for x in row:
            d = orc.digits(x, e, s)
            X = brute.integerise(x, e, s)
            assert list(d) == brute.balanced_digits(X, s), (x, e, s)
            # reconstruction is exact and digit ranges hold
            assert sum(int(dt) * 256 ** (s - 1 - t) for t, dt in enumerate(d)) == X
            assert -127 <= d[0] <= 127
            # rounding bound |x - X 2^(e-P)| <= 2^(e-8s)
            err = abs(Fraction(x) - Fraction(X) * Fraction(2) ** (e - (8 * s - 1)))
            assert err <= Fraction(2) ** (e - 8 * s)


def test_integer_row_special_case(orc):
    """Integer row with max |x| in [64,127]: e = 7 and d_1 = x, others 0."""
    g = synth.rng(5)
    for _ in range(50):
        row = g.integers(-127, 128, 9).astype(float)
        row[0] = float(g.choice([-1, 1]) * g.integers(64, 128))
        e, _ = orc.exponent(row)
        assert e == 7
        for s in (1, 3, 8):
            for x in row:
                d = orc.digits(x, e, s)
                assert d[0] == int(x) and not d[1:].any()


# ---------------------------------------------------------- O5 level sums pins
def test_level_sums_vs_bruteforce(orc):
    g = synth.rng(21)
    for s in (1, 2, 3, 5, 8):
        m, n, k = 3, 4, 5
        DA = g.integers(-128, 128, (s, m, k)).astype(np.int8)
        DB = g.integers(-128, 128, (s, n, k)).astype(np.int8)
        S = orc.level_sums(DA, DB, s)
        Sb = brute.level_sums(DA.tolist(), DB.tolist(), s)
        assert (S == np.array(Sb)).all()


def test_level_sums_closed_forms(orc):
    # all-ones, K = 3*2^16: every entry = 3*2^16
    k = 3 * 2 ** 16
    S = orc.level_sums(np.ones((1, 1, k), np.int8), np.ones((1, 1, k), np.int8), 1)
    assert S[0, 0, 0] == 3 * 2 ** 16
    # worst case -128 x -128: 131071 products fit INT32, 131072 reach 2^31 exactly
    # (SPEC.md:45/51's "2^17 products" bound is off by one)
    for kk, want in ((131071, 2 ** 31 - 2 ** 14), (131072, 2 ** 31)):
        D = np.full((1, 1, kk), -128, np.int8)
        assert orc.level_sums(D, D, 1)[0, 0, 0] == want
    # level L has L-1 pairs: with all digits 1, S_L = (L-1) k for L <= s+1
    s, kk = 5, 7
    D = np.ones((s, 2, kk), np.int8)
    S = orc.level_sums(D, D, s)
    for L in range(2, s + 2):
        assert (S[L - 2] == (L - 1) * kk).all()


# ------------------------------------------------------------ O6 combine pins
@pytest.mark.parametrize("s", [1, 2, 3, 4, 6, 8, 9, 12])
def test_emulated_within_1ulp_of_retained_sum(orc, s):
    """R6: the FP64 ascending combine is within 1 ulp of the exact retained sum."""
    g = synth.rng(300 + s)
    for trial in range(4):
        m, n, k = 3, 3, int(g.integers(1, 6))
        fam = ("uniform", "spread")[trial % 2]
        A = synth.make(fam, m, k, 1000 * s + trial) if fam == "uniform" else \
            synth.spread(m, k, 1000 * s + trial, phi=3.0)
        B = synth.uniform(k, n, 2000 * s + trial)
        P = orc.emulated_product(A, B, s)
        Pex, e, f, S, _, _ = brute.retained_exact(A.tolist(), B.T.tolist(), s)
        Sc = orc.level_sums(*[orc.split_rows(X, s)[0] for X in (A, B.T)], s)
        assert (Sc == np.array(S)).all()
        for i in range(m):
            for j in range(n):
                ex = Pex[i][j]
                if ex == 0:
                    assert P[i, j] == 0.0
                else:
                    assert abs(Fraction(P[i, j]) - ex) <= Fraction(math.ulp(float(ex)))


@pytest.mark.parametrize("s", [1, 2, 4, 7, 8])
def test_closed_form_error_bound_bruteforce(orc, s):
    """|P_exact - (AB)_ij| <= (s+1) k 2^(e_i+f_j-8s)  (SURVEY.md §8(c) bound)."""
    g = synth.rng(400 + s)
    for trial in range(4):
        m, n, k = 2, 3, int(g.integers(1, 7))
        A = synth.spread(m, k, 10 * s + trial, phi=2.0)
        B = synth.spread(k, n, 20 * s + trial, phi=2.0)
        Pex, e, f, _, _, _ = brute.retained_exact(A.tolist(), B.T.tolist(), s)
        T = brute.true_product(A.tolist(), B.T.tolist())
        for i in range(m):
            for j in range(n):
                bound = Fraction(s + 1) * k * Fraction(2) ** (e[i] + f[j] - 8 * s)
                assert abs(Pex[i][j] - T[i][j]) <= bound


@pytest.mark.parametrize("s", [3, 4, 5, 6, 7, 8])
def test_error_bound_64cube(orc, s):
    """Same bound at C1 size (64^3) with the exact product as truth."""
    A = synth.uniform(64, 64, 1)
    B = synth.uniform(64, 64, 2)
    P = orc.emulated_product(A, B, s)
    T = orc.exact_product(A, B)
    e = np.array([orc.exponent(A[i])[0] for i in range(64)])
    f = np.array([orc.exponent(B[:, j])[0] for j in range(64)])
    bound = (s + 1) * 64 * np.exp2(e[:, None] + f[None, :] - 8.0 * s)
    # + the FP64 rounding of the combine (1 ulp, R6)
    bound = bound + np.spacing(np.abs(T)) * 2
    assert (np.abs(P - T) <= bound).all()


def test_monotone_in_s(orc):
    """Max error falls by >= 2^6 per slice until it reaches the FP64 floor."""
    A = synth.uniform(48, 48, 3)
    B = synth.uniform(48, 48, 4)
    T = orc.exact_product(A, B)
    absab = np.abs(A) @ np.abs(B)
    # componentwise metric (reading R13 ii): stable where T ~ 0
    errs = [np.max(np.abs(orc.emulated_product(A, B, s) - T) / absab) for s in range(1, 10)]
    floor = 2.0 ** -53  # one FP64 rounding of the result
    for s in range(1, 9):
        if errs[s - 1] > 64 * floor:
            assert errs[s] <= errs[s - 1] / 64.0, errs
        else:
            assert errs[s] <= 2 * floor, errs


@pytest.mark.parametrize("bits", [7, 8, 10, 15, 16, 23])
def test_integer_exactness_condition(orc, bits):
    """Integer inputs: exact iff T(e_i)+T(f_j) <= s+1 with T(e)=max(1,ceil((e+1)/8))."""
    A = synth.integer(16, 24, 7, bits=bits)
    B = synth.integer(24, 16, 8, bits=bits)
    T = orc.exact_product(A, B)
    e = np.array([orc.exponent(A[i])[0] for i in range(A.shape[0])])
    f = np.array([orc.exponent(B[:, j])[0] for j in range(B.shape[1])])

    def Tn(x):
        return np.maximum(1, np.ceil((x + 1) / 8.0))

    for s in range(1, 9):
        P = orc.emulated_product(A, B, s)
        pred = (Tn(e)[:, None] + Tn(f)[None, :]) <= s + 1
        assert (P[pred] == T[pred]).all()
        if s == 1 and bits == 7:
            assert pred.all()  # plain INT8 GEMM special case


def test_scale_invariance_bitwise(orc):
    """Scaling row i of A by 2^p scales row i of P by exactly 2^p."""
    A = synth.spread(8, 20, 9, phi=1.0)
    B = synth.uniform(20, 6, 10)
    for s in (3, 7):
        P = orc.emulated_product(A, B, s)
        for p in (-700, -3, 5, 300):
            A2 = A.copy()
            A2[2] = np.ldexp(A2[2], p)
            P2 = orc.emulated_product(A2, B, s)
            assert (P2[2] == np.ldexp(P[2], p)).all()
            assert (np.delete(P2, 2, 0) == np.delete(P, 2, 0)).all()


def test_s8_beats_native_fp64(orc):
    """s = 8 at least as accurate as the FP64 triple loop on benign data."""
    A = synth.uniform(64, 64, 12)
    B = synth.uniform(64, 64, 13)
    T = orc.exact_product(A, B)
    e8 = np.max(np.abs(orc.emulated_product(A, B, 8) - T))
    en = np.max(np.abs(orc.fp64_product(A, B) - T))
    assert e8 <= en


# ------------------------------------------------------------- truth (Kulisch)
def test_exact_dot_vs_fraction(orc):
    g = synth.rng(77)
    for trial in range(200):
        k = int(g.integers(1, 12))
        a = g.uniform(-1, 1, k) * np.exp(g.normal(0, 40, k))
        b = g.uniform(-1, 1, k) * np.exp(g.normal(0, 40, k))
        if trial % 5 == 0:  # cancellation: sum = 1 after 1e16-scale terms
            a = np.array([1e16, 1.0, -1e16])
            b = np.array([1.0, 1.0, 1.0])
        if trial % 9 == 0:  # subnormal products
            a = np.array([2.0 ** -1074, 3 * 2.0 ** -1060, 1e-300])
            b = np.array([2.0 ** 60, 2.0 ** -10, -1e-20])
        ex = sum((Fraction(x) * Fraction(y) for x, y in zip(a, b)), Fraction(0))
        got = orc.exact_dot(a, b)
        # reference rounding of the Fraction: float(Fraction) is correctly rounded
        assert got == float(ex), (a, b)


def test_exact_gemm_integer_and_fp64_loop(orc):
    A = synth.integer(10, 30, 1, bits=20)
    B = synth.integer(30, 12, 2, bits=20)
    Tex = orc.exact_product(A, B)
    assert (Tex == (A.astype(object) @ B.astype(object)).astype(float)).all()
    Tn = orc.fp64_product(A, B)
    assert (Tn == Tex).all()  # integer products < 2^53: native FP64 is exact too
    U = synth.uniform(20, 40, 3)
    V = synth.uniform(40, 20, 4)
    Tu = orc.exact_product(U, V)
    Tf = orc.fp64_product(U, V)
    absab = np.abs(U) @ np.abs(V)
    assert (np.abs(Tf - Tu) <= 40 * 2.0 ** -53 * absab * 1.01).all()


# ---------------------------------------------------------------- O7 and BLAS
def test_dgemm_alpha_beta_and_quick_returns(orc):
    A = synth.uniform(5, 4, 1)
    B = synth.uniform(4, 3, 2)
    C = synth.uniform(5, 3, 3)
    s = 6
    P = orc.emulated_product(A, B, s)
    out = orc.dgemm("N", "N", -1.5, A, B, 0.25, C, s)
    assert (out == np.vectorize(lambda p, c: float(Fraction(-1.5) * Fraction(p) + Fraction(0.25) * Fraction(c)))(P, C)).all()
    Cnan = np.full((5, 3), np.nan)
    assert (orc.dgemm("N", "N", 1.0, A, B, 0.0, Cnan, s) == P).all()     # beta=0: C not read
    assert (orc.dgemm("N", "N", 0.0, A, B, 1.0, C, s) == C).all()        # alpha=0, beta=1
    assert (orc.dgemm("N", "N", 0.0, A, B, 0.0, Cnan, s) == 0).all()     # alpha=0, beta=0
    assert (orc.dgemm("N", "N", 0.0, A, B, 2.0, C, s) == 2 * C).all()
    # transposes: op() only re-indexes
    assert (orc.dgemm("T", "N", 1.0, A.T.copy(), B, 0.0, None, s) == P).all()
    assert (orc.dgemm("N", "T", 1.0, A, B.T.copy(), 0.0, None, s) == P).all()
    assert (orc.dgemm("C", "C", 1.0, A.T.copy(), B.T.copy(), 0.0, None, s) == P).all()


def test_nonfinite_rows_propagate(orc):
    A = synth.uniform(4, 5, 1)
    B = synth.uniform(5, 3, 2)
    A[1, 2] = np.inf
    B[0, 2] = np.nan
    P = orc.emulated_product(A, B, 4)
    assert np.isnan(P[1]).all() and np.isnan(P[:, 2]).all()
    ok = np.ones_like(P, bool)
    ok[1] = False
    ok[:, 2] = False
    assert np.isfinite(P[ok]).all()


# ------------------------------------------------------------------- complex
def test_complex_special_cases(orc):
    """a = iI -> C_re = -Bi, C_im = Br; real inputs -> Im == 0."""
    n = 12
    B = synth.integer(n, 7, 4, bits=10, complex_=True)
    iI = 1j * np.eye(n)
    for method in ("4m", "3m"):
        C = orc.zgemm("N", "N", 1.0, iI, B, 0.0, None, 4, method)
        assert (C.real == -B.imag).all() and (C.imag == B.real).all()
        Ar = synth.uniform(6, n, 5).astype(np.complex128)
        Cr = orc.zgemm("N", "N", 1.0, Ar, B.real.astype(np.complex128), 0.0, None, 5, method)
        assert (Cr.imag == 0).all()


@pytest.mark.parametrize("method", ["4m", "3m"])
def test_complex_within_bound_and_conjugation(orc, method):
    A = synth.kkr(40, 40, 1, gamma=1.0)
    B = synth.kkr(40, 40, 2, gamma=1.0)
    T = orc.exact_zproduct(A, B)
    absab = np.abs(A) @ np.abs(B)
    prev = None
    for s in (4, 6, 8):
        C = orc.zgemm("N", "N", 1.0, A, B, 0.0, None, s, method)
        err = np.max(np.abs(C - T) / absab)
        assert err <= 4 * 40 * 2.0 ** (-8 * s + 10) + 1e-15
        if prev is not None:
            assert err <= prev
        prev = err
        # conjugation symmetry within mode precision
        Cc = orc.zgemm("N", "N", 1.0, np.conj(A), np.conj(B), 0.0, None, s, method)
        assert np.max(np.abs(np.conj(Cc) - C) / absab) <= 8 * 40 * 2.0 ** (-8 * s + 10) + 1e-15
    # 'C' flag is conj-transpose: materialised op() gives the same bits
    Cc1 = orc.zgemm("C", "N", 1.0, np.conj(A.T).copy(), B, 0.0, None, 5, method)
    Cn1 = orc.zgemm("N", "N", 1.0, A, B, 0.0, None, 5, method)
    assert (Cc1 == Cn1).all()


def test_complex_alpha_beta(orc):
    A = synth.uniform(6, 5, 1, complex_=True)
    B = synth.uniform(5, 4, 2, complex_=True)
    C = synth.uniform(6, 4, 3, complex_=True)
    al, be = 0.5 - 1.25j, -0.75 + 0.5j
    Pr, Pi = orc.zproduct(A, B, 7, "4m")
    out = orc.zgemm("N", "N", al, A, B, be, C, 7, "4m")
    P = Pr + 1j * Pi
    ref = al * P + be * C
    assert np.max(np.abs(out - ref)) <= 8 * 2.0 ** -53 * np.max(np.abs(ref))
    Cnan = np.full((6, 4), np.nan + 0j)
    o0 = orc.zgemm("N", "N", 1.0, A, B, 0.0, Cnan, 7, "4m")
    assert (o0.real == Pr).all() and (o0.imag == Pi).all()
    assert (orc.zgemm("N", "N", 0.0, A, B, 1.0, C, 7) == C).all()


def test_combine_order_golden(orc):
    """R6 order pinned by hand-derived values (tests/golden/combine_order.txt)."""
    for ln in _golden_lines("combine_order.txt"):
        lhs, want = ln.split("|")
        s, e, f, *S = [int(x) for x in lhs.split()]
        Sarr = np.array(S, dtype=np.int64).reshape(s, 1, 1)
        P = orc.combine(Sarr, [e], [0], [f], [0], s)
        assert P[0, 0] == float(int(want)), ln


# ------------------------------------------------- R9 complex embedding pins
def _hexs(s):
    return [float.fromhex(x) for x in s.split()]


def test_complex_embedding_golden(orc):
    """R9 by hand (tests/golden/complex_embedding.txt): the 4M N-side embedding and the 3M
    combine; the A-side 4M embedding gives different bits on the same input."""
    for ln in _golden_lines("complex_embedding.txt"):
        meth, s_s, a_s, b_s, want_s, alt_s = [x.strip() for x in ln.split("|")]
        ar, ai = _hexs(a_s)
        br, bi = _hexs(b_s)
        wr, wi = _hexs(want_s)
        A = np.array([[complex(ar, ai)]])
        B = np.array([[complex(br, bi)]])
        C = orc.zgemm("N", "N", 1.0, A, B, 0.0, None, int(s_s), meth)
        assert C[0, 0].real == wr and C[0, 0].imag == wi, (ln, C[0, 0])
        if alt_s != "-":
            assert C[0, 0].real != float.fromhex(alt_s)


def _embedded_rows_nside(Aop, Bop):
    """R9 N-side embedding written out as rational rows: A' row i = [Ar_i | Ai_i];
    B'^T rows 2j = [Br_j | -Bi_j] (Re output), 2j+1 = [Bi_j | Br_j] (Im output)."""
    Ar = [[Fraction(float(x.real)) for x in r] + [Fraction(float(x.imag)) for x in r] for r in Aop]
    Bt = []
    for j in range(Bop.shape[1]):
        col = Bop[:, j]
        Bt.append([Fraction(float(x.real)) for x in col] + [-Fraction(float(x.imag)) for x in col])
        Bt.append([Fraction(float(x.imag)) for x in col] + [Fraction(float(x.real)) for x in col])
    return Ar, Bt


def _embedded_rows_aside(Aop, Bop):
    """SURVEY's A-side embedding: rows [Ar | -Ai] (Re) and [Ai | Ar] (Im) against [Br; Bi]."""
    Ar = [[Fraction(float(x.real)) for x in r] + [-Fraction(float(x.imag)) for x in r] for r in Aop]
    Ar += [[Fraction(float(x.imag)) for x in r] + [Fraction(float(x.real)) for x in r] for r in Aop]
    Bt = [[Fraction(float(x.real)) for x in Bop[:, j]] + [Fraction(float(x.imag)) for x in Bop[:, j]]
          for j in range(Bop.shape[1])]
    return Ar, Bt


@pytest.mark.parametrize("s", [2, 3, 4])
def test_4m_is_nside_embedding_bruteforce(orc, s):
    """R9: the oracle's 4M product equals (within R6's 1 ulp) the exact retained sum of the
    N-side embedding, computed by oracle/brute.py from the definitions.  Digits of -x differ
    from -digits(x) only when a low byte of X is 0x80, so the crafted half of the inputs puts
    X(Ai) = odd * 128 (row exponent 1): there the A-side embedding's retained sum is more
    than 2 ulp away for some entry (the top digits of -X and X differ by the carry), so the pin tells the two readings apart."""
    g = synth.rng(900 + s)
    separated = 0
    for trial in range(6):
        m, n, k = 2, 2, int(g.integers(1, 4))
        if trial % 2 == 0:
            A = synth.spread(m, k, 40 * s + trial, phi=2.0, complex_=True)
            B = synth.spread(k, n, 50 * s + trial, phi=2.0, complex_=True)
        else:   # Ar = Br = 1 set e = f = 1, so X = x 2^(8s-2): X(Ai) = 2^(8s-3) + odd*128
            # (low byte 0x80, a carry into the next digit), X(Bi) = odd*256 + odd
            odd = lambda shape: 2 * g.integers(0, 32, shape) + 1  # noqa: E731
            A = 1.0 + 1j * (0.5 + odd((m, k)) * 2.0 ** (9 - 8 * s))
            B = 1.0 + 1j * (odd((k, n)) * 256 + odd((k, n))) * 2.0 ** (2 - 8 * s)
        Pr, Pi = orc.zproduct(A, B, s, "4m")
        Arn, Btn = _embedded_rows_nside(A, B)
        Pn, *_ = brute.retained_exact(Arn, Btn, s)
        Ara, Bta = _embedded_rows_aside(A, B)
        Pa, *_ = brute.retained_exact(Ara, Bta, s)
        for i in range(m):
            for j in range(n):
                for got, exn, exa in ((Pr[i, j], Pn[i][2 * j], Pa[i][j]),
                                      (Pi[i, j], Pn[i][2 * j + 1], Pa[m + i][j])):
                    u = Fraction(math.ulp(float(exn))) if exn != 0 else Fraction(0)
                    assert abs(Fraction(got) - exn) <= u
                    if abs(Fraction(got) - exa) > 2 * u:
                        separated += 1
    assert separated > 0


# ---------------------------------------------- R7 quick return, complex beta
@pytest.mark.parametrize("beta", [0.5 - 0.75j, -1.25 + 0.375j, 0.0 + 2.0j, -3.0 + 0.0j])
def test_quick_complex_beta_exact(orc, beta):
    """R7 quick return (alpha = 0 and k = 0) with a complex beta: C <- beta C.  Dyadic inputs
    make every FP64 step of the fma shapes exact, so the result must equal the exact rational
    product (Fraction) -- a sign or swapped index in the beta_i terms fails."""
    g = synth.rng(77)
    m, n = 5, 4
    C = (g.integers(-64, 65, (m, n)) + 1j * g.integers(-64, 65, (m, n))) / 32.0
    br, bi = Fraction(beta.real), Fraction(beta.imag)
    want_r = [[br * Fraction(C[i, j].real) - bi * Fraction(C[i, j].imag) for j in range(n)] for i in range(m)]
    want_i = [[br * Fraction(C[i, j].imag) + bi * Fraction(C[i, j].real) for j in range(n)] for i in range(m)]
    A = synth.uniform(m, 3, 1, complex_=True)
    B = synth.uniform(3, n, 2, complex_=True)
    for out in (orc.zgemm("N", "N", 0.0, A, B, beta, C, 7, "4m"),
                orc.zgemm("N", "N", 0.0, A, B, beta, C, 7, "3m"),
                orc.zgemm("N", "N", 1.0 + 1.0j, A[:, :0], B[:0, :], beta, C, 7, "4m")):
        for i in range(m):
            for j in range(n):
                assert Fraction(out[i, j].real) == want_r[i][j]
                assert Fraction(out[i, j].imag) == want_i[i][j]


def test_quick_complex_beta_rounded(orc):
    """Non-dyadic data: each component of the quick return is within 2u (|br c| + |bi c'|) of
    the exact beta C (R7's two fma shapes round at most twice)."""
    m, n = 7, 6
    C = synth.uniform(m, n, 5, complex_=True)
    beta = 0.3 - 0.7j
    out = orc.zgemm("N", "N", 0.0, np.zeros((m, 2), complex), np.zeros((2, n), complex), beta, C, 5)
    br, bi = Fraction(beta.real), Fraction(beta.imag)
    u = Fraction(2) ** -53
    for i in range(m):
        for j in range(n):
            cr, ci = Fraction(C[i, j].real), Fraction(C[i, j].imag)
            er, ei = br * cr - bi * ci, br * ci + bi * cr
            assert abs(Fraction(out[i, j].real) - er) <= 2 * u * (abs(br * cr) + abs(bi * ci))
            assert abs(Fraction(out[i, j].imag) - ei) <= 2 * u * (abs(br * ci) + abs(bi * cr))
    # beta == 0: C not read (NaN-safe), zeros
    Cn = np.full((m, n), np.nan + 1j * np.nan)
    z = orc.zgemm("N", "N", 0.0, np.zeros((m, 2), complex), np.zeros((2, n), complex), 0.0, Cn, 5)
    assert (z == 0).all()
