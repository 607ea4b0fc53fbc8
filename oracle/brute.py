"""Exact-rational brute force for tiny Ozaki-I cases -- pins the C oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written independently of
``ozaki_oracle.c``: exponents come from the *definition* (the least power of two
that bounds the row maximum with the 127-rule, searched over integers with
Fractions), digits from exact rational rounding, products in Python integers.

Definitions followed (DESIGN.md readings):
  R3  e = least integer with M < 2^e, bumped by one when M*2^(7-e) > 127.
  R4  X = round_half_even(x * 2^(8s-1-e)), balanced base-256 digits.
  R1  retained pairs t + u <= s + 1.
  R6  the retained sum sum_L S_L 2^(e+f+2-8L) (exact, as a Fraction).
"""
from __future__ import annotations

from fractions import Fraction


def exponent_def(row) -> int:
    """R3 from the definition (no frexp): least e with M < 2^e, then 127-rule."""
    M = max((abs(Fraction(x)) for x in row), default=Fraction(0))
    if M == 0:
        return 0
    e = 0
    while Fraction(2) ** e <= M:
        e += 1
    while Fraction(2) ** (e - 1) > M:
        e -= 1
    if M * Fraction(2) ** (7 - e) > 127:
        e += 1
    return e


def integerise(x, e: int, s: int) -> int:
    """R4: X = RNE(x * 2^(8s-1-e)) as a Python int (Fraction rounding is half-even)."""
    return round(Fraction(x) * Fraction(2) ** (8 * s - 1 - e))


def balanced_digits(X: int, s: int) -> list[int]:
    """Digits d_1..d_s with X = sum d_t 256^(s-t), d_t in [-128,127] for t >= 2.

    Computed by a different route than the C oracle: search the unique digit
    in [-128, 127] congruent to the remainder (instead of a sign-extended byte).
    """
    out = []
    for _ in range(s - 1):
        r = X % 256  # in [0, 255]
        d = r if r < 128 else r - 256
        out.append(d)
        X = (X - d) // 256
    out.append(X)
    return out[::-1]


def split(rows, s: int):
    """Returns (digits[s][r][l] nested lists, exps list)."""
    exps = [exponent_def(r) for r in rows]
    D = [[[0] * len(rows[0]) for _ in rows] for _ in range(s)]
    for i, r in enumerate(rows):
        for l, x in enumerate(r):
            ds = balanced_digits(integerise(x, exps[i], s), s)
            for t in range(s):
                D[t][i][l] = ds[t]
    return D, exps


def level_sums(DA, DB, s: int):
    """S[L-2][i][j] = sum over t+u = L of the exact integer dot products."""
    m, n, k = len(DA[0]), len(DB[0]), len(DA[0][0])
    S = [[[0] * n for _ in range(m)] for _ in range(s)]
    for L in range(2, s + 2):
        for i in range(m):
            for j in range(n):
                acc = 0
                for t in range(1, s + 1):
                    u = L - t
                    if 1 <= u <= s:
                        acc += sum(DA[t - 1][i][l] * DB[u - 1][j][l] for l in range(k))
                S[L - 2][i][j] = acc
    return S


def retained_exact(A_rows, Bt_rows, s: int):
    """Exact rational retained sum P_exact[i][j] and the exponents (e, f)."""
    DA, e = split(A_rows, s)
    DB, f = split(Bt_rows, s)
    S = level_sums(DA, DB, s)
    m, n = len(A_rows), len(Bt_rows)
    P = [[Fraction(0)] * n for _ in range(m)]
    for i in range(m):
        for j in range(n):
            P[i][j] = sum((Fraction(S[L - 2][i][j]) * Fraction(2) ** (e[i] + f[j] + 2 - 8 * L)
                           for L in range(2, s + 2)), Fraction(0))
    return P, e, f, S, DA, DB


def true_product(A_rows, Bt_rows):
    return [[sum((Fraction(a) * Fraction(b) for a, b in zip(ar, br)), Fraction(0))
             for br in Bt_rows] for ar in A_rows]


def ulp(x: float) -> float:
    import math
    return math.ulp(x)
