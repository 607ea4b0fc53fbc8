/*
 * ozaki_oracle.c -- CPU ORACLE for the INT8 Ozaki-I emulation of FP64 GEMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2603_29975_b200/) never links, imports or calls it,
 * and it shares no code, header, constant or helper with the CUDA path.
 *
 * What the paper fixes (§2.2):
 *   "Ozaki-I splits high-precision input matrices into slices as lower-precision
 *    components based on their significant bits and exponent alignment, then
 *    performs low-precision matrix multiplications on these slices and
 *    accumulates them in higher precision."
 * and the precision knob "mantissa bits 31, 39, 47, 55, 63" (§3.2),
 * read as bits = 8s - 1 for s slices (reading R2).
 * Everything below that sentence is a reading written down in DESIGN.md §3
 * (R1..R15); each function names the reading it follows.  Steps O1..O7 are the
 * ones of SURVEY.md §8(c).
 *
 * Conventions of this file (plain, slow, obviously correct):
 *   - op(A) is passed materialised (step O1 is done by the Python wrapper) as a
 *     row-major m x k array: row i of op(A) is contiguous.
 *   - op(B) is passed as its transpose, row-major n x k: column j of op(B) is
 *     contiguous.  So every "row exponent" / "column exponent" scan is a plain
 *     loop over one contiguous array.
 *   - outputs P / C are row-major m x n.
 *   - compiled with -ffp-contract=off: every + and * below is one IEEE
 *     round-to-nearest-even operation, fma() is the only fused operation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ------------------------------------------------------------------------- */
/* O2: exponent of one row (A) or column (B).                 reading R3      */
/*   M = max |x|.  M == 0  -> e = 0 (all digits will be 0).                    */
/*   else e = frexp exponent of M (M < 2^e), and if M * 2^(7-e) > 127 then    */
/*   e += 1 ("127-rule": keeps the top balanced digit inside [-127, 127]).     */
/*   A non-finite entry marks the whole row / column (reading R10).           */
/* ------------------------------------------------------------------------- */
int orc_exponent(const double *x, int64_t n, int *nonfinite)
{
    double M = 0.0;
    *nonfinite = 0;
    for (int64_t l = 0; l < n; ++l) {
        double a = fabs(x[l]);
        if (!isfinite(a))
            *nonfinite = 1;
        else if (a > M)
            M = a;
    }
    if (*nonfinite || M == 0.0)
        return 0;
    int e;
    (void)frexp(M, &e);
    if (ldexp(M, 7 - e) > 127.0)
        e += 1;
    return e;
}

/* ------------------------------------------------------------------------- */
/* O3 + O4: integerise and split one value into s balanced base-256 digits.   */
/*   P = 8s - 1;  X = RNE(x * 2^(P - e))   (reading R4/R5: fixed point, RNE)  */
/*   for t = s down to 2:  d_t = sign-extended low byte of X; X = (X - d_t)/256*/
/*   d_1 = X  (in [-127, 127] thanks to the 127-rule).                        */
/*   d[t-1] receives d_t (most significant first).                             */
/* Returns 0, or -1 if d_1 left [-127,127] (never happens for a valid e).     */
/* ------------------------------------------------------------------------- */
int orc_digits(double x, int e, int s, int8_t *d)
{
    const int P = 8 * s - 1;
    double v = nearbyint(ldexp(x, P - e)); /* default rounding mode = RNE */
    i128 X = (i128)v;                      /* exact: v is an integer < 2^127 */
    for (int t = s; t >= 2; --t) {
        int low = (int)(X & 0xff);
        if (low >= 128)
            low -= 256;
        d[t - 1] = (int8_t)low;
        X = (X - low) / 256;
    }
    if (X < -127 || X > 127)
        return -1;
    d[0] = (int8_t)X;
    return 0;
}

/* Split every row of a row-major rows x k matrix:                            */
/*   digits out: D[(t-1)*rows*k + r*k + l] = d_t of x[r][l]                  */
/*   exps[r], nonfinite[r].  Non-finite rows get all-zero digits.             */
int orc_split_rows(int64_t rows, int64_t k, const double *X, int s,
                   int8_t *D, int32_t *exps, int32_t *nonfinite)
{
    int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        int nf;
        int e = orc_exponent(X + r * k, k, &nf);
        exps[r] = e;
        nonfinite[r] = nf;
        int8_t d[16];
        for (int64_t l = 0; l < k; ++l) {
            if (nf) {
                memset(d, 0, sizeof d);
            } else if (orc_digits(X[r * k + l], e, s, d) != 0) {
                bad |= 1;
            }
            for (int t = 1; t <= s; ++t)
                D[(int64_t)(t - 1) * rows * k + r * k + l] = d[t - 1];
        }
    }
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------------- */
/* O5: level sums over the triangular pair set t + u = L <= s + 1 (reading    */
/* R1).  S[(L-2)*m*n + i*n + j] = sum_{t+u=L} sum_l dA_t[i][l] * dB_u[j][l]   */
/* in exact int64 (no INT32 limit here: the oracle never chunks).             */
/* ------------------------------------------------------------------------- */
void orc_level_sums(int64_t m, int64_t n, int64_t k, int s,
                    const int8_t *DA, const int8_t *DB, int64_t *S)
{
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            for (int L = 2; L <= s + 1; ++L) {
                int64_t acc = 0;
                int tlo = L - s > 1 ? L - s : 1;
                int thi = L - 1 < s ? L - 1 : s;
                for (int t = tlo; t <= thi; ++t) {
                    int u = L - t;
                    const int8_t *a = DA + (int64_t)(t - 1) * m * k + i * k;
                    const int8_t *b = DB + (int64_t)(u - 1) * n * k + j * k;
                    for (int64_t l = 0; l < k; ++l)
                        acc += (int64_t)a[l] * (int64_t)b[l];
                }
                S[(int64_t)(L - 2) * m * n + i * n + j] = acc;
            }
        }
    }
}

/* NEXT-4 variant, reading R21: the FULL pair set, all s^2 slice products.    */
/* Levels L = 2..2s, S_L = sum over 1 <= t, u <= s with t + u = L (the same    */
/* per-level pair formula, no truncation at s + 1).  Output S[(L-2)*m*n+...]   */
/* for L = 2..2s (2s - 1 levels).                                             */
void orc_level_sums_full(int64_t m, int64_t n, int64_t k, int s,
                         const int8_t *DA, const int8_t *DB, int64_t *S)
{
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            for (int L = 2; L <= 2 * s; ++L) {
                int64_t acc = 0;
                int tlo = L - s > 1 ? L - s : 1;
                int thi = L - 1 < s ? L - 1 : s;
                for (int t = tlo; t <= thi; ++t) {
                    int u = L - t;
                    const int8_t *a = DA + (int64_t)(t - 1) * m * k + i * k;
                    const int8_t *b = DB + (int64_t)(u - 1) * n * k + j * k;
                    for (int64_t l = 0; l < k; ++l)
                        acc += (int64_t)a[l] * (int64_t)b[l];
                }
                S[(int64_t)(L - 2) * m * n + i * n + j] = acc;
            }
        }
    }
}

/* R21 combine: as O6 (ascending significance, one RNE per step) over the     */
/* levels L = Lmax .. 2, Lmax = s + 1 (triangular) or 2s (full).              */
void orc_combine_levels(int64_t m, int64_t n, int Lmax, const int64_t *S,
                        const int32_t *e, const int32_t *nfa,
                        const int32_t *f, const int32_t *nfb, double *P)
{
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            if (nfa[i] || nfb[j]) {
                P[i * n + j] = NAN;
                continue;
            }
            double acc = 0.0;
            for (int L = Lmax; L >= 2; --L) {
                double term = (double)S[(int64_t)(L - 2) * m * n + i * n + j] *
                              ldexp(1.0, -8 * (L - 2)); /* exact */
                acc = acc + term;
            }
            P[i * n + j] = ldexp(acc, e[i] + f[j] - 14);
        }
    }
}

/* O2..O6 with the full pair set (R21). */
int orc_emulated_product_full(int64_t m, int64_t n, int64_t k, int s,
                              const double *A, const double *Bt, double *P)
{
    int8_t *DA = malloc((size_t)s * m * k + 1);
    int8_t *DB = malloc((size_t)s * n * k + 1);
    int64_t *S = malloc(sizeof(int64_t) * ((size_t)(2 * s - 1) * m * n + 1));
    int32_t *e = malloc(sizeof(int32_t) * (m + 1)), *nfa = malloc(sizeof(int32_t) * (m + 1));
    int32_t *f = malloc(sizeof(int32_t) * (n + 1)), *nfb = malloc(sizeof(int32_t) * (n + 1));
    int rc = -2;
    if (DA && DB && S && e && nfa && f && nfb) {
        rc = orc_split_rows(m, k, A, s, DA, e, nfa);
        rc |= orc_split_rows(n, k, Bt, s, DB, f, nfb);
        orc_level_sums_full(m, n, k, s, DA, DB, S);
        orc_combine_levels(m, n, 2 * s, S, e, nfa, f, nfb, P);
    }
    free(DA); free(DB); free(S); free(e); free(nfa); free(f); free(nfb);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* O6: combine in FP64, ascending significance (reading R6):                  */
/*   acc = 0; for L = s+1 down to 2: acc = acc + (double)S_L * 2^(-8(L-2))    */
/*   P = ldexp(acc, e_i + f_j - 14)      (level-2 digit unit is 2^(e+f-14))   */
/* A non-finite row of op(A) or column of op(B) gives NaN (reading R10).      */
/* ------------------------------------------------------------------------- */
void orc_combine(int64_t m, int64_t n, int s, const int64_t *S,
                 const int32_t *e, const int32_t *nfa,
                 const int32_t *f, const int32_t *nfb, double *P)
{
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            if (nfa[i] || nfb[j]) {
                P[i * n + j] = NAN;
                continue;
            }
            double acc = 0.0;
            for (int L = s + 1; L >= 2; --L) {
                double term = (double)S[(int64_t)(L - 2) * m * n + i * n + j] *
                              ldexp(1.0, -8 * (L - 2)); /* exact */
                acc = acc + term;
            }
            P[i * n + j] = ldexp(acc, e[i] + f[j] - 14);
        }
    }
}

/* O2..O6 for one real product: P (row-major m x n) = emulated op(A) op(B).   */
/* A: row-major m x k (= op(A)), Bt: row-major n x k (= op(B)^T).             */
int orc_emulated_product(int64_t m, int64_t n, int64_t k, int s,
                         const double *A, const double *Bt, double *P)
{
    int8_t *DA = malloc((size_t)s * m * k + 1);
    int8_t *DB = malloc((size_t)s * n * k + 1);
    int64_t *S = malloc(sizeof(int64_t) * ((size_t)s * m * n + 1));
    int32_t *e = malloc(sizeof(int32_t) * (m + 1)), *nfa = malloc(sizeof(int32_t) * (m + 1));
    int32_t *f = malloc(sizeof(int32_t) * (n + 1)), *nfb = malloc(sizeof(int32_t) * (n + 1));
    int rc = -2;
    if (DA && DB && S && e && nfa && f && nfb) {
        rc = orc_split_rows(m, k, A, s, DA, e, nfa);
        rc |= orc_split_rows(n, k, Bt, s, DB, f, nfb);
        orc_level_sums(m, n, k, s, DA, DB, S);
        orc_combine(m, n, s, S, e, nfa, f, nfb, P);
    }
    free(DA); free(DB); free(S); free(e); free(nfa); free(f); free(nfb);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* O7, real: alpha/beta applied outside the emulation in FP64 (reading R7).    */
/*   beta == 0: C = alpha * P  (C not read)                                   */
/*   else       C = fma(alpha, P, beta * C)                                   */
/* ------------------------------------------------------------------------- */
void orc_apply_real(int64_t mn, double alpha, const double *P, double beta, double *C)
{
    for (int64_t x = 0; x < mn; ++x)
        C[x] = (beta == 0.0) ? alpha * P[x] : fma(alpha, P[x], beta * C[x]);
}

/* O7, complex (reading R7):                                                  */
/*   beta == 0: t = 0 (C not read)                                            */
/*   else t_r = fma(br, Cr, -(bi*Ci)),  t_i = fma(br, Ci, bi*Cr)              */
/*   Cr = fma(ar, Pr, fma(-ai, Pi, t_r)),  Ci = fma(ar, Pi, fma(ai, Pr, t_i)) */
void orc_apply_complex(int64_t mn, double ar, double ai, const double *Pr,
                       const double *Pi, double br, double bi, double *Cr, double *Ci)
{
    for (int64_t x = 0; x < mn; ++x) {
        double tr = 0.0, ti = 0.0;
        if (!(br == 0.0 && bi == 0.0)) {
            tr = fma(br, Cr[x], -(bi * Ci[x]));
            ti = fma(br, Ci[x], bi * Cr[x]);
        }
        double nr = fma(ar, Pr[x], fma(-ai, Pi[x], tr));
        double ni = fma(ar, Pi[x], fma(ai, Pr[x], ti));
        Cr[x] = nr;
        Ci[x] = ni;
    }
}

/* ------------------------------------------------------------------------- */
/* 3M combine (reading R9): C_re = fl(T1 - T2), C_im = fl(fl(T3 - T1) - T2)  */
/* ------------------------------------------------------------------------- */
void orc_combine_3m(int64_t mn, const double *T1, const double *T2, const double *T3,
                    double *Pr, double *Pi)
{
    for (int64_t x = 0; x < mn; ++x) {
        Pr[x] = T1[x] - T2[x];
        Pi[x] = (T3[x] - T1[x]) - T2[x];
    }
}

/* ------------------------------------------------------------------------- */
/* Reference FP64 GEMM (native comparison point, "native FP64    */
/* GEMM as our ground-truth baseline"): plain triple loop, ascending k, fma.  */
/* ------------------------------------------------------------------------- */
void orc_fp64_gemm(int64_t m, int64_t n, int64_t k, const double *A, const double *Bt,
                   double *T)
{
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t l = 0; l < k; ++l)
                acc = fma(A[i * k + l], Bt[j * k + l], acc);
            T[i * n + j] = acc;
        }
}

/* ------------------------------------------------------------------------- */
/* TRUE product: sum_l a_l * b_l exactly, rounded once to FP64 (RNE).         */
/* A long fixed-point (Kulisch-style) accumulator: NLIMB 32-bit limbs kept in */
/* int64 so carries can be deferred; bit b of the accumulator has weight      */
/* 2^(b - KOFF).  Products of two doubles span 2^-2148 .. 2^2048.             */
/* ------------------------------------------------------------------------- */
#define KOFF 2304 /* >= 2*(1074+52)+... so the lowest product bit index is >= 0 */
#define NLIMB 144 /* 4608 bits */

static void kul_add_product(int64_t *acc, double a, double b)
{
    if (a == 0.0 || b == 0.0)
        return;
    int ea, eb;
    double fa = frexp(a, &ea), fb = frexp(b, &eb); /* |f| in [0.5,1) */
    int64_t ma = (int64_t)ldexp(fa, 53), mb = (int64_t)ldexp(fb, 53); /* exact */
    int neg = (ma < 0) != (mb < 0);
    unsigned __int128 p = (unsigned __int128)(ma < 0 ? -ma : ma) *
                          (unsigned __int128)(mb < 0 ? -mb : mb); /* < 2^106 */
    int64_t sh = (int64_t)(ea - 53) + (eb - 53) + KOFF;            /* >= 0 */
    int64_t limb = sh / 32;
    int bit = (int)(sh % 32);
    /* p << bit spans at most 138 bits: five 32-bit limbs */
    unsigned __int128 lo = p << bit; /* low 128 bits */
    unsigned __int128 hi = bit ? (p >> (128 - bit)) : 0;
    uint32_t w[5];
    w[0] = (uint32_t)lo;
    w[1] = (uint32_t)(lo >> 32);
    w[2] = (uint32_t)(lo >> 64);
    w[3] = (uint32_t)(lo >> 96);
    w[4] = (uint32_t)hi;
    for (int q = 0; q < 5; ++q)
        acc[limb + q] += neg ? -(int64_t)w[q] : (int64_t)w[q];
}

static double kul_round(int64_t *acc)
{
    /* propagate carries: afterwards every limb is in [0, 2^32) except the top */
    for (int q = 0; q < NLIMB - 1; ++q) {
        int64_t c = acc[q] >> 32; /* floor division by 2^32 */
        acc[q] -= c * ((int64_t)1 << 32);
        acc[q + 1] += c;
    }
    int neg = acc[NLIMB - 1] < 0;
    if (neg) { /* magnitude: negate every limb, then propagate carries again */
        for (int q = 0; q < NLIMB; ++q)
            acc[q] = -acc[q];
        for (int q = 0; q < NLIMB - 1; ++q) {
            int64_t c = acc[q] >> 32;
            acc[q] -= c * ((int64_t)1 << 32);
            acc[q + 1] += c;
        }
    }
    int top = -1;
    for (int q = NLIMB - 1; q >= 0 && top < 0; --q)
        if (acc[q])
            for (int b = 31; b >= 0; --b)
                if ((acc[q] >> b) & 1) {
                    top = q * 32 + b;
                    break;
                }
    if (top < 0)
        return 0.0;
    /* value = 2^(top - KOFF) * 1.xxx ; keep 53 bits, or fewer if subnormal */
    int64_t e_top = (int64_t)top - KOFF;          /* exponent of the leading bit */
    int64_t lsb = top - 52;                        /* bit index of the last kept bit */
    if (e_top - 52 < -1074)
        lsb = -1074 + KOFF;                        /* subnormal: fixed quantum 2^-1074 */
#define GETBIT(i) ((i) < 0 ? 0 : (int)((acc[(i) / 32] >> ((i) % 32)) & 1))
    uint64_t mant = 0;
    for (int64_t b = top; b >= lsb; --b)
        mant = (mant << 1) | (uint64_t)GETBIT(b);
    int rb = GETBIT(lsb - 1);
    int sticky = 0;
    for (int64_t b = lsb - 2; b >= 0 && !sticky; --b)
        sticky = GETBIT(b);
#undef GETBIT
    if (rb && (sticky || (mant & 1)))
        mant += 1; /* RNE; a carry to 2^53 is exact in double */
    double r = ldexp((double)mant, (int)(lsb - KOFF));
    return neg ? -r : r;
}

double orc_exact_dot(int64_t k, const double *a, const double *b)
{
    int64_t acc[NLIMB];
    memset(acc, 0, sizeof acc);
    for (int64_t l = 0; l < k; ++l)
        kul_add_product(acc, a[l], b[l]);
    return kul_round(acc);
}

void orc_exact_gemm(int64_t m, int64_t n, int64_t k, const double *A, const double *Bt,
                    double *T)
{
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j)
            T[i * n + j] = orc_exact_dot(k, A + i * k, Bt + j * k);
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* BLAS quick return (reading R7): alpha == 0 or k == 0 -> C = beta * C with  */
/* the same FP64 operation shapes as O7; beta == 0 -> C = 0, C not read.      */
/* ------------------------------------------------------------------------- */
void orc_quick_real(int64_t mn, double beta, double *C)
{
    for (int64_t x = 0; x < mn; ++x)
        C[x] = (beta == 0.0) ? 0.0 : beta * C[x];
}

void orc_quick_complex(int64_t mn, double br, double bi, double *Cr, double *Ci)
{
    for (int64_t x = 0; x < mn; ++x) {
        if (br == 0.0 && bi == 0.0) {
            Cr[x] = 0.0;
            Ci[x] = 0.0;
        } else {
            double tr = fma(br, Cr[x], -(bi * Ci[x]));
            double ti = fma(br, Ci[x], bi * Cr[x]);
            Cr[x] = tr;
            Ci[x] = ti;
        }
    }
}

/* ========================================================================= */
/* Ozaki-II (CRT) -- NEXT-1.  PAPER.md:99 (§2.2): "converts floating-point     */
/* matrices into integers, performs multiple matrix multiplications using     */
/* smaller, pairwise coprime moduli and uses the CRT to reconstruct the final */
/* result"; knob = the moduli count.  Steps follow        */
/* SPEC.md [MODULE] ozaki2 (quantize / residue_gemm / crt_reconstruct) with    */
/* DESIGN.md readings R16..R20.  The CRT itself and the final rounding live in */
/* oracle/ozaki2.py (Python big integers / Fraction); these are the two loops  */
/* that are too slow in Python.                                               */
/* ========================================================================= */

/* R17 quantize: row (A) / column (B) power-of-two scale e and integers
 *   Q = RNE(x * 2^(nu - e)),  |Q| < 2^nu.
 * e = frexp exponent of M = max|x| (M < 2^e); if RNE(M * 2^(nu-e)) reaches 2^nu
 * then e += 1.  M == 0 -> e = 0, Q = 0.  Non-finite entry -> row flagged, Q = 0.
 * nu <= 62.  Inputs row-major rows x k (row contiguous).                     */
int orc2_quantize_rows(int64_t rows, int64_t k, const double *X, int nu, int64_t *Q, int *e_out,
                       int *nonfinite)
{
    for (int64_t i = 0; i < rows; ++i) {
        const double *x = X + i * k;
        double M = 0.0;
        int nf = 0;
        for (int64_t j = 0; j < k; ++j) {
            if (!isfinite(x[j])) nf = 1;
            else if (fabs(x[j]) > M) M = fabs(x[j]);
        }
        nonfinite[i] = nf;
        int e = 0;
        if (M > 0.0) {
            (void)frexp(M, &e);
            if (nearbyint(ldexp(M, nu - e)) >= ldexp(1.0, nu)) e += 1;
        }
        e_out[i] = e;
        for (int64_t j = 0; j < k; ++j)
            Q[i * k + j] = (nf || M == 0.0) ? 0 : (int64_t)nearbyint(ldexp(x[j], nu - e));
    }
    return 0;
}

/* Exact integer product Z = QA @ QBt^T with |Q| < 2^62: split Q = h 2^32 + l
 * (l = low 32 bits, unsigned) and accumulate three int128 sums
 *   hh = sum h_a h_b,  mid = sum (h_a l_b + l_a h_b),  ll = sum l_a l_b
 * so Z = hh 2^64 + mid 2^32 + ll (combined with big integers in Python).
 * out[(i n + j) * 6 + {0..5}] = (hh, mid, ll) as (low64, high64) pairs.     */
void orc2_int_gemm(int64_t m, int64_t n, int64_t k, const int64_t *QA, const int64_t *QBt, uint64_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            i128 hh = 0, mid = 0, ll = 0;
            for (int64_t t = 0; t < k; ++t) {
                const int64_t a = QA[i * k + t], b = QBt[j * k + t];
                const i128 ah = a >> 32, bh = b >> 32;
                const i128 al = (uint32_t)(a & 0xffffffff), bl = (uint32_t)(b & 0xffffffff);
                hh += ah * bh;
                mid += ah * bl + al * bh;
                ll += al * bl;
            }
            uint64_t *o = out + (i * n + j) * 6;
            const i128 v[3] = {hh, mid, ll};
            for (int q = 0; q < 3; ++q) {
                o[2 * q] = (uint64_t)v[q];
                o[2 * q + 1] = (uint64_t)(v[q] >> 64);
            }
        }
}

/* R19 residue GEMM for one modulus p: C = (RA @ RBt^T) mod p, centered
 * (p even: [-p/2, p/2-1]; odd: [-(p-1)/2, (p-1)/2]).  RA, RBt int8 residues.  */
void orc2_residue_gemm(int64_t m, int64_t n, int64_t k, const int8_t *RA, const int8_t *RBt, int p,
                       int32_t *C)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            int64_t acc = 0;
            for (int64_t t = 0; t < k; ++t) acc += (int64_t)RA[i * k + t] * RBt[j * k + t];
            int64_t r = acc % p;
            if (r < 0) r += p;
            if (r >= (p + 1) / 2) r -= p;
            C[i * n + j] = (int32_t)r;
        }
}

/* ========================================================================= */
/* Emulated TRSM (NEXT-4c), reading R23.  PAPER.md:115 (§3.2): */
/* LSMS time is "primarily the ZGEMM and ZTRSM"; the paper does not say how a */
/* TRSM is emulated, so R23 reads it as the standard blocked TRSM whose        */
/* off-diagonal updates are the emulated GEMM and whose nb x nb diagonal      */
/* blocks are solved in plain FP64 substitution with this fixed op order:     */
/*   left  (T x = b), T lower: i ascending,  acc = b_i, acc = fma(-T_ij, x_j,  */
/*         acc) for j ascending over j < i, x_i = acc / T_ii (unit: x_i=acc); */
/*         T upper: i descending, j ascending over j > i.                     */
/*   right (x T = b), T upper: j ascending, i ascending over i < j:          */
/*         acc = fma(-T_ij, x_i, acc), x_j = acc / T_jj; T lower: j descending, */
/*         i ascending over i > j.                                            */
/* Complex: acc -= t x as acc_r = fma(-t_r, x_r, fma(t_i, x_i, acc_r)),        */
/* acc_i = fma(-t_r, x_i, fma(-t_i, x_r, acc_i)); division a / t with          */
/* d = fma(t_r, t_r, t_i t_i), x_r = fma(a_r, t_r, a_i t_i) / d,               */
/* x_i = fma(a_i, t_r, -(a_r t_i)) / d.                                        */
/* T is the nb x nb diagonal block of op(A), row-major T[i*kb + j]; X holds    */
/* nvec vectors of length kb, vector v at X[v*kb + .] (solved in place).      */
/* ========================================================================= */
void orc_trsm_diag_real(int right, int lower, int unit, int64_t kb, const double *T, int64_t nvec, double *X)
{
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvec; ++v) {
        double *x = X + v * kb;
        for (int64_t s = 0; s < kb; ++s) {
            /* left: forward over i for lower T; right: forward over j for upper T */
            const int fwd = right ? !lower : lower;
            const int64_t i = fwd ? s : kb - 1 - s;
            double acc = x[i];
            if (!right) {
                const int64_t j0 = lower ? 0 : i + 1, j1 = lower ? i : kb;
                for (int64_t j = j0; j < j1; ++j) acc = fma(-T[i * kb + j], x[j], acc);
                x[i] = unit ? acc : acc / T[i * kb + i];
            } else {
                const int64_t j = i;            /* unknown x_j; terms x_r T_rj */
                const int64_t r0 = lower ? j + 1 : 0, r1 = lower ? kb : j;
                for (int64_t r = r0; r < r1; ++r) acc = fma(-T[r * kb + j], x[r], acc);
                x[j] = unit ? acc : acc / T[j * kb + j];
            }
        }
    }
}

static void cdiv_r23(double ar, double ai, double tr, double ti, double *xr, double *xi)
{
    const double d = fma(tr, tr, ti * ti);
    *xr = fma(ar, tr, ai * ti) / d;
    *xi = fma(ai, tr, -(ar * ti)) / d;
}

/* complex: T and X interleaved (re, im) */
void orc_trsm_diag_complex(int right, int lower, int unit, int64_t kb, const double *T, int64_t nvec, double *X)
{
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvec; ++v) {
        double *x = X + 2 * v * kb;
        for (int64_t s = 0; s < kb; ++s) {
            const int fwd = right ? !lower : lower;
            const int64_t i = fwd ? s : kb - 1 - s;
            double ar = x[2 * i], ai = x[2 * i + 1];
            int64_t r0, r1;
            if (!right) { r0 = lower ? 0 : i + 1; r1 = lower ? i : kb; }
            else        { r0 = lower ? i + 1 : 0; r1 = lower ? kb : i; }
            for (int64_t r = r0; r < r1; ++r) {
                /* left: t = T_ir, x_r;  right: t = T_ri, x_r */
                const int64_t ti_ = right ? (r * kb + i) : (i * kb + r);
                const double tr = T[2 * ti_], tim = T[2 * ti_ + 1];
                const double xr = x[2 * r], xi = x[2 * r + 1];
                ar = fma(-tr, xr, fma(tim, xi, ar));
                ai = fma(-tr, xi, fma(-tim, xr, ai));
            }
            if (unit) {
                x[2 * i] = ar;
                x[2 * i + 1] = ai;
            } else {
                cdiv_r23(ar, ai, T[2 * (i * kb + i)], T[2 * (i * kb + i) + 1], &x[2 * i], &x[2 * i + 1]);
            }
        }
    }
}
