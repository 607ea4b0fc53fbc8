/* A "legacy application": calls Fortran-BLAS dgemm_ and zgemm_ on host arrays.
 * Linked against a stub BLAS (stub_blas.c) that poisons C; under
 * LD_PRELOAD=libozaki_blas.so the calls must reach the Ozaki library instead.
 * Writes m n k, A, B, C (real), then A, B, C (complex) to argv[1].          */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

void dgemm_(const char *, const char *, const int *, const int *, const int *, const double *,
            const double *, const int *, const double *, const int *, const double *, double *,
            const int *);
void zgemm_(const char *, const char *, const int *, const int *, const int *, const double *,
            const double *, const int *, const double *, const int *, const double *, double *,
            const int *);

static uint64_t st = 0x9e3779b97f4a7c15ull;
static double rnd(void) {   /* deterministic, exactly representable: (u - 1/2) * 2^(0..6 - 3) */
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    const double u = (double)(st >> 11) * (1.0 / 9007199254740992.0);
    const int sh = (int)((st >> 5) % 7) - 3;
    double x = u - 0.5;
    for (int i = 0; i < (sh > 0 ? sh : -sh); ++i) x = sh > 0 ? x * 2.0 : x * 0.5;
    return x;
}

int main(int argc, char **argv) {
    if (argc < 2) return 2;
    const int m = 70, n = 45, k = 33;
    double *A = malloc(sizeof(double) * m * k), *B = malloc(sizeof(double) * k * n),
           *C = malloc(sizeof(double) * m * n);
    double *ZA = malloc(16 * m * k), *ZB = malloc(16 * k * n), *ZC = malloc(16 * m * n);
    for (int i = 0; i < m * k; ++i) A[i] = rnd();
    for (int i = 0; i < k * n; ++i) B[i] = rnd();
    for (int i = 0; i < m * n; ++i) C[i] = 0.0;
    for (int i = 0; i < 2 * m * k; ++i) ZA[i] = rnd();
    for (int i = 0; i < 2 * k * n; ++i) ZB[i] = rnd();
    for (int i = 0; i < 2 * m * n; ++i) ZC[i] = 0.0;
    const double one = 1.0, zero = 0.0, zone[2] = {1.0, 0.0}, zzero[2] = {0.0, 0.0};
    dgemm_("N", "N", &m, &n, &k, &one, A, &m, B, &k, &zero, C, &m);
    zgemm_("N", "N", &m, &n, &k, zone, ZA, &m, ZB, &k, zzero, ZC, &m);
    FILE *f = fopen(argv[1], "wb");
    if (!f) return 3;
    const int dims[3] = {m, n, k};
    fwrite(dims, sizeof(int), 3, f);
    fwrite(A, sizeof(double), m * k, f);
    fwrite(B, sizeof(double), k * n, f);
    fwrite(C, sizeof(double), m * n, f);
    fwrite(ZA, 16, m * k, f);
    fwrite(ZB, 16, k * n, f);
    fwrite(ZC, 16, m * n, f);
    fclose(f);
    return 0;
}
