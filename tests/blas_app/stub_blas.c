/* Stand-in for the system BLAS the application was linked against: writes
 * NaN into C, so a result equal to the oracle proves the LD_PRELOADed
 * libozaki_blas.so served the call.                                         */
#include <math.h>
void dgemm_(const char *ta, const char *tb, const int *m, const int *n, const int *k,
            const double *al, const double *A, const int *lda, const double *B, const int *ldb,
            const double *be, double *C, const int *ldc) {
    for (int j = 0; j < *n; ++j)
        for (int i = 0; i < *m; ++i) C[i + (long)j * *ldc] = NAN;
}
void zgemm_(const char *ta, const char *tb, const int *m, const int *n, const int *k,
            const double *al, const double *A, const int *lda, const double *B, const int *ldb,
            const double *be, double *C, const int *ldc) {
    for (int j = 0; j < *n; ++j)
        for (int i = 0; i < 2 * *m; ++i) C[i + 2L * j * *ldc] = NAN;
}
