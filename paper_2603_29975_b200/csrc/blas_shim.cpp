// blas_shim.cpp -- Fortran-BLAS interposition library (libozaki_blas.so).
//
// The paper's deployment contract is "no code change": the application's
// ZGEMM/DGEMM calls are redirected to the emulation underneath it (PAPER.md
// :108-111, §3.1, SCILIB-Accel).  This library exports the reference-BLAS
// Fortran entry points dgemm_/zgemm_ and dtrsm_/ztrsm_ (emulated TRSM, reading R23 -- the
// paper's other hot routine) and the no-underscore aliases, so that
//     LD_PRELOAD=.../libozaki_blas.so ./application
// (or linking against it in place of BLAS) sends every DGEMM/ZGEMM through the
// C ABI of include/ozaki.h.  It holds no arithmetic of its own.
//
// Semantics (include/ozaki.h "BLAS shim"):
//   - Fortran ABI, LP64: every argument by reference, INTEGER = 32-bit int;
//     the hidden CHARACTER-length arguments of gfortran are ignored.
//   - Host operands go through the library's offload path (staged H2D /
//     GEMM / D2H); device operands (CUDA-aware callers) are used in place.
//     The call returns when C is written, as BLAS requires.
//   - Precision knob from the environment, read once: OZAKI_NUM_SLICES
//     (default 7, the 55-bit mode); complex method OZAKI_ZGEMM
//     = "4m" (default) or "3m".
//   - Invalid arguments: the reference-BLAS xerbla message on stderr with the
//     BLAS parameter number, C untouched.  Runtime errors (no sm_100 device,
//     CUDA failure): message on stderr, C untouched.  No CPU fallback.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ozaki.h"

namespace {

int slices_from_env() {
    static const int s = [] {
        const char *e = std::getenv("OZAKI_NUM_SLICES");
        const int v = e ? std::atoi(e) : 7;
        return (v >= 1 && v <= 16) ? v : 7;
    }();
    return s;
}

bool zgemm_3m_from_env() {
    static const bool m3 = [] {
        const char *e = std::getenv("OZAKI_ZGEMM");
        return e && (std::strcmp(e, "3m") == 0 || std::strcmp(e, "3M") == 0);
    }();
    return m3;
}

void report(const char *name, int rc, int slices_param = 14) {
    if (rc < 0) {
        // reference-BLAS xerbla wording; num_slices (GEMM param 14, TRSM 12) comes from the environment
        if (rc == -slices_param)
            std::fprintf(stderr, " ** On entry to %s, OZAKI_NUM_SLICES is out of range [1, 16]\n", name);
        else
            std::fprintf(stderr, " ** On entry to %s parameter number %2d had an illegal value\n", name, -rc);
    } else if (rc > 0) {
        std::fprintf(stderr, " ** %s (ozaki): %s\n", name, ozaki_last_error());
    }
}

// BLAS calls are synchronous: wait for the work enqueued on this thread's stream
// (the offload path already returns after C is written back).
int finish(int rc) {
    return rc == 0 ? ozaki_stream_synchronize() : rc;
}

void dgemm_impl(const char *ta, const char *tb, const int *m, const int *n, const int *k,
                const double *alpha, const double *A, const int *lda, const double *B,
                const int *ldb, const double *beta, double *C, const int *ldc) {
    const int rc = finish(ozaki_dgemm(*ta, *tb, *m, *n, *k, *alpha, A, *lda, B, *ldb, *beta, C, *ldc,
                                      slices_from_env()));
    report("DGEMM ", rc);
}

void zgemm_impl(const char *ta, const char *tb, const int *m, const int *n, const int *k,
                const double *alpha, const double *A, const int *lda, const double *B,
                const int *ldb, const double *beta, double *C, const int *ldc) {
    const int s = slices_from_env();
    const int rc = finish(zgemm_3m_from_env()
                              ? ozaki_zgemm3m(*ta, *tb, *m, *n, *k, alpha, A, *lda, B, *ldb, beta, C, *ldc, s)
                              : ozaki_zgemm(*ta, *tb, *m, *n, *k, alpha, A, *lda, B, *ldb, beta, C, *ldc, s));
    report("ZGEMM ", rc);
}

void dtrsm_impl(const char *side, const char *uplo, const char *ta, const char *diag, const int *m,
                const int *n, const double *alpha, const double *A, const int *lda, double *B, const int *ldb) {
    const int rc = finish(ozaki_dtrsm(*side, *uplo, *ta, *diag, *m, *n, *alpha, A, *lda, B, *ldb,
                                      slices_from_env()));
    report("DTRSM ", rc, 12);
}

void ztrsm_impl(const char *side, const char *uplo, const char *ta, const char *diag, const int *m,
                const int *n, const double *alpha, const double *A, const int *lda, double *B, const int *ldb) {
    const int rc = finish(ozaki_ztrsm(*side, *uplo, *ta, *diag, *m, *n, alpha, A, *lda, B, *ldb,
                                      slices_from_env()));
    report("ZTRSM ", rc, 12);
}

}  // namespace

extern "C" {

// Fortran: SUBROUTINE DTRSM(SIDE,UPLO,TRANSA,DIAG,M,N,ALPHA,A,LDA,B,LDB) -- emulated (R23)
void dtrsm_(const char *side, const char *uplo, const char *ta, const char *diag, const int *m, const int *n,
            const double *alpha, const double *A, const int *lda, double *B, const int *ldb) {
    dtrsm_impl(side, uplo, ta, diag, m, n, alpha, A, lda, B, ldb);
}
void dtrsm(const char *side, const char *uplo, const char *ta, const char *diag, const int *m, const int *n,
           const double *alpha, const double *A, const int *lda, double *B, const int *ldb) {
    dtrsm_impl(side, uplo, ta, diag, m, n, alpha, A, lda, B, ldb);
}
// Fortran: SUBROUTINE ZTRSM(...) with COMPLEX*16 ALPHA, A, B (interleaved re, im); 4M updates
void ztrsm_(const char *side, const char *uplo, const char *ta, const char *diag, const int *m, const int *n,
            const double *alpha, const double *A, const int *lda, double *B, const int *ldb) {
    ztrsm_impl(side, uplo, ta, diag, m, n, alpha, A, lda, B, ldb);
}
void ztrsm(const char *side, const char *uplo, const char *ta, const char *diag, const int *m, const int *n,
           const double *alpha, const double *A, const int *lda, double *B, const int *ldb) {
    ztrsm_impl(side, uplo, ta, diag, m, n, alpha, A, lda, B, ldb);
}

// Fortran: SUBROUTINE DGEMM(TRANSA,TRANSB,M,N,K,ALPHA,A,LDA,B,LDB,BETA,C,LDC)
void dgemm_(const char *ta, const char *tb, const int *m, const int *n, const int *k,
            const double *alpha, const double *A, const int *lda, const double *B, const int *ldb,
            const double *beta, double *C, const int *ldc) {
    dgemm_impl(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}
void dgemm(const char *ta, const char *tb, const int *m, const int *n, const int *k,
           const double *alpha, const double *A, const int *lda, const double *B, const int *ldb,
           const double *beta, double *C, const int *ldc) {
    dgemm_impl(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}
// Fortran: SUBROUTINE ZGEMM(...) with COMPLEX*16 ALPHA, BETA, A, B, C (interleaved re, im)
void zgemm_(const char *ta, const char *tb, const int *m, const int *n, const int *k,
            const double *alpha, const double *A, const int *lda, const double *B, const int *ldb,
            const double *beta, double *C, const int *ldc) {
    zgemm_impl(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}
void zgemm(const char *ta, const char *tb, const int *m, const int *n, const int *k,
           const double *alpha, const double *A, const int *lda, const double *B, const int *ldb,
           const double *beta, double *C, const int *ldc) {
    zgemm_impl(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // extern "C"
