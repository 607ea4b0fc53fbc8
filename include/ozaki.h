/*
 * ozaki.h -- C ABI of the B200 (sm_100a) INT8 Ozaki-I emulation of FP64 GEMM.
 *
 * The operation (§2.2): Ozaki-I "splits high-precision input
 * matrices into slices as lower-precision components based on their significant
 * bits and exponent alignment, then performs low-precision matrix
 * multiplications on these slices and accumulates them in higher precision".
 * The precision knob is the slice count s = num_slices: the paper's modes
 * "mantissa bits 31, 39, 47, 55, 63" (§3.2) are s = 4..8
 * (bits = 8s - 1, reading R2).  The complex routines serve the ZGEMM
 * calls that dominate LSMS in MuST (§3.2).
 *
 * What every call computes (readings R1-R15):
 *   e_i  = power-of-two exponent of row i of op(A)   (127-rule, R3)
 *   f_j  = power-of-two exponent of column j of op(B)
 *   each entry x -> X = RNE(x * 2^(8s-1-e)) -> s balanced INT8 digits (R4)
 *   S_L  = sum_{t+u=L} A_t * B_u^T  exactly (INT8 x INT8 -> INT32), L = 2..s+1 (R1)
 *   acc  = sum_{L=s+1..2} S_L 2^(-8(L-2)) in FP64, ascending (R6)
 *   P    = acc * 2^(e_i + f_j - 14)            (one correctly rounded scaling)
 *   C    = alpha * P + beta * C   in FP64, BLAS semantics (R7)
 * Results are bit-identical to the CPU oracle (oracle/) for every s.
 *
 * Conventions (all routines):
 *   - Matrices are column-major with leading dimensions, exactly as BLAS
 *     dgemm/zgemm.  Complex matrices are interleaved (re, im) doubles.
 *   - A, B, C (and strided-batched bases) are DEVICE pointers owned by the
 *     caller (e.g. torch tensors).  A and B are read-only; C must not share an
 *     element with A or B (OZAKI_ERR_ALIAS).  Views with the same leading
 *     dimension are compared element-exactly, so LAPACK-style updates of
 *     disjoint sub-blocks of one array (A22 -= L21 U12) are accepted; other
 *     combinations (and batched calls) are compared by address span.  When
 *     beta == 0, C is never read (NaN-safe).
 *   - Offload: if A, B and C are all HOST pointers (pinned or pageable), the
 *     call stages batch chunks through device memory on internal streams with
 *     H2D copy / GEMM / D2H copy overlapped, and returns once C is written
 *     back (synchronous for the host; the caller's stream is ordered after it).
 *     Mixed host/device operands return OZAKI_ERR_UNSUPPORTED.
 *   - transa/transb in {'N','n','T','t','C','c'}; for real routines 'C' == 'T'.
 *   - num_slices in [1, 16].
 *   - Calls enqueue work on the calling thread's stream (ozaki_set_stream,
 *     default: the legacy default stream 0) and return without synchronising.
 *     Workspace is allocated stream-ordered (cudaMallocAsync) and freed in
 *     stream order.
 *   - Return value: 0 on success.  -i: parameter i (BLAS position, counted as
 *     in the prototype below) is invalid; NOTHING is enqueued or written.
 *     > 0: runtime error (OZAKI_ERR_*); ozaki_last_error() has the message.
 *   - Non-finite inputs: a row of op(A) / column of op(B) containing Inf/NaN
 *     gives NaN in the corresponding row / column of alpha*P, and the sticky
 *     non-finite counter in ozaki_stats_t is incremented (R10).  There is no
 *     CPU fallback.
 *   - Thread safety: re-entrant; the stream and last-error are thread-local.
 */
#ifndef OZAKI_H
#define OZAKI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OZAKI_OK = 0,
    OZAKI_ERR_CUDA = 1,        /* a CUDA call or kernel launch failed          */
    OZAKI_ERR_ALLOC = 2,       /* workspace allocation failed                 */
    OZAKI_ERR_ARCH = 3,        /* current device is not sm_100 (B200/GB200)   */
    OZAKI_ERR_UNSUPPORTED = 4, /* argument combination not supported          */
    OZAKI_ERR_ALIAS = 5        /* C overlaps A or B                           */
};

/* Counters (monotonic since load or ozaki_reset_stats).  int8_gemm_equiv
 * counts INT8 slice-pair GEMMs in the closed forms of SPEC.md:305-310:
 * s(s+1)/2 per real product, x4 for 4M, x3 for 3M, times batch entries.  */
typedef struct ozaki_stats {
    uint64_t dgemm_calls;
    uint64_t zgemm_calls;     /* 4M */
    uint64_t zgemm3m_calls;   /* 3M */
    uint64_t batch_entries;   /* products computed (1 per non-batched call)   */
    uint64_t int8_gemm_equiv; /* slice-pair INT8 GEMMs (closed form)          */
    uint64_t int8_macs;       /* INT8 multiply-accumulates issued (padded)    */
    uint64_t k_chunks;        /* extra INT32 K-chunks needed (R8)             */
    uint64_t nonfinite_rows;  /* rows/cols that contained Inf/NaN (synced)    */
    uint64_t kernel_launches; /* device kernels launched by the library      */
    uint64_t crt_calls;       /* Ozaki-II calls (ozaki2_*)                   */
} ozaki_stats_t;

/* --- real: C = alpha op(A) op(B) + beta C,  op(A) m x k, op(B) k x n ---------
 * params: 1 transa 2 transb 3 m 4 n 5 k 6 alpha 7 A 8 lda 9 B 10 ldb
 *         11 beta 12 C 13 ldc 14 num_slices                                  */
int ozaki_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
                double alpha, const double *A, int64_t lda,
                const double *B, int64_t ldb,
                double beta, double *C, int64_t ldc, int num_slices);

/* --- complex, 4M real embedding [Ar|Ai] [[Br,Bi],[-Bi,Br]] (R9, N side) -----
 * alpha, beta: HOST pointers to {re, im}.  Same parameter numbering.        */
int ozaki_zgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
                const double *alpha, const double *A, int64_t lda,
                const double *B, int64_t ldb,
                const double *beta, double *C, int64_t ldc, int num_slices);

/* --- complex, 3M: T1=ArBr, T2=AiBi, T3=fl(Ar+Ai)fl(Br+Bi) each emulated,
 *     C_re = fl(T1-T2), C_im = fl(fl(T3-T1)-T2), then alpha/beta (R9)       */
int ozaki_zgemm3m(char transa, char transb, int64_t m, int64_t n, int64_t k,
                  const double *alpha, const double *A, int64_t lda,
                  const double *B, int64_t ldb,
                  const double *beta, double *C, int64_t ldc, int num_slices);

/* --- strided batched: entry b uses A + b*strideA, B + b*strideB,
 *     C + b*strideC (strides in ELEMENTS: doubles for d, complex for z).
 * params: 1 transa 2 transb 3 m 4 n 5 k 6 alpha 7 A 8 lda 9 strideA 10 B
 *         11 ldb 12 strideB 13 beta 14 C 15 ldc 16 strideC 17 batch
 *         18 num_slices.  All entries run in ONE persistent GEMM launch.    */
int ozaki_dgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                double alpha, const double *A, int64_t lda, int64_t strideA,
                                const double *B, int64_t ldb, int64_t strideB,
                                double beta, double *C, int64_t ldc, int64_t strideC,
                                int64_t batch, int num_slices);

int ozaki_zgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                const double *alpha, const double *A, int64_t lda, int64_t strideA,
                                const double *B, int64_t ldb, int64_t strideB,
                                const double *beta, double *C, int64_t ldc, int64_t strideC,
                                int64_t batch, int num_slices);

int ozaki_zgemm3m_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                  const double *alpha, const double *A, int64_t lda, int64_t strideA,
                                  const double *B, int64_t ldb, int64_t strideB,
                                  const double *beta, double *C, int64_t ldc, int64_t strideC,
                                  int64_t batch, int num_slices);

/* --- Ozaki-II (CRT), NEXT-1 of SURVEY.md §8(f) ------------------------------
 * PAPER.md:99 (§2.2): Ozaki-II "converts floating-point matrices into
 * integers, performs multiple matrix multiplications using smaller, pairwise
 * coprime moduli and uses the CRT to reconstruct the final result"; the knob is
 * the moduli count (10..18 in PAPER.md:119, :127).  Readings R16..R20:
 *   moduli   256, 255, 253, 251, 247, ... (greedy pairwise coprime, <= 256)
 *   nu       = min(62, floor((log2 M - ceil(log2 k_eff) - 1) / 2)), M = prod p
 *   e_i, f_j power-of-two row / column exponents; Q = RNE(x 2^(nu - e)), |Q| < 2^nu
 *   per modulus one INT8 GEMM of centred residues, reduced mod p (exact INT32)
 *   Z        = CRT of the residues = the exact integer product Q_A Q_B
 *   P        = RNE(Z 2^(e_i + f_j - 2 nu)) (one rounding); C = alpha P + beta C (R7)
 * Complex: the 4M real embedding of R9 (k_eff = 2k).  Same conventions, error
 * codes and host/device pointer rules as the Ozaki-I routines above;
 * parameter 14 (18 batched) is num_moduli in [1, 20].  Limits:
 * k_eff <= 131071 (INT32 residue sums) else OZAKI_ERR_UNSUPPORTED; nu >= 1
 * (enough moduli for k) else OZAKI_ERR_UNSUPPORTED.  Bit-identical to
 * oracle/ozaki2.py.                                                         */
int ozaki2_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
                 double alpha, const double *A, int64_t lda,
                 const double *B, int64_t ldb,
                 double beta, double *C, int64_t ldc, int num_moduli);
int ozaki2_zgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
                 const double *alpha, const double *A, int64_t lda,
                 const double *B, int64_t ldb,
                 const double *beta, double *C, int64_t ldc, int num_moduli);
int ozaki2_dgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                 double alpha, const double *A, int64_t lda, int64_t strideA,
                                 const double *B, int64_t ldb, int64_t strideB,
                                 double beta, double *C, int64_t ldc, int64_t strideC,
                                 int64_t batch, int num_moduli);
int ozaki2_zgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                 const double *alpha, const double *A, int64_t lda, int64_t strideA,
                                 const double *B, int64_t ldb, int64_t strideB,
                                 const double *beta, double *C, int64_t ldc, int64_t strideC,
                                 int64_t batch, int num_moduli);

/* --- NEXT-4 variant: emulated triangular solve (reading R23) ----------------
 * PAPER.md:115 (§3.2): LSMS time is "primarily the ZGEMM and ZTRSM" (> 80 %).
 * BLAS TRSM semantics, B overwritten by X (column-major, device or host
 * pointers like the GEMMs; host pointers are staged and the call returns when
 * B is written back):
 *   side 'L': op(A) X = alpha B   (A is m x m)
 *   side 'R': X op(A) = alpha B   (A is n x n)
 * uplo 'U'/'L' selects the referenced triangle of A, transa 'N'/'T'/'C'
 * (real 'C' == 'T'), diag 'U' = unit diagonal (not referenced) / 'N'.
 * Method (R23): B <- alpha B (R7's beta*C op shapes; alpha == 0: B = 0, B not
 * read; alpha == 1: unchanged), then over blocks of nb rows (left) / columns
 * (right) of the triangle, forward when op(A) is lower (left) / upper (right)
 * and backward otherwise: the diagonal block is solved by FP64 substitution
 * in the fixed op order of R23 (k_trsm_diag), and the remaining rows / columns
 * of B are updated by the EMULATED GEMM B_R <- -T_RK X_K + B_R (left) or
 * B_R <- -X_K T_KR + B_R (right) with num_slices slices (ozaki_dgemm /
 * ozaki_zgemm 4M).  nb is thread-local (ozaki_set_trsm_block, default 128).
 * Errors (nothing written): -1 side, -2 uplo, -3 transa, -4 diag, -5 m < 0,
 * -6 n < 0, -9 lda < max(1, m or n), -11 ldb < max(1, m), -12 num_slices not
 * in [1, 16]; OZAKI_ERR_ALIAS when A and B overlap.                          */
int ozaki_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
                const double *A, int64_t lda, double *B, int64_t ldb, int num_slices);
int ozaki_ztrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, const double *alpha,
                const double *A, int64_t lda, double *B, int64_t ldb, int num_slices);
/* nb >= 1 (returns -1 otherwise); thread-local, read at each TRSM call.      */
int ozaki_set_trsm_block(int64_t nb);
int64_t ozaki_get_trsm_block(void);

/* --- NEXT-4 variant: the Ozaki-I pair set (reading R21) ----------------------
 * full = 0 (default): the triangular set t + u <= s + 1 of R1, s(s+1)/2 INT8
 * products.  full = 1: all s^2 slice products (levels L = 2..2s, same
 * ascending FP64 combine), i.e. the exact integer product of the integerised
 * operands before one rounding per level step -- more accurate, ~2x the INT8
 * work.  Thread-local, read at each ozaki_*gemm* call (Ozaki-I routines only).
 * The full set needs s <= 8 and s * k_eff <= 131071 (no K-chunking) and the
 * CTA-pair kernel; otherwise the call returns OZAKI_ERR_UNSUPPORTED.
 * ozaki_debug_level_sums then writes 2s - 1 levels.                          */
int ozaki_set_pair_set(int full);
int ozaki_get_pair_set(void);

/* --- NEXT-4 variant: per-block exponent alignment (reading R22) -------------
 * kb = 0 (default): one exponent per row of op(A) / column of op(B).  kb > 0:
 * K is cut into blocks of kb; each block is emulated with its own row /
 * column exponents (same slices, pairs and combine), the block products are
 * summed in ascending block order in FP64 (one RNE each) into a workspace T,
 * then C = alpha T + beta C (R7).  Thread-local, read at each Ozaki-I call;
 * kb >= k is the per-row scheme.  Ozaki-II calls ignore it.  Returns -1 for
 * kb < 0.                                                                    */
int ozaki_set_exponent_block(int64_t kb);
int64_t ozaki_get_exponent_block(void);

/* --- cross-call overlap (performance option, thread-local, default 0) ---------
 * on != 0: consecutive Ozaki-I DGEMM / ZGEMM (4M) calls of this thread on one
 * stream overlap -- a call's split kernel is launched with programmatic
 * dependent launch (PDL) right after the previous call's GEMM and fills the SMs
 * its last wave leaves idle.  When the previous call's C overlaps neither A nor
 * B, the split reads A / B and writes its slices before that GEMM completes
 * (the slices alternate between two persistent workspaces owned by the thread
 * and stream); otherwise it waits.  Each split grid completes only after the
 * previous GEMM, so results and stream order are unchanged.  Caller's promise:
 * no kernel launched with PDL that writes the next call's A or B is placed on
 * the stream between two calls.  on = 0 releases the persistent workspaces.
 * The host-pointer offload path and 3M, Ozaki-II, K-chunked and debug calls run
 * as without it.  Returns 0.                                                 */
int ozaki_set_overlap(int on);
int ozaki_get_overlap(void);

/* --- streams, stats, errors --------------------------------------------- */
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * thread-local; returns 0.                                                 */
int ozaki_set_stream(void *stream);
void *ozaki_get_stream(void);
/* Blocks until all work enqueued on this thread's stream is done (used by the
 * BLAS shim, whose calls are synchronous).  0, or OZAKI_ERR_CUDA.          */
int ozaki_stream_synchronize(void);
/* Synchronises the device once to read the non-finite counter.           */
int ozaki_get_stats(ozaki_stats_t *out);
int ozaki_reset_stats(void);
/* Bytes of device workspace one call of this shape needs.
 * kind: 'd' real, 'z' 4M complex, '3' 3M complex.  -1 on bad arguments.   */
int64_t ozaki_workspace_size(char kind, int64_t m, int64_t n, int64_t k, int64_t batch,
                             int num_slices);
/* Message of the last error on this thread ("" if none).                  */
const char *ozaki_last_error(void);
/* Library version string.                                                 */
const char *ozaki_version(void);

/* --- phase profiler (tracing subsystem) ---------------------
 * When enabled, every kernel the library launches is bracketed by CUDA
 * events on its stream; ozaki_profile_read synchronises on the recorded
 * events, returns per-phase device time and launch counts accumulated since
 * the last read, and clears them.  Phases: 0 = K1 exponent scan, 1 = K1
 * slicing, 2 = K2/K3 slice GEMM + epilogue, 3 = other (3M combine, scale). */
typedef struct ozaki_profile {
    double ms[4];
    uint64_t launches[4];
} ozaki_profile_t;
int ozaki_profile_enable(int on);
int ozaki_profile_read(ozaki_profile_t *out);

/* --- test-only debug entry points (same kernels, extra outputs) -----------
 * ozaki_debug_split: run the split kernels on one operand.
 *   side 'A': rows of op(X) where op(X) = X ('N') or X^T ('T'/'C');
 *             X is rows x cols if trans=='N' else cols x rows (column-major).
 *   side 'B': columns of op(X) where op(X) is cols x rows ... i.e. the
 *             "rows" of the split are the columns of op(B): X is cols x rows
 *             if trans == 'N' else rows x cols.
 *   kind 'd' (real), 'z' (4M embedding; rows_out = 2*rows for side B),
 *        'r','i','s' (3M operands Re, Im, fl(Re+Im) of complex X).
 *   Outputs (DEVICE pointers): slices_out[t][r][l] int8 (t = 0..s-1 most
 *   significant first, r over output rows, l over the output K depth
 *   K' = cols (real/3M) or 2*round_up(cols,32) (4M)),
 *   exps_out[r] int32 (0x3fffffff marks a non-finite row).
 *   Returns the same codes as the GEMM routines.                           */
int ozaki_debug_split(char side, char kind, char trans, int64_t rows, int64_t cols,
                      const double *X, int64_t ldx, int num_slices,
                      int8_t *slices_out, int32_t *exps_out, int64_t *kdepth_out);

/* ozaki_debug_level_sums: the exact INT32 level sums S_L of a real product,
 * S_out[(L-2)*m*n + j*m + i] for L = 2..s+1 (DEVICE pointer, column-major
 * per level).  Same operand conventions as ozaki_dgemm.                   */
int ozaki_debug_level_sums(char transa, char transb, int64_t m, int64_t n, int64_t k,
                           const double *A, int64_t lda, const double *B, int64_t ldb,
                           int num_slices, int32_t *S_out);

/* ozaki_debug_timing: enable (1) / disable (0) per-role clock64 timers in the
 * GEMM kernel; when `out` is non-null, synchronises, copies up to `nslots`
 * counters (summed over CTAs: producer wait, MMA wait-operands, MMA
 * wait-TMEM-drain, MMA lifetime, epilogue wait, drain, store, CTA lifetime)
 * and clears them.  Returns the number of counters.                       */
int ozaki_debug_timing(int enable, uint64_t *out, int nslots);

#ifdef __cplusplus
}
#endif

#endif /* OZAKI_H */
