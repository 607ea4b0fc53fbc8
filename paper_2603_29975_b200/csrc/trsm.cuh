// trsm.cuh -- diagonal-block solve of the emulated TRSM (reading R23, NEXT-4c).
//
// PAPER.md:115 (§3.2): LSMS spends its time "primarily [in] the ZGEMM and ZTRSM".  R23 reads
// the emulated TRSM as a blocked TRSM whose off-diagonal updates are the emulated GEMM (the
// host loop in ozaki.cu) and whose nb x nb diagonal blocks are solved here by FP64
// substitution in a FIXED operation order (the oracle's orc_trsm_diag_* does the same):
//   left  (T x = b): T lower -> i ascending, T upper -> i descending; acc = b_i, then
//         acc = fma(-T_ij, x_j, acc) over the solved j in ascending order; x_i = acc / T_ii
//         (unit diagonal: x_i = acc).
//   right (x T = b): T upper -> j ascending, T lower -> j descending; acc = b_j, then
//         acc = fma(-T_ij, x_i, acc) over the solved i in ascending order; x_j = acc / T_jj.
// Complex: acc -= t x as acc_r = fma(-t_r, x_r, fma(t_i, x_i, acc_r)),
//          acc_i = fma(-t_r, x_i, fma(-t_i, x_r, acc_i));  a / t with d = fma(t_r, t_r, t_i t_i),
//          x_r = fma(a_r, t_r, a_i t_i) / d, x_i = fma(a_i, t_r, -(a_r t_i)) / d.
// T = op(A) restricted to the block: T_ij = A(k0+i, k0+j) ('N'), A(k0+j, k0+i) ('T'),
// conj(A(k0+j, k0+i)) ('C').  One thread per right-hand-side vector (a column of B for the
// left side, a row for the right side); the vector is solved in place in global memory (its
// own elements stay in L1); T elements are warp-uniform loads (broadcast).
#pragma once
#include <cstdint>

namespace ozk {

struct TrsmDiagParams {
    const double *A;   // element (0,0) of A (interleaved re, im when complex)
    int64_t lda;
    double *B;         // element (0,0) of B
    int64_t ldb;
    int64_t k0;        // first row / column of the diagonal block
    int32_t kb;        // block size
    int32_t trans;     // 0 'N', 1 'T', 2 'C'
    int32_t lower;     // op(A) lower triangular
    int32_t unit;      // unit diagonal
    int32_t right;     // side 'R'
    int64_t nvec;      // right-hand-side vectors (n for the left side, m for the right side)
};

template <bool CPLX>
__device__ __forceinline__ void trsm_T(const TrsmDiagParams &p, int64_t i, int64_t j, double &tr, double &ti) {
    const int64_t r = p.trans == 0 ? p.k0 + i : p.k0 + j, c = p.trans == 0 ? p.k0 + j : p.k0 + i;
    if constexpr (CPLX) {
        const double2 v = __ldg(reinterpret_cast<const double2 *>(p.A) + r + c * p.lda);
        tr = v.x;
        ti = p.trans == 2 ? -v.y : v.y;
    } else {
        tr = __ldg(p.A + r + c * p.lda);
        ti = 0.0;
    }
}

template <bool CPLX>
__global__ void __launch_bounds__(128) k_trsm_diag(const TrsmDiagParams p) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= p.nvec) return;
    // element e of this thread's vector: left -> B(k0 + e, v), right -> B(v, k0 + e)
    const int64_t base = p.right ? v + p.k0 * p.ldb : p.k0 + v * p.ldb;
    const int64_t step = p.right ? p.ldb : 1;
    const int kb = p.kb;
    const bool fwd = p.right ? !p.lower : p.lower;
    for (int s = 0; s < kb; ++s) {
        const int i = fwd ? s : kb - 1 - s;
        // solved neighbours: left lower / right upper -> [0, i), else (i, kb)
        const int r0 = fwd ? 0 : i + 1, r1 = fwd ? i : kb;
        if constexpr (CPLX) {
            double2 *x = reinterpret_cast<double2 *>(p.B) + base;
            double2 a = x[(int64_t)i * step];
            for (int r = r0; r < r1; ++r) {
                double tr, ti;
                if (p.right) trsm_T<true>(p, r, i, tr, ti);
                else trsm_T<true>(p, i, r, tr, ti);
                const double2 xr = x[(int64_t)r * step];
                a.x = __fma_rn(-tr, xr.x, __fma_rn(ti, xr.y, a.x));
                a.y = __fma_rn(-tr, xr.y, __fma_rn(-ti, xr.x, a.y));
            }
            if (!p.unit) {
                double tr, ti;
                trsm_T<true>(p, i, i, tr, ti);
                const double d = __fma_rn(tr, tr, __dmul_rn(ti, ti));
                const double re = __ddiv_rn(__fma_rn(a.x, tr, __dmul_rn(a.y, ti)), d);
                const double im = __ddiv_rn(__fma_rn(a.y, tr, -__dmul_rn(a.x, ti)), d);
                a = make_double2(re, im);
            }
            x[(int64_t)i * step] = a;
        } else {
            double *x = p.B + base;
            double a = x[(int64_t)i * step];
            for (int r = r0; r < r1; ++r) {
                double tr, ti;
                if (p.right) trsm_T<false>(p, r, i, tr, ti);
                else trsm_T<false>(p, i, r, tr, ti);
                a = __fma_rn(-tr, x[(int64_t)r * step], a);
            }
            if (!p.unit) {
                double tr, ti;
                trsm_T<false>(p, i, i, tr, ti);
                a = __ddiv_rn(a, tr);
            }
            x[(int64_t)i * step] = a;
        }
    }
}

}  // namespace ozk
