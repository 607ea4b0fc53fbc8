// crt_kernel.cuh -- Ozaki-II reconstruction (NEXT-1, reading R20; PAPER.md:99
// "uses the CRT to reconstruct the final result").
//
// Per output element: the n residues u_q in [0, p_q) (plane q) determine the
// unique Z in (-M/2, M/2] with Z = u_q mod p_q; by the choice of nu (R17) Z is
// the exact integer product Q_A . Q_B.  Computed exactly in 32-bit limbs:
//   S = sum_q u_q W_q   (W_q = (M/p_q) inv_q < M)
//   Z = S mod M  (quotient from an FP64 estimate, corrected to be exact), centred
// then P = RNE(Z 2^(e_i + f_j - 2 nu)) with ONE rounding at the bit position
// of the (normal or subnormal) result, and C = alpha P + beta C as R7.
#pragma once
#include <cstdint>

#include "crt.cuh"
#include "numerics.cuh"

namespace ozk {

constexpr int kCrtLimbs = 5;   // M < 2^160 (kMaxModuli = 20)

struct CrtParams {
    const int8_t *R;
    int64_t plane_bytes, batch_bytes, rows_pad, groups;   // groups = padded columns / 16
    const int32_t *ea, *fb;
    int64_t Mp, Np, batch;
    double *C;
    int64_t ldc, strideC;
    int32_t cplx, ab_unit, nu, n;
    double alpha_r, alpha_i, beta_r, beta_i;
    uint32_t p[kMaxModuli];
    uint32_t W[kMaxModuli][kCrtLimbs];
    uint32_t M[kCrtLimbs + 1];
    uint32_t Mhalf[kCrtLimbs];
    double Minv;                                            // 2^(32(L-1)) / M (quotient from the top two limbs)
};

// RNE(mag * 2^sh) for a non-negative integer mag of L 32-bit limbs, one rounding
// at the precision of the result (53 bits, fewer when subnormal).
template <int L>
__device__ __forceinline__ double round_scaled(const uint32_t (&mag)[L], int sh) {
    // leading limb and the two below it, selected without dynamic register indexing
    int top = -1;
    uint32_t h0 = 0, m1 = 0, m2 = 0;
#pragma unroll
    for (int l = 0; l < L; ++l)
        if (mag[l]) {
            top = l;
            h0 = mag[l];
            m1 = l >= 1 ? mag[l >= 1 ? l - 1 : 0] : 0u;
            m2 = l >= 2 ? mag[l >= 2 ? l - 2 : 0] : 0u;
        }
    if (top < 0) return 0.0;
    // T = the 64 bits below and including the leading one; sticky = anything lower
    uint64_t hi = h0;
    uint64_t T;
    bool sticky = false;
    const int lz = __clz(h0);
    const int BL = 32 * top + 32 - lz;                       // bit length of mag
    {
        const uint64_t w96hi = (hi << 32) | m1;              // bits [32 top - 32, 32 top + 32)
        // T = top 64 bits of (mag[top], m1, m2) left-aligned
        T = lz ? ((w96hi << lz) | ((uint64_t)m2 >> (32 - lz))) : w96hi;
        if (lz && (m2 << lz)) sticky = true;
        if (!lz && m2) sticky = true;
#pragma unroll
        for (int l = 0; l < L; ++l)
            if (l < top - 2 && mag[l]) sticky = true;
    }
    // T carries bits [BL-64, BL) of mag (zeros below when BL < 64); value = T 2^(BL-64+sh)
    const int E = BL - 1 + sh;                               // binary exponent of the exact value
    int prec = 53;
    if (E < -1022) prec = 53 - (-1022 - E);                  // subnormal: fewer significant bits
    if (prec < 0) return 0.0;                                // below half the smallest subnormal
    const int d = 64 - prec;                                 // bits to drop from T (11..64)
    uint64_t Rq;
    if (d >= 64) {
        Rq = 0;                                              // prec == 0: round(T 2^-64) in {0, 1}
        const bool up = (T > (1ull << 63)) || (T == (1ull << 63) && sticky);
        Rq = up ? 1 : 0;
    } else {
        Rq = T >> d;
        const uint64_t rem = T & ((1ull << d) - 1), half = 1ull << (d - 1);
        const bool up = rem > half || (rem == half && (sticky || (Rq & 1ull)));
        Rq += up ? 1 : 0;
    }
    if (Rq == 0) return 0.0;
    // exact: Rq < 2^54, and Rq 2^(BL-64+d+sh) is representable (normal or subnormal)
    return ldexp_rn((double)Rq, BL - 64 + d + sh);
}

// One thread per (row, 4 consecutive columns): 4 lanes share one 16-byte plane
// chunk, so a warp reads 8 rows x 16 B = 128 contiguous bytes per plane.  The moduli
// count N is compile-time (L = ceil(N / 4) limbs holds M for the R16 moduli): all N plane
// words are loaded before any arithmetic, and the sum has no per-modulus branches.
template <int N>
__global__ void __launch_bounds__(256) k_crt(const __grid_constant__ CrtParams P) {
    constexpr int L = (N + 3) / 4;
    const int64_t per_b = P.rows_pad * P.groups * 4;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (idx >= per_b) return;
    const int quad = (int)(idx & 3);
    const int64_t rg = idx >> 2;
    const int64_t G = rg / P.rows_pad, row = rg - G * P.rows_pad;
    const int64_t col0 = G * 16 + quad * 4;
    if (row >= P.Mp || col0 >= P.Np) return;
    const int8_t *src = P.R + b * P.batch_bytes + (G * P.rows_pad + row) * 16 + quad * 4;
    uint32_t words[N];
#pragma unroll
    for (int q = 0; q < N; ++q) words[q] = __ldg(reinterpret_cast<const uint32_t *>(src + (int64_t)q * P.plane_bytes));
    // S_x = sum_q u_q W_q for the 4 elements, 64-bit accumulator per limb
    unsigned long long acc[4][L];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int l = 0; l < L; ++l) acc[x][l] = 0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        const uint32_t word = words[q];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const uint32_t u = (word >> (8 * x)) & 0xffu;   // residue planes hold u in [0, p)
#pragma unroll
            for (int l = 0; l < L; ++l) acc[x][l] += (unsigned long long)u * P.W[q][l];
        }
    }
    const int32_t e = __ldg(P.ea + b * P.Mp + row);
    double Pv[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const int64_t col = col0 + x;
        uint32_t s[L + 1];
        unsigned long long c = 0;
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const unsigned long long t = acc[x][l] + c;
            s[l] = (uint32_t)t;
            c = t >> 32;
        }
        s[L] = (uint32_t)c;
        // q = floor(S / M) < 2^13 from the top 64 bits of S (error < 1), then exact fix-up
        const unsigned long long top = ((unsigned long long)s[L] << 32) | s[L - 1];
        long long qe = (long long)(__ull2double_rn(top) * P.Minv);
        if (qe < 0) qe = 0;
        {
            unsigned long long cm = 0;
            uint32_t br = 0;
#pragma unroll
            for (int l = 0; l <= L; ++l) {
                const unsigned long long prod = (unsigned long long)P.M[l] * (unsigned long long)qe + cm;
                cm = prod >> 32;
                const unsigned long long diff = (unsigned long long)s[l] - (uint32_t)prod - br;
                s[l] = (uint32_t)diff;
                br = (uint32_t)(diff >> 63);
            }
            // qe is floor(S / M) - 1, floor(S / M) or floor(S / M) + 1: the FP64 estimate has a
            // relative error below 2^-51 on a quotient below 2^13 (absolute < 2^-38), and the
            // dropped low limbs add less than 2^(32(L-1)) / M < 2^-15.  So S - qe M lies in
            // [-M, 2M) and ONE correction (add M if negative, else subtract M if >= M) is exact.
            {
                if ((int32_t)s[L] < 0) {                     // negative: add M
                    unsigned long long cc = 0;
#pragma unroll
                    for (int l = 0; l <= L; ++l) {
                        const unsigned long long t = (unsigned long long)s[l] + P.M[l] + cc;
                        s[l] = (uint32_t)t;
                        cc = t >> 32;
                    }
                } else {                                      // s >= M: subtract M
                    unsigned long long bb = 0;
                    uint32_t d[L + 1];
#pragma unroll
                    for (int l = 0; l <= L; ++l) {
                        const unsigned long long t = (unsigned long long)s[l] - P.M[l] - bb;
                        d[l] = (uint32_t)t;
                        bb = (t >> 63) & 1ull;
                    }
                    if (!bb) {
#pragma unroll
                        for (int l = 0; l <= L; ++l) s[l] = d[l];
                    }
                }
            }
        }
        // 0 <= s < M; centre: s > M/2 -> Z = s - M
        unsigned long long bb = 0;
        uint32_t d[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {                        // d = Mhalf - s (borrow -> s > Mhalf)
            const unsigned long long t = (unsigned long long)P.Mhalf[l] - s[l] - bb;
            d[l] = (uint32_t)t;
            bb = (t >> 63) & 1ull;
        }
        const bool neg = bb != 0;
        uint32_t mag[L];
        if (neg) {                                           // |Z| = M - s
            unsigned long long b2 = 0;
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const unsigned long long t = (unsigned long long)P.M[l] - s[l] - b2;
                mag[l] = (uint32_t)t;
                b2 = (t >> 63) & 1ull;
            }
        } else {
#pragma unroll
            for (int l = 0; l < L; ++l) mag[l] = s[l];
        }
        double v = 0.0;
        if (col < P.Np) {
            const int32_t f = __ldg(P.fb + b * P.Np + col);
            if (e == kNonFinite || f == kNonFinite) v = __longlong_as_double(0x7ff8000000000000ll);
            else {
                v = round_scaled<L>(mag, e + f - 2 * P.nu);
                if (neg) v = -v;
            }
        }
        Pv[x] = v;
    }
    // C = alpha P + beta C (R7); complex: columns 2j / 2j+1 are Re / Im (R9)
    if (!P.cplx) {
        double *cp = P.C + b * P.strideC + row + col0 * P.ldc;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            if (col0 + x < P.Np) {
                if (P.ab_unit) *cp = Pv[x];
                else *cp = (P.beta_r == 0.0) ? __dmul_rn(P.alpha_r, Pv[x])
                                             : __fma_rn(P.alpha_r, Pv[x], __dmul_rn(P.beta_r, *cp));
            }
            cp += P.ldc;
        }
    } else {
        double2 *cp = reinterpret_cast<double2 *>(P.C) + b * P.strideC + row + (col0 >> 1) * P.ldc;
        const bool beta0 = P.beta_r == 0.0 && P.beta_i == 0.0;
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
            if (col0 + 2 * c2 < P.Np) {
                const double Pr = Pv[2 * c2], Pi = Pv[2 * c2 + 1];
                if (P.ab_unit) {
                    *cp = make_double2(plus_zero(Pr, Pi), plus_zero(Pi, Pr));
                } else {
                    double tr = 0.0, ti = 0.0;
                    if (!beta0) {
                        const double2 cv = *cp;
                        tr = __fma_rn(P.beta_r, cv.x, -__dmul_rn(P.beta_i, cv.y));
                        ti = __fma_rn(P.beta_r, cv.y, __dmul_rn(P.beta_i, cv.x));
                    }
                    *cp = make_double2(__fma_rn(P.alpha_r, Pr, __fma_rn(-P.alpha_i, Pi, tr)),
                                       __fma_rn(P.alpha_r, Pi, __fma_rn(P.alpha_i, Pr, ti)));
                }
            }
            cp += P.ldc;
        }
    }
}

}  // namespace ozk
