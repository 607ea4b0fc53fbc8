// crt.cuh -- Ozaki-II (CRT) device arithmetic: exponent rule, int64
// quantisation, centred residues (NEXT-1, §2.2 "converts
// floating-point matrices into integers, performs multiple matrix
// multiplications using smaller, pairwise coprime moduli and uses the CRT to
// reconstruct the final result"; readings R16..R20).
//
// Everything here is integer arithmetic on the ALU / IMAD pipes: the FP64 pipe
// is starved while the tensor cores stream (tools/fp64_vs_mma.cu), and the
// reductions mod p must be exact.
#pragma once
#include <cstdint>

#include "numerics.cuh"

namespace ozk {

constexpr int kMaxModuli = 20;   // M < 2^160: five 32-bit limbs (CRT kernel)

// Per-modulus constants, built on the host (ozaki.cu: crt_tables).
//   p      modulus (R16: 256, 255, 253, 251, 247, ...)
//   c21    2^21 mod p,  c42 = 2^42 mod p,  c16 = 2^16 mod p
//   bias28 multiple of p >= 2^28 (makes a folded sum non-negative)
//   bias23 multiple of p >= 2^23
//   m39    ceil(2^39 / p), 32 bits for p > 128 (and 2^31 for p = 256): m39 p - 2^39 < 2^8, so
//          floor(x m39 / 2^39) = floor(x / p) for 0 <= x < 2^31 (Granlund-Montgomery)
struct CrtTab {
    int32_t n;        // moduli count
    int32_t nu;       // R17 quantisation bits
    uint32_t p[kMaxModuli], c21[kMaxModuli], c42[kMaxModuli], c16[kMaxModuli];
    uint32_t bias28[kMaxModuli], bias23[kMaxModuli];
    uint32_t m39[kMaxModuli];   // ceil(2^39 / p) < 2^32: floor(x / p) = umulhi(x, m39) >> 7 for x < 2^31
};

// R17 exponent of a row / column from the bit pattern u of max|x| (finite):
// e = frexp exponent (max|x| < 2^e), plus one when RNE(max|x| 2^(nu-e)) reaches
// 2^nu.  With max|x| = 1.f 2^(e-1): max|x| 2^(nu-e) = 1.f 2^(nu-1), which rounds
// to 2^nu exactly when nu <= 52 and the 52-bit fraction >= 2^52 - 2^(52-nu)
// (the tie rounds to the even 2^nu).  0 -> 0.
__device__ __forceinline__ int32_t crt_exponent(uint64_t u, int nu) {
    if (u == 0) return 0;
    int32_t ex = (int32_t)(u >> 52);
    uint64_t frac = u & kFracMask;
    int32_t e;
    if (ex == 0) {
        const int32_t bl = 64 - __clzll((long long)frac);
        e = bl - 1074;
        frac = (frac << (53 - bl)) & kFracMask;
    } else {
        e = ex - 1022;
    }
    if (nu <= 52 && frac >= (1ull << 52) - (1ull << (52 - nu))) e += 1;
    return e;
}

// x mod p in [0, p) for 0 <= x < 2^31 (m39 = ceil(2^39 / p))
__device__ __forceinline__ uint32_t mod_small(uint32_t x, uint32_t p, uint32_t m39) {
    const uint32_t q = __umulhi(x, m39) >> 7;
    return x - q * p;
}

// R18: residue of an int64 |Q| < 2^62 mod p, NOT centred, in [0, p):
// Q = q2 2^42 + q1 2^21 + q0 (q0, q1 in [0, 2^21), q2 signed |q2| < 2^20),
// folded to q2 c42 + q1 c21 + q0 + bias28 in [0, 2^31).
__device__ __forceinline__ uint32_t residue_u(int32_t q2, uint32_t q1, uint32_t q0, const CrtTab &t, int i) {
    const uint32_t x = (uint32_t)(q2 * (int32_t)t.c42[i]) + q1 * t.c21[i] + q0 + t.bias28[i];
    return mod_small(x, t.p[i], t.m39[i]);
}

// centred representative (even p: [-p/2, p/2-1], odd p: symmetric) as a byte
__device__ __forceinline__ uint32_t centre_byte(uint32_t r, uint32_t p) {
    return (r >= ((p + 1) >> 1)) ? (r - p) & 0xffu : r;
}

// R19 epilogue: (int32 sum of residue products) mod p, as the byte u in [0, p) (not centred:
// the residue planes are read only by k_crt, which needs u).
// v = vh 2^16 + vl with |vh| < 2^15: folded to vh c16 + vl + bias23 in [0, 2^25).
__device__ __forceinline__ uint32_t residue_of_i32(int32_t v, const CrtTab &t, int i) {
    const uint32_t x = (uint32_t)((v >> 16) * (int32_t)t.c16[i]) + (uint32_t)(v & 0xffff) + t.bias23[i];
    return mod_small(x, t.p[i], t.m39[i]);   // u in [0, p): the planes feed only k_crt (p <= 256)
}

// 8 x 8 byte transpose of 8 words of 4 residue bytes each (values i, moduli
// 4j..4j+3) into one 8-byte word per modulus; store at modulus stride `ss`.
__device__ __forceinline__ void crt_store_word(const uint32_t (&w)[8], int j, int n, int8_t *dst, int64_t ss) {
    uint32_t o[8];
    // reuse the digit path's 4x4 transposes (split.cuh's transpose4x4 has the same semantics)
    const uint32_t t0 = __byte_perm(w[0], w[1], 0x5140), t1 = __byte_perm(w[2], w[3], 0x5140);
    const uint32_t t2 = __byte_perm(w[0], w[1], 0x7362), t3 = __byte_perm(w[2], w[3], 0x7362);
    o[0] = __byte_perm(t0, t1, 0x5410);
    o[1] = __byte_perm(t0, t1, 0x7632);
    o[2] = __byte_perm(t2, t3, 0x5410);
    o[3] = __byte_perm(t2, t3, 0x7632);
    const uint32_t u0 = __byte_perm(w[4], w[5], 0x5140), u1 = __byte_perm(w[6], w[7], 0x5140);
    const uint32_t u2 = __byte_perm(w[4], w[5], 0x7362), u3 = __byte_perm(w[6], w[7], 0x7362);
    o[4] = __byte_perm(u0, u1, 0x5410);
    o[5] = __byte_perm(u0, u1, 0x7632);
    o[6] = __byte_perm(u2, u3, 0x5410);
    o[7] = __byte_perm(u2, u3, 0x7632);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const int q = 4 * j + qq;
        if (q < n) *reinterpret_cast<uint2 *>(dst + (int64_t)q * ss) = make_uint2(o[qq], o[4 + qq]);
    }
}

// R17 + R18 for 8 consecutive values: Q = RNE(x 2^(nu-e)) (one DMUL by the
// exact power when representable -- identical to ldexp -- else ldexp_rn), then
// the centred residues of Q (dst0 / dst1) and of -Q (dstn) for every modulus.
__device__ __forceinline__ void residues_store8(const double (&v)[8], double scale, int32_t e,
                                                const CrtTab &t, int8_t *dst0, int8_t *dst1, int8_t *dstn,
                                                int64_t ss) {
    int32_t q2[8];
    uint32_t q1[8], q0[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const double xs = (scale != 0.0) ? __dmul_rn(v[i], scale) : ldexp_rn(v[i], t.nu - e);
        const long long Q = __double2ll_rn(xs);                 // |Q| < 2^nu <= 2^62
        q0[i] = (uint32_t)Q & 0x1fffffu;
        q1[i] = (uint32_t)(Q >> 21) & 0x1fffffu;
        q2[i] = (int32_t)(Q >> 42);
    }
    const int nw = (t.n + 3) >> 2;
    if (!dstn) {
        for (int j = 0; j < nw; ++j) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = 0;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int q = 4 * j + qq;
                if (q < t.n) {
                    const uint32_t p = t.p[q];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        w[i] |= centre_byte(residue_u(q2[i], q1[i], q0[i], t, q), p) << (8 * qq);
                }
            }
            crt_store_word(w, j, t.n, dst0, ss);
            if (dst1) crt_store_word(w, j, t.n, dst1, ss);
        }
        return;
    }
    for (int j = 0; j < nw; ++j) {   // B4M: also the residues of -Q (the -Im block, R9)
        uint32_t w[8], wn[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            w[i] = 0;
            wn[i] = 0;
        }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const int q = 4 * j + qq;
            if (q < t.n) {
                const uint32_t p = t.p[q];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t r = residue_u(q2[i], q1[i], q0[i], t, q);
                    w[i] |= centre_byte(r, p) << (8 * qq);
                    wn[i] |= centre_byte(r ? p - r : 0u, p) << (8 * qq);
                }
            }
        }
        crt_store_word(w, j, t.n, dst0, ss);
        if (dst1) crt_store_word(w, j, t.n, dst1, ss);
        crt_store_word(wn, j, t.n, dstn, ss);
    }
}

}  // namespace ozk
