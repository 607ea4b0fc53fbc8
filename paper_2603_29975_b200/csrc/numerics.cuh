// numerics.cuh -- FP64 bit-level helpers of the Ozaki-I path (device side).
//
// Written from the definitions in DESIGN.md §3 (R3 exponent rule, R4 fixed
// point + balanced digits, R6 one correctly-rounded final scaling) using
// integer operations on IEEE-754 bit patterns; deliberately NOT libm.
#pragma once
#include <cstdint>

namespace ozk {

constexpr int32_t kNonFinite = 0x3fffffff;      // exponent sentinel: row/col had Inf/NaN
constexpr uint64_t kAbsMask = 0x7fffffffffffffffull;
constexpr uint64_t kExpInf = 0x7ff0000000000000ull;
constexpr uint64_t kFracMask = 0x000fffffffffffffull;

// R3: exponent of a row/column from the bit pattern `u` of max |x| (finite,
// any value incl. 0 and subnormals).  M = max|x|; e = least integer with
// M < 2^e (frexp convention); if M * 2^(7-e) > 127 then e += 1.  M == 0 -> 0.
// With M = 1.f * 2^E: e = E + 1 and M*2^(7-e) = 64 * 1.f, which exceeds 127
// exactly when f > 63/64, i.e. the 52-bit fraction field > 63 * 2^46.
__device__ __forceinline__ int32_t exponent_from_maxbits(uint64_t u) {
    if (u == 0) return 0;
    int32_t ex = (int32_t)(u >> 52);
    uint64_t frac = u & kFracMask;
    int32_t e;
    if (ex == 0) {                        // subnormal: M = frac * 2^-1074
        int32_t bl = 64 - __clzll((long long)frac);   // bit length of frac
        e = bl - 1074;
        frac = (frac << (53 - bl)) & kFracMask;   // normalised fraction bits
    } else {
        e = ex - 1022;
    }
    if (frac > (63ull << 46)) e += 1;
    return e;
}

__device__ __forceinline__ double pow2(int n) {   // 2^n for n in [-1022, 1023]
    return __longlong_as_double((long long)((uint64_t)(n + 1023) << 52));
}

// x * 2^n correctly rounded (RNE), x finite.  Normal results are exact
// exponent adjustments; subnormal results come from ONE rounding multiply of
// an exact operand; overflow gives +-Inf.
__device__ __forceinline__ double ldexp_rn(double x, int n) {
    uint64_t b = (uint64_t)__double_as_longlong(x);
    uint64_t sign = b & ~kAbsMask;
    uint64_t a = b & kAbsMask;
    if (a == 0 || n == 0) return x;
    int32_t ex = (int32_t)(a >> 52);
    if (ex == 0) {                         // subnormal input: normalise exactly
        x = __dmul_rn(x, 18014398509481984.0);   // 2^54, exact
        n -= 54;
        b = (uint64_t)__double_as_longlong(x);
        a = b & kAbsMask;
        ex = (int32_t)(a >> 52);
    }
    int32_t E = ex - 1023 + n;             // unbiased exponent of the result
    if (E > 1023) return __longlong_as_double((long long)(sign | kExpInf));
    if (E >= -1022)
        return __longlong_as_double((long long)(sign | ((uint64_t)(E + 1023) << 52) | (a & kFracMask)));
    if (E < -1075) return __longlong_as_double((long long)sign);   // below half the min subnormal
    // y = 1.f * 2^-1022 exactly, then one rounding multiply by 2^(E+1022) in [2^-53, 2^-1]
    double y = __longlong_as_double((long long)(sign | (1ull << 52) | (a & kFracMask)));
    return __dmul_rn(y, pow2(E + 1022));
}

// 2^n is a normal double (n in [-1022, 1023]): then x * 2^n by one DMUL is the
// correctly rounded (RNE) ldexp for every finite x -- exact when the result is
// normal, one rounding of the exact product when it is subnormal, +-Inf on
// overflow.  Sentinel exponents (kNonFinite) fall outside and take the slow path.
__device__ __forceinline__ bool pow2_normal(int n) { return (unsigned)(n + 1022) <= 2045u; }

// x * 2^n, correctly rounded: exact exponent-field add when x and the result
// are normal (the common case, branch-free select); otherwise ldexp_rn.
__device__ __forceinline__ double scale_pow2(double x, int n) {
    const long long b = __double_as_longlong(x);
    const int ex = (int)((b >> 52) & 0x7ff);
    const int E = ex + n;
    const bool fast = (ex != 0) && (ex != 0x7ff) && (E >= 1) && (E <= 2046);
    if (fast) return __longlong_as_double(b + ((long long)n << 52));
    return ldexp_rn(x, n);
}

// RNE(x) to a double for an integer |x| < 2^62, with integer operations only
// (no FP64 instruction): round the magnitude to 53 significant bits, ties to
// even, then assemble sign | exponent | fraction.
__device__ __forceinline__ double i64_to_f64_rn(long long x) {
    const unsigned long long sgn = (unsigned long long)x & 0x8000000000000000ull;
    const unsigned long long a = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
    if (a == 0) return 0.0;
    const int p = 63 - __clzll((long long)a);          // bit length - 1
    unsigned long long m;
    if (p > 52) {
        const int k = p - 52;
        const unsigned long long r = a >> k, rem = a & ((1ull << k) - 1), half = 1ull << (k - 1);
        m = r + ((rem > half || (rem == half && (r & 1ull))) ? 1ull : 0ull);   // may reach 2^53
    } else {
        m = a << (52 - p);
    }
    // m's leading one (bit 52, or 53 after a carry) adds to the exponent field
    return __longlong_as_double((long long)(sgn | (((unsigned long long)(p + 1022) << 52) + m)));
}

// fma(1, x, fma(+-0, y, +0)) of R7 with alpha = 1, beta = 0, in integer operations:
// the inner term is +0 when y is finite and NaN when y is +-Inf / NaN; x + (+0) maps
// -0 to +0 and keeps every other x (NaN stays NaN).
__device__ __forceinline__ double plus_zero(double x, double y) {
    const long long by = __double_as_longlong(y);
    if ((by & (long long)kExpInf) == (long long)kExpInf) return __longlong_as_double(0x7ff8000000000000ll);
    const long long bx = __double_as_longlong(x);
    return __longlong_as_double(bx == (long long)0x8000000000000000ull ? 0ll : bx);
}

// Exact int32 -> double without the XU pipe: 2^52 + 2^31 + x is representable,
// built from bits (hi word 0x43300000, lo word x + 2^31); one exact DADD
// removes the offset.  Same value as __int2double_rn, on the FP64 pipe.
__device__ __forceinline__ double i32_to_f64(uint32_t x) {
    const double biased = __hiloint2double(0x43300000, (int)(x ^ 0x80000000u));
    return __dsub_rn(biased, 4503601774854144.0);   // 2^52 + 2^31
}

}  // namespace ozk
