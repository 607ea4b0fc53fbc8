// split_fast.cuh -- K1 for the production Ozaki-I path (CTA-pair GEMM layout, s <= 12).
//
// Same method and output as k_split_sm (split.cuh): §2.2 ("splits
// high-precision input matrices into slices ... based on their significant bits
// and exponent alignment"), readings R3 (exponent), R4 (X = RNE(x 2^(8s-1-e)),
// balanced base-256 digits), R9 (4M embedding, 3M operands) in DESIGN.md §3.
// The difference is specialisation: the slice count S, the operand mode of each
// side and the tile height (hence every output offset) are compile-time, so one
// item (8 values of one row) costs ~8 LDS + 8 DMUL + 8 F2I + 4 int ops / value +
// the PRMT transposes + S immediate-offset stores per target, and each thread
// keeps one row for the whole CTA (one base pointer, constant strides).
//
// Exponent scan (pass 1): the max of |x| is taken over the IEEE high words only
// (32-bit IMNMX).  R3 needs the full 64-bit max M only when the high word cannot
// decide it: M subnormal / zero (leading bit may sit in the low word) or the
// 127-rule tie (fraction's top 20 bits exactly 0b111111 followed by 14 zeros,
// where "f > 63/64" depends on the low word).  Those rows (warp-uniform) rescan
// with the exact 64-bit max -- so the exponent is bit-identical to k_split_sm.
#pragma once
#include <cstdint>

#include "numerics.cuh"
#include "split.cuh"

namespace ozk {

// R3 from the max high word H = max (hi(x) & 0x7fffffff) of a row (finite: H < 0x7ff00000).
// Returns false when the low words are needed (see header).
__device__ __forceinline__ bool exponent_from_hi(uint32_t H, int32_t &e) {
    const uint32_t ex = H >> 20, f = H & 0xfffffu;
    if (ex == 0 || f == (63u << 14)) return false;
    e = (int32_t)ex - 1022 + (f > (63u << 14) ? 1 : 0);
    return true;
}

// R17 (crt_exponent) from the max high word: e = E + 1 for a normal max 1.f 2^E, plus one when
// nu <= 52 and the top nu fraction bits are all ones.  Decided by the high word unless the max
// is subnormal / zero or (nu > 20 and the 20 high fraction bits are all ones).
__device__ __forceinline__ bool exponent_from_hi_crt(uint32_t H, int nu, int32_t &e) {
    const uint32_t ex = H >> 20, f = H & 0xfffffu;
    if (ex == 0) return false;
    bool bump = false;
    if (nu <= 20) bump = f >= (1u << 20) - (1u << (20 - nu));
    else if (nu <= 52 && f == 0xfffffu) return false;
    e = (int32_t)ex - 1022 + (bump ? 1 : 0);
    return true;
}

constexpr int32_t kExpBiasDef = 4096;   // long-row split: exponents stored as e + 4096 > 0

__device__ __forceinline__ uint32_t hi_abs(double x) {
    return (uint32_t)__double2hiint(x) & 0x7fffffffu;
}

__device__ __forceinline__ void st_global_v2(int8_t *p, uint32_t a, uint32_t b) {
    asm volatile("st.global.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

template <int S>
struct FastDigits {
    static constexpr int NW = (S + 3) / 4;   // 32-bit words of Y holding the S digit bytes
    static constexpr unsigned long long B = 0x0080808080808080ull >> (8 * (8 - (S < 8 ? S : 8)));

    // R4 for 8 values: X = RNE(v * 2^(P-e)) (scale = +-2^(P-e) when that power is a normal
    // double: one exact-or-correctly-rounded DMUL; else ldexp_rn on sgn*v), Y = (X + B) ^ B
    // (byte q = balanced digit of slice S - q).  NEG also forms wn = the digits of X2, where
    // X2 = -X if neg2 else X (a per-lane choice without register-array selects).
    // S <= 8: |X| <= 127 * 2^(8S-8) fits int64; S = 9..12: 128-bit X (|y| >= 2^63 is an
    // integer mantissa * 2^q, exact).
    template <bool NEG>
    __device__ __forceinline__ static void words(const double (&v)[8], double scale, double sgn, int sh,
                                                 uint32_t (&w)[NW][8], uint32_t (&wn)[NW][8],
                                                 bool neg2 = true) {
        if constexpr (S <= 8) {
            long long X[8];
            if (scale != 0.0) {
#pragma unroll
                for (int i = 0; i < 8; ++i) X[i] = __double2ll_rn(__dmul_rn(v[i], scale));
            } else {   // 2^(P-e) is not a normal double (extreme exponents): exact ldexp
#pragma unroll
                for (int i = 0; i < 8; ++i) X[i] = __double2ll_rn(ldexp_rn(sgn * v[i], sh));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const unsigned long long Y = ((unsigned long long)X[i] + B) ^ B;
                w[0][i] = (uint32_t)Y;
                if constexpr (NW > 1) w[1][i] = (uint32_t)(Y >> 32);
                if constexpr (NEG) {
                    const unsigned long long X2 =
                        neg2 ? 0ull - (unsigned long long)X[i] : (unsigned long long)X[i];
                    const unsigned long long Yn = (X2 + B) ^ B;
                    wn[0][i] = (uint32_t)Yn;
                    if constexpr (NW > 1) wn[1][i] = (uint32_t)(Yn >> 32);
                }
            }
        } else {
            unsigned __int128 B2 = 0;
#pragma unroll
            for (int q = 0; q < S - 1; ++q) B2 |= (unsigned __int128)0x80 << (8 * q);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double y = (scale != 0.0) ? __dmul_rn(v[i], scale) : ldexp_rn(sgn * v[i], sh);
                __int128 X;
                if (fabs(y) < 9223372036854775808.0) {
                    X = (__int128)__double2ll_rn(y);
                } else {   // |y| >= 2^63: an integer, mantissa * 2^q with q >= 11
                    const uint64_t bits = (uint64_t)__double_as_longlong(y);
                    const int q = (int)((bits >> 52) & 0x7ff) - 1075;
                    X = (__int128)((bits & kFracMask) | (1ull << 52)) << q;
                    if (bits >> 63) X = -X;
                }
                const unsigned __int128 Y = ((unsigned __int128)X + B2) ^ B2;
#pragma unroll
                for (int j = 0; j < NW; ++j) w[j][i] = (uint32_t)(Y >> (32 * j));
                if constexpr (NEG) {
                    const unsigned __int128 X2 = neg2 ? (unsigned __int128)0 - (unsigned __int128)X
                                                      : (unsigned __int128)X;
                    const unsigned __int128 Yn = (X2 + B2) ^ B2;
#pragma unroll
                    for (int j = 0; j < NW; ++j) wn[j][i] = (uint32_t)(Yn >> (32 * j));
                }
            }
        }
    }

    // 8x8 byte transpose of the words and one 8-byte store per slice; slice t = S - q of
    // byte q goes to block (t - 1) = S - 1 - q of the (tile, k-block) group, BLK bytes apart.
    template <int BLK>
    __device__ __forceinline__ static void store(const uint32_t (&w)[NW][8], int8_t *p) {
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            uint32_t lo[4], hi[4];
            transpose4x4(w[j][0], w[j][1], w[j][2], w[j][3], lo[0], lo[1], lo[2], lo[3]);
            transpose4x4(w[j][4], w[j][5], w[j][6], w[j][7], hi[0], hi[1], hi[2], hi[3]);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int q = 4 * j + qq;
                if (q < S) st_global_v2(p + (S - 1 - q) * BLK, lo[qq], hi[qq]);
            }
        }
    }
};

template <int S>
struct FastDigitsEmit : FastDigits<S> {
    using D = FastDigits<S>;
    // one target: the digits of X
    template <int BLK>
    __device__ __forceinline__ static void emit1(const double (&v)[8], double scale, double sgn, int sh,
                                                 int8_t *p1, const SplitParams &) {
        uint32_t w[D::NW][8], wn[D::NW][8];
        D::template words<false>(v, scale, sgn, sh, w, wn);
        D::template store<BLK>(w, p1);
    }
    // two targets: p1 <- digits of X, p2 <- digits of X2 (-X if neg2 else X)
    template <int BLK>
    __device__ __forceinline__ static void emit2(const double (&v)[8], double scale, double sgn, int sh,
                                                 int8_t *p1, int8_t *p2, bool neg2, const SplitParams &) {
        uint32_t w[D::NW][8], wn[D::NW][8];
        D::template words<true>(v, scale, sgn, sh, w, wn, neg2);
        D::template store<BLK>(w, p1);
        D::template store<BLK>(wn, p2);
    }
};

// Ozaki-II (NEXT-1) counterpart: R17 Q = RNE(v 2^(nu-e)) as int64 and the centred residues
// of Q mod p_q for the NM moduli (R18, crt.cuh), one byte each, modulus-major (stride
// p.ss_bytes).  Processed 4 moduli (one 32-bit word per value) at a time to bound registers.
// NM is a multiple of 4 (the word count is compile-time); the live moduli count is prm.crt.n.
template <int NM>
struct FastResidues {
    static constexpr int NW = (NM + 3) / 4;
    __device__ __forceinline__ static void quantise(const double (&v)[8], double scale, double sgn, int sh,
                                                    int32_t (&q2)[8], uint32_t (&q1)[8], uint32_t (&q0)[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double xs = (scale != 0.0) ? __dmul_rn(v[i], scale) : ldexp_rn(sgn * v[i], sh);
            const long long Q = __double2ll_rn(xs);   // |Q| < 2^nu <= 2^62
            q0[i] = (uint32_t)Q & 0x1fffffu;
            q1[i] = (uint32_t)(Q >> 21) & 0x1fffffu;
            q2[i] = (int32_t)(Q >> 42);
        }
    }
    __device__ __forceinline__ static void store_word(const uint32_t (&w)[8], int j, int nm, int8_t *p,
                                                      int64_t ss) {
        uint32_t lo[4], hi[4];
        transpose4x4(w[0], w[1], w[2], w[3], lo[0], lo[1], lo[2], lo[3]);
        transpose4x4(w[4], w[5], w[6], w[7], hi[0], hi[1], hi[2], hi[3]);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
            if (4 * j + qq < nm) st_global_v2(p + (int64_t)(4 * j + qq) * ss, lo[qq], hi[qq]);
    }
    // centred residue byte of Q (R18) for modulus q: with h = floor(p/2), x = fold(Q) >= 0 and
    // t = floor((x + h) / p), r = x - t p lies in [-h, p - 1 - h] (the centred range: symmetric
    // for odd p, [-128, 127] for p = 256) -- the same value as centre_byte(x mod p).
    __device__ __forceinline__ static uint32_t cres(int32_t q2, uint32_t q1, uint32_t q0, const CrtTab &t, int q) {
        const uint32_t x = (uint32_t)(q2 * (int32_t)t.c42[q]) + q1 * t.c21[q] + q0 + t.bias28[q];
        const uint32_t h = t.p[q] >> 1;
        const uint32_t tq = __umulhi(x + h, t.m39[q]) >> 7;   // floor((x + h) / p), x + h < 2^31
        return x - tq * t.p[q];   // low byte = the centred residue (two's complement)
    }
    // per-byte negation of 4 packed two's-complement bytes (-(-128) wraps to -128 = the centred
    // residue of -Q for p = 256; odd p have symmetric ranges)
    __device__ __forceinline__ static uint32_t neg4(uint32_t w) {
        const uint32_t nw = ~w;
        return ((nw & 0x7f7f7f7fu) + 0x01010101u) ^ (nw & 0x80808080u);
    }
    template <int BLK>
    __device__ __forceinline__ static void emit1(const double (&v)[8], double scale, double sgn, int sh,
                                                 int8_t *p1, const SplitParams &prm) {
        int32_t q2[8];
        uint32_t q1[8], q0[8];
        quantise(v, scale, sgn, sh, q2, q1, q0);
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = 0;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int q = 4 * j + qq;
                if (q < prm.crt.n) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        w[i] = __byte_perm(w[i], cres(q2[i], q1[i], q0[i], prm.crt, q), (0x3210 & ~(0xf << (4 * qq))) | (4 << (4 * qq)));
                }
            }
            store_word(w, j, prm.crt.n, p1, prm.ss_bytes);
        }
    }
    template <int BLK>
    __device__ __forceinline__ static void emit2(const double (&v)[8], double scale, double sgn, int sh,
                                                 int8_t *p1, int8_t *p2, bool neg2, const SplitParams &prm) {
        int32_t q2[8];
        uint32_t q1[8], q0[8];
        quantise(v, scale, sgn, sh, q2, q1, q0);
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = 0;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int q = 4 * j + qq;
                if (q < prm.crt.n) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        w[i] = __byte_perm(w[i], cres(q2[i], q1[i], q0[i], prm.crt, q), (0x3210 & ~(0xf << (4 * qq))) | (4 << (4 * qq)));
                }
            }
            store_word(w, j, prm.crt.n, p1, prm.ss_bytes);
            if (neg2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = neg4(w[i]);
            }
            store_word(w, j, prm.crt.n, p2, prm.ss_bytes);
        }
    }
};

// Exact 64-bit max |x| of row r over the valid depth, straight from global memory (rare path).
template <bool CPLX>
__device__ uint64_t row_max_bits_slow(const SplitParams &p, const void *Xb, int64_t r, int comp, int lane) {
    uint64_t m = 0;
    for (int64_t l = lane; l < p.k; l += 32) {
        const int64_t off = r * p.rs + l * p.ls;
        uint64_t u;
        if constexpr (!CPLX) {
            u = (uint64_t)__double_as_longlong(reinterpret_cast<const double *>(Xb)[off]) & kAbsMask;
        } else {
            const double2 x = reinterpret_cast<const double2 *>(Xb)[off];
            const double im = p.conj ? -x.y : x.y;
            const uint64_t ur = (uint64_t)__double_as_longlong(x.x) & kAbsMask;
            const uint64_t ui = (uint64_t)__double_as_longlong(im) & kAbsMask;
            if (comp == 0) u = ur;
            else if (comp == 1) u = ui;
            else if (comp == 2) u = (uint64_t)__double_as_longlong(__dadd_rn(x.x, im)) & kAbsMask;
            else u = ur > ui ? ur : ui;
        }
        m = u > m ? u : m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t om = __shfl_xor_sync(0xffffffffu, m, o);
        m = om > m ? om : m;
    }
    return m;
}

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
    return __reduce_max_sync(0xffffffffu, v);
}

// One side of the split: RG input rows r0..r0+RG-1 of batch entry b (one warp per row in
// pass 1, 32 * RG threads); MODE and the output tile height TH are compile-time.
//
// LONG (rows of many windows): the exponents come from k_split_exps (already in p.exps) and
// each CTA digitises ONE window (blockIdx.x = row group * nwin + window), so no CTA keeps a
// long row "open" between a first and a second read -- the input is read twice from HBM, but
// every read streams (the windowed single-kernel form re-reads each window from L2 only while
// the open rows of all resident CTAs fit there, which long rows do not).
//
// CRT (Ozaki-II, NEXT-1): S is the moduli count; pass 1 takes the exact 64-bit max and the R17
// exponent (crt_exponent), pass 2 emits residues instead of digits, modulus-major per tile.
template <int S, int MODE, int TH, int RG, bool LONG, bool CRT = false>
__device__ __forceinline__ void split_fast_side(const SplitParams &p, int KW, uint8_t *sbuf) {
    constexpr bool CPLX = (MODE != SPLIT_REAL);
    constexpr int NX = (MODE == SPLIT_3M) ? 3 : 1;   // operands (exponents) per row
    constexpr int BLK = TH * 32;                      // bytes of one (tile, k-block, slice) block
    constexpr int KBS = CRT ? BLK : S * BLK;          // bytes between k-blocks of one tile
    const int P = CRT ? p.crt.nu : 8 * S - 1;         // fixed-point bits (R4) / quantisation bits (R17)
    using D = typename std::conditional<CRT, FastResidues<S>, FastDigitsEmit<S>>::type;
    using Elem = typename std::conditional<CPLX, double2, double>::type;

    __shared__ int32_t s_e[3][RG];
    __shared__ double s_scale[3][RG];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b = blockIdx.y;
    const bool RCONTIG = (p.rs == 1);
    const int ld = KW + (16 / (int)sizeof(Elem));     // padded row stride (elements)
    Elem *slab = reinterpret_cast<Elem *>(sbuf);
    const Elem *X = reinterpret_cast<const Elem *>(p.X) + b * p.bstride;
    constexpr bool FOURM = (MODE == SPLIT_A4M || MODE == SPLIT_B4M);
    const int64_t kpad = FOURM ? p.kh : p.KB * 32;
    const int64_t nwin = (kpad + KW - 1) / KW;
    const int64_t r0 = (LONG ? (int64_t)blockIdx.x / nwin : (int64_t)blockIdx.x) * RG;
    const int64_t wbeg = LONG ? (int64_t)blockIdx.x % nwin : 0, wend = LONG ? wbeg + 1 : nwin;
    const int nrows = (int)min((int64_t)RG, max((int64_t)0, p.rows - r0));

    auto load_window = [&](int64_t w0) {
        const int wlen = (int)min((int64_t)KW, p.k - w0);
        if (wlen > 0) {
            if (RCONTIG) {   // the RG rows are adjacent for each l: thread keeps row tid % RG
                const int row = tid % RG;
                if (row < nrows) {
                    const int64_t gstep = 32 * p.ls;
                    const Elem *g = X + r0 + row + (w0 + tid / RG) * p.ls;
                    Elem *d = slab + row * ld + tid / RG;
#pragma unroll 4
                    for (int l = tid / RG; l < wlen; l += 32) {
                        if (CPLX) cp_async16(d, g);
                        else cp_async8(d, g);
                        g += gstep;
                        d += 32;
                    }
                }
            } else {         // row contiguous along l: one warp per row, 32 consecutive elements
                if (warp < nrows) {
                    const Elem *g = X + (r0 + warp) * p.rs + w0;
                    Elem *d = slab + warp * ld;
#pragma unroll 4
                    for (int l = lane; l < wlen; l += 32) {
                        if (CPLX) cp_async16(d + l, g + l);
                        else cp_async8(d + l, g + l);
                    }
                }
            }
        }
        cp_async_wait_all();
    };

    // ---------------- pass 1: exponents (warp = row)
    if constexpr (LONG) {   // from k_split_exps: biased per-row exponents (0: zero row, ~0u: Inf / NaN)
        if (tid < RG * NX) {
            const int x = tid / RG, rw = tid % RG;
            int32_t e = 0;
            if (rw < nrows) {
                const uint32_t v = p.emax[((int64_t)x * gridDim.y + b) * p.rows + r0 + rw];
                e = (v == 0u) ? 0 : (v == 0xffffffffu ? kNonFinite : (int32_t)v - kExpBiasDef);
                if (wbeg == 0) {   // one CTA per row group publishes the exponents (R3 / R17)
                    int32_t *ex = p.exps + (MODE == SPLIT_3M ? x * p.x_exps : 0) + b * p.rows_out;
                    if (MODE == SPLIT_B4M) {
                        ex[2 * (r0 + rw)] = e;
                        ex[2 * (r0 + rw) + 1] = e;
                    } else {
                        ex[r0 + rw] = e;
                    }
                    if (e == kNonFinite) atomicAdd(p.nonfinite, 1ull);
                }
            }
            s_e[x][rw] = e;
            const int sh = P - e;
            s_scale[x][rw] = (sh >= -1022 && sh <= 1023) ? pow2(sh) : 0.0;
        }
    } else {
    uint32_t hm[NX];
#pragma unroll
    for (int x = 0; x < NX; ++x) hm[x] = 0;
    for (int64_t w = 0; w < nwin; ++w) {
        const int64_t w0 = w * KW;
        if (w > 0) __syncthreads();
        load_window(w0);
        __syncthreads();
        const int wlen = (int)min((int64_t)KW, p.k - w0);
        if (warp < nrows) {
            const Elem *src = slab + warp * ld;
#pragma unroll 4
            for (int l = lane; l < wlen; l += 32) {
                const Elem v = src[l];
                if constexpr (!CPLX) {
                    hm[0] = max(hm[0], hi_abs(v));
                } else if constexpr (MODE == SPLIT_3M) {
                    const double im = p.conj ? -v.y : v.y;
                    hm[0] = max(hm[0], hi_abs(v.x));
                    hm[1] = max(hm[1], hi_abs(v.y));
                    hm[2] = max(hm[2], hi_abs(__dadd_rn(v.x, im)));
                } else {
                    hm[0] = max(hm[0], max(hi_abs(v.x), hi_abs(v.y)));
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < NX; ++x) {
        const uint32_t H = warp_max_u32(hm[x]);
        int32_t e = 0;
        bool nf = false;
        if (warp < nrows) {
            if (H >= 0x7ff00000u) {          // an Inf / NaN in the row (R10)
                nf = true;
                e = kNonFinite;
            } else if (!(CRT ? exponent_from_hi_crt(H, p.crt.nu, e) : exponent_from_hi(H, e))) {
                const int comp = (MODE == SPLIT_3M) ? x : (CPLX ? 3 : 0);
                const uint64_t mx = row_max_bits_slow<CPLX>(p, X, r0 + warp, comp, lane);
                e = CRT ? crt_exponent(mx, p.crt.nu) : exponent_from_maxbits(mx);
            }
        }
        if (lane == 0) {
            if (warp < nrows) {
                int32_t *ex = p.exps + (MODE == SPLIT_3M ? x * p.x_exps : 0) + b * p.rows_out;
                if (MODE == SPLIT_B4M) {
                    ex[2 * (r0 + warp)] = e;
                    ex[2 * (r0 + warp) + 1] = e;
                } else {
                    ex[r0 + warp] = e;
                }
                if (nf) atomicAdd(p.nonfinite, 1ull);
            }
            s_e[x][warp] = e;
            const int sh = P - e;
            s_scale[x][warp] = (sh >= -1022 && sh <= 1023) ? pow2(sh) : 0.0;
        }
    }
    }   // !LONG
    __syncthreads();

    // ---------------- pass 2: digits; thread = (row, 8-value units h = h0 + HSTEP j).
    // 4M: the lanes also split by component c (0 = Re, 1 = Im'), so that one store instruction
    // of a warp fills whole 32-B sectors: B4M rows 2r (Re) and 2r+1 (Im') are adjacent 16-B
    // slots of a core matrix, both halves hh of each come from the same instruction.
    const int row = tid % RG;
    constexpr int HSTEP = FOURM ? 16 : 32;
    const int c = FOURM ? ((tid / RG) & 1) : 0;
    const int h0 = FOURM ? ((tid / RG) >> 1) : tid / RG;
    const int64_t R = (MODE == SPLIT_B4M) ? 2 * (r0 + row) : r0 + row;   // first output row
    const int64_t tile = R / TH, rr = R % TH;
    const int64_t tile_bytes = (int64_t)(CRT ? p.crt.n : S) * BLK * p.KB;
    int8_t *obase = p.out + (b * p.tiles + tile) * tile_bytes + (rr >> 3) * 256 + (rr & 7) * 16 +
                    ((h0 >> 1) & 1) * 128 + (h0 & 1) * 8;
    const int64_t half_off = (p.kh >> 5) * KBS;        // 4M: the second K half (Im / Re block)
    int32_t ex[NX];
    double sc[NX], sg[NX];
    bool live[NX];
#pragma unroll
    for (int x = 0; x < NX; ++x) {
        ex[x] = s_e[x][row];
        live[x] = (row < nrows) && (ex[x] != kNonFinite);
        // R9 conj for 3M's Im operand: RNE is sign-symmetric, so digits of -v = digits with -scale
        sg[x] = (MODE == SPLIT_3M && x == 1 && p.conj) ? -1.0 : 1.0;
        sc[x] = s_scale[x][row] * sg[x];
    }
    const bool anylive = live[0];

    for (int64_t w = wbeg; w < wend; ++w) {
        const int64_t w0 = w * KW;
        if (LONG || nwin > 1) {
            __syncthreads();
            load_window(w0);
            __syncthreads();
        }
        const int wh = (int)((min((int64_t)KW, kpad - w0) + 7) / 8);   // 8-value units in window
        int8_t *op = obase + ((w0 >> 5) + (h0 >> 2)) * (int64_t)KBS;
        for (int h = h0; h < wh; h += HSTEP, op += (HSTEP / 4) * (int64_t)KBS) {
            const int64_t l0 = w0 + 8 * h;
            const int nvalid = (int)min((int64_t)8, max((int64_t)0, p.k - l0));
            const Elem *src = slab + row * ld + 8 * h;
            if constexpr (!CPLX) {
                double v[8];
                if (anylive && nvalid == 8) {
                    const double2 *s2 = reinterpret_cast<const double2 *>(src);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const double2 t = s2[i];
                        v[2 * i] = t.x;
                        v[2 * i + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = (anylive && i < nvalid) ? src[i] : 0.0;
                }
                D::template emit1<BLK>(v, sc[0], sg[0], P - ex[0], op, p);
            } else if constexpr (FOURM) {
                // this lane's component of 8 complex values; Im' = conj ? -Im : Im via -scale (RNE
                // is sign-symmetric).  A4M: row r = [Re | Im'].  B4M (R9 N side): row 2r = [Re | -Im'],
                // row 2r+1 = [Im' | Re]; lane c writes row 2r + c (first half, digits of X) and row
                // 2r + 1 - c (second half, digits of X for Re, of -X for Im'), 16 B apart.
                const double *sv = reinterpret_cast<const double *>(src) + c;
                double v[8];
                if (anylive && nvalid == 8) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = sv[2 * i];
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = (anylive && i < nvalid) ? sv[2 * i] : 0.0;
                }
                const bool negc = (c == 1) && p.conj;
                if constexpr (MODE == SPLIT_A4M) {
                    D::template emit1<BLK>(v, negc ? -sc[0] : sc[0], negc ? -1.0 : 1.0, P - ex[0],
                                           op + (c ? half_off : 0), p);
                } else {
                    D::template emit2<BLK>(v, negc ? -sc[0] : sc[0], negc ? -1.0 : 1.0, P - ex[0], op + 16 * c,
                                           op + half_off + 16 * (1 - c), c == 1, p);
                }
            } else {
                double re[8], im[8];
                if (anylive && nvalid == 8) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const double2 t = src[i];
                        re[i] = t.x;
                        im[i] = t.y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const double2 t = (i < nvalid) ? src[i] : make_double2(0.0, 0.0);
                        re[i] = t.x;
                        im[i] = t.y;
                    }
                }
                {          // SPLIT_3M: regions x = 0 (Re), 1 (Im'), 2 (fl(Re + Im')), own exponents
#pragma unroll
                    for (int x = 0; x < 3; ++x) {
                        double v[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const double imc = p.conj ? -im[i] : im[i];
                            v[i] = live[x] ? (x == 0 ? re[i] : (x == 1 ? im[i] : __dadd_rn(re[i], imc))) : 0.0;
                        }
                        D::template emit1<BLK>(v, sc[x], sg[x], P - ex[x], op + x * p.x_bytes, p);
                    }
                }
            }
        }
    }
}

// Both operands of one product in ONE launch (blockIdx.z = side), A rows in 128-row tiles,
// B rows in 64-row halves (the CTA-pair GEMM's layout).
//
// Cross-call overlap (ozaki_set_overlap): the kernel may be launched with programmatic dependent
// launch right after the previous call's GEMM, which triggers its dependents at its start, so
// these CTAs fill the SMs the GEMM's last wave leaves idle.  `early` (host-decided: the previous
// GEMM's C overlaps neither operand; the slice workspace alternates between two buffers) lets
// the CTA read its operands and write its slices before the previous GEMM has finished;
// otherwise it waits first.  Every CTA waits before exiting, so this grid completes only after
// the previous GEMM -- the next GEMM's own griddepcontrol.wait then orders it after both.
// Without the launch attribute both waits are no-ops.
template <int S, int MA, int MB, int RG, bool LONG = false, bool CRT = false>
// Ozaki-II long rows (CRT && LONG, 512 threads): at most 40 registers so three CTAs share an SM
// (issue-bound integer kernel: occupancy 50 -> 75 %, C3 N=12 split 1.05 -> 0.93 ms).
__global__ void __launch_bounds__(32 * RG, (CRT && LONG) ? 3 : 1) k_split_fast(const __grid_constant__ SplitPair pp, int KW,
                                                         int nwin, int early) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
    extern __shared__ __align__(16) uint8_t sbuf[];
    const int64_t rg = LONG ? (int64_t)blockIdx.x / nwin : (int64_t)blockIdx.x;
    if (blockIdx.z == 0) {
        if (rg * RG < pp.side[0].rows_grid) split_fast_side<S, MA, 128, RG, LONG, CRT>(pp.side[0], KW, sbuf);
    } else {
        if (rg * RG < pp.side[1].rows_grid)
            split_fast_side<S, MB, CRT ? 128 : 64, RG, LONG, CRT>(pp.side[1], KW, sbuf);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// R3 / R17 exponents of long rows (the LONG split's first kernel), split along K: each CTA
// takes a group of rows and a K chunk of p.kchunk, forms the exact 64-bit max |x| of its part of
// each row (NX maxima for SPLIT_3M: Re, Im', fl(Re + Im')) and folds the chunk's exponent into
// p.emax with atomicMax.  The exponent rule is monotone in the max, so the max over chunks of
// the chunk exponents is the exponent of the row max; zero chunks contribute nothing (the
// buffer starts at 0), Inf / NaN chunks contribute ~0u.  Values are e + kExpBias > 0.
//   rows contiguous along l: one warp per row (8 rows per CTA);
//   rows adjacent for each l (rs == 1): lane = row (32 rows per CTA), the 8 warps split l and
//   combine through shared memory.
template <int MODE, bool CRT>
__device__ __forceinline__ void exps_side(const SplitParams &p, int64_t g, int64_t kc, int64_t b) {
    constexpr bool CPLX = (MODE != SPLIT_REAL);
    constexpr int NX = (MODE == SPLIT_3M) ? 3 : 1;
    using Elem = typename std::conditional<CPLX, double2, double>::type;
    __shared__ uint64_t s_m[3][8][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Elem *X = reinterpret_cast<const Elem *>(p.X) + b * p.bstride;
    const bool RCONTIG = (p.rs == 1);
    const int64_t l0 = kc * p.kchunk, l1 = min(p.k, l0 + p.kchunk);
    auto mag = [&](const Elem v, uint64_t (&m)[NX]) {
        if constexpr (!CPLX) {
            const uint64_t u = (uint64_t)__double_as_longlong(v) & kAbsMask;
            m[0] = u > m[0] ? u : m[0];
        } else {
            const uint64_t ur = (uint64_t)__double_as_longlong(v.x) & kAbsMask;
            const uint64_t ui = (uint64_t)__double_as_longlong(v.y) & kAbsMask;
            if constexpr (MODE == SPLIT_3M) {
                const double im = p.conj ? -v.y : v.y;
                const uint64_t us = (uint64_t)__double_as_longlong(__dadd_rn(v.x, im)) & kAbsMask;
                m[0] = ur > m[0] ? ur : m[0];
                m[1] = ui > m[1] ? ui : m[1];
                m[2] = us > m[2] ? us : m[2];
            } else {
                const uint64_t u = ur > ui ? ur : ui;
                m[0] = u > m[0] ? u : m[0];
            }
        }
    };
    auto fold = [&](int64_t r, const uint64_t (&m)[NX]) {
#pragma unroll
        for (int x = 0; x < NX; ++x) {
            if (m[x] == 0) continue;
            const uint32_t v = (m[x] >= kExpInf)
                                   ? 0xffffffffu
                                   : (uint32_t)((CRT ? crt_exponent(m[x], p.crt.nu) : exponent_from_maxbits(m[x])) +
                                                kExpBiasDef);
            atomicMax(p.emax + ((int64_t)x * gridDim.y + b) * p.rows + r, v);
        }
    };
    uint64_t m[NX];
#pragma unroll
    for (int x = 0; x < NX; ++x) m[x] = 0;
    if (!RCONTIG) {
        const int64_t r = g * 8 + warp;
        if (r >= p.rows) return;
        const Elem *gp = X + r * p.rs;
#pragma unroll 8
        for (int64_t l = l0 + lane; l < l1; l += 32) mag(gp[l], m);
#pragma unroll
        for (int x = 0; x < NX; ++x) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t om = __shfl_xor_sync(0xffffffffu, m[x], o);
                m[x] = om > m[x] ? om : m[x];
            }
        }
        if (lane == 0) fold(r, m);
    } else {
        const int64_t r = g * 32 + lane;
        if (r < p.rows) {
            const Elem *gp = X + r + (l0 + warp) * p.ls;
            const int64_t step = 8 * p.ls;
#pragma unroll 8
            for (int64_t l = l0 + warp; l < l1; l += 8, gp += step) mag(*gp, m);
        }
#pragma unroll
        for (int x = 0; x < NX; ++x) s_m[x][warp][lane] = m[x];
        __syncthreads();
        if (warp == 0 && r < p.rows) {
#pragma unroll
            for (int x = 0; x < NX; ++x) {
                uint64_t v = s_m[x][0][lane];
#pragma unroll
                for (int w = 1; w < 8; ++w) v = s_m[x][w][lane] > v ? s_m[x][w][lane] : v;
                m[x] = v;
            }
            fold(r, m);
        }
    }
}

// One CTA per (row group, K chunk) of one side (blockIdx.z) and batch entry (blockIdx.y);
// blockIdx.x = group * chunks + chunk.
template <int MA, int MB, bool CRT = false>
__global__ void __launch_bounds__(256) k_split_exps(const __grid_constant__ SplitPair pp) {
    const SplitParams &q = pp.side[blockIdx.z];
    const int64_t gsz = (q.rs == 1) ? 32 : 8;
    const int64_t nch = (q.k + q.kchunk - 1) / q.kchunk;
    const int64_t g = blockIdx.x / nch, kc = blockIdx.x % nch;
    if (g * gsz >= q.rows) return;
    if (blockIdx.z == 0) exps_side<MA, CRT>(q, g, kc, blockIdx.y);
    else exps_side<MB, CRT>(q, g, kc, blockIdx.y);
}

}  // namespace ozk
