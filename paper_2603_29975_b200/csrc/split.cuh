// split.cuh -- K1: exponent scan + INT8 slicing (the bandwidth-bound half).
//
// Method (§2.2 "splits high-precision input matrices into slices
// ... based on their significant bits and exponent alignment"; readings R3/R4
// in DESIGN.md §3):
//   phase 1 (k_exponent): e_r = exponent rule R3 applied to max |x| of the
//            r-th "row" (row of op(A) / column of op(B)), by a max-reduction of
//            IEEE bit patterns (warp shuffles).
//   phase 2 (k_slice):    X = RNE(x * 2^(8s-1-e_r)), then s balanced base-256
//            digits, written as INT8 into the GEMM's tiled operand layout
//            (DESIGN.md §5): per (row tile, 32-byte K block, slice) one
//            canonical K-major SWIZZLE_NONE block of tile_h rows x 32 bytes,
//            so the GEMM fetches a whole pipeline stage with ONE bulk copy.
//
// Operand "views": element (r, l) of the split matrix lives at
//   X[b*bstride + r*rs + l*ls]          (real: double, complex: double2)
// and, per mode, maps to one or more (output row, output K chunk) targets.
#pragma once
#include <cstdint>

#include "numerics.cuh"

namespace ozk {

enum SplitMode : int {
    SPLIT_REAL = 0,   // real operand
    SPLIT_A4M = 1,    // complex op(A) -> row r: [Re | Im]
    SPLIT_B4M = 2,    // complex op(B) -> columns 2j: [Re ; -Im], 2j+1: [Im ; Re]  (R9, N side)
    SPLIT_RE = 3,     // 3M operands: Re, Im, fl(Re + Im)
    SPLIT_IM = 4,
    SPLIT_SUM = 5,
};

struct SplitParams {
    const void *X;
    int64_t rs, ls;       // element strides between rows / along the K depth
    int64_t bstride;      // element stride between batch entries
    int64_t rows;         // valid input rows
    int64_t k;            // valid input depth
    int64_t rows_grid;    // input rows covered by the slice grid (covers all tile rows)
    int64_t rows_out;     // valid output rows (2*rows for B4M)
    int32_t mode, conj, s, tile_h;
    int64_t tiles;        // output row tiles per batch entry
    int64_t KB;           // 32-byte K blocks per output row
    int64_t kh;           // 4M: start of the second half (multiple of 32), else 0
    int8_t *out;          // tiled slices
    int32_t *exps;        // [batch][rows_out]
    unsigned long long *nonfinite;   // device counter (rows/cols with Inf/NaN)
};

__device__ __forceinline__ bool is_complex_mode(int m) { return m != SPLIT_REAL; }

// |value| bit pattern used for the exponent of mode `mode` at (r, l).
__device__ __forceinline__ uint64_t mag_bits(const SplitParams &p, const void *base, int64_t off) {
    if (p.mode == SPLIT_REAL) {
        double x = __ldg(reinterpret_cast<const double *>(base) + off);
        return (uint64_t)__double_as_longlong(x) & kAbsMask;
    }
    double2 v = __ldg(reinterpret_cast<const double2 *>(base) + off);
    double re = v.x, im = p.conj ? -v.y : v.y;
    uint64_t ur = (uint64_t)__double_as_longlong(re) & kAbsMask;
    uint64_t ui = (uint64_t)__double_as_longlong(im) & kAbsMask;
    switch (p.mode) {
        case SPLIT_RE: return ur;
        case SPLIT_IM: return ui;
        case SPLIT_SUM: return (uint64_t)__double_as_longlong(__dadd_rn(re, im)) & kAbsMask;
        default: return ur > ui ? ur : ui;   // 4M: one exponent for Re and Im (R9)
    }
}

__device__ __forceinline__ void reduce_and_store(const SplitParams &p, int64_t b, int64_t r,
                                                 uint64_t maxb, uint32_t nf) {
    int32_t e = nf ? kNonFinite : exponent_from_maxbits(maxb);
    int32_t *ex = p.exps + b * p.rows_out;
    if (p.mode == SPLIT_B4M) {
        ex[2 * r] = e;
        ex[2 * r + 1] = e;
    } else {
        ex[r] = e;
    }
    if (nf) atomicAdd(p.nonfinite, 1ull);
}

// Phase 1.  RCONTIG: consecutive rows are contiguous (rs == 1): block (32,8),
// thread x = row, y strides the depth, smem max-reduce.  Otherwise each row is
// contiguous along l: one warp per row, lanes stride l, shuffle max-reduce.
template <bool RCONTIG>
__global__ void __launch_bounds__(256) k_exponent(const SplitParams p) {
    const int64_t b = blockIdx.z;
    const void *base = p.mode == SPLIT_REAL
                           ? (const void *)(reinterpret_cast<const double *>(p.X) + b * p.bstride)
                           : (const void *)(reinterpret_cast<const double2 *>(p.X) + b * p.bstride);
    if constexpr (RCONTIG) {
        __shared__ uint64_t smax[8][33];
        __shared__ uint32_t snf[8][33];
        const int64_t r = (int64_t)blockIdx.x * 32 + threadIdx.x;
        uint64_t m = 0;
        uint32_t nf = 0;
        if (r < p.rows) {
            for (int64_t l = threadIdx.y; l < p.k; l += 8) {
                uint64_t u = mag_bits(p, base, r * p.rs + l * p.ls);
                nf |= (u >= kExpInf);
                m = (u < kExpInf && u > m) ? u : m;
            }
        }
        smax[threadIdx.y][threadIdx.x] = m;
        snf[threadIdx.y][threadIdx.x] = nf;
        __syncthreads();
        if (threadIdx.y == 0 && r < p.rows) {
            for (int y = 1; y < 8; ++y) {
                uint64_t o = smax[y][threadIdx.x];
                m = o > m ? o : m;
                nf |= snf[y][threadIdx.x];
            }
            reduce_and_store(p, b, r, m, nf);
        }
    } else {
        const int warp = threadIdx.y, lane = threadIdx.x;
        const int64_t r = (int64_t)blockIdx.x * 8 + warp;
        if (r >= p.rows) return;
        uint64_t m = 0;
        uint32_t nf = 0;
        for (int64_t l = lane; l < p.k; l += 32) {
            uint64_t u = mag_bits(p, base, r * p.rs + l * p.ls);
            nf |= (u >= kExpInf);
            m = (u < kExpInf && u > m) ? u : m;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t om = __shfl_xor_sync(0xffffffffu, m, o);
            m = om > m ? om : m;
            nf |= __shfl_xor_sync(0xffffffffu, nf, o);
        }
        if (lane == 0) reduce_and_store(p, b, r, m, nf);
    }
}

// ------------------------------------------------------------------ digits
// R4: X = RNE(x 2^(P-e)), P = 8s-1; balanced digits via the offset trick:
// with Bofs = sum_{p=0}^{s-2} 128*256^p, Z = X + Bofs has plain base-256 bytes
// (d_t + 128) at positions p = s-t for t >= 2 and d_1 = Z >> 8(s-1).
template <int SMAX>
struct DigitWords {
    uint32_t w[SMAX][4];   // slice t (0 = most significant), 16 bytes
};

template <int SMAX>
__device__ __forceinline__ void put_digits(DigitWords<SMAX> &dw, int i, double x, int32_t e,
                                           int s) {
    const int P = 8 * s - 1;
    const int sh_i = 8 * (i & 3);
    const int wi = i >> 2;
    if constexpr (SMAX <= 8) {
        double v = ldexp_rn(x, P - e);                 // |v| <= 127*2^(8s-8) < 2^63
        long long X = __double2ll_rn(v);
        long long bofs = (long long)(0x0080808080808080ull >> (8 * (8 - s)));   // s-1 bytes
        long long Z = X + bofs;
#pragma unroll
        for (int t = 0; t < SMAX; ++t) {
            if (t < s) {
                int p = s - 1 - t;
                int d = (t == 0) ? (int)(Z >> (8 * p)) : (int)((Z >> (8 * p)) & 0xff) - 128;
                dw.w[t][wi] |= ((uint32_t)d & 0xffu) << sh_i;
            }
        }
    } else {
        double v = ldexp_rn(x, P - e);                 // |v| < 2^127
        __int128 X;
        double av = fabs(v);
        if (av < 9223372036854775808.0) {
            X = (__int128)__double2ll_rn(v);
        } else {                                       // integer >= 2^63: mant * 2^q
            uint64_t bits = (uint64_t)__double_as_longlong(v);
            int q = (int)((bits >> 52) & 0x7ff) - 1075;
            __int128 mant = (__int128)((bits & kFracMask) | (1ull << 52));
            X = mant << q;
            if (bits >> 63) X = -X;
        }
        __int128 bofs = 0;
        for (int p = 0; p < s - 1; ++p) bofs |= (__int128)0x80 << (8 * p);
        __int128 Z = X + bofs;
#pragma unroll
        for (int t = 0; t < SMAX; ++t) {
            if (t < s) {
                int p = s - 1 - t;
                int d = (t == 0) ? (int)(Z >> (8 * p)) : (int)((Z >> (8 * p)) & 0xff) - 128;
                dw.w[t][wi] |= ((uint32_t)d & 0xffu) << sh_i;
            }
        }
    }
}

template <int SMAX>
__device__ __forceinline__ void store_digits(const SplitParams &p, int64_t b, int64_t R,
                                             int64_t Cchunk, const DigitWords<SMAX> &dw) {
    const int64_t tile = R / p.tile_h;
    const int64_t rr = R % p.tile_h;
    const int64_t kb = Cchunk >> 1;
    const int64_t cc = Cchunk & 1;
    const int64_t blk = (int64_t)p.tile_h * 32;   // bytes of one (slice, k-block) block
    int8_t *dst = p.out + (((b * p.tiles + tile) * p.KB + kb) * p.s) * blk + (rr >> 3) * 256 +
                  cc * 128 + (rr & 7) * 16;
#pragma unroll
    for (int t = 0; t < SMAX; ++t) {
        if (t < p.s) {
            uint4 v = make_uint4(dw.w[t][0], dw.w[t][1], dw.w[t][2], dw.w[t][3]);
            *reinterpret_cast<uint4 *>(dst + t * blk) = v;
        }
    }
}

template <int SMAX>
__device__ __forceinline__ void zero_words(DigitWords<SMAX> &dw) {
#pragma unroll
    for (int t = 0; t < SMAX; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) dw.w[t][q] = 0;
}

// Phase 2.  Thread = (input row r, 16-wide chunk c of the input depth).
// block (64, 4): x -> row (coalesced when rows are contiguous, and 8
// consecutive rows write one contiguous 128-B core matrix), y -> chunk.
template <int SMAX>
__global__ void __launch_bounds__(256) k_slice(const SplitParams p) {
    const int64_t b = blockIdx.z;
    const int64_t r = (int64_t)blockIdx.x * 64 + threadIdx.x;
    const int64_t c = (int64_t)blockIdx.y * 4 + threadIdx.y;
    const bool four_m = (p.mode == SPLIT_A4M || p.mode == SPLIT_B4M);
    const int64_t nchunks = four_m ? (p.kh >> 4) : (p.KB * 2);
    if (r >= p.rows_grid || c >= nchunks) return;

    const bool row_ok = r < p.rows;
    int32_t e = 0;
    if (row_ok) e = p.exps[b * p.rows_out + (p.mode == SPLIT_B4M ? 2 * r : r)];
    const bool live = row_ok && e != kNonFinite;
    const int64_t l0 = c * 16;
    DigitWords<SMAX> dw;

    if (p.mode == SPLIT_REAL) {
        const double *base = reinterpret_cast<const double *>(p.X) + b * p.bstride + r * p.rs;
        double x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            int64_t l = l0 + i;
            x[i] = (live && l < p.k) ? __ldg(base + l * p.ls) : 0.0;
        }
        zero_words(dw);
#pragma unroll
        for (int i = 0; i < 16; ++i) put_digits<SMAX>(dw, i, x[i], e, p.s);
        store_digits<SMAX>(p, b, r, c, dw);
        return;
    }

    const double2 *base = reinterpret_cast<const double2 *>(p.X) + b * p.bstride + r * p.rs;
    double re[16], im[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        int64_t l = l0 + i;
        double2 v = (live && l < p.k) ? __ldg(base + l * p.ls) : make_double2(0.0, 0.0);
        re[i] = v.x;
        im[i] = p.conj ? -v.y : v.y;
    }
    if (p.mode == SPLIT_RE || p.mode == SPLIT_IM || p.mode == SPLIT_SUM) {
        zero_words(dw);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            double x = p.mode == SPLIT_RE ? re[i] : (p.mode == SPLIT_IM ? im[i] : __dadd_rn(re[i], im[i]));
            put_digits<SMAX>(dw, i, x, e, p.s);
        }
        store_digits<SMAX>(p, b, r, c, dw);
        return;
    }
    const int64_t c2 = (p.kh >> 4) + c;   // chunk index in the second half
    if (p.mode == SPLIT_A4M) {            // row r = [Re | Im]
        zero_words(dw);
#pragma unroll
        for (int i = 0; i < 16; ++i) put_digits<SMAX>(dw, i, re[i], e, p.s);
        store_digits<SMAX>(p, b, r, c, dw);
        zero_words(dw);
#pragma unroll
        for (int i = 0; i < 16; ++i) put_digits<SMAX>(dw, i, im[i], e, p.s);
        store_digits<SMAX>(p, b, r, c2, dw);
        return;
    }
    // SPLIT_B4M: column 2r = [Re ; -Im], column 2r+1 = [Im ; Re]; -Im is split
    // from the negated FP64 value (balanced digits are not sign-symmetric, R9).
    zero_words(dw);
#pragma unroll
    for (int i = 0; i < 16; ++i) put_digits<SMAX>(dw, i, re[i], e, p.s);
    store_digits<SMAX>(p, b, 2 * r, c, dw);
    store_digits<SMAX>(p, b, 2 * r + 1, c2, dw);
    zero_words(dw);
#pragma unroll
    for (int i = 0; i < 16; ++i) put_digits<SMAX>(dw, i, im[i], e, p.s);
    store_digits<SMAX>(p, b, 2 * r + 1, c, dw);
    zero_words(dw);
#pragma unroll
    for (int i = 0; i < 16; ++i) put_digits<SMAX>(dw, i, -im[i], e, p.s);
    store_digits<SMAX>(p, b, 2 * r, c2, dw);
}

}  // namespace ozk
