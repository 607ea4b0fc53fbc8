// split.cuh -- K1: exponent scan + INT8 slicing (the bandwidth-bound half).
//
// Method (§2.2 "splits high-precision input matrices into slices
// ... based on their significant bits and exponent alignment"; readings R3/R4
// in DESIGN.md §3):
//   pass 1 (k_split): e_r = exponent rule R3 applied to max |x| of the
//            r-th "row" (row of op(A) / column of op(B)), by a max-reduction of
//            IEEE bit patterns.
//   pass 2 (k_split): X = RNE(x * 2^(8s-1-e_r)), then s balanced base-256
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

#include <type_traits>

#include "crt.cuh"
#include "numerics.cuh"

namespace ozk {

__device__ __forceinline__ uint32_t smem_u32_split(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

enum SplitMode : int {
    SPLIT_REAL = 0,   // real operand
    SPLIT_A4M = 1,    // complex op(A) -> row r: [Re | Im]
    SPLIT_B4M = 2,    // complex op(B) -> columns 2j: [Re ; -Im], 2j+1: [Im ; Re]  (R9, N side)
    SPLIT_RE = 3,     // 3M operands: Re, Im, fl(Re + Im)
    SPLIT_IM = 4,
    SPLIT_SUM = 5,
    SPLIT_3M = 6,     // all three 3M operands (Re, Im, fl(Re + Im)) in one pass, regions x = 0, 1, 2
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
    int64_t kbs_bytes;    // bytes between k-blocks of one tile (Ozaki-I: s*blk; Ozaki-II: blk)
    int64_t ss_bytes;     // bytes between slices / moduli  (Ozaki-I: blk;  Ozaki-II: KB*blk)
    int64_t x_bytes;      // SPLIT_3M: bytes between the Re / Im / Sum slice regions
    int64_t x_exps;       // SPLIT_3M: exponents between the three regions
    uint32_t *emax;       // long-row split: per-row biased exponents [NX][batch][rows] (atomicMax)
    int32_t kchunk;       // long-row split: depth per k_split_exps CTA
    CrtTab crt;           // Ozaki-II constants (CRT instantiation only)
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

__device__ __forceinline__ void reduce_and_store(const SplitParams &p, int64_t b, int64_t r, int32_t e,
                                                 uint32_t nf) {
    int32_t *ex = p.exps + b * p.rows_out;
    if (p.mode == SPLIT_B4M) {
        ex[2 * r] = e;
        ex[2 * r + 1] = e;
    } else {
        ex[r] = e;
    }
    if (nf) atomicAdd(p.nonfinite, 1ull);
}

// ------------------------------------------------------------------ digits
// R4: X = RNE(x 2^(P-e)), P = 8s-1; balanced digits via the offset trick:
// with Bofs = sum_{p=0}^{s-2} 128*256^p, Z = X + Bofs has plain base-256 bytes
// (d_t + 128) at positions p = s-t for t >= 2 and d_1 = Z >> 8(s-1).
// 4x4 byte transpose: out[q] byte i = in[i] byte q.
__device__ __forceinline__ void transpose4x4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint32_t &o0, uint32_t &o1, uint32_t &o2, uint32_t &o3) {
    const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a2, a3, 0x5140);
    const uint32_t t2 = __byte_perm(a0, a1, 0x7362), t3 = __byte_perm(a2, a3, 0x7362);
    o0 = __byte_perm(t0, t1, 0x5410);
    o1 = __byte_perm(t0, t1, 0x7632);
    o2 = __byte_perm(t2, t3, 0x5410);
    o3 = __byte_perm(t2, t3, 0x7632);
}

// transpose the 8 values' digit words w[j][i] and store one 8-byte word per slice
template <int NW>
__device__ __forceinline__ void store_planes(const uint32_t (&w)[NW][8], int s, int8_t *dst0, int8_t *dst1,
                                             int64_t blk) {
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        uint32_t lo[4], hi[4];   // slice word halves for byte positions q = 4j .. 4j+3
        transpose4x4(w[j][0], w[j][1], w[j][2], w[j][3], lo[0], lo[1], lo[2], lo[3]);
        transpose4x4(w[j][4], w[j][5], w[j][6], w[j][7], hi[0], hi[1], hi[2], hi[3]);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const int q = 4 * j + qq;
            if (q < s) {
                const int64_t off = (int64_t)(s - 1 - q) * blk;
                const uint2 val = make_uint2(lo[qq], hi[qq]);
                *reinterpret_cast<uint2 *>(dst0 + off) = val;
                if (dst1) *reinterpret_cast<uint2 *>(dst1 + off) = val;
            }
        }
    }
}

// R4 for 8 consecutive values and the s slices of their 8-byte output.
// X = RNE(x 2^(P-e)): x * scale with scale = 2^(P-e) (one exact-or-correctly-
// rounded DMUL, identical to ldexp) when the power is representable, else
// ldexp_rn.  With B = 0x80 in each of the s-1 low bytes, Y = (X + B) XOR B
// holds every balanced digit as a byte (byte q = digit of slice t = s - q);
// an 8x8 byte transpose (PRMT) gives one 8-byte word per slice.  dst0 / dst1
// receive the digits of X, dstn (optional) the digits of -X (RNE is sign-
// symmetric, so -X is exactly the integer of the negated values).
template <int SMAX, bool NEG>
__device__ __forceinline__ void digits_store8_impl(const double (&v)[8], double scale, int32_t e, int s,
                                                   int8_t *dst0, int8_t *dst1, int8_t *dstn, int64_t blk) {
    const int P = 8 * s - 1;
    constexpr int NW = SMAX / 4;   // 32-bit words of Y per value
    uint32_t w[NW][8], wn[NW][8];
    if constexpr (SMAX <= 8) {
        const unsigned long long B = 0x0080808080808080ull >> (8 * (8 - s));
        long long Xs[8];
        if (scale != 0.0) {          // the power 2^(P-e) is a normal double: one exact DMUL
#pragma unroll
            for (int i = 0; i < 8; ++i) Xs[i] = __double2ll_rn(__dmul_rn(v[i], scale));
        } else {
            for (int i = 0; i < 8; ++i) Xs[i] = __double2ll_rn(ldexp_rn(v[i], P - e));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long long X = Xs[i];                                  // |X| <= 127*2^(8s-8)
            const unsigned long long Y = ((unsigned long long)X + B) ^ B;
            w[0][i] = (uint32_t)Y;
            w[1][i] = (uint32_t)(Y >> 32);
            if constexpr (NEG) {
                const unsigned long long Yn = ((unsigned long long)(-X) + B) ^ B;
                wn[0][i] = (uint32_t)Yn;
                wn[1][i] = (uint32_t)(Yn >> 32);
            }
        }
    } else {
        unsigned __int128 B = 0;
        for (int q = 0; q < s - 1; ++q) B |= (unsigned __int128)0x80 << (8 * q);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double x = (scale != 0.0) ? __dmul_rn(v[i], scale) : ldexp_rn(v[i], P - e);   // |x| < 2^127
            __int128 X;
            if (fabs(x) < 9223372036854775808.0) {
                X = (__int128)__double2ll_rn(x);
            } else {                                                         // integer mant * 2^q
                const uint64_t bits = (uint64_t)__double_as_longlong(x);
                const int q = (int)((bits >> 52) & 0x7ff) - 1075;
                X = (__int128)((bits & kFracMask) | (1ull << 52)) << q;
                if (bits >> 63) X = -X;
            }
            const unsigned __int128 Y = ((unsigned __int128)X + B) ^ B;
#pragma unroll
            for (int j = 0; j < NW; ++j) w[j][i] = (uint32_t)(Y >> (32 * j));
            if constexpr (NEG) {
                const unsigned __int128 Yn = ((unsigned __int128)(-X) + B) ^ B;
#pragma unroll
                for (int j = 0; j < NW; ++j) wn[j][i] = (uint32_t)(Yn >> (32 * j));
            }
        }
    }
    store_planes<NW>(w, s, dst0, dst1, blk);
    if constexpr (NEG) store_planes<NW>(wn, s, dstn, nullptr, blk);
}

// dstn == nullptr (every target but 4M's -Im block): no negated digits at all
template <int SMAX>
__device__ __forceinline__ void digits_store8(const double (&v)[8], double scale, int32_t e, int s,
                                              int8_t *dst0, int8_t *dst1, int8_t *dstn, int64_t blk) {
    if (dstn) digits_store8_impl<SMAX, true>(v, scale, e, s, dst0, dst1, dstn, blk);
    else digits_store8_impl<SMAX, false>(v, scale, e, s, dst0, dst1, nullptr, blk);
}

// address of the 8-byte half hh of 16-byte chunk C of output row R, slice 1
__device__ __forceinline__ int8_t *slice_addr(const SplitParams &p, int64_t b, int64_t R, int64_t C, int hh) {
    const int64_t tile = R / p.tile_h, rr = R % p.tile_h, kb = C >> 1, cc = C & 1;
    const int64_t blk = (int64_t)p.tile_h * 32;
    return p.out + (((b * p.tiles + tile) * p.KB + kb) * p.s) * blk + (rr >> 3) * 256 + cc * 128 +
           (rr & 7) * 16 + hh * 8;
}

// ------------------------------------------------------------------
// Shared-memory staged variant (the production K1): the 8-row slab is copied
// into SMEM with cp.async (deep memory-level parallelism, no registers), both
// passes read SMEM.  Rows longer than one window (KW elements) are streamed in
// windows: pass 1 scans all windows, pass 2 reloads them (second read hits L2).
__device__ __forceinline__ void cp_async8(void *smem, const void *g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32_split(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32_split(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// CRT = false: Ozaki-I digits (R3, R4); CRT = true: Ozaki-II exponent, int64
// quantisation and centred residues per modulus (R17, R18), written
// modulus-major within a tile (contiguous k-blocks per modulus).
// Both operands of a GEMM in ONE launch: blockIdx.z selects the side (one launch gap and one
// tail fewer than two launches); the row-contiguity of the view is a runtime property.
struct SplitPair {
    SplitParams side[2];
};

template <int SMAX, bool CPLX, bool CRT = false>
__global__ void __launch_bounds__(256) k_split_sm(const __grid_constant__ SplitPair pp, int KW) {
    // let the dependent GEMM (launched with programmatic stream serialisation) start its
    // prologue as soon as every split CTA is resident; it waits for our completion itself
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const SplitParams &p = pp.side[blockIdx.z];
    if ((int64_t)blockIdx.x * 8 >= p.rows_grid) return;   // the other side needs more row groups
    const bool RCONTIG = (p.rs == 1);                     // 8 rows adjacent in memory for each l
    extern __shared__ __align__(16) uint8_t sbuf[];
    __shared__ int32_t s_e[8];
    __shared__ double s_scale[8];
    __shared__ int32_t s_e3[3][8];         // SPLIT_3M: per-operand exponents / scales
    __shared__ double s_scale3[3][8];
    __shared__ int8_t *s_rowbase[16];      // output row base (tile, row-in-tile part of the address)
    using Elem = typename std::conditional<CPLX, double2, double>::type;
    constexpr int ES = sizeof(Elem);
    const int ld = KW + (16 / ES);                 // padded row stride (elements) against bank conflicts
    Elem *slab = reinterpret_cast<Elem *>(sbuf);
    const int tid = threadIdx.x;
    const int64_t b = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 8;
    const Elem *X = reinterpret_cast<const Elem *>(p.X) + b * p.bstride;
    const bool four_m = (p.mode == SPLIT_A4M || p.mode == SPLIT_B4M);
    const int64_t kpad = four_m ? p.kh : p.KB * 32;  // input depth covered by output chunks
    const int64_t nwin = (kpad + KW - 1) / KW;
    const int nrows = (int)min((int64_t)8, max((int64_t)0, p.rows - r0));
    const int64_t blk = (int64_t)p.tile_h * 32;      // bytes of one (tile, k-block, slice) block
    const int64_t kbs = p.kbs_bytes;                 // bytes between k-blocks of one tile
    const int64_t tile_bytes = (int64_t)p.s * p.KB * blk;

    if (tid < 16) {   // output rows of this block: r0..r0+7 (B4M: 2r0 .. 2r0+15)
        const int64_t R = (p.mode == SPLIT_B4M ? 2 * r0 : r0) + tid;
        const int64_t tile = R / p.tile_h, rr = R % p.tile_h;
        s_rowbase[tid] = p.out + (b * p.tiles + tile) * tile_bytes + (rr >> 3) * 256 + (rr & 7) * 16;
    }

    auto load_window = [&](int64_t w0) {
        const int wlen = (int)min((int64_t)KW, p.k - w0);   // valid elements in this window
        if (wlen <= 0) return;
        if (RCONTIG) {   // 8 rows adjacent in memory for each l
            // blockDim = 256 is a multiple of 8: a thread keeps its row (tid & 7) and walks l
            // in steps of 32 -- pointer increments only, no per-copy index math
            const int row = tid & 7;
            if (row < nrows) {
                const int64_t gstep = 32 * p.ls;
                const Elem *g = X + r0 * p.rs + w0 * p.ls + row + (int64_t)(tid >> 3) * p.ls;
                Elem *d = slab + row * ld + (tid >> 3);
#pragma unroll 4
                for (int l = tid >> 3; l < wlen; l += 32) {
                    if (CPLX) cp_async16(d, g);
                    else cp_async8(d, g);
                    g += gstep;
                    d += 32;
                }
            }
        } else {         // each row contiguous along l
            for (int row = 0; row < nrows; ++row) {
                const Elem *g = X + (r0 + row) * p.rs + w0;
                for (int l = tid; l < wlen; l += blockDim.x) {
                    if (CPLX) cp_async16(slab + row * ld + l, g + l);
                    else cp_async8(slab + row * ld + l, g + l);
                }
            }
        }
        cp_async_wait_all();
    };

    // ---------------- pass 1: exponents
    if (CPLX && !CRT && p.mode == SPLIT_3M) {
        // R9 3M: three operands Re, Im (conj applied) and fl(Re + Im), each with its own exponent
        const int row = tid >> 5, lane = tid & 31;
        uint64_t m3[3] = {0, 0, 0};
        for (int64_t w = 0; w < nwin; ++w) {
            const int64_t w0 = w * KW;
            load_window(w0);
            __syncthreads();
            const int wlen = (int)min((int64_t)KW, p.k - w0);
            if (row < nrows) {
                const double *src = reinterpret_cast<const double *>(slab + row * ld);
                for (int l = lane; l < wlen; l += 32) {
                    const double re = src[2 * l], im = p.conj ? -src[2 * l + 1] : src[2 * l + 1];
                    const uint64_t u0 = (uint64_t)__double_as_longlong(re) & kAbsMask;
                    const uint64_t u1 = (uint64_t)__double_as_longlong(im) & kAbsMask;
                    const uint64_t u2 = (uint64_t)__double_as_longlong(__dadd_rn(re, im)) & kAbsMask;
                    m3[0] = u0 > m3[0] ? u0 : m3[0];
                    m3[1] = u1 > m3[1] ? u1 : m3[1];
                    m3[2] = u2 > m3[2] ? u2 : m3[2];
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int x = 0; x < 3; ++x) {
            uint64_t m = m3[x];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t om = __shfl_xor_sync(0xffffffffu, m, o);
                m = om > m ? om : m;
            }
            if (lane == 0) {
                int32_t e = 0;
                if (row < nrows) {
                    const uint32_t nf3 = (m >= kExpInf);
                    e = nf3 ? kNonFinite : exponent_from_maxbits(m);
                    p.exps[x * p.x_exps + b * p.rows_out + r0 + row] = e;
                    if (nf3) atomicAdd(p.nonfinite, 1ull);
                }
                s_e3[x][row] = e;
                const int sh = 8 * p.s - 1 - e;
                s_scale3[x][row] = (sh >= -1022 && sh <= 1023) ? pow2(sh) : 0.0;
                if (x == 0) s_e[row] = 0;   // pass 2's row-liveness; each operand checks its own e
            }
        }
        __syncthreads();
    } else {
        const int row = tid >> 5, lane = tid & 31;
        uint64_t m = 0;
        uint32_t nf = 0;
        for (int64_t w = 0; w < nwin; ++w) {
            const int64_t w0 = w * KW;
            load_window(w0);
            __syncthreads();
            const int wlen = (int)min((int64_t)KW, p.k - w0);
            if (row < nrows) {
                const Elem *src = slab + row * ld;
                for (int l = lane; l < wlen; l += 32) {
                    const Elem x = src[l];
                    uint64_t u;
                    if constexpr (!CPLX) {
                        u = (uint64_t)__double_as_longlong(x) & kAbsMask;
                    } else {
                        const uint64_t ur = (uint64_t)__double_as_longlong(x.x) & kAbsMask;
                        const uint64_t ui = (uint64_t)__double_as_longlong(x.y) & kAbsMask;   // |conj| = |.|
                        if (p.mode == SPLIT_RE) u = ur;
                        else if (p.mode == SPLIT_IM) u = ui;
                        else if (p.mode == SPLIT_SUM)
                            u = (uint64_t)__double_as_longlong(__dadd_rn(x.x, p.conj ? -x.y : x.y)) & kAbsMask;
                        else u = ur > ui ? ur : ui;
                    }
                    m = u > m ? u : m;   // Inf/NaN patterns exceed every finite |x|
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t om = __shfl_xor_sync(0xffffffffu, m, o);
            m = om > m ? om : m;
        }
        nf = (m >= kExpInf);     // some entry of the row is Inf / NaN (R10)
        if (lane == 0) {
            int32_t e = 0;
            if (row < nrows) {
                e = nf ? kNonFinite : (CRT ? crt_exponent(m, p.crt.nu) : exponent_from_maxbits(m));
                reduce_and_store(p, b, r0 + row, e, nf);
            }
            s_e[row] = e;
            const int sh = (CRT ? p.crt.nu : 8 * p.s - 1) - e;   // 2^(P-e) as one exact DMUL when representable
            s_scale[row] = (sh >= -1022 && sh <= 1023) ? pow2(sh) : 0.0;
        }
        __syncthreads();
    }
    // ---------------- pass 2: digits; one item = (row, 8-value half chunk), all targets
    const int64_t c2off = p.kh >> 4;
    for (int64_t w = 0; w < nwin; ++w) {
        const int64_t w0 = w * KW;
        if (nwin > 1) {
            __syncthreads();
            load_window(w0);
            __syncthreads();
        }
        const int wh = (int)((min((int64_t)KW, kpad - w0) + 7) / 8);   // 8-value units in window
        for (int item = tid; item < 8 * wh; item += blockDim.x) {
            const int row = item & 7;
            const int h = item >> 3;
            const int lw = h * 8;                      // offset in window
            const int64_t l0 = w0 + lw;                // input depth index
            const int32_t e = s_e[row];
            const double scale = s_scale[row];
            const bool live = (row < nrows) && (e != kNonFinite);
            const int nvalid = live ? (int)min((int64_t)8, max((int64_t)0, p.k - l0)) : 0;
            const Elem *src = slab + row * ld + lw;
            const int64_t c = l0 >> 4;
            const int hh = (int)((l0 >> 3) & 1);
            const int64_t coff = (c >> 1) * kbs + (c & 1) * 128 + hh * 8;            // first half
            const int64_t coff2 = ((c + c2off) >> 1) * kbs + ((c + c2off) & 1) * 128 + hh * 8;   // second half
            auto emit = [&](const double (&vv)[8], int8_t *d0, int8_t *d1, int8_t *dn) {
                if constexpr (CRT) residues_store8(vv, scale, e, p.crt, d0, d1, dn, p.ss_bytes);
                else digits_store8<SMAX>(vv, scale, e, p.s, d0, d1, dn, blk);
            };
            if constexpr (!CPLX) {
                double v[8];
                if (nvalid == 8) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = src[i];
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = (i < nvalid) ? src[i] : 0.0;
                }
                emit(v, s_rowbase[row] + coff, nullptr, nullptr);
            } else {
                // one component at a time (8 live values): 0 = Re, 1 = Im (conj applied), 2 = Re + Im
                auto comp8 = [&](int comp, double (&v)[8]) {
                    const double *xe = reinterpret_cast<const double *>(src);
                    if (nvalid == 8 && comp < 2) {          // full item, plain component
                        const double sg = (comp == 1 && p.conj) ? -1.0 : 1.0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[i] = (comp == 0) ? xe[2 * i] : sg * xe[2 * i + 1];
                        return;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        double val = 0.0;
                        if (i < nvalid) {
                            const double re = xe[2 * i], im0 = xe[2 * i + 1];
                            const double im = p.conj ? -im0 : im0;
                            val = comp == 0 ? re : (comp == 1 ? im : __dadd_rn(re, im));
                        }
                        v[i] = val;
                    }
                };
                double v[8];
                switch (p.mode) {
                    case SPLIT_3M:
                        if constexpr (!CRT) {
                            const bool live3 = row < nrows;
#pragma unroll 1
                            for (int x = 0; x < 3; ++x) {
                                const int32_t ex = s_e3[x][row];
                                if (live3 && ex != kNonFinite) comp8(x, v);
                                else {
#pragma unroll
                                    for (int q = 0; q < 8; ++q) v[q] = 0.0;
                                }
                                digits_store8<SMAX>(v, s_scale3[x][row], ex, p.s,
                                                    s_rowbase[row] + x * p.x_bytes + coff, nullptr, nullptr, blk);
                            }
                        }
                        break;
                    case SPLIT_RE:
                    case SPLIT_IM:
                    case SPLIT_SUM:
                        comp8(p.mode == SPLIT_RE ? 0 : (p.mode == SPLIT_IM ? 1 : 2), v);
                        emit(v, s_rowbase[row] + coff, nullptr, nullptr);
                        break;
                    case SPLIT_A4M:   // row r = [Re | Im]
                        comp8(0, v);
                        emit(v, s_rowbase[row] + coff, nullptr, nullptr);
                        comp8(1, v);
                        emit(v, s_rowbase[row] + coff2, nullptr, nullptr);
                        break;
                    default:          // SPLIT_B4M: 2r = [Re | -Im], 2r+1 = [Im | Re] (R9)
                        comp8(0, v);
                        emit(v, s_rowbase[2 * row] + coff, s_rowbase[2 * row + 1] + coff2, nullptr);
                        comp8(1, v);
                        emit(v, s_rowbase[2 * row + 1] + coff, nullptr, s_rowbase[2 * row] + coff2);
                        break;
                }
            }
        }
    }
}

}  // namespace ozk
