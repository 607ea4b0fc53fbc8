// gemm.cuh -- K2 + K3: the slice-pair INT8 GEMM on tcgen05 (kind::i8) with the
// level sums resident in TMEM and the FP64 rescale / accumulate / alpha-beta
// epilogue fused in the same persistent kernel.
//
// Method (§2.2: "performs low-precision matrix multiplications on
// these slices and accumulates them in higher precision"; readings R1, R6, R7):
//   for every output tile (BM = 128 rows of op(A)' x BN columns of op(B)):
//     S_L = sum_{t+u=L} A_t B_u^T   (L = 2..s+1, exact INT32)   -- tcgen05.mma
//     acc = sum_{L=s+1..2} S_L 2^(-8(L-2))  in FP64, ascending   -- epilogue
//     P   = acc * 2^(e_i + f_j - 14);  C = alpha P + beta C       -- epilogue
//
// B200 design:
//   * K-outer loop: one pipeline stage carries ALL s slices of A and of B for a
//     32-byte K block, and every retained pair (t,u) is issued from it, so each
//     slice byte crosses L2->SMEM once per tile (not (s+1)/2 times).  The s
//     level sums live side by side in TMEM: S_L at columns (L-2)*BN, which is
//     why BN = 64 for s <= 8 and BN = 32 for s <= 16 (s*BN <= 512 columns).
//   * Operands arrive pre-tiled by K1 in the canonical no-swizzle K-major
//     layout, so one stage = two cp.async.bulk copies (no tensor maps).
//   * Warp roles: warp 0 = bulk-copy producer, warp 1 = TMEM owner + single
//     thread MMA issuer, warps 2..9 = FP64 epilogue (2 per TMEM lane quarter).
//   * Persistent: grid = min(#tiles, #SMs); tiles (batch, m, n) are walked with
//     a grouped raster so concurrently running CTAs share operand tiles in L2.
#pragma once
// EPI_LEVELS (debug) instantiations `continue` before the FP64 epilogue of the same loop body
#pragma nv_diag_suppress 128
#include <cstdint>

#include "numerics.cuh"
#include "ptx.cuh"

namespace ozk {

enum EpiMode : int { EPI_REAL = 0, EPI_CPLX4M = 1, EPI_LEVELS = 2 };

constexpr int kBM = 128;            // rows per tile (UMMA M)
constexpr int kKB = 32;             // bytes of K per block (one kind::i8 MMA)
constexpr int kNumEpiWarps = 8;
constexpr int kGemmThreads = 64 + 32 * kNumEpiWarps;   // 320
constexpr int kRasterGroup = 8;

struct GemmParams {
    const int8_t *A;        // tiled slices of op(A)'  [batch][tiles_m][KB][s][128x32]
    const int8_t *B;        // tiled slices of op(B)'^T [batch][tiles_n][KB][s][BNx32]
    const int32_t *ea;      // [batch][Mp] row exponents
    const int32_t *fb;      // [batch][N]  column exponents
    int64_t Mp, N, KB;
    int64_t tiles_m, tiles_n, batch;
    int32_t s, kps, stages;
    uint32_t a_kb_bytes, b_kb_bytes;
    double *C;              // real: double elements; complex: interleaved pairs
    int64_t ldc, strideC;   // in elements (complex elements for EPI_CPLX4M)
    double alpha_r, alpha_i, beta_r, beta_i;
    int ab_unit;               // alpha == 1 (+0i) and beta == 0: C = P, no FP64 in the store
    int32_t *S_out;         // EPI_LEVELS
    // K-chunking (reading R8): this launch covers k-blocks [kb_begin, kb_end);
    // chunk_mode 0 = whole K, 1 = first chunk (W = S), 2 = middle (W += S),
    // 3 = last (level sum = W + S, then the FP64 combine).  W holds the exact
    // integer partial level sums in FP64 (< 2^53): W[(L-2)*w_lvl + col*Mp + row].
    int64_t kb_begin, kb_end;
    int32_t chunk_mode;
    double *W;
    int64_t w_lvl;
    // Split-K for small problems: the CTA pairs run splitk work units per
    // tile, unit u = (tile u / splitk, split q = u % splitk) over an equal share of the
    // k-blocks; each writes its EXACT partials -- the int64 prefix of the first pass's levels
    // (R6's exact part) to P0 and the int32 sums of the later levels to PL -- and
    // k_splitk_combine adds them (integers: order-free) and runs the FP64 combine + store.
    // Layout: P0[q][b][col][row], PL[q][li][b][col][row] (li = later level index).
    int32_t splitk;
    int32_t pk_nl;         // later levels per unit (PL planes)
    int64_t *P0;
    int32_t *PL;
    unsigned long long *dbg;   // optional per-CTA role timers (ozaki_debug_timing), null = off
};

// Role timer slots (clock64 cycles summed per CTA) written when p.dbg != null.
enum DbgSlot : int {
    DBG_PROD_WAIT = 0,   // producer waiting for a free stage
    DBG_MMA_WAIT_FULL,   // MMA thread waiting for operands
    DBG_MMA_WAIT_SLOT,   // MMA thread waiting for the epilogue to drain TMEM
    DBG_MMA_TOTAL,       // MMA thread lifetime
    DBG_EPI_WAIT,        // epilogue waiting for a completed pass (warp 2, lane 0)
    DBG_EPI_DRAIN,       // epilogue TMEM -> FP64 accumulate (warp 2)
    DBG_EPI_STORE,       // epilogue ldexp + alpha/beta + store (warp 2)
    DBG_TOTAL,           // CTA lifetime (warp 1)
    DBG_MMA_WAIT_SLOT0,  // part of DBG_MMA_WAIT_SLOT spent before the first pass of a tile
    DBG_EPI_PREFIX,      // part of DBG_EPI_DRAIN spent in the exact-prefix levels (warp 2)
    DBG_EPI_FIRST_ARRIVE,// pass_full -> first slot released, first pass (warp 2)
    DBG_MMA_WAIT_FULL0,  // part of DBG_MMA_WAIT_FULL at the first k-block of a pass
    DBG_MMA_WAIT_FULLP0, // part of DBG_MMA_WAIT_FULL inside pass 0
    DBG_TL0 = 32,        // timeline of CTA 0 (globaltimer ns): slots DBG_TL0 + event
    DBG_NSLOT = 64
};

// debug timers (cold path): accumulate straight into the device buffer so no
// timer stays live in registers across the tile loop
__device__ __forceinline__ void dbg_add(const GemmParams &p, int slot, long long v) {
    atomicAdd(p.dbg + slot, (unsigned long long)v);
}

// Tile index -> (batch entry, row tile, column tile), raster groups of kRasterGroup row tiles.
// 32-bit arithmetic: the host keeps batch x tiles (x split-K units) below 2^31 (make_plan), and
// a 64-bit division is a long software sequence on the critical path of every tile.
__device__ __forceinline__ void decode_tile(const GemmParams &p, int64_t tile, int64_t &b,
                                            int64_t &tm, int64_t &tn) {
    const uint32_t t = (uint32_t)tile, tiles_m = (uint32_t)p.tiles_m, tiles_n = (uint32_t)p.tiles_n;
    const uint32_t per_batch = tiles_m * tiles_n;
    const uint32_t bb = t / per_batch;
    const uint32_t r = t - bb * per_batch;
    const uint32_t gsize = (uint32_t)kRasterGroup * tiles_n;
    const uint32_t group = r / gsize;
    const uint32_t first_m = group * kRasterGroup;
    const uint32_t gm = min((uint32_t)kRasterGroup, tiles_m - first_m);
    const uint32_t in_g = r - group * gsize;
    b = bb;
    tm = first_m + in_g % gm;
    tn = in_g / gm;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm(const __grid_constant__ GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t a_stage = (uint32_t)p.kps * p.a_kb_bytes;
    const uint32_t b_stage = (uint32_t)p.kps * p.b_kb_bytes;
    uint8_t *sA = smem;
    uint8_t *sB = smem + (size_t)p.stages * a_stage;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + (size_t)p.stages * b_stage);
    uint64_t *empty = full + p.stages;
    uint64_t *tfull = empty + p.stages;
    uint64_t *tempty = tfull + 1;
    uint32_t *tholder = reinterpret_cast<uint32_t *>(tempty + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int s = p.s;
    const int64_t total = p.batch * p.tiles_m * p.tiles_n;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < p.stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, kNumEpiWarps);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tholder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tholder;

    if (warp == 0) {
        // ===================== producer: one bulk copy per operand per stage
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
                int64_t b, tm, tn;
                decode_tile(p, tile, b, tm, tn);
                const int8_t *ga = p.A + (b * p.tiles_m + tm) * p.KB * (int64_t)p.a_kb_bytes;
                const int8_t *gb = p.B + (b * p.tiles_n + tn) * p.KB * (int64_t)p.b_kb_bytes;
                for (int64_t kb0 = 0; kb0 < p.KB; kb0 += p.kps) {
                    const uint32_t nk = (uint32_t)min((int64_t)p.kps, p.KB - kb0);
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t ba = nk * p.a_kb_bytes, bb = nk * p.b_kb_bytes;
                    mbar_arrive_expect_tx(&full[stage], ba + bb);
                    bulk_g2s(sA + (size_t)stage * a_stage, ga + kb0 * p.a_kb_bytes, ba, &full[stage]);
                    bulk_g2s(sB + (size_t)stage * b_stage, gb + kb0 * p.b_kb_bytes, bb, &full[stage]);
                    if (++stage == (uint32_t)p.stages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer: all retained pairs from each stage
        constexpr uint32_t idesc = idesc_i8(kBM, BN);
        uint32_t stage = 0, phase = 0, tphase = 0;
        for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
            mbar_wait(tempty, tphase ^ 1);   // epilogue drained the previous tile
            tc_fence_after();
            for (int64_t kb0 = 0; kb0 < p.KB; kb0 += p.kps) {
                const int nk = (int)min((int64_t)p.kps, p.KB - kb0);
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA + (size_t)stage * a_stage);
                    const uint32_t b0 = smem_u32(sB + (size_t)stage * b_stage);
                    for (int kk = 0; kk < nk; ++kk) {
                        for (int t = 0; t < s; ++t) {
                            const uint64_t adesc = smem_desc_kmajor_noswz(
                                a0 + (uint32_t)(kk * s + t) * (kBM * kKB), 128, 256);
                            for (int u = 0; u + t < s; ++u) {
                                const uint64_t bdesc = smem_desc_kmajor_noswz(
                                    b0 + (uint32_t)(kk * s + u) * (BN * kKB), 128, 256);
                                const int lvl = t + u;   // L - 2
                                // first write of level L in this tile overwrites
                                const bool first = (kb0 == 0 && kk == 0 && t == max(0, lvl + 1 - s));
                                mma_i8(tbase + (uint32_t)(lvl * BN), adesc, bdesc, idesc, first ? 0u : 1u);
                            }
                        }
                    }
                    mma_commit(&empty[stage]);   // frees the SMEM stage when these MMAs finish
                }
                __syncwarp();
                if (++stage == (uint32_t)p.stages) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) mma_commit(tfull);    // all level sums of this tile complete
            __syncwarp();
            tphase ^= 1;
        }
    } else {
        // ===================== epilogue: FP64 combine + alpha/beta + store
        const int ew = warp - 2;
        const int q = warp & 3;                  // TMEM lane quarter of this warp
        const int half = ew >> 2;                // which half of the BN columns
        constexpr int kCols = BN / 2;
        uint32_t tphase = 0;
        for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
            int64_t b, tm, tn;
            decode_tile(p, tile, b, tm, tn);
            mbar_wait(tfull, tphase);
            tc_fence_after();
            const int row_local = q * 32 + lane;
            const int64_t grow = tm * kBM + row_local;
            const bool row_ok = grow < p.Mp;
            const int32_t e = row_ok ? p.ea[b * p.Mp + grow] : 0;
            const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
            for (int ch = 0; ch < kCols / 16; ++ch) {
                const int col_local = half * kCols + ch * 16;
                if constexpr (EPI == EPI_LEVELS) {
                    for (int L = s + 1; L >= 2; --L) {
                        uint32_t v[16];
                        tmem_ld_32x32b_x16(tl + (uint32_t)((L - 2) * BN + col_local), v);
                        tmem_wait_ld();
                        if (b == 0 && row_ok) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const int64_t gcol = tn * BN + col_local + j;
                                if (gcol < p.N)
                                    p.S_out[(int64_t)(L - 2) * p.Mp * p.N + gcol * p.Mp + grow] = (int32_t)v[j];
                            }
                        }
                    }
                    continue;
                }
                double acc[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = 0.0;
                for (int L = s + 1; L >= 2; --L) {      // ascending significance (R6)
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tl + (uint32_t)((L - 2) * BN + col_local), v);
                    tmem_wait_ld();
                    const double sc = pow2(-8 * (L - 2));
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        acc[j] = __fma_rn(__int2double_rn((int32_t)v[j]), sc, acc[j]);   // exact product
                }
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    const int64_t gcol = tn * BN + col_local + j;
                    const int32_t f = (gcol < p.N) ? p.fb[b * p.N + gcol] : 0;
                    const int32_t f1 = (gcol + 1 < p.N) ? p.fb[b * p.N + gcol + 1] : 0;
                    const bool enan = (e == kNonFinite);
                    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
                    const double P0 = (enan || f == kNonFinite) ? qnan : ldexp_rn(acc[j], e + f - 14);
                    const double P1 = (enan || f1 == kNonFinite) ? qnan : ldexp_rn(acc[j + 1], e + f1 - 14);
                    if constexpr (EPI == EPI_REAL) {
                        if (row_ok && gcol < p.N) {
                            double *cp = p.C + b * p.strideC + grow + gcol * p.ldc;
                            *cp = (p.beta_r == 0.0) ? __dmul_rn(p.alpha_r, P0)
                                                    : __fma_rn(p.alpha_r, P0, __dmul_rn(p.beta_r, *cp));
                        }
                        if (row_ok && gcol + 1 < p.N) {
                            double *cp = p.C + b * p.strideC + grow + (gcol + 1) * p.ldc;
                            *cp = (p.beta_r == 0.0) ? __dmul_rn(p.alpha_r, P1)
                                                    : __fma_rn(p.alpha_r, P1, __dmul_rn(p.beta_r, *cp));
                        }
                    } else {   // EPI_CPLX4M, R9 N-side embedding: columns (2c, 2c+1) = (Re, Im)
                        if (row_ok && gcol < p.N) {
                            double2 *cp = reinterpret_cast<double2 *>(p.C) + b * p.strideC + grow + (gcol >> 1) * p.ldc;
                            double tr = 0.0, ti = 0.0;
                            if (!(p.beta_r == 0.0 && p.beta_i == 0.0)) {
                                const double2 cv = *cp;
                                tr = __fma_rn(p.beta_r, cv.x, -__dmul_rn(p.beta_i, cv.y));
                                ti = __fma_rn(p.beta_r, cv.y, __dmul_rn(p.beta_i, cv.x));
                            }
                            *cp = make_double2(__fma_rn(p.alpha_r, P0, __fma_rn(-p.alpha_i, P1, tr)),
                                               __fma_rn(p.alpha_r, P1, __fma_rn(p.alpha_i, P0, ti)));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            tphase ^= 1;
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

}  // namespace ozk
