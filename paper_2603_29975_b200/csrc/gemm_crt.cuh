// gemm_crt.cuh -- Ozaki-II residue GEMMs on CTA pairs (NEXT-1; PAPER.md:99
// "performs multiple matrix multiplications using smaller, pairwise coprime
// moduli"; reading R19).
//
// One INT8 GEMM per modulus: C_q = (rA_q . rB_q) mod p_q.  Unlike Ozaki-I's
// level passes, every residue slice feeds exactly ONE product, so the MMA is
// as wide as possible to halve the shared-memory operand traffic per MMA:
// a CTA pair computes a 256 x 256 tile (cta_group::2, M = 256, N = 256, K = 32,
// 128 clk per SM per instruction) reading 4 KB of A and 4 KB of B per CTA.
// TMEM holds two 256-column accumulator slots: the MMA of modulus q+1 runs
// while the epilogue reduces modulus q (no pass-boundary stall).
// NW = 2 (wide tiles, 256 x 512): each k-block's A tile feeds TWO N = 256 MMAs
// (B tiles t and t + 2 of the pair), so the shared-memory port moves 12 KB in and
// reads 16 KB per two MMAs instead of 8 + 8 KB per one; the two accumulators fill
// TMEM, so the MMA of modulus q+1 waits for the epilogue's loads of modulus q.  The
// epilogue is integer-only (mod p by folding + a 40-bit reciprocal multiply)
// and writes centred residue bytes in 16-byte row chunks:
//   R[q][b][col / 16][row][16]        (plane q, batch b; rows padded to 256)
// The CRT kernel (crt_kernel.cuh) turns the planes into FP64.
#pragma once
#include <cstdint>

#include <cudaTypedefs.h>

#include "crt.cuh"
#include "ptx.cuh"

namespace ozk {

constexpr int kCrtEpi = 16;                       // epilogue warps per CTA (4 lane quarters x 4 column quarters)
constexpr int kCrtThreads = 64 + 32 * kCrtEpi;    // 576
constexpr uint32_t kCrtBlk = 128 * 32;            // one (128-row tile, k-block, modulus) block

struct CrtGemmParams {
    CUtensorMap tmA, tmB;      // residue slices as rows of 256 B; box = kpp * 16 rows
    int64_t batch, tiles_m, tiles_n, KB;
    int32_t kpp, stages;
    uint32_t stage_bytes;      // kpp * 2 * kCrtBlk
    int8_t *R;                 // residue planes
    int64_t plane_bytes, batch_bytes, rows_pad;
    unsigned long long *dbg;
    CrtTab crt;
};

template <int NW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCrtThreads, 1)
    k_gemm_crt(const __grid_constant__ CrtGemmParams P) {
    constexpr int NSLOT = (NW == 1) ? 2 : 1;   // accumulator slots of 256 * NW columns
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = P.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * P.stage_bytes);
    uint64_t *empty = full + S;
    uint64_t *slot_full = empty + S;       // [2]
    uint64_t *slot_empty = slot_full + 2;  // [2], leader only
    uint32_t *tholder = reinterpret_cast<uint32_t *>(slot_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int n = P.crt.n;
    const int64_t per_b = P.tiles_m * P.tiles_n;
    const int64_t total = P.batch * per_b;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int j = 0; j < NSLOT; ++j) {
            mbar_init(&slot_full[j], 1);
            mbar_init(&slot_empty[j], 2 * kCrtEpi);
        }
        fence_mbar_init();
        tma_prefetch_desc(&P.tmA);
        tma_prefetch_desc(&P.tmB);
    }
    if (warp == 1) tmem_alloc_pair(tholder, 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tbase = *tholder;

    if (warp == 0) {
        // ------------------------------------------------ producer (both CTAs)
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            const uint32_t abytes = (uint32_t)P.kpp * kCrtBlk;
            const uint32_t leader_full0 = mapa_shared(smem_u32(&full[0]), 0);
            for (int64_t tile = blockIdx.x >> 1; tile < total; tile += gridDim.x >> 1) {
                const int64_t b = tile / per_b, r = tile - b * per_b;
                const int64_t tm = r / P.tiles_n, tn = r - tm * P.tiles_n;
                const int64_t ta = b * (2 * P.tiles_m) + 2 * tm + rank;   // this CTA's 128-row A tile
                // this CTA's 128-row B tiles: j-th MMA of the tile uses tiles 2 (NW tn + j) + rank
                const int64_t tb = b * (2 * NW * P.tiles_n) + 2 * NW * tn + rank;
                for (int q = 0; q < n; ++q) {
                    for (int64_t kb0 = 0; kb0 < P.KB; kb0 += P.kpp) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        const uint32_t lf = leader_full0 + 8u * stage;
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2u * (1 + NW) * abytes);
                        uint8_t *dst = smem + (size_t)stage * P.stage_bytes;
                        const int rowA = (int)(((ta * n + q) * P.KB + kb0) * (kCrtBlk / 256));
                        tma_load_2d_pair(dst, &P.tmA, 0, rowA, lf);
#pragma unroll
                        for (int j = 0; j < NW; ++j) {
                            const int rowB = (int)((((tb + 2 * j) * n + q) * P.KB + kb0) * (kCrtBlk / 256));
                            tma_load_2d_pair(dst + (1 + j) * abytes, &P.tmB, 0, rowB, lf);
                        }
                        if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (rank == 0) {
            constexpr uint32_t idesc = idesc_i8(256, 256);
            const uint64_t dsc = smem_desc_kmajor_noswz(0, 128, 256);
            uint32_t stage = 0, phase = 0, spar = 0x3u;   // bit j: parity to wait for on slot j
            uint32_t g = 0;                               // global modulus-pass counter
            for (int64_t tile = blockIdx.x >> 1; tile < total; tile += gridDim.x >> 1) {
                for (int q = 0; q < n; ++q, ++g) {
                    const uint32_t slot = (NSLOT == 2) ? (g & 1u) : 0u;
                    mbar_wait(&slot_empty[slot], (spar >> slot) & 1u);
                    spar ^= 1u << slot;
                    tc_fence_after();
                    const uint32_t d = tbase + slot * 256u;
                    for (int64_t kb0 = 0; kb0 < P.KB; kb0 += P.kpp) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t sb = smem_u32(smem + (size_t)stage * P.stage_bytes);
                        for (int kk = 0; kk < P.kpp; ++kk) {
                            const uint64_t ad = dsc + ((sb + (uint32_t)kk * kCrtBlk) >> 4);
#pragma unroll
                            for (int j = 0; j < NW; ++j) {
                                const uint64_t bd = dsc + ((sb + (uint32_t)((1 + j) * P.kpp + kk) * kCrtBlk) >> 4);
                                mma_i8_pair_elect(d + 256u * j, ad, bd, idesc, (kb0 + kk > 0) ? 1u : 0u);
                            }
                        }
                        mma_commit_pair_elect(&empty[stage]);
                        if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
                    }
                    mma_commit_pair_elect(&slot_full[slot]);
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (16 warps per CTA)
        const int ew = warp - 2;
        const int qd = warp & 3;            // TMEM lane quarter this warp may access
        const int ch = ew >> 2;             // column quarter [64 NW ch, 64 NW (ch + 1))
        const uint32_t tl = tbase + ((uint32_t)(qd * 32) << 16) + (uint32_t)(64 * NW * ch);
        const uint32_t slot_remote0 = mapa_shared(smem_u32(&slot_empty[0]), 0);
        uint32_t fpar = 0;                  // bit j: parity of the next completion of slot_full[j]
        uint32_t g = 0;
        for (int64_t tile = blockIdx.x >> 1; tile < total; tile += gridDim.x >> 1) {
            const int64_t b = tile / per_b, r = tile - b * per_b;
            const int64_t tm = r / P.tiles_n, tn = r - tm * P.tiles_n;
            const int64_t row = (2 * tm + rank) * 128 + qd * 32 + lane;
            int8_t *rb = P.R + b * P.batch_bytes + row * 16 + (tn * 16 * NW + 4 * NW * ch) * P.rows_pad * 16;
            for (int q = 0; q < n; ++q, ++g) {
                const uint32_t slot = (NSLOT == 2) ? (g & 1u) : 0u;
                mbar_wait(&slot_full[slot], (fpar >> slot) & 1u);
                fpar ^= 1u << slot;
                tc_fence_after();
                int8_t *dst = rb + (int64_t)q * P.plane_bytes;
#pragma unroll
                for (int gp = 0; gp < 2 * NW; ++gp) {   // two 16-column groups in flight per TMEM wait
                    uint32_t v[2][16];
                    tmem_ld_32x32b_x16(tl + slot * 256u + (uint32_t)(32 * gp), v[0]);
                    tmem_ld_32x32b_x16(tl + slot * 256u + (uint32_t)(32 * gp + 16), v[1]);
                    tmem_wait_ld();
                    if (gp == 2 * NW - 1) {   // all loads of this slot done: hand it back
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(slot_remote0 + 8u * slot);
                    }
#pragma unroll
                    for (int hg = 0; hg < 2; ++hg) {
                        const int gg = 2 * gp + hg;
                        uint32_t w[4];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            w[x] = residue_of_i32((int32_t)v[hg][4 * x], P.crt, q) |
                                   (residue_of_i32((int32_t)v[hg][4 * x + 1], P.crt, q) << 8) |
                                   (residue_of_i32((int32_t)v[hg][4 * x + 2], P.crt, q) << 16) |
                                   (residue_of_i32((int32_t)v[hg][4 * x + 3], P.crt, q) << 24);
                        }
                        *reinterpret_cast<uint4 *>(dst + (int64_t)gg * P.rows_pad * 16) =
                            make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
            }
        }
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tbase, 512);
    }
}

}  // namespace ozk
