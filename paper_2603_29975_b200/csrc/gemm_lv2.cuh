// gemm_lv2.cuh -- K2 + K3 on CTA pairs (tcgen05 cta_group::2), the production
// slice GEMM for s <= 12.
//
// Same method and pass structure as gemm_lv.cuh (§2.2; readings
// R1, R6, R7; passes of <= 4 levels in 4 TMEM slots).  The difference is the
// MMA shape: a cluster of two CTAs on one TPC issues M=256 x N=128 x K=32
// kind::i8 MMAs (leader CTA issues).  Each CTA stages only its own 128 rows of
// A and HALF (64 columns) of B, so the shared-memory operand traffic per SM
// drops from 8 KB to 6 KB per 64-clk MMA -- the 1-CTA kernel was bound by the
// SMEM port (MMA operand reads + incoming copies).
//
// Synchronisation (all barriers at identical offsets in both CTAs):
//   full[stage]   leader only: both CTAs' TMA loads (cta_group::2) credit it
//   empty[stage]  both: the leader's MMA commit multicasts to the pair
//   pass_full     both: multicast commit when a level pass is complete
//   slot_empty[j] leader only: 16 arrivals (8 epilogue warps x 2 CTAs)
#pragma once
#include <cstdint>

#include "gemm_lv.cuh"

namespace ozk {

constexpr int kMaxPassMaps = 4;

// R6 step of a level after the integer prefix: acc = fma(S_L, 2^w, acc).  (Measured: removing
// these FP64 instructions entirely, or converting with I2F instead of the DADD magic, does not
// change the C3 / C2x30 GEMM time -- the FP64 combine does not steal tensor cycles.)
#define OZK_LEVEL_FMA(v, sc, a) __fma_rn(i32_to_f64(v), (sc), (a))
constexpr int kEpi2 = 16;                       // epilogue warps per CTA (4 per TMEM lane quarter)
constexpr int kThreads2 = 64 + 32 * kEpi2;      // 576
constexpr int kNC2 = kLvBN / (kEpi2 / 4);       // 32 columns per epilogue thread

struct Lv2Params {
    LvParams lv;                          // operands / epilogue / pass plan
    CUtensorMap tmA[kMaxPassMaps];        // A slices as [rows of 256 B], box = 16 n rows
    CUtensorMap tmB[kMaxPassMaps];        // B slices (64-row tiles), box = 8 n rows
};

// Debug timeline (ozaki_debug_timing): globaltimer at fixed events of CTA 0.
enum TlEvent : int { TL_ENTRY = 0, TL_PROLOGUE, TL_DEPWAIT, TL_TMA0, TL_FULL0, TL_MMA_PASS0, TL_MMA_END,
                     TL_EPI_PASS0, TL_EPI_LAST, TL_EPI_STORE, TL_EXIT, TL_EPI_DRAINED, TL_EPI_F, TL_MMA_SLOT1, TL_EPI_REL0,
                     TL_MMA_FULL1, TL_ENTRY_MAX, TL_EXIT_MAX, TL_MMA_END_MAX };
// The timeline is compiled only into a -DOZK_TIMELINE build (tools/gemm_timeline.py builds one):
// even predicated-off checks in the MMA issuer's loop cost ~9 % of the C3 s=4 GEMM.
#ifdef OZK_TIMELINE
#define OZK_TL(...) __VA_ARGS__
#else
#define OZK_TL(...)
#endif
// latest event over all CTAs (atomicMax of globaltimer)
__device__ __forceinline__ void tl_max(const GemmParams &p, int ev) {
    if (p.dbg) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(p.dbg + DBG_TL0 + ev, t);
    }
}
__device__ __forceinline__ void tl_mark(const GemmParams &p, int ev) {
    if (p.dbg && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.dbg[DBG_TL0 + ev] = t;
    }
}

// Work unit u of the persistent loop: tile u / splitk, k-blocks of split u % splitk (an equal
// share of [kb_begin, kb_end); splitk == 1 is the whole range).
template <bool SPLIT>
__device__ __forceinline__ void lv2_unit(const GemmParams &p, int64_t u, int64_t &tile, int64_t &kb0,
                                         int64_t &kb1, int &q) {
    if constexpr (!SPLIT) {   // unsplit kernels: the original per-tile loop (uniform K bounds)
        tile = u;
        q = 0;
        kb0 = p.kb_begin;
        kb1 = p.kb_end;
        return;
    }
    const uint32_t sk = (uint32_t)p.splitk, uu = (uint32_t)u;   // < 2^31 (make_plan)
    tile = uu / sk;
    q = (int)(uu - (uint32_t)tile * sk);
    if (sk == 1) {
        kb0 = p.kb_begin;
        kb1 = p.kb_end;
        return;
    }
    const uint32_t span = (uint32_t)(p.kb_end - p.kb_begin);   // split-K runs unchunked: span = KB
    kb0 = p.kb_begin + (uint32_t)(((uint64_t)span * (uint32_t)q) / sk);
    kb1 = p.kb_begin + (uint32_t)(((uint64_t)span * (uint32_t)(q + 1)) / sk);
}

template <int S, bool FULL = false, bool SPLIT = false>
__device__ __forceinline__ void lv2_mma_role(const Lv2Params &P2, uint8_t *smem, uint64_t *full,
                                             uint64_t *empty, uint64_t *pass_full,
                                             uint64_t *slot_empty, uint32_t tbase) {
    constexpr PassPlan PP = FULL ? make_pass_plan_full(S) : make_pass_plan(S);
    constexpr uint32_t idesc = idesc_i8(256, kLvBN);
    const LvParams &lp = P2.lv;
    const GemmParams &p = lp.g;
    const int64_t total = p.batch * p.tiles_m * p.tiles_n * (SPLIT ? p.splitk : 1);   // units of 256 x 128 super-tiles
    const int Sg = p.stages;
    uint32_t stage = 0, phase = 0;
    uint32_t slot_par = (1u << kSlots) - 1u;    // bit j: parity to wait for on slot j
    const long long t_begin = p.dbg ? clock64() : 0;
    const uint64_t dA = smem_desc_kmajor_noswz(0, 128, 256);   // 128-row A operand per CTA
    const uint64_t dB = smem_desc_kmajor_noswz(0, 128, 256);   // 64-row B half per CTA
    for (int64_t u = blockIdx.x >> 1; u < total; u += gridDim.x >> 1) {
        int64_t tile, ub, ue;
        int q;
        lv2_unit<SPLIT>(p, u, tile, ub, ue, q);
#pragma unroll
        for (int ps = 0; ps < PP.npass; ++ps) {
            const int hi = PP.hi[ps], lo = PP.lo[ps], tlo = PP.tlo[ps], n = PP.n[ps];
            const uint32_t abytes = (uint32_t)n * kBlk, bbytes = (uint32_t)n * (kBlk / 2);
            const int kpp = lp.pass[ps].kpp;
            for (int64_t kb0 = ub; kb0 < ue; kb0 += kpp) {
                const int nk = (int)min((int64_t)kpp, ue - kb0);
                const bool kfirst = (kb0 == ub);
                long long w0 = p.dbg ? clock64() : 0;
                mbar_wait(&full[stage], phase);
                OZK_TL(if (kfirst && ps == 0 && u == (blockIdx.x >> 1)) tl_mark(p, TL_FULL0);)
                OZK_TL(if (kfirst && ps == 1 && u == (blockIdx.x >> 1)) tl_mark(p, TL_MMA_FULL1);)
                if (p.dbg && (threadIdx.x & 31) == 0) {
                    const long long dw = clock64() - w0;
                    dbg_add(p, DBG_MMA_WAIT_FULL, dw);
                    if (kfirst) dbg_add(p, DBG_MMA_WAIT_FULL0, dw);
                    if (ps == 0) dbg_add(p, DBG_MMA_WAIT_FULLP0, dw);
                }
                tc_fence_after();
                const uint32_t sbase = smem_u32(smem + (size_t)stage * lp.stage_bytes);
                for (int kk = 0; kk < nk; ++kk) {
                    const uint32_t abase = sbase + (uint32_t)kk * (abytes + bbytes);
                    const uint64_t ad0 = dA + (abase >> 4);
                    const uint64_t bd0 = dB + ((abase + abytes) >> 4);
                    if (kfirst && kk == 0) {
#pragma unroll
                        for (int j = 0; j < hi - lo + 1; ++j) {
                            w0 = p.dbg ? clock64() : 0;
                            mbar_wait(&slot_empty[j], (slot_par >> j) & 1u);
                            slot_par ^= 1u << j;
                            if (p.dbg && (threadIdx.x & 31) == 0) {
                                const long long dw = clock64() - w0;
                                dbg_add(p, DBG_MMA_WAIT_SLOT, dw);
                                if (ps == 0) dbg_add(p, DBG_MMA_WAIT_SLOT0, dw);
                            }
                        }
                        tc_fence_after();
                        OZK_TL(if (ps == 1 && u == (blockIdx.x >> 1)) tl_mark(p, TL_MMA_SLOT1);)
                    }
#pragma unroll
                    for (int r = 0; r < S; ++r) {
#pragma unroll
                        for (int j = 0; j < hi - lo + 1; ++j) {
                            const int L = hi - j;
                            const int t0 = pp_max(1, L - S), t1 = pp_min(S, L - 1);
                            const int t = t0 + r;
                            if (t <= t1) {
                                const int u = L - t;
                                const uint32_t acc = (r == 0) ? (uint32_t)(!kfirst || kk != 0) : 1u;
                                mma_i8_pair_elect(tbase + (uint32_t)(j * kLvBN),
                                                  ad0 + (uint64_t)(((t - tlo) * kBlk) >> 4),
                                                  bd0 + (uint64_t)(((u - tlo) * (kBlk / 2)) >> 4), idesc, acc);
                            }
                        }
                    }
                }
                mma_commit_pair_elect(&empty[stage]);
                if (++stage == (uint32_t)Sg) { stage = 0; phase ^= 1; }
            }
            mma_commit_pair_elect(pass_full);
            OZK_TL(if (ps == 0 && u == (blockIdx.x >> 1)) tl_mark(p, TL_MMA_PASS0);)
        }
    }
    OZK_TL(tl_mark(p, TL_MMA_END); tl_max(p, TL_MMA_END_MAX);)
    if (p.dbg && (threadIdx.x & 31) == 0) dbg_add(p, DBG_MMA_TOTAL, clock64() - t_begin);
}

// CHUNK (compile time, reading R8): 0 = whole K in one INT32 accumulation;
// 1 = first/middle K chunk (W = S or W += S, nothing stored to C);
// 2 = last K chunk (level sum = W + S, then the FP64 combine and store);
// 3 = split-K unit (exact partials to P0 / PL, k_splitk_combine finishes).
// FULL (reading R21, NEXT-4): all s^2 pairs, levels 2s .. 2 (s <= 8, CHUNK 0 only).
template <int EPI, int CHUNK, bool FULL = false, bool GAB = true>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    k_gemm_lv2(const __grid_constant__ Lv2Params P2) {
    const LvParams &lp = P2.lv;
    const GemmParams &p = lp.g;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * lp.stage_bytes);
    uint64_t *empty = full + S;
    uint64_t *pass_full = empty + S;
    uint64_t *slot_empty = pass_full + 1;
    uint32_t *tholder = reinterpret_cast<uint32_t *>(slot_empty + kSlots);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int s = p.s;
    const int Lmax = FULL ? 2 * s : s + 1;   // levels Lmax (least significant) .. 2 (R1 / R21)
    constexpr bool SPLIT = (CHUNK == 3);   // split-K units (compile time: the other kernels keep the tile loop)
    const int64_t total = p.batch * p.tiles_m * p.tiles_n * (SPLIT ? p.splitk : 1);   // work units
    if (threadIdx.x == 0) {
        OZK_TL(tl_mark(p, TL_ENTRY); tl_max(p, TL_ENTRY_MAX);)
    }

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(pass_full, 1);
        for (int j = 0; j < kSlots; ++j) mbar_init(&slot_empty[j], 2 * kEpi2);
        fence_mbar_init();
        for (int q = 0; q < lp.npass; ++q) {
            tma_prefetch_desc(&P2.tmA[q]);
            tma_prefetch_desc(&P2.tmB[q]);
        }
    }
    if (warp == 1) tmem_alloc_pair(tholder, 512);
    tc_fence_before();
    cluster_sync();          // barriers of both CTAs initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tbase = *tholder;
    OZK_TL(if (threadIdx.x == 0) tl_mark(p, TL_PROLOGUE);)
    // Programmatic dependent launch: the prologue above overlaps the producer kernel's tail
    // (K1); everything below reads its output (slices, exponents), so wait for its completion.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    OZK_TL(if (threadIdx.x == 0) tl_mark(p, TL_DEPWAIT);)
    // ... and let a dependent launched with PDL (the next call's split, ozaki_set_overlap) start
    // on the SMs this grid's last wave leaves idle; it orders itself after this grid (split_fast.cuh)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ========================= producer (both CTAs): own A rows, own B half
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for (int64_t u = blockIdx.x >> 1; u < total; u += gridDim.x >> 1) {
                int64_t tile, ub, ue, b, tm, tn;
                int q;
                lv2_unit<SPLIT>(p, u, tile, ub, ue, q);
                decode_tile(p, tile, b, tm, tn);
                // A tiles of 128 rows: this CTA's is 2*tm + rank;  B tiles of 64 rows: 2*tn + rank
                const int64_t arow0 = ((b * (2 * p.tiles_m) + 2 * tm + rank) * p.KB) * (int64_t)s * (kBlk / 256);
                const int64_t brow0 = ((b * (2 * p.tiles_n) + 2 * tn + rank) * p.KB) * (int64_t)s * (kBlk / 512);
                for (int ps = 0; ps < lp.npass; ++ps) {
                    const LvPass pa = lp.pass[ps];
                    const uint32_t abytes = (uint32_t)pa.n * kBlk, bbytes = (uint32_t)pa.n * (kBlk / 2);
                    for (int64_t kb0 = ub; kb0 < ue; kb0 += pa.kpp) {
                        const int nk = (int)min((int64_t)pa.kpp, ue - kb0);
                        const long long w0 = p.dbg ? clock64() : 0;
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (p.dbg) dbg_add(p, DBG_PROD_WAIT, clock64() - w0);
                        const uint32_t leader_full = mapa_shared(smem_u32(&full[stage]), 0);
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2u * (abytes + bbytes) * nk);
                        uint8_t *dst = smem + (size_t)stage * lp.stage_bytes;
                        for (int kk = 0; kk < nk; ++kk) {
                            const int64_t kb = kb0 + kk;
                            const int ra = (int)(arow0 + (kb * s + pa.tlo - 1) * (kBlk / 256));
                            const int rb = (int)(brow0 + (kb * s + pa.tlo - 1) * (kBlk / 512));
                            tma_load_2d_pair(dst, &P2.tmA[ps], 0, ra, leader_full);
                            tma_load_2d_pair(dst + abytes, &P2.tmB[ps], 0, rb, leader_full);
                            dst += abytes + bbytes;
                        }
                        OZK_TL(if (u == (blockIdx.x >> 1) && ps == 0 && kb0 == ub) tl_mark(p, TL_TMA0);)
                        if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ========================= MMA issuer: leader CTA only
        if (rank == 0) {
            if constexpr (FULL) {
                switch (s) {
#define OZK_MMA2_CASE(SS) case SS: lv2_mma_role<SS, true, SPLIT>(P2, smem, full, empty, pass_full, slot_empty, tbase); break;
                    OZK_MMA2_CASE(1) OZK_MMA2_CASE(2) OZK_MMA2_CASE(3) OZK_MMA2_CASE(4)
                    OZK_MMA2_CASE(5) OZK_MMA2_CASE(6) OZK_MMA2_CASE(7) OZK_MMA2_CASE(8)
#undef OZK_MMA2_CASE
                    default: break;
                }
            } else {
                switch (s) {
#define OZK_MMA2_CASE(SS) case SS: lv2_mma_role<SS, false, SPLIT>(P2, smem, full, empty, pass_full, slot_empty, tbase); break;
                    OZK_MMA2_CASE(1) OZK_MMA2_CASE(2) OZK_MMA2_CASE(3) OZK_MMA2_CASE(4)
                    OZK_MMA2_CASE(5) OZK_MMA2_CASE(6) OZK_MMA2_CASE(7) OZK_MMA2_CASE(8)
                    OZK_MMA2_CASE(9) OZK_MMA2_CASE(10) OZK_MMA2_CASE(11) OZK_MMA2_CASE(12)
#undef OZK_MMA2_CASE
                    default: break;
                }
            }
        }
    } else {
        // ========================= epilogue (8 warps per CTA, own 128 rows)
        const int ew = warp - 2;
        const int q = warp & 3;
        const int half = ew >> 2;                    // column group: [half * kNC2, +kNC2)
        const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * kNC2);
        uint32_t pphase = 0;
        const bool dbgw = p.dbg && warp == 2 && lane == 0;
        // slot_empty barriers are consecutive 8-byte words: remote address = base + 8 j
        const uint32_t slot_remote0 = mapa_shared(smem_u32(&slot_empty[0]), 0);
        for (int64_t u = blockIdx.x >> 1; u < total; u += gridDim.x >> 1) {
            int64_t tile, ub, ue, b, tm, tn;
            int sq;
            lv2_unit<SPLIT>(p, u, tile, ub, ue, sq);
            decode_tile(p, tile, b, tm, tn);
            const int64_t grow = (2 * tm + rank) * kBM + q * 32 + lane;
            const int32_t e = (grow < p.Mp) ? __ldg(p.ea + b * p.Mp + grow) : 0;
            double acc[kNC2];
#pragma unroll
            for (int j = 0; j < kNC2; ++j) acc[j] = 0.0;
            for (int ps = 0; ps < lp.npass; ++ps) {
                const LvPass pa = lp.pass[ps];
                long long w0 = p.dbg ? clock64() : 0;
                mbar_wait(pass_full, pphase);
                OZK_TL(if (dbgw && u == (blockIdx.x >> 1)) tl_mark(p, ps == 0 ? TL_EPI_PASS0 : TL_EPI_LAST);)
                long long w1 = p.dbg ? clock64() : 0;
                if (dbgw) dbg_add(p, DBG_EPI_WAIT, w1 - w0);
                pphase ^= 1;
                tc_fence_after();
                if constexpr (CHUNK == 3) {
                    // split-K unit: exact partials of this unit's k-blocks, no FP64.  Pass 0 -> the
                    // int64 prefix X = sum_j S_j 2^(8j) of its levels (the exact part of R6, < 2^55
                    // per unit; the units' X add exactly in int64); later levels -> int32 sums.
                    const int nlev = pa.hi - pa.lo + 1;
                    const int np0 = lp.pass[0].hi - lp.pass[0].lo + 1;
                    const int64_t c0 = tn * kLvBN + half * kNC2;
                    const bool rok = grow < p.Mp;
                    const int64_t plane = p.batch * p.N * p.Mp;
                    const int64_t off = (b * p.N + c0) * p.Mp + grow;
                    uint32_t v[16];
                    if (ps == 0) {
                        long long t0[16], t1[16];
                        tmem_ld_32x32b_x16(tl, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) t0[i] = (long long)(int)v[i];
#pragma unroll 1
                        for (int j = 1; j < nlev; ++j) {
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN), v);
                            tmem_wait_ld();
                            const int w = 1 << (8 * j);
#pragma unroll
                            for (int i = 0; i < 16; ++i) t0[i] += (long long)(int)v[i] * w;
                        }
                        tmem_ld_32x32b_x16(tl + 16u, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) t1[i] = (long long)(int)v[i];
#pragma unroll 1
                        for (int j = 1; j < nlev; ++j) {
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + 16), v);
                            tmem_wait_ld();
                            const int w = 1 << (8 * j);
#pragma unroll
                            for (int i = 0; i < 16; ++i) t1[i] += (long long)(int)v[i] * w;
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0)
                            for (int j = 0; j < nlev; ++j) mbar_arrive_cluster(slot_remote0 + 8u * (uint32_t)j);
                        if (rok) {
                            long long *dst = reinterpret_cast<long long *>(p.P0) + (int64_t)sq * plane + off;
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (c0 + i < p.N) dst[(int64_t)i * p.Mp] = t0[i];
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (c0 + 16 + i < p.N) dst[(int64_t)(16 + i) * p.Mp] = t1[i];
                        }
                    } else {
#pragma unroll 1
                        for (int j = 0; j < nlev; ++j) {
                            const int li = (Lmax - np0) - (pa.hi - j);
                            int32_t *dst = p.PL + ((int64_t)sq * p.pk_nl + li) * plane + off;
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN), v);
                            tmem_wait_ld();
                            if (rok) {
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    if (c0 + i < p.N) dst[(int64_t)i * p.Mp] = (int32_t)v[i];
                            }
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + 16), v);
                            tmem_wait_ld();
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(slot_remote0 + 8u * (uint32_t)j);
                            if (rok) {
#pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    if (c0 + 16 + i < p.N) dst[(int64_t)(16 + i) * p.Mp] = (int32_t)v[i];
                            }
                        }
                    }
                } else if constexpr (CHUNK == 0 && EPI != EPI_LEVELS) {
                    // one software pipeline over the pass: chunk c = (level c/2, 16-column
                    // group c%2), the load of chunk c+1 in flight while chunk c is combined;
                    // a level's TMEM slot is released as soon as both its groups are in
                    // registers (before its FP64 work).  Levels in ascending significance (R6).
                    static_assert(kNC2 == 32, "two 16-column groups per level");
                    // acc is carried scaled by 2^(8(s-1)) (exact: power-of-two scaling of
                    // normal values leaves every RNE step unchanged); level L weighs 2^(8(s+1-L)).
                    const int nlev = pa.hi - pa.lo + 1;
                    uint32_t v[16];
                    int j0 = 0;
                    if (ps == 0) {
                        // Integer prefix: the first np <= 4 levels (L = s+1 .. s-2).  With
                        // |S_L| < 2^31, X = sum_j S_j 2^(8j) (< 2^55.01) is exact in int64; R6's
                        // steps over the first three are exact (< 2^53), so R6 rounds once, at the
                        // fourth: acc = RNE53(X) = one I2F.F64.S64 (round-to-nearest-even).  No
                        // FP64-pipe instruction: FP64 is starved while the tensor core streams the
                        // next pass (tools/fp64_vs_mma.cu), I2F and IMAD are not.
                        const int np = nlev < 4 ? nlev : 4;
                        long long t0[16], t1[16];
                        // columns 0..15 of every prefix level, then 16..31 (each slot released
                        // right after its second load); conversions only after the last release
                        tmem_ld_32x32b_x16(tl, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) t0[i] = (long long)(int)v[i];
#pragma unroll 1
                        for (int j = 1; j < np; ++j) {
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN), v);
                            tmem_wait_ld();
                            const int w = 1 << (8 * j);
#pragma unroll
                            for (int i = 0; i < 16; ++i) t0[i] += (long long)(int)v[i] * w;
                        }
                        tmem_ld_32x32b_x16(tl + 16u, v);
                        tmem_wait_ld();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(slot_remote0);
                        OZK_TL(if (dbgw && u == (blockIdx.x >> 1)) tl_mark(p, TL_EPI_REL0);)
                        if (dbgw) dbg_add(p, DBG_EPI_FIRST_ARRIVE, clock64() - w1);
#pragma unroll
                        for (int i = 0; i < 16; ++i) t1[i] = (long long)(int)v[i];
#pragma unroll 1
                        for (int j = 1; j < np; ++j) {
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + 16), v);
                            tmem_wait_ld();
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(slot_remote0 + 8u * (uint32_t)j);
                            const int w = 1 << (8 * j);
#pragma unroll
                            for (int i = 0; i < 16; ++i) t1[i] += (long long)(int)v[i] * w;
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            acc[i] = __ll2double_rn(t0[i]);
                            acc[16 + i] = __ll2double_rn(t1[i]);
                        }
                        j0 = np;
                        if (dbgw) dbg_add(p, DBG_EPI_PREFIX, clock64() - w1);
                    }
#pragma unroll 1
                    for (int j = j0; j < nlev; ++j) {
                        const double sc = pow2(8 * (Lmax - (pa.hi - j)));
                        tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN), v);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[i] = OZK_LEVEL_FMA(v[i], sc, acc[i]);
                        tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + 16), v);
                        tmem_wait_ld();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(slot_remote0 + 8u * (uint32_t)j);
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[16 + i] = OZK_LEVEL_FMA(v[i], sc, acc[16 + i]);
                    }
                } else {
                for (int L = pa.hi; L >= pa.lo; --L) {          // ascending significance (R6)
                    const int j = pa.hi - L;
                    const double sc = pow2(-8 * (L - 2));
#pragma unroll
                        for (int g = 0; g < kNC2 / 32; ++g) {
                            uint32_t v0[16], v1[16];
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + g * 32), v0);
                            tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + g * 32 + 16), v1);
                            tmem_wait_ld();
                            if constexpr (EPI == EPI_LEVELS) {
                                if (b == 0 && grow < p.Mp) {
    #pragma unroll
                                    for (int i = 0; i < 32; ++i) {
                                        const int64_t gcol = tn * kLvBN + half * kNC2 + g * 32 + i;
                                        if (gcol < p.N)
                                            p.S_out[(int64_t)(L - 2) * p.Mp * p.N + gcol * p.Mp + grow] =
                                                (int32_t)(i < 16 ? v0[i] : v1[i - 16]);
                                    }
                                }
                                continue;
                            }
                            if constexpr (CHUNK == 1) {
                                // first/middle K chunk (R8): exact partial level sums W (+)= S
                                const int64_t c0 = tn * kLvBN + half * kNC2 + g * 32;
                                if (grow < p.Mp) {
                                    double *wp = p.W + (int64_t)(L - 2) * p.w_lvl + c0 * p.Mp + grow;
    #pragma unroll 4
                                    for (int i = 0; i < 32; ++i) {
                                        if (c0 + i >= p.N) break;
                                        const double part = i32_to_f64(i < 16 ? v0[i] : v1[i - 16]);
                                        double *q = wp + (int64_t)i * p.Mp;
                                        *q = (p.chunk_mode == 1) ? part : __dadd_rn(*q, part);
                                    }
                                }
                            } else if constexpr (CHUNK == 2) {
                                // last K chunk: level sum = W + S (exact), then the FP64 combine
                                const int64_t c0 = tn * kLvBN + half * kNC2 + g * 32;
                                const bool rok = grow < p.Mp;
                                const double *wp = p.W + (int64_t)(L - 2) * p.w_lvl + c0 * p.Mp + grow;
    #pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    double lvl = i32_to_f64(i < 16 ? v0[i] : v1[i - 16]);
                                    if (rok && c0 + i < p.N) lvl = __dadd_rn(wp[(int64_t)i * p.Mp], lvl);
                                    acc[g * 32 + i] = __fma_rn(lvl, sc, acc[g * 32 + i]);
                                }
                            }
                        }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(slot_remote0 + 8u * (uint32_t)j);
                }
                }
                if (dbgw) dbg_add(p, DBG_EPI_DRAIN, clock64() - w1);
            }
            const long long s0 = p.dbg ? clock64() : 0;
#ifdef OZK_TIMELINE
            if (dbgw) {
                tl_mark(p, TL_EPI_DRAINED);
                // probe: latency of one column-exponent load and one load of C (debug timeline only)
                const int32_t f = __ldg(p.fb + b * p.N + tn * kLvBN);
                const double cv = *(volatile double *)(p.C + b * p.strideC);
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (blockIdx.x == 0) p.dbg[DBG_TL0 + TL_EPI_F] = t + (f == -123456789 ? 1 : 0) + (cv == 1.2345e300 ? 1 : 0);
            }
#endif
            if constexpr (EPI != EPI_LEVELS && CHUNK != 1 && CHUNK != 3)
                lv_store<EPI, kNC2, GAB>(p, b, grow, e, tn * kLvBN + half * kNC2, acc, CHUNK == 0 ? -8 * (Lmax - 2) : 0);
            if (dbgw) dbg_add(p, DBG_EPI_STORE, clock64() - s0);
            OZK_TL(if (dbgw) tl_mark(p, TL_EPI_STORE);)
        }
    }

    tc_fence_before();
    cluster_sync();          // all MMAs done and all TMEM reads of both CTAs finished
    if (threadIdx.x == 0) {
        OZK_TL(tl_mark(p, TL_EXIT); tl_max(p, TL_EXIT_MAX);)
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tbase, 512);
    }
}

// Split-K combine (CHUNK == 3 units wrote the partials): one thread per (row, NC = 2 product
// columns: one complex element for 4M), warps over 32 consecutive rows (coalesced partial
// reads), enough threads to keep the reads in flight.  The level sums are the integer sums of
// the units' partials (order-free); acc = RNE53(X) then R6's FMAs in the pass order, exactly as
// the unsplit epilogue, and the same store (lv_store).
template <int EPI>
__global__ void __launch_bounds__(128) k_splitk_combine(const __grid_constant__ GemmParams p, int Lmax, int np0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int NC = 2;
    const int64_t b = blockIdx.z;
    const int64_t grow = (int64_t)blockIdx.y * 128 + threadIdx.x;
    const int64_t col0 = (int64_t)blockIdx.x * NC;
    const bool rok = grow < p.Mp;
    const int32_t e = rok ? __ldg(p.ea + b * p.Mp + grow) : 0;
    const int64_t plane = p.batch * p.N * p.Mp;
    const int64_t off = (b * p.N + col0) * p.Mp + grow;
    const int sk = p.splitk, nl = p.pk_nl;
    const bool ok0 = rok && col0 < p.N, ok1 = rok && col0 + 1 < p.N;
    long long X0 = 0, X1 = 0;
    {
        const long long *x = reinterpret_cast<const long long *>(p.P0) + off;
#pragma unroll 4
        for (int q = 0; q < sk; ++q) {
            if (ok0) X0 += __ldg(x + (int64_t)q * plane);
            if (ok1) X1 += __ldg(x + (int64_t)q * plane + p.Mp);
        }
    }
    double acc[NC] = {__ll2double_rn(X0), __ll2double_rn(X1)};
    for (int li = 0; li < nl; ++li) {
        const double sc = pow2(8 * (np0 + li));   // level L = Lmax - np0 - li weighs 2^(8(Lmax-L))
        const int32_t *y = p.PL + (int64_t)li * plane + off;
        uint32_t S0 = 0, S1 = 0;
#pragma unroll 4
        for (int q = 0; q < sk; ++q) {
            if (ok0) S0 += (uint32_t)__ldg(y + (int64_t)q * nl * plane);
            if (ok1) S1 += (uint32_t)__ldg(y + (int64_t)q * nl * plane + p.Mp);
        }
        acc[0] = __fma_rn(i32_to_f64(S0), sc, acc[0]);
        acc[1] = __fma_rn(i32_to_f64(S1), sc, acc[1]);
    }
    lv_store<EPI, NC>(p, b, grow, e, col0, acc, -8 * (Lmax - 2));
}

}  // namespace ozk
