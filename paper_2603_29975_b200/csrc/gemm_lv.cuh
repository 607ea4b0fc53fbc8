// gemm_lv.cuh -- K2 + K3, level-pass design (the production kernel for s <= 12).
//
// Same method as gemm.cuh (§2.2; readings R1, R6, R7):
//   S_L = sum_{t+u=L} A_t B_u^T (exact INT32) for L = s+1 .. 2,
//   acc = sum_{L=s+1..2} S_L 2^(-8(L-2)) in FP64 (ascending), P = acc 2^(e+f-14),
//   C = alpha P + beta C.
//
// Why this shape (measured on B200, tools/mma_microbench*.cu):
//   * an M=128 kind::i8 MMA costs >= ~64 clk whatever N is, so only N >= 128
//     reaches the tensor peak (128x128x32 in 64 clk = 8192 MAC/clk/SM);
//   * TMEM holds 512 columns = 4 accumulators of 128x128 INT32, so at most 4
//     levels can be resident: the levels are processed in PASSES of <= 4
//     (descending L, the order the FP64 combine consumes them).  Each pass
//     sweeps K once, loading only the slices its pairs need; the FP64 running
//     sum lives in the epilogue warps' registers across passes;
//   * per-slot barriers let the epilogue drain pass p's levels while the MMA
//     warp already issues pass p+1 into the slots drained first.
//
// Roles: warp 0 bulk-copy producer, warp 1 TMEM owner + MMA issuer (one
// thread), warps 2..9 epilogue (two per TMEM lane quarter, 64 columns each).
#pragma once
// EPI_LEVELS (debug) instantiations `continue` before the FP64 epilogue of the same loop body
#pragma nv_diag_suppress 128
#include <cstdint>

#include "gemm.cuh"
#include "numerics.cuh"
#include "passplan.cuh"
#include "ptx.cuh"

namespace ozk {

constexpr int kLvBN = 128;
constexpr int kMaxPass = 4;
constexpr int kSlots = 4;
constexpr uint32_t kBlk = 128 * kKB;   // bytes of one (slice, k-block) operand block

struct LvPass {
    int32_t hi, lo;      // levels L = hi down to lo (slot j holds L = hi - j)
    int32_t tlo, n;      // slices t (and u) in [tlo, tlo + n) are loaded
    int32_t kpp;         // k-blocks per pipeline stage in this pass
};

struct LvParams {
    GemmParams g;        // operands, exponents, epilogue (BN = 128 tiling)
    int32_t npass;
    uint32_t stage_bytes;
    LvPass pass[kMaxPass];
};

// Final epilogue of one thread: its row `grow`, 64 consecutive product
// columns col0 .. col0+63 held in acc[].  Complex (4M, R9 N-side embedding):
// columns 2c / 2c+1 are Re / Im of complex column col0/2 + c, so each thread
// owns whole complex numbers: one 16-byte store, no lane exchange.
// GAB: compile the beta != 0 (general alpha / beta) store; the production alpha = 1, beta = 0
// kernels instantiate GAB = false so that code does not weigh on their register allocation.
template <int EPI, int NC = 64, bool GAB = true>
__device__ __forceinline__ void lv_store(const GemmParams &p, int64_t b, int64_t grow, int32_t e,
                                         int64_t col0, const double *acc, int nbias = 0) {
    const int lane = threadIdx.x & 31;
    const int ncol = (grow < p.Mp) ? (int)min((int64_t)NC, p.N - col0) : 0;
    // column exponents: lane j holds f of columns col0 + j and col0 + 32 + j
    const int32_t f_lo = (col0 + lane < p.N) ? __ldg(p.fb + b * p.N + col0 + lane) : 0;
    const int32_t f_hi = (NC > 32 && col0 + 32 + lane < p.N) ? __ldg(p.fb + b * p.N + col0 + 32 + lane) : 0;
    const bool beta0 = (p.beta_r == 0.0 && p.beta_i == 0.0);
    const bool enan = (e == kNonFinite);
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    // P = ldexp(acc, e + f - 14) by an integer exponent-field add (scale_pow2: exact, no FP64
    // instruction on the normal path).  Scalar FP64 shares the SM's tensor datapath on B200 and
    // runs ~19x slower while the MMAs of the next tile stream (tools/fp64_vs_mma.cu), so the
    // store avoids FP64 entirely when alpha = 1, beta = 0: then R7's formula reduces bitwise to
    // C = P (real) and, complex, C_r = P_r + 0 (-0 -> +0; NaN if P_i is not finite, from
    // -0 * Inf), C_i likewise.
    if constexpr (EPI == EPI_REAL) {
        double *cp = p.C + b * p.strideC + grow + col0 * p.ldc;
        if (!GAB || p.ab_unit || beta0) {
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const int32_t f = __shfl_sync(0xffffffffu, j < 32 ? f_lo : f_hi, j & 31);
                const double P = (enan || f == kNonFinite) ? qnan : scale_pow2(acc[j], e + f - 14 + nbias);
                if (j < ncol) *cp = p.ab_unit ? P : __dmul_rn(p.alpha_r, P);
                cp += p.ldc;
            }
        } else if constexpr (GAB) {
            // beta != 0: the C values of a group of 8 columns are loaded together before the
            // group's FMAs (one memory latency per group instead of one per column).  Each C
            // element is read once, before this thread writes it, and no other thread touches
            // its cache lines (a warp owns whole 32-row column segments), so the read-only path
            // is safe.
#pragma unroll
            for (int j0 = 0; j0 < NC; j0 += 8) {
                double cv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    cv[i] = (j0 + i < NC && j0 + i < ncol) ? __ldg(cp + (int64_t)(j0 + i) * p.ldc) : 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int j = j0 + i;
                    if (j >= NC) break;
                    const int32_t f = __shfl_sync(0xffffffffu, j < 32 ? f_lo : f_hi, j & 31);
                    const double P = (enan || f == kNonFinite) ? qnan : scale_pow2(acc[j], e + f - 14 + nbias);
                    // beta == 1: beta * C == C exactly (also for -0, Inf, NaN): no DMUL
                    const double t = (p.beta_r == 1.0) ? cv[i] : __dmul_rn(p.beta_r, cv[i]);
                    if (j < ncol) cp[(int64_t)j * p.ldc] = __fma_rn(p.alpha_r, P, t);
                }
            }
        }
    } else {
        double2 *cp = reinterpret_cast<double2 *>(p.C) + b * p.strideC + grow + (col0 >> 1) * p.ldc;
        if (GAB && !p.ab_unit && !beta0) {
            // general alpha / beta: C loaded 4 complex columns at a time ahead of their FMAs
            // (read-only path: see the real case).  (An LU-update special case -- alpha = +-1,
            // beta = 1 as one DADD per component plus exact signed-zero selects -- measured
            // slower on C2 x 30: 0.53 vs 0.47-0.50 ms.)
            const double2 *cq = cp;
#pragma unroll
            for (int c0 = 0; c0 < NC / 2; c0 += 4) {
                double2 cv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    cv[i] = (c0 + i < NC / 2 && 2 * (c0 + i) < ncol) ? __ldg(cq + (int64_t)(c0 + i) * p.ldc)
                                                                      : make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = c0 + i;
                    if (c >= NC / 2) break;
                    const int32_t f = __shfl_sync(0xffffffffu, c < 16 ? f_lo : f_hi, (2 * c) & 31);
                    const int nsc = e + f - 14 + nbias;
                    const bool nan = enan || f == kNonFinite;
                    const double Pr = nan ? qnan : scale_pow2(acc[2 * c], nsc);
                    const double Pi = nan ? qnan : scale_pow2(acc[2 * c + 1], nsc);
                    const double tr = __fma_rn(p.beta_r, cv[i].x, -__dmul_rn(p.beta_i, cv[i].y));
                    const double ti = __fma_rn(p.beta_r, cv[i].y, __dmul_rn(p.beta_i, cv[i].x));
                    const double2 out = make_double2(__fma_rn(p.alpha_r, Pr, __fma_rn(-p.alpha_i, Pi, tr)),
                                                     __fma_rn(p.alpha_r, Pi, __fma_rn(p.alpha_i, Pr, ti)));
                    if (2 * c < ncol) cp[(int64_t)c * p.ldc] = out;
                }
            }
            return;
        }
#pragma unroll
        for (int c = 0; c < NC / 2; ++c) {
            const int32_t f = __shfl_sync(0xffffffffu, c < 16 ? f_lo : f_hi, (2 * c) & 31);
            const int nsc = e + f - 14 + nbias;
            const bool nan = enan || f == kNonFinite;
            const double Pr = nan ? qnan : scale_pow2(acc[2 * c], nsc);
            const double Pi = nan ? qnan : scale_pow2(acc[2 * c + 1], nsc);
            if (2 * c < ncol) {
                if (p.ab_unit) {
                    *cp = make_double2(plus_zero(Pr, Pi), plus_zero(Pi, Pr));
                } else {
                    double tr = 0.0, ti = 0.0;
                    if (!beta0) {
                        const double2 cv = *cp;
                        tr = __fma_rn(p.beta_r, cv.x, -__dmul_rn(p.beta_i, cv.y));
                        ti = __fma_rn(p.beta_r, cv.y, __dmul_rn(p.beta_i, cv.x));
                    }
                    *cp = make_double2(__fma_rn(p.alpha_r, Pr, __fma_rn(-p.alpha_i, Pi, tr)),
                                       __fma_rn(p.alpha_r, Pi, __fma_rn(p.alpha_i, Pr, ti)));
                }
            }
            cp += p.ldc;
        }
    }
}

// MMA issuer for a compile-time slice count S: the pass plan is constexpr, so
// every (level, pair) MMA of a k-block is an unrolled instruction whose
// descriptors are the stage base plus an immediate (the runtime
// loop version was issue-bound at ~180 clk per MMA).
template <int S>
__device__ __forceinline__ void lv_mma_role(const LvParams &lp, uint8_t *smem, uint64_t *full,
                                            uint64_t *empty, uint64_t *pass_full,
                                            uint64_t *slot_empty, uint32_t tbase) {
    constexpr PassPlan PP = make_pass_plan(S);
    constexpr uint32_t idesc = idesc_i8(kBM, kLvBN);
    const GemmParams &p = lp.g;
    const int64_t total = p.batch * p.tiles_m * p.tiles_n;
    const int Sg = p.stages;
    uint32_t stage = 0, phase = 0;
    uint32_t slot_par[kSlots] = {1u, 1u, 1u, 1u};   // parity to wait for (fresh: previous phase done)
    long long t_full = 0, t_slot = 0;
    const long long t_begin = clock64();
    // descriptor of stage base + byte offset: only the 14-bit address field changes
    const uint64_t dbase = smem_desc_kmajor_noswz(0, 128, 256);
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
#pragma unroll
        for (int ps = 0; ps < PP.npass; ++ps) {
            const int hi = PP.hi[ps], lo = PP.lo[ps], tlo = PP.tlo[ps], n = PP.n[ps];
            const uint32_t opb = (uint32_t)n * kBlk;
            const int kpp = lp.pass[ps].kpp;
            for (int64_t kb0 = 0; kb0 < p.KB; kb0 += kpp) {
                const int nk = (int)min((int64_t)kpp, p.KB - kb0);
                long long w0 = p.dbg ? clock64() : 0;
                mbar_wait(&full[stage], phase);
                if (p.dbg) t_full += clock64() - w0;
                tc_fence_after();
                const uint32_t sbase = smem_u32(smem + (size_t)stage * lp.stage_bytes);
                for (int kk = 0; kk < nk; ++kk) {
                    const uint64_t ad0 = dbase + ((sbase + (uint32_t)kk * 2u * opb) >> 4);
                    const uint64_t bd0 = ad0 + (opb >> 4);
                    // slot waits (first k-block of the pass only)
                    if (kb0 == 0 && kk == 0) {
#pragma unroll
                        for (int j = 0; j < hi - lo + 1; ++j) {
                            w0 = p.dbg ? clock64() : 0;
                            mbar_wait(&slot_empty[j], slot_par[j]);
                            slot_par[j] ^= 1u;
                            if (p.dbg) t_slot += clock64() - w0;
                        }
                        tc_fence_after();
                    }
                    // round-robin over the levels of the pass so consecutive MMAs
                    // accumulate into different TMEM slots (an accumulator chain
                    // serialises on MMA latency)
#pragma unroll
                    for (int r = 0; r < S; ++r) {
#pragma unroll
                        for (int j = 0; j < hi - lo + 1; ++j) {
                            const int L = hi - j;
                            const int t0 = pp_max(1, L - S), t1 = pp_min(S, L - 1);
                            const int t = t0 + r;
                            if (t <= t1) {
                                const int u = L - t;
                                const uint32_t acc = (r == 0) ? (uint32_t)(kb0 != 0 || kk != 0) : 1u;
                                mma_i8_elect(tbase + (uint32_t)(j * kLvBN),
                                             ad0 + (uint64_t)(((t - tlo) * kBlk) >> 4),
                                             bd0 + (uint64_t)(((u - tlo) * kBlk) >> 4), idesc, acc);
                            }
                        }
                    }
                }
                mma_commit_elect(&empty[stage]);
                if (++stage == (uint32_t)Sg) { stage = 0; phase ^= 1; }
            }
            mma_commit_elect(pass_full);   // all levels of this pass complete
        }
    }
    if (p.dbg && (threadIdx.x & 31) == 0) {
        atomicAdd(p.dbg + DBG_MMA_WAIT_FULL, (unsigned long long)t_full);
        atomicAdd(p.dbg + DBG_MMA_WAIT_SLOT, (unsigned long long)t_slot);
        atomicAdd(p.dbg + DBG_MMA_TOTAL, (unsigned long long)(clock64() - t_begin));
    }
}

template <int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_lv(const __grid_constant__ LvParams lp) {
    const GemmParams &p = lp.g;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * lp.stage_bytes);
    uint64_t *empty = full + S;
    uint64_t *pass_full = empty + S;
    uint64_t *slot_empty = pass_full + 1;          // kSlots
    uint32_t *tholder = reinterpret_cast<uint32_t *>(slot_empty + kSlots);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int s = p.s;
    const int64_t total = p.batch * p.tiles_m * p.tiles_n;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(pass_full, 1);
        for (int j = 0; j < kSlots; ++j) mbar_init(&slot_empty[j], kNumEpiWarps);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tholder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tholder;
    const int64_t kb_stride = (int64_t)s * kBlk;   // bytes per (tile, k-block) in global

    if (warp == 0) {
        // ========================= producer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            long long t_wait = 0;
            for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
                int64_t b, tm, tn;
                decode_tile(p, tile, b, tm, tn);
                const int8_t *ga = p.A + (b * p.tiles_m + tm) * p.KB * kb_stride;
                const int8_t *gb = p.B + (b * p.tiles_n + tn) * p.KB * kb_stride;
                for (int ps = 0; ps < lp.npass; ++ps) {
                    const LvPass pa = lp.pass[ps];
                    const uint32_t opb = (uint32_t)pa.n * kBlk;   // one operand, one k-block
                    const int64_t toff = (int64_t)(pa.tlo - 1) * kBlk;
                    for (int64_t kb0 = 0; kb0 < p.KB; kb0 += pa.kpp) {
                        const int nk = (int)min((int64_t)pa.kpp, p.KB - kb0);
                        const long long w0 = p.dbg ? clock64() : 0;
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (p.dbg) t_wait += clock64() - w0;
                        mbar_arrive_expect_tx(&full[stage], 2u * opb * nk);
                        uint8_t *dst = smem + (size_t)stage * lp.stage_bytes;
                        for (int kk = 0; kk < nk; ++kk) {
                            const int64_t g = (kb0 + kk) * kb_stride + toff;
                            bulk_g2s(dst, ga + g, opb, &full[stage]);
                            bulk_g2s(dst + opb, gb + g, opb, &full[stage]);
                            dst += 2 * opb;
                        }
                        if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
                    }
                }
            }
            if (p.dbg) atomicAdd(p.dbg + DBG_PROD_WAIT, (unsigned long long)t_wait);
        }
    } else if (warp == 1) {
        // ========================= MMA issuer (whole warp converged, one elected lane issues)
        switch (s) {
#define OZK_MMA_CASE(SS) case SS: lv_mma_role<SS>(lp, smem, full, empty, pass_full, slot_empty, tbase); break;
            OZK_MMA_CASE(1) OZK_MMA_CASE(2) OZK_MMA_CASE(3) OZK_MMA_CASE(4)
            OZK_MMA_CASE(5) OZK_MMA_CASE(6) OZK_MMA_CASE(7) OZK_MMA_CASE(8)
            OZK_MMA_CASE(9) OZK_MMA_CASE(10) OZK_MMA_CASE(11) OZK_MMA_CASE(12)
#undef OZK_MMA_CASE
            default: break;
        }
    } else {
        // ========================= epilogue (8 warps)
        const int ew = warp - 2;
        const int q = warp & 3;          // TMEM lane quarter
        const int half = ew >> 2;        // columns [64*half, 64*half + 64)
        const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * 64);
        uint32_t pphase = 0;
        long long t_w = 0, t_d = 0, t_s = 0;
        for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
            int64_t b, tm, tn;
            decode_tile(p, tile, b, tm, tn);
            const int64_t grow = tm * kBM + q * 32 + lane;
            const int32_t e = (grow < p.Mp) ? __ldg(p.ea + b * p.Mp + grow) : 0;
            double acc[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = 0.0;
            for (int ps = 0; ps < lp.npass; ++ps) {
                const LvPass pa = lp.pass[ps];
                long long w0 = p.dbg ? clock64() : 0;
                mbar_wait(pass_full, pphase);
                long long w1 = p.dbg ? clock64() : 0;
                t_w += w1 - w0;
                pphase ^= 1;
                tc_fence_after();
                for (int L = pa.hi; L >= pa.lo; --L) {          // ascending significance (R6)
                    const int j = pa.hi - L;
                    const double sc = pow2(-8 * (L - 2));
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
                        uint32_t v0[16], v1[16];
                        tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + g * 32), v0);
                        tmem_ld_32x32b_x16(tl + (uint32_t)(j * kLvBN + g * 32 + 16), v1);
                        tmem_wait_ld();
                        if constexpr (EPI == EPI_LEVELS) {   // debug: raw level sums, entry 0
                            if (b == 0 && grow < p.Mp) {
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    const int64_t gcol = tn * kLvBN + half * 64 + g * 32 + i;
                                    if (gcol < p.N)
                                        p.S_out[(int64_t)(L - 2) * p.Mp * p.N + gcol * p.Mp + grow] =
                                            (int32_t)(i < 16 ? v0[i] : v1[i - 16]);
                                }
                            }
                            continue;
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            acc[g * 32 + i] = __fma_rn(i32_to_f64(v0[i]), sc, acc[g * 32 + i]);
                            acc[g * 32 + 16 + i] = __fma_rn(i32_to_f64(v1[i]), sc, acc[g * 32 + 16 + i]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&slot_empty[j]);
                }
                if (p.dbg) t_d += clock64() - w1;
            }
            const long long s0 = p.dbg ? clock64() : 0;
            if constexpr (EPI != EPI_LEVELS) lv_store<EPI>(p, b, grow, e, tn * kLvBN + half * 64, acc);
            if (p.dbg) t_s += clock64() - s0;
        }
        if (p.dbg && warp == 2 && lane == 0) {
            atomicAdd(p.dbg + DBG_EPI_WAIT, (unsigned long long)t_w);
            atomicAdd(p.dbg + DBG_EPI_DRAIN, (unsigned long long)t_d);
            atomicAdd(p.dbg + DBG_EPI_STORE, (unsigned long long)t_s);
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

}  // namespace ozk
