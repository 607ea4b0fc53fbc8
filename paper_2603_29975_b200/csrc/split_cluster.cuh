// split_cluster.cuh -- K1 for long real rows with ONE read of the operand (thread-block clusters).
//
// Same method and output bytes as k_split_fast (split_fast.cuh): §2.2 ("splits
// high-precision input matrices into slices ... based on their significant bits and exponent
// alignment"), readings R3 (row exponent from max |x|, 127-rule) and R4 (X = RNE(x 2^(8s-1-e)),
// balanced base-256 digits) in DESIGN.md §3.
//
// The row exponent needs the max over the WHOLE row before any digit can be formed.  For rows
// longer than one shared-memory window the LONG form of k_split_fast reads every value twice from
// HBM (k_split_exps, then the digit kernel).  Here a cluster of CS CTAs owns a group of RG rows;
// CTA c of the cluster stages the K chunk [c KC, (c+1) KC) of those rows in its shared memory
// (the only HBM read), forms the exact 64-bit partial max |x| of each row over its chunk, and
// pushes its RG partial maxima into every CTA of the cluster (st.async into distributed shared
// memory, completion counted by each receiver's mbarrier -- no cluster-wide barrier after the
// loads, so no CTA waits for stores to drain or for a cluster barrier beyond the partials it
// needs).  Every CTA then holds the exact row max, applies R3, and digitises its chunk straight
// from shared memory.  The max is order-free, so the exponent is bit-identical to the two-pass
// form.
//
// Real operands only (DGEMM long rows: C3, C5), Ozaki-I digits or Ozaki-II residues.  Layout of
// the staged chunk:
//   rows adjacent in memory (rs == 1, op(A) = A): slab[l][row]   (RG * 8 B per l: 64 / 128 B)
//   rows contiguous along K (ls == 1, op(B) = B):  slab[row][l]   (row pitch KC + 2 values)
#pragma once
#include <cstdint>

#include "ptx.cuh"
#include "split_fast.cuh"

namespace ozk {

// rows per CTA and threads: (16, 256) or (8, 128); thread = (row = tid % RG, 8-value unit
// h = tid / RG + (NT / RG) j)

__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// Geometry of one work item (row group r0 of batch entry b, this CTA's K chunk).
struct ClItem {
    int64_t b, r0, l0;
    int kw, kv, nrows;
};
__device__ __forceinline__ ClItem cl_item_geom(const SplitParams &p, int64_t b, int64_t r0, int KC, int RG) {
    ClItem it;
    it.b = b;
    it.r0 = r0;
    it.l0 = (int64_t)cluster_ctarank() * KC;
    const int64_t kpad = p.KB * 32;
    it.kw = (int)max((int64_t)0, min((int64_t)KC, kpad - it.l0));   // depth written (multiple of 32)
    it.kv = (int)max((int64_t)0, min((int64_t)KC, p.k - it.l0));    // valid depth read
    it.nrows = (int)min((int64_t)RG, max((int64_t)0, p.rows - r0));
    return it;
}

// The single HBM read: this CTA's [RG rows x kv] chunk into `slab` (cp.async, not waited for).
template <bool RC, int RG, int NT>
__device__ __forceinline__ void cl_load(const SplitParams &p, const ClItem &it, int KC, double *slab) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double *X = reinterpret_cast<const double *>(p.X) + it.b * p.bstride;
    if constexpr (RC) {
        const double *g0 = X + it.r0 + it.l0 * p.ls;
        if (it.nrows == RG && ((reinterpret_cast<uintptr_t>(g0) | (uintptr_t)(p.ls * 8)) & 15) == 0) {
            // 16-B pieces, RG / 2 per column l (the RG rows of one l are RG * 8 contiguous bytes)
            for (int j = tid; j < it.kv * (RG / 2); j += NT) {
                const int l = j / (RG / 2), c = j % (RG / 2);
                cp_async16(slab + l * RG + 2 * c, g0 + (int64_t)l * p.ls + 2 * c);
            }
        } else {
            for (int j = tid; j < it.kv * RG; j += NT) {
                const int l = j / RG, rr = j % RG;
                if (rr < it.nrows) cp_async8(slab + l * RG + rr, g0 + (int64_t)l * p.ls + rr);
            }
        }
    } else {
        const int LDR = KC + 2;
        for (int rr = warp; rr < it.nrows; rr += NT / 32) {
            const double *g = X + (it.r0 + rr) * p.rs + it.l0;
            double *d = slab + rr * LDR;
            if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
                for (int j = lane; j < it.kv / 2; j += 32) cp_async16(d + 2 * j, g + 2 * j);
                if ((it.kv & 1) && lane == 0) cp_async8(d + it.kv - 1, g + it.kv - 1);
            } else {
                for (int j = lane; j < it.kv; j += 32) cp_async8(d + j, g + j);
            }
        }
    }
}

// Scratch of one CTA (static shared memory of the kernel).
template <int RG, int NT>
struct ClShared {
    uint64_t wmax[NT / 32][RG];
    uint64_t part[RG];        // this CTA's partial maxima
    uint64_t all[16][RG];     // every CTA's partial maxima, pushed by st.async (index: sender rank)
    uint64_t mbar;            // counts the cs * RG * 8 pushed bytes
    int32_t e[RG];
    double scale[RG];
};

__device__ __forceinline__ void st_async_u64(uint32_t cluster_addr, uint64_t v, uint32_t cluster_mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "l"(v), "r"(cluster_mbar)
                 : "memory");
}

// One work item once its chunk is in `slab` (visible to the CTA) and every CTA of the cluster has
// initialised its mbarrier (barrier.cluster.wait done): partial max, push to all CTAs, R3, digits.
template <int S, int TH, bool RC, int RG, int NT, bool CRT>
__device__ __forceinline__ void cl_item(const SplitParams &p, const ClItem &it, int KC, const double *slab,
                                        ClShared<RG, NT> &sh) {
    static_assert(RG == 8 || RG == 16, "rows per CTA");
    static_assert(NT >= 16 * RG, "one push per thread");
    constexpr int HSTEP = NT / RG;          // units of 8 values per sweep of the CTA (multiple of 4)
    constexpr int BLK = TH * 32;            // bytes of one (tile, k-block, slice) block
    constexpr int KBS = CRT ? BLK : S * BLK;   // bytes between k-blocks of one tile
    const int P = CRT ? p.crt.nu : 8 * S - 1;  // R4 fixed-point bits / R17 quantisation bits
    using D = typename std::conditional<CRT, FastResidues<S>, FastDigitsEmit<S>>::type;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int LDR = KC + 2;   // row layout pitch (16-B pad: conflict-free LDS.128 across rows)
    auto at = [&](int row, int l) -> double { return RC ? slab[l * RG + row] : slab[row * LDR + l]; };
    const int kv = it.kv, nrows = it.nrows;
    const uint32_t cs = cluster_nctarank(), kc = cluster_ctarank();

    // ---------------- partial row max over the chunk (exact 64-bit |x| bit patterns)
    const int row = tid % RG, h0 = tid / RG;
    {
        uint64_t m = 0;
        if (row < nrows) {
            for (int h = h0; 8 * h < kv; h += HSTEP) {
                const int nv = min(8, kv - 8 * h);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (i < nv) {
                        const uint64_t u = (uint64_t)__double_as_longlong(at(row, 8 * h + i)) & kAbsMask;
                        m = u > m ? u : m;
                    }
                }
            }
        }
#pragma unroll
        for (int o = RG; o < 32; o <<= 1) {   // lanes l, l ^ RG, ...: the same row
            const uint64_t t = __shfl_xor_sync(0xffffffffu, m, o);
            m = t > m ? t : m;
        }
        if (lane < RG) sh.wmax[warp][lane] = m;
        __syncthreads();
        if (tid < RG) {
            uint64_t v = sh.wmax[0][tid];
#pragma unroll
            for (int w = 1; w < NT / 32; ++w) v = sh.wmax[w][tid] > v ? sh.wmax[w][tid] : v;
            sh.part[tid] = v;
        }
        __syncthreads();
    }
    // ---------------- push: thread t sends row t % RG's partial to CTA t / RG (all[kc][row] there)
    if (tid < (int)cs * RG) {
        const uint32_t dst = (uint32_t)tid / RG;
        st_async_u64(mapa_shared(smem_u32_split(&sh.all[kc][tid % RG]), dst), sh.part[tid % RG],
                     mapa_shared(smem_u32_split(&sh.mbar), dst));
    }
    mbar_wait(&sh.mbar, 0);   // all cs * RG partials of this row group have landed here

    // ---------------- the row max, R3 exponent
    if (tid < RG) {
        uint64_t mx = 0;
        for (uint32_t c = 0; c < cs; ++c) mx = sh.all[c][tid] > mx ? sh.all[c][tid] : mx;
        int32_t e = 0;
        if (tid < nrows) {
            e = (mx >= kExpInf) ? kNonFinite : (CRT ? crt_exponent(mx, p.crt.nu) : exponent_from_maxbits(mx));
            if (kc == 0) {   // one CTA per row group publishes the exponents
                p.exps[it.b * p.rows_out + it.r0 + tid] = e;
                if (e == kNonFinite) atomicAdd(p.nonfinite, 1ull);
            }
        }
        sh.e[tid] = e;
        const int sft = P - e;
        sh.scale[tid] = (sft >= -1022 && sft <= 1023) ? pow2(sft) : 0.0;
    }
    __syncthreads();

    // ---------------- digits from shared memory: thread = (row, units h0 + HSTEP j)
    const int32_t ex = sh.e[row];
    const bool live = (row < nrows) && (ex != kNonFinite);
    const double sc = sh.scale[row];
    const int64_t R = it.r0 + row;
    const int64_t tile = R / TH, rr = R % TH;
    const int64_t tile_bytes = (int64_t)(CRT ? p.crt.n : S) * BLK * p.KB;
    int8_t *op = p.out + (it.b * p.tiles + tile) * tile_bytes + (rr >> 3) * 256 + (rr & 7) * 16 +
                 ((h0 >> 1) & 1) * 128 + (h0 & 1) * 8 + ((it.l0 >> 5) + (h0 >> 2)) * (int64_t)KBS;
    for (int h = h0; 8 * h < it.kw; h += HSTEP, op += (HSTEP / 4) * (int64_t)KBS) {
        const int nv = live ? max(0, min(8, kv - 8 * h)) : 0;
        double v[8];
        if (nv == 8) {
            if constexpr (RC) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = slab[(8 * h + i) * RG + row];
            } else {
                const double2 *s2 = reinterpret_cast<const double2 *>(slab + row * LDR + 8 * h);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double2 t = s2[i];
                    v[2 * i] = t.x;
                    v[2 * i + 1] = t.y;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = (i < nv) ? at(row, 8 * h + i) : 0.0;
        }
        D::template emit1<BLK>(v, sc, 1.0, P - ex, op, p);
    }
}

// blockIdx.x = row group * CS + chunk (cluster dims (CS, 1, 1)), blockIdx.y = batch entry,
// blockIdx.z = side (A: 128-row tiles, B: 64-row halves of the CTA-pair GEMM layout).
// PDL protocol as k_split_fast (cross-call overlap, split_fast.cuh).
// Cluster protocol: each CTA initialises its mbarrier (expecting cs * RG * 8 bytes) and arrives
// (relaxed) on the cluster barrier before its loads; it waits on that barrier only once its own
// chunk is reduced, right before pushing into the other CTAs' shared memory.  A CTA leaves only
// after its own mbarrier has counted every push into it, so no push targets an exited CTA.
// CRT (Ozaki-II, NEXT-1): S is the moduli word count (a multiple of 4), the exponent is R17's,
// the values are quantised to p.crt.nu bits and emitted as residues, 128-row tiles on both sides
// (split_fast.cuh FastResidues).
template <int S, int RG, int NT, bool CRT = false>
__global__ void __launch_bounds__(NT, 3) k_split_cluster(const __grid_constant__ SplitPair pp, int KC, int early) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ __align__(16) uint8_t sbuf[];
    __shared__ ClShared<RG, NT> sh;
    const SplitParams &p = pp.side[blockIdx.z];
    const uint32_t cs = cluster_nctarank();
    const int64_t r0 = (int64_t)(blockIdx.x / cs) * RG;
    // the whole cluster shares the row group, so it leaves together (no dangling cluster barrier)
    if (r0 < p.rows_grid) {
        if (threadIdx.x == 0) {
            mbar_init(&sh.mbar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&sh.mbar, cs * RG * 8);
        }
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
        if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
        double *slab = reinterpret_cast<double *>(sbuf);
        const ClItem it = cl_item_geom(p, blockIdx.y, r0, KC, RG);
        if (p.rs == 1) cl_load<true, RG, NT>(p, it, KC, slab);
        else cl_load<false, RG, NT>(p, it, KC, slab);
        cp_async_wait_all();
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // every mbarrier is initialised
        __syncthreads();
        constexpr int THB = CRT ? 128 : 64;
        if (blockIdx.z == 0) {
            if (p.rs == 1) cl_item<S, 128, true, RG, NT, CRT>(p, it, KC, slab, sh);
            else cl_item<S, 128, false, RG, NT, CRT>(p, it, KC, slab, sh);
        } else {
            if (p.rs == 1) cl_item<S, THB, true, RG, NT, CRT>(p, it, KC, slab, sh);
            else cl_item<S, THB, false, RG, NT, CRT>(p, it, KC, slab, sh);
        }
    } else if (!early) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace ozk
