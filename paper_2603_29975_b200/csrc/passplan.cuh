// passplan.cuh -- compile-time/host pass plan of the level-pass GEMM.
//
// The s levels L = s+1 .. 2 (reading R1: level L holds the L-1
// retained pairs t+u = L) are split into ceil(s/4) consecutive groups of at
// most 4 levels (one 128-column TMEM accumulator per level, 512 columns).
// Among all such splits we take the one minimising the worst pass ratio of
// operand bytes streamed per k-block to MMA clocks per k-block (the L2 -> SMEM
// demand; 128x128x32 MMA = 64 clk, one slice block = 4 KB per operand),
// tie-broken by total bytes.  constexpr so the MMA issuer can be fully
// unrolled per s, and callable from the host planner.
#pragma once

namespace ozk {

struct PassPlan {
    int npass;
    int hi[4], lo[4], tlo[4], n[4];   // levels hi..lo; slices t,u in [tlo, tlo+n)
};

__host__ __device__ constexpr int pp_min(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int pp_max(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int pp_npairs(int L, int s) { return pp_min(s, L - 1) - pp_max(1, L - s) + 1; }

// Levels Lmax .. 2: Lmax = s + 1 for the triangular pair set (R1), 2s for the
// full set (R21, s <= 8 so that the 2s - 1 levels fit 4 passes).
__host__ __device__ constexpr PassPlan make_pass_plan_L(int s, int Lmax) {
    PassPlan best{};
    const int nlev = Lmax - 1;
    const int np = (nlev + 3) / 4;
    double best_worst = 1e30, best_bytes = 1e30;
    for (int c0 = 1; c0 <= 4; ++c0)
        for (int c1 = (np > 1 ? 1 : 0); c1 <= (np > 1 ? 4 : 0); ++c1)
            for (int c2 = (np > 2 ? 1 : 0); c2 <= (np > 2 ? 4 : 0); ++c2)
                for (int c3 = (np > 3 ? 1 : 0); c3 <= (np > 3 ? 4 : 0); ++c3) {
                    if (c0 + c1 + c2 + c3 != nlev) continue;
                    const int c[4] = {c0, c1, c2, c3};
                    PassPlan cand{};
                    cand.npass = np;
                    int hi = Lmax;
                    double worst = 0, bytes = 0;
                    for (int q = 0; q < np; ++q) {
                        const int lo = hi - c[q] + 1;
                        int pairs = 0;
                        for (int L = hi; L >= lo; --L) pairs += pp_npairs(L, s);
                        const int tlo = pp_max(1, lo - s), thi = pp_min(s, hi - 1);
                        const double by = 2.0 * (thi - tlo + 1) * 4096.0;
                        const double ratio = by / (pairs * 64.0);
                        worst = ratio > worst ? ratio : worst;
                        bytes += by;
                        cand.hi[q] = hi;
                        cand.lo[q] = lo;
                        cand.tlo[q] = tlo;
                        cand.n[q] = thi - tlo + 1;
                        hi = lo - 1;
                    }
                    if (worst < best_worst - 1e-9 || (worst < best_worst + 1e-9 && bytes < best_bytes)) {
                        best_worst = worst;
                        best_bytes = bytes;
                        best = cand;
                    }
                }
    return best;
}

__host__ __device__ constexpr PassPlan make_pass_plan(int s) { return make_pass_plan_L(s, s + 1); }
__host__ __device__ constexpr PassPlan make_pass_plan_full(int s) { return make_pass_plan_L(s, 2 * s); }

}  // namespace ozk
