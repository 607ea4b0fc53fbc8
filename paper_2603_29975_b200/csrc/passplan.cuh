// passplan.cuh -- compile-time/host pass plan of the level-pass GEMM.
//
// The s levels L = s+1 .. 2 (reading R1: level L holds the L-1
// retained pairs t+u = L) are split into ceil(s/4) consecutive groups of at
// most 4 levels (one 128-column TMEM accumulator per level, 512 columns).
// The split is chosen by a modelled time per k-block (selection rule below):
// each pass costs max(MMA clocks, shared-memory port clocks), the MMA issuing one
// M=256 x N=128 x K=32 pair instruction per 64 clk and the port moving 128 B/clk per
// SM of TMA writes (6 KB per slice block: 4 KB of A rows + 2 KB of the B half) plus
// MMA operand reads (6 KB per MMA).  A larger first pass also helps the epilogue: pass 0
// is its integer prefix, every later level costs FP64 work, which is starved while the
// tensor core streams.  (The earlier model -- worst ratio of
// TMA bytes to MMA clocks -- chose e.g. {8,7,6},{5,4,3,2} for s = 7, 1.7% more port
// time and one more FP64 level than {8,7,6,5},{4,3,2}.)  constexpr so the MMA issuer can
// be fully unrolled per s, and callable from the host planner.
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
// modelled time per k-block of the split c[0..np) of levels Lmax .. 2 (fills `out`)
__host__ __device__ constexpr double pp_time(int s, int Lmax, int np, const int (&c)[4], PassPlan &out) {
    out = PassPlan{};
    out.npass = np;
    int hi = Lmax;
    double time = 0;
    for (int q = 0; q < np; ++q) {
        const int lo = hi - c[q] + 1;
        int pairs = 0;
        for (int L = hi; L >= lo; --L) pairs += pp_npairs(L, s);
        const int tlo = pp_max(1, lo - s), thi = pp_min(s, hi - 1);
        const double mma = pairs * 64.0;
        const double port = ((thi - tlo + 1) * 6144.0 + pairs * 6144.0) / 128.0;
        time += mma > port ? mma : port;
        out.hi[q] = hi;
        out.lo[q] = lo;
        out.tlo[q] = tlo;
        out.n[q] = thi - tlo + 1;
        hi = lo - 1;
    }
    return time;
}

// Selection: among the splits within 4% of the least modelled time, the one whose smallest
// pass is largest, then the larger first pass, then the lower time.  Measured on C2 x30:
// s = 5 {6..3},{2} beats {6,5},{4,3,2} by 5.5%; s = 7 {8..5},{4,3,2} beats {8,7,6},{5..2} by
// ~2%; s = 6 keeps {7,6,5},{4,3,2} (the model prefers {7..4},{3,2} by 3.4%, measured 1-3% slower).
__host__ __device__ constexpr PassPlan make_pass_plan_L(int s, int Lmax) {
    const int nlev = Lmax - 1;
    const int np = (nlev + 3) / 4;
    double best_time = 1e30;
    for (int c0 = 1; c0 <= 4; ++c0)
        for (int c1 = (np > 1 ? 1 : 0); c1 <= (np > 1 ? 4 : 0); ++c1)
            for (int c2 = (np > 2 ? 1 : 0); c2 <= (np > 2 ? 4 : 0); ++c2)
                for (int c3 = (np > 3 ? 1 : 0); c3 <= (np > 3 ? 4 : 0); ++c3) {
                    if (c0 + c1 + c2 + c3 != nlev) continue;
                    const int c[4] = {c0, c1, c2, c3};
                    PassPlan cand{};
                    const double t = pp_time(s, Lmax, np, c, cand);
                    if (t < best_time) best_time = t;
                }
    PassPlan best{};
    int best_min = -1, best_c0 = -1;
    double best_t = 1e30;
    for (int c0 = 1; c0 <= 4; ++c0)
        for (int c1 = (np > 1 ? 1 : 0); c1 <= (np > 1 ? 4 : 0); ++c1)
            for (int c2 = (np > 2 ? 1 : 0); c2 <= (np > 2 ? 4 : 0); ++c2)
                for (int c3 = (np > 3 ? 1 : 0); c3 <= (np > 3 ? 4 : 0); ++c3) {
                    if (c0 + c1 + c2 + c3 != nlev) continue;
                    const int c[4] = {c0, c1, c2, c3};
                    PassPlan cand{};
                    const double t = pp_time(s, Lmax, np, c, cand);
                    if (t > best_time * 1.04 + 1e-9) continue;
                    int mn = 4;
                    for (int q = 0; q < np; ++q) mn = pp_min(mn, c[q]);
                    const bool better = mn > best_min || (mn == best_min && c0 > best_c0) ||
                                        (mn == best_min && c0 == best_c0 && t < best_t);
                    if (better) {
                        best_min = mn;
                        best_c0 = c0;
                        best_t = t;
                        best = cand;
                    }
                }
    return best;
}

__host__ __device__ constexpr PassPlan make_pass_plan(int s) { return make_pass_plan_L(s, s + 1); }
__host__ __device__ constexpr PassPlan make_pass_plan_full(int s) { return make_pass_plan_L(s, 2 * s); }

}  // namespace ozk
