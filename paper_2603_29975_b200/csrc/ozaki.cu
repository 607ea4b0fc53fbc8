// ozaki.cu -- host runtime of the C ABI declared in include/ozaki.h.
//
// Per call: BLAS argument checks (xerbla-style codes, nothing enqueued on
// error) -> quick returns -> a plan (slice layout, tile grid, pipeline depth)
// -> stream-ordered workspace -> K1 (exponents, slices) for both operands ->
// K2+K3 persistent GEMM with the fused FP64 epilogue.  Everything is enqueued
// on the caller's stream; nothing synchronises the host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <unistd.h>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "crt_kernel.cuh"
#include "gemm.cuh"
#include "gemm_crt.cuh"
#include "gemm_lv.cuh"
#include "gemm_lv2.cuh"
#include "ozaki.h"
#include "split.cuh"
#include "split_fast.cuh"
#include "split_cluster.cuh"
#include "trsm.cuh"

using namespace ozk;

namespace {

thread_local cudaStream_t t_stream = nullptr;
thread_local std::string t_err;
thread_local int t_full_pairs = 0;   // R21 pair set for Ozaki-I calls (ozaki_set_pair_set)
thread_local int64_t t_kblock = 0;    // R22 exponent block along K (0 = per row / column)
thread_local int t_overlap = 0;       // cross-call split / GEMM overlap (ozaki_set_overlap)
thread_local int64_t t_trsm_nb = 128;  // R23 TRSM block (ozaki_set_trsm_block)

// OZAKI_* test / tuning hooks: one scan of the environment per public call
// (env_refresh) instead of a getenv per hook per launch; ozenv() reads the snapshot.
struct EnvSnap {
    int n = 0;
    std::string key[16], val[16];
};
thread_local EnvSnap t_envs;
void env_refresh() {
    EnvSnap &e = t_envs;
    e.n = 0;
    for (char **v = environ; v && *v; ++v) {
        if (strncmp(*v, "OZAKI_", 6) != 0 || e.n >= 16) continue;
        const char *eq = strchr(*v, '=');
        if (!eq) continue;
        e.key[e.n].assign(*v, (size_t)(eq - *v));
        e.val[e.n].assign(eq + 1);
        ++e.n;
    }
}
const char *ozenv(const char *name) {
    const EnvSnap &e = t_envs;
    for (int i = 0; i < e.n; ++i)
        if (e.key[i] == name) return e.val[i].c_str();
    return nullptr;
}

// Cross-call overlap state per (thread, stream, device): two persistent slice workspaces used
// alternately, and whether the last kernel this thread put on the stream is an Ozaki-I GEMM
// (which triggers programmatic dependents at its start) together with the bytes it writes (C).
struct OvState {
    cudaStream_t st = nullptr;
    int dev = -1;
    void *ws[2] = {nullptr, nullptr};
    size_t cap[2] = {0, 0};
    int next = 0;
    bool last_gemm = false;
    uintptr_t c_lo = 0, c_hi = 0;
};
// The persistent workspaces are freed when the thread exits (or on ozaki_set_overlap(0)).
struct OvList {
    std::vector<OvState> v;
    ~OvList() {
        for (auto &o : v)
            for (int i = 0; i < 2; ++i)
                if (o.ws[i]) {
                    int cur = 0;
                    if (cudaGetDevice(&cur) != cudaSuccess) return;   // runtime already torn down
                    cudaSetDevice(o.dev);
                    cudaFree(o.ws[i]);
                    cudaSetDevice(cur);
                }
    }
};
thread_local OvList t_ov_list;
OvState &ov_state(cudaStream_t st) {
    int d = 0;
    cudaGetDevice(&d);
    for (auto &o : t_ov_list.v)
        if (o.st == st && o.dev == d) return o;
    t_ov_list.v.emplace_back();
    t_ov_list.v.back().st = st;
    t_ov_list.v.back().dev = d;
    return t_ov_list.v.back();
}

struct Stats {
    std::atomic<uint64_t> dgemm{0}, zgemm{0}, zgemm3m{0}, entries{0}, equiv{0}, macs{0},
        chunks{0}, launches{0}, crt{0};
} g_stats;

// ------------------------------------------------------------ profiler
enum Phase { PH_EXP = 0, PH_SLICE = 1, PH_GEMM = 2, PH_OTHER = 3 };
struct ProfRec {
    cudaEvent_t a, b;
    int phase;
};
std::atomic<int> g_prof_on{0};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
    // called with g_prof_mu held
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one kernel launch with events when profiling is on.
struct ProfScope {
    cudaEvent_t a = nullptr;
    cudaStream_t st;
    int phase;
    ProfScope(cudaStream_t s, int ph) : st(s), phase(ph) {
        if (!g_prof_on.load(std::memory_order_relaxed)) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        a = prof_event();
        cudaEventRecord(a, st);
    }
    ~ProfScope() {
        if (!a) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        cudaEvent_t b = prof_event();
        cudaEventRecord(b, st);
        g_prof_recs.push_back({a, b, phase});
    }
};

unsigned long long *g_dbg = nullptr;   // role timers (ozaki_debug_timing)
std::atomic<int> g_dbg_on{0};

constexpr int kMaxDev = 64;
struct DevState {
    bool init = false;
    bool ok = false;
    int sms = 0;
    unsigned long long *nonfinite = nullptr;
    uint64_t nonfinite_base = 0;
};
DevState g_dev[kMaxDev];
std::mutex g_mu;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return fail(OZAKI_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

// Dynamic shared memory opt-in, per device and kernel: the attribute belongs to the device
// context, so a process that drives several GPUs sets it once on each; the cache is updated
// under the lock together with the attribute (two threads cannot leave it claiming more than
// the attribute holds).
std::mutex g_attr_mu;
std::unordered_map<const void *, size_t> g_attr[kMaxDev];

cudaError_t smem_optin(const void *fn, size_t smem) {
    if (smem <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t &have = g_attr[dev][fn];
    if (have >= smem) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = smem;
    return e;
}

// Cluster sizes above 8 (non-portable) opt-in, per device and kernel, cached like smem_optin.
std::unordered_map<const void *, bool> g_cl16[kMaxDev];
cudaError_t cluster16_optin(const void *fn) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    bool &have = g_cl16[dev][fn];
    if (have) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) have = true;
    return e;
}

template <int BN, int EPI>
int set_gemm_attr(size_t smem) {
    CUDA_TRY(smem_optin((const void *)k_gemm<BN, EPI>, smem));
    return 0;
}

int device_state(DevState **out) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDev) return fail(OZAKI_ERR_CUDA, "device index %d out of range", dev);
    std::lock_guard<std::mutex> lk(g_mu);
    DevState &d = g_dev[dev];
    if (!d.init) {
        cudaDeviceProp prop;
        CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
        d.init = true;
        d.ok = (prop.major == 10 && prop.minor == 0);
        d.sms = prop.multiProcessorCount;
        if (d.ok) {
            CUDA_TRY(cudaMalloc(&d.nonfinite, sizeof(unsigned long long)));
            CUDA_TRY(cudaMemset(d.nonfinite, 0, sizeof(unsigned long long)));
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;   // keep freed workspace cached in the pool
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
    }
    if (!d.ok) return fail(OZAKI_ERR_ARCH, "device %d is not sm_100 (B200/GB200)", dev);
    *out = &d;
    return 0;
}

bool trans_ok(char t) {
    return t == 'N' || t == 'n' || t == 'T' || t == 't' || t == 'C' || t == 'c';
}
char up(char t) { return (char)(t >= 'a' ? t - 32 : t); }
int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

enum Kind { KIND_REAL = 0, KIND_4M = 1, KIND_3M = 2 };

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// ------------------------------------------------------------------- plan
struct Plan {
    int s, BN;
    bool full = false;   // R21 full pair set (levels 2s .. 2)
    int64_t m, n, k, batch;
    int64_t Mp;          // output rows of the real product
    int64_t Np;          // output columns of the real product (2n for 4M: Re/Im interleaved)
    int64_t kh;          // 4M half width
    int64_t Kp, KB;      // padded depth (bytes) and 32-B blocks
    int64_t tiles_m, tiles_n;
    size_t a_bytes, b_bytes, ea_bytes, fb_bytes;   // per whole batch, 256-B aligned
    size_t a_bytes_entry, b_bytes_entry;           // slice bytes of one batch entry (unaligned)
    int kps, stages;
    size_t smem;
    bool kchunk_needed;      // s * k_eff > 131071 (reading R8)
    bool lv;                 // level-pass kernels (BN = 128)
    bool pair;               // ... on CTA pairs (k_gemm_lv2, M = 256 per pair)
    int a_tile_h, b_tile_h;  // operand row tiles of the split layout
    int npass;
    uint32_t stage_bytes;
    LvPass pass[kMaxPass];
    int splitk = 1;          // split-K units per tile (a7: small problems, CHUNK 3 + k_splitk_combine)
    int pk_np = 0, pk_nl = 0;   // prefix levels (pass 0) / later levels of the split-K partials
    size_t p0_bytes = 0, pl_bytes = 0;
};

// Split-K: when the super-tiles leave two thirds of the CTA pairs idle,
// every tile is cut into S units over equal shares of the k-blocks (>= 4 k-blocks each), so
// up to all pairs work; the units' exact integer partials are added by k_splitk_combine.
// OZAKI_SPLITK=n forces S (tests; 1 = off).
void plan_splitk(Plan &P, int sms) {
    P.splitk = 1;
    if (!P.pair || P.kchunk_needed || P.batch == 0) return;
    const int64_t tiles = P.batch * P.tiles_m * P.tiles_n, pairs = sms / 2;
    int64_t S = 1;
    if (const char *e = ozenv("OZAKI_SPLITK")) {
        S = std::max<int64_t>(1, std::min<int64_t>(atoll(e), P.KB));
    } else if (3 * tiles <= pairs) {   // S >= 3: at S = 2 the partials cost what the split saves
        S = std::min<int64_t>({pairs / tiles, P.KB / 4, 16});   // (DGEMM 1024^3: 60.5 vs 55.8 us)
    }
    if (S <= 1) return;
    P.splitk = (int)S;
    P.pk_np = P.pass[0].hi - P.pass[0].lo + 1;
    P.pk_nl = (P.full ? 2 * P.s : P.s + 1) - 1 - P.pk_np;
    const size_t elems = (size_t)P.batch * P.Mp * P.Np;
    P.p0_bytes = al256((size_t)S * elems * 8);
    P.pl_bytes = al256((size_t)S * P.pk_nl * elems * 4);
}

// Pass plan of the level-pass kernel: make_pass_plan (passplan.cuh, shared
// with the device code) plus the per-pass k-blocks per stage.
void plan_passes(int s, Plan &P) {
    const PassPlan pp = P.full ? make_pass_plan_full(s) : make_pass_plan(s);
    P.npass = pp.npass;
    const uint32_t kb_bytes_per_slice = (uint32_t)(P.a_tile_h + P.b_tile_h) * kKB;   // A + B rows
    uint32_t maxb = 0;
    for (int q = 0; q < pp.npass; ++q) {
        LvPass &pa = P.pass[q];
        pa.hi = pp.hi[q];
        pa.lo = pp.lo[q];
        pa.tlo = pp.tlo[q];
        pa.n = pp.n[q];
        maxb = std::max<uint32_t>(maxb, (uint32_t)pa.n * kb_bytes_per_slice);
    }
    // Stages of at least ~54 KB: a small-s pass (s = 3: 18 KB per k-block) then takes several
    // k-blocks per stage -- fewer barrier round trips per MMA and more bytes in flight.  C3 GEMM,
    // same clock: s = 3 2.53 -> 2.24 ms, s = 4 3.52 -> 3.41 ms; s >= 5 (>= 30 KB per k-block) and
    // C2 x 30 unchanged.  OZAKI_STAGE_KB overrides the minimum (tuning hook).
    {
        uint32_t want = 54u * 1024u;
        if (const char *e = ozenv("OZAKI_STAGE_KB")) want = (uint32_t)std::max(0, atoi(e)) * 1024u;
        if (want > maxb) maxb = want / maxb * maxb;
    }
    P.stage_bytes = maxb;
    for (int q = 0; q < pp.npass; ++q) {
        const uint32_t per = (uint32_t)P.pass[q].n * kb_bytes_per_slice;
        P.pass[q].kpp = (int)std::max<int64_t>(1, std::min<int64_t>(maxb / per, P.KB));
    }
}

// Kernel selection: OZAKI_KERNEL = "pair" (default for s <= 12), "lv1", "flat".
int kernel_choice() {
    static int choice = -1;
    if (choice < 0) {
        const char *e = getenv("OZAKI_KERNEL");
        choice = 2;
        if (e && !strcmp(e, "lv1")) choice = 1;
        if (e && !strcmp(e, "flat")) choice = 0;
    }
    return choice;
}

int make_plan(Kind kind, int64_t m, int64_t n, int64_t k, int64_t batch, int s, Plan &P, bool full = false) {
    P.s = s;
    P.full = full;
    P.BN = (s <= 8) ? 64 : 32;
    P.m = m;
    P.n = n;
    P.k = k;
    P.batch = batch;
    P.Mp = m;
    if (kind == KIND_4M) {   // R9: [Ar|Ai] x [[Br,Bi],[-Bi,Br]], columns interleaved
        P.Np = 2 * n;
        P.kh = rup(k, 32);
        P.Kp = 2 * P.kh;
    } else {
        P.Np = n;
        P.kh = 0;
        P.Kp = rup(k, 32);
    }
    // R8: a level sums (L-1) * k_eff products of magnitude <= 2^14 in INT32; the
    // pair kernel splits K into chunks that respect this (exact FP64 partials),
    // the other kernels need the whole K in one INT32 accumulation.
    const int64_t keff = (kind == KIND_4M) ? 2 * k : k;
    P.kchunk_needed = (int64_t)s * keff > 131071;
    P.KB = P.Kp / 32;
    const int kc = kernel_choice();
    P.lv = (s <= 12) && kc >= 1;
    P.pair = P.lv && kc == 2;
    if (P.kchunk_needed && !P.pair)
        return fail(OZAKI_ERR_UNSUPPORTED,
                    "s*k_eff = %lld exceeds the INT32 level-sum bound 131071 and K-chunking needs the "
                    "CTA-pair kernel (s <= 12)",
                    (long long)((int64_t)s * keff));
    if (full && (!P.pair || s > 8 || P.kchunk_needed))
        return fail(OZAKI_ERR_UNSUPPORTED,
                    "the full pair set (R21) needs the CTA-pair kernel, s <= 8 and s*k_eff <= 131071");
    if (P.lv) P.BN = kLvBN;
    P.a_tile_h = kBM;
    P.b_tile_h = P.pair ? kLvBN / 2 : P.BN;
    if (P.pair) {   // super-tiles of 256 x 128; A in 128-row tiles (padded to pairs), B in 64-row halves
        P.tiles_m = (P.Mp + 2 * kBM - 1) / (2 * kBM);
        P.tiles_n = (P.Np + kLvBN - 1) / kLvBN;
        P.a_bytes_entry = (size_t)s * kBM * kKB * P.KB * (2 * P.tiles_m);
        P.b_bytes_entry = (size_t)s * (kLvBN / 2) * kKB * P.KB * (2 * P.tiles_n);
        P.a_bytes = al256(P.a_bytes_entry * batch);
        P.b_bytes = al256(P.b_bytes_entry * batch);
    } else {
        P.tiles_m = (P.Mp + kBM - 1) / kBM;
        P.tiles_n = (P.Np + P.BN - 1) / P.BN;
        P.a_bytes_entry = (size_t)s * kBM * kKB * P.KB * P.tiles_m;
        P.b_bytes_entry = (size_t)s * P.BN * kKB * P.KB * P.tiles_n;
        P.a_bytes = al256(P.a_bytes_entry * batch);
        P.b_bytes = al256(P.b_bytes_entry * batch);
    }
    const size_t a_kb = (size_t)s * kBM * kKB, b_kb = (size_t)s * P.BN * kKB;
    P.ea_bytes = al256(sizeof(int32_t) * P.Mp * batch);
    P.fb_bytes = al256(sizeof(int32_t) * P.Np * batch);
    const size_t budget = 226 * 1024;
    if (P.lv) {
        plan_passes(s, P);
        P.kps = 1;
        int smax = 8;
        if (const char *e = ozenv("OZAKI_STAGES_MAX")) smax = std::max(2, std::min(16, atoi(e)));
        P.stages = (int)std::min<size_t>((size_t)smax, (budget - 2048) / P.stage_bytes);
        P.smem = (size_t)P.stages * P.stage_bytes + 1024 + 512;
    } else {
        const size_t kb_bytes = a_kb + b_kb;
        P.kps = (int)std::max<size_t>(1, std::min<size_t>(40960 / kb_bytes, (size_t)P.KB));
        P.stages = (int)std::min<size_t>(8, (budget - 2048) / (P.kps * kb_bytes));
        P.smem = (size_t)P.stages * P.kps * kb_bytes + 1024 /*align*/ + 256 /*barriers*/;
    }
    if (P.stages < 2) return fail(OZAKI_ERR_UNSUPPORTED, "pipeline does not fit in shared memory");
    // the kernels decode (batch, tile, split-K unit) in 32-bit arithmetic
    if ((double)P.batch * (double)P.tiles_m * (double)P.tiles_n * 16.0 >= 2147483648.0)
        return fail(OZAKI_ERR_UNSUPPORTED, "batch x tiles = %lld exceeds 2^27", (long long)(P.batch * P.tiles_m * P.tiles_n));
    return 0;
}

size_t plan_workspace(const Plan &P) { return P.a_bytes + P.b_bytes + P.ea_bytes + P.fb_bytes; }

// ------------------------------------------------------------ small kernels
__global__ void k_scale_real(double *C, int64_t m, int64_t n, int64_t ldc, int64_t strideC,
                             double beta) {
    const int64_t b = blockIdx.z;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % m, j = idx / m;
        double *cp = C + b * strideC + i + j * ldc;
        *cp = (beta == 0.0) ? 0.0 : __dmul_rn(beta, *cp);
    }
}

__global__ void k_scale_cplx(double *C, int64_t m, int64_t n, int64_t ldc, int64_t strideC,
                             double br, double bi) {
    const int64_t b = blockIdx.z;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = idx % m, j = idx / m;
        double2 *cp = reinterpret_cast<double2 *>(C) + b * strideC + i + j * ldc;
        if (br == 0.0 && bi == 0.0) {
            *cp = make_double2(0.0, 0.0);
        } else {
            double2 c = *cp;
            *cp = make_double2(__fma_rn(br, c.x, -__dmul_rn(bi, c.y)), __fma_rn(br, c.y, __dmul_rn(bi, c.x)));
        }
    }
}

// 3M: C_re = fl(T1-T2), C_im = fl(fl(T3-T1)-T2), then complex alpha/beta (R7, R9).
__global__ void k_combine_3m(const double *T1, const double *T2, const double *T3, double *C,
                             int64_t m, int64_t n, int64_t ldc, int64_t strideC, double ar,
                             double ai, double br, double bi) {
    const int64_t b = blockIdx.z;
    const int64_t off = b * m * n;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % m, j = idx / m;
        const double t1 = T1[off + idx], t2 = T2[off + idx], t3 = T3[off + idx];
        const double pr = __dsub_rn(t1, t2);
        const double pi = __dsub_rn(__dsub_rn(t3, t1), t2);
        double2 *cp = reinterpret_cast<double2 *>(C) + b * strideC + i + j * ldc;
        double tr = 0.0, ti = 0.0;
        if (!(br == 0.0 && bi == 0.0)) {
            double2 c = *cp;
            tr = __fma_rn(br, c.x, -__dmul_rn(bi, c.y));
            ti = __fma_rn(br, c.y, __dmul_rn(bi, c.x));
        }
        *cp = make_double2(__fma_rn(ar, pr, __fma_rn(-ai, pi, tr)), __fma_rn(ar, pi, __fma_rn(ai, pr, ti)));
    }
}

// R22: C = alpha T + beta C with R7's operation shapes (T: batch x m x n, ld m).
__global__ void k_apply_ab(const double *T, double *C, int64_t m, int64_t n, int64_t ldc, int64_t strideC,
                           int cplx, double ar, double ai, double br, double bi) {
    const int64_t b = blockIdx.z;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % m, j = idx / m;
        if (!cplx) {
            const double P = T[b * m * n + idx];
            double *cp = C + b * strideC + i + j * ldc;
            *cp = (br == 0.0) ? __dmul_rn(ar, P) : __fma_rn(ar, P, __dmul_rn(br, *cp));
        } else {
            const double2 P = reinterpret_cast<const double2 *>(T)[b * m * n + idx];
            double2 *cp = reinterpret_cast<double2 *>(C) + b * strideC + i + j * ldc;
            double tr = 0.0, ti = 0.0;
            if (!(br == 0.0 && bi == 0.0)) {
                const double2 cv = *cp;
                tr = __fma_rn(br, cv.x, -__dmul_rn(bi, cv.y));
                ti = __fma_rn(br, cv.y, __dmul_rn(bi, cv.x));
            }
            *cp = make_double2(__fma_rn(ar, P.x, __fma_rn(-ai, P.y, tr)), __fma_rn(ar, P.y, __fma_rn(ai, P.x, ti)));
        }
    }
}

// Debug: tiled slices -> plain [s][rows_out][kdepth] int8.
__global__ void k_unpack(const int8_t *tiled, int8_t *out, int64_t rows_out, int64_t kdepth,
                         int s, int tile_h, int64_t KB) {
    const int64_t total = (int64_t)s * rows_out * kdepth;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = idx % kdepth;
        const int64_t r = (idx / kdepth) % rows_out;
        const int64_t t = idx / (kdepth * rows_out);
        const int64_t tile = r / tile_h, rr = r % tile_h, kb = l / 32, c = (l % 32) / 16, x = l % 16;
        const int64_t off = ((tile * KB + kb) * s + t) * (int64_t)tile_h * 32 + (rr >> 3) * 256 +
                            c * 128 + (rr & 7) * 16 + x;
        out[idx] = tiled[off];
    }
}

unsigned grid1d(int64_t work, int sms) {
    int64_t g = (work + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 16));
}

// ---------------------------------------------------------------- K1 launch
struct Operand {
    const void *X;
    int64_t rs, ls, bstride;
    int64_t rows, k;
    int mode, conj;
};

SplitParams split_params(const Plan &P, const Operand &op, bool sideA, int8_t *slices, int32_t *exps,
                         DevState *dev, int64_t x_batch) {
    SplitParams sp{};
    sp.X = op.X;
    sp.rs = op.rs;
    sp.ls = op.ls;
    sp.bstride = op.bstride;
    sp.rows = op.rows;
    sp.k = op.k;
    sp.mode = op.mode;
    sp.conj = op.conj;
    sp.s = P.s;
    sp.tile_h = sideA ? P.a_tile_h : P.b_tile_h;
    sp.kbs_bytes = (int64_t)P.s * sp.tile_h * 32;   // layout [tile][kb][slice][block]
    sp.ss_bytes = (int64_t)sp.tile_h * 32;
    sp.tiles = (sideA ? P.tiles_m : P.tiles_n) * (P.pair ? 2 : 1);
    sp.KB = P.KB;
    sp.kh = P.kh;
    sp.rows_out = (op.mode == SPLIT_B4M) ? 2 * op.rows : op.rows;
    sp.rows_grid = (op.rows == 0) ? 0 : ((op.mode == SPLIT_B4M) ? sp.tiles * sp.tile_h / 2 : sp.tiles * sp.tile_h);
    sp.out = slices;
    sp.exps = exps;
    sp.nonfinite = dev->nonfinite;
    // SPLIT_3M: the plan covers 3 x x_batch entries; the three operands go to regions x = 0, 1, 2
    if (op.mode == SPLIT_3M) {
        sp.x_bytes = (int64_t)((sideA ? P.a_bytes_entry : P.b_bytes_entry) * x_batch);
        sp.x_exps = (sideA ? P.Mp : P.Np) * x_batch;
    }
    return sp;
}

// K1 specialised for the production layout (k_split_fast, split_fast.cuh): both operands in one
// launch, CTA-pair tiles (A 128 rows, B 64 rows), s <= 8, Ozaki-I digit layout.  Returns 1 when
// the call does not qualify (the generic k_split_sm runs), else 0 / an error code.
// OZAKI_SPLIT=generic forces the generic kernel (A/B tests).
// LONG form of k_split_fast: 16 rows per CTA (512 threads) for real operands, 8 for complex
template <int S, int MA, int MB>
void launch_split_long(dim3 grid, size_t smem, cudaStream_t st, const SplitPair &pp, int KW, int nwin) {
    constexpr int R = (MA == SPLIT_REAL) ? 16 : 8;
    smem_optin((const void *)k_split_fast<S, MA, MB, R, true>, smem);   // a failure surfaces at launch
    k_split_fast<S, MA, MB, R, true><<<grid, 32 * R, smem, st>>>(pp, KW, nwin, 0);
}

// cudaLaunchKernelEx with programmatic stream serialisation when `pdl` (cross-call overlap)
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// Long-row split, first kernel: K-chunked exponent scan (k_split_exps) into a zeroed buffer of
// biased per-row exponents ([NX][batch][rows] per side, freed in stream order by the caller).
// mode: 0 real, 1 4M, 2 3M.  The digit kernel reads it back (split_fast.cuh LONG).
int launch_exps(SplitPair &pp, unsigned batch, int nx, int mode, bool crt, cudaStream_t st, uint32_t **emax_out) {
    const size_t na = (size_t)nx * batch * std::max<int64_t>(1, pp.side[0].rows);
    const size_t nb = (size_t)nx * batch * std::max<int64_t>(1, pp.side[1].rows);
    uint32_t *emax = nullptr;
    {
        cudaError_t e = cudaMallocAsync((void **)&emax, 4 * (na + nb), st);
        if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "cudaMallocAsync(emax): %s", cudaGetErrorString(e));
    }
    CUDA_TRY(cudaMemsetAsync(emax, 0, 4 * (na + nb), st));
    int64_t ctas = 1;
    for (int sd = 0; sd < 2; ++sd) {
        SplitParams &q = pp.side[sd];
        q.emax = emax + (sd ? na : 0);
        // split K only as far as needed for ~16 CTAs per SM over the side (few long row groups
        // are the slow case: C3's 256 groups of 32 adjacent rows); chunks of >= 256 elements
        static const int sms = [] {
            int d = 0, v = 148;
            cudaGetDevice(&d);
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
            return v;
        }();
        const int64_t groups = (q.rows + (q.rs == 1 ? 31 : 7)) / (q.rs == 1 ? 32 : 8);
        const int64_t gb = groups * batch;
        const int64_t want = gb < 4 * (int64_t)sms ? std::max<int64_t>(1, (16 * (int64_t)sms + gb - 1) / gb) : 1;
        const int64_t kc = (q.k + want - 1) / want;
        q.kchunk = (int32_t)std::max<int64_t>(256, (kc + 255) / 256 * 256);
        ctas = std::max<int64_t>(ctas, groups * ((q.k + q.kchunk - 1) / q.kchunk));
    }
    dim3 ge((unsigned)ctas, batch, 2);
    {
        ProfScope ps(st, PH_EXP);
        if (crt) {
            if (mode == 0) k_split_exps<SPLIT_REAL, SPLIT_REAL, true><<<ge, 256, 0, st>>>(pp);
            else k_split_exps<SPLIT_A4M, SPLIT_B4M, true><<<ge, 256, 0, st>>>(pp);
        } else {
            if (mode == 0) k_split_exps<SPLIT_REAL, SPLIT_REAL><<<ge, 256, 0, st>>>(pp);
            else if (mode == 1) k_split_exps<SPLIT_A4M, SPLIT_B4M><<<ge, 256, 0, st>>>(pp);
            else k_split_exps<SPLIT_3M, SPLIT_3M><<<ge, 256, 0, st>>>(pp);
        }
    }
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    *emax_out = emax;
    return 0;
}

// Cross-call overlap request for the next split launch (set by run() for ozaki_set_overlap):
// pdl = launch with PDL after the previous call's GEMM; early = may read / write before it ends.
thread_local bool t_split_pdl = false, t_split_early = false;

// Long real rows in one HBM read (split_cluster.cuh): a cluster of CS CTAs per 8-row group
// (OZAKI_SPLIT_RG=16: 16 rows), chunk KC <= KCMAX values of K per CTA (32 KB of shared memory at 512).  Returns 1 when the
// shape does not qualify (the two-kernel LONG form runs).  OZAKI_SPLIT_CLUSTER=0 disables it,
// OZAKI_SPLIT_KC sets KCMAX (tuning hook).
// sw: the slice count s (Ozaki-I) or the moduli word count (CRT: a multiple of 4).
template <bool CRT>
int launch_split_cluster(int sw, const SplitPair &pp, unsigned batch, cudaStream_t st, bool pdl, bool early) {
    if (const char *e = ozenv("OZAKI_SPLIT_CLUSTER"))
        if (atoi(e) == 0) return 1;
    // 8 rows x 512 values (32 KB, six CTAs per SM) measured best on C3: split 0.28 ms at s = 3,
    // 0.41 ms at s = 7 (16 rows: 0.31 / 0.45; 8 x 1024: 0.31 / 0.45; two-kernel form 0.57 / 0.74)
    int kcmax = 512, rg = 8;
    if (const char *e = ozenv("OZAKI_SPLIT_KC")) {
        const int v = atoi(e);
        if (v >= 64 && v <= 1024 && v % 32 == 0) kcmax = v;
    }
    if (const char *e = ozenv("OZAKI_SPLIT_RG"))
        if (atoi(e) == 16) rg = 16;
    for (int sd = 0; sd < 2; ++sd) {
        const SplitParams &q = pp.side[sd];
        if (q.mode != SPLIT_REAL || (q.rs != 1 && q.ls != 1)) return 1;
    }
    const int64_t kpad = pp.side[0].KB * 32;
    const int64_t cs = (kpad + kcmax - 1) / kcmax;
    if (cs < 2 || cs > 16) return 1;
    const int KC = (int)(((kpad + cs - 1) / cs + 31) / 32 * 32);
    const int64_t groups = (std::max(pp.side[0].rows_grid, pp.side[1].rows_grid) + rg - 1) / rg;
    if (groups * cs > INT32_MAX) return 1;
    const size_t smem = (size_t)rg * (KC + 2) * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(groups * cs), batch, 2);
    cfg.blockDim = dim3(rg == 16 ? 256 : 128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto prep = [&](const void *kern) -> int {
        CUDA_TRY(smem_optin(kern, smem));
        if (cs > 8) CUDA_TRY(cluster16_optin(kern));
        return 0;
    };
    auto go = [&](auto kern) -> int {
        if (prep((const void *)kern)) {   // no cluster opt-in on this device: the two-kernel form
            cudaGetLastError();
            return 1;
        }
        cfg.numAttrs = pdl ? 2 : 1;
        ProfScope ps(st, PH_SLICE);
        if (cudaLaunchKernelEx(&cfg, kern, pp, KC, early ? 1 : 0) != cudaSuccess) {
            cudaGetLastError();   // e.g. a cluster shape the device cannot co-schedule
            return 1;
        }
        return 0;
    };
#define OZK_CL(S)                                                                                          \
    case S:                                                                                                \
        return rg == 16 ? go(k_split_cluster<S, 16, 256, CRT>) : go(k_split_cluster<S, 8, 128, CRT>);
    if constexpr (CRT) {
        switch (sw) { OZK_CL(4) OZK_CL(8) OZK_CL(12) OZK_CL(16) OZK_CL(20) }
    } else {
        switch (sw) {
            OZK_CL(1) OZK_CL(2) OZK_CL(3) OZK_CL(4) OZK_CL(5) OZK_CL(6)
            OZK_CL(7) OZK_CL(8) OZK_CL(9) OZK_CL(10) OZK_CL(11) OZK_CL(12)
        }
    }
#undef OZK_CL
    return 1;
}

int launch_split_fast(const Plan &P, const SplitParams &a, const SplitParams *b, dim3 grid, cudaStream_t st) {
    const bool pdl = t_split_pdl, early = t_split_early;
    if (!b || !P.pair || P.s < 1 || P.s > 12) return 1;
    if (a.tile_h != 128 || b->tile_h != 64) return 1;
    if (a.kbs_bytes != (int64_t)P.s * 128 * 32 || b->kbs_bytes != (int64_t)P.s * 64 * 32) return 1;
    const bool real = a.mode == SPLIT_REAL && b->mode == SPLIT_REAL;
    const bool fourm = a.mode == SPLIT_A4M && b->mode == SPLIT_B4M;
    const bool threem = a.mode == SPLIT_3M && b->mode == SPLIT_3M;
    if (!real && !fourm && !threem) return 1;
    if (const char *e = ozenv("OZAKI_SPLIT"))
        if (!strcmp(e, "generic")) return 1;
    int KW = real ? 1024 : 512;
    if (const char *kw = ozenv("OZAKI_SPLIT_KW")) {   // tuning hook: window elements per row
        const int v = atoi(kw);
        if (v >= 64 && v <= 1024 && v % 32 == 0) KW = v;
    }
    // rows per CTA (one warp each): 4 -- more, smaller CTAs than 8 rows, so more load / compute
    // phases overlap per SM at the same SMEM per row (measured: equal for 4M, -8% time for 3M)
    int RG = 4;
    // long rows (>= 3 windows): exponents first (k_split_exps), then one CTA per (row group,
    // window) -- OZAKI_SPLIT_LONG=0 / 1 forces the single-kernel / two-kernel form
    const int64_t kpad = fourm ? a.kh : a.KB * 32;
    int nwin = (int)((kpad + KW - 1) / KW);
    if (nwin == 2 && !ozenv("OZAKI_SPLIT_KW")) {   // rows of two windows: one double window
        KW *= 2;                                   // (64 KB per 4-row CTA) beats re-reading the
        nwin = 1;                                  // row from L2 (C4: 0.64 -> 0.47 ms)
    }
    bool lng = nwin >= 3;
    if (const char *lg = ozenv("OZAKI_SPLIT_LONG")) lng = (atoi(lg) != 0) && nwin > 1;
    if (lng && real) {   // one HBM read through a thread-block cluster when the rows fit 16 chunks
        SplitPair pc;
        pc.side[0] = a;
        pc.side[1] = *b;
        const int rc = launch_split_cluster<false>(P.s, pc, grid.y, st, pdl, early);
        if (rc <= 0) {
            if (rc == 0) g_stats.launches += 1;
            return rc;
        }
    }
    if (lng) {   // short windows, more rows per CTA: 128-B reads per l when rows are adjacent
        RG = real ? 16 : 8;
        KW = 256;
        nwin = (int)((kpad + KW - 1) / KW);
    }
    grid.x = (unsigned)((std::max(a.rows_grid, b->rows_grid) + RG - 1) / RG) * (lng ? nwin : 1);
    SplitPair pp;
    pp.side[0] = a;
    pp.side[1] = *b;
    uint32_t *emax = nullptr;
    if (lng) {
        if (int rc = launch_exps(pp, grid.y, threem ? 3 : 1, real ? 0 : (fourm ? 1 : 2), false, st, &emax)) return rc;
    }
    const size_t smem = (size_t)RG * (KW + (real ? 2 : 1)) * (real ? 8 : 16);
    {
        ProfScope ps(st, PH_SLICE);
#define OZK_FAST_RG(S, MA, MB, R)                                                                    \
        {                                                                                            \
            smem_optin((const void *)k_split_fast<S, MA, MB, R>, smem);                               \
            launch_pdl(k_split_fast<S, MA, MB, R>, grid, dim3(32 * R), smem, st, pdl, pp, KW, nwin,   \
                       early ? 1 : 0);                                                               \
        }
#define OZK_FAST_LONG(S, MA, MB) launch_split_long<S, MA, MB>(grid, smem, st, pp, KW, nwin);
#define OZK_FAST(S, MA, MB)                                                                          \
        if (lng) OZK_FAST_LONG(S, MA, MB) else OZK_FAST_RG(S, MA, MB, 4)
#define OZK_FAST_S(S)                                                                                \
        case S:                                                                                      \
            if (real) OZK_FAST(S, SPLIT_REAL, SPLIT_REAL)                                            \
            else if (fourm) OZK_FAST(S, SPLIT_A4M, SPLIT_B4M)                                        \
            else OZK_FAST(S, SPLIT_3M, SPLIT_3M)                                                     \
            break;
        switch (P.s) {
            OZK_FAST_S(1) OZK_FAST_S(2) OZK_FAST_S(3) OZK_FAST_S(4)
            OZK_FAST_S(5) OZK_FAST_S(6) OZK_FAST_S(7) OZK_FAST_S(8)
            OZK_FAST_S(9) OZK_FAST_S(10) OZK_FAST_S(11) OZK_FAST_S(12)
        }
#undef OZK_FAST_S
#undef OZK_FAST
#undef OZK_FAST_RG
#undef OZK_FAST_LONG
    }
    if (emax) cudaFreeAsync(emax, st);
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    return 0;
}

// K1 for one (b == nullptr) or both operands in one launch.
int launch_split_sides(const Plan &P, const SplitParams &a, const SplitParams *b, int64_t gb, cudaStream_t st) {
    SplitPair pp;
    pp.side[0] = a;
    pp.side[1] = b ? *b : a;
    const int64_t rows_grid = std::max(a.rows_grid, b ? b->rows_grid : 0);
    if (rows_grid == 0) return 0;
    const bool cplx = a.mode != SPLIT_REAL;
    dim3 grid((unsigned)((rows_grid + 7) / 8), (unsigned)gb, b ? 2u : 1u);
    if (int rc = launch_split_fast(P, a, b, grid, st); rc <= 0) return rc;   // production layout
    // SMEM window: 8 rows x KW elements (+ pad), 64 KB
    int KW = cplx ? 512 : 1024;
    if (const char *kw = ozenv("OZAKI_SPLIT_KW")) {   // tuning hook: window elements per row
        const int v = atoi(kw);
        if (v >= 64 && v <= 1024) KW = cplx ? std::min(v, 512) : v;
    }
    const size_t smem = (size_t)8 * (KW + (cplx ? 1 : 2)) * (cplx ? 16 : 8);
    {
        ProfScope ps(st, PH_SLICE);
#define OZK_SPLIT(SM, CX)                                                                           \
        {                                                                                           \
            smem_optin((const void *)k_split_sm<SM, CX>, smem);                                     \
            k_split_sm<SM, CX><<<grid, 256, smem, st>>>(pp, KW);                                    \
        }
        if (P.s <= 8) {
            if (cplx) OZK_SPLIT(8, true) else OZK_SPLIT(8, false)
        } else {
            if (cplx) OZK_SPLIT(16, true) else OZK_SPLIT(16, false)
        }
#undef OZK_SPLIT
    }
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    return 0;
}

int launch_split(const Plan &P, const Operand &op, bool sideA, int8_t *slices, int32_t *exps,
                 DevState *dev, cudaStream_t st, int64_t x_batch = 0) {
    const SplitParams sp = split_params(P, op, sideA, slices, exps, dev, x_batch);
    return launch_split_sides(P, sp, nullptr, op.mode == SPLIT_3M ? x_batch : P.batch, st);
}

// both operands of one product in a single launch
int launch_split_ab(const Plan &P, const Operand &oa, int8_t *sa, int32_t *ea, const Operand &ob, int8_t *sb,
                    int32_t *fb, DevState *dev, cudaStream_t st, int64_t x_batch = 0) {
    const SplitParams pa = split_params(P, oa, true, sa, ea, dev, x_batch);
    const SplitParams pb = split_params(P, ob, false, sb, fb, dev, x_batch);
    return launch_split_sides(P, pa, &pb, oa.mode == SPLIT_3M ? x_batch : P.batch, st);
}

// ---------------------------------------------------------------- K2 launch
template <int EPI>
int launch_gemm_lv(const Plan &P, const GemmParams &gp, DevState *dev, cudaStream_t st) {
    CUDA_TRY(smem_optin((const void *)k_gemm_lv<EPI>, P.smem));
    LvParams lp{};
    lp.g = gp;
    lp.npass = P.npass;
    lp.stage_bytes = P.stage_bytes;
    for (int q = 0; q < P.npass; ++q) lp.pass[q] = P.pass[q];
    const int64_t tiles = P.batch * P.tiles_m * P.tiles_n;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, dev->sms);
    {
        ProfScope ps(st, PH_GEMM);
        k_gemm_lv<EPI><<<grid, kGemmThreads, P.smem, st>>>(lp);
    }
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    return 0;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

// Encoded maps are cached per thread by (base, bytes, box): the workspaces come back at the
// same addresses (stream-ordered pool, persistent overlap buffers), and an encode is ~1 µs of
// host time per map (2 x passes maps per GEMM launch).
struct MapCacheEntry {
    const void *base = nullptr;
    size_t bytes = 0;
    uint32_t box = 0;
    CUtensorMap map;
};
thread_local MapCacheEntry t_maps[32];
thread_local unsigned t_maps_next = 0;

int rows_map(CUtensorMap *m, const void *base, size_t bytes, uint32_t box_rows) {
    for (const MapCacheEntry &c : t_maps)
        if (c.base == base && c.bytes == bytes && c.box == box_rows) {
            *m = c.map;
            return 0;
        }
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(OZAKI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    cuuint64_t dims[2] = {256, (cuuint64_t)(bytes / 256)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {256, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(OZAKI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    MapCacheEntry &c = t_maps[t_maps_next++ % 32];
    c.base = base;
    c.bytes = bytes;
    c.box = box_rows;
    c.map = *m;
    return 0;
}

template <int EPI, int CHUNK = 0, bool FULL = false, bool GAB = true>
int launch_gemm_lv2(const Plan &P, const GemmParams &gp, size_t a_avail, size_t b_avail, DevState *dev,
                    cudaStream_t st) {
    CUDA_TRY(smem_optin((const void *)k_gemm_lv2<EPI, CHUNK, FULL, GAB>, P.smem));
    Lv2Params P2;
    std::memset(&P2, 0, sizeof P2);
    P2.lv.g = gp;
    P2.lv.npass = P.npass;
    P2.lv.stage_bytes = P.stage_bytes;
    for (int q = 0; q < P.npass; ++q) {
        P2.lv.pass[q] = P.pass[q];
        if (int rc = rows_map(&P2.tmA[q], gp.A, a_avail, (uint32_t)P.pass[q].n * (kBlk / 256))) return rc;
        if (int rc = rows_map(&P2.tmB[q], gp.B, b_avail, (uint32_t)P.pass[q].n * (kBlk / 512))) return rc;
    }
    const int64_t tiles = gp.batch * gp.tiles_m * gp.tiles_n * gp.splitk;   // work units
    const unsigned pairs = (unsigned)std::min<int64_t>(tiles, dev->sms / 2);
    {
        ProfScope ps(st, PH_GEMM);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(kThreads2);
        cfg.dynamicSmemBytes = P.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlap K1's tail
        attr[0].val.programmaticStreamSerializationAllowed = ozenv("OZAKI_NO_PDL") ? 0 : 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_TRY(cudaLaunchKernelEx(&cfg, k_gemm_lv2<EPI, CHUNK, FULL, GAB>, P2));
    }
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    return 0;
}

template <int BN, int EPI>
int launch_gemm_t(const Plan &P, const GemmParams &gp, DevState *dev, cudaStream_t st) {
    if (int rc = set_gemm_attr<BN, EPI>(P.smem)) return rc;
    const int64_t tiles = P.batch * P.tiles_m * P.tiles_n;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, dev->sms);
    {
        ProfScope ps(st, PH_GEMM);
        k_gemm<BN, EPI><<<grid, kGemmThreads, P.smem, st>>>(gp);
    }
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    return 0;
}

// K-chunked GEMM (reading R8): per batch entry, per column panel (W <= 2 GiB),
// per K chunk (s * chunk_K' <= 131071): chunk 1 writes the exact INT32 partial
// level sums into W (FP64, exact), middle chunks add, the last chunk adds its
// own partial in the epilogue and runs the normal FP64 combine + alpha/beta.
int launch_gemm_chunked(const Plan &P, const GemmParams &g0, int epi, int64_t kc_env, DevState *dev,
                        cudaStream_t st) {
    const int s = P.s;
    int64_t kbc = 131071 / (32 * (int64_t)s);          // k-blocks per chunk
    if (kc_env > 0) kbc = std::min<int64_t>(kbc, kc_env);
    if (kbc < 1) return fail(OZAKI_ERR_UNSUPPORTED, "K chunk too small");
    const int64_t nchunk = (P.KB + kbc - 1) / kbc;
    const int64_t Np = P.Np, Mp = P.Mp;
    int64_t panel = ((int64_t)2 << 30) / ((int64_t)s * Mp * 8);
    panel = std::max<int64_t>(kLvBN, panel / kLvBN * kLvBN);
    panel = std::min<int64_t>(panel, P.tiles_n * kLvBN);
    if (const char *pe = ozenv("OZAKI_PANEL_COLS"))     // test hook: force narrow panels
        panel = std::max<int64_t>(kLvBN, std::min<int64_t>(panel, atoll(pe) / kLvBN * kLvBN));
    double *W = nullptr;
    const size_t wbytes = (size_t)s * Mp * panel * sizeof(double);
    cudaError_t e = cudaMallocAsync((void **)&W, wbytes, st);
    if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "K-chunk workspace (%zu B): %s", wbytes, cudaGetErrorString(e));
    const size_t a_tile_bytes = (size_t)P.KB * s * kBlk;            // one 128-row A tile
    const size_t b_tile_bytes = (size_t)P.KB * s * (kBlk / 2);      // one 64-row B tile
    int rc = 0;
    for (int64_t b = 0; b < P.batch && !rc; ++b) {
        for (int64_t j0 = 0; j0 < Np && !rc; j0 += panel) {
            const int64_t nw = std::min<int64_t>(panel, Np - j0);
            GemmParams gp = g0;
            gp.batch = 1;
            gp.A = g0.A + (size_t)b * (2 * P.tiles_m) * a_tile_bytes;
            gp.B = g0.B + ((size_t)b * (2 * P.tiles_n) + 2 * (j0 / kLvBN)) * b_tile_bytes;
            gp.ea = g0.ea + b * Mp;
            gp.fb = g0.fb + b * Np + j0;
            gp.N = nw;
            gp.tiles_n = (nw + kLvBN - 1) / kLvBN;
            gp.C = (epi == EPI_CPLX4M) ? g0.C + 2 * (b * g0.strideC + (j0 / 2) * g0.ldc)
                                       : g0.C + b * g0.strideC + j0 * g0.ldc;
            gp.W = W;
            gp.w_lvl = Mp * nw;
            const size_t a_avail = (size_t)P.a_bytes - (size_t)(gp.A - g0.A);
            const size_t b_avail = (size_t)P.b_bytes - (size_t)(gp.B - g0.B);
            for (int64_t c = 0; c < nchunk && !rc; ++c) {
                gp.kb_begin = c * kbc;
                gp.kb_end = std::min<int64_t>(P.KB, (c + 1) * kbc);
                gp.chunk_mode = (nchunk == 1) ? 0 : (c == 0 ? 1 : (c + 1 == nchunk ? 3 : 2));
                if (gp.chunk_mode == 0)
                    rc = (epi == EPI_REAL) ? launch_gemm_lv2<EPI_REAL, 0>(P, gp, a_avail, b_avail, dev, st)
                                           : launch_gemm_lv2<EPI_CPLX4M, 0>(P, gp, a_avail, b_avail, dev, st);
                else if (gp.chunk_mode != 3)   // partial chunks store nothing to C: one kernel
                    rc = launch_gemm_lv2<EPI_REAL, 1>(P, gp, a_avail, b_avail, dev, st);
                else
                    rc = (epi == EPI_REAL) ? launch_gemm_lv2<EPI_REAL, 2>(P, gp, a_avail, b_avail, dev, st)
                                           : launch_gemm_lv2<EPI_CPLX4M, 2>(P, gp, a_avail, b_avail, dev, st);
                if (!rc && nchunk > 1) g_stats.chunks += 1;
            }
        }
    }
    cudaFreeAsync(W, st);
    return rc;
}

// Split-K launch: one GEMM over tiles x S units writing exact partials (CHUNK 3), then
// k_splitk_combine (PDL: its launch overlaps the GEMM's tail) sums them and stores C.
int launch_gemm_splitk(const Plan &P, GemmParams gp, int epi, int64_t *P0, int32_t *PL, DevState *dev,
                       cudaStream_t st) {
    gp.splitk = P.splitk;
    gp.pk_nl = P.pk_nl;
    gp.P0 = P0;
    gp.PL = PL;
    int rc = P.full ? launch_gemm_lv2<EPI_REAL, 3, true>(P, gp, P.a_bytes, P.b_bytes, dev, st)
                    : launch_gemm_lv2<EPI_REAL, 3, false>(P, gp, P.a_bytes, P.b_bytes, dev, st);
    if (rc) return rc;
    const int Lmax = P.full ? 2 * P.s : P.s + 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((P.Np + 1) / 2), (unsigned)((P.Mp + 127) / 128), (unsigned)P.batch);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = ozenv("OZAKI_NO_PDL") ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    {
        ProfScope ps(st, PH_OTHER);
        if (epi == EPI_CPLX4M)
            CUDA_TRY(cudaLaunchKernelEx(&cfg, k_splitk_combine<EPI_CPLX4M>, gp, Lmax, P.pk_np));
        else
            CUDA_TRY(cudaLaunchKernelEx(&cfg, k_splitk_combine<EPI_REAL>, gp, Lmax, P.pk_np));
    }
    g_stats.launches += 1;
    return 0;
}

int launch_gemm(const Plan &P, int epi, const int8_t *sa, const int8_t *sb, const int32_t *ea,
                const int32_t *fb, double *C, int64_t ldc, int64_t strideC, const double al[2],
                const double be[2], int32_t *S_out, DevState *dev, cudaStream_t st,
                int64_t *P0 = nullptr, int32_t *PL = nullptr) {
    GemmParams gp{};
    gp.splitk = 1;
    gp.A = sa;
    gp.B = sb;
    gp.ea = ea;
    gp.fb = fb;
    gp.Mp = P.Mp;
    gp.N = P.Np;
    gp.KB = P.KB;
    gp.tiles_m = P.tiles_m;
    gp.tiles_n = P.tiles_n;
    gp.batch = P.batch;
    gp.s = P.s;
    gp.kps = P.kps;
    gp.stages = P.stages;
    gp.a_kb_bytes = (uint32_t)(P.s * kBM * kKB);
    gp.b_kb_bytes = (uint32_t)(P.s * P.BN * kKB);
    gp.C = C;
    gp.ldc = ldc;
    gp.strideC = strideC;
    gp.alpha_r = al[0];
    gp.alpha_i = al[1];
    gp.beta_r = be[0];
    gp.beta_i = be[1];
    gp.ab_unit = (al[0] == 1.0 && al[1] == 0.0 && be[0] == 0.0 && be[1] == 0.0) ? 1 : 0;
    gp.S_out = S_out;
    gp.kb_begin = 0;
    gp.kb_end = P.KB;
    gp.chunk_mode = 0;
    gp.W = nullptr;
    gp.w_lvl = 0;
    if (g_dbg_on.load()) {
        if (!g_dbg) {
            CUDA_TRY(cudaMalloc(&g_dbg, sizeof(unsigned long long) * DBG_NSLOT));
            CUDA_TRY(cudaMemset(g_dbg, 0, sizeof(unsigned long long) * DBG_NSLOT));
        }
        gp.dbg = g_dbg;
    }
    if (P.pair) {
        const char *ev = ozenv("OZAKI_KCHUNK_KB");   // test hook: force a small K chunk
        const int64_t kc_env = ev ? atoll(ev) : 0;
        if ((P.kchunk_needed || kc_env > 0) && epi != EPI_LEVELS)
            return launch_gemm_chunked(P, gp, epi, kc_env, dev, st);
        if (P.splitk > 1 && epi != EPI_LEVELS && P0 && PL)
            return launch_gemm_splitk(P, gp, epi, P0, PL, dev, st);
        if (P.full) {   // R21: all s^2 pairs (planned only without K-chunking)
            if (epi == EPI_REAL) return launch_gemm_lv2<EPI_REAL, 0, true>(P, gp, P.a_bytes, P.b_bytes, dev, st);
            if (epi == EPI_CPLX4M) return launch_gemm_lv2<EPI_CPLX4M, 0, true>(P, gp, P.a_bytes, P.b_bytes, dev, st);
            return launch_gemm_lv2<EPI_LEVELS, 0, true>(P, gp, P.a_bytes, P.b_bytes, dev, st);
        }
        // beta == 0 (C not read): the kernels without the general alpha / beta store
        const bool gab = !(be[0] == 0.0 && be[1] == 0.0);
        if (epi == EPI_REAL)
            return gab ? launch_gemm_lv2<EPI_REAL, 0, false, true>(P, gp, P.a_bytes, P.b_bytes, dev, st)
                       : launch_gemm_lv2<EPI_REAL, 0, false, false>(P, gp, P.a_bytes, P.b_bytes, dev, st);
        if (epi == EPI_CPLX4M)
            return gab ? launch_gemm_lv2<EPI_CPLX4M, 0, false, true>(P, gp, P.a_bytes, P.b_bytes, dev, st)
                       : launch_gemm_lv2<EPI_CPLX4M, 0, false, false>(P, gp, P.a_bytes, P.b_bytes, dev, st);
        return launch_gemm_lv2<EPI_LEVELS>(P, gp, P.a_bytes, P.b_bytes, dev, st);
    }
    if (P.lv) {
        if (epi == EPI_REAL) return launch_gemm_lv<EPI_REAL>(P, gp, dev, st);
        if (epi == EPI_CPLX4M) return launch_gemm_lv<EPI_CPLX4M>(P, gp, dev, st);
        return launch_gemm_lv<EPI_LEVELS>(P, gp, dev, st);
    }
    if (P.BN == 64) {
        if (epi == EPI_REAL) return launch_gemm_t<64, EPI_REAL>(P, gp, dev, st);
        if (epi == EPI_CPLX4M) return launch_gemm_t<64, EPI_CPLX4M>(P, gp, dev, st);
        return launch_gemm_t<64, EPI_LEVELS>(P, gp, dev, st);
    }
    if (epi == EPI_REAL) return launch_gemm_t<32, EPI_REAL>(P, gp, dev, st);
    if (epi == EPI_CPLX4M) return launch_gemm_t<32, EPI_CPLX4M>(P, gp, dev, st);
    return launch_gemm_t<32, EPI_LEVELS>(P, gp, dev, st);
}

// Views of op(A) rows / op(B) columns over column-major storage.
Operand view_A(const double *A, char ta, int64_t m, int64_t k, int64_t lda, int64_t strideA,
               int mode) {
    Operand o{};
    o.X = A;
    o.rows = m;
    o.k = k;
    o.bstride = strideA;
    o.mode = mode;
    if (ta == 'N') {   // row i of A: A[i + l*lda]
        o.rs = 1;
        o.ls = lda;
    } else {           // row i of A^T: column i of A
        o.rs = lda;
        o.ls = 1;
        o.conj = (ta == 'C' && mode != SPLIT_REAL) ? 1 : 0;
    }
    return o;
}

Operand view_B(const double *B, char tb, int64_t n, int64_t k, int64_t ldb, int64_t strideB,
               int mode) {
    Operand o{};
    o.X = B;
    o.rows = n;
    o.k = k;
    o.bstride = strideB;
    o.mode = mode;
    if (tb == 'N') {   // column j of B: B[l + j*ldb]
        o.rs = ldb;
        o.ls = 1;
    } else {           // column j of B^T: row j of B
        o.rs = 1;
        o.ls = ldb;
        o.conj = (tb == 'C' && mode != SPLIT_REAL) ? 1 : 0;
    }
    return o;
}

bool overlaps(const void *a, size_t abytes, const void *b, size_t bbytes) {
    const char *x = (const char *)a, *y = (const char *)b;
    return abytes && bbytes && x < y + bbytes && y < x + abytes;
}

// Exact element overlap of two column-major views X (xr x xc, ld) and C (cr x cc, ld)
// of the SAME leading dimension (e.g. sub-blocks of one LAPACK-style array, where the
// byte spans interleave but the elements are disjoint).  Different leading dimensions
// or misaligned bases: conservatively "overlap".
bool elems_overlap(const void *x, int64_t xr, int64_t xc, int64_t ldx, const void *cp, int64_t cr, int64_t cc,
                   int64_t ldc, size_t es) {
    if (xr == 0 || xc == 0 || cr == 0 || cc == 0) return false;
    if (ldx != ldc) return true;
    const int64_t diff = (const char *)cp - (const char *)x;
    if (diff % (int64_t)es) return true;
    const int64_t ld = ldx, d = diff / (int64_t)es;
    int64_t dc = d / ld, dr = d % ld;                   // C(0,0) sits at X(dr, dc) of the ld-grid
    if (dr < 0) { dr += ld; dc -= 1; }
    auto meet = [](int64_t a0, int64_t a1, int64_t b0, int64_t b1) { return a0 < b1 && b0 < a1; };
    // C rows i' with dr + i' < ld land in grid rows dr + i' of columns dc + j'
    const int64_t r1 = std::min(cr, ld - dr);
    if (r1 > 0 && meet(dr, dr + r1, 0, xr) && meet(dc, dc + cc, 0, xc)) return true;
    // C rows wrapping past ld land in rows dr + i' - ld of columns dc + j' + 1
    if (cr > ld - dr && meet(0, dr + cr - ld, 0, xr) && meet(dc + 1, dc + cc + 1, 0, xc)) return true;
    return false;
}

size_t span_bytes(int64_t rows, int64_t cols, int64_t ld, int64_t stride, int64_t batch, size_t es) {
    if (rows == 0 || cols == 0 || batch == 0) return 0;
    return es * (size_t)((batch - 1) * stride + (cols - 1) * ld + rows);
}

struct Call {
    Kind kind;
    char ta, tb;
    int64_t m, n, k;
    double al[2], be[2];
    const double *A;
    int64_t lda, sA;
    const double *B;
    int64_t ldb, sB;
    double *C;
    int64_t ldc, sC, batch;
    int s;            // Ozaki-I: slices; Ozaki-II (crt): moduli count
    bool batched;
    int32_t *S_out;   // debug level dump (real only)
    bool crt;         // Ozaki-II (NEXT-1)
    bool full;        // Ozaki-I full pair set (R21, NEXT-4)
    int64_t kblock;   // R22 per-block exponents (0: per row / column)
};

int validate(const Call &c) {
    const bool b = c.batched;
    if (!trans_ok(c.ta)) return fail(-1, "transa");
    if (!trans_ok(c.tb)) return fail(-2, "transb");
    if (c.m < 0) return fail(-3, "m < 0");
    if (c.n < 0) return fail(-4, "n < 0");
    if (c.k < 0) return fail(-5, "k < 0");
    const char ta = up(c.ta), tb = up(c.tb);
    if (c.lda < std::max<int64_t>(1, ta == 'N' ? c.m : c.k)) return fail(-8, "lda too small");
    if (b && c.sA < 0) return fail(-9, "strideA < 0");
    if (c.ldb < std::max<int64_t>(1, tb == 'N' ? c.k : c.n)) return fail(b ? -11 : -10, "ldb too small");
    if (b && c.sB < 0) return fail(-12, "strideB < 0");
    if (c.ldc < std::max<int64_t>(1, c.m)) return fail(b ? -15 : -13, "ldc too small");
    if (b && c.sC < 0) return fail(-16, "strideC < 0");
    if (b && c.batch < 0) return fail(-17, "batch < 0");
    if (!c.crt && (c.s < 1 || c.s > 16)) return fail(b ? -18 : -14, "num_slices not in [1,16]");
    if (c.crt && (c.s < 1 || c.s > kMaxModuli)) return fail(b ? -18 : -14, "num_moduli not in [1,20]");
    return 0;
}

int run(const Call &c0);

// ------------------------------------------------------------ host offload
// A, B, C in host memory (pinned or pageable): the library stages batch
// chunks through device buffers on three internal streams so H2D copies,
// the emulated GEMM and D2H copies overlap (chunk i+1 in, i computing, i-1
// out), and returns when C is back in host memory.  This is the analogue of
// the automatic BLAS offload the paper relies on.
enum PtrKind { PTR_DEVICE = 0, PTR_HOST = 1, PTR_BAD = 2 };

PtrKind ptr_kind(const void *p) {
    if (!p) return PTR_DEVICE;   // only reached for empty operands
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return PTR_HOST;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return PTR_DEVICE;
    return PTR_HOST;   // cudaMemoryTypeHost (pinned) or cudaMemoryTypeUnregistered (pageable)
}

struct OffloadCtx {
    bool init = false;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t in_done[2] = {}, comp_done[2] = {}, out_done[2] = {}, start = nullptr;
    char *buf[2] = {nullptr, nullptr};   // staging buffer sets, cached across calls
    size_t cap = 0;
    char *blk = nullptr;                 // one-GEMM 2-D block staging (op(A), op(B), C), cached
    size_t blk_cap = 0;
};
thread_local OffloadCtx t_off[kMaxDev];

int offload_ctx(OffloadCtx **out) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    OffloadCtx &o = t_off[dev];
    if (!o.init) {
        CUDA_TRY(cudaStreamCreateWithFlags(&o.h2d, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&o.comp, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&o.d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaEventCreateWithFlags(&o.in_done[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&o.comp_done[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&o.out_done[i], cudaEventDisableTiming));
        }
        CUDA_TRY(cudaEventCreateWithFlags(&o.start, cudaEventDisableTiming));
        o.init = true;
    }
    *out = &o;
    return 0;
}

// One large GEMM on host pointers (batch == 1), in 2-D blocks: op(A) moves in row blocks and
// op(B) in column blocks, each ONCE (they stay resident), and block (i, j) of C is computed as
// soon as A_i and B_j have arrived, so the D2H copies of C start after the first block instead
// of after all of op(A) (PCIe runs both directions at once).  Order: A_0, B_0, B_1, ..., then
// A_1, A_2, ...  Row exponents come from full rows of op(A) and column exponents are per column,
// so every element is computed exactly as by one call (bitwise).
int run_offload_blocks(const Call &c, int64_t rb, int64_t cb) {
    const size_t es = (c.kind == KIND_REAL) ? 8 : 16;
    const int64_t ew = (c.kind == KIND_REAL) ? 1 : 2;      // doubles per element
    const bool an = c.ta == 'N', bn = c.tb == 'N';
    const int64_t ar = an ? c.m : c.k, br = bn ? c.k : c.n;  // device leading dimensions (packed)
    const bool readC = !(c.be[0] == 0.0 && c.be[1] == 0.0);
    const int64_t I = (c.m + rb - 1) / rb, J = (c.n + cb - 1) / cb;
    OffloadCtx *o = nullptr;
    if (int rc = offload_ctx(&o)) return rc;
    const size_t abytes = al256((size_t)c.m * c.k * es), bbytes = al256((size_t)c.k * c.n * es);
    const size_t need = abytes + bbytes + (size_t)c.m * c.n * es;
    if (o->blk_cap < need) {
        CUDA_TRY(cudaStreamSynchronize(o->d2h));
        CUDA_TRY(cudaStreamSynchronize(o->comp));
        if (o->blk) cudaFree(o->blk);
        o->blk = nullptr;
        o->blk_cap = 0;
        cudaError_t e = cudaMalloc(&o->blk, need);
        if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "offload staging (%zu B): %s", need, cudaGetErrorString(e));
        o->blk_cap = need;
    }
    double *dA = (double *)o->blk;
    double *dB = (double *)(o->blk + abytes);
    double *dC = (double *)(o->blk + abytes + bbytes);
    // events: released on every path (RAII), after the streams are drained
    struct Events {
        std::vector<cudaEvent_t> v;
        ~Events() {
            for (auto &x : v)
                if (x) cudaEventDestroy(x);
        }
    } evs;
    evs.v.assign((size_t)(I + J + 2 * I * J), nullptr);
    std::vector<cudaEvent_t> &ev = evs.v;
    for (auto &x : ev) CUDA_TRY(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    cudaEvent_t *a_done = ev.data(), *b_done = a_done + I, *in_done = b_done + J, *cmp_done = in_done + I * J;
    cudaStream_t user = t_stream;
    CUDA_TRY(cudaEventRecord(o->start, user));
    CUDA_TRY(cudaStreamWaitEvent(o->h2d, o->start, 0));
    auto copy_a = [&](int64_t i) -> int {   // op(A) rows [i0, i1)
        const int64_t i0 = i * rb, h = std::min<int64_t>(rb, c.m - i0);
        if (an)
            CUDA_TRY(cudaMemcpy2DAsync(dA + ew * i0, ar * es, (const char *)c.A + i0 * es, c.lda * es, h * es, c.k,
                                       cudaMemcpyHostToDevice, o->h2d));
        else
            CUDA_TRY(cudaMemcpy2DAsync(dA + ew * i0 * ar, ar * es, (const char *)c.A + i0 * c.lda * es, c.lda * es,
                                       c.k * es, h, cudaMemcpyHostToDevice, o->h2d));
        CUDA_TRY(cudaEventRecord(a_done[i], o->h2d));
        return 0;
    };
    auto copy_b = [&](int64_t j) -> int {   // op(B) columns [j0, j1)
        const int64_t j0 = j * cb, w = std::min<int64_t>(cb, c.n - j0);
        if (bn)
            CUDA_TRY(cudaMemcpy2DAsync(dB + ew * j0 * br, br * es, (const char *)c.B + j0 * c.ldb * es, c.ldb * es,
                                       c.k * es, w, cudaMemcpyHostToDevice, o->h2d));
        else
            CUDA_TRY(cudaMemcpy2DAsync(dB + ew * j0, br * es, (const char *)c.B + j0 * es, c.ldb * es, w * es, c.k,
                                       cudaMemcpyHostToDevice, o->h2d));
        CUDA_TRY(cudaEventRecord(b_done[j], o->h2d));
        return 0;
    };
    int rc = 0;
    for (int64_t i = 0; i < I && !rc; ++i) {
        rc = copy_a(i);
        for (int64_t j = 0; j < J && !rc; ++j) {
            if (i == 0 && (rc = copy_b(j))) break;
            const int64_t i0 = i * rb, h = std::min<int64_t>(rb, c.m - i0);
            const int64_t j0 = j * cb, w = std::min<int64_t>(cb, c.n - j0);
            double *dCij = dC + ew * (i0 + j0 * c.m);
            char *hC = (char *)c.C + (i0 + j0 * c.ldc) * es;
            const int64_t q = i * J + j;
            if (readC) {
                CUDA_TRY(cudaMemcpy2DAsync(dCij, c.m * es, hC, c.ldc * es, h * es, w, cudaMemcpyHostToDevice, o->h2d));
                CUDA_TRY(cudaEventRecord(in_done[q], o->h2d));
                CUDA_TRY(cudaStreamWaitEvent(o->comp, in_done[q], 0));
            }
            CUDA_TRY(cudaStreamWaitEvent(o->comp, a_done[i], 0));
            CUDA_TRY(cudaStreamWaitEvent(o->comp, b_done[j], 0));
            Call d = c;
            d.A = dA + ew * (an ? i0 : i0 * ar);
            d.lda = ar;
            d.B = dB + ew * (bn ? j0 * br : j0);
            d.ldb = br;
            d.C = dCij;
            d.ldc = c.m;
            d.m = h;
            d.n = w;
            d.sA = d.sB = d.sC = 0;
            t_stream = o->comp;
            const int ovs = t_overlap;
            t_overlap = 0;
            rc = run(d);
            t_overlap = ovs;
            t_stream = user;
            if (rc) break;
            CUDA_TRY(cudaEventRecord(cmp_done[q], o->comp));
            CUDA_TRY(cudaStreamWaitEvent(o->d2h, cmp_done[q], 0));
            CUDA_TRY(cudaMemcpy2DAsync(hC, c.ldc * es, dCij, c.m * es, h * es, w, cudaMemcpyDeviceToHost, o->d2h));
        }
    }
    cudaEventRecord(o->start, o->d2h);
    cudaStreamWaitEvent(user, o->start, 0);
    cudaError_t e = cudaStreamSynchronize(o->d2h);
    cudaStreamSynchronize(o->comp);
    cudaStreamSynchronize(o->h2d);
    if (!rc && e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "offload: %s", cudaGetErrorString(e));
    return rc;
}

int run_offload(const Call &c) {
    const size_t es = (c.kind == KIND_REAL) ? 8 : 16;
    const int64_t ar = c.ta == 'N' ? c.m : c.k, ac = c.ta == 'N' ? c.k : c.m;
    const int64_t br = c.tb == 'N' ? c.k : c.n, bc = c.tb == 'N' ? c.n : c.k;
    // A and B are read only when alpha != 0 and k > 0 (else the quick return C = beta C runs on
    // the staged C alone)
    const bool readsAB = !(c.al[0] == 0.0 && c.al[1] == 0.0) && c.k > 0;
    // element span of one entry (leading dimensions kept as given); C moves as m x n with pitch
    // ldc (cudaMemcpy2DAsync), so the rows m..ldc-1 of the caller's array are never written
    const int64_t spanA = readsAB ? (ac - 1) * c.lda + ar : 0, spanB = readsAB ? (bc - 1) * c.ldb + br : 0;
    const int64_t spanC = (c.n - 1) * c.ldc + c.m;
    const bool readC = !(c.be[0] == 0.0 && c.be[1] == 0.0);
    const size_t per_entry = (size_t)(spanA + spanB + spanC) * es;
    size_t chunk_bytes = 32ull << 20;   // ~32 MB per chunk (measured best: 5.6 vs 5.9 ms for C2x30; OZAKI_OFFLOAD_CHUNK_MB overrides)
    if (const char *ce = ozenv("OZAKI_OFFLOAD_CHUNK_MB")) {
        const long long v = atoll(ce);
        if (v >= 1 && v <= 4096) chunk_bytes = (size_t)v << 20;
    }
    int64_t cb = (int64_t)(chunk_bytes / std::max<size_t>(per_entry, 1));
    cb = std::max<int64_t>(1, std::min<int64_t>(cb, (c.batch + 1) / 2 > 0 ? (c.batch + 1) / 2 : 1));
    const int64_t nchunk = (c.batch + cb - 1) / cb;
    OffloadCtx *o = nullptr;
    if (int rc = offload_ctx(&o)) return rc;
    cudaStream_t user = t_stream;
    const size_t set_bytes = (size_t)cb * per_entry;
    if (o->cap < set_bytes) {   // grow the cached staging sets (never freed per call: cudaFree syncs)
        CUDA_TRY(cudaStreamSynchronize(o->d2h));
        for (int i = 0; i < 2; ++i) {
            if (o->buf[i]) cudaFree(o->buf[i]);
            o->buf[i] = nullptr;
        }
        o->cap = 0;
        for (int i = 0; i < 2; ++i) {
            cudaError_t e = cudaMalloc(&o->buf[i], set_bytes);
            if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "offload staging (%zu B): %s", set_bytes, cudaGetErrorString(e));
        }
        o->cap = set_bytes;
    }
    char *buf[2] = {o->buf[0], o->buf[1]};
    CUDA_TRY(cudaEventRecord(o->start, user));
    CUDA_TRY(cudaStreamWaitEvent(o->h2d, o->start, 0));
    int rc = 0;
    const char *hA = (const char *)c.A, *hB = (const char *)c.B;
    char *hC = (char *)c.C;
    for (int64_t ch = 0; ch < nchunk && !rc; ++ch) {
        const int set = (int)(ch & 1);
        const int64_t b0 = ch * cb, nb = std::min<int64_t>(cb, c.batch - b0);
        double *dA = (double *)buf[set];
        double *dB = (double *)(buf[set] + (size_t)cb * spanA * es);
        double *dC = (double *)(buf[set] + (size_t)cb * (spanA + spanB) * es);
        if (ch >= 2) CUDA_TRY(cudaStreamWaitEvent(o->h2d, o->out_done[set], 0));   // buffer set reuse
        for (int64_t i = 0; i < nb; ++i) {
            if (readsAB) {
                CUDA_TRY(cudaMemcpyAsync((char *)dA + (size_t)i * spanA * es, hA + (size_t)(b0 + i) * c.sA * es,
                                         (size_t)spanA * es, cudaMemcpyHostToDevice, o->h2d));
                CUDA_TRY(cudaMemcpyAsync((char *)dB + (size_t)i * spanB * es, hB + (size_t)(b0 + i) * c.sB * es,
                                         (size_t)spanB * es, cudaMemcpyHostToDevice, o->h2d));
            }
            if (readC)
                CUDA_TRY(cudaMemcpy2DAsync((char *)dC + (size_t)i * spanC * es, (size_t)c.ldc * es,
                                           hC + (size_t)(b0 + i) * c.sC * es, (size_t)c.ldc * es,
                                           (size_t)c.m * es, (size_t)c.n, cudaMemcpyHostToDevice, o->h2d));
        }
        CUDA_TRY(cudaEventRecord(o->in_done[set], o->h2d));
        CUDA_TRY(cudaStreamWaitEvent(o->comp, o->in_done[set], 0));
        Call d = c;
        d.A = dA;
        d.B = dB;
        d.C = dC;
        d.sA = spanA;
        d.sB = spanB;
        d.sC = spanC;
        d.batch = nb;
        d.batched = true;
        t_stream = o->comp;
        const int ovs = t_overlap;
        t_overlap = 0;   // chunks are separated by event waits on the staging copies
        rc = run(d);
        t_overlap = ovs;
        t_stream = user;
        if (rc) break;
        CUDA_TRY(cudaEventRecord(o->comp_done[set], o->comp));
        CUDA_TRY(cudaStreamWaitEvent(o->d2h, o->comp_done[set], 0));
        for (int64_t i = 0; i < nb; ++i)
            CUDA_TRY(cudaMemcpy2DAsync(hC + (size_t)(b0 + i) * c.sC * es, (size_t)c.ldc * es,
                                       (char *)dC + (size_t)i * spanC * es, (size_t)c.ldc * es,
                                       (size_t)c.m * es, (size_t)c.n, cudaMemcpyDeviceToHost, o->d2h));
        CUDA_TRY(cudaEventRecord(o->out_done[set], o->d2h));
    }
    // the caller's stream observes completion; host memory is final on return
    cudaEventRecord(o->start, o->d2h);
    cudaStreamWaitEvent(user, o->start, 0);
    cudaError_t e = cudaStreamSynchronize(o->d2h);
    if (!rc && e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "offload: %s", cudaGetErrorString(e));
    return rc;
}

// ============================================================ Ozaki-II (NEXT-1)
// Host tables of reading R16..R20: the greedy moduli, the per-modulus
// reduction constants of crt.cuh and the CRT weights W_q = (M/p_q) inv_q as
// 32-bit limbs (exact multi-limb arithmetic on the host).
struct CrtHost {
    bool ready = false;
    int n = 0, L = 0, bitlen = 0;
    CrtTab tab{};
    uint32_t W[kMaxModuli][kCrtLimbs]{};
    uint32_t M[kCrtLimbs + 1]{};
    uint32_t Mhalf[kCrtLimbs]{};
    double Minv = 0.0;
};
CrtHost g_crt[kMaxModuli + 1];
std::mutex g_crt_mu;

int gcd_i(int a, int b) {
    while (b) {
        const int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

const CrtHost &crt_tables(int n) {
    std::lock_guard<std::mutex> lk(g_crt_mu);
    CrtHost &h = g_crt[n];
    if (h.ready) return h;
    // R16: 256, then the largest integers coprime to all chosen
    std::vector<int> mods{256};
    for (int c = 255; (int)mods.size() < n && c >= 2; --c) {
        bool ok = true;
        for (int q : mods) ok = ok && gcd_i(c, q) == 1;
        if (ok) mods.push_back(c);
    }
    h.n = n;
    h.tab.n = n;
    // M = prod p_q, little-endian 32-bit limbs
    uint32_t M[kCrtLimbs + 1] = {1};
    for (int q = 0; q < n; ++q) {
        uint64_t carry = 0;
        for (int l = 0; l <= kCrtLimbs; ++l) {
            const uint64_t t = (uint64_t)M[l] * (uint32_t)mods[q] + carry;
            M[l] = (uint32_t)t;
            carry = t >> 32;
        }
    }
    int top = kCrtLimbs;
    while (top > 0 && M[top] == 0) --top;
    h.bitlen = 32 * top + (32 - __builtin_clz(M[top]));
    h.L = (h.bitlen + 31) / 32;
    std::memcpy(h.M, M, sizeof M);
    for (int l = 0; l < kCrtLimbs; ++l) h.Mhalf[l] = (M[l] >> 1) | (l + 1 <= kCrtLimbs ? (M[l + 1] << 31) : 0u);
    double md = 0.0;
    for (int l = kCrtLimbs; l >= 0; --l) md = md * 4294967296.0 + (double)M[l];
    h.Minv = 1.0 / md;
    for (int q = 0; q < n; ++q) {
        const uint32_t p = (uint32_t)mods[q];
        // Mq = M / p (exact), r = Mq mod p, inv = r^-1 mod p, W = Mq * inv (< M)
        uint32_t Mq[kCrtLimbs + 1];
        uint64_t rem = 0;
        for (int l = kCrtLimbs; l >= 0; --l) {
            const uint64_t cur = (rem << 32) | M[l];
            Mq[l] = (uint32_t)(cur / p);
            rem = cur % p;
        }
        uint64_t r = 0;
        for (int l = kCrtLimbs; l >= 0; --l) r = ((r << 32) | Mq[l]) % p;
        uint32_t inv = 0;
        for (uint32_t x = 1; x < p; ++x)
            if ((r * x) % p == 1) {
                inv = x;
                break;
            }
        if (p == 1) inv = 0;
        uint64_t carry = 0;
        for (int l = 0; l < kCrtLimbs; ++l) {
            const uint64_t t = (uint64_t)Mq[l] * inv + carry;
            h.W[q][l] = (uint32_t)t;
            carry = t >> 32;
        }
        h.tab.p[q] = p;
        h.tab.c21[q] = (uint32_t)((1ull << 21) % p);
        h.tab.c42[q] = (uint32_t)((1ull << 42) % p);
        h.tab.c16[q] = (uint32_t)((1ull << 16) % p);
        h.tab.bias28[q] = (uint32_t)(((1ull << 28) + p - 1) / p * p);
        h.tab.bias23[q] = (uint32_t)(((1ull << 23) + p - 1) / p * p);
        h.tab.m39[q] = (uint32_t)(((1ull << 39) + p - 1) / p);
    }
    h.ready = true;
    return h;
}

// R17: nu = min(62, largest nu with 2^(2 nu + ceil(log2 k_eff) + 1) <= M), and
// 2^x <= M  <=>  x <= bitlen(M) - 1.
int crt_nu(const CrtHost &h, int64_t keff) {
    int c = 0;
    while ((1ll << c) < keff) ++c;
    int nu = 0;
    while (2 * (nu + 1) + c + 1 <= h.bitlen - 1) ++nu;
    return std::min(nu, 62);
}

// K1' for Ozaki-II through k_split_fast<…, CRT>: both operands in one launch, 128-row tiles on
// both sides, the moduli word count compile-time (n rounded up to a multiple of 4).  Returns 1
// when OZAKI_SPLIT=generic asks for the generic k_split_sm form.
template <int NMX>
void launch_crt_fast(bool real, bool lng, dim3 grid, size_t smem, cudaStream_t st, const SplitPair &pp, int KW,
                     int nwin) {
#define OZK_CRT_K(MA, MB, R, L)                                                                      \
    {                                                                                                \
        smem_optin((const void *)k_split_fast<NMX, MA, MB, R, L, true>, smem);                       \
        k_split_fast<NMX, MA, MB, R, L, true><<<grid, 32 * R, smem, st>>>(pp, KW, nwin, 0);          \
    }
    if (real) {
        if (lng) OZK_CRT_K(SPLIT_REAL, SPLIT_REAL, 16, true) else OZK_CRT_K(SPLIT_REAL, SPLIT_REAL, 4, false)
    } else {
        if (lng) OZK_CRT_K(SPLIT_A4M, SPLIT_B4M, 8, true) else OZK_CRT_K(SPLIT_A4M, SPLIT_B4M, 4, false)
    }
#undef OZK_CRT_K
}

int launch_split_fast_crt(const SplitParams &a, const SplitParams &b, int64_t batch, cudaStream_t st) {
    if (const char *e = ozenv("OZAKI_SPLIT"))
        if (!strcmp(e, "generic")) return 1;
    const bool real = a.mode == SPLIT_REAL;
    const int64_t rows_grid = std::max(a.rows_grid, b.rows_grid);
    if (rows_grid == 0) return 0;
    int KW = real ? 1024 : 512, RG = 4;
    const int64_t kpad = real ? a.KB * 32 : a.kh;
    int nwin = (int)((kpad + KW - 1) / KW);
    if (nwin == 2) {   // one double window instead of re-reading the row (as for Ozaki-I)
        KW *= 2;
        nwin = 1;
    }
    bool lng = nwin >= 3;
    if (const char *lg = ozenv("OZAKI_SPLIT_LONG")) lng = (atoi(lg) != 0) && nwin > 1;
    if (lng) {
        RG = real ? 16 : 8;
        KW = 256;
        nwin = (int)((kpad + KW - 1) / KW);
    }
    SplitPair pp;
    pp.side[0] = a;
    pp.side[1] = b;
    if (lng && real) {   // one HBM read through a thread-block cluster (split_cluster.cuh)
        const int nmx = (a.crt.n + 3) / 4 * 4;
        const int rc = launch_split_cluster<true>(nmx > 20 ? 20 : nmx, pp, (unsigned)batch, st, false, false);
        if (rc <= 0) {
            if (rc == 0) g_stats.launches += 1;
            return rc;
        }
    }
    dim3 grid((unsigned)((rows_grid + RG - 1) / RG) * (lng ? nwin : 1), (unsigned)batch, 2);
    uint32_t *emax = nullptr;
    if (lng) {
        if (int rc = launch_exps(pp, (unsigned)batch, 1, real ? 0 : 1, true, st, &emax)) return rc;
    }
    const size_t smem = (size_t)RG * (KW + (real ? 2 : 1)) * (real ? 8 : 16);
    {
        ProfScope ps(st, PH_SLICE);
        switch ((a.crt.n + 3) / 4) {
            case 1: launch_crt_fast<4>(real, lng, grid, smem, st, pp, KW, nwin); break;
            case 2: launch_crt_fast<8>(real, lng, grid, smem, st, pp, KW, nwin); break;
            case 3: launch_crt_fast<12>(real, lng, grid, smem, st, pp, KW, nwin); break;
            case 4: launch_crt_fast<16>(real, lng, grid, smem, st, pp, KW, nwin); break;
            default: launch_crt_fast<20>(real, lng, grid, smem, st, pp, KW, nwin); break;
        }
    }
    if (emax) cudaFreeAsync(emax, st);
    CUDA_TRY(cudaGetLastError());
    g_stats.launches += 1;
    return 0;
}

int run_crt(const Call &c, DevState *dev, cudaStream_t st) {
    const int n = c.s;
    const CrtHost &h = crt_tables(n);
    const bool cplx = c.kind == KIND_4M;
    const int64_t keff = cplx ? 2 * c.k : c.k;
    if (keff > 131071)
        return fail(OZAKI_ERR_UNSUPPORTED, "Ozaki-II: k_eff = %lld exceeds the INT32 residue-GEMM bound 131071",
                    (long long)keff);
    const int nu = crt_nu(h, keff);
    if (nu < 1) return fail(OZAKI_ERR_UNSUPPORTED, "Ozaki-II: moduli budget too small for k (nu < 1)");
    const int64_t Mp = c.m, Np = cplx ? 2 * c.n : c.n;
    const int64_t kh = cplx ? rup(c.k, 32) : 0;
    const int64_t Kp = cplx ? 2 * kh : rup(c.k, 32);
    const int64_t KB = Kp / 32;
    // residue-GEMM tile width 256 NW (gemm_crt.cuh): NW = 2 reuses each A tile for two MMAs but
    // gives up the accumulator double buffer, which pays off when each modulus's K sweep is long
    // (C3, KB = 256: residue GEMM 10-17 % faster; C2 x 30, KB = 64: 4 % slower).  OZAKI_CRT_NW
    // forces 1 or 2.
    int NW = (KB >= 128) ? 2 : 1;
    if (const char *e = ozenv("OZAKI_CRT_NW")) NW = (atoi(e) == 2) ? 2 : 1;
    const int64_t tiles_m = (Mp + 255) / 256, tiles_n = (Np + 256 * NW - 1) / (256 * NW);
    const size_t a_bytes = al256((size_t)n * kCrtBlk * KB * 2 * tiles_m * c.batch);
    const size_t b_bytes = al256((size_t)n * kCrtBlk * KB * 2 * NW * tiles_n * c.batch);
    const size_t ea_bytes = al256(sizeof(int32_t) * Mp * c.batch), fb_bytes = al256(sizeof(int32_t) * Np * c.batch);
    const int64_t rows_pad = 256 * tiles_m, groups = 16 * NW * tiles_n;
    const int64_t batch_bytes = rows_pad * groups * 16;
    const size_t plane_bytes = (size_t)batch_bytes * c.batch;
    const size_t ws = a_bytes + b_bytes + ea_bytes + fb_bytes + al256(plane_bytes * n);
    void *base = nullptr;
    {
        cudaError_t e = cudaMallocAsync(&base, ws, st);
        if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "cudaMallocAsync(%zu): %s", ws, cudaGetErrorString(e));
    }
    int8_t *sa = (int8_t *)base;
    int8_t *sb = sa + a_bytes;
    int32_t *ea = (int32_t *)(sb + b_bytes);
    int32_t *fb = (int32_t *)((char *)ea + ea_bytes);
    int8_t *planes = (int8_t *)((char *)fb + fb_bytes);
    int rc = 0;

    // ---- K1': R17 quantisation + R18 residues (modulus-major slices, 128-row tiles)
    auto params = [&](const Operand &op, bool sideA, int8_t *out, int32_t *exps) {
        SplitParams sp{};
        sp.X = op.X;
        sp.rs = op.rs;
        sp.ls = op.ls;
        sp.bstride = op.bstride;
        sp.rows = op.rows;
        sp.k = op.k;
        sp.mode = op.mode;
        sp.conj = op.conj;
        sp.s = n;
        sp.tile_h = 128;
        sp.tiles = 2 * (sideA ? tiles_m : NW * tiles_n);
        sp.KB = KB;
        sp.kh = kh;
        sp.rows_out = (op.mode == SPLIT_B4M) ? 2 * op.rows : op.rows;
        sp.rows_grid = (op.rows == 0) ? 0 : ((op.mode == SPLIT_B4M) ? sp.tiles * sp.tile_h / 2 : sp.tiles * sp.tile_h);
        sp.out = out;
        sp.exps = exps;
        sp.nonfinite = dev->nonfinite;
        sp.kbs_bytes = kCrtBlk;
        sp.ss_bytes = (int64_t)KB * kCrtBlk;
        sp.crt = h.tab;
        sp.crt.nu = nu;
        return sp;
    };
    auto split = [&](const SplitParams &sp) -> int {   // generic form, one operand per launch
        if (sp.rows == 0) return 0;
        const bool cx = sp.mode != SPLIT_REAL;
        dim3 grid((unsigned)((sp.rows_grid + 7) / 8), (unsigned)c.batch);
        const int KW = cx ? 512 : 1024;
        const size_t smem = (size_t)8 * (KW + (cx ? 1 : 2)) * (cx ? 16 : 8);
        SplitPair pp;
        pp.side[0] = sp;
        pp.side[1] = sp;
        ProfScope ps(st, PH_SLICE);
#define OZK_SPLIT2(CX)                                                                               \
        {                                                                                            \
            smem_optin((const void *)k_split_sm<8, CX, true>, smem);                                 \
            k_split_sm<8, CX, true><<<grid, 256, smem, st>>>(pp, KW);                               \
        }
        if (cx) OZK_SPLIT2(true) else OZK_SPLIT2(false)
#undef OZK_SPLIT2
        CUDA_TRY(cudaGetLastError());
        g_stats.launches += 1;
        return 0;
    };
    const int ma = cplx ? SPLIT_A4M : SPLIT_REAL, mb = cplx ? SPLIT_B4M : SPLIT_REAL;
    const SplitParams spa = params(view_A(c.A, c.ta, c.m, c.k, c.lda, c.sA, ma), true, sa, ea);
    const SplitParams spb = params(view_B(c.B, c.tb, c.n, c.k, c.ldb, c.sB, mb), false, sb, fb);
    rc = launch_split_fast_crt(spa, spb, c.batch, st);
    if (rc == 1) {
        rc = split(spa);
        if (!rc) rc = split(spb);
    }

    // ---- K2': one INT8 GEMM per modulus, residues of the products (R19)
    if (!rc) {
        CrtGemmParams G;
        std::memset(&G, 0, sizeof G);
        int kpp = 4;
        while (KB % kpp) kpp >>= 1;
        G.kpp = kpp;
        G.stage_bytes = (uint32_t)kpp * (1 + NW) * kCrtBlk;
        G.stages = (int)std::min<int64_t>(8, (int64_t)(224 * 1024) / G.stage_bytes);
        const size_t smem = (size_t)G.stages * G.stage_bytes + 1024 + 512;
        G.batch = c.batch;
        G.tiles_m = tiles_m;
        G.tiles_n = tiles_n;
        G.KB = KB;
        G.R = planes;
        G.plane_bytes = (int64_t)plane_bytes;
        G.batch_bytes = batch_bytes;
        G.rows_pad = rows_pad;
        G.crt = h.tab;
        G.crt.nu = nu;
        rc = rows_map(&G.tmA, sa, a_bytes, (uint32_t)kpp * (kCrtBlk / 256));
        if (!rc) rc = rows_map(&G.tmB, sb, b_bytes, (uint32_t)kpp * (kCrtBlk / 256));
        if (!rc) {
            auto kern = (NW == 2) ? k_gemm_crt<2> : k_gemm_crt<1>;
            CUDA_TRY(smem_optin((const void *)kern, smem));
            const int64_t tiles = c.batch * tiles_m * tiles_n;
            const unsigned pairs = (unsigned)std::min<int64_t>(tiles, dev->sms / 2);
            {
                ProfScope ps(st, PH_GEMM);
                kern<<<2 * pairs, kCrtThreads, smem, st>>>(G);
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "k_gemm_crt: %s", cudaGetErrorString(e));
            g_stats.launches += 1;
        }
    }
    // ---- K3': CRT reconstruction + one rounding + alpha/beta (R20, R7)
    if (!rc) {
        CrtParams Q;
        std::memset(&Q, 0, sizeof Q);
        Q.R = planes;
        Q.plane_bytes = (int64_t)plane_bytes;
        Q.batch_bytes = batch_bytes;
        Q.rows_pad = rows_pad;
        Q.groups = groups;
        Q.ea = ea;
        Q.fb = fb;
        Q.Mp = Mp;
        Q.Np = Np;
        Q.batch = c.batch;
        Q.C = c.C;
        Q.ldc = c.ldc;
        Q.strideC = c.sC;
        Q.cplx = cplx ? 1 : 0;
        Q.ab_unit = (c.al[0] == 1.0 && c.al[1] == 0.0 && c.be[0] == 0.0 && c.be[1] == 0.0) ? 1 : 0;
        Q.nu = nu;
        Q.n = n;
        Q.alpha_r = c.al[0];
        Q.alpha_i = c.al[1];
        Q.beta_r = c.be[0];
        Q.beta_i = c.be[1];
        for (int q = 0; q < n; ++q) {
            Q.p[q] = h.tab.p[q];
            for (int l = 0; l < kCrtLimbs; ++l) Q.W[q][l] = h.W[q][l];
        }
        std::memcpy(Q.M, h.M, sizeof Q.M);
        std::memcpy(Q.Mhalf, h.Mhalf, sizeof Q.Mhalf);
        Q.Minv = std::ldexp(h.Minv, 32 * (h.L - 1));   // top-two-limb quotient estimate
        dim3 grid((unsigned)((rows_pad * groups * 4 + 255) / 256), (unsigned)c.batch);
        {
            ProfScope ps(st, PH_OTHER);
            if (h.L != (n + 3) / 4)   // k_crt<N> holds M in ceil(N / 4) limbs (true for the R16 moduli)
                return fail(OZAKI_ERR_UNSUPPORTED, "Ozaki-II: M needs %d limbs for %d moduli", h.L, n);
            switch (n) {
#define OZK_CRT_N(N) case N: k_crt<N><<<grid, 256, 0, st>>>(Q); break;
                OZK_CRT_N(1) OZK_CRT_N(2) OZK_CRT_N(3) OZK_CRT_N(4) OZK_CRT_N(5) OZK_CRT_N(6) OZK_CRT_N(7)
                OZK_CRT_N(8) OZK_CRT_N(9) OZK_CRT_N(10) OZK_CRT_N(11) OZK_CRT_N(12) OZK_CRT_N(13)
                OZK_CRT_N(14) OZK_CRT_N(15) OZK_CRT_N(16) OZK_CRT_N(17) OZK_CRT_N(18) OZK_CRT_N(19)
                default: k_crt<20><<<grid, 256, 0, st>>>(Q); break;
#undef OZK_CRT_N
            }
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "k_crt: %s", cudaGetErrorString(e));
        g_stats.launches += 1;
    }
    cudaFreeAsync(base, st);
    if (rc) return rc;
    g_stats.entries += (uint64_t)c.batch;
    g_stats.equiv += (uint64_t)n * (cplx ? 4 : 1) * (uint64_t)c.batch;
    g_stats.macs += (uint64_t)n * (uint64_t)(2 * tiles_m * 128) * (uint64_t)(tiles_n * 256) * (uint64_t)Kp *
                    (uint64_t)c.batch;
    g_stats.crt += 1;
    return 0;
}

int run(const Call &c0) {
    t_err.clear();
    if (int rc = validate(c0)) return rc;
    Call c = c0;
    c.ta = up(c.ta);
    c.tb = up(c.tb);
    if (c.kind == KIND_REAL) {   // 'C' == 'T' for real operands
        if (c.ta == 'C') c.ta = 'T';
        if (c.tb == 'C') c.tb = 'T';
    }
    if (c.m == 0 || c.n == 0 || c.batch == 0) return 0;
    // the kernels index batch entries with blockIdx.y / z (at most 65535): larger batches run as
    // consecutive sub-batches, each entry's computation unchanged
    constexpr int64_t kMaxGridBatch = 65535;
    if (c.batch > kMaxGridBatch && !c.S_out) {
        const int64_t ew = (c.kind == KIND_REAL) ? 1 : 2;   // doubles per element
        for (int64_t b0 = 0; b0 < c.batch; b0 += kMaxGridBatch) {
            Call cb = c;
            cb.batch = std::min(kMaxGridBatch, c.batch - b0);
            cb.A = c.A + ew * b0 * c.sA;
            cb.B = c.B + ew * b0 * c.sB;
            cb.C = c.C + ew * b0 * c.sC;
            if (int rc = run(cb)) return rc;
        }
        return 0;
    }
    DevState *dev = nullptr;
    if (int rc = device_state(&dev)) return rc;
    if (!c.S_out) {   // host operands -> pipelined offload (all three must be host)
        const bool readsAB = !(c.al[0] == 0.0 && c.al[1] == 0.0) && c.k > 0;
        const PtrKind kc = ptr_kind(c.C);
        const PtrKind ka = readsAB ? ptr_kind(c.A) : kc, kb = readsAB ? ptr_kind(c.B) : kc;
        if (ka == PTR_HOST || kb == PTR_HOST || kc == PTR_HOST) {
            if (!(ka == PTR_HOST && kb == PTR_HOST && kc == PTR_HOST))
                return fail(OZAKI_ERR_UNSUPPORTED, "A, B, C must all be device or all be host pointers");
            if (!readsAB && c.be[0] == 1.0 && c.be[1] == 0.0) return 0;   // quick return, C unchanged
            if (readsAB && c.batch == 1) {
                // one large GEMM: 2-D blocks of ~128 MB row panels of op(A) / column panels of op(B)
                // (multiples of the 256-row / 128-column super-tile; every block call re-splits its
                // panels, which the GPU hides under the PCIe time)
                const size_t es = (c.kind == KIND_REAL) ? 8 : 16;
                const int64_t per = (int64_t)((128ull << 20) / std::max<size_t>(1, (size_t)c.k * es));
                int64_t rb = std::max<int64_t>(256, per / 256 * 256), cb = std::max<int64_t>(128, per / 128 * 128);
                if (const char *pe = ozenv("OZAKI_OFFLOAD_PANEL_COLS")) cb = std::max<int64_t>(1, atoll(pe));
                if (const char *pe = ozenv("OZAKI_OFFLOAD_PANEL_ROWS")) rb = std::max<int64_t>(1, atoll(pe));
                if (c.n > cb || c.m > rb) return run_offload_blocks(c, rb, cb);
            }
            return run_offload(c);   // (alpha == 0 or k == 0: C = beta C staged through k_scale_*)
        }
    }
    cudaStream_t st = t_stream;
    const size_t es = (c.kind == KIND_REAL) ? 8 : 16;
    const bool cplx = c.kind != KIND_REAL;
    const bool alpha0 = c.al[0] == 0.0 && c.al[1] == 0.0;
    // cross-call overlap: whatever this call launches, the stream's last kernel is no longer a
    // tracked GEMM unless the overlapped main path below sets it again
    OvState *ov = t_overlap ? &ov_state(st) : nullptr;
    const bool prev_gemm = ov && ov->last_gemm;
    const uintptr_t pc_lo = ov ? ov->c_lo : 0, pc_hi = ov ? ov->c_hi : 0;
    if (ov) ov->last_gemm = false;
    const bool beta1 = c.be[0] == 1.0 && c.be[1] == 0.0;

    // C must not alias A or B (only checked when A/B are read)
    if (!alpha0 && c.k > 0) {
        const size_t cb = span_bytes(c.m, c.n, c.ldc, c.sC, c.batch, es);
        const int64_t ar = c.ta == 'N' ? c.m : c.k, ac = c.ta == 'N' ? c.k : c.m;
        const int64_t br = c.tb == 'N' ? c.k : c.n, bc = c.tb == 'N' ? c.n : c.k;
        const bool oa = overlaps(c.C, cb, c.A, span_bytes(ar, ac, c.lda, c.sA, c.batch, es)) &&
                        (c.batch > 1 || elems_overlap(c.A, ar, ac, c.lda, c.C, c.m, c.n, c.ldc, es));
        const bool ob = overlaps(c.C, cb, c.B, span_bytes(br, bc, c.ldb, c.sB, c.batch, es)) &&
                        (c.batch > 1 || elems_overlap(c.B, br, bc, c.ldb, c.C, c.m, c.n, c.ldc, es));
        if (oa || ob) return fail(OZAKI_ERR_ALIAS, "C overlaps A or B");
    }
    // quick return (R7): alpha == 0 or k == 0 -> C = beta C
    if (alpha0 || c.k == 0) {
        if (beta1 || c.S_out) return 0;
        dim3 grid(grid1d(c.m * c.n, dev->sms), 1, (unsigned)c.batch);
        ProfScope ps(st, PH_OTHER);
        if (cplx)
            k_scale_cplx<<<grid, 256, 0, st>>>(c.C, c.m, c.n, c.ldc, c.sC, c.be[0], c.be[1]);
        else
            k_scale_real<<<grid, 256, 0, st>>>(c.C, c.m, c.n, c.ldc, c.sC, c.be[0]);
        CUDA_TRY(cudaGetLastError());
        g_stats.launches += 1;
        return 0;
    }

    if (c.crt) return run_crt(c, dev, st);

    // R22 (NEXT-4): per-block exponents -- emulate each K block with its own exponents into T
    // (T = P_0, then T = P_b + T: one RNE per block), then C = alpha T + beta C.
    if (c.kblock > 0 && c.kblock < c.k && !c.S_out) {
        const size_t tb = al256(es * (size_t)c.m * c.n * c.batch);
        double *T = nullptr;
        {
            cudaError_t e = cudaMallocAsync((void **)&T, tb, st);
            if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "cudaMallocAsync(%zu): %s", tb, cudaGetErrorString(e));
        }
        const int64_t ew = cplx ? 2 : 1;   // doubles per element
        int rc = 0;
        // the block calls run without cross-call overlap: the stream's last kernel is
        // k_apply_ab (writing the user's C), never a tracked GEMM of the temporary T
        const int ovs = t_overlap;
        t_overlap = 0;
        for (int64_t b0 = 0; b0 < c.k && !rc; b0 += c.kblock) {
            Call cb = c;
            cb.k = std::min<int64_t>(c.kblock, c.k - b0);
            cb.A = c.A + ew * (c.ta == 'N' ? b0 * c.lda : b0);
            cb.B = c.B + ew * (c.tb == 'N' ? b0 : b0 * c.ldb);
            cb.C = T;
            cb.ldc = c.m;
            cb.sC = c.m * c.n;
            cb.al[0] = 1.0;
            cb.al[1] = 0.0;
            cb.be[0] = (b0 == 0) ? 0.0 : 1.0;
            cb.be[1] = 0.0;
            cb.kblock = 0;
            cb.batched = true;
            rc = run(cb);
        }
        t_overlap = ovs;
        if (!rc) {
            dim3 grid(grid1d(c.m * c.n, dev->sms), 1, (unsigned)c.batch);
            ProfScope ps(st, PH_OTHER);
            k_apply_ab<<<grid, 256, 0, st>>>(T, c.C, c.m, c.n, c.ldc, c.sC, cplx ? 1 : 0, c.al[0], c.al[1],
                                            c.be[0], c.be[1]);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "apply_ab: %s", cudaGetErrorString(e));
            g_stats.launches += 1;
        }
        cudaFreeAsync(T, st);
        return rc;
    }

    Plan P;
    const Kind pk = (c.kind == KIND_4M) ? KIND_4M : KIND_REAL;
    // 3M: the three real products run as 3 x batch entries of ONE plan / split / GEMM launch
    const int64_t pbatch = (c.kind == KIND_3M) ? 3 * c.batch : c.batch;
    if (int rc = make_plan(pk, c.m, c.n, c.k, pbatch, c.s, P, c.full)) return rc;
    if (!c.S_out) plan_splitk(P, dev->sms);
    size_t ws = plan_workspace(P);
    size_t t_bytes = 0;
    if (c.kind == KIND_3M) t_bytes = al256(sizeof(double) * c.m * c.n * c.batch);
    ws += 3 * t_bytes + P.p0_bytes + P.pl_bytes;

    // cross-call overlap (ozaki_set_overlap): one split + one GEMM launch, slices in the
    // alternate persistent workspace; the split may start under the previous call's GEMM
    // (PDL), and may read / write before that GEMM ends when its C overlaps neither operand
    const bool ovl = ov && (c.kind == KIND_REAL || c.kind == KIND_4M) && !c.S_out && !P.kchunk_needed;
    int ov_slot = 0;
    void *base = nullptr;
    if (ovl) {
        ov_slot = ov->next;
        if (ov->cap[ov_slot] < ws) {   // grow (rare): the buffer may still be read by a GEMM in flight
            CUDA_TRY(cudaStreamSynchronize(st));
            if (ov->ws[ov_slot]) cudaFree(ov->ws[ov_slot]);
            ov->ws[ov_slot] = nullptr;
            ov->cap[ov_slot] = 0;
            cudaError_t e = cudaMalloc(&ov->ws[ov_slot], ws);
            if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "overlap workspace (%zu B): %s", ws, cudaGetErrorString(e));
            ov->cap[ov_slot] = ws;
        }
        base = ov->ws[ov_slot];
    } else {
        cudaError_t e = cudaMallocAsync(&base, ws, st);
        if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "cudaMallocAsync(%zu): %s", ws, cudaGetErrorString(e));
    }
    int8_t *sa = (int8_t *)base;
    int8_t *sb = sa + P.a_bytes;
    int32_t *ea = (int32_t *)(sb + P.b_bytes);
    int32_t *fb = (int32_t *)((char *)ea + P.ea_bytes);
    double *T = (double *)((char *)fb + P.fb_bytes);
    int64_t *P0 = P.splitk > 1 ? (int64_t *)((char *)T + 3 * t_bytes) : nullptr;
    int32_t *PL = P.splitk > 1 ? (int32_t *)((char *)P0 + P.p0_bytes) : nullptr;
    int rc = 0;

    if (c.kind == KIND_REAL || c.kind == KIND_4M) {
        const int ma = (c.kind == KIND_4M) ? SPLIT_A4M : SPLIT_REAL;
        const int mb = (c.kind == KIND_4M) ? SPLIT_B4M : SPLIT_REAL;
        if (ovl && prev_gemm) {
            const int64_t ar = c.ta == 'N' ? c.m : c.k, ac = c.ta == 'N' ? c.k : c.m;
            const int64_t br = c.tb == 'N' ? c.k : c.n, bc = c.tb == 'N' ? c.n : c.k;
            const uintptr_t a0 = (uintptr_t)c.A, a1 = a0 + span_bytes(ar, ac, c.lda, c.sA, c.batch, es);
            const uintptr_t b0 = (uintptr_t)c.B, b1 = b0 + span_bytes(br, bc, c.ldb, c.sB, c.batch, es);
            t_split_pdl = true;
            t_split_early = (a1 <= pc_lo || a0 >= pc_hi) && (b1 <= pc_lo || b0 >= pc_hi);
        }
        rc = launch_split_ab(P, view_A(c.A, c.ta, c.m, c.k, c.lda, c.sA, ma), sa, ea,
                             view_B(c.B, c.tb, c.n, c.k, c.ldb, c.sB, mb), sb, fb, dev, st);
        t_split_pdl = t_split_early = false;
        if (!rc) {
            const int epi = c.S_out ? EPI_LEVELS : (c.kind == KIND_4M ? EPI_CPLX4M : EPI_REAL);
            rc = launch_gemm(P, epi, sa, sb, ea, fb, c.C, c.ldc, c.sC, c.al, c.be, c.S_out, dev, st, P0, PL);
        }
    } else {   // 3M: one fused split per operand (Re, Im, fl(Re+Im) regions) and ONE GEMM launch
               // over 3 x batch entries into T = [T1 | T2 | T3], then the combine
        const double one[2] = {1.0, 0.0}, zero[2] = {0.0, 0.0};
        rc = launch_split_ab(P, view_A(c.A, c.ta, c.m, c.k, c.lda, c.sA, SPLIT_3M), sa, ea,
                             view_B(c.B, c.tb, c.n, c.k, c.ldb, c.sB, SPLIT_3M), sb, fb, dev, st, c.batch);
        if (!rc) rc = launch_gemm(P, EPI_REAL, sa, sb, ea, fb, T, c.m, c.m * c.n, one, zero, nullptr, dev, st, P0, PL);
        if (!rc) {
            dim3 grid(grid1d(c.m * c.n, dev->sms), 1, (unsigned)c.batch);
            ProfScope ps(st, PH_OTHER);
            const int64_t tx = c.m * c.n * c.batch;   // the GEMM wrote T1, T2, T3 back to back
            k_combine_3m<<<grid, 256, 0, st>>>(T, T + tx, T + 2 * tx, c.C, c.m, c.n,
                                              c.ldc, c.sC, c.al[0], c.al[1], c.be[0], c.be[1]);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "combine_3m: %s", cudaGetErrorString(e));
            g_stats.launches += 1;
        }
    }
    if (ovl) {
        if (!rc) {
            ov->next = ov_slot ^ 1;
            ov->last_gemm = true;
            ov->c_lo = (uintptr_t)c.C;
            ov->c_hi = ov->c_lo + span_bytes(c.m, c.n, c.ldc, c.sC, c.batch, es);
        }
    } else {
        cudaFreeAsync(base, st);
    }
    if (rc) return rc;

    const uint64_t pr = c.full ? (uint64_t)c.s * c.s : (uint64_t)c.s * (c.s + 1) / 2;
    const uint64_t mult = c.kind == KIND_REAL ? 1 : (c.kind == KIND_4M ? 4 : 3);
    g_stats.entries += (uint64_t)c.batch;
    g_stats.equiv += pr * mult * (uint64_t)c.batch;
    const uint64_t rows_pad = (uint64_t)P.tiles_m * kBM * (P.pair ? 2 : 1);
    g_stats.macs += pr * (uint64_t)(c.kind == KIND_3M ? 3 : 1) * rows_pad * (uint64_t)P.tiles_n * P.BN *
                    (uint64_t)P.Kp * (uint64_t)c.batch;
    if (c.kind == KIND_REAL) g_stats.dgemm += 1;
    if (c.kind == KIND_4M) g_stats.zgemm += 1;
    if (c.kind == KIND_3M) g_stats.zgemm3m += 1;
    return 0;
}

// ============================================================ emulated TRSM (R23, NEXT-4c)
struct TrsmCall {
    bool cplx;
    char side, uplo, ta, diag;
    int64_t m, n;
    double al[2];
    const double *A;
    int64_t lda;
    double *B;
    int64_t ldb;
    int s;
};

int validate_trsm(const TrsmCall &c) {
    const char sd = up(c.side), ul = up(c.uplo), dg = up(c.diag);
    if (sd != 'L' && sd != 'R') return fail(-1, "side");
    if (ul != 'U' && ul != 'L') return fail(-2, "uplo");
    if (!trans_ok(c.ta)) return fail(-3, "transa");
    if (dg != 'U' && dg != 'N') return fail(-4, "diag");
    if (c.m < 0) return fail(-5, "m < 0");
    if (c.n < 0) return fail(-6, "n < 0");
    if (c.lda < std::max<int64_t>(1, sd == 'L' ? c.m : c.n)) return fail(-9, "lda too small");
    if (c.ldb < std::max<int64_t>(1, c.m)) return fail(-11, "ldb too small");
    if (c.s < 1 || c.s > 16) return fail(-12, "num_slices not in [1,16]");
    return 0;
}

int run_trsm_device(const TrsmCall &c, DevState *dev, cudaStream_t st) {
    const char sd = up(c.side), ul = up(c.uplo), dg = up(c.diag);
    char ta = up(c.ta);
    if (!c.cplx && ta == 'C') ta = 'T';
    const bool left = sd == 'L';
    const int64_t dim = left ? c.m : c.n;
    const size_t es = c.cplx ? 16 : 8;
    const double *A = c.A;
    double *B = c.B;
    // B <- alpha B with R7's quick-return op shapes (alpha == 0: zeros, B not read)
    const bool alpha1 = c.al[0] == 1.0 && c.al[1] == 0.0;
    if (!alpha1) {
        dim3 grid(grid1d(c.m * c.n, dev->sms), 1, 1);
        ProfScope ps(st, PH_OTHER);
        if (c.cplx) k_scale_cplx<<<grid, 256, 0, st>>>(B, c.m, c.n, c.ldb, 0, c.al[0], c.al[1]);
        else k_scale_real<<<grid, 256, 0, st>>>(B, c.m, c.n, c.ldb, 0, c.al[0]);
        CUDA_TRY(cudaGetLastError());
        g_stats.launches += 1;
        if (c.al[0] == 0.0 && c.al[1] == 0.0) return 0;
    }
    const bool lower = (ul == 'L') == (ta == 'N');   // op(A) lower triangular
    const bool forward = left ? lower : !lower;
    const int64_t nb = std::max<int64_t>(1, t_trsm_nb);
    const int64_t nblk = (dim + nb - 1) / nb;
    const double m1[2] = {-1.0, 0.0}, p1[2] = {1.0, 0.0};
    const int ovs = t_overlap;
    t_overlap = 0;   // the diagonal kernels sit between the GEMMs (no PDL early reads)
    const cudaStream_t user = t_stream;
    t_stream = st;
    int rc = 0;
    for (int64_t q = 0; q < nblk && !rc; ++q) {
        const int64_t bi = forward ? q : nblk - 1 - q;
        const int64_t k0 = bi * nb, kb = std::min<int64_t>(nb, dim - k0);
        TrsmDiagParams dp;
        dp.A = A;
        dp.lda = c.lda;
        dp.B = B;
        dp.ldb = c.ldb;
        dp.k0 = k0;
        dp.kb = (int32_t)kb;
        dp.trans = ta == 'N' ? 0 : (ta == 'T' ? 1 : 2);
        dp.lower = lower ? 1 : 0;
        dp.unit = dg == 'U' ? 1 : 0;
        dp.right = left ? 0 : 1;
        dp.nvec = left ? c.n : c.m;
        {
            ProfScope ps(st, PH_OTHER);
            const unsigned g = (unsigned)((dp.nvec + 127) / 128);
            if (c.cplx) k_trsm_diag<true><<<g, 128, 0, st>>>(dp);
            else k_trsm_diag<false><<<g, 128, 0, st>>>(dp);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) { rc = fail(OZAKI_ERR_CUDA, "k_trsm_diag: %s", cudaGetErrorString(e)); break; }
            g_stats.launches += 1;
        }
        // remaining rows (left) / columns (right): [k0 + kb, dim) forward, [0, k0) backward
        const int64_t r0 = forward ? k0 + kb : 0, r1 = forward ? dim : k0;
        if (r1 <= r0) continue;
        const int64_t nr = r1 - r0;
        // T_{R,K} (left) or T_{K,R} (right) as an operand of op(): 'N' -> A(rows, cols) of T,
        // 'T'/'C' -> the mirrored block of A with the same transpose flag
        auto tblock = [&](int64_t row0, int64_t col0) {   // element (0,0) of T(row0.., col0..)
            const int64_t r = ta == 'N' ? row0 : col0, cc = ta == 'N' ? col0 : row0;
            return A + (c.cplx ? 2 : 1) * (r + cc * c.lda);
        };
        const int64_t ew = c.cplx ? 2 : 1;
        Call g{};
        g.kind = c.cplx ? KIND_4M : KIND_REAL;
        g.al[0] = m1[0];
        g.al[1] = m1[1];
        g.be[0] = p1[0];
        g.be[1] = p1[1];
        g.s = c.s;
        g.batch = 1;
        g.batched = false;
        g.full = t_full_pairs != 0;
        g.kblock = t_kblock;
        if (left) {   // B_R <- -T_{R,K} X_K + B_R
            g.ta = ta;
            g.tb = 'N';
            g.m = nr;
            g.n = c.n;
            g.k = kb;
            g.A = tblock(r0, k0);
            g.lda = c.lda;
            g.B = B + ew * k0;
            g.ldb = c.ldb;
            g.C = B + ew * r0;
            g.ldc = c.ldb;
        } else {      // B_R <- -X_K T_{K,R} + B_R
            g.ta = 'N';
            g.tb = ta;
            g.m = c.m;
            g.n = nr;
            g.k = kb;
            g.A = B + ew * k0 * c.ldb;
            g.lda = c.ldb;
            g.B = tblock(k0, r0);
            g.ldb = c.lda;
            g.C = B + ew * r0 * c.ldb;
            g.ldc = c.ldb;
        }
        rc = run(g);
    }
    t_stream = user;
    t_overlap = ovs;
    (void)es;
    return rc;
}

int run_trsm(const TrsmCall &c0) {
    t_err.clear();
    env_refresh();
    if (int rc = validate_trsm(c0)) return rc;
    TrsmCall c = c0;
    if (c.m == 0 || c.n == 0) return 0;
    DevState *dev = nullptr;
    if (int rc = device_state(&dev)) return rc;
    const bool left = up(c.side) == 'L';
    const int64_t dim = left ? c.m : c.n;
    const size_t es = c.cplx ? 16 : 8;
    const bool alpha0 = c.al[0] == 0.0 && c.al[1] == 0.0;
    const size_t abytes = alpha0 ? 0 : es * (size_t)((dim - 1) * c.lda + dim);
    const size_t bbytes = es * (size_t)((c.n - 1) * c.ldb + c.m);
    if (!alpha0 && overlaps(c.A, abytes, c.B, bbytes)) return fail(OZAKI_ERR_ALIAS, "A overlaps B");
    cudaStream_t st = t_stream;
    const PtrKind kb_ = ptr_kind(c.B), ka = alpha0 ? kb_ : ptr_kind(c.A);
    if (ka == PTR_DEVICE && kb_ == PTR_DEVICE) return run_trsm_device(c, dev, st);
    if (!(ka == PTR_HOST && kb_ == PTR_HOST))
        return fail(OZAKI_ERR_UNSUPPORTED, "A and B must both be device or both be host pointers");
    // host pointers: stage A (dim x dim, pitch lda) and B (m x n, pitch ldb), solve, copy B back
    char *buf = nullptr;
    const size_t a_dev = alpha0 ? 0 : es * (size_t)dim * dim, b_dev = es * (size_t)c.m * c.n;
    cudaError_t e = cudaMallocAsync((void **)&buf, al256(a_dev) + b_dev, st);
    if (e != cudaSuccess) return fail(OZAKI_ERR_ALLOC, "TRSM staging: %s", cudaGetErrorString(e));
    TrsmCall d = c;
    d.A = (const double *)buf;
    d.lda = std::max<int64_t>(1, dim);
    d.B = (double *)(buf + al256(a_dev));
    d.ldb = c.m;
    int rc = 0;
    if (!alpha0)
        CUDA_TRY(cudaMemcpy2DAsync(buf, es * dim, c.A, es * c.lda, es * dim, dim, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpy2DAsync(d.B, es * c.m, c.B, es * c.ldb, es * c.m, c.n, cudaMemcpyHostToDevice, st));
    rc = run_trsm_device(d, dev, st);
    if (!rc) CUDA_TRY(cudaMemcpy2DAsync(c.B, es * c.ldb, d.B, es * c.m, es * c.m, c.n, cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(buf, st);
    e = cudaStreamSynchronize(st);
    if (!rc && e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "TRSM: %s", cudaGetErrorString(e));
    return rc;
}

Call make_call(Kind kind, char ta, char tb, int64_t m, int64_t n, int64_t k, const double *al,
               const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb, int64_t sB,
               const double *be, double *C, int64_t ldc, int64_t sC, int64_t batch, int s,
               bool batched) {
    env_refresh();
    Call c{};
    c.kind = kind;
    c.ta = ta;
    c.tb = tb;
    c.m = m;
    c.n = n;
    c.k = k;
    c.al[0] = al[0];
    c.al[1] = kind == KIND_REAL ? 0.0 : al[1];
    c.be[0] = be[0];
    c.be[1] = kind == KIND_REAL ? 0.0 : be[1];
    c.A = A;
    c.lda = lda;
    c.sA = sA;
    c.B = B;
    c.ldb = ldb;
    c.sB = sB;
    c.C = C;
    c.ldc = ldc;
    c.sC = sC;
    c.batch = batch;
    c.s = s;
    c.batched = batched;
    c.full = t_full_pairs != 0;
    c.kblock = t_kblock;
    return c;
}

Call make_call_crt(Kind kind, char ta, char tb, int64_t m, int64_t n, int64_t k, const double *al,
                   const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb, int64_t sB,
                   const double *be, double *C, int64_t ldc, int64_t sC, int64_t batch, int nmod,
                   bool batched) {
    Call c = make_call(kind, ta, tb, m, n, k, al, A, lda, sA, B, ldb, sB, be, C, ldc, sC, batch, nmod, batched);
    c.crt = true;
    return c;
}

}  // namespace

// =========================================================================
extern "C" {

int ozaki_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                int64_t ldc, int num_slices) {
    const double al[2] = {alpha, 0.0}, be[2] = {beta, 0.0};
    return run(make_call(KIND_REAL, transa, transb, m, n, k, al, A, lda, 0, B, ldb, 0, be, C, ldc,
                         0, 1, num_slices, false));
}

int ozaki_zgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, const double *alpha,
                const double *A, int64_t lda, const double *B, int64_t ldb, const double *beta,
                double *C, int64_t ldc, int num_slices) {
    return run(make_call(KIND_4M, transa, transb, m, n, k, alpha, A, lda, 0, B, ldb, 0, beta, C,
                         ldc, 0, 1, num_slices, false));
}

int ozaki_zgemm3m(char transa, char transb, int64_t m, int64_t n, int64_t k, const double *alpha,
                  const double *A, int64_t lda, const double *B, int64_t ldb, const double *beta,
                  double *C, int64_t ldc, int num_slices) {
    return run(make_call(KIND_3M, transa, transb, m, n, k, alpha, A, lda, 0, B, ldb, 0, beta, C,
                         ldc, 0, 1, num_slices, false));
}

int ozaki_dgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                double alpha, const double *A, int64_t lda, int64_t strideA,
                                const double *B, int64_t ldb, int64_t strideB, double beta,
                                double *C, int64_t ldc, int64_t strideC, int64_t batch,
                                int num_slices) {
    const double al[2] = {alpha, 0.0}, be[2] = {beta, 0.0};
    return run(make_call(KIND_REAL, transa, transb, m, n, k, al, A, lda, strideA, B, ldb, strideB,
                         be, C, ldc, strideC, batch, num_slices, true));
}

int ozaki_zgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                const double *alpha, const double *A, int64_t lda,
                                int64_t strideA, const double *B, int64_t ldb, int64_t strideB,
                                const double *beta, double *C, int64_t ldc, int64_t strideC,
                                int64_t batch, int num_slices) {
    return run(make_call(KIND_4M, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB,
                         beta, C, ldc, strideC, batch, num_slices, true));
}

int ozaki_zgemm3m_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                  const double *alpha, const double *A, int64_t lda,
                                  int64_t strideA, const double *B, int64_t ldb, int64_t strideB,
                                  const double *beta, double *C, int64_t ldc, int64_t strideC,
                                  int64_t batch, int num_slices) {
    return run(make_call(KIND_3M, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB,
                         beta, C, ldc, strideC, batch, num_slices, true));
}

// ---- Ozaki-II (CRT), NEXT-1
int ozaki2_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                 int64_t ldc, int num_moduli) {
    const double al[2] = {alpha, 0.0}, be[2] = {beta, 0.0};
    return run(make_call_crt(KIND_REAL, transa, transb, m, n, k, al, A, lda, 0, B, ldb, 0, be, C, ldc, 0, 1,
                             num_moduli, false));
}

int ozaki2_zgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, const double *alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, const double *beta,
                 double *C, int64_t ldc, int num_moduli) {
    return run(make_call_crt(KIND_4M, transa, transb, m, n, k, alpha, A, lda, 0, B, ldb, 0, beta, C, ldc, 0, 1,
                             num_moduli, false));
}

int ozaki2_dgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                 double alpha, const double *A, int64_t lda, int64_t strideA,
                                 const double *B, int64_t ldb, int64_t strideB, double beta, double *C,
                                 int64_t ldc, int64_t strideC, int64_t batch, int num_moduli) {
    const double al[2] = {alpha, 0.0}, be[2] = {beta, 0.0};
    return run(make_call_crt(KIND_REAL, transa, transb, m, n, k, al, A, lda, strideA, B, ldb, strideB, be, C,
                             ldc, strideC, batch, num_moduli, true));
}

int ozaki2_zgemm_strided_batched(char transa, char transb, int64_t m, int64_t n, int64_t k,
                                 const double *alpha, const double *A, int64_t lda, int64_t strideA,
                                 const double *B, int64_t ldb, int64_t strideB, const double *beta,
                                 double *C, int64_t ldc, int64_t strideC, int64_t batch, int num_moduli) {
    return run(make_call_crt(KIND_4M, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta,
                             C, ldc, strideC, batch, num_moduli, true));
}

int ozaki_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
                const double *A, int64_t lda, double *B, int64_t ldb, int num_slices) {
    TrsmCall c{false, side, uplo, transa, diag, m, n, {alpha, 0.0}, A, lda, B, ldb, num_slices};
    return run_trsm(c);
}

int ozaki_ztrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, const double *alpha,
                const double *A, int64_t lda, double *B, int64_t ldb, int num_slices) {
    TrsmCall c{true, side, uplo, transa, diag, m, n, {alpha[0], alpha[1]}, A, lda, B, ldb, num_slices};
    return run_trsm(c);
}

int ozaki_set_trsm_block(int64_t nb) {
    if (nb < 1) return -1;
    t_trsm_nb = nb;
    return 0;
}

int64_t ozaki_get_trsm_block(void) { return t_trsm_nb; }

int ozaki_set_exponent_block(int64_t kb) {
    if (kb < 0) return fail(-1, "exponent block < 0");
    t_kblock = kb;
    return 0;
}

int64_t ozaki_get_exponent_block(void) { return t_kblock; }

int ozaki_set_overlap(int on) {
    t_overlap = on ? 1 : 0;
    if (!on && !t_ov_list.v.empty()) {   // release this thread's persistent workspaces once their GEMMs
        int cur = 0;                 // finished (device-wide sync: a tracked stream may be gone)
        cudaGetDevice(&cur);
        for (auto &o : t_ov_list.v) {
            cudaSetDevice(o.dev);
            cudaDeviceSynchronize();
            for (int i = 0; i < 2; ++i)
                if (o.ws[i]) cudaFree(o.ws[i]);
        }
        cudaSetDevice(cur);
        t_ov_list.v.clear();
    }
    return 0;
}

int ozaki_get_overlap(void) { return t_overlap; }

int ozaki_set_pair_set(int full) {
    t_full_pairs = full ? 1 : 0;
    return 0;
}

int ozaki_get_pair_set(void) { return t_full_pairs; }

int ozaki_set_stream(void *stream) {
    t_stream = (cudaStream_t)stream;
    return 0;
}

void *ozaki_get_stream(void) { return (void *)t_stream; }

int ozaki_stream_synchronize(void) {
    CUDA_TRY(cudaStreamSynchronize(t_stream));
    return 0;
}

int ozaki_get_stats(ozaki_stats_t *out) {
    if (!out) return -1;
    std::memset(out, 0, sizeof *out);
    out->dgemm_calls = g_stats.dgemm;
    out->zgemm_calls = g_stats.zgemm;
    out->zgemm3m_calls = g_stats.zgemm3m;
    out->batch_entries = g_stats.entries;
    out->int8_gemm_equiv = g_stats.equiv;
    out->int8_macs = g_stats.macs;
    out->k_chunks = g_stats.chunks;
    out->kernel_launches = g_stats.launches;
    out->crt_calls = g_stats.crt;
    uint64_t nf = 0;
    std::lock_guard<std::mutex> lk(g_mu);
    for (int d = 0; d < kMaxDev; ++d) {
        if (g_dev[d].init && g_dev[d].ok && g_dev[d].nonfinite) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(d);
            cudaDeviceSynchronize();
            unsigned long long v = 0;
            cudaMemcpy(&v, g_dev[d].nonfinite, sizeof v, cudaMemcpyDeviceToHost);
            nf += v - g_dev[d].nonfinite_base;
            cudaSetDevice(cur);
        }
    }
    out->nonfinite_rows = nf;
    return 0;
}

int ozaki_reset_stats(void) {
    g_stats.dgemm = 0;
    g_stats.zgemm = 0;
    g_stats.zgemm3m = 0;
    g_stats.entries = 0;
    g_stats.equiv = 0;
    g_stats.macs = 0;
    g_stats.chunks = 0;
    g_stats.launches = 0;
    std::lock_guard<std::mutex> lk(g_mu);
    for (int d = 0; d < kMaxDev; ++d) {
        if (g_dev[d].init && g_dev[d].ok && g_dev[d].nonfinite) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(d);
            cudaDeviceSynchronize();
            unsigned long long v = 0;
            cudaMemcpy(&v, g_dev[d].nonfinite, sizeof v, cudaMemcpyDeviceToHost);
            g_dev[d].nonfinite_base = v;
            cudaSetDevice(cur);
        }
    }
    return 0;
}

int64_t ozaki_workspace_size(char kind, int64_t m, int64_t n, int64_t k, int64_t batch,
                             int num_slices) {
    if (m < 0 || n < 0 || k < 0 || batch < 0 || num_slices < 1 || num_slices > 16) return -1;
    Plan P;
    const Kind kd = kind == 'z' ? KIND_4M : KIND_REAL;
    if (make_plan(kd, m, n, k, batch, num_slices, P)) return -1;
    int64_t ws = (int64_t)plan_workspace(P);
    if (kind == '3') ws += 3 * (int64_t)al256(sizeof(double) * m * n * batch);
    return ws;
}

const char *ozaki_last_error(void) { return t_err.c_str(); }

int ozaki_profile_enable(int on) {
    g_prof_on.store(on ? 1 : 0);
    return 0;
}

int ozaki_profile_read(ozaki_profile_t *out) {
    if (!out) return -1;
    std::memset(out, 0, sizeof *out);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    int rc = 0;
    for (const ProfRec &r : g_prof_recs) {
        float ms = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess)
            rc = OZAKI_ERR_CUDA;
        out->ms[r.phase] += ms;
        out->launches[r.phase] += 1;
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    return rc;
}

const char *ozaki_version(void) { return "ozaki-b200 0.1 (sm_100a, tcgen05 kind::i8)"; }

int ozaki_debug_split(char side, char kind, char trans, int64_t rows, int64_t cols,
                      const double *X, int64_t ldx, int num_slices, int8_t *slices_out,
                      int32_t *exps_out, int64_t *kdepth_out) {
    env_refresh();
    t_err.clear();
    side = up(side);
    trans = up(trans);
    if (side != 'A' && side != 'B') return fail(-1, "side");
    int mode;
    switch (kind) {
        case 'd': mode = SPLIT_REAL; break;
        case 'z': mode = side == 'A' ? SPLIT_A4M : SPLIT_B4M; break;
        case 'r': mode = SPLIT_RE; break;
        case 'i': mode = SPLIT_IM; break;
        case 's': mode = SPLIT_SUM; break;
        default: return fail(-2, "kind");
    }
    if (!trans_ok(trans)) return fail(-3, "trans");
    if (rows < 0) return fail(-4, "rows");
    if (cols < 0) return fail(-5, "cols");
    if (num_slices < 1 || num_slices > 16) return fail(-8, "num_slices");
    if (mode == SPLIT_REAL && trans == 'C') trans = 'T';
    DevState *dev = nullptr;
    if (int rc = device_state(&dev)) return rc;
    cudaStream_t st = t_stream;
    // describe the operand as side A (m = rows, k = cols) or side B (n = rows, k = cols)
    Plan P;
    const Kind pk = (kind == 'z') ? KIND_4M : KIND_REAL;
    if (int rc = make_plan(pk, side == 'A' ? rows : 1, side == 'B' ? rows : 1, cols, 1, num_slices, P)) return rc;
    const int64_t stored_rows = (side == 'A') == (trans == 'N') ? rows : cols;
    if (ldx < std::max<int64_t>(1, stored_rows)) return fail(-7, "ldx");
    const bool sideA = side == 'A';
    Operand op = sideA ? view_A(X, trans, rows, cols, ldx, 0, mode) : view_B(X, trans, rows, cols, ldx, 0, mode);
    const size_t sl_bytes = sideA ? P.a_bytes : P.b_bytes;
    const int64_t rows_out = (mode == SPLIT_B4M) ? 2 * rows : rows;
    void *base = nullptr;
    CUDA_TRY(cudaMallocAsync(&base, sl_bytes + al256(4 * (rows_out + 1)), st));
    int8_t *sl = (int8_t *)base;
    int32_t *ex = (int32_t *)(sl + sl_bytes);
    int rc = launch_split(P, op, sideA, sl, ex, dev, st);
    const int64_t kdepth = (mode == SPLIT_A4M || mode == SPLIT_B4M) ? P.Kp : cols;
    if (!rc && rows_out > 0 && kdepth > 0) {
        const int64_t total = (int64_t)num_slices * rows_out * kdepth;
        k_unpack<<<grid1d(total, dev->sms), 256, 0, st>>>(sl, slices_out, rows_out, kdepth, num_slices,
                                                        sideA ? P.a_tile_h : P.b_tile_h, P.KB);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "unpack: %s", cudaGetErrorString(e));
        if (!rc && exps_out) {
            e = cudaMemcpyAsync(exps_out, ex, 4 * rows_out, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) rc = fail(OZAKI_ERR_CUDA, "copy exps: %s", cudaGetErrorString(e));
        }
    }
    cudaFreeAsync(base, st);
    if (kdepth_out) *kdepth_out = kdepth;
    return rc;
}

int ozaki_debug_timing(int enable, uint64_t *out, int nslots) {
    g_dbg_on.store(enable ? 1 : 0);
    if (out && g_dbg) {
        CUDA_TRY(cudaDeviceSynchronize());
        unsigned long long h[DBG_NSLOT] = {0};
        CUDA_TRY(cudaMemcpy(h, g_dbg, sizeof h, cudaMemcpyDeviceToHost));
        for (int i = 0; i < nslots && i < DBG_NSLOT; ++i) out[i] = h[i];
        CUDA_TRY(cudaMemset(g_dbg, 0, sizeof h));
    }
    return DBG_NSLOT;
}

int ozaki_debug_level_sums(char transa, char transb, int64_t m, int64_t n, int64_t k,
                           const double *A, int64_t lda, const double *B, int64_t ldb,
                           int num_slices, int32_t *S_out) {
    const double al[2] = {1.0, 0.0}, be[2] = {0.0, 0.0};
    Call c = make_call(KIND_REAL, transa, transb, m, n, k, al, A, lda, 0, B, ldb, 0, be, nullptr,
                       std::max<int64_t>(1, m), 0, 1, num_slices, false);
    c.S_out = S_out;
    if (!S_out) return fail(-11, "S_out");
    return run(c);
}

}  // extern "C"
