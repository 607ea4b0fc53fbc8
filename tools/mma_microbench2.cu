// mma_microbench2.cu -- cost model for the Ozaki slice GEMM on B200:
//  (1) SS-mode kind::i8 MMA time vs N and operand reuse (same / rotating A, B)
//  (2) TS-mode (A operand in TMEM) MMA time vs N
//  (3) tcgen05.cp 128x256b (smem -> TMEM) throughput
//  (4) L2 -> SMEM bulk-copy bandwidth with all SMs (L2-resident source)
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"

using namespace ozk;

__device__ __forceinline__ uint64_t dnone(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                 :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tc_cp(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" :: "r"(taddr), "l"(sdesc) : "memory");
}

// MODE 0: SS; 1: TS (A from TMEM); 2: tcgen05.cp only
template <int N, int MODE, int NA, int NB>
__global__ void __launch_bounds__(128, 1) mb(unsigned long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    uint8_t *sA = smem;
    uint8_t *sB = smem + 8 * 4096;
    for (int i = threadIdx.x; i < (8 * 4096 + 8 * N * 32) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = holder;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_i8(128, N);
        constexpr int ACC_COLS = (MODE == 1) ? 448 : 512;
        constexpr int NACC = ACC_COLS / N;
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        if (MODE == 1) {   // stage 8 A tiles into TMEM columns 448..511
            for (int j = 0; j < 8; ++j) tc_cp(tbase + 448 + 8 * j, dnone(a0 + j * 4096));
        }
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int sa = (j / (8 / NA)) % NA;   // NA distinct A per 8 MMAs (consecutive reuse)
                const int sb = (j + it) % NB;
                if (MODE == 0) {
                    mma_i8(tbase + (uint32_t)((j % NACC) * N), dnone(a0 + sa * 4096), dnone(b0 + sb * N * 32), idesc, 1u);
                } else if (MODE == 1) {
                    mma_ts(tbase + (uint32_t)((j % NACC) * N), tbase + 448 + 8 * sa, dnone(b0 + sb * N * 32), idesc, 1u);
                } else {
                    tc_cp(tbase + 8 * ((j + it) & 63), dnone(a0 + sa * 4096));
                }
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int N, int MODE, int NA, int NB>
void run(const char *name, int sms) {
    int iters = 2000;
    size_t smem = 8 * 4096 + 8 * N * 32 + 2048;
    cudaFuncSetAttribute(mb<N, MODE, NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned long long *d;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    mb<N, MODE, NA, NB><<<sms, 128, smem>>>(d, 10);
    mb<N, MODE, NA, NB><<<sms, 128, smem>>>(d, iters);
    cudaError_t err = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), d, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto v : h) avg += (double)v;
    avg /= sms;
    double per = avg / (iters * 8.0);
    if (MODE == 2)
        printf("%-34s            : %7.1f clk per 4KB cp (%.1f B/clk)  %s\n", name, per, 4096 / per,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
    else
        printf("%-34s N=%3d A%d B%d: %7.1f clk per MMA  %7.1f MAC/clk/SM  %s\n", name, N, NA, NB, per,
               128.0 * N * 32 / per, err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(d);
}

// ---- L2 -> SMEM bulk copy bandwidth
__global__ void __launch_bounds__(32, 1) l2bw(const uint8_t *src, size_t span, int chunk, int iters,
                                             unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bars[4];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    size_t off = ((size_t)blockIdx.x * 7919 * chunk) % span;
    unsigned long long t0 = clock64();
    uint32_t phase[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        int s = it & 3;
        if (it >= 4) { mbar_wait(&bars[s], phase[s]); phase[s] ^= 1; }
        mbar_arrive_expect_tx(&bars[s], chunk);
        bulk_g2s(smem + s * chunk, src + off, chunk, &bars[s]);
        off += chunk;
        if (off + chunk > span) off = 0;
    }
    for (int s = 0; s < 4; ++s) { mbar_wait(&bars[s], phase[s]); }
    out[blockIdx.x] = clock64() - t0;
}

void run_l2(int sms, size_t span, int chunk, int ctas_per_sm) {
    uint8_t *src;
    cudaMalloc(&src, span);
    cudaMemset(src, 1, span);
    unsigned long long *d;
    int grid = sms * ctas_per_sm;
    cudaMalloc(&d, grid * 8);
    int iters = 4000;
    size_t smem = 4 * chunk + 1024;
    cudaFuncSetAttribute(l2bw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    l2bw<<<grid, 32, smem>>>(src, span, chunk, 64, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    l2bw<<<grid, 32, smem>>>(src, span, chunk, iters, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)grid * iters * chunk;
    printf("bulk L2->SMEM span %4zu MB chunk %6d x%d/SM: %8.1f GB/s (%.1f B/clk/SM at 1.9GHz) %s\n", span >> 20, chunk,
           ctas_per_sm, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / sms / 1.9e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(src);
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, 0, 8, 8>("SS rotA rotB", sms);
    run<64, 0, 1, 8>("SS sameA rotB", sms);
    run<64, 0, 2, 8>("SS A x4 reuse", sms);
    run<64, 0, 1, 1>("SS sameA sameB", sms);
    run<128, 0, 8, 8>("SS rotA rotB", sms);
    run<128, 0, 1, 8>("SS sameA rotB", sms);
    run<96, 0, 8, 8>("SS rotA rotB", sms);
    run<256, 0, 8, 8>("SS rotA rotB", sms);
    run<32, 0, 1, 8>("SS sameA rotB", sms);
    run<32, 1, 8, 8>("TS rotA rotB", sms);
    run<48, 1, 8, 8>("TS rotA rotB", sms);
    run<64, 1, 8, 8>("TS rotA rotB", sms);
    run<64, 1, 1, 8>("TS sameA rotB", sms);
    run<64, 2, 8, 8>("tcgen05.cp 128x256b", sms);
    run_l2(sms, 64u << 20, 32768, 1);
    run_l2(sms, 64u << 20, 16384, 2);
    run_l2(sms, 64u << 20, 49152, 1);
    run_l2(sms, 1024u << 20, 32768, 1);
    return 0;
}
