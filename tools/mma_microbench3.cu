// mma_microbench.cu -- tcgen05.mma kind::i8 throughput vs smem layout / N / cta_group.
// Operands stay resident in shared memory; one thread issues `iters` x 8 MMAs
// into TMEM; we time with clock64 and report MACs per SM clock.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_29975_b200/csrc
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"

using namespace ozk;

__device__ __forceinline__ uint64_t desc_layout(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// LAYOUT: 0 = SWIZZLE_NONE (core matrices 8x16B, LBO 128, SBO 256)
//         1 = SWIZZLE_32B  (rows of 32 B, SBO 256)
//         2 = SWIZZLE_128B (rows of 128 B, K advance +32 B, SBO 1024)
template <int N, int LAYOUT, int NSLICE, int NACCR = 512 / N>
__global__ void __launch_bounds__(128, 1) mb(unsigned long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    constexpr int A_BYTES = 128 * 32;      // one slice of A for one K step (LAYOUT 0/1)
    constexpr int B_BYTES = N * 32;
    constexpr int A_REGION = (LAYOUT == 2) ? 128 * 128 : A_BYTES;   // SW128: 4 K-steps per tile
    constexpr int B_REGION = (LAYOUT == 2) ? N * 128 : B_BYTES;
    uint8_t *sA = smem;
    uint8_t *sB = smem + NSLICE * A_REGION;
    for (int i = threadIdx.x; i < (NSLICE * (A_REGION + B_REGION)) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = holder;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_i8(128, N);
        constexpr int NACC = NACCR;
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int sa = j % NSLICE, sb = (j * 3 + it) % NSLICE;
                uint64_t ad, bd;
                if (LAYOUT == 0) {
                    ad = desc_layout(a0 + sa * A_REGION, 128, 256, 0);
                    bd = desc_layout(b0 + sb * B_REGION, 128, 256, 0);
                } else if (LAYOUT == 1) {
                    ad = desc_layout(a0 + sa * A_REGION, 16, 256, 6);
                    bd = desc_layout(b0 + sb * B_REGION, 16, 256, 6);
                } else {
                    const int ks = (j + it) & 3;
                    ad = desc_layout(a0 + sa * A_REGION + ks * 32, 16, 1024, 2);
                    bd = desc_layout(b0 + sb * B_REGION + ks * 32, 16, 1024, 2);
                }
                mma_i8(tbase + (uint32_t)((j % NACC) * N), ad, bd, idesc, 1u);
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

template <int N, int LAYOUT, int NSLICE, int NACCR = 512 / N>
void run(const char *name, int sms) {
    int iters = 2000;
    constexpr int A_REGION = (LAYOUT == 2) ? 128 * 128 : 128 * 32;
    constexpr int B_REGION = (LAYOUT == 2) ? N * 128 : N * 32;
    size_t smem = NSLICE * (A_REGION + B_REGION) + 2048;
    cudaFuncSetAttribute(mb<N, LAYOUT, NSLICE, NACCR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned long long *d;
    cudaMalloc(&d, sms * sizeof(unsigned long long));
    mb<N, LAYOUT, NSLICE, NACCR><<<sms, 128, smem>>>(d, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mb<N, LAYOUT, NSLICE, NACCR><<<sms, 128, smem>>>(d, iters);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), d, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto v : h) avg += (double)v;
    avg /= sms;
    double macs = (double)iters * 8 * 128 * N * 32;
    printf("%-28s N=%3d slices=%d: %7.1f MAC/clk/SM  (%6.1f clk per MMA)  chip %7.1f TOPS  %s\n", name, N,
           NSLICE, macs / avg, avg / (iters * 8.0), 2 * macs * sms / (ms * 1e-3) / 1e12,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<128, 0, 8, 1>("N128 1 accumulator", sms);
    run<128, 0, 8, 2>("N128 2 accumulators", sms);
    run<128, 0, 8, 4>("N128 4 accumulators", sms);
    run<256, 0, 4, 1>("N256 1 accumulator", sms);
    run<256, 0, 4, 2>("N256 2 accumulators", sms);
    run<64, 0, 8, 1>("N64 1 accumulator", sms);
    return 0;
}
