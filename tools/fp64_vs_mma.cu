// Does scalar FP64 throughput drop while the SM's tensor core runs kind::i8 MMAs?
// warp 0: back-to-back tcgen05.mma (M=128,N=128,K=32, SMEM operands) for `mma_iters`
// warps 1..W: independent DFMA chains (or DADD / IMAD / I2F variants).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_29975_b200/csrc -o tools/fp64_mma tools/fp64_vs_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ozk;

template <int OP>
__global__ void k(int mma_on, int fp_iters, unsigned long long *out, double *sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&holder, 512);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) smem[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = holder;
    volatile __shared__ int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (warp == 0) {
        if (mma_on) {
            const uint64_t da = smem_desc_kmajor_noswz(smem_u32(smem), 128, 256);
            const uint64_t db = smem_desc_kmajor_noswz(smem_u32(smem + 4096), 128, 256);
            constexpr uint32_t idesc = idesc_i8(128, 128);
            long long t0 = clock64();
            int n = 0;
            while (!stop) {
#pragma unroll 1
                for (int r = 0; r < 64; ++r)
                    mma_i8_elect(tb + (uint32_t)((r & 3) * 128), da, db, idesc, 1u);
                n += 64;
                mma_commit_elect(&bar);
                mbar_wait(&bar, ((n / 64) - 1) & 1);
            }
            long long t1 = clock64();
            if (lane == 0) { atomicAdd(out + 2, (unsigned long long)n); atomicAdd(out + 3, (unsigned long long)(t1 - t0)); }
        }
    } else {
        double a[8];
        long long ia[8];
        for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; ia[i] = threadIdx.x + i; }
        long long t0 = clock64();
        for (int it = 0; it < fp_iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) a[i] = __fma_rn(a[i], 0.999, 0.5);
                else if (OP == 1) a[i] = __dadd_rn(a[i], 0.5);
                else if (OP == 2) a[i] = __dmul_rn(a[i], 0.999);
                else if (OP == 3) ia[i] = ia[i] * 3 + 7;   // IMAD.WIDE-ish
                else if (OP == 4) a[i] = __fmaf_rn((float)a[i], 0.999f, 0.5f);
                else if (OP == 5) ia[i] += __double_as_longlong((double)(int)ia[i]) >> 40;             // I2F.F64.S32
                else if (OP == 6) ia[i] += __double_as_longlong((double)(ia[i] | (1ll << 40))) >> 40;  // I2F.F64.S64
                else if (OP == 7) { a[i] = a[i] + 1.0; ia[i] += (long long)__double2ll_rz(a[i]); }  // F2I.S64
            }
        }
        long long t1 = clock64();
        if (lane == 0) atomicAdd(out + 0, (unsigned long long)(t1 - t0));
        if (lane == 0) atomicAdd(out + 1, 1ull);
        double s = 0; for (int i = 0; i < 8; ++i) s += a[i] + (double)ia[i];
        if (s == 1.2345) sink[0] = s;
    }
    __syncwarp();
    if (warp == 1) { __syncwarp(); if (lane == 0) stop = 1; }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
    unsigned long long *d; double *sink;
    cudaMalloc(&d, 32); cudaMalloc(&sink, 8);
    const char *names[] = {"DFMA", "DADD", "DMUL", "IMAD64", "FFMA32", "I2F.S32", "I2F.S64", "DADD+F2I"};
    for (int op = 0; op < 8; ++op)
    for (int mma = 0; mma < 2; ++mma) {
        auto f = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : op == 6 ? k<6> : k<7>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
        const int nw = 16, iters = 4000;
        f<<<148, (nw + 1) * 32, 16384>>>(mma, 10, d, sink);
        cudaMemset(d, 0, 32);
        f<<<148, (nw + 1) * 32, 16384>>>(mma, iters, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        double clk_per_warp = (double)h[0] / h[1];
        double ops_per_clk_sm = (double)iters * 8 * 32 * nw / clk_per_warp;
        printf("%-7s mma=%d: %s  %.1f lane-ops/clk/SM", names[op], mma, cudaGetErrorString(e), ops_per_clk_sm);
        if (mma && h[2]) printf("   MMA: %.1f clk per MMA", (double)h[3] / (148.0) / ((double)h[2] / 148.0));
        printf("\n");
    }
    return 0;
}
