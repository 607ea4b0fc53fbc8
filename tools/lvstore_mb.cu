// Microbenchmark of the pair GEMM's final store (lv_store) in isolation: one CTA of 576
// threads whose 16 "epilogue" warps each store 32 rows x 32 product columns, as in
// k_gemm_lv2's last tile.  Prints cycles per warp for variants (debug aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      -I include -I paper_2603_29975_b200/csrc tools/lvstore_mb.cu -o /tmp/lvstore_mb
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "gemm_lv2.cuh"

using namespace ozk;

__device__ __forceinline__ void bulk_store(void *gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int EPI, int MODE>
__global__ void __launch_bounds__(576, 1) k_mb(GemmParams p, unsigned long long *out, int reps) {
    extern __shared__ __align__(1024) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < 2) return;
    const int ew = warp - 2, q = warp & 3, half = ew >> 2;
    const int64_t grow = q * 32 + lane;
    double acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 1.0 + 1e-3 * (i + lane);
    const int32_t e = (grow < p.Mp) ? __ldg(p.ea + grow) : 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) lv_store<EPI, 32>(p, 0, grow, e, half * 32, acc, 0);
        if (MODE == 1) {   // plain stores only
            double *cp = p.C + grow + half * 32 * p.ldc;
#pragma unroll
            for (int j = 0; j < 32; ++j) cp[(int64_t)j * p.ldc] = acc[j];
        }
        if (MODE == 2) {   // stage column segments in SMEM, one bulk copy per (column, 32 rows)
            // smem tile column-major [128 cols][128 rows]; this warp: rows q*32.., cols half*32..
            double *st = sm + (int64_t)(half * 32) * 128 + q * 32 + lane;
#pragma unroll
            for (int j = 0; j < 32; ++j) st[j * 128] = acc[j];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane < 32) {   // each lane issues one column's 256-B segment
                const int j = lane;
                const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm + (int64_t)(half * 32 + j) * 128 + q * 32);
                bulk_store(p.C + q * 32 + (half * 32 + j) * p.ldc, src, 256);
            }
            bulk_commit_wait();
            __syncwarp();
        }
        acc[0] += 1.0;
    }
    const long long t1 = clock64();
    if (lane == 0) out[ew] = (unsigned long long)(t1 - t0);
}

int main() {
    const int M = 128, N = 128;
    GemmParams p{};
    double *C;
    int32_t *ea, *fb;
    unsigned long long *out;
    cudaMalloc(&C, sizeof(double) * 2 * M * N);
    cudaMalloc(&ea, 4 * M);
    cudaMalloc(&fb, 4 * N);
    cudaMalloc(&out, 8 * 16);
    cudaMemset(ea, 0, 4 * M);
    cudaMemset(fb, 0, 4 * N);
    p.C = C; p.ea = ea; p.fb = fb; p.Mp = M; p.N = N; p.ldc = M; p.strideC = 0; p.ab_unit = 1;
    p.alpha_r = 1.0; p.batch = 1; p.splitk = 1;
    unsigned long long h[16];
    for (int reps : {1, 10}) {
        k_mb<EPI_REAL, 0><<<1, 576>>>(p, out, reps); cudaDeviceSynchronize();
        k_mb<EPI_REAL, 0><<<1, 576>>>(p, out, reps); cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        printf("real lv_store  reps=%d cycles/warp/rep: %.0f (warp0) %.0f (warp15)\n", reps, (double)h[0] / reps, (double)h[15] / reps);
        k_mb<EPI_REAL, 1><<<1, 576>>>(p, out, reps); cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        printf("real plain st  reps=%d cycles/warp/rep: %.0f %.0f\n", reps, (double)h[0] / reps, (double)h[15] / reps);
        p.ldc = M;
        k_mb<EPI_CPLX4M, 0><<<1, 576>>>(p, out, reps); cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        printf("cplx lv_store  reps=%d cycles/warp/rep: %.0f %.0f\n", reps, (double)h[0] / reps, (double)h[15] / reps);
        cudaFuncSetAttribute(k_mb<EPI_REAL, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8);
        k_mb<EPI_REAL, 2><<<1, 576, 128 * 128 * 8>>>(p, out, reps); cudaDeviceSynchronize();
        k_mb<EPI_REAL, 2><<<1, 576, 128 * 128 * 8>>>(p, out, reps); cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        printf("smem + bulk   reps=%d cycles/warp/rep: %.0f %.0f\n", reps, (double)h[0] / reps, (double)h[15] / reps);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
