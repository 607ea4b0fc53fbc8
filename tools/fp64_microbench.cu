// fp64_microbench.cu -- per-SM throughput of DFMA / DADD / I2F.F64 / F2I.S64 / IADD3 on B200.
#include <cstdio>
#include <cstdint>
template <int OP>
__global__ void k(double *out, int iters) {
    double a[8];
    long long li[8];
    int ii[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; li[i] = threadIdx.x + i; ii[i] = threadIdx.x * 3 + i; }
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = __fma_rn(a[i], b, c);
            if (OP == 1) a[i] = __dadd_rn(a[i], c);
            if (OP == 2) a[i] = __int2double_rn(ii[i] + it) + a[i] * 0.0;
            if (OP == 3) li[i] = __double2ll_rn(a[i] + (double)it);
            if (OP == 4) ii[i] = ii[i] * 3 + it;
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + (double)li[i] + ii[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char *name, int sms) {
    double *d; cudaMalloc(&d, sizeof(double) * sms * 8 * 1024);
    int iters = 4096;
    k<OP><<<sms * 4, 256>>>(d, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<sms * 4, 256>>>(d, iters);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = (double)sms * 4 * 256 * iters * 8;
    printf("%-10s %8.2f Gop/s  %6.1f ops/clk/SM (at %.0f MHz)\n", name, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
    cudaFree(d);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("DFMA", sms); run<1>("DADD", sms); run<2>("I2F.F64", sms); run<3>("F2I.S64", sms); run<4>("IMAD", sms);
}
