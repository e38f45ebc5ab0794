// Microbenchmark: fp64 FMA-pipe (DFMA) vs fp64 tensor (DMMA.8x8x4) throughput on one B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_fp64 tools/microbench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

__global__ void dfma_kernel(double *out, double s)
{
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-7);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
    if (r == 123.0) out[threadIdx.x] = r;
}

__global__ void dmma_kernel(double *out, double s)
{
    double c[8][2];
    double a = threadIdx.x * 1e-9 + s, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
    if (r == 123.0) out[threadIdx.x] = r;
}

int main()
{
    double *out;
    cudaMalloc(&out, 1 << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = sms * 2, threads = 32 * warps / 2;
        for (int k = 0; k < 2; ++k) {
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (k == 0) dfma_kernel<<<blocks, threads>>>(out, 0.999999);
                else dmma_kernel<<<blocks, threads>>>(out, 0.999999);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            const double fma_per = (k == 0) ? 8.0 * ITER : 8.0 * ITER * 256.0 / 32.0;  // per thread
            const double flops = 2.0 * fma_per * blocks * threads;
            printf("%s warps/SM=%2d  %.2f ms  %.1f TFLOP/s\n", k ? "DMMA" : "DFMA", warps, ms, flops / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
