// fp64_peak.cu -- microbenchmark: DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on sm_100a,
// alone and interleaved in one warp, to decide whether the banded apply can use
// the FP64 tensor pipe alongside DFMA.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double *out, double a, double b)
{
    double r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += r[i];
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double *out, double a, double b)
{
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void mixed_kernel(double *out, double a, double b)
{
    double c[8][2];
    double r[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += r[i];
    if (s == 12345.678) out[0] = s;
}

template <typename K>
float timeit(K k, int blocks, int threads, double *out)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main()
{
    double *out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int threads : {128, 256, 512}) {
        int blocks = sms * 4;
        double nthr = (double)blocks * threads;
        float t1 = timeit(dfma_kernel, blocks, threads, out);
        double f1 = nthr * ITERS * 16 * 2 / (t1 * 1e-3) / 1e12;
        float t2 = timeit(dmma_kernel, blocks, threads, out);
        // m8n8k4: 8*8*4 = 256 MAC per warp-instruction
        double f2 = (nthr / 32) * ITERS * 8 * 256 * 2 / (t2 * 1e-3) / 1e12;
        float t3 = timeit(mixed_kernel, blocks, threads, out);
        double f3 = ((nthr / 32) * ITERS * 8 * 256 * 2 + nthr * ITERS * 16 * 2) / (t3 * 1e-3) / 1e12;
        printf("threads/blk %d: DFMA %.2f TF/s (%.3f ms) | DMMA %.2f TF/s (%.3f ms) | mixed %.2f TF/s (%.3f ms)\n",
               threads, f1, t1, f2, t2, f3, t3);
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
