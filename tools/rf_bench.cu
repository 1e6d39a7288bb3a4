// rf_bench.cu -- DFMA throughput vs number of register-file source operands (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
// NOPS = number of distinct 64-bit RF sources per DFMA (1: fma(r,c1,c2); 2: fma(x,c,r); 3: fma(x,y,r))
template <int NOPS, int ILP>
__global__ void __launch_bounds__(512) k(int iters, double a, double b, double *out)
{
    double r[ILP], x[ILP], y[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { r[i] = threadIdx.x * 1e-3 + i; x[i] = 1.0 + i * 1e-9 + a * threadIdx.x; y[i] = b * i + 1e-3 * threadIdx.y; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (NOPS == 1) r[i] = fma(r[i], a, b);
            else if (NOPS == 2) r[i] = fma(x[i], a, r[i]);
            else r[i] = fma(x[i], y[(i + 1) % ILP], r[i]);
        }
#pragma unroll
        for (int i = 0; i < ILP; ++i) { if (NOPS == 3) { double t = x[i]; x[i] = y[i]; y[i] = t; } }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += r[i] + x[i] + y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main()
{
    double *out;
    cudaMalloc(&out, 148 * 8 * 512 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int thr = 256; thr <= 512; thr *= 2) {
#define R(N, I)                                                                              \
    {                                                                                        \
        k<N, I><<<148, thr>>>(2000, 1.0000001, 1e-9, out);                                   \
        cudaEventRecord(a);                                                                  \
        k<N, I><<<148, thr>>>(2000, 1.0000001, 1e-9, out);                                   \
        cudaEventRecord(b);                                                                  \
        cudaEventSynchronize(b);                                                             \
        float ms;                                                                            \
        cudaEventElapsedTime(&ms, a, b);                                                     \
        printf("thr %d rf-operands %d ILP %d: %.2f TF/s\n", thr, N, I,                       \
               2.0 * 148 * thr * 2000.0 * I / (ms * 1e-3) / 1e12);                           \
    }
        R(1, 8) R(2, 8) R(3, 8) R(1, 16) R(2, 16) R(3, 16)
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
