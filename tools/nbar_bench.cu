// nbar_bench.cu -- cost of the v2 apply's named-barrier pipeline skeleton (A -> B -> C, double buffers)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
template <int NA, int NB, int NC, int MODE>
__global__ void k(int steps, long long *out)
{
    const int warp = threadIdx.x >> 5;
    long long t0 = clock64();
    if (warp < NA / 32) {
        for (int g = 0; g < steps; ++g) {
            const int b = g & 1;
            if (g >= 2) nb_sync(5 + b, NA + NC);
            nb_arrive(1 + b, NA + NB);
            if (MODE & 1) nb_sync(9, NA);
        }
    } else if (warp < (NA + NB) / 32) {
        for (int g = 0; g < steps; ++g) {
            const int b = g & 1;
            nb_sync(1 + b, NA + NB);
            if (g >= 2) nb_sync(7 + b, NB + NC);
            nb_arrive(3 + b, NB + NC);
        }
    } else {
        for (int g = 0; g < steps; ++g) {
            const int b = g & 1;
            nb_sync(3 + b, NB + NC);
            if (g + 2 < steps) { nb_arrive(5 + b, NA + NC); nb_arrive(7 + b, NB + NC); }
            if (MODE & 2) nb_sync(10, NC);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main()
{
    long long *d; cudaMalloc(&d, 148 * sizeof(long long)); long long h[148];
    const int steps = 2000;
#define R(NA, NB, NC, M) { k<NA, NB, NC, M><<<148, NA + NB + NC>>>(steps, d); cudaDeviceSynchronize(); \
    k<NA, NB, NC, M><<<148, NA + NB + NC>>>(steps, d); cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost); \
    printf("NA %d NB %d NC %d mode %d: %.1f cycles/step (%s)\n", NA, NB, NC, M, (double)h[0] / steps, cudaGetErrorString(cudaGetLastError())); }
    R(128, 128, 256, 0) R(128, 128, 256, 1) R(128, 128, 256, 2) R(128, 128, 256, 3) R(64, 64, 256, 3) R(32, 32, 64, 3)
    return 0;
}
