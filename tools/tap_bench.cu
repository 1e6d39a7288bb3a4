// tap_bench.cu -- how to feed per-row band taps to DFMA on sm_100a.
// A "pass A" shaped loop: each thread holds NC columns of 14 values and
// computes per column 8 outputs x 7 taps (G) + 8 x 5 taps (R) = 96 DFMA;
// taps for the 8 rows are the same for every thread of the CTA and change
// per tile (runtime-uniform row base).
// Variants: 0 taps from smem (broadcast LDS), 1 taps from a
// __grid_constant__ kernel-param array (LDCU), 2 taps from a __constant__
// array (LDCU), 3 taps held in registers (loaded once before the loop).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tap_bench tap_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ROWS = 128;
struct Taps { double t[ROWS * 16]; };   // 16 KB of params
__constant__ double c_taps[ROWS * 16];

template <int V, int NC>
__global__ void __launch_bounds__(256) kern(const __grid_constant__ Taps P, int iters, int rowbase,
                                            double *out)
{
    __shared__ __align__(16) double s_taps[ROWS * 16];
    __shared__ double col[1024 * 4];
    for (int i = threadIdx.x; i < ROWS * 16; i += blockDim.x) s_taps[i] = P.t[i];
    for (int i = threadIdx.x; i < 1024 * 4; i += blockDim.x) col[i] = i * 1e-3;
    __syncthreads();
    double acc[NC][8];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[c][i] = 0;
    double treg[8][12];
    if (V == 3) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < 12; ++k) treg[i][k] = P.t[(rowbase + i) * 16 + k];
    }
    for (int it = 0; it < iters; ++it) {
        const int rb = (rowbase + (it & 7) * 8) & (ROWS - 8);   // uniform, runtime
        double v[NC][14];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int k = 0; k < 14; ++k) v[c][k] = col[((k + it) & 3) * 1024 + c * 256 + threadIdx.x] + k;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double t[12];
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                const int o = (rb + i) * 16 + (k < 7 ? k : k + 1);
                if (V == 0) t[k] = s_taps[o];
                else if (V == 1) t[k] = P.t[o];
                else if (V == 2) t[k] = c_taps[o];
                else if (V == 3) t[k] = treg[i][k];
                else t[k] = P.t[(3 + i) * 16 + (k < 7 ? k : k + 1)];
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                double g = t[0] * v[c][i];
#pragma unroll
                for (int k = 1; k < 7; ++k) g = fma(t[k], v[c][i + k], g);
                double r = t[7] * v[c][i + 1];
#pragma unroll
                for (int k = 1; k < 5; ++k) r = fma(t[7 + k], v[c][i + k + 1], r);
                acc[c][i] = fma(acc[c][i], 0.5, g + r);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < 8; ++i) s += acc[c][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DFMA latency / throughput vs independent chains per thread
template <int ILP>
__global__ void __launch_bounds__(512) chains(int iters, double a, double b, double *out)
{
    double r[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) r[i] = fma(r[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    Taps h;
    for (int i = 0; i < ROWS * 16; ++i) h.t[i] = 1.0 / (i + 1);
    cudaMemcpyToSymbol(c_taps, h.t, sizeof(h.t));
    double *out;
    cudaMalloc(&out, 148 * 8 * 512 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto fn) {
        fn();
        cudaEventRecord(a);
        fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    };
    const int iters = 1000;
    for (int bps = 1; bps <= 2; ++bps) {
        const int g = 148 * bps;
#define RUN(V, NC)                                                                                     \
    {                                                                                                  \
        float ms = timeit([&] { kern<V, NC><<<g, 256>>>(h, iters, 3, out); });                         \
        const double fma = 148.0 * bps * 256 * iters * 96 * NC;                                        \
        printf("ctas/SM %d variant %d cols %d: %.3f ms  %.2f TF/s\n", bps, V, NC, ms,                  \
               2 * fma / (ms * 1e-3) / 1e12);                                                          \
    }
        RUN(0, 1) RUN(1, 1) RUN(2, 1) RUN(3, 1)
        RUN(4, 1)
        RUN(0, 2) RUN(1, 2) RUN(2, 2) RUN(3, 2) RUN(4, 2)
        RUN(0, 4) RUN(1, 4) RUN(3, 4) RUN(4, 4)
    }
    for (int thr = 128; thr <= 512; thr *= 2) {
#define CH(ILP)                                                                                        \
    {                                                                                                  \
        float ms = timeit([&] { chains<ILP><<<148, thr>>>(4000, 1.0000001, 1e-9, out); });             \
        const double fma = 148.0 * thr * 4000 * ILP;                                                   \
        printf("chains thr/SM %d ILP %d: %.2f TF/s\n", thr, ILP, 2 * fma / (ms * 1e-3) / 1e12);         \
    }
        CH(1) CH(2) CH(4) CH(8) CH(16)
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
