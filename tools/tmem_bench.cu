// tmem_bench.cu -- measure tcgen05.ld / tcgen05.st throughput (bytes/clk/SM) and DFMA latency on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>  // 0 = ld, 1 = st, 2 = ld+st
__global__ void tmem_kernel(int iters, unsigned long long *cyc, float *sink)
{
    __shared__ unsigned taddr_s;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned base = taddr_s + ((unsigned)(32 * (warp % 4)) << 16) + (unsigned)((warp / 4) * 128);
    unsigned r[16];
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x + i;
    float acc = 0.f;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned a = base + (unsigned)((it & 7) * 16);
        if (MODE != 0) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
        }
        if (MODE != 1) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(a));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += __uint_as_float(r[it & 15]);
        } else {
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

__global__ void dfma_lat(int iters, unsigned long long *cyc, double *sink)
{
    double x = threadIdx.x * 1e-3;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, 1.0000001, 1e-9);
    unsigned long long t1 = clock64();
    cyc[0] = t1 - t0;
    sink[0] = x;
}

template <int MODE>
void run(const char *name, int threads, unsigned long long *dc, float *sink)
{
    const int iters = 4096;
    tmem_kernel<MODE><<<148, threads>>>(iters, dc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += c[i] / 148.0;
    const double bytes = (double)threads * iters * 16 * 4 * (MODE == 2 ? 2 : 1);
    printf("%s threads %d: %s  %.1f B/clk/SM (%.0f cycles)\n", name, threads, cudaGetErrorString(e), bytes / mean, mean);
}

int main()
{
    unsigned long long *dc;
    float *sink;
    double *ds;
    cudaMalloc(&dc, 148 * 8);
    cudaMalloc(&sink, 148 * 1024 * 4);
    cudaMalloc(&ds, 8);
    for (int t : {128, 256}) {
        run<0>("tmem ld", t, dc, sink);
        run<1>("tmem st", t, dc, sink);
        run<2>("tmem ld+st", t, dc, sink);
    }
    dfma_lat<<<1, 1>>>(10000, dc, ds);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", c / 10000.0);
    return 0;
}
