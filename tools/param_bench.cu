// Microbenchmark (not product code): GPU time of an empty kernel launch as a
// function of its kernel-parameter block size (the fused apply passes ~27 KB of
// tap tables as parameters), timed with CUDA events around each launch, on a
// stream and inside a CUDA graph.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/param_bench tools/param_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES>
struct Blob {
    double v[BYTES / 8];
};

template <int BYTES>
__global__ void empty_kernel(const __grid_constant__ Blob<BYTES> b, double *out)
{
    if (threadIdx.x == 0 && blockIdx.x == 0 && b.v[0] == 12345.0) out[0] = b.v[BYTES / 8 - 1];
}

template <int BYTES>
void run(int grid)
{
    Blob<BYTES> b{};
    double *out;
    cudaMalloc(&out, 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 10; ++i) empty_kernel<BYTES><<<grid, 256, 0, s>>>(b, out);
    cudaStreamSynchronize(s);
    // stream launches, events around each
    float tot = 0.f;
    const int reps = 200;
    for (int i = 0; i < reps; ++i) {
        cudaEventRecord(e0, s);
        empty_kernel<BYTES><<<grid, 256, 0, s>>>(b, out);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
    }
    // back-to-back stream launches (throughput)
    cudaEventRecord(e0, s);
    for (int i = 0; i < reps; ++i) empty_kernel<BYTES><<<grid, 256, 0, s>>>(b, out);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float bb;
    cudaEventElapsedTime(&bb, e0, e1);
    // graph of `reps` launches
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < reps; ++i) empty_kernel<BYTES><<<grid, 256, 0, s>>>(b, out);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float gm;
    cudaEventElapsedTime(&gm, e0, e1);
    printf("param %6d B, grid %4d: event-bracketed %.2f us, back-to-back %.2f us/launch, graph %.2f us/launch\n", BYTES,
           grid, 1e3 * tot / reps, 1e3 * bb / reps, 1e3 * gm / reps);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(out);
}

int main()
{
    run<1024>(296);
    run<8192>(296);
    run<16384>(296);
    run<28672>(296);
    run<32000>(296);
    return 0;
}
