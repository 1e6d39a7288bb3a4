// tma_test2.cu -- bisect the mbarrier / bulk-copy / TMA mechanics on sm_100a.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void v3(int *out)  // plain mbarrier arrive + wait
{
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
    if (threadIdx.x == 0) out[0] = 1;
}

__global__ void v1(const double *g, double *out)  // 1D bulk copy with complete_tx
{
    __shared__ __align__(128) double buf[256];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(2048) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf)), "l"(g), "r"(2048), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
    out[threadIdx.x] = buf[threadIdx.x];
}

__global__ void v2(const __grid_constant__ CUtensorMap map, double *out)  // 2D tensor copy
{
    __shared__ __align__(128) double buf[16 * 16];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(2048) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(su(buf)), "l"(&map), "r"(su(&bar)), "r"(0), "r"(0) : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
    out[threadIdx.x] = buf[threadIdx.x];
}

int main()
{
    double *g, *o;
    int *io;
    cudaMalloc(&g, 1 << 20);
    cudaMalloc(&o, 1 << 16);
    cudaMalloc(&io, 64);
    double h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = i;
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    v3<<<1, 32>>>(io);
    printf("v3 mbarrier: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    v1<<<1, 256>>>(g, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("v1 bulk: %s\n", cudaGetErrorString(e));
    if (e == cudaSuccess) {
        cudaMemcpy(h, o, 2048, cudaMemcpyDeviceToHost);
        printf("  v1 h[5]=%g h[255]=%g\n", h[5], h[255]);
    }
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap m;
    cuuint64_t dims[2] = {64, 64};
    cuuint64_t str[1] = {64 * 8};
    cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    v2<<<1, 256>>>(m, o);
    e = cudaDeviceSynchronize();
    printf("v2 tensor2d (encode %d): %s\n", (int)r, cudaGetErrorString(e));
    if (e == cudaSuccess) {
        cudaMemcpy(h, o, 2048, cudaMemcpyDeviceToHost);
        printf("  v2 h[17]=%g (want 65)\n", h[17]);
    }
    return 0;
}
