// tma_test3.cu -- bisect 3D TMA: box width, issuing lanes, negative coordinates.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void t3(const __grid_constant__ CUtensorMap map, double *out, int boxw, int lanes, int c0, int c1)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bar = (uint64_t *)sm;
    double *buf = (double *)(sm + 1024);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(lanes * boxw * 8) : "memory");
        __syncwarp();
        if (threadIdx.x < lanes) {
            int r = threadIdx.x;
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su(buf + r * boxw)), "l"(&map), "r"(su(bar)), "r"(c0), "r"(c1 + r), "r"(0) : "memory");
        }
    }
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < lanes * boxw; i += blockDim.x) out[i] = buf[i];
}

int main()
{
    const int n1 = 4, n2 = 128, n3n4 = 1920;
    double *g, *o;
    cudaMalloc(&g, (size_t)n1 * n2 * n3n4 * 8);
    cudaMalloc(&o, 1 << 20);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    struct Case { int boxw, lanes, c0, c1; } cases[] = {
        {16, 1, 0, 0}, {176, 1, 0, 0}, {16, 28, 0, 0}, {16, 1, -45, 0}, {16, 1, 0, -3}, {176, 14, -45, -3}, {256, 1, 0, 0}};
    for (auto c : cases) {
        CUtensorMap m;
        cuuint64_t dims[3] = {(cuuint64_t)n3n4, (cuuint64_t)n2, (cuuint64_t)n1};
        cuuint64_t str[2] = {(cuuint64_t)n3n4 * 8, (cuuint64_t)n2 * n3n4 * 8};
        cuuint32_t box[3] = {(cuuint32_t)c.boxw, 1, 1}, es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        size_t smem = 1024 + (size_t)c.lanes * c.boxw * 8;
        cudaFuncSetAttribute(t3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        t3<<<1, 128, smem>>>(m, o, c.boxw, c.lanes, c.c0, c.c1);
        cudaError_t e = cudaDeviceSynchronize();
        printf("box %d lanes %d c0 %d c1 %d encode %d -> %s\n", c.boxw, c.lanes, c.c0, c.c1, (int)r, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
