// tma_test.cu -- standalone check of the TMA/mbarrier PTX helpers used by the fused apply.
#include <cstdio>
#include <vector>
#include <cudaTypedefs.h>
#include "../paper_1001_5460_b200/csrc/tca_fused_impl.cuh"

namespace tca {
tca_status fail(tca_status s, const std::string &) { return s; }
tca_status cuda_fail(cudaError_t, const char *) { return TCA_ERR_CUDA; }
std::atomic<int64_t> g_launches{0};
}

using namespace tca::fused;

template <int BOXW>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap *gmap, double *out, int useg)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bar = (uint64_t *)sm;
    double *buf = (double *)(sm + 1024);
    int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncthreads();
    if (tid < 32) {
        if (tid == 0) mbar_arrive_expect_tx(bar, 2 * 14 * BOXW * 8);
        __syncwarp();
        if (tid < 28) {
            int r = tid >> 1, h = tid & 1;
            tma_load_3d(buf + r * 2 * BOXW + h * BOXW, useg ? gmap : &map, bar, -45 + h * BOXW, -3 + r, 0);
        }
    }
    mbar_wait(bar, 0);
    for (int i = tid; i < 14 * 2 * BOXW; i += blockDim.x) out[i] = buf[i];
}

template <int BOXW>
int run(PFN_cuTensorMapEncodeTiled_v12000 enc, double *d, double *o, const std::vector<double> &h, int useg)
{
    const int n1 = 4, n2 = 128, n3n4 = 1920;
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)n3n4, (cuuint64_t)n2, (cuuint64_t)n1};
    cuuint64_t str[2] = {(cuuint64_t)n3n4 * 8, (cuuint64_t)n2 * n3n4 * 8};
    cuuint32_t box[3] = {BOXW, 1, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap *gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    size_t smem = 1024 + 14 * 2 * BOXW * 8;
    cudaFuncSetAttribute(k<BOXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<BOXW><<<1, 128, smem>>>(m, gm, o, useg);
    cudaError_t e = cudaDeviceSynchronize();
    printf("BOXW %d useg %d encode %d: %s\n", BOXW, useg, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<double> got(14 * 2 * BOXW);
    cudaMemcpy(got.data(), o, got.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 14; ++rr)
        for (int c = 0; c < 2 * BOXW; ++c) {
            int g2 = -3 + rr, f = -45 + c;
            double want = (g2 >= 0 && f >= 0 && f < n3n4) ? h[(size_t)g2 * n3n4 + f] : 0.0;
            if (got[rr * 2 * BOXW + c] != want) bad++;
        }
    printf("  mismatches %d\n", bad);
    return 0;
}

int main(int argc, char **argv)
{
    const int n1 = 4, n2 = 128, n3n4 = 1920;
    std::vector<double> h((size_t)n1 * n2 * n3n4);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 14 * 512 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    int which = argc > 1 ? atoi(argv[1]) : 0;
    if (which == 0) return run<176>(enc, d, o, h, 0);
    if (which == 1) return run<176>(enc, d, o, h, 1);
    if (which == 2) return run<166>(enc, d, o, h, 1);
    return run<166>(enc, d, o, h, 0);
}
