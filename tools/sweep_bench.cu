// Microbenchmark (not product code): cycles per step of the banded forward
// substitution s_i = c0 x_i - c1 s_{i-1} - c2 s_{i-2} - c3 s_{i-3} in shared
// memory, as in tca_precond.cu's sweep, for three loop forms:
//   0: the product form (next step's loads before this step's store)
//   1: unrolled by 4 with register renaming, loads of the group first
//   2: two fibres per thread interleaved (product form per fibre)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/sweep_bench tools/sweep_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int LEN = 128, LB = 64, P = LB + 1;

template <int FORM>
__global__ void __launch_bounds__(256) sweep(double *out, long long *cyc, int reps)
{
    extern __shared__ double sm[];
    double *tb = sm;            // [LEN][8]
    double *v = sm + 8 * LEN;   // [LEN][P]  (FORM 2: two tiles)
    for (int k = threadIdx.x; k < 8 * LEN; k += blockDim.x) tb[k] = 0.1 + 1e-3 * (k % 7);
    const int ntile = FORM == 2 ? 2 : 1;
    for (int k = threadIdx.x; k < ntile * LEN * P; k += blockDim.x) v[k] = 1.0 + 1e-4 * (k % 13);
    __syncthreads();
    const int j = threadIdx.x;
    long long t0 = clock64();
    if (j < LB) {
        for (int rep = 0; rep < reps; ++rep) {
            if (FORM == 0) {
                double w1 = 0, w2 = 0, w3 = 0;
                double c0 = tb[0], c1 = tb[1], c2 = tb[2], c3 = tb[3], x0 = v[j];
                for (int i = 0; i < LEN; ++i) {
                    double n0 = 0, n1 = 0, n2 = 0, n3 = 0, xn = 0;
                    if (i + 1 < LEN) {
                        const double *cn = tb + 8 * (i + 1);
                        n0 = cn[0]; n1 = cn[1]; n2 = cn[2]; n3 = cn[3];
                        xn = v[(i + 1) * P + j];
                    }
                    const double s = fma(-c1, w1, fma(-c2, w2, fma(-c3, w3, c0 * x0)));
                    v[i * P + j] = s;
                    w3 = w2; w2 = w1; w1 = s;
                    c0 = n0; c1 = n1; c2 = n2; c3 = n3; x0 = xn;
                }
            } else if (FORM == 1) {
                double w1 = 0, w2 = 0, w3 = 0;
                for (int i0 = 0; i0 < LEN; i0 += 4) {
                    double x[4], c[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        x[u] = v[(i0 + u) * P + j];
                        const double2 a = *reinterpret_cast<const double2 *>(tb + 8 * (i0 + u));
                        const double2 b = *reinterpret_cast<const double2 *>(tb + 8 * (i0 + u) + 2);
                        c[u][0] = a.x; c[u][1] = a.y; c[u][2] = b.x; c[u][3] = b.y;
                    }
                    double s[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        s[u] = fma(-c[u][1], w1, fma(-c[u][2], w2, fma(-c[u][3], w3, c[u][0] * x[u])));
                        w3 = w2; w2 = w1; w1 = s[u];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[(i0 + u) * P + j] = s[u];
                }
            } else {
                double *v2 = v + LEN * P;
                double w1 = 0, w2 = 0, w3 = 0, y1 = 0, y2 = 0, y3 = 0;
                for (int i = 0; i < LEN; ++i) {
                    const double *cn = tb + 8 * i;
                    const double c0 = cn[0], c1 = cn[1], c2 = cn[2], c3 = cn[3];
                    const double xa = v[i * P + j], xb = v2[i * P + j];
                    const double s = fma(-c1, w1, fma(-c2, w2, fma(-c3, w3, c0 * xa)));
                    const double t = fma(-c1, y1, fma(-c2, y2, fma(-c3, y3, c0 * xb)));
                    v[i * P + j] = s;
                    v2[i * P + j] = t;
                    w3 = w2; w2 = w1; w1 = s;
                    y3 = y2; y2 = y1; y1 = t;
                }
            }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (j < LB) out[blockIdx.x * LB + j] = v[j];
}

template <int FORM>
void run(int blocks_per_sm)
{
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * blocks_per_sm, reps = 20;
    const size_t smem = (8 * LEN + (FORM == 2 ? 2 : 1) * LEN * P) * sizeof(double);
    cudaFuncSetAttribute(sweep<FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double *out;
    long long *cyc;
    cudaMalloc(&out, grid * LB * sizeof(double));
    cudaMalloc(&cyc, grid * sizeof(long long));
    sweep<FORM><<<grid, 256, smem>>>(out, cyc, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    sweep<FORM><<<grid, 256, smem>>>(out, cyc, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double fibres_steps = (double)grid * LB * (FORM == 2 ? 2 : 1) * LEN * reps;
    printf("form %d, %d blocks/SM (smem %zu KB): block0 %.1f cycles/step, %.2f ms, %.2f G fibre-steps/s\n", FORM,
           blocks_per_sm, smem / 1024, (double)c / (LEN * reps), ms, fibres_steps / (ms * 1e-3) / 1e9);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    cudaFree(out);
    cudaFree(cyc);
}

int main()
{
    run<0>(1);
    run<0>(3);
    run<1>(1);
    run<1>(3);
    run<2>(1);
    return 0;
}
