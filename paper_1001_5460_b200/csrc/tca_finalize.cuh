// tca_finalize.cuh -- the scalar steps of Fig. 2 between
// the vector passes: alpha := rho / <p, q>, rho1 := <r, r>, the stop test and
// beta, with the breakdown / non-finite guards.  One source for
// the stand-alone finaliser kernel (tca_kernels.cu) and for the "last CTA"
// epilogues that run it inside the producing kernel (the fused apply's
// <p, q>, cg_update_r's <r, r>): the CTA that arrives last at a device
// counter sums the per-CTA partials in the same fixed order as the kernel
// (deterministic) and updates the scalars, which removes one launch and its
// graph-node gap per reduction.
#pragma once

#include "tca_internal.cuh"

namespace tca {

// which: 0 rho := <r0, r0> (start), 1 alpha, 2 rho1 / stop / beta, 3 PCG beta,
// 4 PCG start, 8 warm-start reference; s = the reduced dot product.  Thread 0.
__device__ __forceinline__ void cg_finalize_scalars(int which, double s, CgScalars *sc, double *hist)
{
    if (which == 8) {                      // warm start: stop reference <b, b> (reading Z28)
        sc->ref = s;
        return;
    }
    if (which == 0) {                      // rho := R+*R
        sc->rho = s;
        sc->rho0 = s;
        sc->ref = s;
        sc->rr = s;
        sc->iters = 0;
        sc->converged = 0;
        sc->status = TCA_OK;
        sc->done = 0;
        sc->xupd = 0;
        if (hist) hist[0] = s;
        if (!isfinite(s)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; }
        else if (s == 0.0) { sc->converged = 1; sc->done = 1; }
        else if (sc->max_iters <= 0) { sc->done = 1; if (sc->rtol2 > 0.0) sc->status = TCA_NOT_CONVERGED; }
    } else if (which == 1) {               // alpha := rho / (P+*Q)
        sc->pq = s;
        sc->xupd = 0;
        if (!isfinite(s)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; }
        else if (!(s > 0.0)) { sc->status = TCA_ERR_BREAKDOWN; sc->done = 1; }
        else { sc->alpha = sc->rho / s; sc->xupd = 1; }
    } else if (which == 2) {               // rho1 := R+*R (PCG: rr); stop test; CG: beta
        const int k = sc->iters + 1;
        sc->iters = k;
        sc->rr = s;
        if (hist) hist[k] = s;
        if (!isfinite(s)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; if (!sc->pcg) sc->rho = s; return; }
        if (s == 0.0) { sc->converged = 1; sc->done = 1; if (!sc->pcg) sc->rho = s; return; }   // Z12
        if (sc->rtol2 > 0.0 && s <= sc->rtol2 * sc->ref) {                                    // Z1, Z2, Z28
            sc->converged = 1; sc->done = 1; if (!sc->pcg) sc->rho = s; return;
        }
        if (k >= sc->max_iters) {
            sc->done = 1;
            if (!sc->pcg) sc->rho = s;
            if (sc->rtol2 > 0.0) sc->status = TCA_NOT_CONVERGED;
            return;
        }
        if (!sc->pcg) {
            sc->beta = s / sc->rho;
            sc->rho = s;
        }
    } else if (which == 3) {               // PCG: rho1 := R+*Z; beta
        if (!isfinite(s)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
        if (!(s > 0.0)) { sc->status = TCA_ERR_BREAKDOWN; sc->done = 1; return; }
        sc->beta = s / sc->rho;
        sc->rho = s;
    } else {                               // 4, PCG start: rho := R+*Z (R = B, Z = P^-1 B)
        if (!isfinite(s)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
        if (!(s > 0.0)) { sc->status = TCA_ERR_BREAKDOWN; sc->done = 1; return; }
        sc->rho = s;
    }
}

// Fixed-order sum of nparts partials by a block of exactly kRedThreads threads
// (the stand-alone finaliser's order); red: kRedThreads / 32 doubles of shared
// memory.  Result in thread 0.
__device__ __forceinline__ double fin_block_sum(const double *part, int nparts, double *red)
{
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kRedThreads) acc += __ldcg(part + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < kRedThreads / 32; ++i) s += red[i];
    }
    __syncthreads();
    return s;
}

// "Last CTA" epilogue of a producer kernel with kRedThreads threads per CTA
// whose thread 0 has written part[blockIdx.x]: the last CTA to arrive at
// sc->fin_cnt[slot] runs finaliser `which` over the gridDim.x partials and
// re-arms the counter.  Every thread of the CTA must call it.  red: shared
// memory for kRedThreads / 32 doubles and one int flag.
__device__ __forceinline__ void fin_last_cta(int which, int slot, const double *part, CgScalars *sc, double *hist,
                                             double *red)
{
    volatile int *last = reinterpret_cast<volatile int *>(red + kRedThreads / 32);
    if (threadIdx.x == 0) {
        __threadfence();   // this CTA's partial before its arrival
        *last = atomicAdd(&sc->fin_cnt[slot], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!*last) return;
    __threadfence();       // every partial (each written before its CTA's arrival)
    const double s = fin_block_sum(part, gridDim.x, red);
    if (threadIdx.x == 0) {
        cg_finalize_scalars(which, s, sc, hist);
        sc->fin_cnt[slot] = 0u;
    }
}

}  // namespace tca
