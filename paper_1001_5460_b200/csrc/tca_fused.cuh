// tca_fused.cuh -- fused banded operator apply (one HBM pass), see tca_band.cu.
#pragma once
#include "tca_internal.cuh"

namespace tca {
bool fused_shape_supported(const tca_operator *op);        // shape/band/tap-table eligibility
tca_status fused_prepare(tca_operator *op);                // build the kernel-parameter block
bool fused_pointers_ok(const void *x, const void *y);      // TMA alignment of the call's tensors
// pq_part (optional): the kernel writes one fp64 partial of <x, y> per CTA
// (op->band_grid entries) -- the CG <p, q> fused into the apply epilogue.
tca_status launch_fused_apply(const tca_operator *op, const void *x, void *y,
                              const int32_t *done, double *pq_part, cudaStream_t s);
// Fused CG step B1' (one GPU): C += alpha P_old (when sc->xupd), P_new = D +
// beta P_old, Q = A P_new, per-CTA <P_new, Q> partials (op->band_grid_fu);
// sc->done: only the pending C update.
bool fused_b1_supported(const tca_operator *op);
tca_status fused_b1_prepare(const tca_operator *op, const void *const *ptrs, const int *kinds, int n, cudaStream_t s);
tca_status launch_fused_b1(const tca_operator *op, const void *pold, void *pnew, const void *d, void *q, void *x,
                           double *pq_part, cudaStream_t s);
// Apply with the deferred C update (one GPU): Q = A P, per-CTA <P, Q> partials
// (op->band_grid_dx), C += alpha P_prev by a streaming warp when sc->xupd
// (sc->done: only that update).
bool fused_dx_supported(const tca_operator *op);
tca_status fused_dx_prepare(const tca_operator *op, const void *const *ptrs, const int *kinds, int n, cudaStream_t s);
tca_status launch_fused_dx(const tca_operator *op, const void *p, void *q, void *x, const void *pprev,
                           double *pq_part, cudaStream_t s);
}  // namespace tca
