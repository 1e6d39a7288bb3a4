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
}  // namespace tca
