// tca_fused.cuh -- fused banded operator apply (one HBM pass), see tca_fused.cu.
#pragma once
#include "tca_internal.cuh"

namespace tca {
bool fused_apply_supported(const tca_operator *op);
tca_status launch_fused_apply(const tca_operator *op, const void *x, void *y,
                              const int32_t *done, cudaStream_t s);
}  // namespace tca
