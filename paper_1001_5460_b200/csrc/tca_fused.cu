// tca_fused.cu -- fused banded apply (placeholder until the streaming kernel lands).
#include "tca_fused.cuh"

namespace tca {
bool fused_apply_supported(const tca_operator *) { return false; }
tca_status launch_fused_apply(const tca_operator *, const void *, void *, const int32_t *,
                              cudaStream_t)
{
    return fail(TCA_ERR_INVALID_ARG, "fused apply not available");
}
}  // namespace tca
