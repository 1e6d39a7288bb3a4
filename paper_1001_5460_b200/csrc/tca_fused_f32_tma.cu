// Instantiation unit of the fused banded apply: T = float, TMA staging = true.
// (Split per unit so nvcc compiles the instantiations in parallel.)
#include "tca_fused_impl.cuh"

namespace tca {
namespace fused {
template tca_status launch_dispatch<float, true>(const tca_operator *, const float *, float *, const int32_t *,
                                             cudaStream_t, const CUtensorMap *);
}  // namespace fused
}  // namespace tca
