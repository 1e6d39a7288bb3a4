// Instantiation unit of the fused banded apply: T = double, TMA staging = false.
// (Split per unit so nvcc compiles the instantiations in parallel.)
#include "tca_fused_impl.cuh"

namespace tca {
namespace fused {
template tca_status launch_dispatch<double, false>(const tca_operator *, const double *, double *, const int32_t *,
                                             cudaStream_t, const CUtensorMap *);
}  // namespace fused
}  // namespace tca
