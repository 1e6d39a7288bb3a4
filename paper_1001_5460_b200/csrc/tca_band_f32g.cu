// Instantiation unit of the fused banded apply, T = float, tap tables in global
// memory (ParamsG: tables larger than the kernel-parameter block).
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch<ParamsG<float>>(const tca_operator *, const ParamsG<float> &, cudaStream_t,
                                                  const CUtensorMap *, const CUtensorMap *);
}  // namespace band
}  // namespace tca
