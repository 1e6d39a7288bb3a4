// Instantiation unit of the fused banded apply, T = double, tap tables in global
// memory with the mode-4 and mode-3 records also in the parameter block
// (ParamsH: tables larger than the block, config 4's shape class).
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch<ParamsH<double>>(const tca_operator *, const ParamsH<double> &, cudaStream_t,
                                                 const CUtensorMap *, const CUtensorMap *);
}  // namespace band
}  // namespace tca
