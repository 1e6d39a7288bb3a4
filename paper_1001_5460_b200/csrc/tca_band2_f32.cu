// Instantiation unit of the warp-specialised fused banded apply (tca_band2.cuh), T = float.
#include "tca_band2.cuh"

namespace tca {
namespace band2 {
template tca_status launch_dispatch<band::Params<float>>(const tca_operator *, const band::Params<float> &, cudaStream_t,
                                                        const CUtensorMap *, const CUtensorMap *);
template tca_status launch_dispatch<band::ParamsG<float>>(const tca_operator *, const band::ParamsG<float> &, cudaStream_t,
                                                         const CUtensorMap *, const CUtensorMap *);
template tca_status launch_dispatch<band::ParamsH<float>>(const tca_operator *, const band::ParamsH<float> &, cudaStream_t,
                                                         const CUtensorMap *, const CUtensorMap *);
template int pp_for<float>(int);
}  // namespace band2
}  // namespace tca
