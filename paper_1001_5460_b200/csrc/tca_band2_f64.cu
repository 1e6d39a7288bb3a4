// Instantiation unit of the warp-specialised fused banded apply (tca_band2.cuh), T = double.
#include "tca_band2.cuh"

namespace tca {
namespace band2 {
template tca_status launch_dispatch<band::Params<double>>(const tca_operator *, const band::Params<double> &, cudaStream_t,
                                                        const CUtensorMap *, const CUtensorMap *);
template tca_status launch_dispatch<band::ParamsG<double>>(const tca_operator *, const band::ParamsG<double> &, cudaStream_t,
                                                         const CUtensorMap *, const CUtensorMap *);
template tca_status launch_dispatch<band::ParamsH<double>>(const tca_operator *, const band::ParamsH<double> &, cudaStream_t,
                                                         const CUtensorMap *, const CUtensorMap *);
template int pp_for<double>(int);
}  // namespace band2
}  // namespace tca
