// Instantiation unit of the fused CG step B1' (band apply that also forms
// P_new = D + beta P_old and updates C), T = float.
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch_fu<Params<float>>(const tca_operator *, const Params<float> &, cudaStream_t,
                                                    const CUtensorMap *, const CUtensorMap *, const CUtensorMap *,
                                                    const FuArgs<float> &);
template int fu_ok_for<float>(int);
}  // namespace band
}  // namespace tca
