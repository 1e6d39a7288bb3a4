// Instantiation unit of the fused CG step B1' (band apply that also forms
// P_new = D + beta P_old and updates C), T = double.
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch_fu<Params<double>>(const tca_operator *, const Params<double> &, cudaStream_t,
                                                    const CUtensorMap *, const CUtensorMap *, const CUtensorMap *,
                                                    const FuArgs<double> &);
template int fu_ok_for<double>(int);
}  // namespace band
}  // namespace tca
