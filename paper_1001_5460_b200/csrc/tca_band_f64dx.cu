// Instantiation unit of the band apply with the deferred C update (MODE 2: a
// streaming warp applies C := C + alpha P_prev beside the operator), T = double.
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch_dx<Params<double>>(const tca_operator *, const Params<double> &, cudaStream_t,
                                                    const CUtensorMap *, const CUtensorMap *, const FuArgs<double> &);
}  // namespace band
}  // namespace tca
