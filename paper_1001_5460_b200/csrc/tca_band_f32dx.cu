// Instantiation unit of the band apply with the deferred C update (MODE 2: a
// streaming warp applies C := C + alpha P_prev beside the operator), T = float.
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch_dx<Params<float>>(const tca_operator *, const Params<float> &, cudaStream_t,
                                                    const CUtensorMap *, const CUtensorMap *, const FuArgs<float> &);
}  // namespace band
}  // namespace tca
