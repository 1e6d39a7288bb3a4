// Instantiation unit of the fused banded apply, T = float (split per dtype so
// nvcc compiles the instantiations in parallel).
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch<Params<float>>(const tca_operator *, const Params<float> &, cudaStream_t, const CUtensorMap *,
                                         const CUtensorMap *);
template int t3_for<float>(int);
template int boxw_for<float>(int);
template int pp_for<float>(int);
template int onebox_for<float>(int);
template int minb_for<float>(int);
template int unit_for<float>(int);
template int pitched_for<float>(int);
template int padded_s3_for<float>(int);
}  // namespace band
}  // namespace tca
