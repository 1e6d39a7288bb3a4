// Instantiation unit of the fused banded apply, T = double (split per dtype so
// nvcc compiles the instantiations in parallel).
#include "tca_band_impl.cuh"

namespace tca {
namespace band {
template tca_status launch_dispatch<Params<double>>(const tca_operator *, const Params<double> &, cudaStream_t, const CUtensorMap *,
                                         const CUtensorMap *);
template int t3_for<double>(int);
template int boxw_for<double>(int);
template int pp_for<double>(int);
template int onebox_for<double>(int);
template int minb_for<double>(int);
template int unit_for<double>(int);
template int pitched_for<double>(int);
template int padded_s3_for<double>(int);
}  // namespace band
}  // namespace tca
