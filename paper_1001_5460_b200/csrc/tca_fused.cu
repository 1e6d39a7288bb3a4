// tca_fused.cu -- host glue of the fused banded apply: support check, TMA
// tensor-map creation (cached per input pointer) and dispatch to the
// instantiation units tca_fused_{f64,f32}_{tma,cp}.cu.
#include <cudaTypedefs.h>
#include <string.h>

#include <mutex>

#include "tca_fused_impl.cuh"

namespace tca {
namespace fused {
extern template tca_status launch_dispatch<double, true>(const tca_operator *, const double *, double *,
                                                          const int32_t *, cudaStream_t, const CUtensorMap *);
extern template tca_status launch_dispatch<double, false>(const tca_operator *, const double *, double *,
                                                           const int32_t *, cudaStream_t, const CUtensorMap *);
extern template tca_status launch_dispatch<float, true>(const tca_operator *, const float *, float *,
                                                         const int32_t *, cudaStream_t, const CUtensorMap *);
extern template tca_status launch_dispatch<float, false>(const tca_operator *, const float *, float *,
                                                          const int32_t *, cudaStream_t, const CUtensorMap *);
}  // namespace fused

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

// TMA can describe the slab boxes when the row strides are 16-byte multiples
// and the base pointer is 16-byte aligned.
bool tma_shape_ok(const tca_operator *op, const void *x)
{
    const uint64_t row = (uint64_t)op->n[2] * op->n[3] * op->esize;
    if (row % 16 != 0) return false;
    if (((uintptr_t)x) % 16 != 0) return false;
    if (op->nloc1 <= 0 || op->nloc1 > (1ll << 31) || op->n[1] > (1ll << 31)) return false;
    return get_encode() != nullptr;
}

tca_status make_tmap(const tca_operator *op, const void *x, CUtensorMap *m)
{
    auto encode = get_encode();
    if (!encode) return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int n4 = (int)op->n[3];
    const int boxw = op->dtype == TCA_F64 ? fused::boxw_for<double>(n4) : fused::boxw_for<float>(n4);
    cuuint64_t dims[3] = {(cuuint64_t)(op->n[2] * op->n[3]), (cuuint64_t)op->n[1], (cuuint64_t)op->nloc1};
    cuuint64_t strides[2] = {(cuuint64_t)(op->n[2] * op->n[3] * op->esize),
                             (cuuint64_t)(op->n[1] * op->n[2] * op->n[3] * op->esize)};
    cuuint32_t box[3] = {(cuuint32_t)boxw, 1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(m, op->dtype == TCA_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, const_cast<void *>(x), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return TCA_OK;
}

// Small per-operator cache of tensor maps keyed by the input pointer.
const CUtensorMap *cached_tmap(const tca_operator *op_c, const void *x, tca_status *st)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    for (auto &e : op->tmaps)
        if (e.ptr == x) return reinterpret_cast<const CUtensorMap *>(e.map);
    TmapSlot slot;
    slot.ptr = x;
    *st = make_tmap(op, x, reinterpret_cast<CUtensorMap *>(slot.map));
    if (*st != TCA_OK) return nullptr;
    if (op->tmaps.size() >= 8) op->tmaps.erase(op->tmaps.begin());
    op->tmaps.push_back(slot);
    return reinterpret_cast<const CUtensorMap *>(op->tmaps.back().map);
}

}  // namespace

bool fused_apply_supported(const tca_operator *op)
{
    if (!op->all_banded) return false;
    const int n4 = (int)op->n[3];
    const size_t smem = op->dtype == TCA_F64 ? fused::smem_for<double>(n4) : fused::smem_for<float>(n4);
    return smem > 0 && smem <= 227 * 1024;
}

tca_status launch_fused_apply(const tca_operator *op, const void *x, void *y, const int32_t *done,
                              cudaStream_t s)
{
    const bool tma = tma_shape_ok(op, x);
    const CUtensorMap *map = nullptr;
    if (tma) {
        tca_status st = TCA_OK;
        map = cached_tmap(op, x, &st);
        if (!map) return st;
    }
    if (op->dtype == TCA_F64) {
        if (tma) return fused::launch_dispatch<double, true>(op, (const double *)x, (double *)y, done, s, map);
        return fused::launch_dispatch<double, false>(op, (const double *)x, (double *)y, done, s, nullptr);
    }
    if (tma) return fused::launch_dispatch<float, true>(op, (const float *)x, (float *)y, done, s, map);
    return fused::launch_dispatch<float, false>(op, (const float *)x, (float *)y, done, s, nullptr);
}

}  // namespace tca
