// tca_band.cu -- host glue of the fused banded apply (tca_band_impl.cuh):
// support check, kernel-parameter tap tables, TMA tensor maps (cached per
// pointer) and dispatch to the per-dtype instantiation units
// tca_band_f64.cu / tca_band_f32.cu.
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "tca_band_impl.cuh"
#include "tca_band2.cuh"
#include "tca_fused.cuh"

namespace tca {
namespace band {
extern template tca_status launch_dispatch<Params<double>>(const tca_operator *, const Params<double> &, cudaStream_t,
                                                   const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<Params<float>>(const tca_operator *, const Params<float> &, cudaStream_t,
                                                  const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<ParamsG<double>>(const tca_operator *, const ParamsG<double> &, cudaStream_t,
                                                            const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<ParamsG<float>>(const tca_operator *, const ParamsG<float> &, cudaStream_t,
                                                           const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<ParamsH<double>>(const tca_operator *, const ParamsH<double> &, cudaStream_t,
                                                            const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<ParamsH<float>>(const tca_operator *, const ParamsH<float> &, cudaStream_t,
                                                           const CUtensorMap *, const CUtensorMap *);
extern template int t3_for<double>(int);
extern template int t3_for<float>(int);
extern template int boxw_for<double>(int);
extern template int boxw_for<float>(int);
extern template int pp_for<double>(int);
extern template int pp_for<float>(int);
extern template int onebox_for<double>(int);
extern template int onebox_for<float>(int);
extern template int minb_for<double>(int);
extern template int unit_for<double>(int);
extern template int unit_for<float>(int);
extern template int pitched_for<double>(int);
extern template int pitched_for<float>(int);
extern template int minb_for<float>(int);
extern template int padded_s3_for<double>(int);
extern template int padded_s3_for<float>(int);
extern template tca_status launch_dispatch_fu<Params<double>>(const tca_operator *, const Params<double> &,
                                                              cudaStream_t, const CUtensorMap *, const CUtensorMap *,
                                                              const CUtensorMap *, const FuArgs<double> &);
extern template tca_status launch_dispatch_fu<Params<float>>(const tca_operator *, const Params<float> &,
                                                             cudaStream_t, const CUtensorMap *, const CUtensorMap *,
                                                             const CUtensorMap *, const FuArgs<float> &);
extern template tca_status launch_dispatch_dx<Params<double>>(const tca_operator *, const Params<double> &,
                                                              cudaStream_t, const CUtensorMap *, const CUtensorMap *,
                                                              const FuArgs<double> &);
extern template tca_status launch_dispatch_dx<Params<float>>(const tca_operator *, const Params<float> &,
                                                             cudaStream_t, const CUtensorMap *, const CUtensorMap *,
                                                             const FuArgs<float> &);
extern template int fu_ok_for<double>(int);
extern template int fu_ok_for<float>(int);
}  // namespace band
namespace band2 {
extern template tca_status launch_dispatch<band::Params<double>>(const tca_operator *, const band::Params<double> &,
                                                                 cudaStream_t, const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<band::Params<float>>(const tca_operator *, const band::Params<float> &,
                                                                cudaStream_t, const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<band::ParamsG<double>>(const tca_operator *, const band::ParamsG<double> &,
                                                                  cudaStream_t, const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<band::ParamsG<float>>(const tca_operator *, const band::ParamsG<float> &,
                                                                 cudaStream_t, const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<band::ParamsH<double>>(const tca_operator *, const band::ParamsH<double> &,
                                                                  cudaStream_t, const CUtensorMap *, const CUtensorMap *);
extern template tca_status launch_dispatch<band::ParamsH<float>>(const tca_operator *, const band::ParamsH<float> &,
                                                                 cudaStream_t, const CUtensorMap *, const CUtensorMap *);
extern template int pp_for<double>(int);
extern template int pp_for<float>(int);
}  // namespace band2

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

// tile extents of the kernel the operator uses (v2: tca_band2.cuh)
int t2_of(const tca_operator *op) { return op->band_v2 ? band2::T2 : band::T2; }

int t3_of(const tca_operator *op)
{
    if (op->band_v2) return band2::T3;
    return op->dtype == TCA_F64 ? band::t3_for<double>((int)op->n[3]) : band::t3_for<float>((int)op->n[3]);
}

// One TMA box per staged slab (Cfg::ONEBOX): the input is viewed as
// (UNIT, n3 n4 / UNIT, n2, slabs) with 128-B inner chunks, which needs n3 n4 to
// be a multiple of UNIT; otherwise each staged row is NB boxes of a 3-D view.
bool onebox_of(const tca_operator *op)
{
    const int n4 = (int)op->n[3];
    const int unit = op->dtype == TCA_F64 ? band::unit_for<double>(n4) : band::unit_for<float>(n4);
    const int ob = op->dtype == TCA_F64 ? band::onebox_for<double>(n4) : band::onebox_for<float>(n4);
    const int pp = op->dtype == TCA_F64 ? band::pp_for<double>(n4) : band::pp_for<float>(n4);
    return ob && (op->n[2] * op->n[3]) % unit == 0 && pp / unit <= 256;
}

// Rows of the four tap tables (mode 4 first so its offsets are compile-time).
struct TableLayout {
    int rows[kD];
    int off[kD];
    int total;
};

TableLayout table_layout(const tca_operator *op)
{
    TableLayout L{};
    const int t3 = t3_of(op);
    const int extra[kD] = {0, t2_of(op), t3, 0};
    const int order[kD] = {3, 2, 1, 0};
    int off = 0;
    for (int i = 0; i < kD; ++i) {
        const int d = order[i];
        L.rows[d] = (int)(d == 0 ? op->nloc1 : op->n[d]) + extra[d] + 2 * band::PADR + 1;
        L.off[d] = off;
        off += L.rows[d];
    }
    L.total = off;
    return L;
}

bool tables_fit(const tca_operator *op);

// Kernel parameters: schedule and table offsets, plus the tap records either in
// the parameter block (Params, when they fit in TAP_BYTES) or in a device
// buffer (ParamsG, n_d ~ 256: config 4).
template <typename T>
tca_status build_params(const tca_operator *op_c, std::vector<unsigned char> &blob, int &grid, bool fu)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    const bool in_block = tables_fit(op);
    if (fu && !in_block) return TCA_OK;   // B1' takes parameter-block tables only (caller checks the blob)
    const TableLayout L = table_layout(op);
    // records kept in the block: all (Params); else modes 4 and 3 (ParamsH) or mode 4 (ParamsG),
    // the whole table also in global memory (table order: mode 4, 3, 2, 1)
    const size_t cap = band::TAP_BYTES / sizeof(T);
    size_t block_rows = (size_t)L.total;
    if (!in_block) {
        if ((size_t)L.off[1] * band::REC <= cap) { op->band_gt = 2; block_rows = (size_t)L.off[1]; }
        else if ((size_t)L.off[2] * band::REC <= cap) { op->band_gt = 1; block_rows = (size_t)L.off[2]; }
        else return fail(TCA_ERR_SHAPE, "band apply: the mode-4 tap table does not fit the parameter block");
    } else if (!fu) {
        op->band_gt = 0;
    }
    blob.assign(op->band_gt == 0 || fu ? sizeof(band::Params<T>) : sizeof(band::ParamsH<T>), 0);
    static_assert(sizeof(band::ParamsG<float>) == sizeof(band::ParamsH<float>), "one blob size");
    auto *p = reinterpret_cast<band::ParamsBase<T> *>(blob.data());
    const int t3 = t3_of(op);
    p->n1 = (int)op->nloc1;
    p->onebox = onebox_of(op) ? 1 : 0;
    p->n2 = (int)op->n[1];
    p->n3 = (int)op->n[2];
    p->tiles3 = (p->n3 + t3 - 1) / t3;
    const int t2 = t2_of(op);
    const long long tiles2 = (p->n2 + t2 - 1) / t2;
    const long long total = tiles2 * p->tiles3 * p->n1;
    // persistent grid over the (tile-major, slab-minor) unit order.  A CTA's
    // cost is its units plus 6 ramp slabs per tile it touches (mode-1 halo of
    // the ring).  Two schedules, the cheaper (max over CTAs) wins:
    //   split: CTA b owns units [total*b/G, total*(b+1)/G) (balanced units;
    //          ranges cross tile boundaries) -- long mode 1 (one GPU);
    //   whole: CTA b owns tile b entirely (tiles <= G) -- short mode 1 (a
    //          mode-1 shard of 16 rows: 22 slab passes instead of up to 26).
    const int minb = op->band_v2 ? 1
                                 : op->dtype == TCA_F64 ? band::minb_for<double>((int)op->n[3])
                                                        : band::minb_for<float>((int)op->n[3]);
    const int G = (int)std::min<long long>(std::min(op->num_sms * minb, band::MAXG), total);
    const long long tiles = tiles2 * p->tiles3;
    long long split_cost = 0;
    for (int b = 0; b < G; ++b) {
        const long long u0 = total * b / G, u1 = total * (b + 1) / G;
        const long long segs = u1 > u0 ? (u1 - 1) / p->n1 - u0 / p->n1 + 1 : 0;
        split_cost = std::max(split_cost, (u1 - u0) + 2 * band::KH1 * segs);
    }
    const long long whole_cost =
        tiles <= std::min<long long>(band::MAXG, (long long)op->num_sms * minb) ? p->n1 + 2 * band::KH1 : (1ll << 60);
    //   lock: tiles < G.  CTA t < tiles owns output slabs [0, L) of tile t; the
    //         G - tiles tail CTAs own slabs [L, n1) of consecutive tiles.  The
    //         main CTAs advance through mode 1 together, so the halo rows one
    //         tile stages were staged by its neighbours moments earlier and hit
    //         L2 (DRAM reads of the split schedule: 3.5x the algorithmic bytes,
    //         profiles/r01_sched_probe.txt); L balances the two kinds of CTA.
    long long lock_cost = 1ll << 60, lockL = 0, ktail = 0;
    if (tiles < G && p->n1 >= 4 * 2 * band::KH1) {
        const long long nt = G - tiles;
        ktail = (tiles + nt - 1) / nt;
        for (long long Lc = 2 * band::KH1; Lc < p->n1; ++Lc) {
            const long long c = std::max(Lc + 2 * band::KH1, ktail * (p->n1 - Lc + 2 * band::KH1));
            if (c < lock_cost) { lock_cost = c; lockL = Lc; }
        }
    }
    // measurement switch: TCA_BAND_SCHED=whole|split|lock forces a schedule
    // B1' prefers the mode-1-synchronous schedules (whole, lock): its halo
    // re-reads of D and P_old then hit L2
    static const char *force = getenv("TCA_BAND_SCHED");
    char pick = whole_cost <= split_cost ? 'w' : 's';
    // (the plain apply is bound inside the SM, not by DRAM: on config 3 lock
    // cuts DRAM reads 893 -> 317 MB per launch but runs 286 vs 278 us, so it is
    // picked only when strictly cheaper)
    if (lock_cost < (pick == 'w' ? whole_cost : split_cost)) pick = 'l';
    if (fu) pick = lock_cost <= whole_cost ? 'l' : 'w';
    if (force && (force[0] == 'w' || force[0] == 's' || force[0] == 'l')) pick = force[0];
    if (pick == 'w' && tiles > band::MAXG) pick = 's';
    if (pick == 'l' && lockL == 0) pick = tiles <= band::MAXG ? 'w' : 's';
    p->o_next = 0;
    if (pick == 'w') {
        for (long long t = 0; t < tiles; ++t) {
            p->s_tile[t].x = (short)(t / p->tiles3);
            p->s_tile[t].y = (short)(t % p->tiles3);
            p->s_o0[t] = 0;
            p->s_cnt[t] = p->n1;
        }
        grid = (int)tiles;
    } else if (pick == 'l') {
        const long long nt = G - tiles;
        for (long long t = 0; t < tiles; ++t) {
            p->s_tile[t].x = (short)(t / p->tiles3);
            p->s_tile[t].y = (short)(t % p->tiles3);
            p->s_o0[t] = 0;
            p->s_cnt[t] = (int)lockL;
        }
        int g = (int)tiles;
        for (long long i = 0; i < nt; ++i) {
            const long long t0 = tiles * i / nt, t1 = tiles * (i + 1) / nt;
            if (t1 <= t0) continue;
            p->s_tile[g].x = (short)(t0 / p->tiles3);
            p->s_tile[g].y = (short)(t0 % p->tiles3);
            p->s_o0[g] = (int)lockL;
            p->s_cnt[g] = (int)((t1 - t0) * (p->n1 - lockL));
            ++g;
        }
        p->o_next = (int)lockL;
        grid = g;
    } else {
        for (int b = 0; b < G; ++b) {
            const long long u0 = total * b / G, u1 = total * (b + 1) / G;
            const long long tile = u0 / p->n1;
            p->s_tile[b].x = (short)(tile / p->tiles3);
            p->s_tile[b].y = (short)(tile % p->tiles3);
            p->s_o0[b] = (int)(u0 % p->n1);
            p->s_cnt[b] = (int)(u1 - u0);
        }
        grid = G;
    }
    op->band_sched = pick;
    p->xoff = op->ghost;
    p->nin = (int)op->nloc1 + 2 * op->ghost;
    p->off1 = L.off[0];
    p->off2 = L.off[1];
    p->off3 = L.off[2];
    std::vector<T> taps((size_t)L.total * band::REC, T(0));
    for (int d = 0; d < kD; ++d) {
        const int nd = (int)(d == 0 ? op->nloc1 : op->n[d]);
        const int row0 = d == 0 ? (int)op->own_lo : 0;   // global row of local row 0 (mode 1 of a shard)
        // mode 1 of a shard also needs the rows of its ghost slabs (neighbours' rows)
        const int rlo = d == 0 ? -band::PADR : 0, rhi = d == 0 ? nd + band::PADR : nd;
        for (int r = rlo; r < rhi; ++r) {
            const int64_t g = row0 + r;
            if (g < 0 || g >= op->n[d]) continue;   // outside the domain: zero rows
            T *rec = taps.data() + (size_t)(L.off[d] + r + band::PADR) * band::REC;
            for (int k = 0; k < 4; ++k) rec[k] = (T)op->bandG[d][(size_t)g * 4 + k];
            for (int k = 0; k < 3; ++k) rec[4 + k] = (T)op->bandR[d][(size_t)g * 3 + k];
        }
    }
    if (in_block) {
        std::memcpy(reinterpret_cast<band::Params<T> *>(blob.data())->taps, taps.data(), taps.size() * sizeof(T));
    } else if (!fu) {   // global tables (uploaded once; freed with the operator) + the block's prefix
        const size_t nb = taps.size() * sizeof(T);
        TCA_CUDA_TRY(dev_get(&op->band_gtaps, nb));
        op->band_gtaps_bytes = nb;
        TCA_CUDA_TRY(cudaMemcpy(op->band_gtaps, taps.data(), nb, cudaMemcpyHostToDevice));
        auto *g = reinterpret_cast<band::ParamsH<T> *>(blob.data());   // same layout as ParamsG
        g->gtaps = (const T *)op->band_gtaps;
        std::memcpy(g->taps, taps.data(), block_rows * band::REC * sizeof(T));
    }
    return TCA_OK;
}

bool tables_fit(const tca_operator *op)
{
    const size_t es = op->esize;
    return (size_t)table_layout(op).total * band::REC * es <= (size_t)band::TAP_BYTES;
}

tca_status make_tmap(const tca_operator *op, const void *ptr, int kind, CUtensorMap *m)
{
    auto encode = get_encode();
    if (!encode) return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int n4 = (int)op->n[3];
    const int t3 = t3_of(op);
    // loads read a ghosted input (nloc1 + 2 ghost slabs), stores write the local output
    const int64_t slabs = kind == 0 ? op->nloc1 + 2 * op->ghost : op->nloc1;
    cuuint64_t dims[3] = {(cuuint64_t)(op->n[2] * op->n[3]), (cuuint64_t)op->n[1], (cuuint64_t)slabs};
    cuuint64_t strides[2] = {(cuuint64_t)(op->n[2] * op->n[3] * op->esize),
                             (cuuint64_t)(op->n[1] * op->n[2] * op->n[3] * op->esize)};
    cuuint32_t box[3];
    if (kind == 0) {
        const int boxw = op->dtype == TCA_F64 ? band::boxw_for<double>(n4) : band::boxw_for<float>(n4);
        box[0] = (cuuint32_t)boxw;
        box[1] = 1;
        box[2] = 1;
    } else {
        box[0] = (cuuint32_t)(t3 * n4);
        box[1] = band::T2;
        box[2] = 1;
    }
    cuuint32_t es[4] = {1, 1, 1, 1};
    const int s3 = op->band_v2 ? 0 : (op->dtype == TCA_F64 ? band::padded_s3_for<double>(n4) : band::padded_s3_for<float>(n4));
    if (s3) {   // padded staging (Cfg::PADDED): 4-D (n4, n3, n2, slabs) with a fibre box of s3 > n4 (zero fill)
        const auto dt = op->dtype == TCA_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        cuuint64_t d4[4] = {(cuuint64_t)n4, (cuuint64_t)op->n[2], (cuuint64_t)op->n[1], (cuuint64_t)slabs};
        cuuint64_t s4[3] = {(cuuint64_t)n4 * op->esize, (cuuint64_t)(op->n[2] * n4) * op->esize,
                            (cuuint64_t)(op->n[1] * op->n[2] * n4) * op->esize};
        cuuint32_t b4[4] = {(cuuint32_t)s3, (cuuint32_t)(kind == 0 ? t3 + 6 : t3),
                            (cuuint32_t)(kind == 0 ? band::PR : band::T2), 1};
        CUresult r = encode(m, dt, 4, const_cast<void *>(ptr), d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled (padded) failed (" + std::to_string((int)r) + ")");
        return TCA_OK;
    }
    if (op->band_v2) {   // tca_band2.cuh: slab box (UNIT, PP/UNIT, PR, 1) of a 4-D view; store box (T3 n4, T2, 1)
        const auto dt = op->dtype == TCA_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        CUresult r;
        if (kind == 0) {
            const cuuint64_t unit = band2::UNIT, F = (cuuint64_t)(op->n[2] * op->n[3]);
            const int pp = op->dtype == TCA_F64 ? band2::pp_for<double>(n4) : band2::pp_for<float>(n4);
            cuuint64_t d4[4] = {unit, F / unit, (cuuint64_t)op->n[1], (cuuint64_t)slabs};
            cuuint64_t s4[3] = {unit * op->esize, F * op->esize, F * (cuuint64_t)op->n[1] * op->esize};
            cuuint32_t b4[4] = {(cuuint32_t)unit, (cuuint32_t)(pp / unit), (cuuint32_t)band2::PR, 1};
            r = encode(m, dt, 4, const_cast<void *>(ptr), d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            box[0] = (cuuint32_t)(band2::T3 * n4);
            box[1] = band2::T2;
            box[2] = 1;
            r = encode(m, dt, 3, const_cast<void *>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS)
            return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled (v2) failed (" + std::to_string((int)r) + ")");
        return TCA_OK;
    }
    const bool pitched = (op->dtype == TCA_F64 ? band::pitched_for<double>(n4) : band::pitched_for<float>(n4)) != 0;
    if (kind == 0 && (onebox_of(op) || pitched)) {   // whole staged slab (PR rows x PP elements) as one box
        // chunk: Cfg::UNIT elements, or 16 B for a pitched fp32 slab whose n3 n4 is not a multiple of UNIT
        const cuuint64_t unit = onebox_of(op) ? (cuuint64_t)(op->dtype == TCA_F64 ? band::unit_for<double>(n4)
                                                                                  : band::unit_for<float>(n4))
                                              : 16 / op->esize;
        const cuuint64_t F = (cuuint64_t)(op->n[2] * op->n[3]);
        const int pp = op->dtype == TCA_F64 ? band::pp_for<double>(n4) : band::pp_for<float>(n4);
        cuuint64_t d4[4] = {unit, F / unit, (cuuint64_t)op->n[1], (cuuint64_t)slabs};
        cuuint64_t s4[3] = {unit * op->esize, F * op->esize, F * (cuuint64_t)op->n[1] * op->esize};
        cuuint32_t b4[4] = {(cuuint32_t)unit, (cuuint32_t)(pp / unit), (cuuint32_t)band::PR, 1};
        CUresult r = encode(m, op->dtype == TCA_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                            4, const_cast<void *>(ptr), d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled (4-D) failed (" + std::to_string((int)r) + ")");
        return TCA_OK;
    }
    CUresult r = encode(m, op->dtype == TCA_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, const_cast<void *>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TCA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return TCA_OK;
}

// Per-operator cache of tensor maps keyed by (pointer, kind); the descriptors
// live in a device buffer of kTmapSlots slots (round-robin replacement).
const CUtensorMap *cached_tmap(const tca_operator *op_c, const void *ptr, int kind, cudaStream_t s, tca_status *st,
                               int *slot_out)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    for (auto &e : op->tmaps)
        if (e.ptr == ptr && e.kind == kind) {
            *slot_out = e.slot;
            return reinterpret_cast<const CUtensorMap *>(op->tmap_dev) + e.slot;
        }
    if (!op->tmap_dev) {
        cudaError_t e = dev_get(&op->tmap_dev, sizeof(TmapSlot::map) * kTmapSlots);
        if (e == cudaSuccess) {
            op->tmap_host = (uint64_t *)pinned_get(sizeof(TmapSlot::map) * kTmapSlots);
            if (!op->tmap_host) e = cudaErrorMemoryAllocation;
        }
        for (int i = 0; i < kTmapSlots && e == cudaSuccess; ++i)
            e = cudaEventCreateWithFlags(&op->tmap_ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) { *st = cuda_fail(e, "tensor-map buffer"); return nullptr; }
    }
    TmapSlot slot;
    slot.ptr = ptr;
    slot.kind = kind;
    *st = make_tmap(op, ptr, kind, reinterpret_cast<CUtensorMap *>(slot.map));
    if (*st != TCA_OK) return nullptr;
    if ((int)op->tmaps.size() < kTmapSlots) {
        slot.slot = (int)op->tmaps.size();
        op->tmaps.push_back(slot);
    } else {
        int tries = 0;   // round-robin over the slots not pinned by a captured graph
        while ((op->tmap_pinned >> op->tmap_next) & 1u) {
            op->tmap_next = (op->tmap_next + 1) % kTmapSlots;
            if (++tries > kTmapSlots) { *st = fail(TCA_ERR_INVALID_ARG, "tensor-map slots exhausted"); return nullptr; }
        }
        slot.slot = op->tmap_next;
        for (auto &e : op->tmaps)
            if (e.slot == slot.slot) e = slot;
        op->tmap_next = (op->tmap_next + 1) % kTmapSlots;
        // a recycled slot may still be read by an earlier launch: wait for it
        cudaError_t e = cudaEventSynchronize(op->tmap_ev[slot.slot]);
        if (e != cudaSuccess) { *st = cuda_fail(e, "tensor-map slot event"); return nullptr; }
    }
    // stream-ordered upload from a host copy that lives as long as the operator
    std::memcpy(op->tmap_host + (size_t)slot.slot * 16, slot.map, sizeof(CUtensorMap));
    cudaError_t e = cudaMemcpyAsync(reinterpret_cast<CUtensorMap *>(op->tmap_dev) + slot.slot,
                                    op->tmap_host + (size_t)slot.slot * 16, sizeof(CUtensorMap),
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { *st = cuda_fail(e, "tensor-map upload"); return nullptr; }
    *slot_out = slot.slot;
    return reinterpret_cast<const CUtensorMap *>(op->tmap_dev) + slot.slot;
}

template <typename T>
tca_status launch_t(const tca_operator *op, const void *x, void *y, const int32_t *done, double *pq_part,
                    cudaStream_t s)
{
    tca_status st = TCA_OK;
    int xs = 0, ys = 0;
    const CUtensorMap *xm = cached_tmap(op, x, 0, s, &st, &xs);
    if (!xm) return st;
    const CUtensorMap *ym = cached_tmap(op, y, 1, s, &st, &ys);
    if (!ym) return st;
    // the parameter block is prebuilt at create; patch the per-call pointers
    band::ParamsBase<T> *p = reinterpret_cast<band::ParamsBase<T> *>(const_cast<unsigned char *>(op->band_params.data()));
    p->x = (const T *)x;
    p->y = (T *)y;
    p->done = done;
    p->pq_part = pq_part;
    // CG's finaliser 1 in the last CTA: the one-pass kernel (MODE 0) with
    // 256-thread CTAs (n4 <= 16, tca_finalize.cuh's block size), single GPU
    op->band_fin_done = op->band_fin_req && pq_part && !op->band_v2 && !op->transport && op->n[3] <= 16;
    p->fin_sc = op->band_fin_done ? op->sc : nullptr;
    p->fin_hist = op->hist;
    {
        static const char *e = getenv("TCA_BAND_DEBUG");
        p->dbg = e ? atoi(e) : 0;
    }
    if (op->band_v2) {
        if (op->band_gt == 2) TCA_TRY(band2::launch_dispatch(op, *static_cast<band::ParamsH<T> *>(p), s, xm, ym));
        else if (op->band_gt == 1) TCA_TRY(band2::launch_dispatch(op, *static_cast<band::ParamsG<T> *>(p), s, xm, ym));
        else TCA_TRY(band2::launch_dispatch(op, *static_cast<band::Params<T> *>(p), s, xm, ym));
    } else if (op->band_gt == 2) {
        TCA_TRY(band::launch_dispatch(op, *static_cast<band::ParamsH<T> *>(p), s, xm, ym));
    } else if (op->band_gt == 1) {
        TCA_TRY(band::launch_dispatch(op, *static_cast<band::ParamsG<T> *>(p), s, xm, ym));
    } else {
        TCA_TRY(band::launch_dispatch(op, *static_cast<band::Params<T> *>(p), s, xm, ym));
    }
    // the slots are in use until this launch completes; a launch captured into a
    // CUDA graph keeps using them for the graph's lifetime: pin them instead
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TCA_CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    tca_operator *o = const_cast<tca_operator *>(op);
    if (cs != cudaStreamCaptureStatusNone) {
        o->tmap_pinned |= (1u << xs) | (1u << ys);
    } else {
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[xs], s));
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[ys], s));
    }
    return TCA_OK;
}

}  // namespace

bool fused_shape_supported(const tca_operator *op)
{
    if (!op->all_banded) return false;
    const int n4 = (int)op->n[3];
    if (t3_of(op) == 0) return false;
    (void)n4;
    if ((op->n[2] * op->n[3] * op->esize) % 16 != 0) return false;   // TMA global stride rule
    if (op->nloc1 <= 0 || op->nloc1 > (1ll << 30) || op->n[1] > (1ll << 30)) return false;
    return get_encode() != nullptr;   // (tables that do not fit the parameter block go to global memory)
}

// The warp-specialised kernel (tca_band2.cuh) takes 9 <= n4 <= 16 (instantiated:
// 15, 16) when the slab is one TMA box of 8-element chunks.  Opt-in
// (TCA_BAND_V2=1): measured slower than band_apply_kernel on config 3 (DESIGN.md
// 6.1, shared-memory traffic per unknown 31 vs 24 words).
static bool v2_eligible(const tca_operator *op)
{
    static const char *e = getenv("TCA_BAND_V2");
    if (!(e && e[0] == '1')) return false;
    const int n4 = (int)op->n[3];
    if ((n4 != 15 && n4 != 16) || op->dtype != TCA_F64) return false;
    return (op->n[2] * op->n[3]) % band2::UNIT == 0;
}

tca_status fused_prepare(tca_operator *op)
{
    op->band_v2 = v2_eligible(op) ? 1 : 0;
    if (op->dtype == TCA_F64) return build_params<double>(op, op->band_params, op->band_grid, false);
    return build_params<float>(op, op->band_params, op->band_grid, false);
}

bool fused_b1_supported(const tca_operator *op)
{
    if (op->band_v2) return false;   // B1' is an instantiation of the first kernel
    if (op->ghost != 0 || op->band_gt || op->band_params.empty()) return false;   // one GPU, block tables
    const int n4 = (int)op->n[3];
    const bool pitched = (op->dtype == TCA_F64 ? band::pitched_for<double>(n4) : band::pitched_for<float>(n4)) != 0;
    if (!pitched && !onebox_of(op)) return false;   // one TMA box per staged slab
    return (op->dtype == TCA_F64 ? band::fu_ok_for<double>(n4) : band::fu_ok_for<float>(n4)) != 0;
}

namespace {
template <typename T>
tca_status launch_b1_t(const tca_operator *op_c, const void *pold, void *pnew, const void *d, void *q, void *x,
                       double *pq_part, cudaStream_t s)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    if (op->band_params_fu.empty()) return fail(TCA_ERR_INVALID_ARG, "fused CG step: not prepared");
    tca_status st = TCA_OK;
    int ps = 0, ds = 0;
    const CUtensorMap *pm = cached_tmap(op, pold, 0, s, &st, &ps);
    if (!pm) return st;
    const CUtensorMap *dm = cached_tmap(op, d, 0, s, &st, &ds);
    if (!dm) return st;
    int qs = 0;
    const CUtensorMap *qm = cached_tmap(op, q, 1, s, &st, &qs);
    if (!qm) return st;
    auto *p = reinterpret_cast<band::Params<T> *>(op->band_params_fu.data());
    p->x = (const T *)pold;
    p->y = (T *)q;
    p->done = &op->sc->done;
    p->pq_part = pq_part;
    {
        static const char *e = getenv("TCA_BAND_DEBUG");   // measurement switches (results invalid)
        p->dbg = e ? atoi(e) : 0;
    }
    const band::FuArgs<T> fa{(T *)x, (T *)pnew, op->sc};
    TCA_TRY(band::launch_dispatch_fu(op, *p, s, pm, qm, dm, fa));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TCA_CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
        op->tmap_pinned |= (1u << ps) | (1u << ds) | (1u << qs);
    } else {
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[ps], s));
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[ds], s));
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[qs], s));
    }
    return TCA_OK;
}
}  // namespace

// Parameter block and tensor maps of B1' created before any graph capture: a
// map first made inside a capture would be uploaded only when the graph runs,
// not for eager launches after it.
tca_status fused_b1_prepare(const tca_operator *op_c, const void *const *ptrs, const int *kinds, int n,
                            cudaStream_t s)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    if (op->band_params_fu.empty()) {
        if (op->dtype == TCA_F64) TCA_TRY(build_params<double>(op, op->band_params_fu, op->band_grid_fu, true));
        else TCA_TRY(build_params<float>(op, op->band_params_fu, op->band_grid_fu, true));
        if (op->band_params_fu.empty()) return fail(TCA_ERR_INVALID_ARG, "fused CG step: tables not in block");
    }
    for (int i = 0; i < n; ++i) {
        tca_status st = TCA_OK;
        int slot = 0;
        if (!cached_tmap(op, ptrs[i], kinds[i], s, &st, &slot)) return st;
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[slot], s));
    }
    return TCA_OK;
}

tca_status launch_fused_b1(const tca_operator *op, const void *pold, void *pnew, const void *d, void *q, void *x,
                           double *pq_part, cudaStream_t s)
{
    if (op->dtype == TCA_F64) return launch_b1_t<double>(op, pold, pnew, d, q, x, pq_part, s);
    return launch_b1_t<float>(op, pold, pnew, d, q, x, pq_part, s);
}

// Apply with the deferred C update (MODE 2): q = A p and the
// per-CTA <p, q> partials (op->band_grid_dx entries), and C += alpha P_prev by
// a streaming warp when sc->xupd (sc->done: only that update).  One GPU,
// parameter-block tables; the mode-1-synchronous schedule of B1' (lock/whole).
bool fused_dx_supported(const tca_operator *op)
{
    if (op->band_v2) return false;
    if (op->ghost != 0 || op->band_gt || op->band_params.empty()) return false;
    return true;
}

tca_status fused_dx_prepare(const tca_operator *op_c, const void *const *ptrs, const int *kinds, int n, cudaStream_t s)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    if (op->band_params_dx.empty()) {
        if (op->dtype == TCA_F64) TCA_TRY(build_params<double>(op, op->band_params_dx, op->band_grid_dx, true));
        else TCA_TRY(build_params<float>(op, op->band_params_dx, op->band_grid_dx, true));
        if (op->band_params_dx.empty()) return fail(TCA_ERR_INVALID_ARG, "deferred-x apply: tables not in block");
    }
    for (int i = 0; i < n; ++i) {
        tca_status st = TCA_OK;
        int slot = 0;
        if (!cached_tmap(op, ptrs[i], kinds[i], s, &st, &slot)) return st;
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[slot], s));
    }
    return TCA_OK;
}

namespace {
template <typename T>
tca_status launch_dx_t(const tca_operator *op_c, const void *p, void *q, void *x, const void *pprev,
                       double *pq_part, cudaStream_t s)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    if (op->band_params_dx.empty()) return fail(TCA_ERR_INVALID_ARG, "deferred-x apply: not prepared");
    tca_status st = TCA_OK;
    int ps = 0, qs = 0;
    const CUtensorMap *pm = cached_tmap(op, p, 0, s, &st, &ps);
    if (!pm) return st;
    const CUtensorMap *qm = cached_tmap(op, q, 1, s, &st, &qs);
    if (!qm) return st;
    auto *prm = reinterpret_cast<band::Params<T> *>(op->band_params_dx.data());
    prm->x = (const T *)p;
    prm->y = (T *)q;
    prm->done = &op->sc->done;
    prm->pq_part = pq_part;
    {
        static const char *e = getenv("TCA_BAND_DEBUG");   // measurement switches (results invalid)
        prm->dbg = e ? atoi(e) : 0;
    }
    const band::FuArgs<T> fa{(T *)x, (T *)const_cast<void *>(pprev), op->sc};
    TCA_TRY(band::launch_dispatch_dx(op, *prm, s, pm, qm, fa));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TCA_CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
        op->tmap_pinned |= (1u << ps) | (1u << qs);
    } else {
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[ps], s));
        TCA_CUDA_TRY(cudaEventRecord(op->tmap_ev[qs], s));
    }
    return TCA_OK;
}
}  // namespace

tca_status launch_fused_dx(const tca_operator *op, const void *p, void *q, void *x, const void *pprev,
                           double *pq_part, cudaStream_t s)
{
    if (op->dtype == TCA_F64) return launch_dx_t<double>(op, p, q, x, pprev, pq_part, s);
    return launch_dx_t<float>(op, p, q, x, pprev, pq_part, s);
}

bool fused_pointers_ok(const void *x, const void *y)
{
    return ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0);
}

tca_status launch_fused_apply(const tca_operator *op, const void *x, void *y, const int32_t *done, double *pq_part,
                              cudaStream_t s)
{
    if (op->dtype == TCA_F64) return launch_t<double>(op, x, y, done, pq_part, s);
    return launch_t<float>(op, x, y, done, pq_part, s);
}

}  // namespace tca
