// tca_abi.cu -- host side of libtca: the extern "C" entry points of
// include/tca.h, operator setup (G_d = A_d^T A_d, R_d = L_d^T L_d, band
// detection, tap tables), and the orchestration of the device kernels.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "tca_fused.cuh"
#include "tca_internal.cuh"

namespace tca {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

tca_status fail(tca_status s, const std::string &msg)
{
    set_error(msg);
    return s;
}

tca_status cuda_fail(cudaError_t e, const char *what)
{
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TCA_ERR_OOM : TCA_ERR_CUDA;
}

static bool all_finite(const double *a, size_t k)
{
    for (size_t i = 0; i < k; ++i)
        if (!isfinite(a[i])) return false;
    return true;
}

// G = M^T M for an r x c row-major M (fp64, ascending k sums).  Only the
// nonzeros of each row of M contribute (B-spline rows have <= 4): O(r nnz^2)
// instead of O(r c^2); skipped products are exact zeros, so the sums are the
// same as the dense loop's.
// Small pinned host buffers (CG scalar mirror, tensor-map staging) come from a
// process-wide free list: cudaMallocHost costs milliseconds and varies, and an
// operator is created per solve.
static std::mutex g_pinned_mu;
static std::vector<std::pair<size_t, void *>> g_pinned_free;

void *pinned_get(size_t bytes)
{
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        for (size_t i = 0; i < g_pinned_free.size(); ++i)
            if (g_pinned_free[i].first == bytes) {
                void *p = g_pinned_free[i].second;
                g_pinned_free.erase(g_pinned_free.begin() + (long)i);
                return p;
            }
    }
    void *p = nullptr;
    return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}

void pinned_put(void *p, size_t bytes)
{
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.emplace_back(bytes, p);
}

// Small device buffers (tap tables, reduction partials, scalars, histories,
// tensor maps) are recycled through a process-wide size-keyed free list:
// cudaFree synchronises the device and, measured on B200, occasionally stalls
// for hundreds of milliseconds; an operator is created and destroyed per solve.
// (Tensor-sized workspaces use the stream-ordered pool instead.)
static std::mutex g_dev_mu;
static std::vector<std::pair<size_t, void *>> g_dev_free;

cudaError_t dev_get(void **p, size_t bytes)
{
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        for (size_t i = 0; i < g_dev_free.size(); ++i)
            if (g_dev_free[i].first == bytes) {
                *p = g_dev_free[i].second;
                g_dev_free.erase(g_dev_free.begin() + (long)i);
                return cudaSuccess;
            }
    }
    return cudaMalloc(p, bytes);
}

void dev_put(void *p, size_t bytes)
{
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    g_dev_free.emplace_back(bytes, p);
}

static std::vector<double> gram(const double *M, int64_t r, int64_t c)
{
    std::vector<double> G((size_t)(c * c), 0.0);
    std::vector<int64_t> nz;
    nz.reserve((size_t)c);
    for (int64_t k = 0; k < r; ++k) {
        nz.clear();
        for (int64_t a = 0; a < c; ++a)
            if (M[k * c + a] != 0.0) nz.push_back(a);
        for (size_t i = 0; i < nz.size(); ++i)
            for (size_t j = i; j < nz.size(); ++j)
                G[nz[i] * c + nz[j]] += M[k * c + nz[i]] * M[k * c + nz[j]];
    }
    for (int64_t a = 0; a < c; ++a)
        for (int64_t b = a + 1; b < c; ++b) G[b * c + a] = G[a * c + b];
    return G;
}

static int half_bandwidth(const std::vector<double> &G, int64_t n)
{
    int hb = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j)
            if (G[i * n + j] != 0.0) hb = std::max(hb, (int)std::llabs(i - j));
    return hb;
}

static bool cholesky_ok(const std::vector<double> &G, int64_t n)
{
    std::vector<double> L(G);
    for (int64_t j = 0; j < n; ++j) {
        double d = L[j * n + j];
        for (int64_t k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
        if (!(d > 0.0) || !isfinite(d)) return false;
        d = sqrt(d);
        L[j * n + j] = d;
        for (int64_t i = j + 1; i < n; ++i) {
            double s = L[i * n + j];
            for (int64_t k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
            L[i * n + j] = s / d;
        }
    }
    return true;
}

static std::mutex g_attr_mu;
static std::map<std::pair<const void *, int>, size_t> g_attr_set;

tca_status set_max_dynamic_smem(const void *func, size_t bytes)
{
    int dev = 0;
    TCA_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t &cur = g_attr_set[{func, dev}];
    if (bytes > cur) {
        TCA_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        cur = bytes;
    }
    return TCA_OK;
}

template <typename T>
static tca_status upload(const std::vector<double> &h, void **dptr, size_t *bytes)
{
    std::vector<T> c(h.size());
    for (size_t i = 0; i < h.size(); ++i) c[i] = (T)h[i];
    size_t nb = std::max<size_t>(c.size(), 1) * sizeof(T);
    TCA_CUDA_TRY(dev_get(dptr, nb));
    *bytes += nb;
    if (!c.empty()) TCA_CUDA_TRY(cudaMemcpy(*dptr, c.data(), c.size() * sizeof(T), cudaMemcpyHostToDevice));
    return TCA_OK;
}

static tca_status upload_dtype(tca_dtype dt, const std::vector<double> &h, void **dptr,
                               size_t *bytes)
{
    return dt == TCA_F64 ? upload<double>(h, dptr, bytes) : upload<float>(h, dptr, bytes);
}

// Build a compressed-band matrix from a dense rows x cols fp64 matrix.
// width_hint > 0 forces the centred offset form start[r] = r - width_hint/2.
static tca_status make_band(tca_dtype dt, const std::vector<double> &M, int rows, int cols,
                            int centred_half, BandMat *out, size_t *bytes)
{
    std::vector<int> start(rows);
    int W = 0;
    if (centred_half >= 0) {
        W = 2 * centred_half + 1;
        for (int r = 0; r < rows; ++r) start[r] = r - centred_half;
    } else {
        for (int r = 0; r < rows; ++r) {
            int lo = cols, hi = -1;
            for (int c = 0; c < cols; ++c)
                if (M[(size_t)r * cols + c] != 0.0) { lo = std::min(lo, c); hi = c; }
            if (hi < 0) { start[r] = 0; continue; }
            start[r] = lo;
            W = std::max(W, hi - lo + 1);
        }
        if (W == 0) W = 1;
    }
    std::vector<double> taps((size_t)rows * W, 0.0);
    for (int r = 0; r < rows; ++r)
        for (int w = 0; w < W; ++w) {
            int c = start[r] + w;
            if (c >= 0 && c < cols) taps[(size_t)r * W + w] = M[(size_t)r * cols + c];
        }
    out->rows = rows;
    out->cols = cols;
    out->W = W;
    out->dense = (W == cols);
    out->reach_lo = out->reach_hi = 0;
    for (int r = 0; r < rows; ++r) {
        out->reach_lo = std::max(out->reach_lo, -start[r]);
        out->reach_hi = std::max(out->reach_hi, start[r] + W - cols);
    }
    out->win16 = 0;
    for (int r0 = 0; r0 < rows; r0 += 16) {
        int lo = start[r0], hi = start[r0];
        for (int r = r0; r < std::min(rows, r0 + 16); ++r) {
            lo = std::min(lo, start[r]);
            hi = std::max(hi, start[r]);
        }
        out->win16 = std::max(out->win16, hi + W - lo);
    }
    for (int r = 0; r < rows && out->dense; ++r)
        if (start[r] != 0) out->dense = false;
    TCA_CUDA_TRY(dev_get((void **)&out->start, sizeof(int) * std::max(rows, 1)));
    *bytes += sizeof(int) * std::max(rows, 1);
    TCA_CUDA_TRY(cudaMemcpy(out->start, start.data(), sizeof(int) * rows, cudaMemcpyHostToDevice));
    out->tap_bytes = std::max<size_t>(taps.size(), 1) * (dt == TCA_F64 ? sizeof(double) : sizeof(float));
    return upload_dtype(dt, taps, &out->taps, bytes);
}

tca_status make_dense_mat(tca_dtype dt, const std::vector<double> &M, int n, BandMat *out, size_t *bytes)
{
    return make_band(dt, M, n, n, -1, out, bytes);
}

static void free_band(BandMat &b)
{
    dev_put(b.start, sizeof(int) * std::max(b.rows, 1));
    dev_put(b.taps, b.tap_bytes);
    b.start = nullptr;
    b.taps = nullptr;
}

static int64_t inner_of(const int64_t *ext, int d)
{
    int64_t p = 1;
    for (int e = d + 1; e < kD; ++e) p *= ext[e];
    return p;
}

static int64_t outer_of(const int64_t *ext, int d)
{
    int64_t p = 1;
    for (int e = 0; e < d; ++e) p *= ext[e];
    return p;
}

// One mode product: dense fp64 factors run on the FP64 tensor cores (DMMA),
// everything else on the compressed-band kernel.
template <typename T>
static void mode_product(const T *X, T *Y, int64_t outer, const BandMat &M, int64_t inner, double alpha,
                         bool accumulate, const int32_t *done, cudaStream_t s)
{
    if constexpr (sizeof(T) == 8) {
        if (M.dense && M.rows >= 8 && M.cols >= 8) {
            launch_dense_mode_product_dmma((const double *)X, (double *)Y, outer, M.rows, M.cols, inner,
                                           (const double *)M.taps, alpha, accumulate, done, s);
            return;
        }
    }
    launch_band_mode_product<T>(X, Y, outer, M, inner, alpha, accumulate, done, s);
}

template <typename T>
static tca_status apply_multipass_t(const tca_operator *op, const T *x, T *y,
                                    const int32_t *done, cudaStream_t s)
{
    int64_t ext[kD] = {op->nloc1, op->n[1], op->n[2], op->n[3]};
    // Kronecker term: mode products D..1 (Eq. 5 lets us pick any order).
    std::vector<int> active;
    for (int d = kD - 1; d >= 0; --d)
        if (d < op->order) active.push_back(d);
    const T *in = x;
    T *bufs[2] = {(T *)op->t0, (T *)op->t1};
    int nb = 0;
    for (size_t i = 0; i < active.size(); ++i) {
        const int d = active[i];
        T *out = (i + 1 == active.size()) ? y : bufs[nb];
        mode_product<T>(in, out, outer_of(ext, d), op->Gm[d], inner_of(ext, d), 1.0, false, done, s);
        in = out;
        nb ^= 1;
    }
    // Regulariser: y += lambda * (x x_d R_d) for each mode (Eq. 9 Kronecker sum).
    for (int d = 0; d < op->order; ++d)
        if (op->has_reg[d])
            launch_band_mode_product<T>(x, y, outer_of(ext, d), op->Rm[d], inner_of(ext, d),
                                        op->lambda, true, done, s);
    return TCA_OK;
}

tca_status apply_multipass(const tca_operator *op_c, const void *x, void *y,
                           const int32_t *done, cudaStream_t s)
{
    tca_operator *op = const_cast<tca_operator *>(op_c);
    if (!op->t0) {   // lazily: only operators whose apply cannot take the fused path use it
        const size_t vb = (size_t)op->N * op->esize;
        TCA_CUDA_TRY(cudaMallocAsync(&op->t0, vb, s));
        TCA_CUDA_TRY(cudaMallocAsync(&op->t1, vb, s));
        op->device_bytes += 2 * vb;
    }
    if (op->dtype == TCA_F64)
        return apply_multipass_t<double>(op, (const double *)x, (double *)y, done, s);
    return apply_multipass_t<float>(op, (const float *)x, (float *)y, done, s);
}

// pq_part != NULL asks the fused kernel for per-CTA partials of <x, y>; the
// caller must check fused_used() to know whether they were produced.
static bool fused_used(const tca_operator *op, const void *x, const void *y)
{
    return op->apply_path == 1 && fused_pointers_ok(x, y);
}

static tca_status apply_dispatch(const tca_operator *op, const void *x, void *y,
                                 const int32_t *done, cudaStream_t s, double *pq_part = nullptr)
{
    if (op->apply_path == 2) {   // Kronecker sum only (Eq. 9): one stencil pass
        if (op->dtype == TCA_F64)
            launch_ksum_apply<double>((const double *)x, (double *)y, op->N, op->n, (const double *)op->ks_taps,
                                      op->ks_off, done, s);
        else
            launch_ksum_apply<float>((const float *)x, (float *)y, op->N, op->n, (const float *)op->ks_taps,
                                     op->ks_off, done, s);
        TCA_CUDA_TRY(cudaGetLastError());
        if (op->scat) return launch_scatter(op, 0, x, y, nullptr, done, s);   // + sum_k w_k <w_k, x>
        return TCA_OK;
    }
    if (fused_used(op, x, y)) return launch_fused_apply(op, x, y, done, pq_part, s);
    return apply_multipass(op, x, y, done, s);
}

// Successive rectangular mode products in[...] -> out[...] (forward model or rhs).
template <typename T>
static tca_status chain_products(const tca_operator *op, const T *in, T *out,
                                 const int64_t *ext_in, const int64_t *ext_out,
                                 const BandMat *mats, const std::vector<int> &order,
                                 cudaStream_t s)
{
    int64_t ext[kD];
    for (int d = 0; d < kD; ++d) ext[d] = ext_in[d];
    // size of the largest intermediate
    size_t maxi = 0;
    {
        int64_t e2[kD];
        for (int d = 0; d < kD; ++d) e2[d] = ext_in[d];
        for (size_t i = 0; i + 1 < order.size(); ++i) {
            e2[order[i]] = ext_out[order[i]];
            size_t sz = 1;
            for (int d = 0; d < kD; ++d) sz *= (size_t)e2[d];
            maxi = std::max(maxi, sz);
        }
    }
    T *tmp[2] = {nullptr, nullptr};
    if (order.size() > 1) {
        TCA_CUDA_TRY(cudaMallocAsync((void **)&tmp[0], maxi * sizeof(T), s));
        if (order.size() > 2) TCA_CUDA_TRY(cudaMallocAsync((void **)&tmp[1], maxi * sizeof(T), s));
    }
    std::vector<int> rest = order;
    const T *cur = in;
    int tsel = 0;
    // opt-in (TCA_RHS_FUSE1=1): first pass = mode 1 together with the contiguous
    // last mode L when mode 1 comes first and L contracts (launch_band_win_last:
    // the pass writes the tensor with L already contracted).  Measured slower on
    // config 3 (1.89 ms for the fused pass + 0.59 ms for modes 2-3, vs 1.98 ms
    // for the default chain)
    static const bool fuse1 = getenv("TCA_RHS_FUSE1") && getenv("TCA_RHS_FUSE1")[0] == '1';
    if (fuse1 && rest.size() >= 2 && rest[0] == 0) {
        const int L = *std::max_element(rest.begin(), rest.end());
        bool ok = L > 0 && ext_out[L] <= ext_in[L] && !mats[0].dense && !mats[L].dense;
        for (int e = L + 1; e < kD && ok; ++e) ok = ext_in[e] == 1 && ext_out[e] == 1;
        if (ok) {
            int64_t K = 1;
            for (int e = 1; e < L; ++e) K *= ext[e];
            T *dst = rest.size() == 2 ? out : tmp[tsel];
            if (launch_band_win_last<T>(cur, dst, K, (int)ext[L], mats[0], mats[L], s)) {
                ext[0] = ext_out[0];
                ext[L] = ext_out[L];
                cur = dst;
                tsel ^= 1;
                rest.erase(std::remove(rest.begin(), rest.end(), L), rest.end());
                rest.erase(rest.begin());
            }
        }
    }
    // the last two products on the two fastest non-trivial modes (d, d+1): one
    // plane pass (launch_band_plane2) when the plane fits shared memory
    size_t nsep = rest.size();
    int pd = -1;
    if (rest.size() >= 2) {
        const int a = rest[rest.size() - 2], c = rest[rest.size() - 1];
        const int d = std::min(a, c);
        bool trailing_unit = std::max(a, c) == d + 1;
        for (int e = d + 2; e < kD && trailing_unit; ++e) trailing_unit = ext[e] == 1 && ext_out[e] == 1;
        if (trailing_unit && !mats[d].dense && !mats[d + 1].dense) {
            pd = d;
            nsep -= 2;
        }
    }
    for (size_t i = 0; i < rest.size(); ++i) {
        const int d = rest[i];
        T *dst = (i + 1 == rest.size()) ? out : tmp[tsel];
        if (i == nsep && pd >= 0) {
            int64_t planes = 1;
            for (int e = 0; e < pd; ++e) planes *= ext[e];
            if (launch_band_plane2<T>(cur, out, planes, (int)ext[pd], (int)ext[pd + 1], mats[pd], mats[pd + 1], s)) {
                cur = out;
                break;
            }
        }
        mode_product<T>(cur, dst, outer_of(ext, d), mats[d], inner_of(ext, d), 1.0, false, nullptr, s);
        ext[d] = ext_out[d];
        cur = dst;
        tsel ^= 1;
    }
    if (order.empty()) {
        size_t sz = 1;
        for (int d = 0; d < kD; ++d) sz *= (size_t)ext[d];
        TCA_CUDA_TRY(cudaMemcpyAsync(out, in, sz * sizeof(T), cudaMemcpyDeviceToDevice, s));
    }
    if (tmp[0]) TCA_CUDA_TRY(cudaFreeAsync(tmp[0], s));
    if (tmp[1]) TCA_CUDA_TRY(cudaFreeAsync(tmp[1], s));
    return TCA_OK;
}

template <typename T>
static tca_status rhs_t(const tca_operator *op, const T *ydata, T *b, cudaStream_t s)
{
    int64_t ein[kD] = {op->data_hi - op->data_lo, op->m[1], op->m[2], op->m[3]};
    int64_t eout[kD] = {op->nloc1, op->n[1], op->n[2], op->n[3]};
    std::vector<int> order;
    for (int d = 0; d < op->order; ++d) order.push_back(d);
    // contract the modes that shrink the tensor most first (PAPER.md:83 cost-driven
    // order); ties keep the slowest mode first (measured faster on config 3 than
    // contiguous-first with the generic kernel: 7.3 vs 13.0 ms)
    std::stable_sort(order.begin(), order.end(), [&](int a, int c) {
        return (double)ein[a] / eout[a] > (double)ein[c] / eout[c];
    });
    return chain_products<T>(op, ydata, b, ein, eout, op->At, order, s);
}

template <typename T>
static tca_status forward_t(const tca_operator *op, const T *x, T *y, double sigma,
                            uint64_t seed, cudaStream_t s)
{
    // shard-local: data rows [data_lo, data_hi) from unknown rows [xf_lo, xf_hi)
    int64_t ein[kD] = {op->xf_hi - op->xf_lo, op->n[1], op->n[2], op->n[3]};
    int64_t eout[kD] = {op->data_hi - op->data_lo, op->m[1], op->m[2], op->m[3]};
    const int64_t N = ein[0] * ein[1] * ein[2] * ein[3];
    const int64_t M = eout[0] * eout[1] * eout[2] * eout[3];
    T *xt = nullptr;
    if (!x) {   // x_true generated in place, position keyed (global unknown index)
        TCA_CUDA_TRY(cudaMallocAsync((void **)&xt, std::max<int64_t>(N, 1) * sizeof(T), s));
        launch_gen_normal<T>(xt, N, op->xf_lo * op->slab, stream_key(seed, 0), 1.0, false, s);
        x = xt;
    }
    std::vector<int> order;
    for (int d = 0; d < op->order; ++d) order.push_back(d);
    std::stable_sort(order.begin(), order.end(), [&](int a, int c) {
        return (double)eout[a] / ein[a] < (double)eout[c] / ein[c];
    });
    TCA_TRY(chain_products<T>(op, x, y, ein, eout, op->Af, order, s));
    const int64_t mslab = op->m[1] * op->m[2] * op->m[3];
    if (sigma != 0.0) launch_gen_normal<T>(y, M, op->data_lo * mslab, stream_key(seed, 1), sigma, true, s);
    if (xt) TCA_CUDA_TRY(cudaFreeAsync(xt, s));
    return TCA_OK;
}

// Timed apply: an event pair around the launch when instrumentation is on.
// Inside a CUDA-graph capture the pair is recorded as external event nodes of
// the graph (real timestamps at every replay), harvested per graph instance.
template <typename Fn>
static tca_status timed_call(tca_operator *op, cudaStream_t s, Fn &&fn)
{
    if (!op->timing) return fn();
    if (op->capturing && !op->cap_ev) return fn();   // not a sampled iteration of the chunk
    if (op->cap_ev) {
        cudaEvent_t a, b;
        TCA_CUDA_TRY(cudaEventCreate(&a));
        op->cap_ev->push_back(a);
        TCA_CUDA_TRY(cudaEventCreate(&b));
        op->cap_ev->push_back(b);
        TCA_CUDA_TRY(cudaEventRecordWithFlags(a, s, cudaEventRecordExternal));
        TCA_TRY(fn());
        TCA_CUDA_TRY(cudaEventRecordWithFlags(b, s, cudaEventRecordExternal));
        return TCA_OK;
    }
    if (op->tev_used + 2 > op->tev.size()) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            TCA_CUDA_TRY(cudaEventCreate(&e));
            op->tev.push_back(e);
        }
    }
    cudaEvent_t a = op->tev[op->tev_used], b = op->tev[op->tev_used + 1];
    op->tev_used += 2;
    TCA_CUDA_TRY(cudaEventRecord(a, s));
    TCA_TRY(fn());
    TCA_CUDA_TRY(cudaEventRecord(b, s));
    return TCA_OK;
}

static tca_status timed_apply(tca_operator *op, const void *x, void *y, const int32_t *done,
                              cudaStream_t s, double *pq_part = nullptr)
{
    return timed_call(op, s, [&] { return apply_dispatch(op, x, y, done, s, pq_part); });
}

// y = M x for a caller tensor x of the local shape: a sharded operator first
// copies x into its ghosted buffer and exchanges the halo (tca_apply's path)
static tca_status apply_any(tca_operator *o, const void *x, void *y, cudaStream_t s, bool timed)
{
    if (o->transport) {
        const size_t sb = (size_t)o->slab * o->esize;
        const size_t xb = (size_t)(o->nloc1 + 2 * o->ghost) * sb;
        if (!o->x_ext) {
            TCA_CUDA_TRY(cudaMallocAsync(&o->x_ext, xb, s));
            TCA_CUDA_TRY(cudaMemsetAsync(o->x_ext, 0, xb, s));
            o->device_bytes += xb;
        }
        TCA_CUDA_TRY(cudaMemcpyAsync((char *)o->x_ext + (size_t)o->ghost * sb, x, (size_t)o->nloc1 * sb,
                                     cudaMemcpyDeviceToDevice, s));
        TCA_TRY(o->transport->halo(1, (char *)o->x_ext, sb, o->nloc1, s));
        x = o->x_ext;
    }
    if (timed) return timed_apply(o, x, y, nullptr, s);
    return apply_dispatch(o, x, y, nullptr, s);
}

static tca_status harvest_pairs(tca_operator *op, const cudaEvent_t *ev, size_t n)
{
    for (size_t i = 0; i + 1 < n; i += 2) {
        float ms = 0.f;
        TCA_CUDA_TRY(cudaEventSynchronize(ev[i + 1]));
        TCA_CUDA_TRY(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        op->apply_ms += ms;
        op->apply_count += 1;
    }
    return TCA_OK;
}

// Event pairs of the last replay of graph instance g.
static tca_status harvest_graph(tca_operator *op, int g)
{
    if (!op->gpend[g]) return TCA_OK;
    op->gpend[g] = false;
    return harvest_pairs(op, op->gev[g].data(), op->gev[g].size());
}

// Fold the recorded event pairs into apply_ms / apply_count (after a sync).
static tca_status harvest_timing(tca_operator *op)
{
    for (int g = 0; g < 2; ++g) TCA_TRY(harvest_graph(op, g));
    TCA_TRY(harvest_pairs(op, op->tev.data(), op->tev_used));
    op->tev_used = 0;
    return TCA_OK;
}

// Host wait at the solvers' synchronisation points: on a sharded operator the
// transport's (NCCL: polls the asynchronous error state, aborts on an error or
// timeout and returns TCA_ERR_NCCL instead of hanging on a dead peer)
static tca_status sync_solve(tca_operator *op, cudaStream_t s)
{
    if (op->transport) return op->transport->wait(s);
    TCA_CUDA_TRY(cudaStreamSynchronize(s));
    return TCA_OK;
}

// Dot-product finalisation: single GPU one kernel; sharded: local sum, all-reduce
// of the fp64 scalar over the shards, then the scalar update.
static tca_status cg_reduce(tca_operator *op, int which, const double *part, int nparts, cudaStream_t s)
{
    if (!op->transport) {
        launch_cg_finalize(which, part, nparts, op->sc, op->hist, s, 0);
        return TCA_OK;
    }
    launch_cg_finalize(which, part, nparts, op->sc, op->hist, s, 1);
    TCA_TRY(op->transport->allreduce(&op->sc->red[which], 1, s));
    launch_cg_finalize(which, part, nparts, op->sc, op->hist, s, 2);
    return TCA_OK;
}

// R := R - alpha Q and its <r, r> partials, then finaliser 2 (rho1, stop
// test, beta): single GPU inside cg_update_r's last CTA (tca_finalize.cuh: one
// launch and one graph-node gap less per iteration; TCA_NO_FUSED_FIN=1
// measures the separate kernel), sharded through cg_reduce's all-reduce
template <typename T>
static tca_status update_r_reduce(tca_operator *op, T *r, const T *q, cudaStream_t s)
{
    static const bool no_fin = getenv("TCA_NO_FUSED_FIN") != nullptr;
    if (!op->transport && !no_fin) {
        launch_cg_update_r<T>(r, q, op->N, op->sc, op->part, s, true, op->hist);
        return TCA_OK;
    }
    launch_cg_update_r<T>(r, q, op->N, op->sc, op->part, s);
    return cg_reduce(op, 2, op->part, kRedBlocks, s);
}

static tca_status halo_p(tca_operator *op, cudaStream_t s)
{
    if (!op->transport) return TCA_OK;
    return op->transport->halo(0, (char *)op->p, (size_t)op->slab * op->esize, op->nloc1, s);
}

// z = P^-1 r (PCG): banded factors by the in-place sweep kernel, dense factors
// (F_d^-1 formed at setup) by the dense mode product on the FP64 tensor cores.
template <typename T>
static tca_status apply_precond(tca_operator *op, const T *r, T *z, const int32_t *done, cudaStream_t s)
{
    const T *cur = r;
    for (int d = 0; d < op->order; ++d) {
        int64_t outer = 1, inner = 1;
        for (int e = 0; e < d; ++e) outer *= op->n[e];
        for (int e = d + 1; e < kD; ++e) inner *= op->n[e];
        if (op->pc_banded[d]) {
            TCA_TRY(launch_precond_sweep<T>(op, d, cur, z, outer, inner, done, s));
            cur = z;
        } else {   // out of place: ping-pong between z and the preconditioner scratch
            T *dst = (cur == z) ? (T *)op->pc_tmp : z;
            mode_product<T>(cur, dst, outer, op->pc_inv[d], inner, 1.0, false, done, s);
            cur = dst;
        }
    }
    if (cur != z) TCA_CUDA_TRY(cudaMemcpyAsync(z, cur, (size_t)op->N * op->esize, cudaMemcpyDeviceToDevice, s));
    return TCA_OK;
}

// Single-reduction CG: W := A*R with R+*W from the apply, R+*R from the update
// kernel, both reduced together (one all-reduce of two scalars when sharded).
// The CGSR vectors: R in the ghosted buffer (op->p, the apply input), P in
// op->r, S in op->sr_s, W in op->q.
template <typename T>
static tca_status cgsr_apply_reduce(tca_operator *op, int which, cudaStream_t s)
{
    T *rg = (T *)op->p, *r = (T *)op->p_own, *w = (T *)op->q;
    const int32_t *done = &op->sc->done;
    double *prw = op->part + kRedBlocks;
    int nrw = kRedBlocks;
    static const bool no_fused_dot = getenv("TCA_NO_FUSED_DOT") != nullptr;
    if (fused_used(op, rg, w) && !no_fused_dot) {
        TCA_TRY(timed_apply(op, rg, w, which == 7 ? nullptr : done, s, prw));   // W := A*R, R+*W
        nrw = op->band_grid;
    } else {
        TCA_TRY(timed_apply(op, rg, w, which == 7 ? nullptr : done, s));
        launch_dot_partials<T>(r, w, op->N, prw, which == 7 ? nullptr : done, s);
    }
    if (!op->transport) {
        launch_cgsr_finalize(which, op->part, kRedBlocks, prw, nrw, op->sc, op->hist, s, 0);
        return TCA_OK;
    }
    launch_cgsr_finalize(which, op->part, kRedBlocks, prw, nrw, op->sc, op->hist, s, 1);
    TCA_TRY(op->transport->allreduce(&op->sc->red[3], 2, s));   // gamma and delta together
    launch_cgsr_finalize(which, op->part, kRedBlocks, prw, nrw, op->sc, op->hist, s, 2);
    return TCA_OK;
}

// One iteration of Fig. 2 (op->solver == 0), of its preconditioned form
// (1: Z := P^-1 R, rho := R+*Z, P := Z + beta P) or of the single-reduction
// rearrangement (2, reading Z24).
template <typename T>
static tca_status cg_iteration(tca_operator *op, T *x, cudaStream_t s)
{
    T *r = (T *)op->r, *pe = (T *)op->p, *p = (T *)op->p_own, *q = (T *)op->q;
    const int32_t *done = &op->sc->done;
    if (op->solver == 3) {   // tensor Jacobi (Fig. 1): U := U - R*E; R := A*U - B; R+*R
        launch_jacobi_update<T>(x, (const T *)op->r, (const T *)op->jac_e, op->N, op->sc, s);
        TCA_TRY(timed_apply(op, x, q, done, s));
        launch_jacobi_resid<T>((T *)op->r, q, (const T *)op->jac_b, op->N, op->part, done, s);
        launch_jacobi_finalize(1, op->part, kRedBlocks, op->sc, op->hist, s);
        return TCA_OK;
    }
    if (op->solver == 2) {   // P := R + beta P, S := W + beta S, C += alpha P, R -= alpha S, R+*R
        launch_cgsr_update<T>(x, (T *)op->r, (T *)op->sr_s, (T *)op->p_own, (const T *)op->q, op->N, op->sc,
                              op->part, s);
        TCA_TRY(halo_p(op, s));                                         // ghost slabs of R
        return cgsr_apply_reduce<T>(op, 6, s);                          // W := A*R; gamma, delta, alpha, beta
    }
    if (op->b1 == 1) {   // fused step B1': C += alpha P_old, P := R|Z + beta P_old, Q := A*P, P+*Q
        T *pold = (T *)(op->pcur ? op->p2 : op->p_own), *pnew = (T *)(op->pcur ? op->p_own : op->p2);
        const T *d = op->solver == 1 ? (const T *)op->z : r;
        TCA_TRY(timed_call(op, s, [&] { return launch_fused_b1(op, pold, pnew, d, q, x, op->part, s); }));
        op->pcur ^= 1;
        TCA_TRY(cg_reduce(op, 1, op->part, op->band_grid_fu, s));     // alpha
        TCA_TRY(update_r_reduce<T>(op, r, q, s));       // R := R - alpha*Q, R+*R; rho1 (PCG: R+*R), stop, beta
        if (op->solver == 1) {
            T *z = (T *)op->z;
            TCA_TRY(apply_precond<T>(op, r, z, done, s));              // Z := P^-1 R
            launch_dot_partials<T>(r, z, op->N, op->part, done, s);    // R+*Z
            TCA_TRY(cg_reduce(op, 3, op->part, kRedBlocks, s));        // rho1, beta
        }
        return TCA_OK;   // C and P are updated by the next step's B1' (or b1_finish)
    }
    if (op->dx == 1) {   // deferred C update: Q := A*P, P+*Q, C += alpha_prev P_prev in the apply (MODE 2)
        T *pc = (T *)(op->pcur ? op->p2 : op->p_own), *pp = (T *)(op->pcur ? op->p_own : op->p2);
        TCA_TRY(timed_call(op, s, [&] { return launch_fused_dx(op, pc, q, x, pp, op->part, s); }));
        TCA_TRY(cg_reduce(op, 1, op->part, op->band_grid_dx, s));   // alpha
        TCA_TRY(update_r_reduce<T>(op, r, q, s));     // R := R - alpha*Q, R+*R; rho1 (PCG: R+*R), stop, beta
        const T *d = r;
        if (op->solver == 1) {
            T *z = (T *)op->z;
            TCA_TRY(apply_precond<T>(op, r, z, done, s));            // Z := P^-1 R
            launch_dot_partials<T>(r, z, op->N, op->part, done, s);  // R+*Z
            TCA_TRY(cg_reduce(op, 3, op->part, kRedBlocks, s));      // rho1, beta
            d = z;
        }
        launch_cg_update_p<T>(pp, pc, d, op->N, op->sc, s);          // P_next := R|Z + beta*P (other buffer)
        op->pcur ^= 1;
        return TCA_OK;   // C += alpha P: by the next apply (or after the loop)
    }
    static const bool no_fused_dot = getenv("TCA_NO_FUSED_DOT") != nullptr;   // measurement switch
    static const bool no_fin = getenv("TCA_NO_FUSED_FIN") != nullptr;   // measurement switch
    if (fused_used(op, pe, q) && !no_fused_dot) {
        op->band_fin_req = !no_fin;                                   // alpha in the apply's last CTA
        op->band_fin_done = false;
        const tca_status st = timed_apply(op, pe, q, done, s, op->part);   // Q := A*(P*D), P+*Q in the epilogue
        op->band_fin_req = false;
        TCA_TRY(st);
        if (!op->band_fin_done) TCA_TRY(cg_reduce(op, 1, op->part, op->band_grid, s));   // alpha
    } else {
        TCA_TRY(timed_apply(op, pe, q, done, s));                     // Q := A*(P*D)
        launch_dot_partials<T>(p, q, op->N, op->part, done, s);      // P+*Q
        TCA_TRY(cg_reduce(op, 1, op->part, kRedBlocks, s));          // alpha
    }
    TCA_TRY(update_r_reduce<T>(op, r, q, s));         // R := R - alpha*Q, R+*R; rho1 (PCG: R+*R), stop, beta
    const T *d = r;
    if (op->solver == 1) {
        T *z = (T *)op->z;
        TCA_TRY(apply_precond<T>(op, r, z, done, s));                // Z := P^-1 R
        launch_dot_partials<T>(r, z, op->N, op->part, done, s);      // R+*Z
        TCA_TRY(cg_reduce(op, 3, op->part, kRedBlocks, s));          // rho1, beta
        d = z;
    }
    const int64_t hb = (int64_t)kHG * op->slab;   // elements of the 3 boundary slabs
    if (op->transport && op->transport->async_halo() && op->nloc1 > 2 * kHG && (hb * op->esize) % 16 == 0) {
        // the boundary slabs of P first; their halo exchange runs on a side
        // stream under the update of the interior slabs (joined before the
        // next apply, which is the only reader of the ghost slabs)
        const int64_t n = op->N;
        if (!op->hstream) {
            TCA_CUDA_TRY(cudaStreamCreateWithFlags(&op->hstream, cudaStreamNonBlocking));
            TCA_CUDA_TRY(cudaEventCreateWithFlags(&op->hfork, cudaEventDisableTiming));
            TCA_CUDA_TRY(cudaEventCreateWithFlags(&op->hjoin, cudaEventDisableTiming));
        }
        launch_cg_update_xp<T>(x, p, d, hb, op->sc, s);                              // slabs [0, 3)
        launch_cg_update_xp<T>(x + n - hb, p + n - hb, d + n - hb, hb, op->sc, s);   // slabs [nloc-3, nloc)
        TCA_CUDA_TRY(cudaEventRecord(op->hfork, s));
        TCA_CUDA_TRY(cudaStreamWaitEvent(op->hstream, op->hfork, 0));
        TCA_TRY(halo_p(op, op->hstream));
        TCA_CUDA_TRY(cudaEventRecord(op->hjoin, op->hstream));
        launch_cg_update_xp<T>(x + hb, p + hb, d + hb, n - 2 * hb, op->sc, s);       // interior
        TCA_CUDA_TRY(cudaStreamWaitEvent(s, op->hjoin, 0));
        return TCA_OK;
    }
    launch_cg_update_xp<T>(x, p, d, op->N, op->sc, s);               // C := C + alpha*P*D, P := R|Z + beta*P
    return halo_p(op, s);                                             // ghost slabs of P
}

// CG iterations as CUDA graphs: chunks of kGraphChunk iterations captured once
// (per x pointer and timing mode) and relaunched; the first iteration runs
// eagerly (it creates the tensor maps the captured applies use).  Removes the
// per-launch host cost (the fused apply carries a ~31 KB parameter block), which
// dominates the small configs.  Later kernels of a converged solve are no-ops
// (device `done` flag), so the returned x is exactly x_k.
constexpr int kGraphChunk = 32;
constexpr int kTimingStride = 16;   // timed iterations per captured chunk: every 16th

static void destroy_graphs(tca_operator *op)
{
    for (int g = 0; g < 2; ++g) {
        if (op->gexec[g]) cudaGraphExecDestroy(op->gexec[g]);
        op->gexec[g] = nullptr;
        op->gpend[g] = false;
        for (cudaEvent_t e : op->gev[g]) cudaEventDestroy(e);
        op->gev[g].clear();
    }
    op->gx = nullptr;
    // the captured launches were the only users of pinned tensor-map slots
    // (launches after the caller's stream joined the graph stream are ordered
    // after any replay, so the slots may be recycled again)
    op->tmap_pinned = 0;
}

template <typename T>
static tca_status capture_chunk(tca_operator *op, T *x, int g)
{
    cudaGraph_t graph = nullptr;
    TCA_CUDA_TRY(cudaStreamBeginCapture(op->gstream, cudaStreamCaptureModeThreadLocal));
    tca_status st = TCA_OK;
    const int64_t k0 = g_launches.load();
    // timing samples the applies of every kTimingStride-th iteration of the
    // chunk: an external event node pair costs ~20 us of replay time, which
    // timing every apply would add to the solve it measures
    op->capturing = true;
    for (int i = 0; i < kGraphChunk && st == TCA_OK; ++i) {
        op->cap_ev = op->timing && i % kTimingStride == 0 ? &op->gev[g] : nullptr;
        st = cg_iteration<T>(op, x, op->gstream);
    }
    cudaError_t e = cudaStreamEndCapture(op->gstream, &graph);
    op->capturing = false;
    op->cap_ev = nullptr;
    // captured launches run at each replay, not now (single-threaded per operator)
    op->gkernels[g] = g_launches.load() - k0;
    count_launch(-op->gkernels[g]);
    if (st != TCA_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    TCA_CUDA_TRY(e);
    e = cudaGraphInstantiate(&op->gexec[g], graph, 0);
    cudaGraphDestroy(graph);
    TCA_CUDA_TRY(e);
    return TCA_OK;
}

template <typename T>
static tca_status cg_graph_loop(tca_operator *op, T *x, double rtol, int32_t max_iters, cudaStream_t s)
{
    TCA_TRY(cg_iteration<T>(op, x, s));   // eager first iteration
    int done_iters = 1;
    if (!op->gstream) {
        TCA_CUDA_TRY(cudaStreamCreateWithFlags(&op->gstream, cudaStreamNonBlocking));
        TCA_CUDA_TRY(cudaEventCreateWithFlags(&op->gfork, cudaEventDisableTiming));
        TCA_CUDA_TRY(cudaEventCreateWithFlags(&op->gjoin, cudaEventDisableTiming));
    }
    // with timing, two instances alternate: instance g's events are read while
    // the other instance is queued behind it, so the GPU never drains
    const int ng = op->timing ? 2 : 1;
    if (!op->gexec[0] || op->gx != (const void *)x || op->gtimed != op->timing || op->gsolver != op->solver ||
        op->gb != op->jac_b) {
        TCA_TRY(harvest_timing(op));
        destroy_graphs(op);
        for (int g = 0; g < ng; ++g) TCA_TRY(capture_chunk<T>(op, x, g));
        op->gx = x;
        op->gtimed = op->timing;
        op->gsolver = op->solver;
        op->gb = op->jac_b;
    }
    TCA_CUDA_TRY(cudaEventRecord(op->gfork, s));
    TCA_CUDA_TRY(cudaStreamWaitEvent(op->gstream, op->gfork, 0));
    int g = 0;
    while (done_iters + kGraphChunk <= max_iters) {
        TCA_TRY(harvest_graph(op, g));   // its previous replay (the other instance is queued)
        TCA_CUDA_TRY(cudaGraphLaunch(op->gexec[g], op->gstream));
        count_launch(op->gkernels[g]);
        op->gpend[g] = op->timing != 0;
        done_iters += kGraphChunk;
        if (rtol > 0.0) {   // tolerance stop: check the device flag once per chunk
            TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_host, op->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost,
                                         op->gstream));
            TCA_TRY(sync_solve(op, op->gstream));
            if (op->sc_host->done) break;
        }
        g = (g + 1) % ng;
    }
    if (!op->sc_host->done || rtol <= 0.0)
        for (; done_iters < max_iters; ++done_iters) TCA_TRY(cg_iteration<T>(op, x, op->gstream));
    TCA_CUDA_TRY(cudaEventRecord(op->gjoin, op->gstream));
    TCA_CUDA_TRY(cudaStreamWaitEvent(s, op->gjoin, 0));
    return TCA_OK;
}

// E := InvMainDiag(A) once per operator (tensor Jacobi)
template <typename T>
static tca_status jacobi_prepare(tca_operator *op, cudaStream_t s)
{
    if (op->jac_e) return TCA_OK;
    int nmax = 1;
    for (int d = 0; d < kD; ++d) nmax = std::max(nmax, (int)op->n[d]);
    bool have_g = true;
    std::vector<double> dg((size_t)4 * nmax, 0.0), dr((size_t)4 * nmax, 0.0);
    for (int d = 0; d < kD; ++d) {
        const int nd = (int)op->n[d];
        bool nz = false;
        for (int i = 0; i < nd; ++i) {
            dg[(size_t)d * nmax + i] = op->Gh[d][(size_t)i * nd + i];
            nz = nz || op->Gh[d][(size_t)i * nd + i] != 0.0;
            if (op->has_reg[d]) dr[(size_t)d * nmax + i] = op->Rh[d][(size_t)i * nd + i];
        }
        // an all-zero G_d (Gram form without a product term) makes the product term vanish
        have_g = have_g && nz;
    }
    double *buf = nullptr;
    const size_t nb = sizeof(double) * 8 * nmax;
    TCA_CUDA_TRY(dev_get((void **)&buf, nb));
    TCA_CUDA_TRY(cudaMemcpyAsync(buf, dg.data(), nb / 2, cudaMemcpyHostToDevice, s));
    TCA_CUDA_TRY(cudaMemcpyAsync(buf + 4 * nmax, dr.data(), nb / 2, cudaMemcpyHostToDevice, s));
    TCA_CUDA_TRY(cudaMallocAsync(&op->jac_e, (size_t)op->N * op->esize, s));
    launch_jacobi_diag<T>((T *)op->jac_e, op->N, op->n, buf, buf + 4 * nmax, nmax, op->lambda, have_g, s);
    TCA_CUDA_TRY(cudaStreamSynchronize(s));
    dev_put(buf, nb);
    return TCA_OK;
}

// Fig. 2 / PCG / single-reduction CG / tensor Jacobi from the start phase
// through the last iteration on the general (multi-kernel, graph-captured) path.
template <typename T>
static tca_status cg_run(tca_operator *op, const T *b, T *x, double rtol, int32_t max_iters, CgScalars h,
                         cudaStream_t s, int pcg, int x0_zero)
{
    double *part_bb = op->part + 2 * kRedBlocks;   // <b, b> partials (warm start)
    if (pcg == 3) {   // tensor Jacobi: U := 0, E := InvMainDiag(A), R := A*U - B
        h.thr = rtol;
        *op->sc_host = h;
        TCA_CUDA_TRY(cudaMemcpyAsync(op->sc, op->sc_host, sizeof(CgScalars), cudaMemcpyHostToDevice, s));
        TCA_TRY(jacobi_prepare<T>(op, s));
        op->jac_b = b;
        TCA_CUDA_TRY(cudaMemsetAsync(x, 0, (size_t)op->N * op->esize, s));
        TCA_TRY(timed_apply(op, x, (T *)op->q, nullptr, s));
        launch_jacobi_resid<T>((T *)op->r, (const T *)op->q, b, op->N, op->part, nullptr, s);
        launch_jacobi_finalize(0, op->part, kRedBlocks, op->sc, op->hist, s);
    } else if (pcg == 2) {   // single-reduction CG: R := B - A*C (ghosted), P := 0, S := 0, W := A*R
        if (!op->sr_s) TCA_CUDA_TRY(cudaMallocAsync(&op->sr_s, (size_t)op->N * op->esize, s));
        if (x0_zero) {
            launch_cg_init<T>(b, x, (T *)op->p_own, (T *)op->r, op->N, op->part, s);   // gamma0 partials
        } else {   // warm start (Fig. 2's R := B - A*C)
            TCA_TRY(apply_any(op, x, op->q, s, false));
            launch_resid2<T>(b, (const T *)op->q, (T *)op->p_own, nullptr, op->N, op->part, part_bb, s);
        }
        TCA_CUDA_TRY(cudaMemsetAsync(op->r, 0, (size_t)op->N * op->esize, s));
        TCA_CUDA_TRY(cudaMemsetAsync(op->sr_s, 0, (size_t)op->N * op->esize, s));
        TCA_TRY(halo_p(op, s));
        TCA_TRY(cgsr_apply_reduce<T>(op, 7, s));
        if (!x0_zero) TCA_TRY(cg_reduce(op, 8, part_bb, kRedBlocks, s));           // stop reference <b, b>
    } else if (x0_zero) {
        launch_cg_init<T>(b, x, (T *)op->r, (T *)op->p_own, op->N, op->part, s);   // C := 0, R := B, P := R
        TCA_TRY(cg_reduce(op, 0, op->part, kRedBlocks, s));                       // rho0 := R+*R
    } else {   // warm start: R := B - A*C, P := R (Fig. 2; reading Z28)
        TCA_TRY(apply_any(op, x, op->q, s, false));
        launch_resid2<T>(b, (const T *)op->q, (T *)op->r, (T *)op->p_own, op->N, op->part, part_bb, s);
        TCA_TRY(cg_reduce(op, 0, op->part, kRedBlocks, s));                       // rho0 := R+*R
        TCA_TRY(cg_reduce(op, 8, part_bb, kRedBlocks, s));                        // stop reference <b, b>
    }
    if (pcg == 1) {   // Z := P^-1 R, P := Z, rho := R+*Z
        T *z = (T *)op->z;
        TCA_TRY(apply_precond<T>(op, (const T *)op->r, z, &op->sc->done, s));
        TCA_CUDA_TRY(cudaMemcpyAsync(op->p_own, z, (size_t)op->N * op->esize, cudaMemcpyDeviceToDevice, s));
        launch_dot_partials<T>((const T *)op->r, z, op->N, op->part, &op->sc->done, s);
        TCA_TRY(cg_reduce(op, 4, op->part, kRedBlocks, s));
    }
    TCA_TRY(halo_p(op, s));
    static const bool no_graph = getenv("TCA_NO_GRAPH") != nullptr;   // measurement switch
    if (pcg == 3) rtol = 1.0;   // Jacobi stops on its threshold: poll the device flag per chunk
    // graphs also with an NCCL transport (its calls are stream-ordered and
    // capture into the graph); not with the host-synchronised local transport
    if ((!op->transport || op->transport->capturable()) && !no_graph && max_iters > 1) {
        TCA_TRY(cg_graph_loop<T>(op, x, rtol, max_iters, s));
    } else if (rtol <= 0.0) {
        for (int k = 0; k < max_iters; ++k) TCA_TRY(cg_iteration<T>(op, x, s));
    } else {
        const int chunk = 32;
        for (int k = 0; k < max_iters; k += chunk) {
            const int c = std::min(chunk, max_iters - k);
            for (int i = 0; i < c; ++i) TCA_TRY(cg_iteration<T>(op, x, s));
            TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_host, op->sc, sizeof(CgScalars),
                                         cudaMemcpyDeviceToHost, s));
            TCA_TRY(sync_solve(op, s));
            if (op->timing) TCA_TRY(harvest_timing(op));
            if (op->sc_host->done) break;
        }
    }
    if (op->b1 == 1)   // the last step's pending C := C + alpha P (x only: done is set)
        launch_cg_update_xp<T>(x, (T *)(op->pcur ? op->p2 : op->p_own), (const T *)op->r, op->N, op->sc, s);
    if (op->dx == 1)   // the last iteration's pending C := C + alpha P (its P: the buffer before the flip)
        launch_cg_update_xp<T>(x, (T *)(op->pcur ? op->p_own : op->p2), (const T *)op->r, op->N, op->sc, s);
    return TCA_OK;
}

template <typename T>
static tca_status cg_t(tca_operator *op, const T *b, T *x, double rtol, int32_t max_iters,
                       tca_cg_report *rep, cudaStream_t s, int pcg = 0, int x0_zero = 1)
{
    double *part_bb = op->part + 2 * kRedBlocks;   // <b, b> partials (warm start, report)
    CgScalars h{};
    h.rtol2 = rtol > 0.0 ? rtol * rtol : 0.0;
    h.max_iters = max_iters;
    h.pcg = pcg == 1;
    op->solver = pcg;
    const bool tiny = pcg == 0 && tiny_cg_eligible(op);
    const bool gridc = !tiny && pcg == 0 && grid_cg_eligible(op);
    if (op->b1 < 0) {   // fused step B1' for Fig. 2 / PCG on one GPU: opt-in (TCA_B1=1), see DESIGN.md 6.5
        const char *b1env = getenv("TCA_B1");
        const bool want_b1 = b1env && b1env[0] == '1';
        op->b1 = (want_b1 && fused_used(op, op->p_own, op->q) && fused_b1_supported(op)) ? 1 : 0;
        if (op->b1 == 1) {
            cudaError_t e = cudaMallocAsync(&op->p2, (size_t)op->N * op->esize, s);
            if (e != cudaSuccess) { op->b1 = 0; cudaGetLastError(); }
        }
    }
    if (op->dx < 0) {   // deferred C update in the apply: default on for fp32 (TCA_DX=0|1 forces)
        const char *e = getenv("TCA_DX");
        const bool want = (e && (e[0] == '0' || e[0] == '1') ? e[0] == '1' : op->dtype == TCA_F32) && op->b1 != 1;
        op->dx = (want && !op->transport && fused_used(op, op->p_own, op->q) && fused_dx_supported(op)) ? 1 : 0;
        if (op->dx == 1 && !op->p2) {
            cudaError_t e2 = cudaMallocAsync(&op->p2, (size_t)op->N * op->esize, s);
            if (e2 != cudaSuccess) { op->dx = 0; cudaGetLastError(); }
        }
    }
    const int b1_saved = op->b1, dx_saved = op->dx;
    if (pcg == 2 || pcg == 3 || tiny || gridc) op->b1 = 0;   // single-reduction CG, Jacobi, whole-solve engines: own steps
    if (pcg == 2 || pcg == 3 || tiny || gridc || op->b1 == 1) op->dx = 0;
    op->pcur = 0;
    if (op->dx == 1) {
        const void *ptrs[3] = {op->p_own, op->p2, op->q};
        const int kinds[3] = {0, 0, 1};
        TCA_TRY(fused_dx_prepare(op, ptrs, kinds, 3, s));
    }
    if (op->b1 == 1) {
        const void *ptrs[4] = {op->p_own, op->p2, pcg == 1 ? op->z : op->r, op->q};
        const int kinds[4] = {0, 0, 0, 1};
        TCA_TRY(fused_b1_prepare(op, ptrs, kinds, 4, s));
    }
    *op->sc_host = h;
    TCA_CUDA_TRY(cudaMemcpyAsync(op->sc, op->sc_host, sizeof(CgScalars), cudaMemcpyHostToDevice, s));
    TCA_CUDA_TRY(cudaEventRecord(op->ev0, s));
    if (tiny) TCA_TRY(launch_tiny_cg(op, b, x, x0_zero, s));        // whole solve in one block (tca_tiny.cu)
    else {
        bool launched = false;   // whole solve, one cooperative grid (tca_grid.cu)
        if (gridc) TCA_TRY(launch_grid_cg(op, b, x, x0_zero, s, &launched));
        if (!launched) TCA_TRY(cg_run<T>(op, b, x, rtol, max_iters, h, s, pcg, x0_zero));
    }
    op->b1 = b1_saved;
    op->dx = dx_saved;
    TCA_CUDA_TRY(cudaGetLastError());
    TCA_CUDA_TRY(cudaEventRecord(op->ev1, s));
    if (rep) {   // true residual |b - M x_k| / |b| (reading Z2): one more apply, after the timed solve
        TCA_TRY(apply_any(op, x, op->q, s, false));
        launch_resid2<T>(b, (const T *)op->q, nullptr, nullptr, op->N, op->part, part_bb, s);
        launch_cg_finalize(8, op->part, kRedBlocks, op->sc, nullptr, s, 1);
        launch_cg_finalize(9, part_bb, kRedBlocks, op->sc, nullptr, s, 1);
        if (op->transport) TCA_TRY(op->transport->allreduce(&op->sc->red[8], 2, s));
    }
    TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_host, op->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
    TCA_TRY(sync_solve(op, s));
    if (op->timing) TCA_TRY(harvest_timing(op));
    const CgScalars &r = *op->sc_host;
    if (rep) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, op->ev0, op->ev1);
        rep->iterations = r.iters;
        rep->converged = r.converged;
        rep->status = r.status;
        rep->rho0 = r.rho0;
        rep->rho_final = r.rr;
        rep->relres_final = r.red[9] > 0.0 ? sqrt(r.red[8] / r.red[9]) : (r.red[8] > 0.0 ? INFINITY : 0.0);
        rep->seconds = ms * 1e-3;
        if (rep->rho_history && rep->history_capacity > 0) {
            const int cnt = std::min(rep->history_capacity, r.iters + 1);
            TCA_CUDA_TRY(cudaMemcpy(rep->rho_history, op->hist, sizeof(double) * cnt,
                                    cudaMemcpyDeviceToHost));
        }
    }
    return (tca_status)r.status;
}

static tca_status check_op(const tca_operator *op)
{
    if (!op) return fail(TCA_ERR_INVALID_ARG, "op is NULL");
    return TCA_OK;
}

}  // namespace tca

using namespace tca;

extern "C" {

const char *tca_version(void) { return "tca 0.1 sm_100a"; }

const char *tca_last_error(void) { return g_last_error.c_str(); }

const char *tca_status_string(tca_status s)
{
    switch (s) {
    case TCA_OK: return "TCA_OK";
    case TCA_ERR_INVALID_ARG: return "TCA_ERR_INVALID_ARG";
    case TCA_ERR_SHAPE: return "TCA_ERR_SHAPE";
    case TCA_ERR_NOT_SPD: return "TCA_ERR_NOT_SPD";
    case TCA_ERR_OOM: return "TCA_ERR_OOM";
    case TCA_ERR_CUDA: return "TCA_ERR_CUDA";
    case TCA_ERR_NCCL: return "TCA_ERR_NCCL";
    case TCA_ERR_BREAKDOWN: return "TCA_ERR_BREAKDOWN";
    case TCA_ERR_NONFINITE: return "TCA_ERR_NONFINITE";
    case TCA_NOT_CONVERGED: return "TCA_NOT_CONVERGED";
    }
    return "TCA_UNKNOWN_STATUS";
}

void tca_operator_destroy(tca_operator *op)
{
    if (!op) return;
    for (int d = 0; d < kD; ++d) {
        free_band(op->Gm[d]);
        free_band(op->Rm[d]);
        free_band(op->At[d]);
        free_band(op->Af[d]);
        free_band(op->pc_inv[d]);
    }
    delete op->transport;
    destroy_graphs(op);
    if (op->gstream) cudaStreamDestroy(op->gstream);
    if (op->gfork) cudaEventDestroy(op->gfork);
    if (op->gjoin) cudaEventDestroy(op->gjoin);
    if (op->hstream) cudaStreamDestroy(op->hstream);
    if (op->hfork) cudaEventDestroy(op->hfork);
    if (op->hjoin) cudaEventDestroy(op->hjoin);
    // every stream that used the operator is done before its memory goes back
    cudaDeviceSynchronize();
    void *pooled[] = {op->r, op->p, op->q, op->t0, op->t1, op->x_ext, op->z, op->pc_tmp, op->sr_s, op->p2,
                      op->jac_e, op->sc_t, op->sc_perm, op->sc_tstart, op->sc_coef, op->grid_ws};   // stream-ordered pool
    for (void *b : pooled)
        if (b) cudaFreeAsync(b, 0);
    dev_put(op->part, sizeof(double) * kRedBlocks * 3);
    dev_put(op->sc, sizeof(CgScalars));
    dev_put(op->hist, sizeof(double) * op->hist_cap);
    dev_put(op->tmap_dev, sizeof(TmapSlot::map) * kTmapSlots);
    dev_put(op->band_gtaps, op->band_gtaps_bytes);
    dev_put(op->ks_taps, op->ks_bytes);
    for (int d = 0; d < kD; ++d) dev_put(op->pc_tab[d], op->pc_tab_bytes[d]);
    pinned_put(op->sc_host, sizeof(CgScalars));
    pinned_put(op->tmap_host, sizeof(TmapSlot::map) * kTmapSlots);
    for (cudaEvent_t e : op->tmap_ev)
        if (e) cudaEventDestroy(e);
    if (op->ev0) cudaEventDestroy(op->ev0);
    if (op->ev1) cudaEventDestroy(op->ev1);
    for (cudaEvent_t e : op->tev) cudaEventDestroy(e);
    delete op;
}

// Gram form (tca_operator_create_gram): G_d / R_d given directly, A_d = I.
static tca_status create_impl(tca_operator **out, int order, const int64_t *n, const int64_t *m,
                              const double *const *A, const double *const *L, double lambda, tca_dtype dtype,
                              const tca_dist *dist, void *stream, bool gram_form, const double *const *Gin,
                              const double *const *Rin)
{
    if (!out) return fail(TCA_ERR_INVALID_ARG, "op (output pointer) is NULL");
    *out = nullptr;
    if (order < 1 || order > 4) return fail(TCA_ERR_INVALID_ARG, "order must be in 1..4");
    if (!n || !m || !A) return fail(TCA_ERR_INVALID_ARG, "n, m and A must be non-NULL");
    if (dtype != TCA_F64 && dtype != TCA_F32) return fail(TCA_ERR_INVALID_ARG, "dtype must be TCA_F64 or TCA_F32");
    if (!isfinite(lambda) || lambda < 0.0) return fail(TCA_ERR_INVALID_ARG, "lambda must be finite and >= 0");
    for (int d = 0; d < order; ++d) {
        if (n[d] < 1 || n[d] > (1 << 20)) return fail(TCA_ERR_SHAPE, "n[" + std::to_string(d) + "] out of range");
        if (m[d] < 1 || m[d] > (1 << 20)) return fail(TCA_ERR_SHAPE, "m[" + std::to_string(d) + "] out of range");
        if (!A[d]) return fail(TCA_ERR_INVALID_ARG, "A[" + std::to_string(d) + "] is NULL");
        if (!all_finite(A[d], (size_t)(n[d] * m[d])))
            return fail(TCA_ERR_INVALID_ARG, "A[" + std::to_string(d) + "] has non-finite entries");
        if (L && L[d] && n[d] >= 3 && !all_finite(L[d], (size_t)((n[d] - 2) * n[d])))
            return fail(TCA_ERR_INVALID_ARG, "L[" + std::to_string(d) + "] has non-finite entries");
    }
    {
        double vol = 1.0;   // generic mode products index a (rows x inner) plane with 32 bits
        for (int d = 0; d < order; ++d) vol *= (double)std::max(n[d], m[d]);
        if (vol >= 4294967295.0) return fail(TCA_ERR_SHAPE, "problem too large: prod max(n_d, m_d) must be < 2^32");
    }
    int64_t layout[4] = {0, n[0], 0, m[0]};   // own_lo, own_hi, data_lo, data_hi
    // sharded = a transport is given (nranks >= 1; one rank is the whole domain
    // with empty halos -- the single-GPU case of the distributed code path)
    const bool sharded = dist && (dist->nranks > 1 || dist->nccl_comm || dist->local_group);
    if (dist) {
        if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)
            return fail(TCA_ERR_INVALID_ARG, "dist: rank must be in [0, nranks)");
        if (sharded && !dist->nccl_comm && !dist->local_group)
            return fail(TCA_ERR_INVALID_ARG, "dist: a sharded operator needs nccl_comm or local_group");
        if (sharded && dist->nccl_comm && dist->local_group)
            return fail(TCA_ERR_INVALID_ARG, "dist: give exactly one of nccl_comm and local_group");
        if (sharded) TCA_TRY(shard_layout(n[0], A[0], m[0], dist->rank, dist->nranks, layout));
    }
    cudaStream_t s = (cudaStream_t)stream;

    tca_operator *op = new tca_operator();
    op->own_lo = layout[0];
    op->own_hi = layout[1];
    op->data_lo = layout[2];
    op->data_hi = layout[3];
    if (sharded) {
        op->rank = dist->rank;
        op->nranks = dist->nranks;
        op->comm = dist->nccl_comm;
        op->ghost = kHG;
        // unknown rows the shard's data rows touch (forward model, x NULL)
        op->xf_lo = n[0];
        op->xf_hi = 0;
        for (int64_t k = op->data_lo; k < op->data_hi; ++k)
            for (int64_t c = 0; c < n[0]; ++c)
                if (A[0][k * n[0] + c] != 0.0) {
                    op->xf_lo = std::min(op->xf_lo, c);
                    op->xf_hi = std::max(op->xf_hi, c + 1);
                }
        if (op->xf_hi <= op->xf_lo) { op->xf_lo = 0; op->xf_hi = 0; }
    } else {
        op->xf_lo = 0;
        op->xf_hi = n[0];
    }
    op->order = order;
    op->gram_form = gram_form;
    op->dtype = dtype;
    op->esize = dtype == TCA_F64 ? 8 : 4;
    op->lambda = lambda;
    for (int d = 0; d < order; ++d) {
        op->n[d] = n[d];
        op->m[d] = m[d];
    }
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&op->num_sms, cudaDevAttrMultiProcessorCount, dev);
        // rhs / forward-model / host-solve temporaries are stream-ordered
        // allocations of up to several GB: keep freed blocks in the device's
        // default pool (no unmap/remap of GBs at every synchronisation)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    size_t bytes = 0;
    tca_status st = TCA_OK;
    bool all_banded = true;
    for (int d = 0; d < kD && st == TCA_OK; ++d) {
        const int nd = (int)op->n[d], md = (int)op->m[d];
        std::vector<double> G, R, Ad;
        if (d < order && gram_form) {   // factors given: G_d (or none: zero), R_d (Eq. 9 Kronecker sum)
            G.assign((size_t)nd * nd, 0.0);
            if (Gin && Gin[d]) G.assign(Gin[d], Gin[d] + (size_t)nd * nd);
            if (Rin && Rin[d] && lambda > 0.0) {
                R.assign(Rin[d], Rin[d] + (size_t)nd * nd);
                op->has_reg[d] = 1;
                op->hbR[d] = half_bandwidth(R, nd);
            }
            for (int i = 0; i < nd && st == TCA_OK; ++i)
                for (int j = 0; j < i; ++j)
                    if (G[(size_t)i * nd + j] != G[(size_t)j * nd + i] ||
                        (!R.empty() && R[(size_t)i * nd + j] != R[(size_t)j * nd + i])) {
                        st = fail(TCA_ERR_INVALID_ARG, "G_" + std::to_string(d + 1) + " / R_" + std::to_string(d + 1) +
                                                           " must be symmetric");
                        break;
                    }
            if (st != TCA_OK) break;
            Ad.assign(A[d], A[d] + (size_t)md * nd);
        } else if (d < order) {
            G = gram(A[d], md, nd);                       // G_d = A_d^T A_d
            if (!cholesky_ok(G, nd)) {
                st = fail(TCA_ERR_NOT_SPD, "G_" + std::to_string(d + 1) + " = A^T A is not positive definite (A lacks full column rank)");
                break;
            }
            if (L && L[d] && nd >= 3 && lambda > 0.0) {
                R = gram(L[d], nd - 2, nd);               // R_d = L_d^T L_d
                op->has_reg[d] = 1;
                op->hbR[d] = half_bandwidth(R, nd);
            }
            Ad.assign(A[d], A[d] + (size_t)md * nd);
        } else {
            G.assign(1, 1.0);
            Ad.assign(1, 1.0);
        }
        op->Gh[d] = G;
        op->Rh[d] = R;
        op->hbG[d] = half_bandwidth(G, nd);
        const bool banded = op->hbG[d] <= kHG && (!op->has_reg[d] || op->hbR[d] <= kHR);
        if (banded) op->banded_mask |= (1 << d);
        else all_banded = false;
        st = make_band(dtype, G, nd, nd, banded ? kHG : -1, &op->Gm[d], &bytes);
        if (st != TCA_OK) break;
        if (op->has_reg[d]) {
            st = make_band(dtype, R, nd, nd, op->hbR[d] <= kHR ? kHR : -1, &op->Rm[d], &bytes);
            if (st != TCA_OK) break;
        }
        // A_d^T (rows n_d, cols m_d) for the rhs; A_d (rows m_d, cols n_d) for the
        // forward model.  Mode 1 of a shard: A_1^T rows [own_lo, own_hi) over data
        // columns [data_lo, data_hi); A_1 rows [data_lo, data_hi) over unknown
        // columns [xf_lo, xf_hi) (shard-local rhs and data, no communication).
        {
            const int64_t rlo = d == 0 ? op->own_lo : 0, rhi = d == 0 ? op->own_hi : nd;
            const int64_t clo = d == 0 ? op->data_lo : 0, chi = d == 0 ? op->data_hi : md;
            const int tr = (int)(rhi - rlo), tc = (int)(chi - clo);
            std::vector<double> At((size_t)tr * tc);
            for (int i = 0; i < tc; ++i)
                for (int j = 0; j < tr; ++j) At[(size_t)j * tc + i] = Ad[(size_t)(clo + i) * nd + rlo + j];
            st = make_band(dtype, At, tr, tc, -1, &op->At[d], &bytes);
            if (st != TCA_OK) break;
            const int64_t frlo = clo, frhi = chi;
            const int64_t fclo = d == 0 ? op->xf_lo : 0, fchi = d == 0 ? op->xf_hi : nd;
            const int fr = (int)(frhi - frlo), fc = (int)(fchi - fclo);
            std::vector<double> Af((size_t)fr * fc);
            for (int i = 0; i < fr; ++i)
                for (int j = 0; j < fc; ++j) Af[(size_t)i * fc + j] = Ad[(size_t)(frlo + i) * nd + fclo + j];
            st = make_band(dtype, Af, fr, fc, -1, &op->Af[d], &bytes);
            if (st != TCA_OK) break;
        }
        // symmetric band rows for the fused banded kernel
        op->bandG[d].assign((size_t)nd * 4, 0.0);
        op->bandR[d].assign((size_t)nd * 3, 0.0);
        for (int r = 0; r < nd; ++r) {
            for (int k = 0; k <= kHG; ++k)
                if (r + k < nd && k <= op->hbG[d]) op->bandG[d][(size_t)r * 4 + k] = G[(size_t)r * nd + r + k];
            if (op->has_reg[d])
                for (int k = 0; k <= kHR; ++k)
                    if (r + k < nd) op->bandR[d][(size_t)r * 3 + k] = lambda * R[(size_t)r * nd + r + k];
        }
    }
    if (st != TCA_OK) {
        tca_operator_destroy(op);
        return st;
    }
    op->all_banded = all_banded;
    op->nloc1 = op->own_hi - op->own_lo;
    op->slab = op->n[1] * op->n[2] * op->n[3];
    op->N = op->nloc1 * op->slab;
    op->Mloc = (op->data_hi - op->data_lo) * op->m[1] * op->m[2] * op->m[3];
    op->apply_path = fused_shape_supported(op) ? 1 : 0;
    if (gram_form && !Gin && !sharded) {   // Kronecker sum only, banded R_d: the stencil path
        bool ok = true;
        for (int d = 0; d < kD; ++d) ok = ok && (!op->has_reg[d] || op->hbR[d] <= kHR);
        if (ok) {
            std::vector<double> t;
            for (int d = 0; d < kD; ++d) {
                op->ks_off[d] = (int)(t.size() / 5);
                const int nd = (int)op->n[d];
                for (int r = 0; r < nd; ++r)
                    for (int k = -2; k <= 2; ++k) {
                        const int c = r + k;
                        t.push_back(op->has_reg[d] && c >= 0 && c < nd ? lambda * op->Rh[d][(size_t)r * nd + c] : 0.0);
                    }
            }
            std::vector<unsigned char> raw(t.size() * op->esize);
            if (dtype == TCA_F64) std::memcpy(raw.data(), t.data(), raw.size());
            else
                for (size_t i = 0; i < t.size(); ++i) reinterpret_cast<float *>(raw.data())[i] = (float)t[i];
            cudaError_t e0 = dev_get(&op->ks_taps, raw.size());
            if (e0 == cudaSuccess) e0 = cudaMemcpy(op->ks_taps, raw.data(), raw.size(), cudaMemcpyHostToDevice);
            if (e0 != cudaSuccess) {
                tca_operator_destroy(op);
                return cuda_fail(e0, "Kronecker-sum taps");
            }
            op->ks_bytes = raw.size();
            op->apply_path = 2;
        }
    }
    if (sharded && op->apply_path != 1) {
        tca_operator_destroy(op);
        return fail(TCA_ERR_INVALID_ARG,
                    "dist: sharded operators need the fused banded path (all modes banded, supported n4, "
                    "n3*n4*esize a multiple of 16 B)");
    }
    if (op->apply_path == 1) {
        const tca_status fs = fused_prepare(op);
        if (fs != TCA_OK) {
            tca_operator_destroy(op);
            return fs;
        }
    }
    if (sharded) op->transport = make_transport(dist);

    const size_t vb = (size_t)op->N * op->esize;
    const size_t pb = (size_t)(op->nloc1 + 2 * op->ghost) * op->slab * op->esize;   // ghosted p
    cudaError_t e = cudaSuccess;
    // the vector workspaces come from the device's stream-ordered pool (kept at
    // a maximal release threshold above): an operator created after another was
    // destroyed reuses its memory without new mappings
    e = cudaMallocAsync(&op->r, vb, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&op->p, pb, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(op->p, 0, pb, s);   // ghosts beyond the domain stay 0
    if (e == cudaSuccess) op->p_own = (char *)op->p + (size_t)op->ghost * op->slab * op->esize;
    if (e == cudaSuccess) e = cudaMallocAsync(&op->q, vb, s);
    if (e == cudaSuccess) e = dev_get((void **)&op->part, sizeof(double) * kRedBlocks * 3);
    if (e == cudaSuccess) e = dev_get((void **)&op->sc, sizeof(CgScalars));
    if (e == cudaSuccess) {
        op->sc_host = (CgScalars *)pinned_get(sizeof(CgScalars));
        if (!op->sc_host) e = cudaErrorMemoryAllocation;
    }
    if (e == cudaSuccess) e = cudaEventCreate(&op->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&op->ev1);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        tca_status rs = cuda_fail(e, "tca_operator_create workspace");
        tca_operator_destroy(op);
        return rs;
    }
    bytes += vb * 2 + pb + sizeof(double) * kRedBlocks * 2 + sizeof(CgScalars);
    op->device_bytes = bytes;
    *out = op;
    return TCA_OK;
}

tca_status tca_operator_create(tca_operator **out, int order, const int64_t *n, const int64_t *m,
                               const double *const *A, const double *const *L, double lambda,
                               tca_dtype dtype, const tca_dist *dist, void *stream)
{
    return create_impl(out, order, n, m, A, L, lambda, dtype, dist, stream, false, nullptr, nullptr);
}

tca_status tca_operator_create_gram(tca_operator **out, int order, const int64_t *n, const double *const *G,
                                    const double *const *R, double lambda, tca_dtype dtype, const tca_dist *dist,
                                    void *stream)
{
    if (!out) return fail(TCA_ERR_INVALID_ARG, "op (output pointer) is NULL");
    *out = nullptr;
    if (order < 1 || order > 4 || !n) return fail(TCA_ERR_INVALID_ARG, "order must be in 1..4 and n non-NULL");
    if (!G && !R) return fail(TCA_ERR_INVALID_ARG, "G and R are both NULL (empty operator)");
    std::vector<std::vector<double>> eye((size_t)order);
    const double *Ap[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int d = 0; d < order; ++d) {
        if (n[d] < 1 || n[d] > 4096) return fail(TCA_ERR_SHAPE, "n[" + std::to_string(d) + "] out of range");
        if (G && !G[d]) return fail(TCA_ERR_INVALID_ARG, "G[" + std::to_string(d) + "] is NULL (give all or none)");
        if (G && !all_finite(G[d], (size_t)(n[d] * n[d])))
            return fail(TCA_ERR_INVALID_ARG, "G[" + std::to_string(d) + "] has non-finite entries");
        if (R && R[d] && !all_finite(R[d], (size_t)(n[d] * n[d])))
            return fail(TCA_ERR_INVALID_ARG, "R[" + std::to_string(d) + "] has non-finite entries");
        eye[d].assign((size_t)(n[d] * n[d]), 0.0);
        for (int64_t i = 0; i < n[d]; ++i) eye[d][(size_t)(i * n[d] + i)] = 1.0;
        Ap[d] = eye[d].data();
    }
    return create_impl(out, order, n, n, Ap, nullptr, lambda, dtype, dist, stream, true, G, R);
}

tca_status tca_operator_create_scattered(tca_operator **out, int order, const int64_t *n, int64_t K,
                                        const double *t, const double *const *L, double lambda, tca_dtype dtype,
                                        void *stream)
{
    if (!out) return fail(TCA_ERR_INVALID_ARG, "op (output pointer) is NULL");
    *out = nullptr;
    if (order < 1 || order > 4 || !n) return fail(TCA_ERR_INVALID_ARG, "order must be in 1..4 and n non-NULL");
    if (K < 0) return fail(TCA_ERR_INVALID_ARG, "K must be >= 0");
    if (K > 0 && !t) return fail(TCA_ERR_INVALID_ARG, "t is NULL");
    std::vector<std::vector<double>> eye((size_t)order), R((size_t)order);
    const double *Ap[4] = {nullptr, nullptr, nullptr, nullptr}, *Rp[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int d = 0; d < order; ++d) {
        if (n[d] < 1 || n[d] > 4096) return fail(TCA_ERR_SHAPE, "n[" + std::to_string(d) + "] out of range");
        eye[d].assign((size_t)(n[d] * n[d]), 0.0);
        for (int64_t i = 0; i < n[d]; ++i) eye[d][(size_t)(i * n[d] + i)] = 1.0;
        Ap[d] = eye[d].data();
        if (L && L[d] && n[d] >= 3) {   // R_d = L_d^T L_d (reading Z7)
            const int64_t nd = n[d];
            if (!all_finite(L[d], (size_t)((nd - 2) * nd)))
                return fail(TCA_ERR_INVALID_ARG, "L[" + std::to_string(d) + "] has non-finite entries");
            R[d].assign((size_t)(nd * nd), 0.0);
            for (int64_t k = 0; k < nd - 2; ++k)
                for (int64_t i = 0; i < nd; ++i) {
                    const double a = L[d][k * nd + i];
                    if (a == 0.0) continue;
                    for (int64_t j = 0; j < nd; ++j) R[d][(size_t)(i * nd + j)] += a * L[d][k * nd + j];
                }
            Rp[d] = R[d].data();
        }
    }
    for (int64_t k = 0; k < K; ++k)
        for (int d = 0; d < order; ++d) {
            const double v = t[k * order + d];
            if (!(v >= 0.0 && v <= (double)(n[d] - 1)))
                return fail(TCA_ERR_INVALID_ARG, "t[" + std::to_string(k) + "][" + std::to_string(d) +
                                                     "] outside [0, n_d - 1] (or not finite)");
        }
    tca_operator *op = nullptr;
    TCA_TRY(create_impl(&op, order, n, n, Ap, nullptr, lambda, dtype, nullptr, stream, true, nullptr, Rp));
    if (op->apply_path != 2) {
        tca_operator_destroy(op);
        return fail(TCA_ERR_INVALID_ARG, "scattered operator: L_d must give banded R_d (half-bandwidth <= 2)");
    }
    op->scat = true;
    op->Mloc = K;
    tca_status st = scatter_prepare(op, K, t, (cudaStream_t)stream);
    if (st != TCA_OK) {
        tca_operator_destroy(op);
        return st;
    }
    *out = op;
    return TCA_OK;
}

tca_status tca_operator_query(const tca_operator *op, int64_t *own_lo, int64_t *own_hi,
                              int64_t *data_lo, int64_t *data_hi, int *banded_mask,
                              int *half_bw, size_t *device_bytes)
{
    TCA_TRY(check_op(op));
    if (own_lo) *own_lo = op->own_lo;
    if (own_hi) *own_hi = op->own_hi;
    if (data_lo) *data_lo = op->data_lo;
    if (data_hi) *data_hi = op->data_hi;
    if (banded_mask) *banded_mask = op->banded_mask & ((1 << op->order) - 1);
    if (half_bw)
        for (int d = 0; d < op->order; ++d) half_bw[d] = op->hbG[d];
    if (device_bytes) *device_bytes = op->device_bytes;
    return TCA_OK;
}

int tca_operator_apply_path(const tca_operator *op) { return op ? op->apply_path : -1; }

int tca_operator_cg_fused_step(const tca_operator *op) { return op ? op->b1 : -1; }

int tca_operator_cg_deferred_x(const tca_operator *op) { return op ? op->dx : -1; }

int tca_operator_cg_engine(const tca_operator *op)
{
    if (!op) return -1;
    if (tiny_cg_eligible(op)) return 1;
    return grid_cg_eligible(op) ? 2 : 0;
}

tca_status tca_apply(const tca_operator *op, const void *x, void *y, void *stream)
{
    TCA_TRY(check_op(op));
    if (!x || !y) return fail(TCA_ERR_INVALID_ARG, "x and y must be non-NULL device pointers");
    if (x == y) return fail(TCA_ERR_INVALID_ARG, "x and y must not alias");
    cudaStream_t s = (cudaStream_t)stream;
    tca_operator *o = const_cast<tca_operator *>(op);
    TCA_TRY(apply_any(o, x, y, s, true));   // sharded: ghosted copy of x, halo exchange, then the apply
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

tca_status tca_operator_set_timing(tca_operator *op, int enable)
{
    TCA_TRY(check_op(op));
    op->timing = enable ? 1 : 0;
    return TCA_OK;
}

tca_status tca_operator_get_timing(tca_operator *op, double *apply_ms, int64_t *apply_count,
                                   int reset)
{
    TCA_TRY(check_op(op));
    TCA_TRY(harvest_timing(op));
    if (apply_ms) *apply_ms = op->apply_ms;
    if (apply_count) *apply_count = op->apply_count;
    if (reset) {
        op->apply_ms = 0.0;
        op->apply_count = 0;
    }
    return TCA_OK;
}

int64_t tca_kernel_launches(void) { return g_launches.load(); }

tca_status tca_rhs(const tca_operator *op, const void *ydata, void *b, void *stream)
{
    TCA_TRY(check_op(op));
    if (!ydata || !b) return fail(TCA_ERR_INVALID_ARG, "ydata and b must be non-NULL device pointers");
    cudaStream_t s = (cudaStream_t)stream;
    if (op->scat) {   // b = sum_k y_k w_k
        TCA_CUDA_TRY(cudaMemsetAsync(b, 0, (size_t)op->N * op->esize, s));
        return launch_scatter(op, 1, nullptr, b, ydata, nullptr, s);
    }
    if (op->gram_form) return fail(TCA_ERR_INVALID_ARG, "tca_rhs: operator was created from its factors (no A_d)");
    if (op->dtype == TCA_F64) TCA_TRY(rhs_t<double>(op, (const double *)ydata, (double *)b, s));
    else TCA_TRY(rhs_t<float>(op, (const float *)ydata, (float *)b, s));
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

static tca_status solve_common(tca_operator *op, const void *b, void *x, double rtol, int32_t max_iters,
                               tca_cg_report *rep, void *stream, int pcg, int x0_zero = 1)
{
    TCA_TRY(check_op(op));
    if (!b || !x) return fail(TCA_ERR_INVALID_ARG, "b and x must be non-NULL device pointers");
    if (b == x) return fail(TCA_ERR_INVALID_ARG, "b and x must not alias");
    if (max_iters < 0) return fail(TCA_ERR_INVALID_ARG, "max_iters must be >= 0");
    if (!isfinite(rtol)) return fail(TCA_ERR_INVALID_ARG, "rtol must be finite");
    cudaStream_t s = (cudaStream_t)stream;
    if (op->hist_cap < max_iters + 1) {
        destroy_graphs(op);   // captured iterations reference the old history buffer
        TCA_CUDA_TRY(cudaStreamSynchronize(s));
        dev_put(op->hist, sizeof(double) * op->hist_cap);
        op->hist = nullptr;
        op->hist_cap = 0;
        TCA_CUDA_TRY(dev_get((void **)&op->hist, sizeof(double) * (max_iters + 1)));
        op->hist_cap = max_iters + 1;
    }
    if ((pcg == 1 || pcg == 3) && op->scat)
        return fail(TCA_ERR_INVALID_ARG, pcg == 1 ? "tca_pcg_solve: no Kronecker-factor preconditioner for a scattered-data "
                                                    "operator"
                                                  : "tca_jacobi_solve: not available for a scattered-data operator");
    if (pcg == 3 && (op->nranks > 1 || op->transport))
        return fail(TCA_ERR_INVALID_ARG, "tca_jacobi_solve: not available on a sharded operator");
    if (pcg == 3 && rtol < 0.0) return fail(TCA_ERR_INVALID_ARG, "tca_jacobi_solve: threshold must be >= 0");
    if (pcg == 1) {
        if (op->nranks > 1)
            return fail(TCA_ERR_INVALID_ARG, "tca_pcg_solve: the mode-1 factor solve crosses shards (not available on a "
                                             "sharded operator)");
        TCA_TRY(precond_prepare(op, s));
    }
    if (op->dtype == TCA_F64)
        return cg_t<double>(op, (const double *)b, (double *)x, rtol, max_iters, rep, s, pcg, x0_zero);
    return cg_t<float>(op, (const float *)b, (float *)x, rtol, max_iters, rep, s, pcg, x0_zero);
}

tca_status tca_cg_solve(tca_operator *op, const void *b, void *x, int x0_zero, double rtol,
                        int32_t max_iters, tca_cg_report *rep, void *stream)
{
    return solve_common(op, b, x, rtol, max_iters, rep, stream, 0, x0_zero);
}

tca_status tca_pcg_solve(tca_operator *op, const void *b, void *x, int x0_zero, double rtol,
                        int32_t max_iters, tca_cg_report *rep, void *stream)
{
    return solve_common(op, b, x, rtol, max_iters, rep, stream, 1, x0_zero);
}

tca_status tca_jacobi_solve(tca_operator *op, const void *b, void *x, double threshold, int32_t max_iters,
                            tca_cg_report *rep, void *stream)
{
    return solve_common(op, b, x, threshold, max_iters, rep, stream, 3);
}

tca_status tca_cgsr_solve(tca_operator *op, const void *b, void *x, int x0_zero, double rtol,
                        int32_t max_iters, tca_cg_report *rep, void *stream)
{
    return solve_common(op, b, x, rtol, max_iters, rep, stream, 2, x0_zero);
}

tca_status tca_precond_apply(tca_operator *op, const void *r, void *z, void *stream)
{
    TCA_TRY(check_op(op));
    if (!r || !z) return fail(TCA_ERR_INVALID_ARG, "r and z must be non-NULL device pointers");
    if (op->nranks > 1 || op->scat)
        return fail(TCA_ERR_INVALID_ARG, "tca_precond_apply: not available on a sharded or scattered-data operator");
    cudaStream_t s = (cudaStream_t)stream;
    TCA_TRY(precond_prepare(op, s));
    if (op->dtype == TCA_F64) return apply_precond<double>(op, (const double *)r, (double *)z, nullptr, s);
    return apply_precond<float>(op, (const float *)r, (float *)z, nullptr, s);
}

tca_status tca_precond_info(tca_operator *op, double *eps, int *lower_bandwidth, void *stream)
{
    TCA_TRY(check_op(op));
    if (op->nranks > 1 || op->scat)
        return fail(TCA_ERR_INVALID_ARG, "tca_precond_info: not available on a sharded or scattered-data operator");
    TCA_TRY(precond_prepare(op, (cudaStream_t)stream));
    for (int d = 0; d < op->order; ++d) {
        if (eps) eps[d] = op->pc_eps[d];
        if (lower_bandwidth) lower_bandwidth[d] = op->pc_lbw[d];
    }
    return TCA_OK;
}

tca_status tca_solve_host(tca_operator *op, const void *ydata_host, void *x_host, double rtol,
                          int32_t max_iters, tca_cg_report *rep, void *stream)
{
    TCA_TRY(check_op(op));
    if (!ydata_host || !x_host) return fail(TCA_ERR_INVALID_ARG, "ydata_host and x_host must be non-NULL");
    cudaStream_t s = (cudaStream_t)stream;
    void *yd = nullptr, *bd = nullptr, *xd = nullptr;
    const size_t yb = (size_t)op->Mloc * op->esize, vb = (size_t)op->N * op->esize;
    TCA_CUDA_TRY(cudaMallocAsync(&yd, yb, s));
    TCA_CUDA_TRY(cudaMallocAsync(&bd, vb, s));
    TCA_CUDA_TRY(cudaMallocAsync(&xd, vb, s));
    TCA_CUDA_TRY(cudaMemcpyAsync(yd, ydata_host, yb, cudaMemcpyHostToDevice, s));
    tca_status st = tca_rhs(op, yd, bd, stream);
    if (st == TCA_OK || st == TCA_NOT_CONVERGED) {
        st = tca_cg_solve(op, bd, xd, 1, rtol, max_iters, rep, stream);
        cudaMemcpyAsync(x_host, xd, vb, cudaMemcpyDeviceToHost, s);
    }
    cudaFreeAsync(yd, s);
    cudaFreeAsync(bd, s);
    cudaFreeAsync(xd, s);
    TCA_CUDA_TRY(cudaStreamSynchronize(s));
    return st;
}

// Pipelined host-to-host solves: the H2D of item i+1 (copy stream) overlaps the
// rhs and CG of item i, the D2H of item i overlaps item i+1.  Two ydata
// buffers and two x staging buffers; one b and one x work buffer (the CG
// graphs stay cached on one x pointer).
tca_status tca_solve_host_batch(tca_operator *op, int count, const void *const *ydata_host, void *const *x_host,
                                double rtol, int32_t max_iters, tca_cg_report *reps, void *stream)
{
    TCA_TRY(check_op(op));
    if (count < 0) return fail(TCA_ERR_INVALID_ARG, "count must be >= 0");
    if (count > 0 && (!ydata_host || !x_host)) return fail(TCA_ERR_INVALID_ARG, "ydata_host and x_host arrays are NULL");
    for (int i = 0; i < count; ++i)
        if (!ydata_host[i] || !x_host[i]) return fail(TCA_ERR_INVALID_ARG, "ydata_host[i] and x_host[i] must be non-NULL");
    if (count == 0) return TCA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t yb = (size_t)op->Mloc * op->esize, vb = (size_t)op->N * op->esize;
    cudaStream_t cs = nullptr;
    void *yd[2] = {nullptr, nullptr}, *xs[2] = {nullptr, nullptr}, *bd = nullptr, *xd = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_rhs[2] = {}, ev_x[2] = {}, ev_d2h[2] = {};
    // st: the first error (CUDA or a solver error); a non-converged item only sets
    // any_nc, so later items still run and every x_host[i] is written
    tca_status st = TCA_OK;
    bool any_nc = false;
    auto cu = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess && st == TCA_OK) st = cuda_fail(e, what);
        return st == TCA_OK;
    };
    bool ok = cu(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream");
    for (int k = 0; k < 2 && ok; ++k) {
        ok = cu(cudaMallocAsync(&yd[k], yb, s), "ydata buffers") && cu(cudaMallocAsync(&xs[k], vb, s), "x staging");
        for (cudaEvent_t *e : {&ev_h2d[k], &ev_rhs[k], &ev_x[k], &ev_d2h[k]})
            if (ok) ok = cu(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "events");
    }
    if (ok) ok = cu(cudaMallocAsync(&bd, vb, s), "b") && cu(cudaMallocAsync(&xd, vb, s), "x");
    // the copy stream starts after the allocations (stream-ordered on s)
    if (ok) ok = cu(cudaEventRecord(ev_rhs[0], s), "event") && cu(cudaEventRecord(ev_rhs[1], s), "event") &&
                 cu(cudaEventRecord(ev_d2h[0], s), "event") && cu(cudaEventRecord(ev_d2h[1], s), "event");
    auto h2d = [&](int i) {
        const int k = i & 1;
        return cu(cudaStreamWaitEvent(cs, ev_rhs[k], 0), "wait") &&   // buffer k consumed by item i-2's rhs
               cu(cudaMemcpyAsync(yd[k], ydata_host[i], yb, cudaMemcpyHostToDevice, cs), "H2D ydata") &&
               cu(cudaEventRecord(ev_h2d[k], cs), "event");
    };
    if (ok) ok = h2d(0);
    for (int i = 0; i < count && ok; ++i) {
        const int k = i & 1;
        if (i + 1 < count && !(ok = h2d(i + 1))) break;
        if (!(ok = cu(cudaStreamWaitEvent(s, ev_h2d[k], 0), "wait"))) break;
        tca_status r = tca_rhs(op, yd[k], bd, stream);
        if (r != TCA_OK) { st = r; break; }
        if (!(ok = cu(cudaEventRecord(ev_rhs[k], s), "event"))) break;
        r = tca_cg_solve(op, bd, xd, 1, rtol, max_iters, reps ? &reps[i] : nullptr, stream);
        if (r == TCA_NOT_CONVERGED) any_nc = true;
        else if (r != TCA_OK) { st = r; break; }
        // x -> staging k (free once item i-2's D2H is done), D2H on the copy stream
        if (!(ok = cu(cudaStreamWaitEvent(s, ev_d2h[k], 0), "wait") &&
                   cu(cudaMemcpyAsync(xs[k], xd, vb, cudaMemcpyDeviceToDevice, s), "x staging copy") &&
                   cu(cudaEventRecord(ev_x[k], s), "event") && cu(cudaStreamWaitEvent(cs, ev_x[k], 0), "wait") &&
                   cu(cudaMemcpyAsync(x_host[i], xs[k], vb, cudaMemcpyDeviceToHost, cs), "D2H x") &&
                   cu(cudaEventRecord(ev_d2h[k], cs), "event")))
            break;
    }
    if (cs) {
        cudaError_t e = cudaStreamSynchronize(cs);
        if (e != cudaSuccess && st == TCA_OK) st = cuda_fail(e, "copy stream");
        cudaEventRecord(ev_h2d[0], cs);
        cudaStreamWaitEvent(s, ev_h2d[0], 0);
    }
    for (int k = 0; k < 2; ++k) {
        if (yd[k]) cudaFreeAsync(yd[k], s);
        if (xs[k]) cudaFreeAsync(xs[k], s);
    }
    if (bd) cudaFreeAsync(bd, s);
    if (xd) cudaFreeAsync(xd, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && st == TCA_OK) st = cuda_fail(e, "stream");
    for (int k = 0; k < 2; ++k)
        for (cudaEvent_t ev : {ev_h2d[k], ev_rhs[k], ev_x[k], ev_d2h[k]})
            if (ev) cudaEventDestroy(ev);
    if (cs) cudaStreamDestroy(cs);
    if (st == TCA_OK && any_nc) return TCA_NOT_CONVERGED;
    return st;
}

tca_status tca_generate_normal(void *out, tca_dtype dtype, int64_t count, int64_t offset,
                               uint64_t seed, uint32_t stream_id, double scale, void *stream)
{
    if (!out && count > 0) return fail(TCA_ERR_INVALID_ARG, "out is NULL");
    if (count < 0 || offset < 0) return fail(TCA_ERR_INVALID_ARG, "count and offset must be >= 0");
    if (dtype != TCA_F64 && dtype != TCA_F32) return fail(TCA_ERR_INVALID_ARG, "bad dtype");
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t key = stream_key(seed, stream_id);
    if (dtype == TCA_F64) launch_gen_normal<double>((double *)out, count, offset, key, scale, false, s);
    else launch_gen_normal<float>((float *)out, count, offset, key, scale, false, s);
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

tca_status tca_forward_model(const tca_operator *op, const void *x, void *ydata, double sigma,
                             uint64_t seed, void *stream)
{
    TCA_TRY(check_op(op));
    if (!ydata) return fail(TCA_ERR_INVALID_ARG, "ydata is NULL");
    if (op->scat) {   // y_k = <w_k, x> + sigma noise_k (x NULL: x_true of the seed)
        cudaStream_t s = (cudaStream_t)stream;
        void *xt = nullptr;
        if (!x) {
            TCA_CUDA_TRY(cudaMallocAsync(&xt, std::max<int64_t>(op->N, 1) * op->esize, s));
            if (op->dtype == TCA_F64) launch_gen_normal<double>((double *)xt, op->N, 0, stream_key(seed, 0), 1.0, false, s);
            else launch_gen_normal<float>((float *)xt, op->N, 0, stream_key(seed, 0), 1.0, false, s);
            x = xt;
        }
        TCA_CUDA_TRY(cudaMemsetAsync(ydata, 0, (size_t)op->sc_K * op->esize, s));
        TCA_TRY(launch_scatter(op, 2, x, ydata, nullptr, nullptr, s));
        if (sigma != 0.0) {
            if (op->dtype == TCA_F64)
                launch_gen_normal<double>((double *)ydata, op->sc_K, 0, stream_key(seed, 1), sigma, true, s);
            else
                launch_gen_normal<float>((float *)ydata, op->sc_K, 0, stream_key(seed, 1), sigma, true, s);
        }
        if (xt) TCA_CUDA_TRY(cudaFreeAsync(xt, s));
        TCA_CUDA_TRY(cudaGetLastError());
        return TCA_OK;
    }
    if (op->gram_form) return fail(TCA_ERR_INVALID_ARG, "tca_forward_model: operator was created from its factors");
    if (op->nranks > 1 && x) return fail(TCA_ERR_INVALID_ARG, "sharded forward model takes x = NULL");
    cudaStream_t s = (cudaStream_t)stream;
    if (op->dtype == TCA_F64) TCA_TRY(forward_t<double>(op, (const double *)x, (double *)ydata, sigma, seed, s));
    else TCA_TRY(forward_t<float>(op, (const float *)x, (float *)ydata, sigma, seed, s));
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

}  // extern "C"
