// tca_scatter.cu -- scattered-data normal operator (DESIGN.md
// reading Z27 and 6.6).  Sec. 4 of the paper: the system of
// a spline reconstruction from scattered measurements is a sum of rank-1
// (CANDECOMP) sample terms and is applied without storing the system or its
// decomposition:
//   data term  q += sum_k w_k <w_k, x>,   w_k = a_{k,1} (x) ... (x) a_{k,D},
//   rhs        b  = sum_k y_k w_k,        forward  y_k = <w_k, x>,
// a_{k,d}[i] = beta3(t_{k,d} - i), the centred cubic B-spline of reading Z5.
//
// B200 design: samples are bucketed once (host counting sort at create) by the
// tile of coefficient cells they fall in -- TB x TB x TB cells of modes 1-3, the
// whole of mode 4.  One CTA per non-empty tile stages the tile's coefficient
// footprint (TB+3 per tiled mode, n4+3 along mode 4, zero outside the domain)
// in shared memory, runs one sample per warp (each lane two of the 4x4x4
// (i1,i2,i3) support rows, 4 contiguous i4 taps each): gather <w_k, x> from
// shared memory, warp reduction, scatter-add into a shared accumulator (fp64
// shared-memory atomics), and adds the accumulator to HBM once per tile with
// global atomics (footprints of neighbouring tiles overlap by 3 cells).
// Orders D < 4 run as 4-mode problems with leading size-1 modes whose weight
// is 1 (not a B-spline).
#include <algorithm>
#include <cmath>
#include <vector>

#include "tca_internal.cuh"

namespace tca {

namespace {

constexpr int kScatThreads = 256;

__device__ __forceinline__ double beta3(double u)
{
    u = fabs(u);
    if (u < 1.0) return 2.0 / 3.0 - u * u + 0.5 * u * u * u;
    if (u < 2.0) {
        const double v = 2.0 - u;
        return v * v * v * (1.0 / 6.0);
    }
    return 0.0;
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// MODE 0: out += data term of x; 1: out += sum_k yk[perm] w_k (rhs); 2: out[perm[k]] = <w_k, x>
template <typename T, int MODE>
__global__ void __launch_bounds__(kScatThreads)
scatter_kernel(ScatGeom g, const double4 *__restrict__ ts, const int *__restrict__ perm,
               const int *__restrict__ tstart, const T *__restrict__ x, T *__restrict__ out,
               const T *__restrict__ yk, const int32_t *done)
{
    if (done && *done) return;
    const int tile = blockIdx.x;
    const int s0 = tstart[tile], s1 = tstart[tile + 1];
    if (s0 == s1) return;
    extern __shared__ __align__(16) unsigned char scat_smem[];
    T *xs = reinterpret_cast<T *>(scat_smem);
    const int FP = g.F[0] * g.F[1] * g.F[2] * g.F[3];
    T *qs = xs + (MODE == 1 ? 0 : FP);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tc2 = tile % g.nt[2], tc1 = (tile / g.nt[2]) % g.nt[1], tc0 = tile / (g.nt[2] * g.nt[1]);
    // footprint origin (coefficient index of footprint index 0) per mode
    const int lo[4] = {g.real[0] ? tc0 * g.TB - 1 : 0, g.real[1] ? tc1 * g.TB - 1 : 0,
                       g.real[2] ? tc2 * g.TB - 1 : 0, -1};
    const int64_t st3 = g.n[3], st2 = (int64_t)g.n[2] * st3, st1 = (int64_t)g.n[1] * st2;
    for (int f = tid; f < FP; f += kScatThreads) {
        const int f3 = f % g.F[3], f2 = (f / g.F[3]) % g.F[2], f1 = (f / (g.F[3] * g.F[2])) % g.F[1],
                  f0 = f / (g.F[3] * g.F[2] * g.F[1]);
        const int i0 = lo[0] + f0, i1 = lo[1] + f1, i2 = lo[2] + f2, i3 = lo[3] + f3;
        const bool in = i0 >= 0 && i0 < g.n[0] && i1 >= 0 && i1 < g.n[1] && i2 >= 0 && i2 < g.n[2] && i3 >= 0 &&
                        i3 < g.n[3];
        if (MODE != 1) xs[f] = in ? x[i0 * st1 + i1 * st2 + i2 * st3 + i3] : T(0);
        if (MODE != 2) qs[f] = T(0);
    }
    __syncthreads();
    // lane -> support rows (j0, j1, j2) and (j0 + 2, j1, j2) of the 4x4x4 rows;
    // absent modes use row 0 only (weight 1)
    const int ja = lane >> 4, jb = (lane >> 2) & 3, jc = lane & 3;
    for (int s = s0 + warp; s < s1; s += kScatThreads / 32) {
        const double4 tt = ts[s];
        const double tv[4] = {tt.x, tt.y, tt.z, tt.w};
        int fb[4];
        double wa, wb, w1, w2, w3[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int c = (int)floor(tv[d]);
            fb[d] = g.real[d] ? c - 1 - lo[d] : 0;   // footprint index of support row 0
        }
        {
            const double c0 = floor(tv[0]), c1 = floor(tv[1]), c2 = floor(tv[2]), c3 = floor(tv[3]);
            wa = g.real[0] ? beta3(tv[0] - (c0 - 1.0 + ja)) : (ja == 0 ? 1.0 : 0.0);
            wb = g.real[0] ? beta3(tv[0] - (c0 + 1.0 + ja)) : 0.0;
            w1 = g.real[1] ? beta3(tv[1] - (c1 - 1.0 + jb)) : (jb == 0 ? 1.0 : 0.0);
            w2 = g.real[2] ? beta3(tv[2] - (c2 - 1.0 + jc)) : (jc == 0 ? 1.0 : 0.0);
#pragma unroll
            for (int j = 0; j < 4; ++j) w3[j] = beta3(tv[3] - (c3 - 1.0 + j));
        }
        // footprint offsets of the lane's two rows (absent modes: row 0 only)
        const int r1 = g.real[1] ? jb : 0, r2 = g.real[2] ? jc : 0;
        const int ra = g.real[0] ? ja : 0, rb = g.real[0] ? ja + 2 : 0;
        const int base12 = ((fb[1] + r1) * g.F[2] + fb[2] + r2) * g.F[3] + fb[3];
        const int oa = (fb[0] + ra) * g.F[1] * g.F[2] * g.F[3] + base12;
        const int ob = (fb[0] + rb) * g.F[1] * g.F[2] * g.F[3] + base12;
        const double pa = wa * w1 * w2, pb = wb * w1 * w2;
        double coef;
        if (MODE != 1) {
            double sa = 0.0, sb = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sa = fma(w3[j], (double)xs[oa + j], sa);
                sb = fma(w3[j], (double)xs[ob + j], sb);
            }
            coef = warp_sum(fma(pa, sa, pb * sb));   // <w_k, x>
            if (MODE == 2) {
                if (lane == 0) out[perm[s]] = (T)coef;
                continue;
            }
        } else {
            coef = (double)yk[perm[s]];
        }
        const double ca = coef * pa, cb = coef * pb;
        if (ca != 0.0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicAdd(&qs[oa + j], (T)(ca * w3[j]));
        }
        if (cb != 0.0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicAdd(&qs[ob + j], (T)(cb * w3[j]));
        }
    }
    if (MODE == 2) return;
    __syncthreads();
    for (int f = tid; f < FP; f += kScatThreads) {
        const T v = qs[f];
        if (v == T(0)) continue;
        const int f3 = f % g.F[3], f2 = (f / g.F[3]) % g.F[2], f1 = (f / (g.F[3] * g.F[2])) % g.F[1],
                  f0 = f / (g.F[3] * g.F[2] * g.F[1]);
        const int i0 = lo[0] + f0, i1 = lo[1] + f1, i2 = lo[2] + f2, i3 = lo[3] + f3;
        if (i0 >= 0 && i0 < g.n[0] && i1 >= 0 && i1 < g.n[1] && i2 >= 0 && i2 < g.n[2] && i3 >= 0 && i3 < g.n[3])
            atomicAdd(&out[i0 * st1 + i1 * st2 + i2 * st3 + i3], v);
    }
}

template <typename T, int MODE>
tca_status launch_mode(const tca_operator *op, const void *x, void *out, const void *yk, const int32_t *done,
                       cudaStream_t s)
{
    const ScatGeom &g = op->sg;
    const size_t fp = (size_t)g.F[0] * g.F[1] * g.F[2] * g.F[3];
    const size_t smem = fp * sizeof(T) * (MODE == 0 ? 2 : 1);
    static size_t attr = 0;
    if (smem > attr) {
        TCA_CUDA_TRY(cudaFuncSetAttribute(scatter_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        attr = smem;
    }
    count_launch();
    scatter_kernel<T, MODE><<<(unsigned)op->sc_ntiles, kScatThreads, smem, s>>>(
        g, (const double4 *)op->sc_t, (const int *)op->sc_perm, (const int *)op->sc_tstart, (const T *)x, (T *)out,
        (const T *)yk, done);
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

}  // namespace

// Bucket the samples by tile (counting sort) and upload them.  t: K x order
// host coordinates, each in [0, n_d - 1].
tca_status scatter_prepare(tca_operator *op, int64_t K, const double *t, cudaStream_t s)
{
    const int D = op->order;
    ScatGeom g{};
    for (int d = 0; d < 4; ++d) {
        const int e = d - (4 - D);   // internal mode d = user mode e (leading modes padded)
        g.n[d] = e >= 0 ? (int)op->n[e] : 1;
        g.real[d] = e >= 0 ? 1 : 0;
    }
    // tile: TB cells of the real modes among 1-3; the footprint pair (xs, qs)
    // fits two CTAs per SM when it can, one otherwise
    const size_t es = op->esize;
    int TB = 0;
    for (int cap : {113 * 1024, 227 * 1024}) {
        for (int tb : {4, 2, 1}) {
            size_t fp = (size_t)(g.n[3] + 3);
            for (int d = 0; d < 3; ++d) fp *= g.real[d] ? (size_t)(tb + 3) : 1;
            if (fp * es * 2 <= (size_t)cap) { TB = tb; break; }
        }
        if (TB) break;
    }
    if (!TB) return fail(TCA_ERR_SHAPE, "scattered operator: the last mode is too long for a shared-memory tile");
    g.TB = TB;
    int64_t ntiles = 1;
    for (int d = 0; d < 3; ++d) {
        g.nt[d] = g.real[d] ? (g.n[d] + TB - 1) / TB : 1;
        g.F[d] = g.real[d] ? TB + 3 : 1;
        ntiles *= g.nt[d];
    }
    g.F[3] = g.n[3] + 3;
    if (ntiles >= (1ll << 31) || K >= (1ll << 31)) return fail(TCA_ERR_SHAPE, "scattered operator: too many samples");
    std::vector<int> tileof((size_t)K), cnt((size_t)ntiles + 1, 0);
    for (int64_t k = 0; k < K; ++k) {
        int64_t id = 0;
        for (int d = 0; d < 3; ++d) {
            const int e = d - (4 - D);
            const int c = e >= 0 ? (int)std::floor(t[k * D + e]) : 0;
            id = id * g.nt[d] + (g.real[d] ? std::min(c, g.n[d] - 1) / TB : 0);
        }
        tileof[(size_t)k] = (int)id;
        ++cnt[(size_t)id + 1];
    }
    for (int64_t i = 0; i < ntiles; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
    std::vector<double> ts((size_t)K * 4);
    std::vector<int> perm((size_t)K);
    {
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t k = 0; k < K; ++k) {
            const int p = pos[(size_t)tileof[(size_t)k]]++;
            perm[(size_t)p] = (int)k;
            for (int d = 0; d < 4; ++d) {
                const int e = d - (4 - D);
                ts[(size_t)p * 4 + d] = e >= 0 ? t[k * D + e] : 0.0;
            }
        }
    }
    op->sg = g;
    op->sc_K = K;
    op->sc_ntiles = (int)ntiles;
    const size_t bt = std::max<size_t>(ts.size(), 4) * sizeof(double), bp = std::max<size_t>(perm.size(), 1) * sizeof(int),
                 bs = cnt.size() * sizeof(int);
    TCA_CUDA_TRY(cudaMallocAsync(&op->sc_t, bt, s));
    TCA_CUDA_TRY(cudaMallocAsync(&op->sc_perm, bp, s));
    TCA_CUDA_TRY(cudaMallocAsync(&op->sc_tstart, bs, s));
    if (K > 0) {
        TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_t, ts.data(), ts.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_perm, perm.data(), perm.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    }
    TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_tstart, cnt.data(), bs, cudaMemcpyHostToDevice, s));
    TCA_CUDA_TRY(cudaStreamSynchronize(s));   // host vectors go out of scope
    op->device_bytes += bt + bp + bs;
    return TCA_OK;
}

// mode 0: y += data term of x; 1: y += W^T yk (y zeroed by the caller); 2: yk_out = W x
tca_status launch_scatter(const tca_operator *op, int mode, const void *x, void *out, const void *yk,
                          const int32_t *done, cudaStream_t s)
{
    if (op->sc_K == 0) return TCA_OK;
    if (op->dtype == TCA_F64) {
        if (mode == 0) return launch_mode<double, 0>(op, x, out, yk, done, s);
        if (mode == 1) return launch_mode<double, 1>(op, x, out, yk, done, s);
        return launch_mode<double, 2>(op, x, out, yk, done, s);
    }
    if (mode == 0) return launch_mode<float, 0>(op, x, out, yk, done, s);
    if (mode == 1) return launch_mode<float, 1>(op, x, out, yk, done, s);
    return launch_mode<float, 2>(op, x, out, yk, done, s);
}

}  // namespace tca
