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
// in shared memory, runs one sample per thread (its 4 x 4 B-spline weights in
// registers): gather <w_k, x> from shared memory, scatter-add into a shared
// accumulator (fp64 shared-memory atomics), and adds the accumulator to HBM
// once per tile with global atomics (footprints of neighbouring tiles overlap
// by 3 cells).
// Orders D < 4 run as 4-mode problems with leading size-1 modes whose weight
// is 1 (not a B-spline).
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "tca_internal.cuh"

namespace tca {

namespace {

constexpr int kScatThreads = 256;

// MODE 0: out += data term of x; 1: out += sum_k yk[perm] w_k (rhs); 2: out[perm[k]] = <w_k, x>
// FULL: all four modes are B-spline modes (order 4): compile-time support loops
template <typename T, int MODE, bool FULL>
__global__ void __launch_bounds__(kScatThreads)
scatter_kernel(ScatGeom g, const double4 *__restrict__ ts, const int *__restrict__ perm,
               const int *__restrict__ tstart, const T *__restrict__ x, T *__restrict__ out,
               const T *__restrict__ yk, const int32_t *done, double *__restrict__ coefg)
{
#define RL(d) (FULL || g.real[d])
    if (done && *done) return;
    const int tile = blockIdx.x;
    const int s0 = tstart[tile], s1 = tstart[tile + 1];
    if (s0 == s1) return;
    extern __shared__ __align__(16) unsigned char scat_smem[];
    T *xs = reinterpret_cast<T *>(scat_smem);
    const int FP = g.F[0] * g.F[1] * g.F[2] * g.F[3];
    T *qs = xs;   // one footprint buffer: x for the gather, then the accumulator
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tc2 = tile % g.nt[2], tc1 = (tile / g.nt[2]) % g.nt[1], tc0 = tile / (g.nt[2] * g.nt[1]);
    // footprint origin (coefficient index of footprint index 0) per mode
    const int lo[4] = {RL(0) ? tc0 * g.TB - 1 : 0, RL(1) ? tc1 * g.TB - 1 : 0,
                       RL(2) ? tc2 * g.TB - 1 : 0, -1};
    const int64_t st3 = g.n[3], st2 = (int64_t)g.n[2] * st3, st1 = (int64_t)g.n[1] * st2;
    // footprint rows (f0, f1, f2) one warp each, lanes along mode 4 (no divisions per element)
    const int N12 = g.F[1] * g.F[2];
    for (int r12 = warp; r12 < N12; r12 += kScatThreads / 32) {   // one division pair per (f1, f2)
        const int f1 = r12 / g.F[2], f2 = r12 - f1 * g.F[2];
        const int i1 = lo[1] + f1, i2 = lo[2] + f2;
        const bool in12 = i1 >= 0 && i1 < g.n[1] && i2 >= 0 && i2 < g.n[2];
        for (int f0 = 0; f0 < g.F[0]; ++f0) {
            const int i0 = lo[0] + f0, row = f0 * N12 + r12;
            const bool rin = in12 && i0 >= 0 && i0 < g.n[0];
            const T *xr = x + (rin ? i0 * st1 + i1 * st2 + i2 * st3 : 0);
            for (int f3 = lane; f3 < g.F[3]; f3 += 32) {
                const int i3 = f3 - 1;
                if (MODE != 1) xs[row * g.F[3] + f3] = (rin && i3 >= 0 && i3 < g.n[3]) ? xr[i3] : T(0);
                if (MODE == 1) qs[row * g.F[3] + f3] = T(0);
            }
        }
    }
    __syncthreads();
    // Samples in chunks of kScatThreads: (1) gather, one sample per thread (its
    // 4 x 4 B-spline weights in registers, the 4^D support read from shared
    // memory) -> coefficient in shared memory; (2) scatter, one sample per warp,
    // each lane two of the 4x4x4 (i1,i2,i3) support rows x 4 i4 taps, so a
    // warp's 32 shared-memory atomics of one instruction never collide.
    const int J0 = RL(0) ? 4 : 1, J1 = RL(1) ? 4 : 1, J2 = RL(2) ? 4 : 1;
    const int S2 = g.F[3], S1 = g.F[2] * S2, S0 = g.F[1] * S1;
    double *coefs = coefg;   // per sorted sample (apply); rhs reads yk directly
    const int ja = lane >> 4, jb = (lane >> 2) & 3, jc = lane & 3;
    for (int c0s = s0; c0s < s1; c0s += kScatThreads) {
        const int cn = min(kScatThreads, s1 - c0s);
        if (MODE != 1 && tid < cn) {   // <w_k, x>
            const int s = c0s + tid;
            const double4 tt = ts[s];
            const double tv[4] = {tt.x, tt.y, tt.z, tt.w};
            double w[4][4];
            int o = 0;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const double c = floor(tv[d]);
                if (RL(d)) {
                    // cubic B-spline blending functions of u = t - floor(t):
                    // beta3(u+1), beta3(u), beta3(1-u), beta3(2-u) (rows c-1 .. c+2)
                    const double u = tv[d] - c, u2 = u * u, u3 = u2 * u, v = 1.0 - u;
                    w[d][0] = v * v * v * (1.0 / 6.0);
                    w[d][1] = fma(0.5, u3, 2.0 / 3.0 - u2);
                    w[d][2] = fma(-0.5, u3, fma(0.5, u2, fma(0.5, u, 1.0 / 6.0)));
                    w[d][3] = u3 * (1.0 / 6.0);
                } else {
                    w[d][0] = 1.0;
                    w[d][1] = w[d][2] = w[d][3] = 0.0;
                }
                const int fbd = RL(d) ? (int)c - 1 - lo[d] : 0;   // footprint index of support row 0
                o += fbd * (d == 0 ? S0 : d == 1 ? S1 : d == 2 ? S2 : 1);
            }
            double acc = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < 4; ++j0) {
                if (j0 >= J0) break;
#pragma unroll
                for (int j1 = 0; j1 < 4; ++j1) {
                    if (j1 >= J1) break;
                    const double p01 = w[0][j0] * w[1][j1];
#pragma unroll
                    for (int j2 = 0; j2 < 4; ++j2) {
                        if (j2 >= J2) break;
                        const T *xr = xs + o + j0 * S0 + j1 * S1 + j2 * S2;
                        double r = 0.0;
#pragma unroll
                        for (int j3 = 0; j3 < 4; ++j3) r = fma(w[3][j3], (double)xr[j3], r);
                        acc = fma(p01 * w[2][j2], r, acc);
                    }
                }
            }
            if (MODE == 2) out[perm[s]] = (T)acc;
            else coefs[s] = acc;
        }
    }
    if (MODE == 2) return;
    if (MODE == 0) {   // the footprint buffer becomes the accumulator
        __syncthreads();
        for (int f = tid; f < FP; f += kScatThreads) qs[f] = T(0);
        __syncthreads();
    }
    for (int c0s = s0; c0s < s1; c0s += kScatThreads) {
        const int cn = min(kScatThreads, s1 - c0s);
        for (int i = warp; i < cn; i += kScatThreads / 32) {
            const double coef = MODE == 0 ? coefs[c0s + i] : (double)yk[perm[c0s + i]];
            if (coef == 0.0) continue;
            const double4 tt = ts[c0s + i];
            const double tv[4] = {tt.x, tt.y, tt.z, tt.w};
            int fb[4];
            double wsel[3][2], w3[4];
            const int jsel[3][2] = {{ja, ja + 2}, {jb, jb}, {jc, jc}};
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const double c = floor(tv[d]);
                fb[d] = RL(d) ? (int)c - 1 - lo[d] : 0;
                const double u = tv[d] - c, u2 = u * u, u3 = u2 * u, v = 1.0 - u;
                const double bl[4] = {v * v * v * (1.0 / 6.0), fma(0.5, u3, 2.0 / 3.0 - u2),
                                      fma(-0.5, u3, fma(0.5, u2, fma(0.5, u, 1.0 / 6.0))), u3 * (1.0 / 6.0)};
                if (d == 3) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) w3[j] = bl[j];
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = jsel[d][h];
                        // select without local-memory indexing
                        const double bj = j == 0 ? bl[0] : j == 1 ? bl[1] : j == 2 ? bl[2] : bl[3];
                        wsel[d][h] = RL(d) ? bj : (j == 0 ? 1.0 : 0.0);
                    }
                }
            }
            const int r1 = RL(1) ? jb : 0, r2 = RL(2) ? jc : 0;
            const int ra = RL(0) ? ja : 0, rb = RL(0) ? ja + 2 : 0;
            const int base12 = (fb[1] + r1) * S1 + (fb[2] + r2) * S2 + fb[3];
            const double p12 = coef * wsel[1][0] * wsel[2][0];
            const double ca = p12 * wsel[0][0], cb = RL(0) ? p12 * wsel[0][1] : 0.0;
            if (ca != 0.0) {
                T *qa = qs + (fb[0] + ra) * S0 + base12;
#pragma unroll
                for (int j = 0; j < 4; ++j) atomicAdd(&qa[j], (T)(ca * w3[j]));
            }
            if (cb != 0.0) {
                T *qb = qs + (fb[0] + rb) * S0 + base12;
#pragma unroll
                for (int j = 0; j < 4; ++j) atomicAdd(&qb[j], (T)(cb * w3[j]));
            }
        }
    }
    if (MODE == 2) return;
    __syncthreads();
    for (int r12 = warp; r12 < N12; r12 += kScatThreads / 32) {
        const int f1 = r12 / g.F[2], f2 = r12 - f1 * g.F[2];
        const int i1 = lo[1] + f1, i2 = lo[2] + f2;
        if (!(i1 >= 0 && i1 < g.n[1] && i2 >= 0 && i2 < g.n[2])) continue;
        for (int f0 = 0; f0 < g.F[0]; ++f0) {
            const int i0 = lo[0] + f0, row = f0 * N12 + r12;
            if (i0 < 0 || i0 >= g.n[0]) continue;
            T *orow = out + i0 * st1 + i1 * st2 + i2 * st3;
            for (int f3 = lane; f3 < g.F[3]; f3 += 32) {
                const int i3 = f3 - 1;
                const T v = qs[row * g.F[3] + f3];
                if (v != T(0) && i3 >= 0 && i3 < g.n[3]) atomicAdd(&orow[i3], v);
            }
        }
    }
#undef RL
}

template <typename T, int MODE>
tca_status launch_mode(const tca_operator *op, const void *x, void *out, const void *yk, const int32_t *done,
                       cudaStream_t s)
{
    const ScatGeom &g = op->sg;
    const size_t fp = (size_t)g.F[0] * g.F[1] * g.F[2] * g.F[3];
    const size_t smem = fp * sizeof(T);
    const bool full = op->order == 4;
    TCA_TRY(set_max_dynamic_smem(full ? (const void *)scatter_kernel<T, MODE, true>
                                      : (const void *)scatter_kernel<T, MODE, false>, smem));
    count_launch();
    (full ? scatter_kernel<T, MODE, true> : scatter_kernel<T, MODE, false>)<<<(unsigned)op->sc_ntiles, kScatThreads, smem, s>>>(
        g, (const double4 *)op->sc_t, (const int *)op->sc_perm, (const int *)op->sc_tstart, (const T *)x, (T *)out,
        (const T *)yk, done, (double *)op->sc_coef);
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
    // tile: TB cells of the real modes among 1-3; the kernel's one footprint
    // buffer fits two CTAs per SM (113 KB each) when it can, one (227 KB) otherwise
    const size_t es = op->esize;
    int TB = 0;
    for (int cap : {113 * 1024, 227 * 1024}) {
        for (int tb : {4, 2, 1}) {
            size_t fp = (size_t)(g.n[3] + 3);
            for (int d = 0; d < 3; ++d) fp *= g.real[d] ? (size_t)(tb + 3) : 1;
            if (fp * es <= (size_t)cap) { TB = tb; break; }
        }
        if (TB) break;
    }
    if (!TB) return fail(TCA_ERR_SHAPE, "scattered operator: the last mode is too long for a shared-memory tile");
    if (const char *e = getenv("TCA_SCAT_TB")) {   // measurement switch: force the tile width
        const int tb = atoi(e);
        size_t fp = (size_t)(g.n[3] + 3);
        for (int d = 0; d < 3; ++d) fp *= g.real[d] ? (size_t)(tb + 3) : 1;
        if (tb >= 1 && fp * es <= 227 * 1024) TB = tb;
    }
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
    TCA_CUDA_TRY(cudaMallocAsync(&op->sc_coef, std::max<size_t>(perm.size(), 1) * sizeof(double), s));
    if (K > 0) {
        TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_t, ts.data(), ts.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_perm, perm.data(), perm.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    }
    TCA_CUDA_TRY(cudaMemcpyAsync(op->sc_tstart, cnt.data(), bs, cudaMemcpyHostToDevice, s));
    TCA_CUDA_TRY(cudaStreamSynchronize(s));   // host vectors go out of scope
    op->device_bytes += bt + bp + bs + std::max<size_t>(perm.size(), 1) * sizeof(double);   // + sc_coef
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
