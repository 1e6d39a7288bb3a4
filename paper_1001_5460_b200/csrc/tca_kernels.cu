// tca_kernels.cu -- generic (correctness-rung) kernels of libtca:
//   * compressed-band mode-d product (any band width, rectangular or dense),
//     the one-dimensional transformation of Eq. 4;
//   * CG vector updates and dot-product partials (Fig. 2, PAPER.md:193-221;
//     inner product Eq. A13; elementwise ops A.4,
//     PAPER.md:441-452) with device-resident fp64 scalars;
//   * the seeded counter-based normal generator (reading Z9).
// Reductions are deterministic: a fixed grid writes per-block partials that
// one block sums in a fixed order (no floating-point atomics).
#include <math.h>

#include <algorithm>

#include "tca_internal.cuh"
#include "tca_finalize.cuh"

namespace tca {

std::atomic<int64_t> g_launches{0};

// L2 hand-off between the CG vector kernels (default; TCA_L2REV=0 measures the
// plain streaming form): cg_update_r sweeps the vector from its end (the
// apply's last output slabs, high i1, are the ones still in L2) and keeps R
// L2-normal (Q evict-first), so the R it wrote last (low indices) is still in
// L2 when cg_update_xp sweeps from the start and reads it L2-normal.
// Config 3 CG: f64 597.9 -> 592.3 us, f32 369.4 -> 362.2 us per iteration
// (profiles/r02_l2_handoff_probe.txt); with 4 vectors in flight per thread in
// the reverse sweep f64 577.4 -> 569.1 us, f32 361.4 -> 356.9 us
// (profiles/r02_unroll_probe.txt).  The <r, r> partials are summed in the
// sweep's (fixed) order: deterministic.
static int l2_handoff()
{
    static const int on = [] {
        const char *e = getenv("TCA_L2REV");
        return e && e[0] == '0' ? 0 : 1;
    }();
    return on;
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum for blockDim.x == kRedThreads; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v)
{
    __shared__ double sm[kRedThreads / 32];
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sm[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < kRedThreads / 32; ++i) s += sm[i];
    }
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------- band mode product
// Y[o, r, t] = alpha * sum_w taps[r, w] X[o, start[r] + w, t]  (+ Y[o, r, t]).
// One CTA row of the grid per outer index o (grid.y, strided); threads cover
// the (r, t) plane of that slice linearly with t fastest (coalesced loads of
// every tap row), 32-bit index math within the slice.
template <typename T>
__global__ void __launch_bounds__(256)
band_mode_product_kernel(const T *__restrict__ X, T *__restrict__ Y, int64_t outer,
                         int rows, int cols, int inner,
                         const int *__restrict__ start, const T *__restrict__ taps,
                         int W, T alpha, int accumulate, const int32_t *done)
{
    if (done && *done) return;
    const unsigned plane = (unsigned)rows * (unsigned)inner;
    for (int64_t o = blockIdx.y; o < outer; o += gridDim.y) {
        const T *xo = X + o * (int64_t)cols * inner;
        T *yo = Y + o * (int64_t)plane;
        for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < plane; idx += gridDim.x * blockDim.x) {
            const unsigned r = idx / (unsigned)inner;
            const unsigned t = idx - r * (unsigned)inner;
            const int s0 = __ldg(start + r);
            const T *xp = xo + t;
            const T *tp = taps + (int64_t)r * W;
            T acc = T(0);
            for (int w = 0; w < W; ++w) {
                const int c = s0 + w;
                if (c >= 0 && c < cols) acc = fma(__ldg(tp + w), __ldg(xp + (int64_t)c * inner), acc);
            }
            acc *= alpha;
            if (accumulate) acc += yo[idx];
            yo[idx] = acc;
        }
    }
}

// Window-staged form for fibres of >= 32 elements and rows of <= 16 taps: a
// block of 128 threads owns kRB = 16 consecutive output rows x kCB = 128
// consecutive (o, t) positions (flattened, t fastest: coalesced rows when
// inner >= 128, inner-long segments otherwise).  It stages the union of the
// rows' input windows (BandMat::win16 <= kKWIN rows; rows outside [0, cols)
// zero-filled) in shared memory with asynchronous copies (LDGSTS, the whole
// window in flight), so each input element is read ~window / 16 times instead
// of W times (config 3's rhs modes 1 and 2: 38 staged rows for 16 output rows
// of 8 taps).  Warp w then owns rows w, w + 4, w + 8, w + 12: their W taps sit
// in registers and each output costs W shared loads + W FMAs.  Small blocks
// (39 KB of window in fp64) keep several per SM so one block's loads overlap
// another's arithmetic.
constexpr int kRB = 16, kCB = 128, kKWIN = 48;

template <typename T, int WC>
__global__ void __launch_bounds__(kCB)
band_mode_product_win_kernel(const T *__restrict__ X, T *__restrict__ Y, int64_t total, int rows, int cols,
                             int64_t inner, const int *__restrict__ start, const T *__restrict__ taps, T alpha,
                             int accumulate, const int32_t *done)
{
    if (done && *done) return;
    extern __shared__ __align__(16) unsigned char win_raw[];
    T *sm = reinterpret_cast<T *>(win_raw);
    constexpr int NW = kCB / 32, RPW = kRB / NW;   // warps, rows per warp
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = blockIdx.x * kRB;   // row groups fastest: neighbours share window rows in L2
    const int nr = min(kRB, rows - r0);
    int base = __ldg(start + r0), top = base;
    for (int k = 1; k < nr; ++k) {
        const int sr = __ldg(start + r0 + k);
        base = min(base, sr);
        top = max(top, sr);
    }
    top += WC;   // window rows [base, top), <= kKWIN (host-checked win16)
    T tp[RPW][WC];
    int off[RPW];
#pragma unroll
    for (int h = 0; h < RPW; ++h) {
        const int k = warp + NW * h;
        const bool ok = k < nr;
        off[h] = ok ? __ldg(start + r0 + k) - base : 0;
#pragma unroll
        for (int w = 0; w < WC; ++w) tp[h][w] = ok ? __ldg(taps + (int64_t)(r0 + k) * WC + w) : T(0);
    }
    const bool aligned = inner % kCB == 0;   // a chunk never straddles two outer indices
    const int cv0 = max(base, 0), cv1 = min(top, cols);
    for (int64_t f0 = (int64_t)blockIdx.y * kCB; f0 < total; f0 += (int64_t)gridDim.y * kCB) {
        const int64_t oc = aligned ? f0 / inner : 0;   // the chunk's outer index (aligned case)
        {   // stage column f0 + tid of the window
            const int64_t f = f0 + threadIdx.x;
            const bool live = f < total;
            int64_t o, t;
            if (aligned) { o = oc; t = f - oc * inner; }
            else { o = live ? f / inner : 0; t = live ? f - o * inner : 0; }
            __syncthreads();   // previous chunk's reads of sm are done
            T *row = sm + threadIdx.x;
            for (int c = base; c < cv0; ++c) row[(c - base) * kCB] = T(0);           // rows before column 0
            for (int c = max(cv1, base); c < top; ++c) row[(c - base) * kCB] = T(0); // rows past the last column
            if (live) {
                const T *src = X + o * (int64_t)cols * inner + t + (int64_t)cv0 * inner;
                unsigned dst = (unsigned)__cvta_generic_to_shared(row + (cv0 - base) * kCB);
                for (int c = cv0; c < cv1; ++c, src += inner, dst += kCB * sizeof(T)) {
                    if (sizeof(T) == 8)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
                }
            } else {
                for (int c = cv0; c < cv1; ++c) row[(c - base) * kCB] = T(0);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            __syncthreads();
        }
        constexpr int NI = kCB / 32;
        int64_t yb[NI];
        bool lv[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int64_t f = f0 + i * 32 + lane;
            lv[i] = f < total;
            if (aligned) {
                yb[i] = oc * (int64_t)rows * inner + (f - oc * inner);
            } else {
                const int64_t o = lv[i] ? f / inner : 0;
                yb[i] = o * (int64_t)rows * inner + (f - o * inner);
            }
        }
#pragma unroll
        for (int h = 0; h < RPW; ++h) {
            const int k = warp + NW * h;
            if (k >= nr) break;
            const T *sp = sm + off[h] * kCB + lane;
            T *yr = Y + (int64_t)(r0 + k) * inner;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                T acc = T(0);
#pragma unroll
                for (int w = 0; w < WC; ++w) acc = fma(tp[h][w], sp[w * kCB + i * 32], acc);
                if (lv[i]) {
                    acc *= alpha;
                    if (accumulate) acc += yr[yb[i]];
                    yr[yb[i]] = acc;
                }
            }
        }
    }
}

template <typename T, int WC>
static void launch_win(const T *X, T *Y, int64_t outer, const BandMat &M, int64_t inner, double alpha,
                       bool accumulate, const int32_t *done, cudaStream_t s)
{
    const int64_t total = outer * inner;
    const int64_t bx = (M.rows + kRB - 1) / kRB;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // ~16 resident blocks per SM over all row groups, each looping over chunks
    const int64_t by = std::max<int64_t>(1, std::min<int64_t>((total + kCB - 1) / kCB,
                                                              std::max<int64_t>(1, (int64_t)sms * 16 / bx)));
    const size_t smem = (size_t)M.win16 * kCB * sizeof(T);
    set_max_dynamic_smem((const void *)band_mode_product_win_kernel<T, WC>, smem);
    band_mode_product_win_kernel<T, WC><<<dim3((unsigned)bx, (unsigned)by), kCB, smem, s>>>(
        X, Y, total, M.rows, M.cols, inner, M.start, (const T *)M.taps, (T)alpha, accumulate ? 1 : 0, done);
}

// Mode 1 (the slowest) and the last mode L (contiguous fibres of c4 elements)
// in one pass, for the first product of a chain: X is (cols, K c4), Y is
// (rows, K r4).  The window kernel's staging and mode-1 arithmetic on chunks of
// FPC = kCB / c4 whole mode-L fibres; the 16 x FPC c4 mode-1 results go to
// shared memory and are contracted along mode L (M4: r4 x c4 band rows) before
// the store, so the pass writes the tensor with mode L already contracted
// (config 3's rhs: 4.0 GB in, 1.0 GB out instead of 2.0 GB).
template <typename T, int WC>
__global__ void __launch_bounds__(kCB)
band_win_last_kernel(const T *__restrict__ X, T *__restrict__ Y, int64_t K, int rows, int cols, int c4, int r4,
                     const int *__restrict__ start, const T *__restrict__ taps, const int *__restrict__ s4,
                     const T *__restrict__ t4, int w4)
{
    extern __shared__ __align__(16) unsigned char win_raw[];
    T *sm = reinterpret_cast<T *>(win_raw);
    constexpr int NW = kCB / 32, RPW = kRB / NW, NI = kCB / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int FPC = kCB / c4, CW = FPC * c4;           // whole fibres per chunk, chunk width
    const int64_t inner = K * c4, inner_o = K * r4;
    const int r0 = blockIdx.x * kRB;
    const int nr = min(kRB, rows - r0);
    int base = __ldg(start + r0), top = base;
    for (int k = 1; k < nr; ++k) {
        const int sr = __ldg(start + r0 + k);
        base = min(base, sr);
        top = max(top, sr);
    }
    top += WC;
    T tp[RPW][WC];
    int off[RPW];
#pragma unroll
    for (int h = 0; h < RPW; ++h) {
        const int k = warp + NW * h;
        const bool ok = k < nr;
        off[h] = ok ? __ldg(start + r0 + k) - base : 0;
#pragma unroll
        for (int w = 0; w < WC; ++w) tp[h][w] = ok ? __ldg(taps + (int64_t)(r0 + k) * WC + w) : T(0);
    }
    const int cv0 = max(base, 0), cv1 = min(top, cols);
    const int up = CW | 1;   // pitch of the mode-1 results in shared memory
    for (int64_t ch = blockIdx.y; ch * FPC < K; ch += gridDim.y) {
        const int64_t f0 = ch * CW;                      // first column of the chunk
        const int fib = (int)min((int64_t)FPC, K - ch * FPC);
        const int cw = fib * c4;
        {   // stage column tid of the window
            __syncthreads();
            T *row = sm + threadIdx.x;
            const bool live = threadIdx.x < cw;
            for (int c = base; c < cv0; ++c) row[(c - base) * kCB] = T(0);
            for (int c = max(cv1, base); c < top; ++c) row[(c - base) * kCB] = T(0);
            if (live) {
                const T *src = X + f0 + threadIdx.x + (int64_t)cv0 * inner;
                unsigned dst = (unsigned)__cvta_generic_to_shared(row + (cv0 - base) * kCB);
                for (int c = cv0; c < cv1; ++c, src += inner, dst += kCB * sizeof(T)) {
                    if (sizeof(T) == 8)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
                }
            } else {
                for (int c = cv0; c < cv1; ++c) row[(c - base) * kCB] = T(0);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            __syncthreads();
        }
        T u[RPW][NI];
#pragma unroll
        for (int h = 0; h < RPW; ++h) {
            const T *sp = sm + off[h] * kCB + lane;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                T acc = T(0);
#pragma unroll
                for (int w = 0; w < WC; ++w) acc = fma(tp[h][w], sp[w * kCB + i * 32], acc);
                u[h][i] = acc;
            }
        }
        __syncthreads();   // window reads done: the buffer takes the mode-1 results
#pragma unroll
        for (int h = 0; h < RPW; ++h) {
            const int k = warp + NW * h;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int c = i * 32 + lane;
                if (k < nr && c < CW) sm[k * up + c] = u[h][i];
            }
        }
        __syncthreads();
        // mode L: Y[r0 + k, (ch FPC + f) r4 + j] = sum_w t4[j, w] U[k, f c4 + s4[j] + w];
        // thread (half, t): output column t = (f, j) of rows half*8 .. half*8+7,
        // the row's taps (clipped to the fibre) in registers
        const int per = fib * r4;
        const int half = threadIdx.x >> 6;
        for (int t = threadIdx.x & 63; t < per; t += 64) {
            const int f = t / r4, j = t - f * r4;
            const int sj = __ldg(s4 + j);
            const int wlo = max(0, -sj), whi = min(w4, c4 - sj);
            T tw[16];
#pragma unroll
            for (int w = 0; w < 16; ++w) tw[w] = (w >= wlo && w < whi) ? __ldg(t4 + j * w4 + w) : T(0);
            const T *ub = sm + f * c4 + sj;
            for (int k = half * (kRB / 2); k < min(nr, (half + 1) * (kRB / 2)); ++k) {
                const T *ur = ub + k * up;
                T acc = T(0);
#pragma unroll
                for (int w = 0; w < 16; ++w)
                    if (w >= wlo && w < whi) acc = fma(tw[w], ur[w], acc);
                Y[(int64_t)(r0 + k) * inner_o + (ch * FPC + f) * r4 + j] = acc;
            }
        }
    }
}

template <typename T, int WC>
static void launch_win_last_w(const T *X, T *Y, int64_t K, int c4, const BandMat &M1, const BandMat &M4,
                              cudaStream_t s)
{
    const int64_t bx = (M1.rows + kRB - 1) / kRB;
    const int FPC = kCB / c4;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t chunks = (K + FPC - 1) / FPC;
    const int64_t by = std::max<int64_t>(1, std::min<int64_t>(chunks, std::max<int64_t>(1, (int64_t)sms * 16 / bx)));
    const size_t smem = std::max<size_t>((size_t)M1.win16 * kCB, (size_t)kRB * ((FPC * c4) | 1)) * sizeof(T);
    set_max_dynamic_smem((const void *)band_win_last_kernel<T, WC>, smem);
    band_win_last_kernel<T, WC><<<dim3((unsigned)bx, (unsigned)by), kCB, smem, s>>>(
        X, Y, K, M1.rows, M1.cols, c4, M4.rows, M1.start, (const T *)M1.taps, M4.start, (const T *)M4.taps, M4.W);
}

template <typename T>
bool launch_band_win_last(const T *X, T *Y, int64_t K, int c4, const BandMat &M1, const BandMat &M4, cudaStream_t s)
{
    if (M1.W > 16 || M1.win16 > kKWIN || M1.rows < 2 || c4 > kCB || c4 < 1 || M4.cols != c4 || K <= 0) return false;
    count_launch();
    switch (M1.W) {
#define TCA_WL_CASE(w) \
    case w: launch_win_last_w<T, w>(X, Y, K, c4, M1, M4, s); return true;
        TCA_WL_CASE(1) TCA_WL_CASE(2) TCA_WL_CASE(3) TCA_WL_CASE(4) TCA_WL_CASE(5) TCA_WL_CASE(6)
        TCA_WL_CASE(7) TCA_WL_CASE(8) TCA_WL_CASE(9) TCA_WL_CASE(10) TCA_WL_CASE(11) TCA_WL_CASE(12)
        TCA_WL_CASE(13) TCA_WL_CASE(14) TCA_WL_CASE(15) TCA_WL_CASE(16)
#undef TCA_WL_CASE
    }
    return false;
}

// Two fastest modes in one pass (rhs / forward model tail, PAPER.md:83's
// successive mode products): for each plane o of an (outer, c3, c4) tensor,
//   Z[a, j] = sum_w M4[j, w] X[o, a, s4[j] + w]        (mode D,   a < c3, j < r4)
//   Y[o, i, j] = sum_w M3[i, w] Z[s3[i] + w, j]         (mode D-1, i < r3)
// with the plane and Z in shared memory: the tensor is read once and only the
// contracted plane is written (config 3's rhs: 256 x 30 -> 128 x 15 per (i1, i2),
// 1 GB in and 0.25 GB out instead of 1.5 GB + 0.75 GB over two passes).
// Plane rows have an odd pitch (c4 | 1) so the column reads of stage 1 are
// conflict-free; stage 1: warp per output column j (its taps in registers),
// lanes over rows a; stage 2: half-warp per output row i, lanes over j.
constexpr int kPlaneThreads = 512;

// copies a plane into [row][p4] with the data at column offset g4: one 8- or
// 4-byte asynchronous copy per element, flat index (row = e / c4 through an fp32
// reciprocal: exact for e < 2^22)
template <typename T>
__device__ __forceinline__ void plane_load_async(T *xs, const T *xp, int nin, int c4, float inv_c4, int p4, int g4)
{
    const unsigned base = (unsigned)__cvta_generic_to_shared(xs + g4);
    for (int e = threadIdx.x; e < nin; e += kPlaneThreads) {
        const int a = (int)(((float)e + 0.5f) * inv_c4);
        const unsigned dst = base + (unsigned)((e + a * (p4 - c4)) * (int)sizeof(T));
        if (sizeof(T) == 8)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(xp + e) : "memory");
        else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(xp + e) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Persistent (one block per SM), double-buffered: the next plane's copies are
// in flight while this one is computed.  Zero guard columns (g4 each side of a
// plane row) and guard rows (g3 above / below Z) stand in for the columns a
// band row reaches past the matrix (their taps are zero), so the inner loops
// have no bounds tests.  Mode-D taps live in registers (warp per column j for
// the whole kernel); mode-(D-1) taps in a shared table.
template <typename T, int WC>
__global__ void __launch_bounds__(kPlaneThreads, 1)
band_plane2_kernel(const T *__restrict__ X, T *__restrict__ Y, int64_t planes, int c3, int c4, int r3, int r4,
                   const int *__restrict__ s3, const T *__restrict__ t3, int w3, int g3, const int *__restrict__ s4,
                   const T *__restrict__ t4, int w4, int g4)
{
    extern __shared__ __align__(16) unsigned char pl_raw[];
    const int p4 = (c4 + 2 * g4) | 1;       // odd pitch: conflict-free column reads
    const int pz = r4 | 1;
    const int zrows = c3 + 2 * g3;
    T *xs0 = reinterpret_cast<T *>(pl_raw);  // 2 x [c3][p4]
    T *zs = xs0 + 2 * (size_t)c3 * p4;      // [zrows][pz]; data rows start at g3
    T *t3s = zs + (size_t)zrows * pz;       // [r3][WC]
    int *s3s = reinterpret_cast<int *>(t3s + (size_t)r3 * WC);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = kPlaneThreads / 32;
    const int nin = c3 * c4, nout = r3 * r4;
    // one-time: zero guards, stage the mode-(D-1) table
    for (int e = threadIdx.x; e < 2 * c3 * p4; e += kPlaneThreads) xs0[e] = T(0);
    for (int e = threadIdx.x; e < zrows * pz; e += kPlaneThreads) zs[e] = T(0);
    for (int e = threadIdx.x; e < r3 * WC; e += kPlaneThreads) {
        const int i = e / WC, w = e - i * WC;
        t3s[e] = w < w3 ? t3[(int64_t)i * w3 + w] : T(0);
    }
    for (int i = threadIdx.x; i < r3; i += kPlaneThreads) s3s[i] = s3[i] + g3;
    __syncthreads();
    int64_t o = blockIdx.x;
    const float inv_c4 = 1.0f / (float)c4;
    if (o < planes) plane_load_async(xs0, X + o * (int64_t)nin, nin, c4, inv_c4, p4, g4);
    for (int b = 0; o < planes; o += gridDim.x, b ^= 1) {
        const T *xs = xs0 + (size_t)b * c3 * p4;
        const int64_t on = o + gridDim.x;
        if (on < planes) {
            plane_load_async(xs0 + (size_t)(b ^ 1) * c3 * p4, X + on * (int64_t)nin, nin, c4, inv_c4, p4, g4);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();   // plane o staged (every thread's copies)
        // stage 1: mode D, warp per output column j, lanes over rows a
        for (int j = warp; j < r4; j += NW) {
            const int sj = __ldg(s4 + j) + g4;
            T tp[WC];
#pragma unroll
            for (int w = 0; w < WC; ++w) tp[w] = w < w4 ? __ldg(t4 + (int64_t)j * w4 + w) : T(0);
            for (int a = lane; a < c3; a += 64) {   // two rows per lane: independent FMA chains
                const bool two = a + 32 < c3;
                const T *row = xs + a * p4 + sj;
                const T *row2 = two ? row + 32 * p4 : row;
                T acc = T(0), acc2 = T(0);
#pragma unroll
                for (int w = 0; w < WC; ++w) {
                    acc = fma(tp[w], row[w], acc);
                    acc2 = fma(tp[w], row2[w], acc2);
                }
                zs[(a + g3) * pz + j] = acc;
                if (two) zs[(a + 32 + g3) * pz + j] = acc2;
            }
        }
        __syncthreads();
        // stage 2: mode D-1, half-warp per output row i, lanes over j
        T *yp = Y + o * (int64_t)nout;
        const int half = lane >> 4, hl = lane & 15;
        for (int i0 = 2 * warp; i0 < r3; i0 += 4 * NW) {   // rows i and i + 2 NW per half-warp
            const int i = i0 + half, i2 = i + 2 * NW;
            if (i >= r3) continue;
            const bool two = i2 < r3;
            const T *tr = t3s + i * WC, *tr2 = t3s + (two ? i2 : i) * WC;
            const T *zc = zs + s3s[i] * pz, *zc2 = zs + s3s[two ? i2 : i] * pz;
            for (int j = hl; j < r4; j += 16) {
                T acc = T(0), acc2 = T(0);
#pragma unroll
                for (int w = 0; w < WC; ++w) {
                    acc = fma(tr[w], zc[w * pz + j], acc);
                    acc2 = fma(tr2[w], zc2[w * pz + j], acc2);
                }
                yp[i * r4 + j] = acc;
                if (two) yp[i2 * r4 + j] = acc2;
            }
        }
        __syncthreads();   // zs and xs[b] free before the next plane's stages / copies
    }
}

template <typename T, int WC>
static void launch_plane2_w(const T *X, T *Y, int64_t planes, int c3, int c4, const BandMat &M3, const BandMat &M4,
                            size_t smem, cudaStream_t s)
{
    set_max_dynamic_smem((const void *)band_plane2_kernel<T, WC>, smem);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(planes, (int64_t)sms));   // one per SM
    const int g3 = std::max(M3.reach_lo, M3.reach_hi), g4 = std::max(M4.reach_lo, M4.reach_hi);
    band_plane2_kernel<T, WC><<<(unsigned)grid, kPlaneThreads, smem, s>>>(
        X, Y, planes, c3, c4, M3.rows, M4.rows, M3.start, (const T *)M3.taps, M3.W, g3, M4.start,
        (const T *)M4.taps, M4.W, g4);
}

template <typename T>
bool launch_band_plane2(const T *X, T *Y, int64_t planes, int c3, int c4, const BandMat &M3, const BandMat &M4,
                        cudaStream_t s)
{
    const int wmax = std::max(M3.W, M4.W);
    if (wmax > 16 || M3.cols != c3 || M4.cols != c4 || planes <= 0 || (int64_t)c3 * c4 >= (1 << 22)) return false;
    const int w = wmax <= 4 ? 4 : wmax <= 8 ? 8 : wmax <= 12 ? 12 : 16;
    const int g3 = std::max(M3.reach_lo, M3.reach_hi), g4 = std::max(M4.reach_lo, M4.reach_hi);
    const size_t p4 = (size_t)((c4 + 2 * g4) | 1), pz = (size_t)(M4.rows | 1);
    const size_t smem = (2 * (size_t)c3 * p4 + (size_t)(c3 + 2 * g3) * pz + (size_t)M3.rows * w) * sizeof(T) +
                        (size_t)M3.rows * sizeof(int);
    if (smem > 220 * 1024) return false;
    count_launch();
    switch (w) {
    case 4: launch_plane2_w<T, 4>(X, Y, planes, c3, c4, M3, M4, smem, s); break;
    case 8: launch_plane2_w<T, 8>(X, Y, planes, c3, c4, M3, M4, smem, s); break;
    case 12: launch_plane2_w<T, 12>(X, Y, planes, c3, c4, M3, M4, smem, s); break;
    default: launch_plane2_w<T, 16>(X, Y, planes, c3, c4, M3, M4, smem, s); break;
    }
    return true;
}

// Short planes (mode D of a wide tensor: rows x 1) would leave most of every
// block idle in the (plane, outer) mapping: there the flat index runs over
// outer x plane instead.
template <typename T>
__global__ void __launch_bounds__(256)
band_mode_product_flat_kernel(const T *__restrict__ X, T *__restrict__ Y, int64_t total, int rows, int cols,
                              int inner, const int *__restrict__ start, const T *__restrict__ taps, int W, T alpha,
                              int accumulate, const int32_t *done)
{
    if (done && *done) return;
    const int64_t plane = (int64_t)rows * inner;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = idx / plane;
        const int64_t rem = idx - o * plane;
        const int r = (int)(rem / inner), t = (int)(rem - (int64_t)r * inner);
        const int s0 = __ldg(start + r);
        const T *xp = X + o * (int64_t)cols * inner + t;
        const T *tp = taps + (int64_t)r * W;
        T acc = T(0);
        for (int w = 0; w < W; ++w) {
            const int c = s0 + w;
            if (c >= 0 && c < cols) acc = fma(__ldg(tp + w), __ldg(xp + (int64_t)c * inner), acc);
        }
        acc *= alpha;
        if (accumulate) acc += Y[idx];
        Y[idx] = acc;
    }
}

template <typename T>
void launch_band_mode_product(const T *X, T *Y, int64_t outer, const BandMat &M,
                              int64_t inner, double alpha, bool accumulate,
                              const int32_t *done, cudaStream_t s)
{
    const int64_t plane = (int64_t)M.rows * inner;
    if (plane == 0 || outer == 0) return;
    const int64_t target = 148 * 16;   // enough CTAs to fill the GPU
    count_launch();
    if (plane < 64 * 256 && outer > 1) {
        const int64_t total = plane * outer;
        const int64_t bx = std::min<int64_t>((total + 255) / 256, 8 * target);
        band_mode_product_flat_kernel<T><<<(unsigned)bx, 256, 0, s>>>(
            X, Y, total, M.rows, M.cols, (int)inner, M.start, (const T *)M.taps, M.W, (T)alpha, accumulate ? 1 : 0,
            done);
        return;
    }
    if (inner >= 32 && M.rows >= 2 && M.W <= 16 && M.win16 <= kKWIN) {
        switch (M.W) {
#define TCA_WIN_CASE(w) \
    case w: launch_win<T, w>(X, Y, outer, M, inner, alpha, accumulate, done, s); return;
            TCA_WIN_CASE(1) TCA_WIN_CASE(2) TCA_WIN_CASE(3) TCA_WIN_CASE(4) TCA_WIN_CASE(5) TCA_WIN_CASE(6)
            TCA_WIN_CASE(7) TCA_WIN_CASE(8) TCA_WIN_CASE(9) TCA_WIN_CASE(10) TCA_WIN_CASE(11) TCA_WIN_CASE(12)
            TCA_WIN_CASE(13) TCA_WIN_CASE(14) TCA_WIN_CASE(15) TCA_WIN_CASE(16)
#undef TCA_WIN_CASE
        }
    }
    // plane < 2^32 is guaranteed by the extent limits checked at create
    int64_t bx = (plane + 255) / 256;
    int64_t by = outer;
    if (bx > target) bx = target;
    if (by > 65535) by = 65535;
    if (bx * by > 8 * target) by = std::max<int64_t>(1, 8 * target / bx);
    band_mode_product_kernel<T><<<dim3((unsigned)bx, (unsigned)by), 256, 0, s>>>(
        X, Y, outer, M.rows, M.cols, (int)inner, M.start, (const T *)M.taps, M.W, (T)alpha,
        accumulate ? 1 : 0, done);
}

// ---------------------------------------------------------------- dense mode product on FP64 tensor cores
// Y[o, r, t] = alpha * sum_c M[r, c] X[o, c, t] (+ Y) for a dense M (rows x cols):
// per fibre f = (o, t) a GEMM  Y[r, f] = M[r, :] X[:, f].  One warp computes
// 8 x 8 output tiles (8 rows of M x 8 consecutive fibres) with
// mma.sync.m8n8k4.f64 (DMMA: tcgen05 has no f64 kind, SURVEY.md reading Z14),
// K stepped by 4 over the columns of M; fragments are read straight from
// global memory (M is at most a few hundred rows; X fibres are coalesced over
// t).  Used for dense modes (config 1's Gaussian A_d) in fp64.
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256)
dense_mode_product_dmma_kernel(const double *__restrict__ X, double *__restrict__ Y, int64_t nfib, int rows,
                               int cols, int64_t inner, const double *__restrict__ M, double alpha, int accumulate,
                               const int32_t *done)
{
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int rtiles = (rows + 7) / 8;
    const int64_t ftiles = (nfib + 7) / 8;
    const int ar = lane >> 2, ak = lane & 3;          // A fragment: M[r0 + ar][k + ak]
    const int bk = lane & 3, bn = lane >> 2;          // B fragment: X[k + bk][f0 + bn]
    const int dr = lane >> 2, dn = 2 * (lane & 3);    // D fragment: Y[r0 + dr][f0 + dn + {0,1}]
    for (int64_t tile = warp; tile < (int64_t)rtiles * ftiles; tile += nwarps) {
        const int r0 = (int)(tile % rtiles) * 8;
        const int64_t f0 = (tile / rtiles) * 8;
        const int64_t fb = f0 + bn;
        const bool bvalid = fb < nfib;
        const int64_t ob = bvalid ? fb / inner : 0, tb = bvalid ? fb - ob * inner : 0;
        const double *xb = X + ob * (int64_t)cols * inner + tb;
        const int ra = r0 + ar;
        const double *ma = M + (int64_t)(ra < rows ? ra : 0) * cols;
        double d0 = 0.0, d1 = 0.0;
        for (int k = 0; k < cols; k += 4) {
            const int ka = k + ak, kb = k + bk;
            const double a = (ra < rows && ka < cols) ? __ldg(ma + ka) : 0.0;
            const double b = (bvalid && kb < cols) ? __ldg(xb + (int64_t)kb * inner) : 0.0;
            dmma884(d0, d1, a, b);
        }
        const int r = r0 + dr;
        if (r < rows) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t f = f0 + dn + h;
                if (f < nfib) {
                    const int64_t o = f / inner, t = f - o * inner;
                    double *yp = Y + (o * rows + r) * inner + t;
                    double v = alpha * (h ? d1 : d0);
                    if (accumulate) v += *yp;
                    *yp = v;
                }
            }
        }
    }
}

// Shared-memory tiled form: a block computes a 64-row x 64-fibre tile of Y,
// stepping K by 16: the M tile (64 x 16) and the X tile (16 x 64: 16 rows of
// 64 fibres) are staged in shared memory (double-buffered, the next step's
// global loads in registers while this step's DMMAs run), and each of the 8
// warps computes a 16 x 32 sub-tile as 2 x 4 m8n8k4 accumulators, so every
// fragment element loaded from shared memory feeds 2-4 DMMAs (the direct
// kernel above reloads both operands from global memory for every DMMA).
constexpr int kDBM = 64, kDBN = 64, kDBK = 16, kDPA = kDBK + 4, kDPB = kDBN + 4;

__global__ void __launch_bounds__(256)
dense_mode_product_dmma_tiled_kernel(const double *__restrict__ X, double *__restrict__ Y, int64_t nfib, int rows,
                                     int cols, int64_t inner, const double *__restrict__ M, double alpha,
                                     int accumulate, const int32_t *done)
{
    if (done && *done) return;
    __shared__ double As[2][kDBM * kDPA];
    __shared__ double Bs[2][kDBK * kDPB];
    __shared__ int64_t fbase[kDBN];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = blockIdx.y * kDBM;
    const int64_t f0 = (int64_t)blockIdx.x * kDBN;
    if (tid < kDBN) {
        const int64_t f = f0 + tid;
        if (f < nfib) {
            const int64_t o = f / inner, t = f - o * inner;
            fbase[tid] = o * (int64_t)cols * inner + t;
        } else {
            fbase[tid] = -1;
        }
    }
    __syncthreads();
    const bool kfast = inner == 1;   // fibres contiguous: load each fibre's k-run (coalesced)
    // this thread's 4 A and 4 B tile elements (global -> registers -> shared)
    double ra[4], rb[4];
    auto gload = [&](int k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + u * 256;
            const int m = e / kDBK, k = e % kDBK;   // A: k fastest
            const int rr = r0 + m, kk = k0 + k;
            ra[u] = (rr < rows && kk < cols) ? __ldg(M + (int64_t)rr * cols + kk) : 0.0;
            int bk, bn;
            if (kfast) { bn = e / kDBK; bk = e % kDBK; }
            else { bk = e / kDBN; bn = e % kDBN; }
            const int64_t fb = fbase[bn];
            const int kb = k0 + bk;
            rb[u] = (fb >= 0 && kb < cols) ? __ldg(X + fb + (int64_t)kb * inner) : 0.0;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + u * 256;
            As[buf][(e / kDBK) * kDPA + e % kDBK] = ra[u];
            int bk, bn;
            if (kfast) { bn = e / kDBK; bk = e % kDBK; }
            else { bk = e / kDBN; bn = e % kDBN; }
            Bs[buf][bk * kDPB + bn] = rb[u];
        }
    };
    const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;   // warp sub-tile origin
    const int ar = lane >> 2, ak = lane & 3, bk = lane & 3, bn = lane >> 2;
    double d[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) d[i][j][0] = d[i][j][1] = 0.0;
    const int nk = (cols + kDBK - 1) / kDBK;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int ks = 0; ks < nk; ++ks) {
        const int buf = ks & 1;
        if (ks + 1 < nk) gload((ks + 1) * kDBK);
#pragma unroll
        for (int kk = 0; kk < kDBK; kk += 4) {
            double af[2], bf[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) af[i] = As[buf][(wm + i * 8 + ar) * kDPA + kk + ak];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][(kk + bk) * kDPB + wn + j * 8 + bn];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(d[i][j][0], d[i][j][1], af[i], bf[j]);
        }
        if (ks + 1 < nk) {
            sstore(buf ^ 1);   // the other buffer: last read one step ago, before this step's barrier
            __syncthreads();
        }
    }
    const int dr = lane >> 2, dn = 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int r = r0 + wm + i * 8 + dr;
        if (r >= rows) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int fl = wn + j * 8 + dn + h;
                const int64_t f = f0 + fl;
                if (f < nfib) {
                    const int64_t o = f / inner, t = f - o * inner;
                    double *yp = Y + (o * rows + r) * inner + t;
                    double v = alpha * d[i][j][h];
                    if (accumulate) v += *yp;
                    *yp = v;
                }
            }
    }
}

void launch_dense_mode_product_dmma(const double *X, double *Y, int64_t outer, int rows, int cols,
                                    int64_t inner, const double *M, double alpha, bool accumulate,
                                    const int32_t *done, cudaStream_t s)
{
    const int64_t nfib = outer * inner;
    if (nfib == 0 || rows == 0) return;
    static const bool direct = getenv("TCA_DMMA_DIRECT") != nullptr;   // measurement switch: the untiled kernel
    if (!direct && rows >= 32 && cols >= 16 && (nfib + kDBN - 1) / kDBN < (1ll << 31) && (rows + kDBM - 1) / kDBM < 65536) {
        count_launch();
        dense_mode_product_dmma_tiled_kernel<<<dim3((unsigned)((nfib + kDBN - 1) / kDBN), (unsigned)((rows + kDBM - 1) / kDBM)),
                                               256, 0, s>>>(X, Y, nfib, rows, cols, inner, M, alpha, accumulate ? 1 : 0,
                                                            done);
        return;
    }
    const int64_t tiles = (int64_t)((rows + 7) / 8) * ((nfib + 7) / 8);
    int64_t blocks = (tiles + 7) / 8;   // 8 warps per block, one tile per warp per pass
    if (blocks > 148 * 16) blocks = 148 * 16;
    count_launch();
    dense_mode_product_dmma_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, Y, nfib, rows, cols, inner, M, alpha,
                                                                    accumulate ? 1 : 0, done);
}

// ---------------------------------------------------------------- generator (Z9)
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t stream_key(uint64_t seed, uint32_t stream_id)
{
    return mix64(seed * kGamma + (uint64_t)stream_id);
}

__device__ __forceinline__ double u01(uint64_t z)
{
    return ((double)(z >> 11) + 0.5) * 0x1.0p-53;
}

__device__ __forceinline__ double normal_at(uint64_t key, uint64_t j)
{
    const double u1 = u01(mix64(key + (2 * j) * kGamma));
    const double u2 = u01(mix64(key + (2 * j + 1) * kGamma));
    const double two_pi = 6.283185307179586;  // (2 * pi) rounded to double
    const double a = __dmul_rn(two_pi, u2);
    return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(a));
}

template <typename T>
__global__ void gen_normal_kernel(T *out, int64_t count, int64_t offset, uint64_t key,
                                  double scale, int accumulate)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = __dmul_rn(scale, normal_at(key, (uint64_t)(offset + i)));
        if (accumulate) v = __dadd_rn((double)out[i], v);
        out[i] = (T)v;
    }
}

template <typename T>
void launch_gen_normal(T *out, int64_t count, int64_t offset, uint64_t key, double scale,
                       bool accumulate, cudaStream_t s)
{
    if (count <= 0) return;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    count_launch();
    gen_normal_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(out, count, offset, key, scale,
                                                         accumulate ? 1 : 0);
}

// ---------------------------------------------------------------- CG vector kernels
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
cg_init_kernel(const T *__restrict__ b, T *__restrict__ x, T *__restrict__ r,
               T *__restrict__ p, int64_t N, double *part)
{
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const T v = b[i];
        r[i] = v;          // R := B - A*0
        p[i] = v;          // P := R
        x[i] = T(0);       // C := 0
        acc += (double)v * (double)v;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// d = b - q (r, p optional outputs), partials of <d, d> and <b, b>
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
resid2_kernel(const T *__restrict__ b, const T *__restrict__ q, T *__restrict__ r, T *__restrict__ p, int64_t N,
              double *part_dd, double *part_bb)
{
    double dd = 0.0, bb = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const T bv = b[i];
        const T d = bv - q[i];
        if (r) r[i] = d;
        if (p) p[i] = d;
        dd += (double)d * (double)d;
        bb += (double)bv * (double)bv;
    }
    const double s1 = block_sum(dd);
    __syncthreads();
    const double s2 = block_sum(bb);
    if (threadIdx.x == 0) {
        part_dd[blockIdx.x] = s1;
        part_bb[blockIdx.x] = s2;
    }
}

template <typename T>
void launch_resid2(const T *b, const T *q, T *r, T *p, int64_t N, double *part_dd, double *part_bb, cudaStream_t s)
{
    count_launch();
    resid2_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(b, q, r, p, N, part_dd, part_bb);
}

// 16-byte vector views (2 doubles or 4 floats) for the streaming CG kernels:
// each thread moves VW elements per access; a scalar tail covers N % VW.
template <typename T> struct Vec;
template <> struct Vec<double> { using V = double2; static constexpr int W = 2; };
template <> struct Vec<float> { using V = float4; static constexpr int W = 4; };

template <typename V> __device__ __forceinline__ double vdot(const V &a, const V &b);
template <> __device__ __forceinline__ double vdot<double2>(const double2 &a, const double2 &b)
{
    return fma(a.x, b.x, a.y * b.y);
}
template <> __device__ __forceinline__ double vdot<float4>(const float4 &a, const float4 &b)
{
    return (double)a.x * b.x + (double)a.y * b.y + (double)a.z * b.z + (double)a.w * b.w;
}
__device__ __forceinline__ double2 vaxpy(double2 y, double a, double2 x) { return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y)); }
__device__ __forceinline__ float4 vaxpy(float4 y, float a, float4 x)
{
    return make_float4(fmaf(a, x.x, y.x), fmaf(a, x.y, y.y), fmaf(a, x.z, y.z), fmaf(a, x.w, y.w));
}

template <typename T>
__device__ __forceinline__ bool aligned16(const T *p) { return ((uintptr_t)p & 15) == 0; }

template <typename T>
__global__ void __launch_bounds__(kRedThreads)
dot_partials_kernel(const T *__restrict__ a, const T *__restrict__ b, int64_t N,
                    double *part, const int32_t *done)
{
    if (done && *done) return;
    using V = typename Vec<T>::V;
    constexpr int VW = Vec<T>::W;
    double acc = 0.0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    int64_t nv = 0;
    if (aligned16(a) && aligned16(b)) {
        nv = N / VW;
        const V *av = reinterpret_cast<const V *>(a), *bv = reinterpret_cast<const V *>(b);
        for (int64_t i = tid; i < nv; i += nth) acc += vdot(__ldcs(av + i), __ldcs(bv + i));
    }
    for (int64_t i = nv * VW + tid; i < N; i += nth) acc += (double)a[i] * (double)b[i];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// The CG updates in two streaming passes, 8 words per unknown (Fig. 2 as
// written: 9):  R := R - alpha Q with the R+*R partials (read r, q; write r),
// then, once beta is known,  C := C + alpha P  and  P := R + beta P  in one pass
// over p (read x, p, r; write x, p).  x_{k+1} = x_k + alpha_k p_k uses the p_k
// the apply read, so the iterates are exactly Fig. 2's.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
cg_update_r_kernel(T *__restrict__ r, const T *__restrict__ q, int64_t N, CgScalars *sc, double *part, int fin,
                   double *hist, int rev)
{
    if (sc->done) return;
    using V = typename Vec<T>::V;
    constexpr int VW = Vec<T>::W;
    const T alpha = (T)sc->alpha;
    double acc = 0.0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    int64_t nv = 0;
    if (aligned16(r) && aligned16(q)) {
        nv = N / VW;
        V *rv = reinterpret_cast<V *>(r);
        const V *qv = reinterpret_cast<const V *>(q);
        if (rev) {   // L2 hand-off (see l2_handoff): last slabs first, R kept in L2 for cg_update_xp;
                     // 4 vectors of R and Q in flight per thread (f64 CG 577.4 -> 569.1 us per iteration)
#ifndef TCA_R_UNR
#define TCA_R_UNR 4   // vectors in flight per thread (2: same within noise, 8: +8 us; profiles/r02_runroll_probe.txt)
#endif
            constexpr int U = TCA_R_UNR;
            int64_t i = nv - 1 - tid;
            for (; i - (U - 1) * nth >= 0; i -= U * nth) {
                V ra[U], qa[U];
#pragma unroll
                for (int u = 0; u < U; ++u) { ra[u] = __ldcg(rv + i - u * nth); qa[u] = __ldcs(qv + i - u * nth); }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const V rn = vaxpy(ra[u], -alpha, qa[u]);
                    __stcg(rv + i - u * nth, rn);
                    acc += vdot(rn, rn);
                }
            }
            for (; i >= 0; i -= nth) {
                const V rn = vaxpy(__ldcg(rv + i), -alpha, __ldcs(qv + i));
                __stcg(rv + i, rn);
                acc += vdot(rn, rn);
            }
        } else {
            for (int64_t i = tid; i < nv; i += nth) {
                const V rn = vaxpy(__ldcs(rv + i), -alpha, __ldcs(qv + i));   // R := R - alpha*Q
                __stcs(rv + i, rn);
                acc += vdot(rn, rn);                                           // rho1 := R+*R (partials)
            }
        }
    }
    for (int64_t i = nv * VW + tid; i < N; i += nth) {
        const T rv = r[i] - alpha * q[i];
        r[i] = rv;
        acc += (double)rv * (double)rv;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    if (fin) {   // rho1, stop test, beta in the last CTA (tca_finalize.cuh)
        __shared__ double red[kRedThreads / 32 + 1];
        fin_last_cta(2, 1, part, sc, hist, red);
    }
}

// C := C + alpha*P*D when this iteration's alpha is valid (sc->xupd), then
// P := R + beta*P unless the solve stopped at this iteration.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
cg_update_xp_kernel(T *__restrict__ x, T *__restrict__ p, const T *__restrict__ r, int64_t N, const CgScalars *sc,
                    int keep_r)
{
    if (!sc->xupd) return;
    using V = typename Vec<T>::V;
    constexpr int VW = Vec<T>::W;
    const T alpha = (T)sc->alpha;
    const T beta = (T)sc->beta;
    const bool upd_p = !sc->done;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    int64_t nv = 0;
    if (aligned16(x) && aligned16(p) && aligned16(r)) {
        nv = N / VW;
        V *xv = reinterpret_cast<V *>(x), *pv = reinterpret_cast<V *>(p);
        const V *rv = reinterpret_cast<const V *>(r);
        if (upd_p) {
            for (int64_t i = tid; i < nv; i += nth) {
                const V pi = __ldcs(pv + i), xi = __ldcs(xv + i), ri = keep_r ? __ldcg(rv + i) : __ldcs(rv + i);
                __stcs(xv + i, vaxpy(xi, alpha, pi));   // C := C + alpha*P*D
                __stcs(pv + i, vaxpy(ri, beta, pi));    // P := R + beta*P
            }
        } else {
            for (int64_t i = tid; i < nv; i += nth) __stcs(xv + i, vaxpy(__ldcs(xv + i), alpha, __ldcs(pv + i)));
        }
    }
    for (int64_t i = nv * VW + tid; i < N; i += nth) {
        const T pi = p[i];
        x[i] = x[i] + alpha * pi;
        if (upd_p) p[i] = r[i] + beta * pi;
    }
}

// P_next := D + beta*P (D = R, or Z in PCG) into the other buffer of the P
// pair, unless the solve stopped at this iteration (3 words).  The x update of
// this iteration is deferred to the next apply (MODE 2 of the band apply),
// which still reads P from its own buffer.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
cg_update_p_kernel(T *__restrict__ pn, const T *__restrict__ p, const T *__restrict__ d, int64_t N, const CgScalars *sc)
{
    if (sc->done) return;
    using V = typename Vec<T>::V;
    constexpr int VW = Vec<T>::W;
    const T beta = (T)sc->beta;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    int64_t nv = 0;
    if (aligned16(pn) && aligned16(p) && aligned16(d)) {
        nv = N / VW;
        V *pnv = reinterpret_cast<V *>(pn);
        const V *pv = reinterpret_cast<const V *>(p), *dv = reinterpret_cast<const V *>(d);
        // D (= R, just written by cg_update_r's reverse sweep) read L2-normal from the
        // start: the L2 hand-off; 4 vectors of D and P in flight per thread
        int64_t i = tid;
        for (; i + 3 * nth < nv; i += 4 * nth) {
            V da[4], pa[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { da[u] = __ldcg(dv + i + u * nth); pa[u] = __ldcs(pv + i + u * nth); }
#pragma unroll
            for (int u = 0; u < 4; ++u) __stcs(pnv + i + u * nth, vaxpy(da[u], beta, pa[u]));
        }
        for (; i < nv; i += nth) __stcs(pnv + i, vaxpy(__ldcg(dv + i), beta, __ldcs(pv + i)));
    }
    for (int64_t i = nv * VW + tid; i < N; i += nth) pn[i] = d[i] + beta * p[i];
}

// Single-reduction CG (Chronopoulos-Gear, reading Z24): one
// streaming pass per iteration before the apply,
//   P := R + beta*P;  S := W + beta*S;  C := C + alpha*P;  R := R - alpha*S
// with the R+*R partials of the new R (9 words per unknown; the apply then
// reads R and produces W = A*R and R+*W: one reduction point per iteration).
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
cgsr_update_kernel(T *__restrict__ x, T *__restrict__ p, T *__restrict__ sv, T *__restrict__ r,
                   const T *__restrict__ w, int64_t N, const CgScalars *sc, double *part)
{
    if (sc->done) return;
    using V = typename Vec<T>::V;
    constexpr int VW = Vec<T>::W;
    const T alpha = (T)sc->alpha, beta = (T)sc->beta;
    double acc = 0.0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    int64_t nv = 0;
    if (aligned16(x) && aligned16(p) && aligned16(sv) && aligned16(r) && aligned16(w)) {
        nv = N / VW;
        V *xv = reinterpret_cast<V *>(x), *pv = reinterpret_cast<V *>(p), *svv = reinterpret_cast<V *>(sv),
          *rv = reinterpret_cast<V *>(r);
        const V *wv = reinterpret_cast<const V *>(w);
        for (int64_t i = tid; i < nv; i += nth) {
            const V ri = __ldcs(rv + i);
            const V pn = vaxpy(ri, beta, __ldcs(pv + i));                // P := R + beta*P
            const V sn = vaxpy(__ldcs(wv + i), beta, __ldcs(svv + i));   // S := W + beta*S
            __stcs(pv + i, pn);
            __stcs(svv + i, sn);
            __stcs(xv + i, vaxpy(__ldcs(xv + i), alpha, pn));           // C := C + alpha*P
            const V rn = vaxpy(ri, -alpha, sn);                          // R := R - alpha*S
            __stcs(rv + i, rn);
            acc += vdot(rn, rn);
        }
    }
    for (int64_t i = nv * VW + tid; i < N; i += nth) {
        const T pn = r[i] + beta * p[i];
        const T sn = w[i] + beta * sv[i];
        p[i] = pn;
        sv[i] = sn;
        x[i] = x[i] + alpha * pn;
        const T rn = r[i] - alpha * sn;
        r[i] = rn;
        acc += (double)rn * (double)rn;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

template <typename T>
void launch_cgsr_update(T *x, T *p, T *sv, T *r, const T *w, int64_t N, const CgScalars *sc, double *part,
                        cudaStream_t s)
{
    count_launch();
    cgsr_update_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(x, p, sv, r, w, N, sc, part);
}

template <typename T>
void launch_cg_init(const T *b, T *x, T *r, T *p, int64_t N, double *part, cudaStream_t s)
{
    count_launch();
    cg_init_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(b, x, r, p, N, part);
}

template <typename T>
void launch_dot_partials(const T *a, const T *b, int64_t N, double *part,
                         const int32_t *done, cudaStream_t s)
{
    count_launch();
    dot_partials_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(a, b, N, part, done);
}

template <typename T>
void launch_cg_update_r(T *r, const T *q, int64_t N, CgScalars *sc, double *part, cudaStream_t s, bool fin,
                        double *hist)
{
    count_launch();
    cg_update_r_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(r, q, N, sc, part, fin ? 1 : 0, hist, l2_handoff());
}

template <typename T>
void launch_cg_update_p(T *pn, const T *p, const T *d, int64_t N, const CgScalars *sc, cudaStream_t s)
{
    count_launch();
    cg_update_p_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(pn, p, d, N, sc);
}

template <typename T>
void launch_cg_update_xp(T *x, T *p, const T *r, int64_t N, const CgScalars *sc, cudaStream_t s)
{
    count_launch();
    cg_update_xp_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(x, p, r, N, sc, l2_handoff());
}

// ---------------------------------------------------------------- finalisers
// One block of kRedThreads sums the kRedBlocks partials in a fixed order.
__global__ void __launch_bounds__(kRedThreads)
cg_finalize_kernel(int which, const double *__restrict__ part, int nparts, CgScalars *sc, double *hist, int stage)
{
    if (which != 0 && which != 7 && which < 8 && sc->done) {
        // stopped in an earlier iteration: this iteration's x update is void
        if (which == 1 && stage != 1 && threadIdx.x == 0) sc->xupd = 0;
        return;
    }
    double s = 0.0;
    if (stage != 2) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < nparts; i += kRedThreads) acc += part[i];
        s = block_sum(acc);
        if (threadIdx.x != 0) return;
        if (stage == 1) {   // local sum only; the all-reduce and stage 2 follow
            sc->red[which] = s;
            return;
        }
    } else {
        if (threadIdx.x != 0) return;
        s = sc->red[which];
    }
    cg_finalize_scalars(which, s, sc, hist);   // tca_finalize.cuh
}

// Single-reduction CG finaliser: gamma = R+*R (update-kernel partials) and
// delta = R+*W (apply partials) in one step; which = 7 starts the solve (R = B,
// W = A*B), which = 6 closes an iteration.  Stage 1 leaves the two local sums
// in red[3], red[4] for ONE all-reduce of two fp64 values; stage 2 finishes.
__global__ void __launch_bounds__(kRedThreads)
cgsr_finalize_kernel(int which, const double *__restrict__ prr, int nrr, const double *__restrict__ prw, int nrw,
                     CgScalars *sc, double *hist, int stage)
{
    if (which == 6 && sc->done) return;
    double g = 0.0, dl = 0.0;
    if (stage != 2) {
        double a = 0.0, b = 0.0;
        for (int i = threadIdx.x; i < nrr; i += kRedThreads) a += prr[i];
        g = block_sum(a);
        __syncthreads();
        for (int i = threadIdx.x; i < nrw; i += kRedThreads) b += prw[i];
        dl = block_sum(b);
        if (threadIdx.x != 0) return;
        if (stage == 1) {
            sc->red[3] = g;
            sc->red[4] = dl;
            return;
        }
    } else {
        if (threadIdx.x != 0) return;
        g = sc->red[3];
        dl = sc->red[4];
    }
    if (which == 7) {   // gamma0 = <r0, r0>, delta0 = <r0, A r0> (r0 = b when x0 = 0)
        sc->rho = g;
        sc->rho0 = g;
        sc->ref = g;
        sc->rr = g;
        sc->iters = 0;
        sc->converged = 0;
        sc->status = TCA_OK;
        sc->done = 0;
        sc->xupd = 0;
        sc->beta = 0.0;
        if (hist) hist[0] = g;
        if (!isfinite(g)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
        if (g == 0.0) { sc->converged = 1; sc->done = 1; return; }
        if (sc->max_iters <= 0) { sc->done = 1; if (sc->rtol2 > 0.0) sc->status = TCA_NOT_CONVERGED; return; }
        if (!isfinite(dl)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
        if (!(dl > 0.0)) { sc->status = TCA_ERR_BREAKDOWN; sc->done = 1; return; }
        sc->alpha = g / dl;
        return;
    }
    const int k = sc->iters + 1;   // which == 6: gamma1, delta of the new R
    sc->iters = k;
    sc->rr = g;
    if (hist) hist[k] = g;
    if (!isfinite(g)) { sc->rho = g; sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
    if (g == 0.0) { sc->rho = g; sc->converged = 1; sc->done = 1; return; }
    if (sc->rtol2 > 0.0 && g <= sc->rtol2 * sc->ref) { sc->rho = g; sc->converged = 1; sc->done = 1; return; }
    if (k >= sc->max_iters) {
        sc->rho = g;
        sc->done = 1;
        if (sc->rtol2 > 0.0) sc->status = TCA_NOT_CONVERGED;
        return;
    }
    const double beta = g / sc->rho;
    const double den = dl - beta * g / sc->alpha;
    sc->rho = g;
    if (!isfinite(den)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
    if (!(den > 0.0)) { sc->status = TCA_ERR_BREAKDOWN; sc->done = 1; return; }
    sc->beta = beta;
    sc->alpha = g / den;
}

void launch_cgsr_finalize(int which, const double *prr, int nrr, const double *prw, int nrw, CgScalars *sc,
                          double *hist, cudaStream_t s, int stage)
{
    count_launch();
    cgsr_finalize_kernel<<<1, stage == 2 ? 32 : kRedThreads, 0, s>>>(which, prr, nrr, prw, nrw, sc, hist, stage);
}

// ---------------------------------------------------------------- Kronecker-sum apply (Eq. 9)
// y = sum_d (mode-d lambda R_d) x for an operator without a Kronecker-product
// term (factor form, tca_operator_create_gram with G = NULL): one thread per
// output, the <= 5 taps of each mode from taps[(off_d + r) * 5 + k + 2]
// (zero outside the band and the domain); neighbour loads hit L1/L2.  One HBM
// read and one write per element (the separable Poisson stencil).
template <typename T>
__global__ void __launch_bounds__(256)
ksum_apply_kernel(const T *__restrict__ x, T *__restrict__ y, int64_t N, int n1, int n2, int n3, int n4,
                  const T *__restrict__ taps, int o1, int o2, int o3, int o4, const int32_t *done)
{
    if (done && *done) return;
    const int64_t s4 = 1, s3 = n4, s2 = (int64_t)n3 * n4, s1 = (int64_t)n2 * n3 * n4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = i;
        const int i4 = (int)(rem % n4); rem /= n4;
        const int i3 = (int)(rem % n3); rem /= n3;
        const int i2 = (int)(rem % n2); rem /= n2;
        const int i1 = (int)rem;
        T acc = T(0);
#pragma unroll
        for (int k = -2; k <= 2; ++k) {
            if (i1 + k >= 0 && i1 + k < n1) acc = fma(__ldg(taps + (int64_t)(o1 + i1) * 5 + k + 2), __ldg(x + i + k * s1), acc);
            if (i2 + k >= 0 && i2 + k < n2) acc = fma(__ldg(taps + (int64_t)(o2 + i2) * 5 + k + 2), __ldg(x + i + k * s2), acc);
            if (i3 + k >= 0 && i3 + k < n3) acc = fma(__ldg(taps + (int64_t)(o3 + i3) * 5 + k + 2), __ldg(x + i + k * s3), acc);
            if (i4 + k >= 0 && i4 + k < n4) acc = fma(__ldg(taps + (int64_t)(o4 + i4) * 5 + k + 2), __ldg(x + i + k * s4), acc);
        }
        y[i] = acc;
    }
}

template <typename T>
void launch_ksum_apply(const T *x, T *y, int64_t N, const int64_t *n, const T *taps, const int *off,
                       const int32_t *done, cudaStream_t s)
{
    count_launch();
    const int64_t blocks = std::min<int64_t>((N + 255) / 256, 148 * 16);
    ksum_apply_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(x, y, N, (int)n[0], (int)n[1], (int)n[2], (int)n[3], taps,
                                                          off[0], off[1], off[2], off[3], done);
}

// ---------------------------------------------------------------- tensor Jacobi (Fig. 1)
// E := InvMainDiag(A): diag[i] = prod_d G_d[i_d, i_d] + lambda sum_d R_d[i_d, i_d]
// from per-mode diagonals dg (4 x nmax, zero when there is no product term) and
// dr (4 x nmax, zero for modes without a regulariser).
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
jacobi_diag_kernel(T *__restrict__ e, int64_t N, int n1, int n2, int n3, int n4, const double *__restrict__ dg,
                   const double *__restrict__ dr, int nmax, double lam, int have_g)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = i;
        const int i4 = (int)(rem % n4); rem /= n4;
        const int i3 = (int)(rem % n3); rem /= n3;
        const int i2 = (int)(rem % n2); rem /= n2;
        const int i1 = (int)rem;
        const double pk = have_g ? dg[i1] * dg[nmax + i2] * dg[2 * nmax + i3] * dg[3 * nmax + i4] : 0.0;
        const double sm = dr[i1] + dr[nmax + i2] + dr[2 * nmax + i3] + dr[3 * nmax + i4];
        e[i] = (T)(1.0 / (pk + lam * sm));
    }
}

// R := Q - B (Q = A*U) with the R+*R partials
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
jacobi_resid_kernel(T *__restrict__ r, const T *__restrict__ q, const T *__restrict__ b, int64_t N, double *part,
                    const int32_t *done)
{
    if (done && *done) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = q[i] - b[i];
        r[i] = v;
        acc += (double)v * (double)v;
    }
    const double sm = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = sm;
}

// U := U - R*E
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
jacobi_update_kernel(T *__restrict__ u, const T *__restrict__ r, const T *__restrict__ e, int64_t N,
                     const CgScalars *sc)
{
    if (sc->done) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        u[i] = u[i] - r[i] * e[i];
}

// R+*R against the absolute threshold ("WHILE R+*R > threshold");
// which = 0 after the initial residual, 1 after each update
__global__ void __launch_bounds__(kRedThreads)
jacobi_finalize_kernel(int which, const double *__restrict__ part, int nparts, CgScalars *sc, double *hist)
{
    if (which == 1 && sc->done) return;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kRedThreads) acc += part[i];
    const double s = block_sum(acc);
    if (threadIdx.x != 0) return;
    int k = 0;
    if (which == 0) {
        sc->rho0 = s;
        sc->iters = 0;
        sc->status = TCA_OK;
        sc->converged = 0;
        sc->done = 0;
    } else {
        k = sc->iters + 1;
        sc->iters = k;
    }
    sc->rho = s;
    sc->rr = s;
    if (hist) hist[k] = s;
    if (!isfinite(s)) { sc->status = TCA_ERR_NONFINITE; sc->done = 1; return; }
    if (s <= sc->thr) { sc->converged = 1; sc->done = 1; return; }
    if (k >= sc->max_iters) { sc->status = TCA_NOT_CONVERGED; sc->done = 1; }
}

template <typename T>
void launch_jacobi_diag(T *e, int64_t N, const int64_t *n, const double *dg, const double *dr, int nmax, double lam,
                        bool have_g, cudaStream_t s)
{
    count_launch();
    jacobi_diag_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(e, N, (int)n[0], (int)n[1], (int)n[2], (int)n[3], dg, dr,
                                                              nmax, lam, have_g ? 1 : 0);
}

template <typename T>
void launch_jacobi_resid(T *r, const T *q, const T *b, int64_t N, double *part, const int32_t *done, cudaStream_t s)
{
    count_launch();
    jacobi_resid_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(r, q, b, N, part, done);
}

template <typename T>
void launch_jacobi_update(T *u, const T *r, const T *e, int64_t N, const CgScalars *sc, cudaStream_t s)
{
    count_launch();
    jacobi_update_kernel<T><<<kRedBlocks, kRedThreads, 0, s>>>(u, r, e, N, sc);
}

void launch_jacobi_finalize(int which, const double *part, int nparts, CgScalars *sc, double *hist, cudaStream_t s)
{
    count_launch();
    jacobi_finalize_kernel<<<1, kRedThreads, 0, s>>>(which, part, nparts, sc, hist);
}

void launch_cg_finalize(int which, const double *part, int nparts, CgScalars *sc, double *hist,
                        cudaStream_t s, int stage)
{
    count_launch();
    cg_finalize_kernel<<<1, stage == 2 ? 32 : kRedThreads, 0, s>>>(which, part, nparts, sc, hist, stage);
}

// ---------------------------------------------------------------- instantiations
#define TCA_INST(T)                                                                       \
    template bool launch_band_win_last<T>(const T *, T *, int64_t, int, const BandMat &,   \
                                          const BandMat &, cudaStream_t);                 \
    template bool launch_band_plane2<T>(const T *, T *, int64_t, int, int, const BandMat &, \
                                        const BandMat &, cudaStream_t);                   \
    template void launch_band_mode_product<T>(const T *, T *, int64_t, const BandMat &,    \
                                              int64_t, double, bool, const int32_t *,     \
                                              cudaStream_t);                              \
    template void launch_gen_normal<T>(T *, int64_t, int64_t, uint64_t, double, bool,     \
                                       cudaStream_t);                                     \
    template void launch_cg_init<T>(const T *, T *, T *, T *, int64_t, double *,          \
                                    cudaStream_t);                                        \
    template void launch_resid2<T>(const T *, const T *, T *, T *, int64_t, double *,      \
                                   double *, cudaStream_t);                               \
    template void launch_dot_partials<T>(const T *, const T *, int64_t, double *,         \
                                         const int32_t *, cudaStream_t);                  \
    template void launch_cg_update_r<T>(T *, const T *, int64_t, CgScalars *, double *,   \
                                        cudaStream_t, bool, double *);                    \
    template void launch_cg_update_xp<T>(T *, T *, const T *, int64_t, const CgScalars *, \
                                         cudaStream_t);                                   \
    template void launch_cg_update_p<T>(T *, const T *, const T *, int64_t,               \
                                        const CgScalars *, cudaStream_t);                 \
    template void launch_cgsr_update<T>(T *, T *, T *, T *, const T *, int64_t,            \
                                        const CgScalars *, double *, cudaStream_t);       \
    template void launch_ksum_apply<T>(const T *, T *, int64_t, const int64_t *, const T *, \
                                       const int *, const int32_t *, cudaStream_t);       \
    template void launch_jacobi_diag<T>(T *, int64_t, const int64_t *, const double *,     \
                                        const double *, int, double, bool, cudaStream_t); \
    template void launch_jacobi_resid<T>(T *, const T *, const T *, int64_t, double *,     \
                                         const int32_t *, cudaStream_t);                  \
    template void launch_jacobi_update<T>(T *, const T *, const T *, int64_t,              \
                                          const CgScalars *, cudaStream_t);

TCA_INST(double)
TCA_INST(float)

}  // namespace tca
