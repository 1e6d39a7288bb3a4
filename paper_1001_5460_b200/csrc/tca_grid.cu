// tca_grid.cu -- whole-solve CG engine for mid-size problems.
//
// Fig. 2 as ONE persistent cooperative kernel (one block per
// SM, all co-resident) whose phases are separated by grid-wide barriers, for
// problems too large for the single-block engine (tca_tiny.cu) but small enough
// that the vectors stay in L2 (config 1: 48^3 unknowns, dense Gaussian modes;
// config 2: 32^3 x 16).  On the general engine such a solve is ~10 kernel
// launches per iteration (graph-replayed), 50-110 us per iteration of latency
// for a few microseconds of work.
//
// Vectors live in global memory (L2-resident); every load of a vector written
// inside the kernel bypasses L1 (ld.global.cg), so a CTA never reads a stale
// line another SM wrote before the last barrier.  An iteration, D = order:
//   phase 0 (mode D, fibres along i_D):   P := R + beta P_old   (P ping-pongs,
//            so neighbours still read P_old), T = G_D x_D P, Q = lambda R_D x_D P
//   phase k (mode D-k):                   T' = G x T, Q += lambda R x P
//   last    (mode 1):                     Q += G_1 x_1 T + lambda R_1 x_1 P,
//                                          <P, Q> partials
//   update:                               alpha; C += alpha P, R -= alpha Q,
//                                          <R, R> partials; rho1, stop, beta
// = D + 1 grid barriers per iteration (Eq. 4's successive mode products,
// PAPER.md:68-73, and Eq. 9's Kronecker-sum regulariser).
// Each phase works on tiles of F whole fibres of its mode: the tile is staged
// in shared memory and every output row is a band (or dense) row of the mode's
// matrix, whose table is in shared memory for the whole solve.
// Same semantics as cg_t / cg_iteration (tca_abi.cu): readings Z1-Z3, Z10,
// Z12, Z28, the guards, the rho history, warm start.
#include "tca_internal.cuh"

namespace tca {

namespace {

// block size (grid_threads): 512 threads, or 1024 when a block owns >= 2048
// elements per phase (config 2: 43.2 -> 39.2 us per iteration; config 1 with
// 747 elements per block: 20.7 at 512 vs 26.1 us at 1024 -- the extra warps
// only lengthen the block barriers)
constexpr size_t kGridSmem = 200 * 1024;
constexpr int kMaxF = 1024;
constexpr size_t kTileBudget = 150 * 1024;   // S + P fibre tiles

struct GridMode {
    int n, inner;
    int64_t outer;       // N / (n * inner)
    int F, lgF, ftiles;  // fibres per tile (a power of two), its log2, tiles of this mode's phase
    int gW, rW;          // taps per row (rW = 0: no regulariser)
    int gP, rP;          // shared-memory row pitches of the tables (odd: lanes on different rows hit different banks)
    int dense_mma;       // fp64 dense G with n, F multiples of 8 and one 8 x 8 output tile per warp: DMMA
    int fb_off;          // byte offset of this block's precomputed fibre bases (-1: computed per tile)
    int fb_tpb;          // tiles per block covered by the precomputed table
    int g_off, r_off;    // byte offsets of the tables in shared memory
    int gs_off, rs_off;  // byte offsets of the row starts (int)
    const void *gt, *rt;
    const int *gs, *rs;
};

struct GridArgs {
    const void *b;
    void *x;              // C (in: warm start; out: solution)
    void *r, *q, *t0, *t1;
    void *p0, *p1;        // P ping-pong
    double *part;         // 2 x gridDim partials
    unsigned *bar;        // [0] arrivals, [1] generation
    CgScalars *sc;
    double *hist;
    int x0_zero;
    int64_t N;
    int order;
    int tile_off;         // byte offset of the fibre tiles in shared memory
    // fused first phase (modes D-1 and D on whole planes, D >= 2): planes of
    // na x nc elements, PT planes per tile, odd pitches
    int fuse2, na, nc, PT, ptiles, pc, pz;
    int64_t planes;
    int dbg;              // measurement switches (TCA_GRID_DBG): 1 skip the fibre phases, 2 the update loop, 4 the phases' arithmetic, 8 their loads
    double lambda;
    GridMode md[kD];
};

__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// D(8x8) += A(8x4) B(4x8) on the FP64 tensor cores (fragment layout of mma.sync m8n8k4)
__device__ __forceinline__ void grid_dmma884(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ float ldcg(const float *p) { return __ldcg(p); }

// Grid-wide barrier (all blocks co-resident: cooperative launch): one atomic
// per block on a counter whose top bit flips when the last block arrives
// (block 0 adds 2^31 - (grid - 1), the others 1), then a spin on that bit.
// The counter never needs a reset.
__device__ __forceinline__ void grid_sync(unsigned *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        unsigned old, cur;
        // release: this block's writes (ordered before it by the CTA barrier) are
        // visible to any block that acquires the flipped counter
        asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
    }
    __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double *red)
{
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) v += __shfl_xor_sync(0xffffffffu, v, k);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int k = 16; k > 0; k >>= 1) s += __shfl_xor_sync(0xffffffffu, s, k);
    }
    return s;   // valid in thread 0
}

// every block: the sum of the gridDim partials in a fixed order (same value
// everywhere).  (A single-warp variant, 5 partials per lane, measured slower:
// 21.4 vs 20.7 us per config-1 iteration.)
__device__ __forceinline__ double grid_total(const double *part, double *red)
{
    double v = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += __ldcg(part + i);
    v = block_sum(v, red);
    __syncthreads();
    if (threadIdx.x == 0) red[32] = v;
    __syncthreads();
    return red[32];
}

// sum_w tp[w] col[(s0 + w) * F] over the columns inside [0, n) (taps outside are
// zero).  WC > 0: compile-time width (the banded forms, unrolled); WC = 0: any
// width (dense rows), four independent chains.  Rows whose window lies inside
// the fibre take the unchecked loop.
template <int WC, typename T>
__device__ __forceinline__ T band_row(const T *tp, int s0, int Wrt, int n, const T *col, int F)
{
    const int W = WC > 0 ? WC : Wrt;
    if (s0 >= 0 && s0 + W <= n) {
        const T *c = col + s0 * F;
        if (WC > 0) {
            T a0 = T(0), a1 = T(0);
#pragma unroll
            for (int w = 0; w < WC; ++w) {
                if (w & 1) a1 = fma(tp[w], c[w * F], a1);
                else a0 = fma(tp[w], c[w * F], a0);
            }
            return a0 + a1;
        }
        T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
        int w = 0;
        for (; w + 3 < W; w += 4) {
            a0 = fma(tp[w], c[w * F], a0);
            a1 = fma(tp[w + 1], c[(w + 1) * F], a1);
            a2 = fma(tp[w + 2], c[(w + 2) * F], a2);
            a3 = fma(tp[w + 3], c[(w + 3) * F], a3);
        }
        for (; w < W; ++w) a0 = fma(tp[w], c[w * F], a0);
        return (a0 + a1) + (a2 + a3);
    }
    T a0 = T(0);
    for (int w = 0; w < W; ++w) {
        const int cc = s0 + w;
        if (cc >= 0 && cc < n) a0 = fma(tp[w], col[cc * F], a0);
    }
    return a0;
}

template <typename T>
__device__ __forceinline__ T band_row_any(const T *tp, int s0, int W, int n, const T *col, int F)
{
    switch (W) {
    case 3: return band_row<3>(tp, s0, W, n, col, F);
    case 5: return band_row<5>(tp, s0, W, n, col, F);
    case 7: return band_row<7>(tp, s0, W, n, col, F);
    case 9: return band_row<9>(tp, s0, W, n, col, F);
    default: return band_row<0>(tp, s0, W, n, col, F);
    }
}

// One phase over the fibres of mode m: for every fibre tile,
//   stage S = src fibres (S = P_old/R -> P when first), optional PS = P fibres
//   dst[r] = sum_w G[r, w] S[start_r + w]           (dst != nullptr)
//   q[r] (+)= lambda sum_w R[r, w] P[start_r + w] (+ G... when last)
template <typename T>
__device__ void fibre_phase(const GridArgs &a, const unsigned char *sm, T *tile, int m, bool first, bool last,
                            const T *src, T *dst, const T *pn_in, T *pn_out, T beta, double &pq)
{
    const GridMode &md = a.md[m];
    const int n = md.n, F = md.F, PF = F + 1;   // odd pitch: conflict-free along f and along c
    const int inner = md.inner;
    T *S = tile;                  // [n][PF] staged input fibres
    T *PS = S + n * PF;           // [n][PF] P fibres (regulariser, <p, q>, first-phase P)
    T *QS = PS + n * PF;          // [n][PF] Q accumulated by the earlier phases
    int *fbase = reinterpret_cast<int *>(QS + n * PF);   // [F] fibre base offsets
    const int lgF = md.lgF;
    const bool cfast = inner == 1;   // fibres contiguous: element order c-fastest (coalesced)
    const float inv_n = 1.0f / (float)n;
    const T *gt = reinterpret_cast<const T *>(sm + md.g_off);
    const int *gs = reinterpret_cast<const int *>(sm + md.gs_off);
    const T *rt = reinterpret_cast<const T *>(sm + md.r_off);
    const int *rs = reinterpret_cast<const int *>(sm + md.rs_off);
    const T *pold = (const T *)(first ? pn_in : nullptr);
    const T *rv = (const T *)a.r;
    T *q = (T *)a.q;
    const T lam = (T)a.lambda;
    const int nfib = (int)(md.outer * inner);
    const int nel = n * F;
    const bool need_p = first || md.rW > 0 || last;
    const bool need_q = !first && (md.rW > 0 || last);
    const int *fpre = md.fb_off >= 0 ? reinterpret_cast<const int *>(sm + md.fb_off) : nullptr;
    for (int ti = blockIdx.x, kt = 0; ti < md.ftiles; ti += gridDim.x, ++kt) {
        __syncthreads();   // previous tile's reads of the tiles / fbase done
        if (fpre) {        // fibre bases precomputed at kernel start (the same every iteration)
            fbase = const_cast<int *>(fpre) + kt * F;
        } else {
            for (int f = threadIdx.x; f < F; f += blockDim.x) {
                const int fid = ti * F + f;
                if (fid < nfib) {
                    const int o = fid / inner, t = fid - o * inner;
                    fbase[f] = o * n * inner + t;
                } else {
                    fbase[f] = -1;
                }
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < nel; e += blockDim.x) {
            int c, f;
            if (cfast) { f = (int)(((float)e + 0.5f) * inv_n); c = e - f * n; }
            else { c = e >> lgF; f = e & (F - 1); }
            const int fb = fbase[f];
            T sv = T(0), pv = T(0), qv = T(0);
            if (fb >= 0 && !(a.dbg & 8)) {
                const int g = fb + c * inner;
                if (first) {   // P := R + beta P_old, written by the (unique) owner of this element
                    pv = fma(beta, ldcg(pold + g), ldcg(rv + g));
                    pn_out[g] = pv;
                    sv = pv;
                } else {
                    sv = ldcg(src + g);
                    if (need_p) pv = ldcg(pn_in + g);
                    if (need_q) qv = ldcg(q + g);
                }
            }
            S[c * PF + f] = sv;
            PS[c * PF + f] = pv;
            QS[c * PF + f] = qv;
        }
        __syncthreads();
        bool mma = false;
        if constexpr (sizeof(T) == 8) {
            // dense G on the FP64 tensor cores: warp w computes the 8 x 8 output
            // tile w of G S (K = n in steps of 4), written back over S
            if (md.dense_mma && !(a.dbg & 4)) {
                mma = true;
                const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nrt = n >> 3;
                const bool mine = warp < nrt * (F >> 3);
                const int r0 = (warp % nrt) * 8, f0 = (warp / nrt) * 8;
                double d0 = 0.0, d1 = 0.0;
                if (mine) {
                    const double *ga = reinterpret_cast<const double *>(gt) + (r0 + (lane >> 2)) * md.gP + (lane & 3);
                    const double *sb = reinterpret_cast<const double *>(S) + (lane & 3) * PF + f0 + (lane >> 2);
                    for (int k = 0; k < n; k += 4) grid_dmma884(d0, d1, ga[k], sb[k * PF]);
                }
                __syncthreads();   // every warp has read S
                if (mine) {
                    double *o = reinterpret_cast<double *>(S) + (r0 + (lane >> 2)) * PF + f0 + 2 * (lane & 3);
                    o[0] = d0;
                    o[1] = d1;
                }
                __syncthreads();
            }
        }
        for (int e = threadIdx.x; e < nel && !(a.dbg & 4); e += blockDim.x) {
            int r, f;
            if (cfast) { f = (int)(((float)e + 0.5f) * inv_n); r = e - f * n; }
            else { r = e >> lgF; f = e & (F - 1); }
            const int fb = fbase[f];
            if (fb < 0) continue;
            const int g = fb + r * inner;
            const T acc = mma ? S[r * PF + f] : band_row_any(gt + r * md.gP, gs[r], md.gW, n, S + f, PF);
            const T reg = md.rW > 0 ? band_row_any(rt + r * md.rP, rs[r], md.rW, n, PS + f, PF) : T(0);
            if (last) {   // Q += G_1 T + lambda R_1 P (or, D = 1: Q = G P + lambda R P)
                const T qv = QS[r * PF + f] + fma(lam, reg, acc);
                q[g] = qv;
                pq += (double)PS[r * PF + f] * (double)qv;
            } else {
                dst[g] = acc;
                if (first) q[g] = lam * reg;
                else if (md.rW > 0) q[g] = fma(lam, reg, QS[r * PF + f]);
            }
        }
    }
}

// First phase on whole (i_{D-1}, i_D) planes (both fastest modes in one phase):
//   P := R + beta P_old (own elements), Z = G_D x_D P, RQ = lambda R_D x_D P,
//   T = G_{D-1} x_{D-1} Z, Q = RQ + lambda R_{D-1} x_{D-1} P   (D > 2: T -> dst)
//   D == 2 (last): Q += T, <P, Q> partials
template <typename T>
__device__ void plane_phase(const GridArgs &a, const unsigned char *sm, T *tile, bool last, const T *pold, T *pn,
                            T beta, T *dst, double &pq)
{
    const GridMode &ma = a.md[a.order - 2], &mc = a.md[a.order - 1];
    const int na = a.na, nc = a.nc, PT = a.PT, pc = a.pc, pz = a.pz;
    const int pl = na * nc;
    T *S = tile;                        // [PT][na][pc] P
    T *Z = S + (size_t)PT * na * pc;    // [PT][na][pz] G_D P
    T *RQ = Z + (size_t)PT * na * pz;   // [PT][na][pz] lambda R_D P
    const T *gtc = reinterpret_cast<const T *>(sm + mc.g_off), *gta = reinterpret_cast<const T *>(sm + ma.g_off);
    const int *gsc = reinterpret_cast<const int *>(sm + mc.gs_off), *gsa = reinterpret_cast<const int *>(sm + ma.gs_off);
    const T *rtc = reinterpret_cast<const T *>(sm + mc.r_off), *rta = reinterpret_cast<const T *>(sm + ma.r_off);
    const int *rsc = reinterpret_cast<const int *>(sm + mc.rs_off), *rsa = reinterpret_cast<const int *>(sm + ma.rs_off);
    const T *rv = (const T *)a.r;
    T *q = (T *)a.q;
    const T lam = (T)a.lambda;
    const float inv_nc = 1.0f / (float)nc, inv_pl = 1.0f / (float)pl;
    const int nel = PT * pl;
    for (int ti = blockIdx.x; ti < a.ptiles; ti += gridDim.x) {
        const int64_t o0 = (int64_t)ti * PT;
        const int np = (int)min((int64_t)PT, a.planes - o0);
        const int ne = np * pl;
        __syncthreads();   // previous tile's reads done
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {   // contiguous: the tile's planes are one run
            const int pp = (int)(((float)e + 0.5f) * inv_pl), w = e - pp * pl;
            const int ai = (int)(((float)w + 0.5f) * inv_nc), ci = w - ai * nc;
            const int64_t g = o0 * pl + e;
            T pv = T(0);
            if (!(a.dbg & 8)) pv = fma(beta, ldcg(pold + g), ldcg(rv + g));
            pn[g] = pv;
            S[((size_t)pp * na + ai) * pc + ci] = pv;
        }
        __syncthreads();
        // stage 1: mode D along the contiguous index
        for (int e = threadIdx.x; e < ne && !(a.dbg & 4); e += blockDim.x) {
            const int pp = (int)(((float)e + 0.5f) * inv_pl), w = e - pp * pl;
            const int ai = (int)(((float)w + 0.5f) * inv_nc), j = w - ai * nc;
            const T *row = S + ((size_t)pp * na + ai) * pc;
            Z[((size_t)pp * na + ai) * pz + j] = band_row_any(gtc + j * mc.gP, gsc[j], mc.gW, nc, row, 1);
            RQ[((size_t)pp * na + ai) * pz + j] =
                mc.rW > 0 ? lam * band_row_any(rtc + j * mc.rP, rsc[j], mc.rW, nc, row, 1) : T(0);
        }
        __syncthreads();
        // stage 2: mode D-1
        for (int e = threadIdx.x; e < ne && !(a.dbg & 4); e += blockDim.x) {
            const int pp = (int)(((float)e + 0.5f) * inv_pl), w = e - pp * pl;
            const int i = (int)(((float)w + 0.5f) * inv_nc), j = w - i * nc;
            const T *zc = Z + (size_t)pp * na * pz + j;
            const T t = band_row_any(gta + i * ma.gP, gsa[i], ma.gW, na, zc, pz);
            T qv = RQ[((size_t)pp * na + i) * pz + j];
            if (ma.rW > 0) qv = fma(lam, band_row_any(rta + i * ma.rP, rsa[i], ma.rW, na, S + (size_t)pp * na * pc + j, pc), qv);
            const int64_t g = o0 * pl + e;
            if (last) {
                qv += t;
                pq += (double)S[((size_t)pp * na + i) * pc + j] * (double)qv;
            } else {
                dst[g] = t;
            }
            q[g] = qv;
        }
    }
}

// The operator phases of one iteration (Q := A P, P := R + beta P_old formed on
// the way), D - 1 grid barriers inside (with the fused first phase D - 2); the
// caller synchronises after.  pq: this thread's <P, Q> partial.
template <typename T>
__device__ void operator_phases(const GridArgs &a, const unsigned char *sm, T *tile, T *pold, T *pn, T beta,
                                T *const *tb, double &pq)
{
    const int D = a.order;
    if (a.fuse2) {
        plane_phase<T>(a, sm, tile, D == 2, pold, pn, beta, tb[0], pq);
        for (int k = 2; k < D; ++k) {   // modes D-2 .. 1 (0-based D-1-k)
            grid_sync(a.bar);
            const int j = k - 2;
            fibre_phase<T>(a, sm, tile, D - 1 - k, false, k == D - 1, tb[j & 1], tb[(j + 1) & 1], pn, pn, beta, pq);
        }
        return;
    }
    for (int k = 0; k < D; ++k) {
        if (k > 0) grid_sync(a.bar);
        fibre_phase<T>(a, sm, tile, D - 1 - k, k == 0, k == D - 1, k == 0 ? nullptr : tb[(k - 1) & 1], tb[k & 1],
                       k == 0 ? pold : pn, pn, beta, pq);
    }
}

template <typename T, int NT>
__global__ void __launch_bounds__(NT, 1) grid_cg_kernel(const __grid_constant__ GridArgs a)
{
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[40];
    const int D = a.order;
    const int64_t N = a.N;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gstride = (int64_t)gridDim.x * blockDim.x;
    // ---- tap tables -> shared memory (start offsets as stored)
    for (int d = 0; d < D; ++d) {
        const GridMode &m = a.md[d];
        T *g = reinterpret_cast<T *>(sm + m.g_off);
        for (int i = threadIdx.x; i < m.n * m.gW; i += blockDim.x) g[(i / m.gW) * m.gP + i % m.gW] = ((const T *)m.gt)[i];
        int *gs = reinterpret_cast<int *>(sm + m.gs_off);
        for (int i = threadIdx.x; i < m.n; i += blockDim.x) gs[i] = m.gs[i];
        if (m.rW > 0) {
            T *rr = reinterpret_cast<T *>(sm + m.r_off);
            for (int i = threadIdx.x; i < m.n * m.rW; i += blockDim.x) rr[(i / m.rW) * m.rP + i % m.rW] = ((const T *)m.rt)[i];
            int *rs = reinterpret_cast<int *>(sm + m.rs_off);
            for (int i = threadIdx.x; i < m.n; i += blockDim.x) rs[i] = m.rs[i];
        }
    }
    // fibre bases of this block's tiles, per mode (constant for the whole solve)
    for (int d = 0; d < D; ++d) {
        const GridMode &m = a.md[d];
        if (m.fb_off < 0) continue;
        int *fp = reinterpret_cast<int *>(sm + m.fb_off);
        const int nfib = (int)(m.outer * m.inner);
        for (int e = threadIdx.x; e < m.fb_tpb * m.F; e += blockDim.x) {
            const int kt = e / m.F, f = e - kt * m.F;
            const int ti = blockIdx.x + kt * (int)gridDim.x;
            const int fid = ti * m.F + f;
            if (ti < m.ftiles && fid < nfib) {
                const int o = fid / m.inner, t = fid - o * m.inner;
                fp[e] = o * m.n * m.inner + t;
            } else {
                fp[e] = -1;
            }
        }
    }
    T *tile = reinterpret_cast<T *>(sm + a.tile_off);
    const T *b = (const T *)a.b;
    T *x = (T *)a.x, *r = (T *)a.r, *q = (T *)a.q;
    T *pb[2] = {(T *)a.p0, (T *)a.p1};
    T *tb[2] = {(T *)a.t0, (T *)a.t1};
    double *part = a.part;
    CgScalars *sc = a.sc;
    const double rtol2 = sc->rtol2;
    const int max_iters = sc->max_iters;
    // ---- start: R := B - A*C (warm start: one apply of C through the phases), P_old := 0
    double rr = 0.0, bb = 0.0;
    if (!a.x0_zero) {
        for (int64_t i = gtid; i < N; i += gstride) {
            r[i] = x[i];        // phase 0 forms P := R + 0 * P_old = C
            pb[0][i] = T(0);
        }
        grid_sync(a.bar);
        double dummy = 0.0;
        operator_phases<T>(a, sm, tile, pb[0], pb[1], T(0), tb, dummy);
        grid_sync(a.bar);
        for (int64_t i = gtid; i < N; i += gstride) {   // Q = A*C
            const T bi = b[i], ri = T(bi - ldcg(q + i));
            r[i] = ri;
            pb[0][i] = T(0);
            rr += (double)ri * (double)ri;
            bb += (double)bi * (double)bi;
        }
    } else {
        for (int64_t i = gtid; i < N; i += gstride) {
            const T bi = b[i];
            x[i] = T(0);
            r[i] = bi;
            pb[0][i] = T(0);
            rr += (double)bi * (double)bi;
        }
    }
    double v = block_sum(rr, red);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
    v = block_sum(bb, red);
    if (threadIdx.x == 0) part[gridDim.x + blockIdx.x] = v;
    grid_sync(a.bar);
    double rho = grid_total(part, red);
    const double ref = a.x0_zero ? rho : grid_total(part + gridDim.x, red);   // stop reference <b, b> (Z28)
    const double rho0 = rho;
    double rho_last = rho;
    int status = TCA_OK, converged = 0, iters = 0;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (lead && a.hist) a.hist[0] = rho;
    bool done = false;
    if (!isfinite(rho)) { status = TCA_ERR_NONFINITE; done = true; }
    else if (rho == 0.0) { converged = 1; done = true; }
    else if (max_iters <= 0) { done = true; if (rtol2 > 0.0) status = TCA_NOT_CONVERGED; }
    T beta = T(0);
    int cur = 0;   // P_old in pb[cur], P in pb[cur ^ 1]
    bool first_it = true;
    while (!done) {
        // part[0, grid) (the <p, q> partials) is rewritten below: every block must
        // have read the start reductions.  Later iterations pass D - 1 >= 1 phase
        // barriers and the <r, r> barrier between two uses of a partial buffer.
        if (first_it || D == 1) grid_sync(a.bar);
        first_it = false;
        double pq = 0.0;
        T *pn = pb[cur ^ 1];
        if (!(a.dbg & 1)) operator_phases<T>(a, sm, tile, pb[cur], pn, beta, tb, pq);
        if (a.dbg & 13) pq = 1.0;
        pq = block_sum(pq, red);
        if (threadIdx.x == 0) part[blockIdx.x] = pq;
        grid_sync(a.bar);
        pq = grid_total(part, red);                        // P+*Q
        if (!isfinite(pq)) { status = TCA_ERR_NONFINITE; break; }
        if (!(pq > 0.0)) { status = TCA_ERR_BREAKDOWN; break; }
        const T alpha = (T)(rho / pq);
        double r1 = (a.dbg & 2) ? rho * 0.5 : 0.0;
        for (int64_t i = gtid; i < N && !(a.dbg & 2); i += gstride) {
            const T pv = ldcg(pn + i);
            x[i] = fma(alpha, pv, x[i]);                      // C := C + alpha*P*D
            const T ri = fma(-alpha, ldcg(q + i), r[i]);       // R := R - alpha*Q
            r[i] = ri;
            r1 += (double)ri * (double)ri;
        }
        r1 = block_sum(r1, red);
        if (threadIdx.x == 0) part[gridDim.x + blockIdx.x] = r1;
        grid_sync(a.bar);
        const double rho1 = grid_total(part + gridDim.x, red);   // rho1 := R+*R
        iters += 1;
        rho_last = rho1;
        if (lead && a.hist) a.hist[iters] = rho1;
        if (!isfinite(rho1)) { status = TCA_ERR_NONFINITE; break; }
        if (rho1 == 0.0) { converged = 1; break; }                         // Z12
        if (rtol2 > 0.0 && rho1 <= rtol2 * ref) { converged = 1; break; }  // Z1, Z2, Z28
        if (iters >= max_iters) { if (rtol2 > 0.0) status = TCA_NOT_CONVERGED; break; }
        beta = (T)(rho1 / rho);
        rho = rho1;
        cur ^= 1;
    }
    if (lead) {
        sc->rho = rho_last;
        sc->rr = rho_last;
        sc->rho0 = rho0;
        sc->ref = ref;
        sc->iters = iters;
        sc->converged = converged;
        sc->status = status;
        sc->done = 1;
    }
}

int grid_threads(const tca_operator *op)
{
    return op->N / op->num_sms >= 2048 ? 1024 : 512;
}

// shared-memory plan and the per-mode tiling; 0 when not eligible
size_t grid_plan(const tca_operator *op, int grid, GridArgs *out)
{
    GridArgs a{};
    a.order = op->order;
    a.N = op->N;
    a.lambda = op->lambda;
    const size_t es = op->esize;
    size_t off = 0;
    int64_t inner = 1;
    size_t tile_max = 0;
    for (int d = op->order - 1; d >= 0; --d) {
        GridMode &m = a.md[d];
        m.n = (int)op->n[d];
        m.inner = (int)inner;
        m.outer = op->N / ((int64_t)m.n * inner);
        const int64_t nfib = m.outer * inner;
        // the fewest tile rounds per block: the widest power-of-two tile within
        // the shared-memory budget that still gives every block a tile (a phase
        // is then as few load round trips + compute passes per block as fit)
        int F = kMaxF, lg = 10;
        auto tile_bytes = [&](int f) { return 3 * (size_t)m.n * (f + 1) * es + 4 * (size_t)f; };
        while (F > 1 && ((nfib + F - 1) / F < grid || tile_bytes(F) > kTileBudget)) {
            F >>= 1;
            --lg;
        }
        m.F = F;
        m.lgF = lg;
        m.ftiles = (int)((nfib + F - 1) / F);
        tile_max = std::max(tile_max, tile_bytes(F));
        const BandMat &g = op->Gm[d];
        static const bool no_mma = getenv("TCA_GRID_NOMMA") != nullptr;   // measurement switch
        m.dense_mma = !no_mma && es == 8 && g.dense && m.n % 8 == 0 && F % 8 == 0 &&
                      (m.n / 8) * (F / 8) <= grid_threads(op) / 32;
        m.gW = g.W;
        m.gP = g.W | 1;
        m.gt = g.taps;
        m.gs = g.start;
        m.g_off = (int)off;
        off += (size_t)m.n * m.gP * es;
        m.gs_off = (int)off;
        off += (size_t)m.n * sizeof(int);
        off = (off + 15) & ~(size_t)15;
        if (op->has_reg[d]) {
            const BandMat &rm = op->Rm[d];
            m.rW = rm.W;
            m.rP = rm.W | 1;
            m.rt = rm.taps;
            m.rs = rm.start;
            m.r_off = (int)off;
            off += (size_t)m.n * m.rP * es;
            m.rs_off = (int)off;
            off += (size_t)m.n * sizeof(int);
            off = (off + 15) & ~(size_t)15;
        }
        inner *= m.n;
    }
    // fuse the two fastest modes when a plane (three arrays) fits the tile budget
    static const bool no_fuse = getenv("TCA_GRID_NOFUSE") != nullptr;   // measurement switch
    if (op->order >= 2 && !no_fuse) {
        const int na = (int)op->n[op->order - 2], nc = (int)op->n[op->order - 1];
        const int pc = nc | 1, pz = nc | 1;
        auto pbytes = [&](int pt) { return (size_t)pt * na * (pc + 2 * pz) * es; };
        const int64_t planes = op->N / ((int64_t)na * nc);
        // only with a plane for every block: fewer, larger tiles lose more to
        // the idle blocks than the saved phase (config 1: 48 planes, 30.5 vs
        // 24.7 us per iteration; config 2: 1024 planes, 44.3 vs 50.8 us)
        if (pbytes(1) <= kTileBudget && planes >= grid) {
            int PT = 1;
            while (PT < 64 && pbytes(2 * PT) <= kTileBudget && (planes + PT - 1) / PT > grid) PT *= 2;
            a.fuse2 = 1;
            a.na = na;
            a.nc = nc;
            a.PT = PT;
            a.pc = pc;
            a.pz = pz;
            a.planes = planes;
            a.ptiles = (int)((planes + PT - 1) / PT);
            tile_max = std::max(tile_max, pbytes(PT));
        }
    }
    // precomputed fibre-base tables (when small): tiles per block x F ints per mode
    {
        size_t fb_total = 0;
        for (int d = 0; d < op->order; ++d) {
            const GridMode &m = a.md[d];
            fb_total += (size_t)((m.ftiles + grid - 1) / grid) * m.F * sizeof(int);
        }
        const bool pre = fb_total <= 32 * 1024;
        for (int d = 0; d < op->order; ++d) {
            GridMode &m = a.md[d];
            m.fb_off = -1;
            if (!pre) continue;
            m.fb_tpb = (m.ftiles + grid - 1) / grid;
            m.fb_off = (int)off;
            off += (size_t)m.fb_tpb * m.F * sizeof(int);
            off = (off + 15) & ~(size_t)15;
        }
    }
    a.tile_off = (int)off;
    off += tile_max;
    if (out) *out = a;
    return off;
}

int grid_blocks(const tca_operator *op)
{
    return op->num_sms;   // one block per SM (cooperative: all co-resident)
}

template <typename T>
tca_status launch_t(tca_operator *op, const void *b, void *x, int x0_zero, cudaStream_t s, bool *launched)
{
    *launched = false;
    const int grid = grid_blocks(op);
    GridArgs a{};
    const size_t smem = grid_plan(op, grid, &a);
    if (!op->grid_ws) {   // t1, second P buffer, partials, barrier words
        const size_t vb = (size_t)op->N * op->esize;
        op->grid_ws_bytes = 2 * vb + 2 * (size_t)grid * sizeof(double) + 64;
        TCA_CUDA_TRY(cudaMallocAsync(&op->grid_ws, op->grid_ws_bytes, s));
        TCA_CUDA_TRY(cudaMemsetAsync(op->grid_ws, 0, op->grid_ws_bytes, s));
        op->device_bytes += op->grid_ws_bytes;
    }
    char *w = (char *)op->grid_ws;
    const size_t vb = (size_t)op->N * op->esize;
    a.b = b;
    a.x = x;
    a.r = op->r;
    a.q = op->q;
    a.t0 = op->t0 ? op->t0 : nullptr;
    a.p0 = op->p_own;
    a.p1 = w;
    a.t1 = w + vb;
    a.part = (double *)(w + 2 * vb);
    a.bar = (unsigned *)(w + 2 * vb + 2 * (size_t)grid * sizeof(double));
    a.sc = op->sc;
    a.hist = op->hist;
    a.x0_zero = x0_zero;
    static const int dbg = getenv("TCA_GRID_DBG") ? atoi(getenv("TCA_GRID_DBG")) : 0;
    a.dbg = dbg;
    if (!a.t0) {
        TCA_CUDA_TRY(cudaMallocAsync(&op->t0, vb, s));
        TCA_CUDA_TRY(cudaMallocAsync(&op->t1, vb, s));
        op->device_bytes += 2 * vb;
        a.t0 = op->t0;
    }
    const int nt = grid_threads(op);
    const void *kern = nt == 1024 ? (const void *)grid_cg_kernel<T, 1024> : (const void *)grid_cg_kernel<T, 512>;
    TCA_TRY(set_max_dynamic_smem(kern, smem));
    // every block must be co-resident (the grid barrier spins): otherwise (a
    // shared or partitioned GPU) the caller runs the general engine
    int per_sm = 0;
    TCA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
    if (per_sm * op->num_sms < grid) return TCA_OK;
    void *args[] = {(void *)&a};
    const cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(nt), args, smem, s);
    if (e == cudaErrorCooperativeLaunchTooLarge) {
        cudaGetLastError();
        return TCA_OK;
    }
    TCA_CUDA_TRY(e);
    count_launch();
    *launched = true;
    return TCA_OK;
}

}  // namespace

bool grid_cg_eligible(const tca_operator *op)
{
    const char *e = getenv("TCA_GRID");   // read per call: tests pin the general path per operator   // measurement switch: TCA_GRID=0 keeps the general path
    if (e && e[0] == '0') return false;
    if (op->transport || op->scat || op->apply_path == 2 || op->order < 1) return false;
    if (op->N > (int64_t)1 << 21) return false;   // vectors stay L2-resident (8 x 16 MB fp64)
    for (int d = 0; d < op->order; ++d)
        if (!op->Gm[d].taps || op->n[d] > 1024) return false;
    int coop = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (!coop) return false;
    return grid_plan(op, op->num_sms, nullptr) <= kGridSmem;
}

tca_status launch_grid_cg(tca_operator *op, const void *b, void *x, int x0_zero, cudaStream_t s, bool *launched)
{
    if (op->dtype == TCA_F64) return launch_t<double>(op, b, x, x0_zero, s, launched);
    return launch_t<float>(op, b, x, x0_zero, s, launched);
}

}  // namespace tca
