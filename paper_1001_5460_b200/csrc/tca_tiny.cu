// tca_tiny.cu -- whole-solve CG engine for small problems.
//
// Fig. 2 run by ONE thread block: the whole solve is one
// kernel launch instead of ~10 launches per iteration.  Small problems
// (config 0: 12^3 unknowns) are launch-latency bound on the general engine.
//
// Each thread owns the elements idx = tid + j*1024 (j < E) for the whole
// solve, so the vectors only the owner touches live in registers: x (C), r
// (R), q (Q) and the regulariser sum.  Only p (P, read by the neighbours of
// the mode products) and the two mode-product temporaries are in shared
// memory, with zero guard bands so the centred band rows need no bounds test
// (their taps outside the matrix are zero).  The tap tables are copied to
// shared memory at the start.  One iteration:
//   pass 1      t0 = G_D x_D p,  s = lambda sum_d R_d x_d p   (Eq. 9; registers)
//   pass 2..D   t  = G_d x_d t'; the last pass forms q = t + s in registers
//               and the <p, q> partial                        (Eq. 4)
//   reduce      alpha = rho / <p, q>
//   update      x += alpha p, r -= alpha q, <r, r> partial; reduce; beta
//   p = r + beta p
// = D + 2 block barriers per iteration.  Same semantics as cg_t / cg_iteration
// in tca_abi.cu: readings Z1-Z3, Z10 (fp64 scalars), Z12, Z28 (stop reference
// <b, b> on a warm start), the breakdown and non-finite guards, the rho history.
#include "tca_internal.cuh"

namespace tca {

namespace {

constexpr int kTinyThreads = 1024;
constexpr int kTinyWarps = kTinyThreads / 32;
constexpr size_t kTinySmem = 224 * 1024;

struct TinyMode {
    int n, inner;            // extent, stride (elements) of mode d
    int gW, rW;              // taps per row of G_d, R_d (rW = 0: no regulariser)
    int g_off, r_off;        // byte offsets of the tap tables in shared memory
    int gs_off, rs_off;      // byte offsets of the start - row offsets (int)
    const void *gt, *rt;     // global tap tables (BandMat)
    const int *gs, *rs;      // global row starts
};

struct TinyArgs {
    const void *b;
    void *x;
    CgScalars *sc;
    double *hist;
    int x0_zero;
    int N, order, guard;
    int vec_off;             // byte offset of the three guarded vectors
    double lambda;
    TinyMode md[kD];
};

// Fixed-order block sum in fp64: every warp reduces the kTinyWarps partials
// identically, so all threads get the same value (deterministic).
__device__ __forceinline__ double block_sum_d(double v, double *red)
{
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) v += __shfl_xor_sync(0xffffffffu, v, k);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = red[threadIdx.x & 31];
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) s += __shfl_xor_sync(0xffffffffu, s, k);
    return s;
}

// out[j] = sum_w taps[r][w] src[idx_j + (soff[r] + w) * inner],  r = coordinate of idx_j in mode d
template <typename T, int E, int WC>
__device__ __forceinline__ void band_rows(const T *src, const T *taps, const int *soff, int Wrt, int inner,
                                          int shift, const uint64_t (&co)[E], int N, T (&out)[E])
{
    const int W = WC > 0 ? WC : Wrt;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const int idx = threadIdx.x + j * kTinyThreads;
        T acc = T(0);
        if (idx < N) {
            const int r = (int)((co[j] >> shift) & 0xfffu);
            const T *tp = taps + r * W;
            const T *sp = src + idx + soff[r] * inner;
            if (WC > 0) {
#pragma unroll
                for (int w = 0; w < WC; ++w) acc = fma(tp[w], sp[w * inner], acc);
            } else {
                for (int w = 0; w < W; ++w) acc = fma(tp[w], sp[w * inner], acc);
            }
        }
        out[j] = acc;
    }
}

template <typename T, int E>
__device__ __forceinline__ void mode_rows(const T *src, const unsigned char *sm, const TinyMode &m, bool reg,
                                          const uint64_t (&co)[E], int shift, int N, T (&out)[E])
{
    const T *taps = reinterpret_cast<const T *>(sm + (reg ? m.r_off : m.g_off));
    const int *soff = reinterpret_cast<const int *>(sm + (reg ? m.rs_off : m.gs_off));
    const int W = reg ? m.rW : m.gW;
    if (W == 2 * kHG + 1) band_rows<T, E, 2 * kHG + 1>(src, taps, soff, W, m.inner, shift, co, N, out);
    else if (W == 2 * kHR + 1) band_rows<T, E, 2 * kHR + 1>(src, taps, soff, W, m.inner, shift, co, N, out);
    else band_rows<T, E, 0>(src, taps, soff, W, m.inner, shift, co, N, out);
}

// q = M p for the thread's elements (registers); p, t0, t1: guarded shared vectors.
// Ends with t0/t1 free; no trailing barrier (the caller's reduction has one).
template <typename T, int E>
__device__ __forceinline__ void apply_rows(const TinyArgs &a, const unsigned char *sm, const T *p, T *t0, T *t1,
                                           const uint64_t (&co)[E], T (&q)[E])
{
    const int N = a.N, D = a.order;
    T tmp[E];
#pragma unroll
    for (int j = 0; j < E; ++j) q[j] = T(0);
    for (int d = 0; d < D; ++d)   // Eq. 9 regulariser: lambda sum_d R_d x_d p
        if (a.md[d].rW > 0) {
            mode_rows<T, E>(p, sm, a.md[d], true, co, 12 * d, N, tmp);
#pragma unroll
            for (int j = 0; j < E; ++j) q[j] = fma((T)a.lambda, tmp[j], q[j]);
        }
    // Kronecker term: mode products D..1 (Eq. 5: any order)
    const T *src = p;
    for (int d = D - 1; d >= 1; --d) {
        T *dst = ((D - 1 - d) & 1) ? t1 : t0;
        mode_rows<T, E>(src, sm, a.md[d], false, co, 12 * d, N, tmp);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int idx = threadIdx.x + j * kTinyThreads;
            if (idx < N) dst[idx] = tmp[j];
        }
        __syncthreads();
        src = dst;
    }
    mode_rows<T, E>(src, sm, a.md[0], false, co, 0, N, tmp);
#pragma unroll
    for (int j = 0; j < E; ++j) q[j] = tmp[j] + q[j];
}

// Owner-only vectors (x, r): registers, or shared memory when E >= 4 elements
// per thread would spill (XS).
template <typename T, int E, bool XS>
struct OwnVec {
    T v[E];
    __device__ __forceinline__ void bind(T *) {}
    __device__ __forceinline__ T &operator()(int j) { return v[j]; }
};
template <typename T, int E>
struct OwnVec<T, E, true> {
    T *base;
    __device__ __forceinline__ void bind(T *b) { base = b + threadIdx.x; }
    __device__ __forceinline__ T &operator()(int j) { return base[j * kTinyThreads]; }
};

template <typename T, int E>
__global__ void __launch_bounds__(kTinyThreads, 1) tiny_cg_kernel(const __grid_constant__ TinyArgs a)
{
    constexpr bool XS = E >= 4;
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[2][kTinyWarps];
    const int N = a.N, G = a.guard;
    T *p = reinterpret_cast<T *>(sm + a.vec_off) + G;
    T *t0 = p + N + 2 * G;
    T *t1 = t0 + N + 2 * G;
    // ---- tap tables -> shared memory (row starts as offsets start[r] - r)
    for (int d = 0; d < a.order; ++d) {
        const TinyMode &m = a.md[d];
        const T *gt = (const T *)m.gt;
        T *gs = reinterpret_cast<T *>(sm + m.g_off);
        for (int i = threadIdx.x; i < m.n * m.gW; i += kTinyThreads) gs[i] = gt[i];
        int *go = reinterpret_cast<int *>(sm + m.gs_off);
        for (int i = threadIdx.x; i < m.n; i += kTinyThreads) go[i] = m.gs[i] - i;
        if (m.rW > 0) {
            const T *rt = (const T *)m.rt;
            T *rs = reinterpret_cast<T *>(sm + m.r_off);
            for (int i = threadIdx.x; i < m.n * m.rW; i += kTinyThreads) rs[i] = rt[i];
            int *ro = reinterpret_cast<int *>(sm + m.rs_off);
            for (int i = threadIdx.x; i < m.n; i += kTinyThreads) ro[i] = m.rs[i] - i;
        }
    }
    // zero guard bands (read by centred band rows at the tensor faces, times a zero tap)
    for (int i = threadIdx.x; i < G; i += kTinyThreads) {
        p[-1 - i] = p[N + i] = T(0);
        t0[-1 - i] = t0[N + i] = T(0);
        t1[-1 - i] = t1[N + i] = T(0);
    }
    // ---- element coordinates (12 bits per mode) and the start R := B - A*C, P := R
    uint64_t co[E];
    OwnVec<T, E, XS> x, r;
    x.bind(t1 + N + G);
    r.bind(t1 + 2 * N + G);
    T q[E];
    const T *bg = (const T *)a.b;
    T *xg = (T *)a.x;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const int idx = threadIdx.x + j * kTinyThreads;
        uint64_t c = 0;
        int rem = idx;
        for (int d = a.order - 1; d >= 0; --d) {
            c |= (uint64_t)(rem % a.md[d].n) << (12 * d);
            rem /= a.md[d].n;
        }
        co[j] = c;
        if (idx < N) {
            x(j) = a.x0_zero ? T(0) : xg[idx];
            p[idx] = x(j);
        }
        q[j] = T(0);
    }
    __syncthreads();
    if (!a.x0_zero) apply_rows<T, E>(a, sm, p, t0, t1, co, q);   // Q := A*C (warm start, Fig. 2)
    double rr = 0.0, bb = 0.0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const int idx = threadIdx.x + j * kTinyThreads;
        if (idx < N) {
            const T bi = bg[idx];
            r(j) = a.x0_zero ? bi : T(bi - q[j]);
            rr += (double)r(j) * (double)r(j);
            bb += (double)bi * (double)bi;
        }
    }
    __syncthreads();   // p (= C) fully read by the warm-start apply
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const int idx = threadIdx.x + j * kTinyThreads;
        if (idx < N) p[idx] = r(j);
    }
    CgScalars *sc = a.sc;
    const double rtol2 = sc->rtol2;
    const int max_iters = sc->max_iters;
    double rho = block_sum_d(rr, red[0]);   // (its barrier also publishes p)
    const double ref = a.x0_zero ? rho : block_sum_d(bb, red[1]);   // stop reference <b, b> (Z28)
    int status = TCA_OK, converged = 0, iters = 0;
    double rho_last = rho;
    if (threadIdx.x == 0 && a.hist) a.hist[0] = rho;
    bool done = false;
    if (!isfinite(rho)) { status = TCA_ERR_NONFINITE; done = true; }
    else if (rho == 0.0) { converged = 1; done = true; }
    else if (max_iters <= 0) { done = true; if (rtol2 > 0.0) status = TCA_NOT_CONVERGED; }
    const double rho0 = rho;
    __syncthreads();   // red[] of the start reductions fully read
    while (!done) {
        apply_rows<T, E>(a, sm, p, t0, t1, co, q);          // Q := A*(P*D)
        double pq = 0.0;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int idx = threadIdx.x + j * kTinyThreads;
            if (idx < N) pq += (double)p[idx] * (double)q[j];
        }
        pq = block_sum_d(pq, red[0]);                       // P+*Q
        if (!isfinite(pq)) { status = TCA_ERR_NONFINITE; break; }
        if (!(pq > 0.0)) { status = TCA_ERR_BREAKDOWN; break; }
        const T alpha = (T)(rho / pq);
        double r1 = 0.0;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int idx = threadIdx.x + j * kTinyThreads;
            if (idx < N) {
                x(j) = fma(alpha, p[idx], x(j));            // C := C + alpha*P*D
                r(j) = fma(-alpha, q[j], r(j));             // R := R - alpha*Q
                r1 += (double)r(j) * (double)r(j);
            }
        }
        const double rho1 = block_sum_d(r1, red[1]);        // rho1 := R+*R
        iters += 1;
        rho_last = rho1;
        if (threadIdx.x == 0 && a.hist) a.hist[iters] = rho1;
        if (!isfinite(rho1)) { status = TCA_ERR_NONFINITE; break; }
        if (rho1 == 0.0) { converged = 1; break; }                         // Z12
        if (rtol2 > 0.0 && rho1 <= rtol2 * ref) { converged = 1; break; }  // Z1, Z2, Z28
        if (iters >= max_iters) { if (rtol2 > 0.0) status = TCA_NOT_CONVERGED; break; }
        const T beta = (T)(rho1 / rho);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int idx = threadIdx.x + j * kTinyThreads;
            if (idx < N) p[idx] = fma(beta, p[idx], r(j));  // P := R + beta P (own elements)
        }
        rho = rho1;
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const int idx = threadIdx.x + j * kTinyThreads;
        if (idx < N) xg[idx] = x(j);
    }
    if (threadIdx.x == 0) {
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

constexpr int kTinyMaxE = 8;

int tiny_e(const tca_operator *op)
{
    const int64_t e = (op->N + kTinyThreads - 1) / kTinyThreads;
    return e <= 1 ? 1 : e <= 2 ? 2 : e <= 4 ? 4 : e <= 8 ? 8 : 0;
}

// shared-memory plan; 0 when the problem does not fit
size_t tiny_plan(const tca_operator *op, TinyArgs *a)
{
    const size_t es = op->esize;
    size_t off = 0;
    int inner = 1, guard = 0;
    TinyArgs t{};
    t.order = op->order;
    t.N = (int)op->N;
    t.lambda = op->lambda;
    for (int d = op->order - 1; d >= 0; --d) {
        TinyMode &m = t.md[d];
        m.n = (int)op->n[d];
        m.inner = inner;
        const BandMat &g = op->Gm[d];
        m.gW = g.W;
        m.gt = g.taps;
        m.gs = g.start;
        m.g_off = (int)off;
        off += (size_t)m.n * m.gW * es;
        m.gs_off = (int)off;
        off += (size_t)m.n * sizeof(int);
        off = (off + 15) & ~(size_t)15;
        if (op->has_reg[d]) {
            const BandMat &rm = op->Rm[d];
            m.rW = rm.W;
            m.rt = rm.taps;
            m.rs = rm.start;
            m.r_off = (int)off;
            off += (size_t)m.n * m.rW * es;
            m.rs_off = (int)off;
            off += (size_t)m.n * sizeof(int);
            off = (off + 15) & ~(size_t)15;
        }
        // rows reaching past the faces of the mode (BandMat reach; taps there are zero)
        int reach = std::max(g.reach_lo, g.reach_hi);
        if (op->has_reg[d]) reach = std::max(reach, std::max(op->Rm[d].reach_lo, op->Rm[d].reach_hi));
        guard = std::max(guard, reach * inner);
        inner *= m.n;
    }
    t.guard = guard;
    t.vec_off = (int)off;
    off += 3 * ((size_t)op->N + 2 * guard) * es;
    if (tiny_e(op) >= 4) off += 2 * (size_t)op->N * es;   // x, r in shared memory (OwnVec XS)
    if (a) *a = t;
    return off;
}

template <typename T, int E>
tca_status launch_te(const TinyArgs &a, size_t smem, cudaStream_t s)
{
    TCA_TRY(set_max_dynamic_smem((const void *)tiny_cg_kernel<T, E>, smem));
    count_launch();
    tiny_cg_kernel<T, E><<<1, kTinyThreads, smem, s>>>(a);
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

template <typename T>
tca_status launch_t(const tca_operator *op, const void *b, void *x, int x0_zero, cudaStream_t s)
{
    TinyArgs a{};
    const size_t smem = tiny_plan(op, &a);
    a.b = b;
    a.x = x;
    a.sc = op->sc;
    a.hist = op->hist;
    a.x0_zero = x0_zero;
    switch (tiny_e(op)) {
    case 1: return launch_te<T, 1>(a, smem, s);
    case 2: return launch_te<T, 2>(a, smem, s);
    case 4: return launch_te<T, 4>(a, smem, s);
    case 8: if constexpr (sizeof(T) == 4) return launch_te<T, 8>(a, smem, s); break;
    }
    return fail(TCA_ERR_INVALID_ARG, "single-block CG engine: problem too large");
}

}  // namespace

bool tiny_cg_eligible(const tca_operator *op)
{
    const char *e = getenv("TCA_TINY");   // read per call: tests pin the general path per operator   // measurement switch: TCA_TINY=0 keeps the general path
    if (e && e[0] == '0') return false;
    if (op->transport || op->scat || op->apply_path == 2 || op->order < 1) return false;
    const int E = tiny_e(op);
    if (E == 0 || (op->esize == 8 && E > 4) || E > kTinyMaxE) return false;
    for (int d = 0; d < op->order; ++d)
        if (!op->Gm[d].taps || op->n[d] > 4095) return false;
    return tiny_plan(op, nullptr) <= kTinySmem;
}

tca_status launch_tiny_cg(const tca_operator *op, const void *b, void *x, int x0_zero, cudaStream_t s)
{
    if (op->dtype == TCA_F64) return launch_t<double>(op, b, x, x0_zero, s);
    return launch_t<float>(op, b, x, x0_zero, s);
}

}  // namespace tca
