// tca_precond.cu -- the separable (Kronecker-factor) preconditioner of PCG
// (reading Z22):
//
//   P = F_1 (x) ... (x) F_D,   F_d = G_d + eps_d R_d,   eps_d = lambda / prod_{e != d} gbar_e
//
// with gbar_e = det(G_e)^(1/n_e), the geometric mean of G_e's eigenvalues.
// P^-1 = F_1^-1 (x) ... (x) F_D^-1 applies as D successive one-dimensional
// solves (Eq. 4's separable structure; the paper's "direct
// tensor solvers", used per mode): every mode-d fibre is solved
// with the Cholesky factor F_d = C_d C_d^T by a forward and a back sweep.
//
// Host: factors in fp64 (dense Cholesky of n_d x n_d, n_d <= 256).  A banded
// factor (lower bandwidth <= 3: the B-spline modes; a banded SPD matrix has a
// banded Cholesky factor) is stored as rows [1/C_ii, C_i,i-1, C_i,i-2, C_i,i-3]
// and solved by the sweep kernel below; a dense factor (Gaussian modes) is
// replaced by the explicit F_d^-1 and applied as a dense mode product on the
// FP64 tensor cores (tca_abi.cu apply_precond).
// Sweep kernel: one thread per fibre, fibres ordered with the mode's inner
// index fastest so a warp's accesses at each step are contiguous; the last
// three solved values stay in registers.
#include <cmath>
#include <algorithm>
#include <cstring>

#include "tca_internal.cuh"

namespace tca {

namespace {

// element-granular asynchronous global -> shared copy (LDGSTS): the whole
// tile's loads are in flight at once without holding registers
template <typename T>
__device__ __forceinline__ void cp_async_elem(T *sdst, const T *gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sa), "l"(gsrc), "n"(sizeof(T)) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Forward sweep C w = v then back sweep C^T u = w along one fibre
// (element i at v[i * inner]); src may equal dst (in place).  Loads are
// issued U at a time ahead of the (sequential) recurrence so that U memory
// requests per thread are in flight; the grid is a bounded set of threads
// (grid-stride over the fibres) so that the forward results each thread
// re-reads in its back sweep are still in L2.
template <typename T, int U>
__global__ void __launch_bounds__(256, 2)
precond_sweep_kernel(const T *src, T *dst, int64_t outer, int len, int64_t inner, const T *__restrict__ tab,
                     const int32_t *done)
{
    if (done && *done) return;
    const int64_t lines = outer * inner;
    for (int64_t line = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; line < lines;
         line += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = line / inner, t = line - o * inner;
        const int64_t base = o * (int64_t)len * inner + t;
        const T *x = src + base;
        T *z = dst + base;
        T w1 = T(0), w2 = T(0), w3 = T(0);   // z[i-1], z[i-2], z[i-3]
        for (int i0 = 0; i0 < len; i0 += U) {
            T v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = (i0 + u < len) ? x[(int64_t)(i0 + u) * inner] : T(0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u;
                if (i < len) {
                    const T *c = tab + (int64_t)i * 8;   // forward row [f0..f3] (see precond_prepare)
                    const T s = fma(-c[1], w1, fma(-c[2], w2, fma(-c[3], w3, c[0] * v[u])));
                    z[(int64_t)i * inner] = s;
                    w3 = w2; w2 = w1; w1 = s;
                }
            }
        }
        T u1 = T(0), u2 = T(0), u3 = T(0);   // u[i+1], u[i+2], u[i+3]
        for (int i0 = len - 1; i0 >= 0; i0 -= U) {
            T v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = (i0 - u >= 0) ? z[(int64_t)(i0 - u) * inner] : T(0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 - u;
                if (i >= 0) {
                    const T *c = tab + (int64_t)i * 8 + 4;   // backward row [b0..b3]
                    const T s = fma(-c[1], u1, fma(-c[2], u2, fma(-c[3], u3, c[0] * v[u])));
                    z[(int64_t)i * inner] = s;
                    u3 = u2; u2 = u1; u1 = s;
                }
            }
        }
    }
}

// Shared-memory form: a block of LB threads stages LB whole fibres (len x LB
// elements, coalesced: for inner >= LB a step i of the LB fibres is LB
// consecutive elements, for inner == 1 the LB fibres are one contiguous run),
// solves each fibre in shared memory (thread j walks column j: conflict-free
// with the odd pitch LB + 1) and writes the tile back: exactly one read and one
// write of the tensor per mode.
template <typename T>
__global__ void __launch_bounds__(256)
precond_sweep_smem_kernel(const T *src, T *dst, int64_t outer, int len, int64_t inner, const T *__restrict__ tab,
                          int LB, const int32_t *done)
{
    if (done && *done) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    T *tb = reinterpret_cast<T *>(smraw);   // [len][8] factor rows
    T *v = tb + 8 * len;                     // [len][LB + 1]
    const int P = LB + 1, NT = blockDim.x, tid = threadIdx.x;
    const int64_t lines = outer * inner;
    const int64_t l0 = (int64_t)blockIdx.x * LB;
    const int nl = (int)((lines - l0) < LB ? (lines - l0) : LB);
    for (int k = tid; k < 8 * len; k += NT) tb[k] = tab[k];
    // all NT threads move the tile: thread -> fibre jj = tid % LB, steps i = tid / LB (+ NT / LB)
    const int jj = tid % LB, i0 = tid / LB, di = NT / LB;
    int64_t gb = 0;
    if (jj < nl) {
        const int64_t line = l0 + jj, o = line / inner;
        gb = o * len * inner + (line - o * inner);
    }
    const int tot = nl * len;
    if (inner == 1) {   // the block's fibres are one contiguous run
        const T *g = src + l0 * len;
        for (int k = tid; k < tot; k += NT) {
            const int j = k / len, i = k - j * len;
            cp_async_elem(v + i * P + j, g + k);
        }
    } else if (jj < nl) {   // step i of consecutive fibres: consecutive addresses
        for (int i = i0; i < len; i += di) cp_async_elem(v + i * P + jj, src + gb + (int64_t)i * inner);
    }
    cp_async_wait_all();
    __syncthreads();
    const int j = tid;
    if (j < nl) {
        T w1 = T(0), w2 = T(0), w3 = T(0);
        // one DFMA on the recurrence's critical path per step (s_{i-1} enters last);
        // the next step's coefficients and input are loaded before this step's
        // store (the table and the tile share the shared-memory buffer, so the
        // compiler would otherwise order every load after the previous store)
        T c0 = tb[0], c1 = tb[1], c2 = tb[2], c3 = tb[3], x0 = v[j];
        for (int i = 0; i < len; ++i) {
            T n0 = T(0), n1 = T(0), n2 = T(0), n3 = T(0), xn = T(0);
            if (i + 1 < len) {
                const T *cn = tb + 8 * (i + 1);
                n0 = cn[0]; n1 = cn[1]; n2 = cn[2]; n3 = cn[3];
                xn = v[(i + 1) * P + j];
            }
            const T s = fma(-c1, w1, fma(-c2, w2, fma(-c3, w3, c0 * x0)));
            v[i * P + j] = s;
            w3 = w2; w2 = w1; w1 = s;
            c0 = n0; c1 = n1; c2 = n2; c3 = n3; x0 = xn;
        }
        T u1 = T(0), u2 = T(0), u3 = T(0);
        {
            const T *cb = tb + 8 * (len - 1) + 4;
            c0 = cb[0]; c1 = cb[1]; c2 = cb[2]; c3 = cb[3];
        }
        x0 = v[(len - 1) * P + j];
        for (int i = len - 1; i >= 0; --i) {
            T n0 = T(0), n1 = T(0), n2 = T(0), n3 = T(0), xn = T(0);
            if (i > 0) {
                const T *cn = tb + 8 * (i - 1) + 4;
                n0 = cn[0]; n1 = cn[1]; n2 = cn[2]; n3 = cn[3];
                xn = v[(i - 1) * P + j];
            }
            const T s = fma(-c1, u1, fma(-c2, u2, fma(-c3, u3, c0 * x0)));
            v[i * P + j] = s;
            u3 = u2; u2 = u1; u1 = s;
            c0 = n0; c1 = n1; c2 = n2; c3 = n3; x0 = xn;
        }
    }
    __syncthreads();
    if (inner == 1) {
        T *g = dst + l0 * len;
        for (int k = tid; k < tot; k += NT) {
            const int jq = k / len, i = k - jq * len;
            g[k] = v[i * P + jq];
        }
    } else if (jj < nl) {
#pragma unroll 4
        for (int i = i0; i < len; i += di) dst[gb + (int64_t)i * inner] = v[i * P + jj];
    }
}

// Dense Cholesky F = C C^T (C lower, row-major); false if F is not SPD.
bool cholesky(const std::vector<double> &F, int n, std::vector<double> &C)
{
    C.assign((size_t)n * n, 0.0);
    for (int j = 0; j < n; ++j) {
        double s = F[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) s -= C[(size_t)j * n + k] * C[(size_t)j * n + k];
        if (!(s > 0.0)) return false;
        const double cjj = std::sqrt(s);
        C[(size_t)j * n + j] = cjj;
        for (int i = j + 1; i < n; ++i) {
            double t = F[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) t -= C[(size_t)i * n + k] * C[(size_t)j * n + k];
            C[(size_t)i * n + j] = t / cjj;
        }
    }
    return true;
}

}  // namespace

tca_status precond_prepare(tca_operator *op, cudaStream_t s)
{
    if (op->pc_ready) return TCA_OK;
    // gbar_d from the Cholesky diagonal of G_d: log det = 2 sum log C_ii
    double gbar[kD];
    std::vector<double> C;
    for (int d = 0; d < kD; ++d) {
        const int n = (int)op->n[d];
        if (!cholesky(op->Gh[d], n, C)) return fail(TCA_ERR_NOT_SPD, "G_" + std::to_string(d + 1) + " not SPD");
        double ls = 0.0;
        for (int i = 0; i < n; ++i) ls += std::log(C[(size_t)i * n + i]);
        gbar[d] = std::exp(2.0 * ls / n);
    }
    size_t bytes = 0;
    for (int d = 0; d < kD; ++d) {
        const int n = (int)op->n[d];
        double pr = 1.0;
        for (int e = 0; e < op->order; ++e)
            if (e != d) pr *= gbar[e];
        const double eps = op->lambda / pr;   // (used only where mode d has a regulariser)
        op->pc_eps[d] = eps;
        std::vector<double> F(op->Gh[d]);
        if (op->has_reg[d])
            for (size_t i = 0; i < F.size(); ++i) F[i] += eps * op->Rh[d][i];
        if (!cholesky(F, n, C))
            return fail(TCA_ERR_NOT_SPD, "preconditioner factor F_" + std::to_string(d + 1) + " not SPD");
        int w = 0;   // lower bandwidth of C
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < i; ++k)
                if (C[(size_t)i * n + k] != 0.0 && i - k > w) w = i - k;
        op->pc_lbw[d] = w;
        op->pc_banded[d] = w <= 3;
        if (!op->pc_banded[d]) {   // dense factor: F_d^-1 = C^-T C^-1, column by column
            std::vector<double> Fi((size_t)n * n), v(n);
            for (int j = 0; j < n; ++j) {
                for (int i = 0; i < n; ++i) {   // C v = e_j
                    double t = i == j ? 1.0 : 0.0;
                    for (int k = 0; k < i; ++k) t -= C[(size_t)i * n + k] * v[k];
                    v[i] = t / C[(size_t)i * n + i];
                }
                for (int i = n - 1; i >= 0; --i) {   // C^T u = v
                    double t = v[i];
                    for (int k = i + 1; k < n; ++k) t -= C[(size_t)k * n + i] * v[k];
                    v[i] = t / C[(size_t)i * n + i];
                }
                for (int i = 0; i < n; ++i) Fi[(size_t)i * n + j] = v[i];
            }
            TCA_TRY(make_dense_mat(op->dtype, Fi, n, &op->pc_inv[d], &bytes));
            continue;
        }
        // banded rows, the 1/C_ii scaling folded into the sweeps' coefficients:
        //   forward  s_i = f0 v_i - f1 s_{i-1} - f2 s_{i-2} - f3 s_{i-3},  f0 = 1/C_ii, f_k = C_{i,i-k}/C_ii
        //   backward u_i = b0 w_i - b1 u_{i+1} - b2 u_{i+2} - b3 u_{i+3},  b0 = 1/C_ii, b_k = C_{i+k,i}/C_ii
        // (zero where i-k or i+k leaves the fibre)
        op->pc_w[d] = 3;
        std::vector<double> tab((size_t)n * 8, 0.0);
        for (int i = 0; i < n; ++i) {
            const double c0 = 1.0 / C[(size_t)i * n + i];
            tab[(size_t)i * 8] = c0;
            tab[(size_t)i * 8 + 4] = c0;
            for (int k = 1; k <= 3; ++k) {
                if (i - k >= 0) tab[(size_t)i * 8 + k] = C[(size_t)i * n + i - k] * c0;
                if (i + k < n) tab[(size_t)i * 8 + 4 + k] = C[(size_t)(i + k) * n + i] * c0;
            }
        }
        std::vector<unsigned char> raw(tab.size() * op->esize);
        if (op->dtype == TCA_F64) std::memcpy(raw.data(), tab.data(), raw.size());
        else
            for (size_t i = 0; i < tab.size(); ++i) reinterpret_cast<float *>(raw.data())[i] = (float)tab[i];
        TCA_CUDA_TRY(dev_get(&op->pc_tab[d], raw.size()));
        op->pc_tab_bytes[d] = raw.size();
        TCA_CUDA_TRY(cudaMemcpyAsync(op->pc_tab[d], raw.data(), raw.size(), cudaMemcpyHostToDevice, s));
        TCA_CUDA_TRY(cudaStreamSynchronize(s));
        bytes += raw.size();
    }
    TCA_CUDA_TRY(cudaMallocAsync(&op->z, (size_t)op->N * op->esize, s));
    bytes += (size_t)op->N * op->esize;
    bool any_dense = false;
    for (int d = 0; d < op->order; ++d) any_dense |= !op->pc_banded[d];
    if (any_dense) {
        TCA_CUDA_TRY(cudaMallocAsync(&op->pc_tmp, (size_t)op->N * op->esize, s));
        bytes += (size_t)op->N * op->esize;
    }
    op->device_bytes += bytes;
    op->pc_ready = true;
    return TCA_OK;
}

template <typename T>
tca_status launch_precond_sweep(const tca_operator *op, int d, const T *src, T *dst, int64_t outer, int64_t inner,
                                const int32_t *done, cudaStream_t s)
{
    const int len = (int)op->n[d];
    const int64_t lines = outer * inner;
    // shared-memory tiles of LB fibres (LB a multiple of 32, <= 256, tile <= ~100 KB)
    {
        const size_t es = sizeof(T);
        // ~3 tiles per SM; all 256 threads move a tile, LB of them sweep it
        int LB = (int)((75 * 1024 / es - 8 * (size_t)len) / (len + 2));
        LB = std::min(256, LB / 32 * 32);
        while (LB > 32 && 256 % LB) LB -= 32;   // LB divides the 256 movers
        if (LB >= 32) {
            const size_t smem = (8 * (size_t)len + (size_t)len * (LB + 1)) * es;
            if (smem > 100 * 1024) LB = 0;
        }
        if (LB >= 32) {
            const size_t smem = (8 * (size_t)len + (size_t)len * (LB + 1)) * es;
            TCA_TRY(set_max_dynamic_smem((const void *)precond_sweep_smem_kernel<T>, 110 * 1024));
            count_launch();
            precond_sweep_smem_kernel<T><<<(unsigned)((lines + LB - 1) / LB), 256, smem, s>>>(
                src, dst, outer, len, inner, (const T *)op->pc_tab[d], LB, done);
            TCA_CUDA_TRY(cudaGetLastError());
            return TCA_OK;
        }
    }
    // bounded grid: ~512 resident fibre threads per SM keep each thread's forward
    // results (len elements) in L2 for its back sweep
    const int64_t cap = (int64_t)op->num_sms * 2;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((lines + 255) / 256, cap));
    count_launch();
    precond_sweep_kernel<T, 8><<<blocks, 256, 0, s>>>(src, dst, outer, len, inner, (const T *)op->pc_tab[d], done);
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

template tca_status launch_precond_sweep<double>(const tca_operator *, int, const double *, double *, int64_t,
                                                 int64_t, const int32_t *, cudaStream_t);
template tca_status launch_precond_sweep<float>(const tca_operator *, int, const float *, float *, int64_t, int64_t,
                                                const int32_t *, cudaStream_t);

}  // namespace tca
