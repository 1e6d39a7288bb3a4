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
#include <cstring>

#include "tca_internal.cuh"

namespace tca {

namespace {

// Forward sweep C w = v then back sweep C^T u = w along one fibre
// (element i at v[i * inner]); src may equal dst.
template <typename T, int W>
__global__ void __launch_bounds__(256)
precond_sweep_kernel(const T *src, T *dst, int64_t outer, int len, int64_t inner,
                     const T *__restrict__ tab, const int32_t *done)
{
    if (done && *done) return;
    const int64_t line = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (line >= outer * inner) return;
    const int64_t o = line / inner, t = line - o * inner;
    const int64_t base = o * (int64_t)len * inner + t;
    const T *x = src + base;
    T *z = dst + base;
    static_assert(W >= 1 && W <= 3, "banded factor rows");
    {
        constexpr int R = W + 1;
        T w1 = T(0), w2 = T(0), w3 = T(0);   // z[i-1], z[i-2], z[i-3]
        for (int i = 0; i < len; ++i) {
            const T *c = tab + (int64_t)i * R;
            T s = x[(int64_t)i * inner];
            s -= c[1] * w1;                   // entries beyond the fibre start are 0 in the table
            if (W >= 2) s -= c[2] * w2;
            if (W >= 3) s -= c[3] * w3;
            s *= c[0];
            z[(int64_t)i * inner] = s;
            w3 = w2; w2 = w1; w1 = s;
        }
        T u1 = T(0), u2 = T(0), u3 = T(0);   // u[i+1], u[i+2], u[i+3]
        for (int i = len - 1; i >= 0; --i) {
            T s = z[(int64_t)i * inner];
            if (i + 1 < len) s -= tab[(int64_t)(i + 1) * R + 1] * u1;
            if (W >= 2 && i + 2 < len) s -= tab[(int64_t)(i + 2) * R + 2] * u2;
            if (W >= 3 && i + 3 < len) s -= tab[(int64_t)(i + 3) * R + 3] * u3;
            s *= tab[(int64_t)i * R];
            z[(int64_t)i * inner] = s;
            u3 = u2; u2 = u1; u1 = s;
        }
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
        const int W = 3;   // banded rows: [1/C_ii, C_i,i-1, C_i,i-2, C_i,i-3]
        op->pc_w[d] = W;
        std::vector<double> tab((size_t)n * (W + 1), 0.0);
        for (int i = 0; i < n; ++i) {
            tab[(size_t)i * (W + 1)] = 1.0 / C[(size_t)i * n + i];
            for (int k = 1; k <= W && k <= i; ++k) tab[(size_t)i * (W + 1) + k] = C[(size_t)i * n + i - k];
        }
        std::vector<unsigned char> raw(tab.size() * op->esize);
        if (op->dtype == TCA_F64) std::memcpy(raw.data(), tab.data(), raw.size());
        else
            for (size_t i = 0; i < tab.size(); ++i) reinterpret_cast<float *>(raw.data())[i] = (float)tab[i];
        TCA_CUDA_TRY(cudaMalloc(&op->pc_tab[d], raw.size()));
        TCA_CUDA_TRY(cudaMemcpyAsync(op->pc_tab[d], raw.data(), raw.size(), cudaMemcpyHostToDevice, s));
        TCA_CUDA_TRY(cudaStreamSynchronize(s));
        bytes += raw.size();
    }
    TCA_CUDA_TRY(cudaMalloc(&op->z, (size_t)op->N * op->esize));
    bytes += (size_t)op->N * op->esize;
    bool any_dense = false;
    for (int d = 0; d < op->order; ++d) any_dense |= !op->pc_banded[d];
    if (any_dense) {
        TCA_CUDA_TRY(cudaMalloc(&op->pc_tmp, (size_t)op->N * op->esize));
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
    const unsigned blocks = (unsigned)((lines + 255) / 256);
    count_launch();
    precond_sweep_kernel<T, 3><<<blocks, 256, 0, s>>>(src, dst, outer, len, inner, (const T *)op->pc_tab[d], done);
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

template tca_status launch_precond_sweep<double>(const tca_operator *, int, const double *, double *, int64_t,
                                                 int64_t, const int32_t *, cudaStream_t);
template tca_status launch_precond_sweep<float>(const tca_operator *, int, const float *, float *, int64_t, int64_t,
                                                const int32_t *, cudaStream_t);

}  // namespace tca
