/*
 * tca_oracle.c -- plain, slow, obviously-correct CPU oracle (fp64).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1001_5460_b200/,
 * include/, the CUDA library) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg use it.  It shares no code, header, table or constant with the
 * CUDA path.
 *
 * What it computes (arxiv 1001.5460, PAPER.md line numbers):
 *   G_d = A_d^T A_d, R_d = L_d^T L_d      A.7 "patterns like A^T A from matrix
 *                                          normal equations"
 *   apply  y = (G_1 x ... x G_D) x + lam * sum_d (I x .. R_d .. x I) x
 *          Eq. 4 separable transformation as successive one-dimensional
 *          products, Eq. 9's Kronecker sum for the
 *          regulariser; operator per BASELINE.json configs.
 *   rhs    b = (A_1^T x ... x A_D^T) y   (Eq. 4 with rectangular factors,
 *          Table 1 up/down-sampling row)
 *   dot    <a,b> = sum a o b              Eq. A13/A14
 *   CG     Fig. 2 step by step with readings Z1 (loop
 *          guard erratum), Z2 (relative threshold on rho), Z3 (x0 = 0),
 *          Z12 (rho == 0 guard) from DESIGN.md.
 *
 * Conventions: tensors are dense row-major, mode 1 slowest;
 * every sum runs in ascending index order; inner loops visit
 * each matrix row's actual nonzero range [first nonzero, last nonzero],
 * found by scanning the row (no bandwidth is assumed).  Skipped terms are
 * exact zeros.  OpenMP only splits independent output elements; dots use a
 * fixed chunking so results do not depend on the thread count.
 *
 * Parity pins: see tests/test_oracle_pins.py (P1-P9 of DESIGN.md).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_DOT_CHUNK 4096

static void row_range(const double *row, int64_t len, int64_t *lo, int64_t *hi)
{
    int64_t a = 0, b = len - 1;
    while (a < len && row[a] == 0.0) a++;
    while (b >= 0 && row[b] == 0.0) b--;
    *lo = a;
    *hi = b; /* empty row: lo = len, hi = -1 */
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    int t = 1;
#pragma omp parallel
    {
#pragma omp single
        t = omp_get_num_threads();
    }
    return t;
#else
    return 1;
#endif
}

/* G[a,c] = sum_k A[k,a] * A[k,c]; A is m x n row-major, G is n x n. */
void orc_gram(int64_t m, int64_t n, const double *A, double *G)
{
    for (int64_t a = 0; a < n; a++)
        for (int64_t c = 0; c < n; c++) {
            double s = 0.0;
            for (int64_t k = 0; k < m; k++)
                s += A[k * n + a] * A[k * n + c];
            G[a * n + c] = s;
        }
}

/* T = M^T for an r x c row-major M. */
void orc_transpose(int64_t r, int64_t c, const double *M, double *T)
{
    for (int64_t i = 0; i < r; i++)
        for (int64_t j = 0; j < c; j++)
            T[j * r + i] = M[i * c + j];
}

/*
 * Mode-d product Y = X x_d M  (Eq. 4 one-dimensional transformation):
 *   Y[o, a, in] = sum_c M[a, c] X[o, c, in]
 * X has shape s[0..D-1]; M is rows x s[d]; Y has shape s with s[d] -> rows.
 */
void orc_mode_product(int D, const int64_t *s, const double *X, int d,
                      int64_t rows, const double *M, double *Y)
{
    int64_t outer = 1, inner = 1, cols = s[d];
    for (int e = 0; e < d; e++) outer *= s[e];
    for (int e = d + 1; e < D; e++) inner *= s[e];
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * (rows > 0 ? rows : 1));
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (rows > 0 ? rows : 1));
    for (int64_t a = 0; a < rows; a++) row_range(M + a * cols, cols, &lo[a], &hi[a]);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t o = 0; o < outer; o++)
        for (int64_t a = 0; a < rows; a++) {
            double *y = Y + (o * rows + a) * inner;
            for (int64_t t = 0; t < inner; t++) {
                double acc = 0.0;
                for (int64_t c = lo[a]; c <= hi[a]; c++)
                    acc += M[a * cols + c] * X[(o * cols + c) * inner + t];
                y[t] = acc;
            }
        }
    free(lo);
    free(hi);
}

static int64_t prod(const int64_t *n, int D)
{
    int64_t p = 1;
    for (int d = 0; d < D; d++) p *= n[d];
    return p;
}

/*
 * y = (G_1 x ... x G_D) x + lam * sum_d x x_d R_d.
 * Kronecker term: successive mode products in mode order 1..D (Eq. 4);
 * regulariser: one mode product per mode, summed in mode order (Eq. 9).
 * R may be NULL (lam ignored) or hold NULL entries (that mode has no term);
 * G with NULL entries means no Kronecker-product term (Eq. 9).
 */
void orc_apply(int D, const int64_t *n, const double *const *G,
               const double *const *R, double lam, const double *x, double *y)
{
    int64_t N = prod(n, D);
    double *t0 = (double *)malloc(sizeof(double) * N);
    double *t1 = (double *)malloc(sizeof(double) * N);
    int have_g = G != NULL;
    for (int d = 0; d < D && have_g; d++) have_g = G[d] != NULL;
    if (have_g) {
        memcpy(t0, x, sizeof(double) * N);
        for (int d = 0; d < D; d++) {
            orc_mode_product(D, n, t0, d, n[d], G[d], t1);
            double *sw = t0; t0 = t1; t1 = sw;
        }
    } else {   /* no Kronecker-product term (Eq. 9's separable Poisson form) */
        memset(t0, 0, sizeof(double) * N);
    }
    /* t0 = Kronecker term */
    double *reg = (double *)calloc(N, sizeof(double));
    if (R) {
        for (int d = 0; d < D; d++) {
            if (!R[d]) continue;
            orc_mode_product(D, n, x, d, n[d], R[d], t1);
            for (int64_t i = 0; i < N; i++) reg[i] += t1[i];
        }
    }
    for (int64_t i = 0; i < N; i++) y[i] = t0[i] + lam * reg[i];
    free(t0);
    free(t1);
    free(reg);
}

/*
 * b = (A_1^T x ... x A_D^T) y: successive mode products with the transposed
 * factors in mode order 1..D.  A[d] is m_d x n_d row-major; y has shape m.
 */
void orc_rhs(int D, const int64_t *n, const int64_t *m, const double *const *A,
             const double *y, double *b)
{
    int64_t s[8];
    for (int d = 0; d < D; d++) s[d] = m[d];
    int64_t cur = prod(m, D);
    double *t0 = (double *)malloc(sizeof(double) * cur);
    memcpy(t0, y, sizeof(double) * cur);
    for (int d = 0; d < D; d++) {
        double *At = (double *)malloc(sizeof(double) * m[d] * n[d]);
        orc_transpose(m[d], n[d], A[d], At);
        int64_t next = cur / m[d] * n[d];
        double *t1 = (double *)malloc(sizeof(double) * next);
        orc_mode_product(D, s, t0, d, n[d], At, t1);
        s[d] = n[d];
        free(At);
        free(t0);
        t0 = t1;
        cur = next;
    }
    memcpy(b, t0, sizeof(double) * cur);
    free(t0);
}

/*
 * One output of the apply from the plain definition (no successive
 * products):  y[i] = sum_j prod_d G_d[i_d, j_d] x[j]
 *                    + lam * sum_d sum_k R_d[i_d, k] x[i with i_d -> k].
 */
double orc_apply_point(int D, const int64_t *n, const double *const *G,
                       const double *const *R, double lam, const double *x,
                       const int64_t *i)
{
    int64_t lo[8], hi[8], j[8], stride[8];
    int empty = 0;
    stride[D - 1] = 1;
    for (int d = D - 2; d >= 0; d--) stride[d] = stride[d + 1] * n[d + 1];
    for (int d = 0; d < D; d++) {
        row_range(G[d] + i[d] * n[d], n[d], &lo[d], &hi[d]);
        if (lo[d] > hi[d]) empty = 1;
        j[d] = lo[d];
    }
    double kron = 0.0;
    while (!empty) {
        double w = 1.0;
        int64_t lin = 0;
        for (int d = 0; d < D; d++) {
            w *= G[d][i[d] * n[d] + j[d]];
            lin += j[d] * stride[d];
        }
        kron += w * x[lin];
        int d = D - 1;
        while (d >= 0) {
            if (++j[d] <= hi[d]) break;
            j[d] = lo[d];
            d--;
        }
        if (d < 0) break;
    }
    double reg = 0.0;
    if (R) {
        int64_t base = 0;
        for (int d = 0; d < D; d++) base += i[d] * stride[d];
        for (int d = 0; d < D; d++) {
            if (!R[d]) continue;
            double s = 0.0;
            for (int64_t k = 0; k < n[d]; k++) {
                double r = R[d][i[d] * n[d] + k];
                if (r != 0.0) s += r * x[base + (k - i[d]) * stride[d]];
            }
            reg += s;
        }
    }
    return kron + lam * reg;
}

/* One output of the rhs: b[i] = sum_k prod_d A_d[k_d, i_d] y[k]. */
double orc_rhs_point(int D, const int64_t *n, const int64_t *m,
                     const double *const *A, const double *y, const int64_t *i)
{
    int64_t lo[8], hi[8], k[8], stride[8];
    stride[D - 1] = 1;
    for (int d = D - 2; d >= 0; d--) stride[d] = stride[d + 1] * m[d + 1];
    for (int d = 0; d < D; d++) {
        lo[d] = m[d];
        hi[d] = -1;
        for (int64_t r = 0; r < m[d]; r++)
            if (A[d][r * n[d] + i[d]] != 0.0) {
                if (r < lo[d]) lo[d] = r;
                hi[d] = r;
            }
        if (lo[d] > hi[d]) return 0.0;
        k[d] = lo[d];
    }
    double acc = 0.0;
    for (;;) {
        double w = 1.0;
        int64_t lin = 0;
        for (int d = 0; d < D; d++) {
            w *= A[d][k[d] * n[d] + i[d]];
            lin += k[d] * stride[d];
        }
        acc += w * y[lin];
        int d = D - 1;
        while (d >= 0) {
            if (++k[d] <= hi[d]) break;
            k[d] = lo[d];
            d--;
        }
        if (d < 0) break;
    }
    return acc;
}

/* <a,b> = sum_i a_i b_i (Eq. A13): ascending sums inside fixed chunks of
 * ORC_DOT_CHUNK, then an ascending sum of the chunk sums. */
double orc_dot(int64_t N, const double *a, const double *b)
{
    int64_t nchunk = (N + ORC_DOT_CHUNK - 1) / ORC_DOT_CHUNK;
    if (nchunk == 0) return 0.0;
    double *part = (double *)malloc(sizeof(double) * nchunk);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nchunk; c++) {
        int64_t e = (c + 1) * ORC_DOT_CHUNK;
        if (e > N) e = N;
        double s = 0.0;
        for (int64_t i = c * ORC_DOT_CHUNK; i < e; i++) s += a[i] * b[i];
        part[c] = s;
    }
    double s = 0.0;
    for (int64_t c = 0; c < nchunk; c++) s += part[c];
    free(part);
    return s;
}

/* status codes (oracle-local; the product has its own) */
#define ORC_OK 0
#define ORC_BREAKDOWN 7
#define ORC_NONFINITE 8
#define ORC_NOT_CONVERGED 9

/*
 * Tensor CG, Fig. 2, step by step:
 *   R := B - A*C  (x0_zero: C = 0, Z3: R = B; else C is the caller's x);
 *   P := R;  rho := R+*R
 *   REPEAT  Q := A*(P*D)              (D: frame relabel only, Z4)
 *           alpha := rho / (P+*Q)
 *           C := C + alpha*P*D
 *           R := R - alpha*Q
 *           rho1 := R+*R
 *           [stop test, Z1/Z2/Z12/Z20]
 *           P := R + (rho1/rho)*P;  rho := rho1
 * Stop: rho1 == 0, or rtol > 0 and rho1 <= rtol^2 * <b, b> (= rho0 when C = 0;
 * reading Z28), or k+1 == max_iters.
 * hist (optional, >= max_iters+1 entries) receives rho_0 .. rho_k.
 * Returns the status; *iters = completed iterations.
 */
int orc_cg_x0(int D, const int64_t *n, const double *const *G,
              const double *const *R, double lam, const double *b, double *x,
              int x0_zero, double rtol, int max_iters, double *hist, int *iters,
              double *rho_final)
{
    int64_t N = prod(n, D);
    double *r = (double *)malloc(sizeof(double) * N);
    double *p = (double *)malloc(sizeof(double) * N);
    double *q = (double *)malloc(sizeof(double) * N);
    int status = ORC_OK;
    if (x0_zero) {
        memcpy(r, b, sizeof(double) * N);       /* R := B - A*0 */
        memset(x, 0, sizeof(double) * N);       /* C := 0 */
    } else {                                    /* warm start: x holds C */
        orc_apply(D, n, G, R, lam, x, q);
        for (int64_t i = 0; i < N; i++) r[i] = b[i] - q[i];   /* R := B - A*C */
    }
    memcpy(p, r, sizeof(double) * N);           /* P := R */
    double rho = orc_dot(N, r, r);              /* rho := R+*R */
    /* stop reference (Z2, Z28): <b, b>, which is rho_0 when C = 0 */
    double rho0 = x0_zero ? rho : orc_dot(N, b, b);
    if (hist) hist[0] = rho;
    *iters = 0;
    if (!isfinite(rho)) {
        status = ORC_NONFINITE;
    } else if (rho > 0.0) {
        for (int k = 0; k < max_iters; k++) {
            orc_apply(D, n, G, R, lam, p, q);                        /* Q := A*(P*D) */
            double pq = orc_dot(N, p, q);
            if (!isfinite(pq)) { status = ORC_NONFINITE; break; }
            if (!(pq > 0.0)) { status = ORC_BREAKDOWN; break; }
            double alpha = rho / pq;                                 /* alpha := rho/(P+*Q) */
            for (int64_t i = 0; i < N; i++) x[i] = x[i] + alpha * p[i]; /* C := C + alpha*P*D */
            for (int64_t i = 0; i < N; i++) r[i] = r[i] - alpha * q[i]; /* R := R - alpha*Q */
            double rho1 = orc_dot(N, r, r);                          /* rho1 := R+*R */
            *iters = k + 1;
            if (hist) hist[k + 1] = rho1;
            if (!isfinite(rho1)) { rho = rho1; status = ORC_NONFINITE; break; }
            if (rho1 == 0.0) { rho = rho1; break; }                  /* Z12 */
            if (rtol > 0.0 && rho1 <= rtol * rtol * rho0) { rho = rho1; break; } /* Z1, Z2 */
            if (k + 1 == max_iters) {
                rho = rho1;
                if (rtol > 0.0) status = ORC_NOT_CONVERGED;
                break;
            }
            double beta = rho1 / rho;
            for (int64_t i = 0; i < N; i++) p[i] = r[i] + beta * p[i]; /* P := R + (rho1/rho)*P */
            rho = rho1;                                              /* rho := rho1 */
        }
    }
    if (rho_final) *rho_final = rho;
    free(r);
    free(p);
    free(q);
    return status;
}

/* Fig. 2 from C = 0 (reading Z3). */
int orc_cg(int D, const int64_t *n, const double *const *G,
           const double *const *R, double lam, const double *b, double *x,
           double rtol, int max_iters, double *hist, int *iters,
           double *rho_final)
{
    return orc_cg_x0(D, n, G, R, lam, b, x, 1, rtol, max_iters, hist, iters, rho_final);
}

/* ------------------------------------------------------------------------
 * Preconditioned CG with the separable (Kronecker-factor) preconditioner
 * P = F_1 (x) ... (x) F_D,  F_d = G_d + eps_d R_d  (reading Z22;
 * SURVEY.md 8(f)1).  The paper's "direct tensor solvers"
 * applied per mode through the separable structure of Eq. 4:
 * P^-1 = F_1^-1 (x) ... (x) F_D^-1 is D successive one-dimensional solves.
 *   gbar_e = det(G_e)^(1/n_e)   (geometric mean of the eigenvalues of G_e;
 *                                det from the Cholesky diagonal)
 *   eps_d  = lam / prod_{e != d} gbar_e
 * ---------------------------------------------------------------------- */

/* Dense Cholesky F = C C^T (C lower, row-major n x n).  Returns 0, or -1 when
 * F is not positive definite. */
int orc_cholesky(int64_t n, const double *F, double *C)
{
    memset(C, 0, sizeof(double) * n * n);
    for (int64_t j = 0; j < n; j++) {
        double s = F[j * n + j];
        for (int64_t k = 0; k < j; k++) s -= C[j * n + k] * C[j * n + k];
        if (!(s > 0.0)) return -1;
        double cjj = sqrt(s);
        C[j * n + j] = cjj;
        for (int64_t i = j + 1; i < n; i++) {
            double t = F[i * n + j];
            for (int64_t k = 0; k < j; k++) t -= C[i * n + k] * C[j * n + k];
            C[i * n + j] = t / cjj;
        }
    }
    return 0;
}

/* gbar = det(G)^(1/n) = exp((2/n) sum_i log C_ii).  Returns NAN if G is not SPD. */
double orc_geomean_eig(int64_t n, const double *G)
{
    double *C = (double *)malloc(sizeof(double) * n * n);
    double s = 0.0;
    int bad = orc_cholesky(n, G, C);
    for (int64_t i = 0; i < n && !bad; i++) s += log(C[i * n + i]);
    free(C);
    return bad ? NAN : exp(2.0 * s / (double)n);
}

/* The factors F_d = G_d + eps_d R_d (R may be NULL or hold NULL entries);
 * F[d] receives n_d x n_d, eps[d] the weight.  Returns 0 or -1 (not SPD). */
int orc_precond_factors(int D, const int64_t *n, const double *const *G,
                        const double *const *R, double lam, double *const *F, double *eps)
{
    double gbar[8];
    for (int d = 0; d < D; d++) {
        gbar[d] = orc_geomean_eig(n[d], G[d]);
        if (!(gbar[d] > 0.0)) return -1;
    }
    for (int d = 0; d < D; d++) {
        double pr = 1.0;
        for (int e = 0; e < D; e++)
            if (e != d) pr *= gbar[e];
        eps[d] = lam / pr;
        for (int64_t i = 0; i < n[d] * n[d]; i++)
            F[d][i] = G[d][i] + ((R && R[d]) ? eps[d] * R[d][i] : 0.0);
    }
    return 0;
}

/*
 * z = P^-1 r: for d = 1..D, every mode-d fiber v (stride `inner`) is replaced
 * by the solution of F_d w = v, by forward substitution with C_d and back
 * substitution with C_d^T (F_d = C_d C_d^T).  C[d]: Cholesky factors.
 */
void orc_precond_apply(int D, const int64_t *n, const double *const *C, const double *r, double *z)
{
    int64_t N = prod(n, D);
    memcpy(z, r, sizeof(double) * N);
    for (int d = 0; d < D; d++) {
        int64_t outer = 1, inner = 1, len = n[d];
        for (int e = 0; e < d; e++) outer *= n[e];
        for (int e = d + 1; e < D; e++) inner *= n[e];
        const double *Cd = C[d];
#pragma omp parallel for collapse(2) schedule(static)
        for (int64_t o = 0; o < outer; o++)
            for (int64_t t = 0; t < inner; t++) {
                double *v = z + o * len * inner + t;
                for (int64_t i = 0; i < len; i++) {         /* C w' = v */
                    double s = v[i * inner];
                    for (int64_t k = 0; k < i; k++) s -= Cd[i * len + k] * v[k * inner];
                    v[i * inner] = s / Cd[i * len + i];
                }
                for (int64_t i = len - 1; i >= 0; i--) {    /* C^T w = w' */
                    double s = v[i * inner];
                    for (int64_t k = i + 1; k < len; k++) s -= Cd[k * len + i] * v[k * inner];
                    v[i * inner] = s / Cd[i * len + i];
                }
            }
    }
}

/*
 * Preconditioned CG (the textbook preconditioned form of Fig. 2's iteration):
 *   C := 0 (or the caller's x);  R := B - A*C;  Z := P^-1 R;  P := Z;
 *   rho := R+*Z;  stop reference <b, b>
 *   REPEAT  Q := A*P;  alpha := rho / (P+*Q)
 *           C := C + alpha*P;  R := R - alpha*Q;  rr := R+*R
 *           [stop test on rr exactly as orc_cg's on rho1 (Z1/Z2/Z12/Z20)]
 *           Z := P^-1 R;  rho1 := R+*Z  (<= 0 or non-finite: breakdown)
 *           P := Z + (rho1/rho)*P;  rho := rho1
 * hist receives rr_0 .. rr_k; *rr_final the last rr.
 */
int orc_pcg_x0(int D, const int64_t *n, const double *const *G,
               const double *const *R, double lam, const double *b, double *x,
               int x0_zero, double rtol, int max_iters, double *hist, int *iters, double *rr_final)
{
    int64_t N = prod(n, D);
    double *Fs[8] = {0}, *Cs[8] = {0}, eps[8];
    int status = ORC_OK;
    for (int d = 0; d < D; d++) {
        Fs[d] = (double *)malloc(sizeof(double) * n[d] * n[d]);
        Cs[d] = (double *)malloc(sizeof(double) * n[d] * n[d]);
    }
    int bad = orc_precond_factors(D, n, G, R, lam, Fs, eps);
    for (int d = 0; d < D && !bad; d++) bad = orc_cholesky(n[d], Fs[d], Cs[d]);
    double *r = (double *)malloc(sizeof(double) * N);
    double *z = (double *)malloc(sizeof(double) * N);
    double *p = (double *)malloc(sizeof(double) * N);
    double *q = (double *)malloc(sizeof(double) * N);
    if (x0_zero) {
        memset(x, 0, sizeof(double) * N);
        memcpy(r, b, sizeof(double) * N);
    } else {   /* warm start: R := B - A*C */
        orc_apply(D, n, G, R, lam, x, q);
        for (int64_t i = 0; i < N; i++) r[i] = b[i] - q[i];
    }
    double rr = orc_dot(N, r, r), rr0 = x0_zero ? rr : orc_dot(N, b, b);
    if (hist) hist[0] = rr;
    *iters = 0;
    if (bad) {
        status = ORC_BREAKDOWN;
    } else if (!isfinite(rr)) {
        status = ORC_NONFINITE;
    } else if (rr > 0.0) {
        orc_precond_apply(D, n, (const double *const *)Cs, r, z);
        memcpy(p, z, sizeof(double) * N);
        double rho = orc_dot(N, r, z);
        for (int k = 0; k < max_iters; k++) {
            orc_apply(D, n, G, R, lam, p, q);
            double pq = orc_dot(N, p, q);
            if (!isfinite(pq)) { status = ORC_NONFINITE; break; }
            if (!(pq > 0.0)) { status = ORC_BREAKDOWN; break; }
            double alpha = rho / pq;
            for (int64_t i = 0; i < N; i++) x[i] = x[i] + alpha * p[i];
            for (int64_t i = 0; i < N; i++) r[i] = r[i] - alpha * q[i];
            rr = orc_dot(N, r, r);
            *iters = k + 1;
            if (hist) hist[k + 1] = rr;
            if (!isfinite(rr)) { status = ORC_NONFINITE; break; }
            if (rr == 0.0) break;
            if (rtol > 0.0 && rr <= rtol * rtol * rr0) break;
            if (k + 1 == max_iters) {
                if (rtol > 0.0) status = ORC_NOT_CONVERGED;
                break;
            }
            orc_precond_apply(D, n, (const double *const *)Cs, r, z);
            double rho1 = orc_dot(N, r, z);
            if (!isfinite(rho1)) { status = ORC_NONFINITE; break; }
            if (!(rho1 > 0.0)) { status = ORC_BREAKDOWN; break; }
            double beta = rho1 / rho;
            for (int64_t i = 0; i < N; i++) p[i] = z[i] + beta * p[i];
            rho = rho1;
        }
    }
    if (rr_final) *rr_final = rr;
    for (int d = 0; d < D; d++) {
        free(Fs[d]);
        free(Cs[d]);
    }
    free(r);
    free(z);
    free(p);
    free(q);
    return status;
}

int orc_pcg(int D, const int64_t *n, const double *const *G,
            const double *const *R, double lam, const double *b, double *x,
            double rtol, int max_iters, double *hist, int *iters, double *rr_final)
{
    return orc_pcg_x0(D, n, G, R, lam, b, x, 1, rtol, max_iters, hist, iters, rr_final);
}

/* ------------------------------------------------------------------------
 * Single-reduction CG (Chronopoulos & Gear's rearrangement of Fig. 2's CG;
 * SURVEY.md 8(f)2, reading Z24).  Same Krylov iterates as Fig. 2 in
 * exact arithmetic; the two inner products of an iteration are taken together
 * after the one apply, so a distributed solve needs one reduction per step:
 *   C := 0 (or the caller's x);  R := B - A*C;  W := A*R;  gamma := R+*R;  delta := R+*W
 *   alpha := gamma / delta;  beta := 0;  P := 0;  S := 0
 *   REPEAT  P := R + beta*P;  S := W + beta*S        (S = A*P)
 *           C := C + alpha*P;  R := R - alpha*S
 *           W := A*R;  gamma1 := R+*R;  delta := R+*W
 *           [stop test on gamma1 exactly as orc_cg's on rho1]
 *           beta := gamma1/gamma;  alpha := gamma1 / (delta - beta*gamma1/alpha)
 *           gamma := gamma1
 * (alpha's denominator <= 0 or non-finite: breakdown).  hist: gamma_0..gamma_k.
 * ---------------------------------------------------------------------- */
int orc_cgsr_x0(int D, const int64_t *n, const double *const *G,
                const double *const *R, double lam, const double *b, double *x,
                int x0_zero, double rtol, int max_iters, double *hist, int *iters, double *rr_final)
{
    int64_t N = prod(n, D);
    double *r = (double *)malloc(sizeof(double) * N);
    double *w = (double *)malloc(sizeof(double) * N);
    double *p = (double *)calloc(N, sizeof(double));
    double *s = (double *)calloc(N, sizeof(double));
    int status = ORC_OK;
    if (x0_zero) {
        memset(x, 0, sizeof(double) * N);
        memcpy(r, b, sizeof(double) * N);
    } else {   /* warm start: R := B - A*C */
        orc_apply(D, n, G, R, lam, x, w);
        for (int64_t i = 0; i < N; i++) r[i] = b[i] - w[i];
    }
    double gamma = orc_dot(N, r, r), gamma0 = x0_zero ? gamma : orc_dot(N, b, b);
    if (hist) hist[0] = gamma;
    *iters = 0;
    if (!isfinite(gamma)) {
        status = ORC_NONFINITE;
    } else if (gamma > 0.0 && max_iters > 0) {
        orc_apply(D, n, G, R, lam, r, w);
        double delta = orc_dot(N, r, w);
        double alpha = gamma / delta, beta = 0.0;
        if (!isfinite(delta)) status = ORC_NONFINITE;
        else if (!(delta > 0.0)) status = ORC_BREAKDOWN;
        for (int k = 0; k < max_iters && status == ORC_OK; k++) {
            for (int64_t i = 0; i < N; i++) p[i] = r[i] + beta * p[i];
            for (int64_t i = 0; i < N; i++) s[i] = w[i] + beta * s[i];
            for (int64_t i = 0; i < N; i++) x[i] = x[i] + alpha * p[i];
            for (int64_t i = 0; i < N; i++) r[i] = r[i] - alpha * s[i];
            orc_apply(D, n, G, R, lam, r, w);
            double gamma1 = orc_dot(N, r, r);
            delta = orc_dot(N, r, w);
            *iters = k + 1;
            if (hist) hist[k + 1] = gamma1;
            if (!isfinite(gamma1)) { gamma = gamma1; status = ORC_NONFINITE; break; }
            if (gamma1 == 0.0) { gamma = gamma1; break; }
            if (rtol > 0.0 && gamma1 <= rtol * rtol * gamma0) { gamma = gamma1; break; }
            if (k + 1 == max_iters) {
                gamma = gamma1;
                if (rtol > 0.0) status = ORC_NOT_CONVERGED;
                break;
            }
            beta = gamma1 / gamma;
            double den = delta - beta * gamma1 / alpha;
            gamma = gamma1;
            if (!isfinite(den)) { status = ORC_NONFINITE; break; }
            if (!(den > 0.0)) { status = ORC_BREAKDOWN; break; }
            alpha = gamma1 / den;
        }
    }
    if (rr_final) *rr_final = gamma;
    free(r);
    free(w);
    free(p);
    free(s);
    return status;
}

int orc_cgsr(int D, const int64_t *n, const double *const *G,
             const double *const *R, double lam, const double *b, double *x,
             double rtol, int max_iters, double *hist, int *iters, double *rr_final)
{
    return orc_cgsr_x0(D, n, G, R, lam, b, x, 1, rtol, max_iters, hist, iters, rr_final);
}

/* ------------------------------------------------------------------------
 * Tensor Jacobi (Fig. 1a/1b), step by step:
 *   E := InvMainDiag(A);  R := A*U - B;  WHILE R+*R > threshold DO
 *   U := U - R*E;  R := A*U - B;  END
 * with U = 0 initially (reading Z26) and at most max_iters updates.  The main
 * diagonal of A = (G_1 x .. x G_D) + lam sum_d (mode-d R_d) is
 *   diag[i] = prod_d G_d[i_d, i_d] + lam sum_d R_d[i_d, i_d]
 * (G may hold NULL entries: no Kronecker-product term, Eq. 9's Poisson form).
 * hist (>= max_iters + 1): R+*R at every evaluation.  Returns ORC_OK when
 * R+*R <= threshold, ORC_NOT_CONVERGED after max_iters updates.
 * ---------------------------------------------------------------------- */
int orc_jacobi(int D, const int64_t *n, const double *const *G, const double *const *R, double lam,
               const double *b, double *u, double threshold, int max_iters, double *hist, int *iters,
               double *rr_final)
{
    int64_t N = prod(n, D);
    double *e = (double *)malloc(sizeof(double) * N);
    double *r = (double *)malloc(sizeof(double) * N);
    int status = ORC_OK;
    int have_g = 1;
    for (int d = 0; d < D; d++) have_g = have_g && G && G[d];
    for (int64_t i = 0; i < N; i++) {          /* E := InvMainDiag(A) */
        int64_t rem = i, idx[8];
        for (int d = D - 1; d >= 0; d--) { idx[d] = rem % n[d]; rem /= n[d]; }
        double pk = have_g ? 1.0 : 0.0, sm = 0.0;
        for (int d = 0; d < D; d++) {
            if (have_g) pk *= G[d][idx[d] * n[d] + idx[d]];
            if (R && R[d]) sm += R[d][idx[d] * n[d] + idx[d]];
        }
        e[i] = 1.0 / (pk + lam * sm);
    }
    memset(u, 0, sizeof(double) * N);
    orc_apply(D, n, G, R, lam, u, r);           /* R := A*U - B */
    for (int64_t i = 0; i < N; i++) r[i] -= b[i];
    double rho = orc_dot(N, r, r);
    if (hist) hist[0] = rho;
    int k = 0;
    while (rho > threshold) {                   /* WHILE R+*R > threshold */
        if (!isfinite(rho)) { status = ORC_NONFINITE; break; }
        if (k == max_iters) { status = ORC_NOT_CONVERGED; break; }
        for (int64_t i = 0; i < N; i++) u[i] -= r[i] * e[i];   /* U := U - R*E */
        orc_apply(D, n, G, R, lam, u, r);                        /* R := A*U - B */
        for (int64_t i = 0; i < N; i++) r[i] -= b[i];
        rho = orc_dot(N, r, r);
        k++;
        if (hist) hist[k] = rho;
    }
    *iters = k;
    if (rr_final) *rr_final = rho;
    free(e);
    free(r);
    return status;
}

/* ------------------------------------------------------------------------
 * Scattered-data normal operator (reading Z27).
 * Sec. 4: spline reconstruction from scattered
 * measurements, the system decomposed as a sum of rank-1 (CANDECOMP) terms and
 * applied without storing the system or its decomposition:
 *   w_k = a_{k,1} (x) ... (x) a_{k,D},   a_{k,d}[i] = beta3(t_{k,d} - i)
 *   data term  y = sum_k w_k <w_k, x>   (= W^T W x, W the K x N sample matrix)
 *   rhs        b = sum_k yk_k w_k       (= W^T yk)
 *   forward    yk_k = <w_k, x>          (= W x)
 * beta3: the centred cardinal cubic B-spline of reading Z5; t in coefficient
 * grid units (row k of t holds sample k's D coordinates).  Every a_{k,d}[i]
 * is evaluated for all i in [0, n_d) and zero weights are skipped.
 * ---------------------------------------------------------------------- */
static double orc_beta3(double u)
{
    u = fabs(u);
    if (u < 1.0) return 2.0 / 3.0 - u * u + 0.5 * u * u * u;
    if (u < 2.0) { double v = 2.0 - u; return v * v * v / 6.0; }
    return 0.0;
}

/* nonzero entries of a_{k,d}: indices idx[0..cnt) ascending, values val */
static int orc_sample_weights(double t, int64_t n, int64_t *idx, double *val, int cap)
{
    int cnt = 0;
    for (int64_t i = 0; i < n; i++) {
        double w = orc_beta3(t - (double)i);
        if (w != 0.0 && cnt < cap) { idx[cnt] = i; val[cnt] = w; cnt++; }
    }
    return cnt;
}

#define ORC_SCAT_CAP 8

/* visit every nonzero of w_k: flat index and weight, modes in order 1..D
 * (mode D fastest), calling f(flat, weight, ctx) */
static void orc_sample_visit(int D, const int64_t *n, const double *tk,
                             void (*f)(int64_t, double, void *), void *ctx)
{
    int64_t idx[4][ORC_SCAT_CAP];
    double val[4][ORC_SCAT_CAP];
    int cnt[4];
    for (int d = 0; d < D; d++) {
        cnt[d] = orc_sample_weights(tk[d], n[d], idx[d], val[d], ORC_SCAT_CAP);
        if (cnt[d] == 0) return;
    }
    int j[4] = {0, 0, 0, 0};
    for (;;) {
        int64_t flat = 0;
        double w = 1.0;
        for (int d = 0; d < D; d++) {
            flat = flat * n[d] + idx[d][j[d]];
            w *= val[d][j[d]];
        }
        f(flat, w, ctx);
        int d = D - 1;
        while (d >= 0 && ++j[d] == cnt[d]) { j[d] = 0; d--; }
        if (d < 0) break;
    }
}

struct orc_scat_ctx { const double *x; double *y; double s; };
static void orc_scat_gather(int64_t flat, double w, void *c)
{
    struct orc_scat_ctx *q = (struct orc_scat_ctx *)c;
    q->s += w * q->x[flat];
}
static void orc_scat_scatter(int64_t flat, double w, void *c)
{
    struct orc_scat_ctx *q = (struct orc_scat_ctx *)c;
    q->y[flat] += q->s * w;
}

/* y += sum_k w_k <w_k, x> */
void orc_scattered_data(int D, const int64_t *n, int64_t K, const double *t, const double *x, double *y)
{
    for (int64_t k = 0; k < K; k++) {
        struct orc_scat_ctx c = {x, y, 0.0};
        orc_sample_visit(D, n, t + k * D, orc_scat_gather, &c);    /* <w_k, x> */
        orc_sample_visit(D, n, t + k * D, orc_scat_scatter, &c);   /* y += <w_k, x> w_k */
    }
}

/* b = sum_k yk_k w_k */
void orc_scattered_rhs(int D, const int64_t *n, int64_t K, const double *t, const double *yk, double *b)
{
    memset(b, 0, sizeof(double) * prod(n, D));
    for (int64_t k = 0; k < K; k++) {
        struct orc_scat_ctx c = {NULL, b, yk[k]};
        orc_sample_visit(D, n, t + k * D, orc_scat_scatter, &c);
    }
}

/* yk_k = <w_k, x> */
void orc_scattered_forward(int D, const int64_t *n, int64_t K, const double *t, const double *x, double *yk)
{
    for (int64_t k = 0; k < K; k++) {
        struct orc_scat_ctx c = {x, NULL, 0.0};
        orc_sample_visit(D, n, t + k * D, orc_scat_gather, &c);
        yk[k] = c.s;
    }
}
