/*
 * tca.h -- C ABI of the B200 tensor-CG library (libtca.so).
 *
 * The library solves the regularised separable tensor equation of
 * arxiv 1001.5460 ("Solving Tensor Structured Problems with Computational
 * Tensor Algebra"):
 *
 *     M x = b,   M = (G_1 (x) ... (x) G_D) + lambda * sum_d (I (x) .. R_d .. (x) I)
 *     G_d = A_d^T A_d,  R_d = L_d^T L_d,   b = (A_1^T (x) ... (x) A_D^T) y
 *
 *   - the tensor equation A.U = B and its matrix equivalent: PAPER.md:100-109 (Eq. 8)
 *   - separable transformation applied mode by mode: PAPER.md:68-73 (Eq. 4)
 *   - Kronecker-sum operator (regulariser form): PAPER.md:176-182 (Eq. 9)
 *   - A^T A from matrix normal equations: PAPER.md:507-509 (A.7)
 *   - tensor conjugate gradients: PAPER.md:186-227 (Fig. 2)
 *   - inner product <A,B> = sum A o B: PAPER.md:487-505 (Eq. A13/A14)
 *
 * Conventions (all entry points):
 *   - Tensors are dense, row-major, mode 1 slowest, mode D contiguous
 *     (SPEC.md:148).  A tensor "of shape n" has prod(n_d) elements of the
 *     operator's dtype (double for TCA_F64, float for TCA_F32).
 *   - Tensor arguments of tca_apply / tca_rhs / tca_cg_solve are DEVICE
 *     pointers owned by the caller; the host variants (*_host) take HOST
 *     pointers (pinned memory recommended) and copy inside the call.
 *   - Per-mode matrices (A_d, L_d) are HOST fp64 row-major arrays, copied at
 *     create; the caller may free them afterwards.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Device-pointer calls are stream-ordered and asynchronous
 *     unless stated otherwise.
 *   - Every call validates all arguments before launching anything and
 *     returns a tca_status; nothing aborts or throws across the ABI.
 *     tca_last_error() returns a thread-local message naming the reason.
 *   - There is no CPU fallback: every numerical step runs in the library's
 *     CUDA kernels (sm_100a).
 */
#ifndef TCA_H
#define TCA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TCA_OK = 0,
    TCA_ERR_INVALID_ARG = 1, /* NULL pointer, bad order/extent/dtype/lambda   */
    TCA_ERR_SHAPE = 2,       /* matrix shapes inconsistent with n, m          */
    TCA_ERR_NOT_SPD = 3,     /* some G_d is not positive definite (A_d rank)  */
    TCA_ERR_OOM = 4,         /* device allocation failed                      */
    TCA_ERR_CUDA = 5,        /* CUDA runtime error (message in last_error)    */
    TCA_ERR_NCCL = 6,        /* NCCL error in a distributed operator          */
    TCA_ERR_BREAKDOWN = 7,   /* CG: <p, Mp> <= 0                */
    TCA_ERR_NONFINITE = 8,   /* CG: NaN/Inf in a dot product                  */
    TCA_NOT_CONVERGED = 9    /* CG: rtol not reached in max_iters (x valid)   */
} tca_status;

typedef enum { TCA_F64 = 0, TCA_F32 = 1 } tca_dtype;

/* Opaque operator: per-mode tap tables, workspaces, device scalars. */
typedef struct tca_operator tca_operator;

/*
 * Distributed (mode-1 sharded) operator description.  NULL = single GPU.
 * mode 1 (slowest) is split into nranks contiguous row
 * blocks; rank r owns unknown rows [own_lo, own_hi) = [n1*r/P, n1*(r+1)/P)
 * of every tensor (tca_operator_query), needs n1 >= 3*P, and reads the data
 * rows [data_lo, data_hi) (support of its unknown rows in A_1) for tca_rhs,
 * so the rhs is formed shard-locally without communication.  Per apply the
 * 3 boundary mode-1 slabs are exchanged with each neighbour; CG all-reduces
 * its two fp64 dot products.  Exactly one transport is given:
 *   nccl_comm    an ncclComm_t of nranks ranks, one GPU each (tca_nccl_*),
 *                owned by the caller; collectives run on the call's stream;
 *   local_group  a tca_local_group of nranks shards driven by host threads
 *                of one process (test transport for fewer GPUs than shards:
 *                host-synchronised copies; every rank must call the same
 *                entry points concurrently from its own thread).
 * Sharded operators need the fused banded path (all modes banded).  nranks = 1
 * with a transport is allowed (the whole domain, empty halos).
 */
typedef struct {
    int rank;
    int nranks;
    void *nccl_comm;
    void *local_group;
} tca_dist;

/* CG report (SPEC.md:446-449 SolveReport).  rho_history is caller-owned,
 * optional (NULL), and must hold history_capacity >= max_iters+1 doubles. */
typedef struct {
    int32_t iterations;   /* completed CG iterations k                       */
    int32_t converged;    /* 1 if rho_k <= rtol^2 <b, b> or rho_k == 0        */
    int32_t status;       /* tca_status of the solve                         */
    int32_t pad;
    double rho0;          /* <r0, r0> (= <b, b> when x0 = 0)                 */
    double rho_final;     /* recursive <r_k, r_k>                            */
    double relres_final;  /* true residual |b - M x_k|_2 / |b|_2 (reading Z2),
                             from one extra apply after the solve; 0 when
                             b = 0 and M x_k = 0                              */
    double seconds;       /* device time of the solve (CUDA events; the
                             relres_final apply is not included)            */
    double *rho_history;  /* rho_0 .. rho_k (optional)                       */
    int32_t history_capacity;
    int32_t pad2;
} tca_cg_report;

/*
 * Create the operator M for an order-D problem (1 <= order <= 4).
 *   n[d]  unknown extents, m[d] data extents (d = 0..order-1), n[d] >= 1.
 *   A[d]  host fp64 m[d] x n[d] row-major (the per-mode basis).
 *   L     NULL (no regulariser) or D host pointers to (n[d]-2) x n[d]
 *         row-major fp64 matrices; an entry may be NULL or have n[d] < 3
 *         (that mode then has no regulariser term).
 *   lambda >= 0, finite.
 *   dtype  storage and arithmetic type of tensors and taps; CG scalars
 *          (dots, alpha, beta) are always fp64.
 *   dist   NULL for one GPU, or a tca_dist (mode-1 sharding).
 * Forms G_d = A_d^T A_d and R_d = L_d^T L_d in fp64 on the host, detects the
 * half-bandwidth of each G_d (banded path when <= 3 and R_d's <= 2, dense
 * path otherwise), checks G_d positive definite (Cholesky), uploads tap
 * tables and allocates workspaces (r, p, q, halo, reduction scratch).
 * Synchronises `stream` before returning.  *op receives NULL on error.
 */
tca_status tca_operator_create(tca_operator **op, int order, const int64_t *n,
                               const int64_t *m, const double *const *A,
                               const double *const *L, double lambda,
                               tca_dtype dtype, const tca_dist *dist,
                               void *stream);

/*
 * Create the operator from its factors instead of A_d, L_d:
 *   M = (G_1 (x) ... (x) G_D) + lambda sum_d (mode-d R_d)
 * G NULL: no Kronecker-product term -- Eq. 9's separable Poisson operator
 * sum_d (mode-d R_d), e.g. R_d the 1-D finite-difference
 * Laplacian tridiag(-1, 2, -1) and lambda = 1 (reading Z25).  G (if given) and
 * R: D host fp64 n_d x n_d symmetric row-major matrices (R entries may be
 * NULL: no term for that mode); copied at create.  The operator supports
 * tca_apply and the solvers; tca_rhs / tca_forward_model return
 * TCA_ERR_INVALID_ARG (there is no A_d).  M must be SPD for the CG solvers.
 */
tca_status tca_operator_create_gram(tca_operator **op, int order, const int64_t *n,
                                    const double *const *G, const double *const *R,
                                    double lambda, tca_dtype dtype, const tca_dist *dist,
                                    void *stream);

/*
 * Query an operator.  Any output pointer may be NULL.
 *   own_lo/own_hi     mode-1 unknown rows held by this rank ([0,n1) on 1 GPU)
 *   data_lo/data_hi   mode-1 data rows this rank's tca_rhs reads
 *   banded_mask       bit d set when mode d uses the banded path
 *   half_bandwidth    D ints: half-bandwidth of G_d
 *   device_bytes      bytes of device memory the operator holds (the
 *                     matrix-free contract: O(N) + O(sum n_d^2), never N^2)
 */
tca_status tca_operator_query(const tca_operator *op, int64_t *own_lo,
                              int64_t *own_hi, int64_t *data_lo,
                              int64_t *data_hi, int *banded_mask,
                              int *half_bandwidth, size_t *device_bytes);

/* Which kernel tca_apply uses: 1 = fused banded one-pass apply (every mode
 * banded, n4 in {1,2,4,7,8,15,16,32}, tap tables fit the kernel-parameter
 * block, n3*n4*esize a multiple of 16 B), 0 = generic per-mode passes (dense
 * modes or other shapes), -1 = op is NULL.  A fused-eligible operator still
 * takes the generic path for a call whose x or y is not 16-byte aligned. */
int tca_operator_apply_path(const tca_operator *op);

/*
 * Scattered-data operator (reading Z27 and 6.6):
 * the normal equations of a cubic B-spline fit to K scattered samples, Sec. 4
 * of the paper, held as its rank-1 (CANDECOMP) sample
 * terms, never as a matrix:
 *   M x = sum_k w_k <w_k, x> + lambda sum_d (mode-d L_d^T L_d) x,
 *   w_k = a_{k,1} (x) ... (x) a_{k,D},  a_{k,d}[i] = beta3(t[k*order+d] - i)
 * with beta3 the centred cubic B-spline of reading Z5.
 *   n: order extents (<= 4096 each); t: HOST array K x order (row-major),
 *      sample coordinates in coefficient-grid units, each in [0, n_d - 1];
 *      copied (bucketed by tile) at create, the caller may free it.
 *   L: as in tca_operator_create (NULL: no regulariser).
 * On such an operator tca_apply / tca_cg_solve / tca_cgsr_solve use M;
 * tca_rhs takes ydata = K sample values (device, original sample order) and
 * forms sum_k y_k w_k; tca_forward_model writes the K values <w_k, x> (+ noise)
 * (x NULL: the seed's x_true); tca_solve_host(_batch) takes K host values.
 * PCG, Jacobi and the preconditioner calls return TCA_ERR_INVALID_ARG.
 * Single GPU (no dist).  Sums use atomics: results are reproducible to
 * rounding, not bit-for-bit.  Errors: TCA_ERR_INVALID_ARG (NULL/non-finite/
 * out-of-range t, bad L), TCA_ERR_SHAPE (n, or a last mode too long for the
 * shared-memory tile), TCA_ERR_CUDA.
 */
tca_status tca_operator_create_scattered(tca_operator **op, int order,
                                         const int64_t *n, int64_t K,
                                         const double *t,
                                         const double *const *L,
                                         double lambda, tca_dtype dtype,
                                         void *stream);

/* Whether CG / PCG solves on this operator run the fused step B1' (SURVEY.md
 * 8(a) a5): ONE kernel per iteration forms P := R|Z + beta P,
 * applies the pending C := C + alpha P and computes Q = M P with <P, Q>
 * (reads R|Z, P, C; writes P, C, Q), instead of a separate update pass.
 * Opt-in: used only when the environment has TCA_B1=1 at the operator's first
 * solve (measured slower than the default three-kernel iteration on config 3,
 * DESIGN.md 6.5).  1 = yes, 0 = no (not requested, sharded operator, non-fused
 * apply path, tables outside the parameter block, or a shape whose shared-
 * memory plan does not fit: fp64 n4 = 16, 32), -1 = not decided yet
 * (no CG solve so far) or op NULL.  Results are the same iterates either way. */
int tca_operator_cg_fused_step(const tca_operator *op);

/* Whether CG / PCG solves on this operator defer the x update of Fig. 2
 * (C := C + alpha P) into the next iteration's operator
 * apply, where one extra warp per CTA streams it beside the banded apply
 * (DESIGN.md 6.5): the iteration's vector kernels then move 6 words per
 * unknown (R := R - alpha Q; P_next := R|Z + beta P into a second P buffer)
 * instead of 8.  Same arithmetic, same iterates.  Default on for fp32 fused
 * operators on one GPU (the extra warp costs no occupancy there), off for fp64
 * (its apply would lose registers); TCA_DX=1|0 in the environment at the first
 * solve forces it.  1 = yes, 0 = no, -1 = not decided yet or op NULL. */
int tca_operator_cg_deferred_x(const tca_operator *op);

/* Which engine tca_cg_solve uses on this operator: 1 = single-block engine
 * (tca_tiny.cu: the whole Fig. 2 solve, in ONE kernel launch
 * by one 1024-thread block: p and two apply temporaries in shared memory, x,
 * r, q in registers (shared memory above two elements per thread); chosen for
 * fp64 N <= 4096, fp32 N <= 8192, n_d <= 4095, when the tap tables and vectors
 * fit 224 KB of shared memory, single GPU, not scattered, not a Kronecker-sum-
 * only operator; the environment switch TCA_TINY=0 disables it), 2 = one
 * cooperative grid (tca_grid.cu: the whole solve in ONE persistent kernel, one
 * block per SM, phases separated by grid-wide barriers, vectors L2-resident;
 * chosen when the single-block engine is not, for N <= 2^21 and n_d <= 1024
 * with the tap tables and fibre tiles in 200 KB of shared memory, single GPU,
 * not scattered, not Kronecker-sum-only; TCA_GRID=0 disables it; a solve
 * still runs the general engine if the device cannot co-schedule every block
 * at that moment, e.g. a shared GPU), 0 = general
 * multi-kernel engine, -1 = op NULL.  Same iterates, stop rules, guards and
 * report on every engine (readings Z1-Z3, Z10, Z12, Z28). */
int tca_operator_cg_engine(const tca_operator *op);

/* y = M x.  x, y: device tensors of the local shape (rows [own_lo, own_hi)
 * of mode 1 on a sharded operator); x and y must not alias. */
tca_status tca_apply(const tca_operator *op, const void *x, void *y,
                     void *stream);

/* b = (A_1^T (x) ... (x) A_D^T) ydata.  ydata: device tensor of shape
 * (data_hi-data_lo, m_2, ..., m_D); b: device tensor of the local unknown
 * shape.  Uses a temporary device workspace of at most prod(m)/ratio
 * elements (stream-ordered allocation). */
tca_status tca_rhs(const tca_operator *op, const void *ydata, void *b,
                   void *stream);

/*
 * Solve M x = b by tensor CG (Fig. 2).
 *   x0_zero != 0: start from C = 0 (reading Z3; the initial apply is skipped,
 *             R := B); x is output only.
 *   x0_zero == 0: x holds the start C on entry (warm start): R := B - A*C
 *             (Fig. 2's first line) with one apply.
 *   rtol > 0: stop when rho_k <= rtol^2 * <b, b> (reading Z2; <b, b> = rho_0
 *             when x0 = 0, reading Z28 for a warm start) or rho_k == 0,
 *             status TCA_NOT_CONVERGED if max_iters is reached first;
 *   rtol <= 0: run exactly max_iters iterations (stopping early only if
 *             rho_k == 0, reading Z12).
 * b, x: device tensors of the local shape (not aliasing).  The iteration runs
 * entirely on the device (scalars in device memory, no host round trip per
 * iteration).  With rep != NULL the report's relres_final costs one more
 * apply after the solve.  Synchronises `stream` before filling *rep.
 * Errors: TCA_ERR_INVALID_ARG (NULL/aliasing tensors, max_iters < 0,
 * non-finite rtol), TCA_ERR_BREAKDOWN (<p, Mp> <= 0),
 * TCA_ERR_NONFINITE (NaN/Inf in a dot product), TCA_NOT_CONVERGED (x valid).
 */
tca_status tca_cg_solve(tca_operator *op, const void *b, void *x, int x0_zero,
                        double rtol, int32_t max_iters, tca_cg_report *rep,
                        void *stream);

/*
 * Preconditioned CG (reading Z22) with the
 * separable Kronecker-factor preconditioner
 *   P = F_1 (x) ... (x) F_D,  F_d = G_d + eps_d R_d,
 *   eps_d = lambda / prod_{e != d} gbar_e,  gbar_e = det(G_e)^(1/n_e)
 * (the geometric mean of G_e's eigenvalues), applied as D successive
 * one-dimensional Cholesky solves (Eq. 4's separable structure, PAPER.md:68-73,
 * with the per-mode "direct tensor solver" of PAPER.md:116).  Iteration:
 *   R := B, Z := P^-1 R, P := Z, rho := R+*Z; repeat Q := M P,
 *   alpha := rho / P+*Q, C += alpha P, R -= alpha Q, [stop test on R+*R exactly
 *   as tca_cg_solve's], Z := P^-1 R, rho1 := R+*Z, P := Z + (rho1/rho) P.
 * Arguments (x0_zero included: R := B - A*C before Z := P^-1 R), stop rule,
 * report and stream semantics as tca_cg_solve (the report's rho values and
 * history are R+*R).  The factors are formed on the
 * first call (host fp64 Cholesky, n_d <= 256) and kept by the operator.
 * TCA_ERR_INVALID_ARG on a sharded operator (nranks > 1: the mode-1 solve
 * would cross shards); TCA_ERR_BREAKDOWN if R+*Z <= 0.
 */
tca_status tca_pcg_solve(tca_operator *op, const void *b, void *x, int x0_zero,
                         double rtol, int32_t max_iters, tca_cg_report *rep,
                         void *stream);

/*
 * Tensor Jacobi (Fig. 1a/1b), the paper's stationary solver:
 *   E := inverse main diagonal of M; U := 0 (reading Z26); R := M U - B;
 *   WHILE R+*R > threshold DO U := U - R*E; R := M U - B END
 * threshold: absolute bound on R+*R (Fig. 1c uses 1e-4), >= 0.
 * At most max_iters updates (status TCA_NOT_CONVERGED if the bound is not
 * reached).  x receives U.  Report as tca_cg_solve (rho values and history are
 * R+*R).  Single GPU only (TCA_ERR_INVALID_ARG on a sharded operator).
 */
tca_status tca_jacobi_solve(tca_operator *op, const void *b, void *x, double threshold,
                            int32_t max_iters, tca_cg_report *rep, void *stream);

/*
 * Single-reduction CG (reading Z24): Chronopoulos
 * and Gear's rearrangement of Fig. 2's recurrences with the
 * same Krylov iterates in exact arithmetic:
 *   R := B, W := M R, gamma := R+*R, delta := R+*W, alpha := gamma/delta,
 *   beta := 0, P := S := 0; repeat P := R + beta P, S := W + beta S,
 *   C += alpha P, R -= alpha S, W := M R, gamma1 := R+*R, delta := R+*W,
 *   [stop test on gamma1 exactly as tca_cg_solve's], beta := gamma1/gamma,
 *   alpha := gamma1 / (delta - beta gamma1 / alpha).
 * Both inner products of an iteration are reduced together after the apply:
 * one reduction point per iteration (one all-reduce of two fp64 values on a
 * sharded operator) instead of two.  Arguments (x0_zero: R := B - A*C),
 * stop rule, report (rho = R+*R) and stream semantics as tca_cg_solve; works
 * on sharded operators.
 */
tca_status tca_cgsr_solve(tca_operator *op, const void *b, void *x, int x0_zero,
                          double rtol, int32_t max_iters, tca_cg_report *rep,
                          void *stream);

/* z = P^-1 r with the PCG preconditioner above (device tensors of the local
 * shape, z may equal r).  Stream-ordered. */
tca_status tca_precond_apply(tca_operator *op, const void *r, void *z, void *stream);

/* The preconditioner's eps_d and the lower bandwidth of each Cholesky factor
 * (order entries each; either pointer may be NULL).  Forms the factors if needed. */
tca_status tca_precond_info(tca_operator *op, double *eps, int *lower_bandwidth,
                            void *stream);

/*
 * End-to-end solve from HOST buffers: copies ydata_host (data shape of this
 * rank) to the device, forms the rhs, runs tca_cg_solve and copies x back to
 * x_host (local unknown shape).  Synchronises `stream`.
 */
tca_status tca_solve_host(tca_operator *op, const void *ydata_host,
                          void *x_host, double rtol, int32_t max_iters,
                          tca_cg_report *rep, void *stream);

/*
 * Pipelined end-to-end solves of `count` independent data sets with the same
 * operator (the same bases and lambda): item i copies ydata_host[i] to the
 * device, forms its rhs, runs tca_cg_solve and copies x back to x_host[i].
 * The H2D of item i+1 runs on an internal copy stream while item i computes
 * and the D2H of item i while item i+1 computes, so on a compute-bound solve
 * the PCIe transfers are hidden (SURVEY.md 8(d) time-to-solution with host
 * I/O).  Host buffers: caller-owned, pinned for overlap (pageable works but
 * serialises), shapes as in tca_solve_host.  Device memory: two ydata and two
 * x staging buffers besides the operator's.  reps: NULL or `count` reports.
 * Returns the first error (later items are not started), else
 * TCA_NOT_CONVERGED if any item did not converge, else TCA_OK.  Synchronises
 * `stream` and the copy stream before returning.
 */
tca_status tca_solve_host_batch(tca_operator *op, int count,
                                const void *const *ydata_host,
                                void *const *x_host, double rtol,
                                int32_t max_iters, tca_cg_report *reps,
                                void *stream);

void tca_operator_destroy(tca_operator *op);

/*
 * Shard layout (host only, no device needed): for an n1 x ... problem whose
 * mode-1 basis A1 is m1 x n1 (row-major fp64), rank `rank` of `nranks` owns
 * unknown rows [out4[0], out4[1]) and reads data rows [out4[2], out4[3]).
 * TCA_ERR_SHAPE when n1 < 3 * nranks.
 */
tca_status tca_shard_layout(int64_t n1, int64_t m1, const double *A1, int rank,
                            int nranks, int64_t *out4);

/* NCCL bootstrap (libnccl.so.2 is loaded at first use): rank 0 creates the
 * 128-byte unique id, the caller broadcasts it (e.g. torch.distributed), every
 * rank creates its communicator on its current device. */
tca_status tca_nccl_get_unique_id(void *uid128);
tca_status tca_nccl_comm_create(void **comm, int nranks, const void *uid128, int rank);
void tca_nccl_comm_destroy(void *comm);

/* In-process shard group for the local transport (see tca_dist). */
tca_status tca_local_group_create(void **group, int nranks);
void tca_local_group_destroy(void *group);

/*
 * Seeded synthetic input generator (reading Z9): out[i] = scale *
 * normal(seed, stream_id, offset + i), i < count, where normal(.) is the
 * Box-Muller transform of the counter generator
 *   u64(seed, s, j) = mix64(mix64(seed * GAMMA + s) + j * GAMMA)
 * (SplitMix64 output function, GAMMA = 0x9E3779B97F4A7C15) with
 *   normal(j) = sqrt(-2 ln U(2j)) cos(2 pi U(2j+1)),  U = ((u64>>11)+0.5) 2^-53.
 * out: device array of `count` elements of dtype.
 */
tca_status tca_generate_normal(void *out, tca_dtype dtype, int64_t count,
                               int64_t offset, uint64_t seed,
                               uint32_t stream_id, double scale, void *stream);

/*
 * Synthetic data of the operator's problem: ydata = (A_1 (x) ... (x) A_D) x
 *   + sigma * normal(seed, 1, global data linear index), for this rank's data
 * rows.  x: device tensor of the full unknown shape (or NULL: x_true is then
 * generated in place from stream 0, position keyed).  ydata as in tca_rhs.
 */
tca_status tca_forward_model(const tca_operator *op, const void *x, void *ydata,
                             double sigma, uint64_t seed, void *stream);

/*
 * Timing instrumentation (measurement only; off by default).  When enabled,
 * tca_cg_solve and tca_apply record a CUDA event pair on `stream` around
 * the operator-apply launches (eager launches: every one; inside CG's graph
 * chunks of 32 iterations: the applies of iterations 0 and 16 of each chunk,
 * as external event nodes of the captured graph -- a node pair costs ~20 us
 * of replay time, so timing every apply would slow the solve it measures --
 * two alternating instances so that one is read while the other runs);
 * tca_operator_get_timing returns the summed device
 * time (ms) and the number of timed applies since the last reset.
 */
tca_status tca_operator_set_timing(tca_operator *op, int enable);
tca_status tca_operator_get_timing(tca_operator *op, double *apply_ms,
                                   int64_t *apply_count, int reset);

/* Number of CUDA kernel launches the library has issued so far (process-wide;
   the kernels of a replayed CG graph chunk count at every replay). */
int64_t tca_kernel_launches(void);

const char *tca_status_string(tca_status s);
const char *tca_last_error(void);

/* Library build information: "tca <version> sm_100a" */
const char *tca_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TCA_H */
