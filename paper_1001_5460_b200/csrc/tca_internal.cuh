// tca_internal.cuh -- internal declarations of libtca (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>
#include <atomic>

#include "../../include/tca.h"

namespace tca {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
tca_status fail(tca_status s, const std::string &msg);
tca_status cuda_fail(cudaError_t e, const char *what);

#define TCA_CUDA_TRY(expr)                                           \
    do {                                                             \
        cudaError_t e_ = (expr);                                     \
        if (e_ != cudaSuccess) return ::tca::cuda_fail(e_, #expr);   \
    } while (0)

#define TCA_TRY(expr)                                                \
    do {                                                             \
        tca_status s_ = (expr);                                      \
        if (s_ != TCA_OK) return s_;                                 \
    } while (0)

// ---------------------------------------------------------------- layout
// Every problem is padded to order 4 with trailing extents 1 (G = [1], no
// regulariser), so mode 1 is always the slowest (streamed / sharded) mode
// and mode 4 the contiguous one.
constexpr int kD = 4;
constexpr int kHG = 3;  // half-bandwidth of the banded G taps (7 taps)
constexpr int kHR = 2;  // half-bandwidth of the banded R taps (5 taps)
constexpr int kRedBlocks = 592;   // 4 x 148: fixed grid of every dot partial
constexpr int kRedThreads = 256;

// Compressed band rows of a rows x cols matrix:
//   (M v)[r] = sum_{w < W} taps[r*W + w] * v[start[r] + w]   (zero outside [0, cols))
struct BandMat {
    int rows = 0, cols = 0, W = 0;
    int *start = nullptr;  // device, rows
    void *taps = nullptr;  // device, rows*W of the operator dtype
    size_t tap_bytes = 0;
    bool dense = false;    // W == cols and start == 0: taps is the dense row-major matrix
    int reach_lo = 0;      // rows a band row reads before column 0 (max over rows of -start[r])
    int reach_hi = 0;      // ... and past column cols - 1 (max of start[r] + W - cols); taps there are zero
    int win16 = 0;         // largest input window (max start + W - min start) of 16 consecutive rows
};

// Device-resident CG scalars (always fp64, reading Z10).
struct CgScalars {
    double rho;      // <r_k, r_k> (CG) or <r_k, z_k> (PCG)
    double rho0;     // <r_0, r_0> = <b, b>
    double pq;       // <p_k, q_k>
    double alpha;    // rho / pq
    double beta;     // rho1 / rho
    double rtol2;    // rtol^2 (<= 0: fixed iterations)
    int32_t iters;   // completed iterations
    int32_t max_iters;
    int32_t done;    // 1: later kernels of the solve are no-ops
    int32_t status;  // tca_status
    int32_t converged;
    int32_t xupd;    // 1: this iteration's alpha is valid (x := x + alpha p pending)
    double rr;       // <r_k, r_k> (the residual; == rho for plain CG)
    int32_t pcg;     // 1: preconditioned (rho = <r, z>; beta set by finalize 3)
    double thr;      // tensor Jacobi: absolute threshold on R+*R
    int32_t pad;
    double ref;      // stop reference: rtol is relative to <b, b> (= rho0 when x0 = 0; reading Z28)
    double red[10];  // reduced dot products (stage sum -> all-reduce -> stage apply); 8, 9: |b - Mx|^2, |b|^2
    uint32_t fin_cnt[2];   // CTA arrival counters of the finalisers fused into their producer kernels
                           // (0: the band apply's alpha, 1: cg_update_r's rho1); zero between launches
};

// Exchange steps of a mode-1 sharded operator (tca_dist.cu).
class Transport {
  public:
    virtual ~Transport() {}
    // in-place sum over ranks of `count` fp64 values in device memory
    virtual tca_status allreduce(double *dev, int count, cudaStream_t s) = 0;
    // fill the 3 ghost slabs on each side of a ghosted buffer
    //   ext = [3 ghost | nloc own | 3 ghost] slabs of slab_bytes each
    // from the neighbours' boundary slabs; which = 0 (CG p) or 1 (apply input)
    virtual tca_status halo(int which, char *ext, size_t slab_bytes, int64_t nloc, cudaStream_t s) = 0;
    // true when the exchanges are stream-ordered device operations that can be
    // captured into a CUDA graph (NCCL); false for host-synchronised ones
    virtual bool capturable() const { return false; }
    // true when halo() may be issued on a side stream joined by events (overlap)
    virtual bool async_halo() const { return false; }
    // host wait for stream s (NCCL: polls the communicator's error state, with a timeout)
    virtual tca_status wait(cudaStream_t s)
    {
        const cudaError_t e = cudaStreamSynchronize(s);
        return e == cudaSuccess ? TCA_OK : cuda_fail(e, "stream");
    }
};
Transport *make_transport(const tca_dist *d);
tca_status shard_layout(int64_t n1, const double *A1, int64_t m1, int rank, int nranks, int64_t out[4]);

// A cached TMA tensor map (CUtensorMap is 128 bytes, 64-byte aligned).
struct alignas(64) TmapSlot {
    uint64_t map[16];
    const void *ptr = nullptr;
    int kind = 0;   // 0: slab-load map of an apply input, 1: tile-store map of an apply output
    int slot = 0;   // index in the operator's device descriptor buffer
};
constexpr int kTmapSlots = 32;

// Scattered-data operator geometry (tca_scatter.cu): 4 internal modes (orders
// D < 4 padded in front with size-1 modes), tiles of TB cells along modes 1-3.
struct ScatGeom {
    int n[4];      // internal extents
    int real[4];   // 1: B-spline mode, 0: padded mode (weight 1)
    int TB;        // cells per tile along the real modes among 1-3
    int nt[3];     // tiles along modes 1-3
    int F[4];      // shared-memory footprint extents (TB+3 | 1, n4+3)
};

}  // namespace tca

struct tca_operator {
    std::vector<tca::TmapSlot> tmaps;    // TMA descriptors of recent apply inputs/outputs
    void *tmap_dev = nullptr;            // device copies (kTmapSlots x 128 B)
    uint64_t *tmap_host = nullptr;       // pinned host staging of the descriptors
    cudaEvent_t tmap_ev[tca::kTmapSlots] = {};   // last launch reading each slot
    int tmap_next = 0;
    uint32_t tmap_pinned = 0;            // bit i: slot i is referenced by a captured CUDA graph
    int order = 0;
    bool gram_form = false;              // created from G_d / R_d (tca_operator_create_gram): no A_d
    void *ks_taps = nullptr;             // Kronecker-sum-only operator (apply_path 2): rows of lambda R_d, 5 taps
    size_t ks_bytes = 0;
    int ks_off[tca::kD] = {0, 0, 0, 0};
    int64_t n[tca::kD] = {1, 1, 1, 1};   // global unknown extents (padded)
    int64_t m[tca::kD] = {1, 1, 1, 1};   // global data extents (padded)
    tca_dtype dtype = TCA_F64;
    size_t esize = 8;
    double lambda = 0.0;
    int hbG[tca::kD] = {0, 0, 0, 0};
    int hbR[tca::kD] = {0, 0, 0, 0};
    int has_reg[tca::kD] = {0, 0, 0, 0};
    int banded_mask = 0;                 // bit d: G_d hb <= 3 (and R_d hb <= 2)
    bool all_banded = false;

    // symmetric band rows for the fused banded kernel (host, fp64):
    // bandG[d][r*4 + k] = G_d[r, r+k] (k = 0..3), bandR[d][r*3 + k] = lambda R_d[r, r+k] (k = 0..2)
    std::vector<double> bandG[tca::kD];
    std::vector<double> bandR[tca::kD];
    std::vector<unsigned char> band_params;   // prebuilt kernel-parameter block (tap tables)
    char band_sched = 0;                      // schedule of the last band-apply parameter build: w(hole) / s(plit) / l(ock)
    int band_gt = 0;                          // tap tables: 0 block; global (band_gtaps) with modes 4 (1) or 4+3 (2) in the block
    void *band_gtaps = nullptr;
    size_t band_gtaps_bytes = 0;
    // dense host G_d, R_d (fp64; R_d empty without a regulariser) for the PCG factors
    std::vector<double> Gh[tca::kD], Rh[tca::kD];
    // Kronecker-factor preconditioner (tca_precond.cu; built on first use)
    bool pc_ready = false;
    double pc_eps[tca::kD] = {0, 0, 0, 0};
    int pc_w[tca::kD] = {0, 0, 0, 0};            // sub-diagonals stored per factor row
    int pc_lbw[tca::kD] = {0, 0, 0, 0};          // lower bandwidth of the Cholesky factor
    bool pc_banded[tca::kD] = {false, false, false, false};
    void *pc_tab[tca::kD] = {nullptr, nullptr, nullptr, nullptr};   // device factor rows (tca_precond.cu)
    size_t pc_tab_bytes[tca::kD] = {0, 0, 0, 0};
    tca::BandMat pc_inv[tca::kD];                // dense factors: F_d^-1 (dense mode product)
    void *z = nullptr;                           // PCG workspace z = P^-1 r
    void *pc_tmp = nullptr;                      // scratch of the dense-factor mode products
    void *sr_s = nullptr;                        // single-reduction CG: S = A P (lazy)
    void *grid_ws = nullptr;                     // cooperative-grid CG engine workspace (lazy)
    size_t grid_ws_bytes = 0;
    void *jac_e = nullptr;                       // tensor Jacobi: E = inverse main diagonal (lazy)
    const void *jac_b = nullptr;                 // tensor Jacobi: B of the running solve
    // generic compressed-band forms
    tca::BandMat Gm[tca::kD], Rm[tca::kD], At[tca::kD], Af[tca::kD];

    // sharding (mode 1)
    int rank = 0, nranks = 1;
    void *comm = nullptr;
    tca::Transport *transport = nullptr;
    int ghost = 0;            // ghost slabs on each side of p / x_ext (3 when sharded)
    int64_t slab = 0;         // elements per mode-1 slab (n2 n3 n4)
    void *x_ext = nullptr;    // ghosted copy of a tca_apply input (sharded, lazy)
    int64_t own_lo = 0, own_hi = 0, data_lo = 0, data_hi = 0;
    int64_t xf_lo = 0, xf_hi = 0;   // unknown rows read by the shard-local forward model
    int64_t nloc1 = 0;        // own_hi - own_lo
    int64_t N = 0;            // local unknowns
    int64_t Mloc = 0;         // local data points

    // workspaces
    void *r = nullptr, *q = nullptr;
    void *p = nullptr;        // ghosted: [ghost | nloc1 own | ghost] slabs
    void *p_own = nullptr;    // p + ghost slabs
    void *t0 = nullptr, *t1 = nullptr;   // multi-pass temporaries (lazy)
    double *part = nullptr;              // kRedBlocks reduction partials (x3)
    tca::CgScalars *sc = nullptr;        // device scalars
    tca::CgScalars *sc_host = nullptr;   // pinned mirror
    double *hist = nullptr;              // device rho history
    int hist_cap = 0;
    size_t device_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int num_sms = 148;
    int band_grid = 0;                   // persistent grid of the fused banded apply
    // scattered-data operator (tca_operator_create_scattered): sample term on top
    // of the Kronecker-sum regulariser (apply_path 2)
    bool scat = false;
    tca::ScatGeom sg{};
    int64_t sc_K = 0;
    int sc_ntiles = 0;
    void *sc_t = nullptr, *sc_perm = nullptr, *sc_tstart = nullptr;   // samples bucketed by tile
    void *sc_coef = nullptr;             // <w_k, x> per sorted sample (apply scratch)
    // fused CG step B1' (apply that also forms P_new and updates C): its own
    // parameter block and schedule (whole tile columns: every CTA at the same
    // mode-1 slab, so the halo re-reads hit L2), two P buffers (P_old is read
    // by neighbouring CTAs while P_new is written)
    std::vector<unsigned char> band_params_fu;
    int band_grid_fu = 0;
    std::vector<unsigned char> band_params_dx;   // apply with the deferred C update (MODE 2)
    int band_grid_dx = 0;
    int dx = -1;                         // deferred C update in the apply: -1 not decided, 0 off, 1 on
    int b1 = -1;                         // -1: not decided, 0: off, 1: on
    void *p2 = nullptr;                  // second P buffer
    int pcur = 0;                        // 0: P in p_own, 1: P in p2
    int apply_path = 0;                  // 0 = generic multi-pass, 1 = fused banded, 2 = Kronecker-sum stencil
    int band_v2 = 0;                     // fused banded apply: 1 = warp-specialised kernel (tca_band2.cuh)
    mutable bool band_fin_req = false;   // next fused apply with <p, q> partials: run CG's finaliser 1 in its last CTA
    mutable bool band_fin_done = false;  // ... and the last launch did (else the caller runs cg_reduce)
    // CUDA-graph replay of CG chunks
    // (two instances when timing: each carries its own captured event pairs, so
    // one can be harvested while the other runs)
    cudaStream_t gstream = nullptr;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    const void *gx = nullptr;
    int gtimed = 0;                      // the instances were captured with timing events
    int gsolver = 0;                     // ... for this solver's iteration
    const void *gb = nullptr;            // ... and this right-hand side (the Jacobi iteration reads B)
    int solver = 0;                      // iteration being run/captured: 0 CG (Fig. 2), 1 PCG, 2 single-reduction CG
    int64_t gkernels[2] = {0, 0};        // kernel launches captured in instance g (added per replay)
    bool gpend[2] = {false, false};      // instance g has launched and its events are unharvested
    std::vector<cudaEvent_t> gev[2];     // captured (external) event pairs of instance g
    std::vector<cudaEvent_t> *cap_ev = nullptr;   // event list being captured into (sampled iteration)
    bool capturing = false;              // a chunk is being captured (applies outside the sample run plain)
    cudaEvent_t gfork = nullptr, gjoin = nullptr;
    // sharded CG: the halo of p on a side stream under the interior p update
    cudaStream_t hstream = nullptr;
    cudaEvent_t hfork = nullptr, hjoin = nullptr;
    // timing instrumentation
    int timing = 0;
    std::vector<cudaEvent_t> tev;        // pairs (start, stop)
    size_t tev_used = 0;
    double apply_ms = 0.0;
    int64_t apply_count = 0;
};

namespace tca {

// ---------------------------------------------------------------- kernels (tca_kernels.cu)
// Y[o, r, t] = alpha * sum_w taps[r,w] X[o, start[r]+w, t]  (+ Y[o,r,t] if accumulate)
template <typename T>
void launch_band_mode_product(const T *X, T *Y, int64_t outer, const BandMat &M,
                              int64_t inner, double alpha, bool accumulate,
                              const int32_t *done, cudaStream_t s);

// mode 1 and the contiguous last mode of a (cols, K c4) tensor in one pass (M1: rows x
// cols, M4: r4 x c4); false when not applicable (nothing launched)
template <typename T>
bool launch_band_win_last(const T *X, T *Y, int64_t K, int c4, const BandMat &M1, const BandMat &M4, cudaStream_t s);

// the two fastest modes of an (planes, c3, c4) tensor in one pass (M3: rows r3 x
// cols c3, M4: r4 x c4); false when the plane does not fit shared memory (nothing launched)
template <typename T>
bool launch_band_plane2(const T *X, T *Y, int64_t planes, int c3, int c4, const BandMat &M3, const BandMat &M4,
                        cudaStream_t s);

// dense fp64 mode product on the FP64 tensor cores (DMMA); M row-major rows x cols
void launch_dense_mode_product_dmma(const double *X, double *Y, int64_t outer, int rows, int cols,
                                    int64_t inner, const double *M, double alpha, bool accumulate,
                                    const int32_t *done, cudaStream_t s);

template <typename T>
void launch_gen_normal(T *out, int64_t count, int64_t offset, uint64_t key,
                       double scale, bool accumulate, cudaStream_t s);

// CG vector kernels; every one is a no-op once sc->done != 0.
template <typename T>
void launch_cg_init(const T *b, T *x, T *r, T *p, int64_t N, double *part,
                    cudaStream_t s);
template <typename T>
void launch_dot_partials(const T *a, const T *b, int64_t N, double *part,
                         const int32_t *done, cudaStream_t s);
tca_status precond_prepare(tca_operator *op, cudaStream_t s);
tca_status scatter_prepare(tca_operator *op, int64_t K, const double *t, cudaStream_t s);
tca_status launch_scatter(const tca_operator *op, int mode, const void *x, void *out, const void *yk,
                          const int32_t *done, cudaStream_t s);
// process-wide free list of small pinned host buffers (tca_abi.cu)
void *pinned_get(size_t bytes);
// process-wide free list of small device buffers (tca_abi.cu)
cudaError_t dev_get(void **p, size_t bytes);
void dev_put(void *p, size_t bytes);
void pinned_put(void *p, size_t bytes);
// single-reduction CG (tca_kernels.cu)
template <typename T>
void launch_cgsr_update(T *x, T *p, T *sv, T *r, const T *w, int64_t N, const CgScalars *sc, double *part,
                        cudaStream_t s);
void launch_cgsr_finalize(int which, const double *prr, int nrr, const double *prw, int nrw, CgScalars *sc,
                          double *hist, cudaStream_t s, int stage = 0);
// Kronecker-sum apply (operators without a product term; tca_kernels.cu)
template <typename T>
void launch_ksum_apply(const T *x, T *y, int64_t N, const int64_t *n, const T *taps, const int *off,
                       const int32_t *done, cudaStream_t s);
// tensor Jacobi (tca_kernels.cu)
template <typename T>
void launch_jacobi_diag(T *e, int64_t N, const int64_t *n, const double *dg, const double *dr, int nmax, double lam,
                        bool have_g, cudaStream_t s);
template <typename T>
void launch_jacobi_resid(T *r, const T *q, const T *b, int64_t N, double *part, const int32_t *done, cudaStream_t s);
template <typename T>
void launch_jacobi_update(T *u, const T *r, const T *e, int64_t N, const CgScalars *sc, cudaStream_t s);
void launch_jacobi_finalize(int which, const double *part, int nparts, CgScalars *sc, double *hist, cudaStream_t s);
// banded PCG factor solve along mode d (tca_precond.cu); src may equal dst
template <typename T>
tca_status launch_precond_sweep(const tca_operator *op, int d, const T *src, T *dst, int64_t outer, int64_t inner,
                                const int32_t *done, cudaStream_t s);
// dense n x n matrix in the operator's dtype (tca_abi.cu)
tca_status make_dense_mat(tca_dtype dt, const std::vector<double> &M, int n, BandMat *out, size_t *bytes);
template <typename T>
// fin: run finaliser 2 (rho1, stop test, beta) in the kernel's last CTA
// (single GPU; a sharded solve all-reduces the partials first)
void launch_cg_update_r(T *r, const T *q, int64_t N, CgScalars *sc, double *part, cudaStream_t s,
                        bool fin = false, double *hist = nullptr);
// d = b - q: r and p (either may be NULL) receive d; part_dd / part_bb the
// per-block partials of <d, d> and <b, b> (warm start R := B - A*C, and the
// true residual of the report)
template <typename T>
void launch_resid2(const T *b, const T *q, T *r, T *p, int64_t N, double *part_dd, double *part_bb, cudaStream_t s);
template <typename T>
void launch_cg_update_xp(T *x, T *p, const T *r, int64_t N, const CgScalars *sc, cudaStream_t s);
template <typename T>
void launch_cg_update_p(T *pn, const T *p, const T *d, int64_t N, const CgScalars *sc, cudaStream_t s);

// finalisers (one block): 0 = init rho, 1 = pq -> alpha, 2 = rr -> beta/stop,
// 8 = stop reference <b, b> of a warm start (stage 1 only: red[8], red[9] for the report)
// stage: 0 = sum the partials and apply (single GPU), 1 = sum into sc->red[which]
// only, 2 = apply from sc->red[which] (after the all-reduce)
void launch_cg_finalize(int which, const double *part, int nparts, CgScalars *sc,
                        double *hist, cudaStream_t s, int stage = 0);

uint64_t stream_key(uint64_t seed, uint32_t stream_id);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) once per (kernel,
// device, size): the attribute is per device, and the library may drive
// several devices from several host threads (tca_abi.cu)
tca_status set_max_dynamic_smem(const void *func, size_t bytes);
// whole-solve single-block CG for small problems (tca_tiny.cu)
bool tiny_cg_eligible(const tca_operator *op);
tca_status launch_tiny_cg(const tca_operator *op, const void *b, void *x, int x0_zero, cudaStream_t s);
// whole-solve cooperative-grid CG for mid-size problems (tca_grid.cu)
bool grid_cg_eligible(const tca_operator *op);
// *launched = false (TCA_OK): the blocks cannot all be co-resident on this device
// right now; the caller runs the general engine
tca_status launch_grid_cg(tca_operator *op, const void *b, void *x, int x0_zero, cudaStream_t s, bool *launched);

// process-wide count of kernel launches issued by the library
extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// ---------------------------------------------------------------- host helpers (tca_abi.cu)
tca_status apply_multipass(const tca_operator *op, const void *x, void *y,
                           const int32_t *done, cudaStream_t s);

}  // namespace tca
