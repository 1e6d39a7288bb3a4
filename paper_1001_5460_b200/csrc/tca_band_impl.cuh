// tca_band_impl.cuh -- fused banded operator apply, one HBM pass.
// Instantiated per dtype in tca_band_f64.cu / tca_band_f32.cu.
//
//   q = (G_1 (x) G_2 (x) G_3 (x) G_4) p + sum_d (mode-d lambda R_d) p
//
// Eq. 4 applies the separable operator as successive
// one-dimensional transformations; Eq. 5 lets us pick their
// order; Eq. 9 gives the Kronecker-sum regulariser.  Every
// G_d has half-bandwidth <= 3 and every R_d <= 2 (checked at create).
//
// B200 design:
//   * A CTA (256 threads, 1 per SM, persistent) owns a tile of T2 = 8 mode-2
//     rows x T3 mode-3 columns x all n4 and STREAMS mode 1: input slab j
//     (i1 = j) is staged in shared memory once by TMA (halo 3 in i2 and i3,
//     out-of-domain boxes zero-filled = the truncated band of reading Z15).
//   * In-slice modes are applied in the order 2 -> 3 -> 4 (mode 2 on the
//     halo-extended columns):
//       pass A  column owner along i2:  U2 = G2 p, RA = lambda R2 p
//       pass B  8 outputs along i3:     U3 = G3 U2, RB = RA + lambda R3 p
//       pass C  E <= 8 outputs along i4 (the ring owner):
//               S = G4 U3 + lambda R4 p + RB, then mode 1 as a 6-slot
//               register ring over j (G1 S and lambda R1 p), and emission of
//               the finished output slab j-3 to a staging buffer that one
//               thread stores with a TMA bulk tensor store.
//   * Every band loop is written in PUSH form (one input value, consecutive
//     DFMAs into the outputs it touches) and every tap is a kernel-parameter
//     (constant bank) operand -- compile-time offsets for mode 4, uniform
//     runtime offsets (LDCU) for modes 1-3 -- so a DFMA reads one or two
//     register-file operands (profiles/r01_microbench_fp64_operands.txt: three
//     RF operands cap DFMA at ~60 % of peak).
//   * Two CTA barriers per slab; the staged slabs are NSTAGE deep (mbarrier
//     completion), the output staging is double-buffered.
//   * A CTA owns a contiguous range of (tile, i1) units; a range that starts
//     or ends inside a tile pays 6 ramp slabs (mode-1 halo).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "tca_internal.cuh"
#include "tca_finalize.cuh"

#include <type_traits>

#ifndef TCA_RING_F2
#define TCA_RING_F2 1   // fp32 mode-1 ring on FFMA2
#endif

#ifndef TCA_BAND_DBG
#define TCA_BAND_DBG 1   // TCA_BAND_DEBUG phase switches compiled in
#endif

namespace tca {
namespace band {

// CTA shape per n4 (Cfg): NTHR threads, MINB CTAs per SM.  n4 <= 16: two
// 256-thread CTAs per SM (each with its own barriers and TMA pipeline, so one
// CTA's barrier/memory phases overlap the other's compute; with the
// shift-register ring the code fits the instruction cache); n4 = 32: one
// 512-thread CTA.
constexpr int T2 = 8;            // mode-2 rows per tile
constexpr int PR = T2 + 6;       // staged rows (halo 3 + 3)
constexpr int REC = 7;           // tap record per row: G[r,r..r+3], lambda R[r,r..r+2]
constexpr int PADR = 6;          // zero rows below each table (row r at record off + r + PADR)
constexpr int KH1 = 3;           // mode-1 half-bandwidth: a slab range needs 3 ramp slabs each side
constexpr int TAP_BYTES = 27 * 1024;
constexpr int MAXG = 320;        // max persistent CTAs (>= 2 x SM count)

// Kernel parameters (constant bank).  The per-CTA schedule is precomputed on
// the host so that every control value in the kernel is warp-uniform (no
// integer division on device): the compiler then keeps tile coordinates in
// uniform registers and loads taps with LDCU into uniform-register operands.
template <typename T>
struct ParamsBase {
    const T *x;
    T *y;
    const int32_t *done;
    double *pq_part;       // optional: per-CTA partial <x, y> of the emitted outputs (CG's <p, q>)
    CgScalars *fin_sc;     // optional (with pq_part; MODE 0, 256-thread CTAs): the last CTA runs
    double *fin_hist;      // CG's finaliser 1 (alpha := rho / <p, q>, tca_finalize.cuh)
    int n1, n2, n3, tiles3;   // n1: output slabs (local rows of a sharded operator)
    int xoff, nin;            // input slab j lives at slab j + xoff of an input of nin slabs (ghosts)
    int off3, off2, off1;     // record offsets (rows) of the mode-3/2/1 tables; mode 4 at 0
    int dbg;                  // phase switches for bisecting (TCA_BAND_DEBUG; 0 in production)
    int onebox;               // 1: a slab is ONE 4-D TMA box (Cfg::ONEBOX and n3 n4 % UNIT == 0)
    int o_next;               // first output slab of a CTA's second and later tiles (0; lockstep tails: L)
    short2 s_tile[MAXG];   // CTA b starts at tile (x = mode-2 tile, y = mode-3 tile) ...
    int s_o0[MAXG];        // ... at output slab s_o0 ...
    int s_cnt[MAXG];       // ... and processes s_cnt (tile, slab) units
};
// taps in the parameter block (constant bank: LDCU into uniform-register operands)
template <typename T>
struct Params : ParamsBase<T> {
    using value_type = T;
    T taps[TAP_BYTES / sizeof(T)];
};
// tables too large for the parameter block (n_d ~ 256): the whole table in
// global memory, read through the read-only path (register operands), and the
// records of its first NBM modes (mode 4; with NBM = 2 also mode 3) in the block
// as well, so that the mode-4 taps stay compile-time constant-bank operands and
// mode 3's (pass B) uniform-register ones (config 4: pass C + ring 10.4 -> ... ms,
// DESIGN.md 6.1)
template <typename T, int NBM>
struct ParamsGT : ParamsBase<T> {
    using value_type = T;
    static constexpr int block_modes = NBM;
    const T *gtaps;
    T taps[TAP_BYTES / sizeof(T)];
};
template <typename T>
using ParamsG = ParamsGT<T, 1>;   // mode 4 in the block, modes 1-3 global
template <typename T>
using ParamsH = ParamsGT<T, 2>;   // modes 4 and 3 in the block, modes 1-2 global

// Fused CG step B1': the apply kernel also
// forms its own input, P_new = D + beta P_old (D = R, or Z in PCG), applies the
// pending C := C + alpha P_old and writes P_new, so one HBM pass reads D, P_old
// and C and writes P_new, C and Q (6 words per unknown; Fig. 2's order).
template <typename T>
struct FuArgs {
    T *x;                 // C (own slabs)
    T *pn;                // P_new (own slabs); P_old is the kernel input a.x
    const CgScalars *sc;  // alpha (of the previous iteration), beta, xupd, done
};

template <typename T, int N4>
struct Cfg {
    static constexpr int NSEG = (N4 + 3) / 4;        // ring segments along i4
    static constexpr int E = (N4 + NSEG - 1) / NSEG; // elements per segment (<= 4: ring 24 doubles)
    static constexpr int NTHR = N4 > 16 ? 512 : 256;
    static constexpr int MINB = NTHR == 512 ? 1 : 2;  // CTAs per SM
    static constexpr bool RING_SHIFT = true;          // mode-1 ring form (see ring_step; the rotating form is kept for reference)
    static constexpr int T3 = NTHR / (T2 * NSEG);    // mode-3 columns per tile
    static_assert(NTHR % (T2 * NSEG) == 0, "unsupported n4");
    // PADDED: when the mode-4 fibre is a multiple of 32 B (n4 = 4, 8, 16, 32 fp64),
    // the T3 fibres a pass-C warp reads at stride n4 fall on the same banks
    // (config 4, n4 = 32: 8x the ideal wavefronts); the slab is then staged by a
    // 4-D TMA box (S3, T3 + 6, PR, 1) whose fibre extent S3 = n4 + 16 B overruns
    // the tensor (zero fill), so every shared buffer has fibre pitch S3
    static constexpr bool PADDED = (N4 * (int)sizeof(T)) % 32 == 0;
    static constexpr int S3 = PADDED ? N4 + 16 / (int)sizeof(T) : N4;   // i3 pitch in shared memory
    static constexpr int W = (T3 + 6) * S3;          // halo-extended flat columns
    static constexpr int WI = T3 * S3;               // interior flat columns
    static constexpr int VEC = 16 / (int)sizeof(T);  // TMA coordinate granularity (16 B)
    // two-CTA tiles (PITCHED): the slab box uses 8-element chunks (64 B fp64,
    // 32 B fp32) and a row pitch picked against the pass-B/C bank patterns
    // (pick_pp); measured on config 3: fp64 283 -> 276 us (128-B chunks at a
    // 128-B pitch before), 32-B fp64 chunks 281 us; fp32 249 -> 234 us
    static constexpr bool PITCHED = NTHR == 256;
    static constexpr int UNIT = PITCHED ? 8 : 128 / (int)sizeof(T);
    // ONEBOX: the input map is 4-D (UNIT, n3 n4 / UNIT, n2, n1) and a whole staged
    // slab (PR rows of PP elements) is one TMA box, start aligned to UNIT elements
    // (host picks it when n3 n4 % UNIT == 0; otherwise NB boxes per row for
    // fp64, 16-B chunks for PITCHED fp32)
    static constexpr bool ONEBOX = true;
    static constexpr int NEED = PADDED ? W : W + UNIT - 1;
    static constexpr int boxw_for_nb(int nb) { return ((NEED + nb - 1) / nb + UNIT - 1) / UNIT * UNIT; }
    static constexpr int pick_nb()
    {
        int best = 1, tot = 1 << 30;
        for (int nb = 1; nb <= 12; ++nb) {
            const int bw = boxw_for_nb(nb);
            if (bw <= 256 && nb * bw < tot) { tot = nb * bw; best = nb; }
        }
        return best;
    }
    static constexpr int NB = pick_nb();
    static constexpr int BOXW = boxw_for_nb(NB);
    static constexpr int PP_BOXES = NB * BOXW;       // staged row pitch (128-B multiple)
    static constexpr int BL = 4;                     // pass-B outputs per item
    static constexpr int NBLK = T3 / BL;
    // pass B: each warp covers whole mode-2 rows of the block (RPW rows of N4
    // lanes) so its 32 lanes never put three rows on one bank pair of the
    // 128-B-aligned (TMA) slab rows
    // rows start at lane multiples of LW (N4 rounded up to a power of two): each
    // half-warp phase of a 64-bit access then covers one row of N4 consecutive
    // elements, bank-conflict-free at any row pitch (with rows packed at stride
    // N4 the phase that straddles two rows conflicted: profiles/r03_smem_wavefronts.txt)
    static constexpr int LW = N4 <= 1 ? 1 : N4 <= 2 ? 2 : N4 <= 4 ? 4 : N4 <= 8 ? 8 : N4 <= 16 ? 16 : 32;
    static constexpr int RPW = (32 / LW < T2) ? 32 / LW : T2;
    static constexpr int WPB = (T2 + RPW - 1) / RPW;  // warps per block
    static_assert(N4 <= 32, "pass B lane map");
    static constexpr size_t al(size_t e) { return (e * sizeof(T) + 127) / 128 * 128 / sizeof(T); }
    // row pitches of the intermediate tiles: congruent to N4 modulo one bank
    // sweep (128 B) so that pass-B lanes (i2, i4) of consecutive i2 rows hit
    // consecutive banks (conflict-free)
    static constexpr int BANKS = 128 / (int)sizeof(T);
    static constexpr int WP = W + (((N4 - W) % BANKS) + BANKS) % BANKS;    // U2 pitch
    // RA/U3/RB pitch: the candidate in [WI, WI + BANKS) with the fewest shared-
    // memory wavefronts for the two warp access patterns that read these
    // buffers -- pass B lanes (RPW mode-2 rows x N4) and pass C lanes
    // (32 / T3 mode-2 rows x T3 columns of stride N4) -- counted per 4-byte bank
    // shared-memory wavefronts of one warp access: 64-bit accesses are served per
    // half-warp phase (lanes 0-15, 16-31), each phase costing the largest number
    // of words one 4-byte bank holds; 32-bit accesses as one phase
    static constexpr int wavefronts(int X, int pass)
    {
        constexpr int PH = sizeof(T) == 8 ? 16 : 32;   // lanes per phase
        int total = 0;
        for (int p0 = 0; p0 < 32; p0 += PH) {
            int cnt[32] = {};   // words per 4-byte bank (the lanes' addresses are all distinct)
            int worst = 0;
            for (int l = p0; l < p0 + PH; ++l) {
                if (pass == 0 && (l >= RPW * LW || l % LW >= N4)) continue;
                const int idx = pass == 0 ? (l / LW) * X + l % LW        // pass B
                                          : (l / T3) * X + (l % T3) * S3;  // pass C
                for (int h = 0; h < (int)sizeof(T) / 4; ++h) ++cnt[(idx * ((int)sizeof(T) / 4) + h) % 32];
            }
            for (int b = 0; b < 32; ++b) worst = cnt[b] > worst ? cnt[b] : worst;
            total += worst;
        }
        return total;
    }
    static constexpr int pick_wip()
    {
        int best = WI, bc = 1 << 30;
        for (int X = WI; X < WI + BANKS; ++X) {
            const int c = wavefronts(X, 0) + wavefronts(X, 1);
            if (c < bc) { bc = c; best = X; }
        }
        return best;
    }
    static constexpr int WIP = pick_wip();
    static constexpr int pick_pp()
    {
        if (PADDED) return W;   // the 4-D box lands densely: [PR][T3 + 6][S3]
        if (!PITCHED) return PP_BOXES;
        const int p0 = (NEED + UNIT - 1) / UNIT * UNIT;
        int best = p0, bc = 1 << 30;
        for (int X = p0; X < p0 + BANKS; X += UNIT) {
            const int c = wavefronts(X, 0) + wavefronts(X, 1);
            if (c < bc) { bc = c; best = X; }
        }
        return best;
    }
    static constexpr int PP = pick_pp();             // staged row pitch
    static constexpr size_t U2E = al((size_t)T2 * WP);   // smem buffers, each 128-B aligned
    static constexpr size_t WIE = al((size_t)T2 * WIP);
    static constexpr size_t OUTE = al((size_t)T2 * WI);  // TMA store source: dense [T2][WI]
    static constexpr size_t rest_elems = U2E + 3 * WIE + 2 * OUTE;
    static constexpr size_t stage_elems = al((size_t)PR * PP);
    static constexpr size_t SMEM_CAP = MINB == 1 ? 227 * 1024 : 113 * 1024;   // per CTA
    static constexpr int NSTAGE = ((3 * stage_elems + rest_elems) * sizeof(T) + 256 <= SMEM_CAP) ? 3 : 2;
    static constexpr size_t smem_bytes = (NSTAGE * stage_elems + rest_elems) * sizeof(T) + 128;
    // B1': D stages (NSTAGE_FU) + P_old stages (NSTAGE_FU - 1), RB aliases RA,
    // Q stored from registers (no output staging)
    // (Q stored from registers); XB: C of the next own slab, prefetched with
    // cp.async (each thread its own 16-B vectors: no registers held across passes)
    static constexpr size_t XBE = al((size_t)T2 * WI);
    static constexpr size_t rest_fu = U2E + 2 * WIE + XBE;
    static constexpr int NSTAGE_FU = ((5 * stage_elems + rest_fu) * sizeof(T) + 256 <= SMEM_CAP) ? 3 : 2;
    static constexpr size_t smem_fu = ((2 * NSTAGE_FU - 1) * stage_elems + rest_fu) * sizeof(T) + 128;
    static constexpr bool FU_OK = !PADDED && smem_fu <= SMEM_CAP;
    static_assert(T3 % BL == 0, "T3");
    static_assert(NBLK * WPB <= NTHR / 32, "pass B: one item per warp");
    static_assert(PADDED || WI <= 256, "store box");
    static_assert(!PADDED || (S3 <= 256 && (S3 * sizeof(T)) % 16 == 0), "padded box");
    static_assert(PADDED || PITCHED || ((PR * PP * sizeof(T)) % 128 == 0 && (BOXW * sizeof(T)) % 128 == 0),
                  "TMA alignment");
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2,
                                            int c3)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, const void *src, int c0, int c1, int c2, int c3)
{
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }


// ---------------------------------------------------------------- taps
// rec(r) = taps + (off + r + PADR) * REC; G(r, k) = G[r, r+k], R(r, k) = lambda R[r, r+k]
// (symmetric: G[r, r-k] = G[r-k, r]).  Tables are zero outside the domain rows.
// M: the mode the table belongs to (selects block or global records for ParamsGT)
template <int M, typename T>
__device__ __forceinline__ T tapG(const Params<T> &a, int off, int r, int k)
{
#ifdef TCA_DBG_CONST_TAPS
    if (M != 4) { off = 0; r = 0; }   // timing experiment: compile-time tap addresses (wrong results)
#endif
    return k >= 0 ? a.taps[(off + r + PADR) * REC + k] : a.taps[(off + r + k + PADR) * REC - k];
}
template <int M, typename T>
__device__ __forceinline__ T tapR(const Params<T> &a, int off, int r, int k)
{
#ifdef TCA_DBG_CONST_TAPS
    if (M != 4) { off = 0; r = 0; }
#endif
    return k >= 0 ? a.taps[(off + r + PADR) * REC + 4 + k] : a.taps[(off + r + k + PADR) * REC + 4 - k];
}
template <int M, typename T, int NBM>
__device__ __forceinline__ T tapG(const ParamsGT<T, NBM> &a, int off, int r, int k)
{
    const int i = k >= 0 ? (off + r + PADR) * REC + k : (off + r + k + PADR) * REC - k;
    if constexpr (M == 4 || (M == 3 && NBM >= 2)) return a.taps[i];
    else return __ldg(a.gtaps + i);
}
template <int M, typename T, int NBM>
__device__ __forceinline__ T tapR(const ParamsGT<T, NBM> &a, int off, int r, int k)
{
    const int i = k >= 0 ? (off + r + PADR) * REC + 4 + k : (off + r + k + PADR) * REC + 4 - k;
    if constexpr (M == 4 || (M == 3 && NBM >= 2)) return a.taps[i];
    else return __ldg(a.gtaps + i);
}

// ---------------------------------------------------------------- pass C + ring (per segment)
// Shift-register form (fp32): 6-slot ring: before slab j, acc[k] holds the partial sum of
// output slab j-3+k (k = 0..5).  Slab j finishes output j-3 (emitted), adds its
// contributions to outputs j-2..j+2 while shifting them down one slot (each
// DFMA writes the slot its input vacates: no register moves, no rotation
// copies of the code) and starts output j+3 in slot 5.
template <typename T, int E>
__device__ __forceinline__ void ring_step(T (&acc)[6][E], const T (&s)[E], const T (&q)[E], const T (&pc)[E],
                                          const T (&g1)[7], const T (&r1)[5], T (&ov)[E], bool dot, double &pq)
{
    // s: in-slice Kronecker part (goes through G1), q: in-slice regulariser
    // part (identity in mode 1: added to output j only), pc: p itself (R1).
    T pd[E];                            // p_j where it enters <p, Mp>, else 0 (one select per element)
#pragma unroll
    for (int e = 0; e < E; ++e) pd[e] = dot ? pc[e] : T(0);
#pragma unroll
    for (int e = 0; e < E; ++e) ov[e] = fma(g1[0], s[e], acc[0][e]);   // o = -3: finishes output j-3
#pragma unroll
    for (int o = -2; o <= 2; ++o) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            T v = acc[o + 3][e];
            if (o == 0) pq = fma((double)pd[e], (double)v, pq);   // <p_j, old> (see below)
            v = fma(g1[o + 3], s[e], v);
            v = fma(r1[o + 2], pc[e], v);
            if (o == 0) {
                v += q[e];
                // <p, Mp> without a p history: M is block-symmetric along mode 1,
                // so <p, Mp> = sum_j <p_j, M_jj p_j + 2 sum_{j'<j} M_jj' p_j'> and the
                // slot of output j holds exactly sum_{j'<j} M_jj' p_j' before slab j
                // is added:  contribution = <p_j, old> + <p_j, new>
                pq = fma((double)pd[e], (double)v, pq);
            }
            acc[o + 2][e] = v;
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) acc[5][e] = g1[6] * s[e];               // o = +3: first term of output j+3
}

// fp32 shift ring on sm_100's packed FMA (FFMA2: two elements of a segment per
// instruction, the mode-1 tap broadcast), same summation order as ring_step
template <int E>
__device__ __forceinline__ void ring_step_f2(float (&acc)[6][E], const float (&s)[E], const float (&q)[E],
                                             const float (&pc)[E], const float (&g1)[7], const float (&r1)[5],
                                             float (&ov)[E], bool dot, double &pq)
{
    static_assert(E % 2 == 0, "pairs");
    float pd[E];
#pragma unroll
    for (int e = 0; e < E; ++e) pd[e] = dot ? pc[e] : 0.0f;
#pragma unroll
    for (int h = 0; h < E / 2; ++h) {
        const float2 sh = make_float2(s[2 * h], s[2 * h + 1]), ph = make_float2(pc[2 * h], pc[2 * h + 1]);
        const float2 o = __ffma2_rn(make_float2(g1[0], g1[0]), sh, make_float2(acc[0][2 * h], acc[0][2 * h + 1]));
        ov[2 * h] = o.x;
        ov[2 * h + 1] = o.y;
#pragma unroll
        for (int k = -2; k <= 2; ++k) {
            float2 v = make_float2(acc[k + 3][2 * h], acc[k + 3][2 * h + 1]);
            if (k == 0) {
                pq = fma((double)pd[2 * h], (double)v.x, pq);
                pq = fma((double)pd[2 * h + 1], (double)v.y, pq);
            }
            v = __ffma2_rn(make_float2(g1[k + 3], g1[k + 3]), sh, v);
            v = __ffma2_rn(make_float2(r1[k + 2], r1[k + 2]), ph, v);
            if (k == 0) {
                v.x += q[2 * h];
                v.y += q[2 * h + 1];
                pq = fma((double)pd[2 * h], (double)v.x, pq);
                pq = fma((double)pd[2 * h + 1], (double)v.y, pq);
            }
            acc[k + 2][2 * h] = v.x;
            acc[k + 2][2 * h + 1] = v.y;
        }
        acc[5][2 * h] = g1[6] * s[2 * h];
        acc[5][2 * h + 1] = g1[6] * s[2 * h + 1];
    }
}

// Rotating form (fp64): output slab o lives in slot (o - j0) mod 6; at slab j
// the slot of j-3 is emitted and reused for j+3; the rotation is a compile-time
// parameter (6 copies of the code).  Measured on B200 (config 3): fp64 320 us
// rotating vs 327 us shift-register; fp32 296 us rotating vs 266 us shift.
template <typename T, int E, int ROT>
__device__ __forceinline__ void ring_step_rot(T (&acc)[6][E], const T (&s)[E], const T (&q)[E], const T (&pc)[E],
                                          const T (&g1)[7], const T (&r1)[5], T (&ov)[E], bool dot, double &pq)
{
    // s: in-slice Kronecker part (goes through G1), q: in-slice regulariser
    // part (identity in mode 1: added to output j only), pc: p itself (R1).
    constexpr int SE = (ROT + 3) % 6;   // slot of j-3 == slot of j+3
    T pd[E];                            // p_j where it enters <p, Mp>, else 0 (one select per element)
#pragma unroll
    for (int e = 0; e < E; ++e) pd[e] = dot ? pc[e] : T(0);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        ov[e] = fma(g1[0], s[e], acc[SE][e]);   // o = -3: finishes output j-3
        acc[SE][e] = g1[6] * s[e];              // o = +3: first term of output j+3
    }
#pragma unroll
    for (int o = -2; o <= 2; ++o) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            T v = acc[(ROT + o + 6) % 6][e];
            if (o == 0) pq = fma((double)pd[e], (double)v, pq);   // <p_j, old> (see below)
            v = fma(g1[o + 3], s[e], v);
            v = fma(r1[o + 2], pc[e], v);
            if (o == 0) {
                v += q[e];
                // <p, Mp> without a p history: M is block-symmetric along mode 1,
                // so <p, Mp> = sum_j <p_j, M_jj p_j + 2 sum_{j'<j} M_jj' p_j'> and the
                // slot of output j holds exactly sum_{j'<j} M_jj' p_j' before slab j
                // is added:  contribution = <p_j, old> + <p_j, new>
                pq = fma((double)pd[e], (double)v, pq);
            }
            acc[(ROT + o + 6) % 6][e] = v;
        }
    }
}

template <typename T, int N4, int SEG, typename PA, bool FU>
__device__ __forceinline__ void pass_c(const PA &a, T (&acc)[6][Cfg<T, N4>::E], const T *U3, const T *RB,
                                       const T *P, T *OUT, int pos, int rot, int j, bool live, bool emit, int a2,
                                       int a3, int o0, int o1, double &pq, int qoff)
{
    using C = Cfg<T, N4>;
    constexpr int E = C::E;
    constexpr int e0 = SEG * E;
    constexpr int e1 = (e0 + E < N4) ? e0 + E : N4;
    constexpr int NE = e1 - e0;
    constexpr int ulo = e0 - 3 > 0 ? e0 - 3 : 0;
    constexpr int uhi = e1 + 3 < N4 ? e1 + 3 : N4;
    constexpr int plo = e0 - 2 > 0 ? e0 - 2 : 0;
    constexpr int phi = e1 + 2 < N4 ? e1 + 2 : N4;
    const int i2 = pos / C::T3, i3 = pos % C::T3;
    // mode-1 taps of input slab j: G1[j+o, j], lambda R1[j+o, j] -- fetched first so
    // their latency hides behind the window loads and the mode-4 products
    T g1[7], r1[5];
    const int b1 = __shfl_sync(0xffffffffu, a.off1 + j, 0);   // uniform table row base (LDCU, UR operands)
#pragma unroll
    for (int o = -3; o <= 3; ++o) g1[o + 3] = tapG<1>(a, 0, b1 + o, -o);
#pragma unroll
    for (int o = -2; o <= 2; ++o) r1[o + 2] = tapR<1>(a, 0, b1 + o, -o);
    T s[E], q[E], pc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { s[e] = T(0); q[e] = T(0); pc[e] = T(0); }
    if (live) {
        const T *u3 = U3 + i2 * C::WIP + i3 * C::S3;
        const T *rb = RB + i2 * C::WIP + i3 * C::S3;
        const T *pp = P + (i2 + 3) * C::PP + (i3 + 3) * C::S3;
        T uw[uhi - ulo], pw[phi - plo];
#pragma unroll
        for (int k = ulo; k < uhi; ++k) uw[k - ulo] = u3[k];
#pragma unroll
        for (int k = plo; k < phi; ++k) pw[k - plo] = pp[k];
#pragma unroll
        for (int e = 0; e < NE; ++e) q[e] = rb[e0 + e];
        // G4 U3 (push form, compile-time taps: constant-bank operands)
#pragma unroll
        for (int k = ulo; k < uhi; ++k)
#pragma unroll
            for (int e = e0; e < e1; ++e)
                if (k - e >= -3 && k - e <= 3) s[e - e0] = fma(tapG<4>(a, 0, e, k - e), uw[k - ulo], s[e - e0]);
        // lambda R4 p
#pragma unroll
        for (int k = plo; k < phi; ++k)
#pragma unroll
            for (int e = e0; e < e1; ++e)
                if (k - e >= -2 && k - e <= 2) q[e - e0] = fma(tapR<4>(a, 0, e, k - e), pw[k - plo], q[e - e0]);
#pragma unroll
        for (int e = 0; e < NE; ++e) pc[e] = pw[e0 + e - plo];
    }
    T *out;
    bool st = emit;
    if constexpr (FU) {   // OUT: output slab j-3 in HBM; qoff: this thread's element in it (-1: clipped)
        out = OUT + qoff + e0;
        st = emit && qoff >= 0;
    } else {
        out = OUT + (pos / C::T3) * C::WI + (pos % C::T3) * C::S3 + e0;
    }
    T ov[E];
    const bool dot = a.pq_part != nullptr && j >= o0 && j < o1;   // input slab j is one of this CTA's
    if constexpr (C::RING_SHIFT && std::is_same<T, float>::value && E % 2 == 0 && TCA_RING_F2) {
        ring_step_f2<E>(acc, s, q, pc, g1, r1, ov, dot, pq);
    } else if constexpr (C::RING_SHIFT) {
        ring_step<T, E>(acc, s, q, pc, g1, r1, ov, dot, pq);
    } else {
        switch (rot) {
#define TCA_ROT(R)                                                      \
    case R:                                                             \
        ring_step_rot<T, E, R>(acc, s, q, pc, g1, r1, ov, dot, pq);     \
        break;
            TCA_ROT(0) TCA_ROT(1) TCA_ROT(2) TCA_ROT(3) TCA_ROT(4) default: ring_step_rot<T, E, 5>(acc, s, q, pc, g1, r1, ov, dot, pq);
#undef TCA_ROT
        }
    }
    if (st) {
#pragma unroll
        for (int e = 0; e < NE; ++e) out[e] = ov[e];
    }
}

template <typename T, int N4, int SEG, typename PA, bool FU>
__device__ __forceinline__ void pass_c_dispatch(const PA &a, T (&acc)[6][Cfg<T, N4>::E], const T *U3,
                                                const T *RB, const T *P, T *OUT, int seg, int pos, int rot, int j,
                                                bool live, bool emit, int a2, int a3, int o0, int o1, double &pq,
                                                int qoff)
{
    if constexpr (SEG < Cfg<T, N4>::NSEG) {
        if (seg == SEG) pass_c<T, N4, SEG, PA, FU>(a, acc, U3, RB, P, OUT, pos, rot, j, live, emit, a2, a3, o0, o1, pq, qoff);
        else pass_c_dispatch<T, N4, SEG + 1, PA, FU>(a, acc, U3, RB, P, OUT, seg, pos, rot, j, live, emit, a2, a3, o0, o1, pq, qoff);
    }
}

// ---------------------------------------------------------------- pass B (compile-time block B)
template <typename T, int N4, int B, typename PA>
__device__ __forceinline__ void pass_b(const PA &a, const T *U2, const T *RA, const T *P, T *U3, T *RB,
                                       int a3, int warp, int lane)
{
    using C = Cfg<T, N4>;
    if constexpr (B < C::NBLK) {
        if (warp / C::WPB != B) {
            pass_b<T, N4, B + 1, PA>(a, U2, RA, P, U3, RB, a3, warp, lane);
            return;
        }
        constexpr int h0b = B * C::BL;
        const int r3 = __shfl_sync(0xffffffffu, a.off3 + a3 + h0b, 0);   // uniform table row base (all lanes)
        if (lane >= C::RPW * C::LW || lane % C::LW >= N4) return;
        const int i2 = (warp % C::WPB) * C::RPW + lane / C::LW, i4 = lane % C::LW;
        if (i2 >= T2) return;
        constexpr int h0 = B * C::BL;
        const T *u2 = U2 + i2 * C::WP + h0 * C::S3 + i4;
        const T *pp = P + (i2 + 3) * C::PP + (h0 + 1) * C::S3 + i4;
        const int ob = i2 * C::WIP + h0 * C::S3 + i4;
        T v[C::BL + 6], w[C::BL + 4], u[C::BL], rr[C::BL];
#pragma unroll
        for (int m = 0; m < C::BL + 6; ++m) v[m] = u2[m * C::S3];
#pragma unroll
        for (int m = 0; m < C::BL + 4; ++m) w[m] = pp[m * C::S3];
#pragma unroll
        for (int o = 0; o < C::BL; ++o) { u[o] = T(0); rr[o] = RA[ob + o * C::S3]; }
        // pull form, one output row at a time: the row's 12 taps can be loaded
        // (uniform) ahead of its 12 DFMAs; same summation order as the push form
        // taps of row o+1 are fetched while row o computes (hand pipelining:
        // the scheduler otherwise issues each LDCU right before its DFMA)
        T tg[2][7], tr[2][5];
#pragma unroll
        for (int k = -3; k <= 3; ++k) tg[0][k + 3] = tapG<3>(a, 0, r3, k);
#pragma unroll
        for (int k = -2; k <= 2; ++k) tr[0][k + 2] = tapR<3>(a, 0, r3, k);
#pragma unroll
        for (int o = 0; o < C::BL; ++o) {
            if (o + 1 < C::BL) {
#pragma unroll
                for (int k = -3; k <= 3; ++k) tg[(o + 1) & 1][k + 3] = tapG<3>(a, 0, r3 + o + 1, k);
#pragma unroll
                for (int k = -2; k <= 2; ++k) tr[(o + 1) & 1][k + 2] = tapR<3>(a, 0, r3 + o + 1, k);
            }
#pragma unroll
            for (int k = -3; k <= 3; ++k) u[o] = fma(tg[o & 1][k + 3], v[o + 3 + k], u[o]);
#pragma unroll
            for (int k = -2; k <= 2; ++k) rr[o] = fma(tr[o & 1][k + 2], w[o + 2 + k], rr[o]);
        }
#pragma unroll
        for (int o = 0; o < C::BL; ++o) {
            U3[ob + o * C::S3] = u[o];
            RB[ob + o * C::S3] = rr[o];
        }
    }
}

// ---------------------------------------------------------------- kernel
template <typename T> struct V16;   // 16-byte vectors (B1' streaming parts)
template <> struct V16<double> { using V = double2; };
template <> struct V16<float> { using V = float4; };
__device__ __forceinline__ double2 v_axpy(double2 y, double a, double2 x) { return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y)); }
__device__ __forceinline__ float4 v_axpy(float4 y, float a, float4 x)
{
    return make_float4(fmaf(a, x.x, y.x), fmaf(a, x.y, y.y), fmaf(a, x.z, y.z), fmaf(a, x.w, y.w));
}

// Deferred C update (MODE 2): one extra warp per CTA streams
// C := C + alpha P_prev over the CTA's share of the vector while the other
// NTHR threads apply the operator.  P_prev is the previous iteration's search
// direction (kept in the other buffer of a ping-pong pair) and alpha its step
// (sc->alpha, valid when sc->xupd): the x update of Fig. 2
// executed one iteration late, so the apply -- bound inside the SM, its DRAM
// traffic a fraction of the peak -- carries the 3 words of the x update that
// the vector kernels otherwise add to every iteration.  Loads: 16-B vectors,
// XU of C and of P_prev in flight per lane (the DRAM latency is hidden by
// the outstanding loads, not by other warps).
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Deferred C update (MODE 2): one extra warp per CTA streams
// C := C + alpha P_prev over the CTA's share of the vector while the other
// NTHR threads apply the operator.  P_prev is the previous iteration's search
// direction (the other buffer of a ping-pong pair) and alpha its step
// (sc->alpha, valid when sc->xupd): the x update of Fig. 2
// executed one iteration late, so the apply -- bound inside the SM, its DRAM
// traffic a fraction of the peak -- carries the 3 words of the x update that
// the vector kernels otherwise add to every iteration.  Chunks of the share are
// bulk-prefetched into L2 two ahead of their 16-B loads (XU vectors of C and of
// P_prev in flight per lane).  Used where the extra warp costs no occupancy
// (fp32: 95 registers; fp64's 116-register body would be cut to 96 and spill).
template <typename T>
__device__ __forceinline__ void x_stream(const FuArgs<T> &f, size_t n, int lane)
{
    if (!f.sc->xupd) return;   // no valid alpha: first iteration, or the solve stopped earlier
    const T alpha = (T)f.sc->alpha;
    using V = typename V16<T>::V;
    constexpr int VW = 16 / (int)sizeof(T);
    constexpr int XU = 8;
    constexpr int CH = 32 * XU * 4;   // vectors per chunk
    const size_t nv = n / VW;
    const size_t v0 = nv * blockIdx.x / gridDim.x, v1 = nv * (blockIdx.x + 1) / gridDim.x;
    V *xv = reinterpret_cast<V *>(f.x);
    const V *pv = reinterpret_cast<const V *>(f.pn);
    auto pf = [&](size_t c0) {
        if (lane == 0 && c0 < v1) {
            const size_t c1 = c0 + CH < v1 ? c0 + CH : v1;
            prefetch_l2(xv + c0, (unsigned)((c1 - c0) * 16));
            prefetch_l2(pv + c0, (unsigned)((c1 - c0) * 16));
        }
    };
    pf(v0);
    pf(v0 + CH);
    for (size_t c = v0; c < v1; c += CH) {
        pf(c + 2 * CH);
        const size_t ce = c + CH < v1 ? c + CH : v1;
        size_t i = c + lane;
        for (; i + (XU - 1) * 32 < ce; i += XU * 32) {
            V xr[XU], pr[XU];
#pragma unroll
            for (int u = 0; u < XU; ++u) {
                xr[u] = __ldcs(xv + i + u * 32);
                pr[u] = __ldcs(pv + i + u * 32);
            }
#pragma unroll
            for (int u = 0; u < XU; ++u) __stcs(xv + i + u * 32, v_axpy(xr[u], alpha, pr[u]));
        }
        for (; i < ce; i += 32) __stcs(xv + i, v_axpy(__ldcs(xv + i), alpha, __ldcs(pv + i)));
    }
    if (blockIdx.x == 0)   // scalar tail
        for (size_t k = nv * VW + lane; k < n; k += 32) f.x[k] = fma(alpha, f.pn[k], f.x[k]);
}

// CTA barrier of the NTHR operator threads (MODE 2: the streaming warp does not take part)
template <int MODE, int NTHR>
__device__ __forceinline__ void cta_sync()
{
    if constexpr (MODE == 2) asm volatile("bar.sync 1, %0;\n" ::"n"(NTHR) : "memory");
    else __syncthreads();
}

// MODE: 0 the apply; 1 the fused CG step B1' (FuArgs: C, P_new); 2 the apply
// with the deferred C update (an extra streaming warp; FuArgs: C, P_prev as pn)
template <typename T, int N4, typename PA, int MODE>
__device__ __forceinline__ void band_apply_body(const CUtensorMap *__restrict__ xmp, const CUtensorMap *__restrict__ ymp,
                                                const PA &a, const CUtensorMap *__restrict__ rmp, const FuArgs<T> &f)
{
    using C = Cfg<T, N4>;
    constexpr bool FU = MODE == 1;
    constexpr int W = C::W, WI = C::WI, PP = C::PP, T3 = C::T3, E = C::E, NTHR = C::NTHR;
    constexpr int NS = FU ? C::NSTAGE_FU : C::NSTAGE;   // input stages
    const int dbg = TCA_BAND_DBG ? a.dbg : 0;   // phase switches (measurement builds only)
    if constexpr (MODE == 2) {
        if (threadIdx.x >= NTHR) {   // the streaming warp
            if (!(dbg & 4096)) x_stream<T>(f, (size_t)a.n1 * a.n2 * a.n3 * N4, threadIdx.x & 31);
            return;
        }
    }
    if constexpr (FU) {
        if (*a.done) {   // stopped: only the pending C := C + alpha P_old of the last iteration
            if (f.sc->xupd) {
                const T alpha = (T)f.sc->alpha;
                const size_t n = (size_t)a.n1 * a.n2 * a.n3 * N4;
                const T *po = a.x + (size_t)a.xoff * a.n2 * a.n3 * N4;
                for (size_t i = blockIdx.x * (size_t)NTHR + threadIdx.x; i < n; i += (size_t)gridDim.x * NTHR)
                    f.x[i] = fma(alpha, po[i], f.x[i]);
            }
            return;
        }
    } else {
        if (a.done && *a.done) {
            if constexpr (MODE == 0 && NTHR == kRedThreads)   // finaliser 1 of a stopped solve: no x update
                if (a.fin_sc && blockIdx.x == 0 && threadIdx.x == 0) a.fin_sc->xupd = 0;
            return;
        }
    }
    if (dbg & 16) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    T *Pst = reinterpret_cast<T *>(smem_raw + 128);
    T *POst = Pst + NS * C::stage_elems;                                   // B1': P_old stages
    T *U2 = FU ? POst + (NS - 1) * C::stage_elems : Pst + NS * C::stage_elems;
    T *RA = U2 + C::U2E;
    T *U3 = RA + C::WIE;
    T *RB = FU ? RA : U3 + C::WIE;   // B1': pass B updates RA in place
    T *OUTB = RB + C::WIE;   // [2][OUTE] (not used by B1')
    T *XB = U3 + C::WIE;     // B1': C of the next own slab, [vector][VW]
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    // B1' scalars of this step: P_new = D + beta P_old, C += alpha P_old (xu)
    T alpha = T(0), beta = T(0);
    bool xu = false;
    if constexpr (FU) {
        alpha = (T)f.sc->alpha;
        beta = (T)f.sc->beta;
        xu = f.sc->xupd != 0;
    }
    using V = typename V16<T>::V;
    constexpr int VW = 16 / (int)sizeof(T);
    constexpr int NVR = WI / VW;                     // 16-B vectors per interior row
    constexpr int NV = T2 * NVR;
    constexpr int XIT = (NV + NTHR - 1) / NTHR;      // vectors per thread
    static_assert(WI % VW == 0, "interior rows are whole vectors");
    const int F = a.n3 * N4;                         // row stride (elements)
    const size_t slabE = (size_t)a.n2 * F;           // slab stride (elements)
    // xmp/ymp: tensor maps in global memory (a descriptor in a >4 KB parameter
    // block is not usable by the TMA unit)
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cta_sync<MODE, NTHR>();
    if (dbg & 32) return;

    const int seg = tid / (NTHR / C::NSEG);   // warp-uniform
    const int pos = tid % (NTHR / C::NSEG);   // (i2, i3) of the ring owner

    // per-CTA schedule (uniform): tile (t2i, t3i) from slab o0, cnt units in total
    int t2i = a.s_tile[blockIdx.x].x, t3i = a.s_tile[blockIdx.x].y;
    int o0 = a.s_o0[blockIdx.x];
    int cnt = a.s_cnt[blockIdx.x];
    unsigned gi = 0, gc = 0;   // slabs issued / consumed (stage = g % NSTAGE, parity (g / NSTAGE) & 1)
    T acc[6][E];
    double pq = 0.0;           // <x, y> partial of this thread's emitted outputs
    for (; cnt > 0; o0 = a.o_next, t3i = (t3i + 1 == a.tiles3) ? 0 : t3i + 1, t2i += (t3i == 0) ? 1 : 0) {
        const int o1 = (a.n1 - o0 < cnt) ? a.n1 : o0 + cnt;
        cnt -= o1 - o0;
        const int a2 = __shfl_sync(0xffffffffu, t2i * T2, 0);   // provably warp-uniform
        const int a3 = __shfl_sync(0xffffffffu, t3i * T3, 0);
        const int b2 = __shfl_sync(0xffffffffu, a.off2 + t2i * T2, 0);   // uniform mode-2 table row base
        const int ca = (a3 - 3) * N4;                              // flat column of staged column 0
        // B1' per-tile element offsets within a slab (-1: outside the domain):
        // this thread's 16-B vectors of the interior, and its ring outputs
        // B1' per-tile element offsets within a slab (-1: outside the domain):
        // this thread's 16-B vectors of the interior, and its ring outputs
        int voff[XIT], qoff = -1;
        auto fetch_x = [&](int js) {   // cp.async of C's slab js (own vectors) into XB
            const T *xg = f.x + (size_t)js * slabE;
#pragma unroll
            for (int it = 0; it < XIT; ++it)
                if (voff[it] >= 0) cp_async16(XB + (tid + it * NTHR) * VW, xg + voff[it]);
            cp_async_commit();
        };
        if constexpr (FU) {
#pragma unroll
            for (int it = 0; it < XIT; ++it) {
                const int v = tid + it * NTHR, r = v / NVR, cv = v % NVR;
                voff[it] = (v < NV && a2 + r < a.n2 && a3 * N4 + cv * VW < F) ? (a2 + r) * F + a3 * N4 + cv * VW : -1;
            }
            const int q2 = a2 + pos / C::T3, q3 = a3 + pos % C::T3;
            qoff = (q2 < a.n2 && q3 < a.n3) ? q2 * F + q3 * N4 : -1;
            const int jx0 = o0 > -a.xoff ? o0 : -a.xoff;   // first own slab
            if (xu && jx0 < o1) fetch_x(jx0);
        }
        // boxes start 16-B aligned (per-row boxes) or UNIT-aligned (one box per slab)
        const bool onebox = C::PITCHED || (C::ONEBOX && a.onebox);
        const int cal = onebox ? C::UNIT : C::VEC;
        int delta = ((ca % cal) + cal) % cal;
        int cchunk = (ca - delta) / C::UNIT;                       // onebox: first chunk
        if constexpr (C::PITCHED) {   // one box always; 16-B chunks when n3 n4 % UNIT != 0
            if (!a.onebox) {
                delta = ((ca % C::VEC) + C::VEC) % C::VEC;
                cchunk = (ca - delta) / C::VEC;
            }
        }
        if constexpr (C::PADDED) {   // 4-D box (fibre, i3, i2, slab): staged column 0 is i3 = a3 - 3
            delta = 0;
            cchunk = a3 - 3;
        }
        const int j0 = o0 - 3, j1 = o1 + 3;
        const int jb = j0 > -a.xoff ? j0 : -a.xoff, je = j1 < a.nin - a.xoff ? j1 : a.nin - a.xoff;
#pragma unroll
        for (int s = 0; s < 6; ++s)
#pragma unroll
            for (int e = 0; e < E; ++e) acc[s][e] = T(0);

        // prologue: stage the first NSTAGE-1 in-range slabs
        // stage slab js: NB boxes per staged row, issued round-robin by lane 0 of
        // every warp (one warp issuing all of them serialises ~30 UTMALDG)
        auto issue = [&](int js) {
            if (dbg & 256) { ++gi; return; }   // compute-only timing: no loads
            const unsigned st = gi % NS;
            T *dst = Pst + st * C::stage_elems;
            if constexpr (FU) {   // D and P_old slabs, one barrier (host guarantees one box per slab)
                if (tid == 0) {
                    mbar_arrive_expect_tx(bar + st, (unsigned)(2 * PR * PP * sizeof(T)));
                    tma_load_4d(dst, rmp, bar + st, 0, cchunk, a2 - 3, js + a.xoff);
                    tma_load_4d(POst + (gi % (NS - 1)) * C::stage_elems, xmp, bar + st, 0, cchunk, a2 - 3,
                                js + a.xoff);
                }
                ++gi;
                return;
            }
            if (onebox || C::PADDED) {
                if (tid == 0) {
                    mbar_arrive_expect_tx(bar + st, (unsigned)(PR * PP * sizeof(T)));
                    tma_load_4d(dst, xmp, bar + st, 0, cchunk, a2 - 3, js + a.xoff);
                }
                ++gi;
                return;
            }
            if (tid == 0) mbar_arrive_expect_tx(bar + st, (unsigned)(C::NB * PR * C::BOXW * sizeof(T)));
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < (C::NB * PR + NTHR / 32 - 1) / (NTHR / 32); ++k) {
                    const int b = warp + k * (NTHR / 32);
                    if (b < C::NB * PR) {
                        const int r = b / C::NB, h = b % C::NB;
                        tma_load_3d(dst + r * PP + h * C::BOXW, xmp, bar + st,
                                    ca - delta + h * C::BOXW, a2 - 3 + r,
                                    js + a.xoff);
                    }
                }
            }
            ++gi;
        };
        if (!(dbg & 8))
            for (int js = jb; js < je && js < jb + NS - 1; ++js) issue(js);
        int next = jb + NS - 1;   // next slab to stage
        int rot = 0;                     // ring rotation (rotating form only)
        int pending = -1;                // output slab whose staging buffer awaits its TMA store
#pragma unroll 1
        for (int j = j0; j < j1; ++j) {
            const bool live = j >= jb && j < je && !(dbg & 8);
            T *P = Pst + (gc % NS) * C::stage_elems + delta;
            if (live && !(dbg & (128 | 256))) mbar_wait(bar + gc % NS, (gc / NS) & 1);
            const T *PO = POst + (gc % (NS > 1 ? NS - 1 : 1)) * C::stage_elems + delta;   // B1': P_old slab j
            const bool own = FU && live && j >= o0 && j < o1;

            // ---- pass A: G2 (all halo-extended columns), lambda R2 (interior columns)
            if (live && !(dbg & 4)) {
#pragma unroll 1
                for (int t = tid; t < W; t += NTHR) {
                    // interior columns (G2 and R2) on the first threads, the halo
                    // columns (G2 only) after them: the heavy columns fill warps
                    // 0-3, one per scheduler, instead of doubling up on one
                    int c = t;
                    if constexpr (W <= NTHR) c = t < WI ? 3 * C::S3 + t : (t < WI + 3 * C::S3 ? t - WI : t);
                    T v[PR];
                    if (FU && !(dbg & 2048)) {   // P_new := D + beta P_old on the staged slab (halo included)
#pragma unroll
                        for (int s = 0; s < PR; ++s) {
                            v[s] = fma(beta, PO[s * PP + c], P[s * PP + c]);
                            if (s >= 3 && s < 3 + T2) P[s * PP + c] = v[s];   // rows read by passes B, C
                        }
                    } else {
#pragma unroll
                        for (int s = 0; s < PR; ++s) v[s] = P[s * PP + c];
                    }
                    T u[T2];
#pragma unroll
                    for (int r = 0; r < T2; ++r) u[r] = T(0);
                    // symmetric band (G[r, r+k] = G[r+k, r]): each stored record tap
                    // G[r, r+k] (k > 0) serves output r (input row r+k) and output r+k
                    // (input row r) -- 38 uniform tap loads for the 56 DFMAs of G2 on
                    // 8 rows (the records of halo rows -3..-1 cover the top edge)
#pragma unroll
                    for (int r = -3; r < T2; ++r) {
#pragma unroll
                        for (int k = (r < 0 ? -r : 0); k <= 3; ++k) {
                            const T t = tapG<2>(a, 0, b2 + r, k);
                            if (r >= 0) u[r] = fma(t, v[r + 3 + k], u[r]);
                            if (k > 0 && r + k < T2) u[r + k] = fma(t, v[r + 3], u[r + k]);
                        }
                    }
#pragma unroll
                    for (int r = 0; r < T2; ++r) U2[r * C::WP + c] = u[r];
                    const int ci = c - 3 * C::S3;
                    if (ci >= 0 && ci < WI) {
#pragma unroll
                        for (int r = 0; r < T2; ++r) u[r] = T(0);
#pragma unroll
                        for (int r = -2; r < T2; ++r) {
#pragma unroll
                            for (int k = (r < 0 ? -r : 0); k <= 2; ++k) {
                                const T t = tapR<2>(a, 0, b2 + r, k);
                                if (r >= 0) u[r] = fma(t, v[r + 3 + k], u[r]);
                                if (k > 0 && r + k < T2) u[r + k] = fma(t, v[r + 3], u[r + k]);
                            }
                        }
#pragma unroll
                        for (int r = 0; r < T2; ++r) RA[r * C::WIP + ci] = u[r];
                    }
                }
            }
            if (FU && own && xu && !(dbg & 512)) {   // C := C + alpha P_old (interior of slab j)
                cp_async_wait_all();
                T *xs = f.x + (size_t)j * slabE;
#pragma unroll
                for (int it = 0; it < XIT; ++it) {
                    const int v = tid + it * NTHR;
                    if (voff[it] >= 0) {
                        const V xv = *reinterpret_cast<const V *>(XB + v * VW);
                        const V po = *reinterpret_cast<const V *>(PO + (v / NVR + 3) * PP + 3 * N4 + (v % NVR) * VW);
                        *reinterpret_cast<V *>(xs + voff[it]) = v_axpy(xv, alpha, po);
                    }
                }
                if (j + 1 < o1) fetch_x(j + 1);
            }
            cta_sync<MODE, NTHR>();   // bar1: U2/RA complete; all threads finished slab j-1

            if (pending >= 0) {   // uniform: every thread tracks the same pending slab
                if (tid == 0 && !(dbg & (1 | 256))) {
                    // staging buffer of output slab `pending` (written in pass C of slab pending+3)
                    if constexpr (C::PADDED) tma_store_4d(ymp, OUTB + ((pending + 3) & 1) * C::OUTE, 0, a3, a2, pending);
                    else tma_store_3d(ymp, OUTB + ((pending + 3) & 1) * C::OUTE, a3 * N4, a2, pending);
                    bulk_commit();
                    bulk_wait_read<1>();
                }
                pending = -1;
            }
            if (live && next < je && !(dbg & 64)) {   // stage slab `next` into the stage last read in slab j-1
                issue(next);
                ++next;
            }
            if (own && !(dbg & 1024)) {   // B1': P_new of slab j (own interior) to HBM
                T *ps = f.pn + (size_t)j * slabE;
#pragma unroll
                for (int it = 0; it < XIT; ++it) {
                    const int v = tid + it * NTHR;
                    if (voff[it] >= 0)
                        *reinterpret_cast<V *>(ps + voff[it]) =
                            *reinterpret_cast<const V *>(P + (v / NVR + 3) * PP + 3 * N4 + (v % NVR) * VW);
                }
            }
            // ---- pass B: G3 on U2, lambda R3 on p (8 outputs along i3 per item; item = warp)
            if (live && !(dbg & 4)) pass_b<T, N4, 0, PA>(a, U2, RA, P, U3, RB, a3, warp, lane);
            cta_sync<MODE, NTHR>();   // bar2: U3/RB complete

            // ---- pass C + mode-1 ring + emission of output slab j-3
            const bool emit = (j - 3 >= o0) && (j - 3 < o1);
            T *OUT = FU ? a.y + (ptrdiff_t)(j - 3) * (ptrdiff_t)slabE : OUTB + (j & 1) * C::OUTE;
            if (!(dbg & 2)) pass_c_dispatch<T, N4, 0, PA, FU>(a, acc, U3, RB, P, OUT, seg, pos, rot, j, live, emit, a2, a3, o0, o1, pq, qoff);
            if (!FU && emit) {
                fence_proxy_async();
                pending = j - 3;
            }
            if (live) ++gc;
            rot = rot == 5 ? 0 : rot + 1;
        }
        cta_sync<MODE, NTHR>();
        if (!FU && pending >= 0) {
            if (tid == 0 && !(dbg & (1 | 256))) {
                if constexpr (C::PADDED) tma_store_4d(ymp, OUTB + ((pending + 3) & 1) * C::OUTE, 0, a3, a2, pending);
                else tma_store_3d(ymp, OUTB + ((pending + 3) & 1) * C::OUTE, a3 * N4, a2, pending);
                bulk_commit();
            }
            pending = -1;
        }
        if (!FU) {
            if (tid == 0) bulk_wait<0>();   // the next segment rewrites the staging buffers
            cta_sync<MODE, NTHR>();
        }
    }
    if (a.pq_part) {   // fixed-order CTA reduction of the <x, y> partials (deterministic)
        double *red = reinterpret_cast<double *>(smem_raw + 128);   // stage memory is idle now
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pq += __shfl_xor_sync(0xffffffffu, pq, o);
        if (lane == 0) red[warp] = pq;
        cta_sync<MODE, NTHR>();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NTHR / 32; ++w) t += red[w];
            a.pq_part[blockIdx.x] = t;
        }
        if constexpr (MODE == 0 && NTHR == kRedThreads)
            if (a.fin_sc) fin_last_cta(1, 0, a.pq_part, a.fin_sc, a.fin_hist, red);   // alpha in the last CTA
    }
}

template <typename T, int N4, typename PA, int MODE>
__global__ void __launch_bounds__(Cfg<T, N4>::NTHR + (MODE == 2 ? 32 : 0), Cfg<T, N4>::MINB)
band_apply_kernel(const CUtensorMap *__restrict__ xmp, const CUtensorMap *__restrict__ ymp,
                  const __grid_constant__ PA a, const CUtensorMap *__restrict__ rmp, const __grid_constant__ FuArgs<T> f)
{
    band_apply_body<T, N4, PA, MODE>(xmp, ymp, a, rmp, f);
}


// ---------------------------------------------------------------- host side
template <typename T, int N4, typename PA, int MODE>
tca_status launch_n4(const tca_operator *op, const PA &prm, cudaStream_t s, const CUtensorMap *xm,
                     const CUtensorMap *ym, const CUtensorMap *rm, const FuArgs<T> &fa)
{
    using C = Cfg<T, N4>;
    constexpr bool FU = MODE == 1;
    if constexpr (FU && !C::FU_OK) {
        return fail(TCA_ERR_INVALID_ARG, "fused CG step: shape does not fit shared memory");
    } else {
        constexpr size_t smem = FU ? C::smem_fu : C::smem_bytes;
        auto kern = band_apply_kernel<T, N4, PA, MODE>;
        TCA_TRY(set_max_dynamic_smem((const void *)kern, smem));
        count_launch();
        const int grid = MODE == 1 ? op->band_grid_fu : MODE == 2 ? op->band_grid_dx : op->band_grid;
        kern<<<(unsigned)grid, C::NTHR + (MODE == 2 ? 32 : 0), smem, s>>>(xm, ym, prm, rm, fa);
        TCA_CUDA_TRY(cudaGetLastError());
        return TCA_OK;
    }
}

#define TCA_BAND_N4_LIST(X) X(1) X(2) X(4) X(7) X(8) X(15) X(16) X(32)

template <typename T>
int t3_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::T3;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int pp_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::PP;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int onebox_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::ONEBOX ? 1 : 0;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int unit_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::UNIT;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int pitched_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::PITCHED ? 1 : 0;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int minb_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::MINB;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 1;
}

template <typename T>
int boxw_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::BOXW;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int padded_s3_for(int n4)   // fibre pitch of the padded 4-D staging, 0 when the layout is flat
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::PADDED ? Cfg<T, n>::S3 : 0;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int fu_ok_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::FU_OK ? 1 : 0;
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename PA>
tca_status launch_dispatch(const tca_operator *op, const PA &prm, cudaStream_t s, const CUtensorMap *xm,
                           const CUtensorMap *ym)
{
    using T = typename PA::value_type;
    const FuArgs<T> none{};
    switch ((int)op->n[3]) {
#define TCA_CASE(n) \
    case n: return launch_n4<T, n, PA, 0>(op, prm, s, xm, ym, nullptr, none);
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return fail(TCA_ERR_INVALID_ARG, "band apply: unsupported n4");
}

// B1' (fused CG step): xm = P_old map, rm = D map, output Q = prm.y
template <typename PA>
tca_status launch_dispatch_fu(const tca_operator *op, const PA &prm, cudaStream_t s, const CUtensorMap *xm,
                              const CUtensorMap *ym, const CUtensorMap *rm, const FuArgs<typename PA::value_type> &fa)
{
    using T = typename PA::value_type;
    switch ((int)op->n[3]) {
#define TCA_CASE(n) \
    case n: return launch_n4<T, n, PA, 1>(op, prm, s, xm, ym, rm, fa);
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return fail(TCA_ERR_INVALID_ARG, "band apply: unsupported n4");
}

// apply with the deferred C update (MODE 2): fa = {C, P_prev, scalars}
template <typename PA>
tca_status launch_dispatch_dx(const tca_operator *op, const PA &prm, cudaStream_t s, const CUtensorMap *xm,
                              const CUtensorMap *ym, const FuArgs<typename PA::value_type> &fa)
{
    using T = typename PA::value_type;
    switch ((int)op->n[3]) {
#define TCA_CASE(n) \
    case n: return launch_n4<T, n, PA, 2>(op, prm, s, xm, ym, nullptr, fa);
        TCA_BAND_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return fail(TCA_ERR_INVALID_ARG, "band apply: unsupported n4");
}

}  // namespace band
}  // namespace tca
