// tca_band2.cuh -- fibre-owner fused banded apply (v3, opt-in TCA_BAND_V2=1),
// 9 <= n4 <= 16, fp64.
//
//   q = (G_1 (x) G_2 (x) G_3 (x) G_4) p + sum_d (mode-d lambda R_d) p
//
// Same operator as tca_band_impl.cuh (Eq. 4, applied as
// successive one-dimensional transformations in an order Eq. 5, PAPER.md:75-81,
// allows; Eq. 9's Kronecker-sum regulariser), re-partitioned
// to cut the shared-memory traffic that bounds band_apply_kernel (about 24
// words per unknown):
//
//   * one persistent 512-thread CTA per SM owns a tile of T2 = 8 mode-2 rows x
//     T3 = 16 mode-3 columns x all n4 and streams mode 1 slab by slab; the
//     input slab (halo 3 in i2 and i3) arrives by one TMA box;
//   * AB warps (8, 88 registers): mode 2 (column owners over the 8 rows,
//     symmetric uniform taps) into U2, then mode 3 (column owners along i3, 8
//     outputs each) with lambda R2 + lambda R3 into U3 and RB;
//   * C warps (8, 168 registers via setmaxnreg): each thread owns half of a
//     mode-4 fibre (8 elements; the half is warp-uniform, so mode-4 taps are
//     compile-time): mode 4 in registers, the 6-slot mode-1 ring, CG's <p, q>,
//     the output staged for one TMA tensor store per slab;
//   * AB runs up to two slabs ahead of C through double-buffered U3/RB and
//     named barriers; C releases each input stage and issues the next TMA load.
// Shared-memory traffic per unknown: about 17 words.  Measured on config 3:
// 271 us vs 277 us for band_apply_kernel -- the pipeline's synchronisation and
// instruction-fetch overhead (88 us with all compute off) eats the saving
// (DESIGN.md 6.1), so band_apply_kernel stays the default.
#pragma once

#include "tca_band_impl.cuh"

#include <cstdio>
#include <type_traits>

namespace tca {
namespace band2 {

using band::Params;
using band::ParamsBase;
using band::ParamsG;
using band::ParamsH;
using band::tapG;
using band::tapR;

constexpr int T2 = 8;          // mode-2 rows per tile
constexpr int T3 = 16;         // mode-3 columns per tile
constexpr int PR = T2 + 6;     // staged rows (halo 3 + 3)
constexpr int CW = T3 + 6;     // staged / U2 mode-3 columns (halo 3 + 3)
constexpr int N4P = 16;        // padded mode-4 extent of U2
constexpr int FP = 18;         // fibre pitch of RA/RB/U3 (16 + 2: C's lanes on distinct bank groups)
constexpr int NAB = 256, NC = 256;
constexpr int NTHR = NAB + NC;
constexpr int UNIT = 8;        // TMA chunk of the staged slab box (elements)
constexpr int NS = 3;          // input stages

// named barriers (0 is __syncthreads)
constexpr int BAR_AB = 1;         // AB warps (phase boundaries)
constexpr int BAR_FULL = 2;       // +b: AB produced U3/RB[b]          (AB arrive, C sync)
constexpr int BAR_EMPTY = 4;      // +b: C released U3/RB[b]           (C arrive, AB sync)
constexpr int BAR_C = 6;          // C warps: the input stage is read

template <typename T, int N4>
struct Cfg {
    static_assert(N4 >= 9 && N4 <= 16, "v3 takes 9 <= n4 <= 16");
    static constexpr int W = CW * N4;                                   // staged flat columns
    // a tile starts at a3 = 16 t, so the staged box's offset in its first chunk,
    // (3 - a3) n4 mod 8 = -3 n4 mod 8, is the same for every tile
    static constexpr int DELTA = ((-3 * N4) % UNIT + UNIT) % UNIT;
    static constexpr int PP = (W + DELTA + UNIT - 1) / UNIT * UNIT;     // staged row pitch (elements)
    static constexpr size_t al(size_t e) { return (e * sizeof(T) + 127) / 128 * 128 / sizeof(T); }
    static constexpr size_t STG = al((size_t)PR * PP);
    static constexpr size_t U2E = al((size_t)T2 * W);              // [T2][CW * N4] (flat, as staged)
    static constexpr size_t TE = al((size_t)T2 * T3 * FP);   // RA (= RB, updated in place), U3
    static constexpr size_t OUTE = al((size_t)T2 * T3 * N4);  // output staging: dense [T2][T3 n4] (TMA store box)
    static constexpr size_t smem_bytes = 128 + (NS * STG + U2E + 4 * TE + OUTE) * sizeof(T);
    static_assert(smem_bytes <= 227 * 1024, "shared memory");
    static_assert(PP / UNIT <= 256, "TMA box");
};

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n)
{
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// measurement build only (-DTCA_BAND2_PROF): per-phase clock64 sums of block 0
#ifdef TCA_BAND2_PROF
static __device__ unsigned long long g_b2prof[64];
#define B2_PROF_INIT \
    long long _pt = clock64(); \
    long long _pa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define B2_PROF(k) \
    { \
        const long long _n = clock64(); \
        _pa[k] += _n - _pt; \
        _pt = _n; \
    }
#define B2_PROF_DONE(base) \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) \
        for (int _k = 0; _k < 8; ++_k) atomicAdd(&g_b2prof[(base) + _k], (unsigned long long)_pa[_k]);
#else
#define B2_PROF_INIT
#define B2_PROF(k)
#define B2_PROF_DONE(base)
#endif

// ---------------------------------------------------------------- per-CTA schedule
// Segments (tile, output slabs [o0, o1)) in the order of tca_band.cu's
// schedule: CTA b starts at tile s_tile[b] and slab s_o0[b] and processes
// s_cnt[b] (tile, slab) units, tile-major.  A segment takes o1 - o0 + 6 steps
// (input slabs o0-3 .. o1+2: the mode-1 ring's ramps).
struct Sched {
    int t2i, t3i, o0, cnt, n1, tiles3, o_next;
    __device__ bool next(int &a2, int &a3, int &s0, int &s1)
    {
        if (cnt <= 0) return false;
        s0 = o0;
        s1 = (n1 - o0 < cnt) ? n1 : o0 + cnt;
        cnt -= s1 - s0;
        a2 = t2i * T2;
        a3 = t3i * T3;
        o0 = o_next;
        t3i = (t3i + 1 == tiles3) ? 0 : t3i + 1;
        t2i += (t3i == 0) ? 1 : 0;
        return true;
    }
};

// Live input slabs of the CTA in step order (the producer's cursor): slab j of a
// segment is live when the (ghosted) input holds it.
struct LiveCursor {
    Sched sc;
    int a2, a3, j, je, xoff, nin;
    __device__ bool next(int &oa2, int &oa3, int &oj)
    {
        while (j >= je) {
            int s0, s1;
            if (!sc.next(a2, a3, s0, s1)) return false;
            j = max(s0 - 3, -xoff);
            je = min(s1 + 3, nin - xoff);
        }
        oa2 = a2;
        oa3 = a3;
        oj = j++;
        return true;
    }
};

__device__ __forceinline__ int2 stage_of(int a3, int n4)   // first 8-element chunk of the staged box, offset in it
{
    const int ca = (a3 - 3) * n4;
    const int delta = ((ca % UNIT) + UNIT) % UNIT;
    return make_int2((ca - delta) / UNIT, delta);
}


// ---------------------------------------------------------------- C warps
// Thread f of a half: fibre (i2 = a2 + f / 16, i3 = a3 + f % 16), elements
// [8 H, 8 H + 8) of it (H compile-time: mode-4 taps at compile-time offsets).
template <typename T, int N4, int H, typename PA>
__device__ __forceinline__ void c_loop(const CUtensorMap *xmp, const CUtensorMap *ymp, const PA &a, const Sched &sc0,
                                       int gtot, uint64_t *bar, T *Xst, T *RA, T *U3, T *OUT, int f, bool producer,
                                       int dbg, double &pq)
{
    using C = Cfg<T, N4>;
    constexpr int PP = C::PP;
    constexpr int E0 = 8 * H;                                  // first element of this half
    constexpr int E1 = (E0 + 8 < N4) ? E0 + 8 : N4;            // one past the last
    constexpr int NE = E1 - E0;
    constexpr int WLO = (E0 - 3 > 0) ? E0 - 3 : 0;             // U3 window
    constexpr int WHI = (E1 + 3 < N4) ? E1 + 3 : N4;
    constexpr int PLO = (E0 - 2 > 0) ? E0 - 2 : 0;             // p window
    constexpr int PHI = (E1 + 2 < N4) ? E1 + 2 : N4;
    const int r = f >> 4, o = f & 15;
    const int F = a.n3 * N4;
    LiveCursor prod{sc0, 0, 0, 0, 0, a.xoff, a.nin};   // producer cursor (one thread)
    unsigned gi = 0;                                   // live slabs issued
    auto issue = [&]() {
        int pa2, pa3, pj;
        if (!prod.next(pa2, pa3, pj)) return;
        const unsigned st = gi % NS;
        band::mbar_arrive_expect_tx(bar + st, (unsigned)(PR * PP * sizeof(T)));
        band::tma_load_4d(Xst + st * C::STG, xmp, bar + st, 0, stage_of(pa3, N4).x, pa2 - 3, pj + a.xoff);
        ++gi;
    };
    (void)issue;
    if (producer && !(dbg & 4))
        for (int s = 0; s < NS; ++s) issue();
    T acc[6][8];
    unsigned gc = 0;
    B2_PROF_INIT
    Sched sc = sc0;
    int a2, a3, o0, o1, g = 0;
    while (sc.next(a2, a3, o0, o1)) {
#pragma unroll
        for (int k = 0; k < 6; ++k)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[k][e] = T(0);
        const int delta = stage_of(a3, N4).y;
        const int jb = max(o0 - 3, -a.xoff), je = min(o1 + 3, a.nin - a.xoff);
        const bool inside = a2 + r < a.n2 && a3 + o < a.n3;
        for (int j = o0 - 3; j < o1 + 3; ++j, ++g) {
            const int b = g & 1;
            const bool live = j >= jb && j < je;
            const bool emit = j - 3 >= o0 && j - 3 < o1;
            const bool dot = a.pq_part != nullptr && j >= o0 && j < o1;
            // mode-1 taps of input slab j: G1[j+k, j], lambda R1[j+k, j] (uniform registers)
            T g1[7], r1[5];
            const int b1 = __shfl_sync(0xffffffffu, a.off1 + j, 0);
#pragma unroll
            for (int k = -3; k <= 3; ++k) g1[k + 3] = tapG<1>(a, 0, b1 + k, -k);
#pragma unroll
            for (int k = -2; k <= 2; ++k) r1[k + 2] = tapR<1>(a, 0, b1 + k, -k);
            T *out = OUT + r * (T3 * N4) + o * N4;   // staging of output slab j - 3
            if (producer && !(dbg & 8)) band::bulk_wait_read<0>();   // the last store has read OUT
            B2_PROF(0);
            nb_sync(BAR_FULL + b, NAB + NC);
            B2_PROF(1);
            const T *u3 = U3 + b * C::TE + f * FP;
            const T *rb = RA + b * C::TE + f * FP;
            const T *xp = Xst + (gc % NS) * C::STG + delta + (r + 3) * PP + (o + 3) * N4;
            const bool use = live && !(dbg & 2);
            if (live && !(dbg & 4)) band::mbar_wait(bar + gc % NS, (gc / NS) & 1);   // (complete; orders the TMA data)
            // U3, RB and p of the half fibre (+ mode-4 halo), each read once, in a window
            // that slides with the element (a compiler barrier per element keeps the
            // loads from being hoisted above the ring's registers)
            T uw[N4], pw[N4], qw[N4];
#pragma unroll
            for (int k = WLO; k < WHI; ++k) uw[k] = use ? u3[k] : T(0);
#pragma unroll
            for (int k = PLO; k < PHI; ++k) pw[k] = use ? xp[k] : T(0);
#pragma unroll
            for (int k = E0; k < E1; ++k) qw[k] = use ? rb[k] : T(0);
#pragma unroll
            for (int e = E0; e < E1; ++e) {
                if (dbg & 16) break;
                // mode 4 (compile-time taps): s = G4 U3, q = RB + lambda R4 p; pc = p
                // (two partial sums each: shorter dependent chains)
                T s0 = T(0), s1 = T(0), q0 = qw[e], q1 = T(0);
                const T pc = pw[e];
#pragma unroll
                for (int k = (e - 3 > 0 ? e - 3 : 0); k <= (e + 3 < N4 - 1 ? e + 3 : N4 - 1); ++k) {
                    if ((k - e) & 1) s1 = fma(tapG<4>(a, 0, e, k - e), uw[k], s1);
                    else s0 = fma(tapG<4>(a, 0, e, k - e), uw[k], s0);
                }
#pragma unroll
                for (int k = (e - 2 > 0 ? e - 2 : 0); k <= (e + 2 < N4 - 1 ? e + 2 : N4 - 1); ++k) {
                    if ((k - e) & 1) q1 = fma(tapR<4>(a, 0, e, k - e), pw[k], q1);
                    else q0 = fma(tapR<4>(a, 0, e, k - e), pw[k], q0);
                }
                const T s = s0 + s1, q = q0 + q1;
                // mode-1 shift ring (tca_band_impl.cuh ring_step, one element); the finished
                // output element goes straight to HBM
                T(&ac)[6][8] = acc;
                const int i = e - E0;
                const T pd = dot ? pc : T(0);
                if (emit) out[e] = fma(g1[0], s, ac[0][i]);
#pragma unroll
                for (int kk = -2; kk <= 2; ++kk) {
                    T v = ac[kk + 3][i];
                    if (kk == 0) pq = fma((double)pd, (double)v, pq);
                    v = fma(g1[kk + 3], s, v);
                    v = fma(r1[kk + 2], pc, v);
                    if (kk == 0) {
                        v += q;
                        pq = fma((double)pd, (double)v, pq);
                    }
                    ac[kk + 2][i] = v;
                }
                ac[5][i] = g1[6] * s;
            }
            (void)NE;
            (void)inside;
            B2_PROF(2);
            if (emit) band::fence_proxy_async();   // OUT writes -> the TMA store (async proxy)
            if (live || emit) {   // every C thread has read the stage / written OUT
                nb_sync(BAR_C, NC);
                if (live) {
                    ++gc;
                    if (producer && !(dbg & 4)) issue();   // the producer refills the stage
                }
                if (emit && producer && !(dbg & 8)) {
                    band::tma_store_3d(ymp, OUT, a3 * N4, a2, j - 3);
                    band::bulk_commit();
                }
            }
            B2_PROF(3);
            if (g + 2 < gtot) nb_arrive(BAR_EMPTY + b, NAB + NC);
        }
    }
    B2_PROF_DONE(32 + 8 * H)
}

// ---------------------------------------------------------------- kernel
template <typename T, int N4, typename PA>
__global__ void __launch_bounds__(NTHR, 1)
band3_kernel(const CUtensorMap *__restrict__ xmp, const CUtensorMap *__restrict__ ymp, const __grid_constant__ PA a)
{
    using C = Cfg<T, N4>;
    constexpr int PP = C::PP;
    if (a.done && *a.done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    T *Xst = reinterpret_cast<T *>(smem_raw + 128);
    T *U2 = Xst + NS * C::STG;   // [T2][CW][N4P] (single buffer, AB-internal)
    T *RA = U2 + C::U2E;         // [2][TE]: [T2][T3][FP]
    T *U3 = RA + 2 * C::TE;      // [2][TE]
    T *OUT = U3 + 2 * C::TE;     // [OUTE] (single buffer: its TMA store is waited for one step later)
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) band::mbar_init(bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int dbg = TCA_BAND_DBG ? a.dbg : 0;   // phase switches (measurement only): 1 AB, 2 C compute off

    const Sched sc0{a.s_tile[blockIdx.x].x, a.s_tile[blockIdx.x].y, a.s_o0[blockIdx.x], a.s_cnt[blockIdx.x], a.n1,
                    a.tiles3, a.o_next};
    int gtot = 0;   // pipeline steps of this CTA
    {
        Sched t = sc0;
        int a2, a3, s0, s1;
        while (t.next(a2, a3, s0, s1)) gtot += s1 - s0 + 6;
    }
    const int F = a.n3 * N4;   // elements per mode-2 row of a slab
    double pq = 0.0;

    if (warp < NAB / 32) {
        // =========================== AB: mode 2 (+ lambda R2), mode 3 (+ lambda R3)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
        Sched sc = sc0;
        int a2, a3, o0, o1, g = 0;
        unsigned gc = 0;   // live slabs consumed (stage = gc % NS)
        // phase B item: column (r, i4) along i3, outputs o in [8 h, 8 h + 8)
        const int bi4 = tid & 15, br = (tid >> 4) & 7, bh = tid >> 7;
        B2_PROF_INIT
        while (sc.next(a2, a3, o0, o1)) {
            const int b2 = __shfl_sync(0xffffffffu, a.off2 + a2, 0);               // mode-2 rows of the tile
            const int b3 = __shfl_sync(0xffffffffu, a.off3 + a3 + 8 * bh, 0);      // mode-3 rows of this half
            const int delta = stage_of(a3, N4).y;
            const int jb = max(o0 - 3, -a.xoff), je = min(o1 + 3, a.nin - a.xoff);
            for (int j = o0 - 3; j < o1 + 3; ++j, ++g) {
                const int b = g & 1;
                const bool live = j >= jb && j < je;
                B2_PROF(6);
                if (g >= 2) nb_sync(BAR_EMPTY + b, NAB + NC);   // C is done with RA/RB[b], U3[b] (step g-2)
                B2_PROF(0);
                nb_sync(BAR_AB, NAB);                           // phase B of step g-1 is done with U2
                B2_PROF(1);
                if (live) {
                    if (!(dbg & 4)) band::mbar_wait(bar + gc % NS, (gc / NS) & 1);
                    B2_PROF(2);
                    const T *X = Xst + (gc % NS) * C::STG + delta;
                    T *ra = RA + b * C::TE;
                    if (!(dbg & 1)) {
                        // ---- phase A: column owners c over the staged flat columns (i3', i4)
#pragma unroll 1
                        for (int c = tid; c < C::W; c += NAB) {
                            T v[PR];
#pragma unroll
                            for (int s = 0; s < PR; ++s) v[s] = X[s * PP + c];
                            const int c3 = c / N4, i4 = c - c3 * N4;
                            T u[T2];
#pragma unroll
                            for (int q = 0; q < T2; ++q) u[q] = T(0);
                            // symmetric band: tap G[r, r+k] serves output r (input r+k) and r+k (input r)
#pragma unroll
                            for (int q = -3; q < T2; ++q)
#pragma unroll
                                for (int k = (q < 0 ? -q : 0); k <= 3; ++k) {
                                    const T t = tapG<2>(a, 0, b2 + q, k);
                                    if (q >= 0) u[q] = fma(t, v[q + 3 + k], u[q]);
                                    if (k > 0 && q + k < T2) u[q + k] = fma(t, v[q + 3], u[q + k]);
                                }
#pragma unroll
                            for (int q = 0; q < T2; ++q) U2[q * C::W + c] = u[q];
                            if (c3 >= 3 && c3 < 3 + T3) {   // lambda R2 on the interior columns
#pragma unroll
                                for (int q = 0; q < T2; ++q) u[q] = T(0);
#pragma unroll
                                for (int q = -2; q < T2; ++q)
#pragma unroll
                                    for (int k = (q < 0 ? -q : 0); k <= 2; ++k) {
                                        const T t = tapR<2>(a, 0, b2 + q, k);
                                        if (q >= 0) u[q] = fma(t, v[q + 3 + k], u[q]);
                                        if (k > 0 && q + k < T2) u[q + k] = fma(t, v[q + 3], u[q + k]);
                                    }
#pragma unroll
                                for (int q = 0; q < T2; ++q) ra[(q * T3 + c3 - 3) * FP + i4] = u[q];
                            }
                        }
                    }
                    B2_PROF(3);
                    nb_sync(BAR_AB, NAB);   // U2 and RA complete
                    B2_PROF(4);
                    if (!(dbg & 1) && bi4 < N4) {
                        // ---- phase B: column (br, bi4) along i3, outputs o = 8 bh .. 8 bh + 7
                        const T *u2 = U2 + br * C::W + 8 * bh * N4 + bi4;            // U2 col 8bh + m
                        const T *xp = X + (br + 3) * PP + (8 * bh + 1) * N4 + bi4;   // i3 = a3 + 8bh - 2 + m
                        T *u3b = U3 + b * C::TE;
                        T w[T2 + 6], pz[T2 + 4], u[T2], rr[T2];
#pragma unroll
                        for (int m = 0; m < T2 + 6; ++m) w[m] = u2[m * N4];
#pragma unroll
                        for (int q = 0; q < T2; ++q) u[q] = T(0);
#pragma unroll
                        for (int q = -3; q < T2; ++q)
#pragma unroll
                            for (int k = (q < 0 ? -q : 0); k <= 3; ++k) {
                                const T t = tapG<3>(a, 0, b3 + q, k);
                                if (q >= 0) u[q] = fma(t, w[q + 3 + k], u[q]);
                                if (k > 0 && q + k < T2) u[q + k] = fma(t, w[q + 3], u[q + k]);
                            }
#pragma unroll
                        for (int q = 0; q < T2; ++q) u3b[(br * T3 + 8 * bh + q) * FP + bi4] = u[q];
                        // lambda R3 (+ R2 from phase A) after G3: fewer live registers
#pragma unroll
                        for (int m = 0; m < T2 + 4; ++m) pz[m] = xp[m * N4];
#pragma unroll
                        for (int q = 0; q < T2; ++q) rr[q] = ra[(br * T3 + 8 * bh + q) * FP + bi4];
#pragma unroll
                        for (int q = -2; q < T2; ++q)
#pragma unroll
                            for (int k = (q < 0 ? -q : 0); k <= 2; ++k) {
                                const T t = tapR<3>(a, 0, b3 + q, k);
                                if (q >= 0) rr[q] = fma(t, pz[q + 2 + k], rr[q]);
                                if (k > 0 && q + k < T2) rr[q + k] = fma(t, pz[q + 2], rr[q + k]);
                            }
#pragma unroll
                        for (int q = 0; q < T2; ++q) ra[(br * T3 + 8 * bh + q) * FP + bi4] = rr[q];   // RB in place
                    }
                    ++gc;
                    B2_PROF(5);
                }
                nb_arrive(BAR_FULL + b, NAB + NC);
            }
        }
        B2_PROF_DONE(0)
    } else {
        // =========================== C: mode 4 + mode-1 ring per half fibre, output to HBM
        asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
        const int tc = tid - NAB;
        const int hh = __shfl_sync(0xffffffffu, tc >> 7, 0);   // elements [8 hh, 8 hh + 8) (warp-uniform)
        if (hh == 0) c_loop<T, N4, 0>(xmp, ymp, a, sc0, gtot, bar, Xst, RA, U3, OUT, tc & 127, tc == 0, dbg, pq);
        else c_loop<T, N4, 1>(xmp, ymp, a, sc0, gtot, bar, Xst, RA, U3, OUT, tc & 127, false, dbg, pq);
        if (tc == 0) band::bulk_wait<0>();
    }
    if (a.pq_part) {   // fixed-order CTA reduction of the <x, y> partials (deterministic)
        __syncthreads();
        double *red = reinterpret_cast<double *>(smem_raw + 128);   // stage memory is idle now
#pragma unroll
        for (int k = 16; k > 0; k >>= 1) pq += __shfl_xor_sync(0xffffffffu, pq, k);
        if (lane == 0) red[warp] = pq;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NTHR / 32; ++w) t += red[w];
            a.pq_part[blockIdx.x] = t;
        }
    }
}

// ---------------------------------------------------------------- host side
template <typename T, int N4, typename PA>
tca_status launch_n4(const tca_operator *op, const PA &prm, cudaStream_t s, const CUtensorMap *xm,
                     const CUtensorMap *ym)
{
    using C = Cfg<T, N4>;
    TCA_TRY(set_max_dynamic_smem((const void *)band3_kernel<T, N4, PA>, C::smem_bytes));
    count_launch();
    band3_kernel<T, N4, PA><<<(unsigned)op->band_grid, NTHR, C::smem_bytes, s>>>(xm, ym, prm);
    TCA_CUDA_TRY(cudaGetLastError());
#ifdef TCA_BAND2_PROF
    {   // per-phase cycles of block 0: AB (per warp), C half 0, C half 1 (per warp)
        unsigned long long h[64];
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(h, g_b2prof, sizeof(h));
        const char *nm[3] = {"AB", "C0", "C1"};
        const int base[3] = {0, 32, 40}, nw[3] = {NAB / 32, NC / 64, NC / 64};
        for (int gr = 0; gr < 3; ++gr) {
            fprintf(stderr, "band3 prof %s:", nm[gr]);
            for (int k = 0; k < 8; ++k) fprintf(stderr, " %llu", h[base[gr] + k] / nw[gr]);
            fprintf(stderr, "\n");
        }
        const unsigned long long z[64] = {};
        cudaMemcpyToSymbol(g_b2prof, z, sizeof(z));
    }
#endif
    return TCA_OK;
}

#define TCA_BAND2_N4_LIST(X) X(15) X(16)

template <typename T>
int pp_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Cfg<T, n>::PP;
        TCA_BAND2_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename PA>
tca_status launch_dispatch(const tca_operator *op, const PA &prm, cudaStream_t s, const CUtensorMap *xm,
                           const CUtensorMap *ym)
{
    using T = typename PA::value_type;
    if constexpr (!std::is_same<T, double>::value) {
        return fail(TCA_ERR_INVALID_ARG, "band apply v3: fp64 only");
    } else {
        switch ((int)op->n[3]) {
#define TCA_CASE(n) \
    case n: return launch_n4<T, n, PA>(op, prm, s, xm, ym);
            TCA_BAND2_N4_LIST(TCA_CASE)
#undef TCA_CASE
        }
        return fail(TCA_ERR_INVALID_ARG, "band apply v3: unsupported n4");
    }
}

}  // namespace band2
}  // namespace tca
