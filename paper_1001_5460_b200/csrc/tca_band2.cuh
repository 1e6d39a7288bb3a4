// tca_band2.cuh -- warp-specialised fused banded apply (v2), n4 <= 16.
//
//   q = (G_1 (x) G_2 (x) G_3 (x) G_4) p + sum_d (mode-d lambda R_d) p
//
// Same operator and summation structure as tca_band_impl.cuh (Eq. 4,
// PAPER.md:68-73 applied as successive one-dimensional transformations in the
// order Eq. 5 allows: modes 2 -> 3 -> 4 in shared memory,
// mode 1 streamed through a register ring; Eq. 9's Kronecker-sum regulariser,
// PAPER.md:176-182), re-partitioned for instruction issue:
//
//   * One persistent 384-thread CTA per SM owns a tile of T2 = 4 mode-2 rows x
//     T3 = 16 mode-3 columns x all n4 and streams mode 1 slab by slab.  The
//     input slab (halo 3 in i2 and i3) arrives by ONE TMA box per slab.
//   * The warps are specialised and pipelined through double-buffered shared
//     tiles with named barriers (no CTA-wide barrier per slab):
//       A (2 warps)  mode 2: U2 = G2 p on the halo-extended columns, RA =
//                    lambda R2 p (off-diagonal taps), and a padded copy XP of
//                    the centre rows of p; each warp owns two fixed mode-2
//                    rows, so its 22 taps stay in registers for the whole tile;
//       B (2 warps)  mode 3: U3 = G3 U2, RB = RA + lambda R3 p with the merged
//                    centre lambda (R2[i2,i2] + R3[i3,i3]); each thread owns
//                    two fixed mode-3 rows (taps in registers);
//       C (8 warps)  mode 4 (compile-time taps, constant-bank operands) and the
//                    mode-1 shift ring (uniform taps) of tca_band_impl.cuh,
//                    CG's <p, q> epilogue, emission of output slab j-3 through
//                    a TMA tensor store.
//     A runs up to two slabs ahead of C.  The work split per slab (DFMA): A
//     ~14 k, B ~12 k, C ~26 k on 2 / 2 / 8 warps, one A or B warp and two C
//     warps per SM sub-partition.
//   * Intermediate tiles use a padded fibre layout ([.. ][i3][FP], i4
//     contiguous, FP = 18 doubles / 20 floats) so that every B and C access is
//     a 16-byte vector access with the minimum number of shared-memory
//     wavefronts (fibre pitch coprime with the 8 16-byte bank groups).
#pragma once

#include "tca_band_impl.cuh"

#include <cstdio>

namespace tca {
namespace band2 {

using band::Params;
using band::ParamsBase;
using band::ParamsG;
using band::ParamsH;
using band::tapG;
using band::tapR;

constexpr int T2 = 4;          // mode-2 rows per tile
constexpr int T3 = 16;         // mode-3 columns per tile
constexpr int PR = T2 + 6;     // staged rows (halo 3 + 3)
constexpr int CW = T3 + 6;     // U2 columns (halo 3 + 3)
constexpr int XW = T3 + 4;     // XP columns (halo 2 + 2)
constexpr int N4P = 16;        // padded mode-4 extent
constexpr int NA = 128, NB = 128, NC = 256;
constexpr int NTHR = NA + NB + NC;
#ifndef TCA_B2_UNIT
#define TCA_B2_UNIT 8
#endif
constexpr int UNIT = TCA_B2_UNIT;   // TMA chunk of the staged slab box (elements)
constexpr int MAXG = band::MAXG;

// named barriers (0 is __syncthreads)
constexpr int BAR_FULL_AB = 1;    // +b: A produced U2/RA/XP[b]        (A arrive, B sync)
constexpr int BAR_FULL_BC = 3;    // +b: B produced U3/RB[b]           (B arrive, C sync)
constexpr int BAR_EMPTY_XP = 5;   // +b: C released XP[b] (and U2[b])  (C arrive, A sync)
constexpr int BAR_EMPTY_U3 = 7;   // +b: C released U3/RB[b]           (C arrive, B sync)
constexpr int BAR_A = 9;          // A warps: staged slab fully read
constexpr int BAR_C = 10;         // C warps: output staging written

template <typename T, int N4>
struct Cfg {
    static_assert(N4 >= 9 && N4 <= 16, "v2 takes 9 <= n4 <= 16");
    static constexpr int W = CW * N4;                                   // staged flat columns
    static constexpr int PP = (W + UNIT - 1 + UNIT - 1) / UNIT * UNIT;  // staged row pitch (elements)
    static constexpr int FP = sizeof(T) == 8 ? 18 : 20;                 // padded fibre pitch
    static constexpr int NS = 4;                                        // input stages
    static constexpr size_t al(size_t e) { return (e * sizeof(T) + 127) / 128 * 128 / sizeof(T); }
    static constexpr size_t STG = al((size_t)PR * PP);
    static constexpr size_t U2E = al((size_t)T2 * CW * FP);
    static constexpr size_t TE = al((size_t)T2 * T3 * FP);   // RA (= RB, updated in place by B), U3
    static constexpr size_t XPE = al((size_t)T2 * XW * FP);
    static constexpr size_t OUTE = al((size_t)T2 * T3 * N4); // TMA store source: dense [T2][T3 n4]
    static constexpr size_t smem_bytes = 128 + (NS * STG + 2 * (U2E + 2 * TE + XPE + OUTE)) * sizeof(T);
    static_assert(smem_bytes <= 227 * 1024, "shared memory");
    static_assert(PP / UNIT <= 256 && T3 * N4 <= 256, "TMA box");
};

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n)
{
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

template <typename T> struct V2;
template <> struct V2<double> { using V = double2; };
template <> struct V2<float> { using V = float2; };
template <typename T>
__device__ __forceinline__ void st2(T *p, T a, T b)
{
    *reinterpret_cast<typename V2<T>::V *>(p) = typename V2<T>::V{a, b};
}
template <typename T>
__device__ __forceinline__ void ld2(const T *p, T &a, T &b)
{
    const typename V2<T>::V v = *reinterpret_cast<const typename V2<T>::V *>(p);
    a = v.x;
    b = v.y;
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
    if (blockIdx.x == 0 && lane == 0) \
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
    int t2i, t3i, o0, cnt, n1, tiles3;
    __device__ bool next(int &a2, int &a3, int &s0, int &s1)
    {
        if (cnt <= 0) return false;
        s0 = o0;
        s1 = (n1 - o0 < cnt) ? n1 : o0 + cnt;
        cnt -= s1 - s0;
        a2 = t2i * T2;
        a3 = t3i * T3;
        o0 = 0;
        t3i = (t3i + 1 == tiles3) ? 0 : t3i + 1;
        t2i += (t3i == 0) ? 1 : 0;
        return true;
    }
};

// ---------------------------------------------------------------- C: mode 4 of one segment (compile-time taps)
// s = G4 U3, q = RB + lambda R4 p, pc = p over the elements [4 SEG, 4 SEG + 4) of
// this thread's fibre (pad elements >= N4 are zero).
template <typename T, int N4, int SEG, typename PA>
__device__ __forceinline__ void mode4(const PA &a, const T *u3, const T *rb, const T *xp, T (&s)[4], T (&q)[4],
                                      T (&pc)[4])
{
    constexpr int e0 = 4 * SEG;
    constexpr int e1 = (e0 + 4 < N4) ? e0 + 4 : N4;
    constexpr int ulo = ((e0 - 3 > 0) ? e0 - 3 : 0) & ~1;
    constexpr int uhi = (((e1 + 3 < N4) ? e1 + 3 : N4) + 1) & ~1;
    constexpr int plo = ((e0 - 2 > 0) ? e0 - 2 : 0) & ~1;
    constexpr int phi = (((e1 + 2 < N4) ? e1 + 2 : N4) + 1) & ~1;
    T uw[N4P], pw[N4P];
#pragma unroll
    for (int k = ulo; k < uhi; k += 2) ld2(u3 + k, uw[k], uw[k + 1]);
#pragma unroll
    for (int k = plo; k < phi; k += 2) ld2(xp + k, pw[k], pw[k + 1]);
    ld2(rb + e0, q[0], q[1]);
    ld2(rb + e0 + 2, q[2], q[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = T(0);
    // push form: one input value, consecutive DFMAs into the outputs it touches
#pragma unroll
    for (int k = ulo; k < uhi; ++k)
#pragma unroll
        for (int e = e0; e < e1; ++e)
            if (k < N4 && k - e >= -3 && k - e <= 3) s[e - e0] = fma(tapG<4>(a, 0, e, k - e), uw[k], s[e - e0]);
#pragma unroll
    for (int k = plo; k < phi; ++k)
#pragma unroll
        for (int e = e0; e < e1; ++e)
            if (k < N4 && k - e >= -2 && k - e <= 2) q[e - e0] = fma(tapR<4>(a, 0, e, k - e), pw[k], q[e - e0]);
#pragma unroll
    for (int e = 0; e < 4; ++e) pc[e] = (e0 + e < N4) ? pw[e0 + e] : T(0);
#pragma unroll
    for (int e = e1 - e0; e < 4; ++e) { s[e] = T(0); q[e] = T(0); }
}

template <typename T, int N4, int SEG, typename PA>
__device__ __forceinline__ void mode4_dispatch(int seg, const PA &a, const T *u3, const T *rb, const T *xp, T (&s)[4],
                                               T (&q)[4], T (&pc)[4])
{
    if constexpr (SEG < 4) {
        if (seg == SEG) mode4<T, N4, SEG, PA>(a, u3, rb, xp, s, q, pc);
        else mode4_dispatch<T, N4, SEG + 1, PA>(seg, a, u3, rb, xp, s, q, pc);
    }
}

// ---------------------------------------------------------------- kernel
template <typename T, int N4, typename PA>
__global__ void __launch_bounds__(NTHR, 1)
band2_kernel(const CUtensorMap *__restrict__ xmp, const CUtensorMap *__restrict__ ymp, const __grid_constant__ PA a)
{
    using C = Cfg<T, N4>;
    constexpr int NS = C::NS, PP = C::PP, FP = C::FP;
    if (a.done && *a.done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    T *Xst = reinterpret_cast<T *>(smem_raw + 128);
    T *U2 = Xst + NS * C::STG;   // [2][U2E]
    T *RA = U2 + 2 * C::U2E;     // [2][TE]
    T *U3 = RA + 2 * C::TE;      // [2][TE]
    T *RB = RA;                  // B turns RA into RB in place (each thread its own entries)
    T *XP = U3 + 2 * C::TE;      // [2][XPE]
    T *OUT = XP + 2 * C::XPE;    // [2][OUTE]
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) band::mbar_init(bar + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    Sched sc0{a.s_tile[blockIdx.x].x, a.s_tile[blockIdx.x].y, a.s_o0[blockIdx.x], a.s_cnt[blockIdx.x], a.n1, a.tiles3};
    int gtot = 0;   // total pipeline steps of this CTA
    {
        Sched t = sc0;
        int a2, a3, s0, s1;
        while (t.next(a2, a3, s0, s1)) gtot += s1 - s0 + 6;
    }
    const int F = a.n3 * N4;   // elements per mode-2 row of a slab
    const int dbg = TCA_BAND_DBG ? a.dbg : 0;   // phase switches (measurement only): 1 A, 2 B, 4 C compute off
    double pq = 0.0;

    if (warp < NA / 32) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
        // =========================== A: mode 2 (+ lambda R2 off-diagonal, XP copy)
        const int R0 = 2 * (warp & 1);   // output rows R0, R0 + 1 of the tile (warp-uniform)
        const int half = warp >> 1;      // interior columns [3 + 8 half, 11 + 8 half), halo side half
        const int m = lane & 7;    // i4 pair (2m, 2m + 1)
        const bool e0ok = 2 * m < N4, e1ok = 2 * m + 1 < N4;
        B2_PROF_INIT
        unsigned gi = 0, gc = 0;   // live slabs issued / consumed (stage = k % NS)
        Sched sc = sc0;
        int a2, a3, o0, o1, g = 0;
        while (sc.next(a2, a3, o0, o1)) {
            T gt[2][7], rt[2][4];   // taps of rows a2+R0, a2+R0+1: G2[i2, i2+k], lambda R2[i2, i2+k] (k != 0)
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
                for (int k = -3; k <= 3; ++k) gt[rr][k + 3] = tapG<2>(a, a.off2, a2 + R0 + rr, k);
                rt[rr][0] = tapR<2>(a, a.off2, a2 + R0 + rr, -2);
                rt[rr][1] = tapR<2>(a, a.off2, a2 + R0 + rr, -1);
                rt[rr][2] = tapR<2>(a, a.off2, a2 + R0 + rr, 1);
                rt[rr][3] = tapR<2>(a, a.off2, a2 + R0 + rr, 2);
            }
            const int ca = (a3 - 3) * N4;                // flat column of staged column 0
            const int delta = ((ca % UNIT) + UNIT) % UNIT;
            const int cchunk = (ca - delta) / UNIT;
            const int jb = max(o0 - 3, -a.xoff), je = min(o1 + 3, a.nin - a.xoff);
            int nxt = jb;
            auto issue = [&]() {   // leader: stage input slab nxt
                while (gi < gc + NS && nxt < je) {
                    const unsigned st = gi % NS;
                    band::mbar_arrive_expect_tx(bar + st, (unsigned)(PR * PP * sizeof(T)));
                    band::tma_load_4d(Xst + st * C::STG, xmp, bar + st, 0, cchunk, a2 - 3, nxt + a.xoff);
                    ++gi;
                    ++nxt;
                }
            };
            if (tid == 0 && !(dbg & 32)) issue();
            for (int j = o0 - 3; j < o1 + 3; ++j, ++g) {
                const int b = g & 1;
                const bool live = j >= jb && j < je;
                B2_PROF(3);
                if (g >= 2) nb_sync(BAR_EMPTY_XP + b, NA + NC);
                B2_PROF(0);
                if (live && !(dbg & 32)) band::mbar_wait(bar + gc % NS, (gc / NS) & 1);
                B2_PROF(1);
                if (live && !(dbg & 1)) {
                    const T *X = Xst + (gc % NS) * C::STG + delta + R0 * PP;
                    T *u2 = U2 + b * C::U2E + R0 * CW * FP;
                    T *ra = RA + b * C::TE + R0 * T3 * FP;
                    T *xp = XP + b * C::XPE + R0 * XW * FP;
                    // items (i3', m): 2 interior rounds of 4 columns x 8 pairs (G and R),
                    // then 3 halo columns ({0,1,2} or {19,20,21}; G only)
#pragma unroll 1
                    for (int it = 0; it < 3; ++it) {
                        const bool inner = it < 2;
                        int c3;
                        if (inner) {
                            c3 = 3 + 8 * half + it * 4 + (lane >> 3);
                        } else {
                            const int h = lane >> 3;   // 0..3 (3 used)
                            if (h >= 3) continue;
                            c3 = half ? 19 + h : h;
                        }
                        const T *x = X + c3 * N4 + 2 * m;
                        T v0[8], v1[8];
#pragma unroll
                        for (int s = 0; s < 8; ++s) {
                            v0[s] = e0ok ? x[s * PP] : T(0);
                            v1[s] = e1ok ? x[s * PP + 1] : T(0);
                        }
                        T g00 = T(0), g01 = T(0), g10 = T(0), g11 = T(0);
#pragma unroll
                        for (int s = 0; s < 8; ++s) {
                            if (s <= 6) {
                                g00 = fma(gt[0][s], v0[s], g00);
                                g01 = fma(gt[0][s], v1[s], g01);
                            }
                            if (s >= 1) {
                                g10 = fma(gt[1][s - 1], v0[s], g10);
                                g11 = fma(gt[1][s - 1], v1[s], g11);
                            }
                        }
                        st2(u2 + c3 * FP + 2 * m, g00, g01);
                        st2(u2 + (CW + c3) * FP + 2 * m, g10, g11);
                        if (inner) {
                            // row rr: R2 taps k = -2, -1, 1, 2 at input rows s = 3 + rr + k
                            T r00 = T(0), r01 = T(0), r10 = T(0), r11 = T(0);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int k = i < 2 ? i - 2 : i - 1;
                                r00 = fma(rt[0][i], v0[3 + k], r00);
                                r01 = fma(rt[0][i], v1[3 + k], r01);
                                r10 = fma(rt[1][i], v0[4 + k], r10);
                                r11 = fma(rt[1][i], v1[4 + k], r11);
                            }
                            st2(ra + (c3 - 3) * FP + 2 * m, r00, r01);
                            st2(ra + (T3 + c3 - 3) * FP + 2 * m, r10, r11);
                        }
                        if (c3 >= 1 && c3 <= XW) {   // XP: centre rows of p, columns i3' in [1, 21)
                            st2(xp + (c3 - 1) * FP + 2 * m, v0[3], v1[3]);
                            st2(xp + (XW + c3 - 1) * FP + 2 * m, v0[4], v1[4]);
                        }
                    }
                }
                B2_PROF(2);
                nb_arrive(BAR_FULL_AB + b, NA + NB);
                if (live) {
                    ++gc;
                    nb_sync(BAR_A, NA);   // every A thread is done with the stage
                    if (tid == 0 && !(dbg & 32)) issue();
                }
            }
        }
        B2_PROF_DONE(0)
    } else if (warp < (NA + NB) / 32) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
        // =========================== B: mode 3 (+ lambda R3, merged centre)
        const int tb = tid - NA;
        const int m = tb & 7;            // i4 pair
        const int op = (tb >> 3) & 7;    // output columns o = 2 op, 2 op + 1
        const int rh = tb >> 6;          // rows 2 rh, 2 rh + 1
        B2_PROF_INIT
        Sched sc = sc0;
        int a2, a3, o0, o1, g = 0;
        while (sc.next(a2, a3, o0, o1)) {
            T gt[2][7], rt[2][4], cen[2][2];
#pragma unroll
            for (int ol = 0; ol < 2; ++ol) {
                const int i3 = a3 + 2 * op + ol;
#pragma unroll
                for (int k = -3; k <= 3; ++k) gt[ol][k + 3] = tapG<3>(a, a.off3, i3, k);
                rt[ol][0] = tapR<3>(a, a.off3, i3, -2);
                rt[ol][1] = tapR<3>(a, a.off3, i3, -1);
                rt[ol][2] = tapR<3>(a, a.off3, i3, 1);
                rt[ol][3] = tapR<3>(a, a.off3, i3, 2);
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) cen[rr][ol] = tapR<2>(a, a.off2, a2 + 2 * rh + rr, 0) + tapR<3>(a, a.off3, i3, 0);
            }
            const int jb = max(o0 - 3, -a.xoff), je = min(o1 + 3, a.nin - a.xoff);
            for (int j = o0 - 3; j < o1 + 3; ++j, ++g) {
                const int b = g & 1;
                const bool live = j >= jb && j < je;
                B2_PROF(3);
                nb_sync(BAR_FULL_AB + b, NA + NB);
                B2_PROF(0);
                if (g >= 2) nb_sync(BAR_EMPTY_U3 + b, NB + NC);
                B2_PROF(1);
                if (live && !(dbg & 2)) {
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {   // unrolled: cen[rr] stays in registers
                        const int r = 2 * rh + rr;
                        const T *u2 = U2 + b * C::U2E + (r * CW + 2 * op) * FP + 2 * m;
                        const T *xp = XP + b * C::XPE + (r * XW + 2 * op) * FP + 2 * m;
                        const T *ra = RA + b * C::TE + (r * T3 + 2 * op) * FP + 2 * m;
                        T u00 = T(0), u01 = T(0), u10 = T(0), u11 = T(0);   // [o][i4]
                        T w00, w01, w10, w11;
                        ld2(ra, w00, w01);
                        ld2(ra + FP, w10, w11);
#pragma unroll
                        for (int p = 0; p < 8; ++p) {   // U2 column i3' = 2 op + p
                            T x0, x1;
                            ld2(u2 + p * FP, x0, x1);
                            if (p <= 6) {
                                u00 = fma(gt[0][p], x0, u00);
                                u01 = fma(gt[0][p], x1, u01);
                            }
                            if (p >= 1) {
                                u10 = fma(gt[1][p - 1], x0, u10);
                                u11 = fma(gt[1][p - 1], x1, u11);
                            }
                        }
#pragma unroll
                        for (int p = 0; p < 6; ++p) {   // XP column i3'' = 2 op + p (= i3 + 2)
                            T x0, x1;
                            ld2(xp + p * FP, x0, x1);
                            // output ol: k = p - ol - 2
                            if (p <= 4) {
                                const int k = p - 2;
                                const T t = k == 0 ? cen[rr][0] : rt[0][k < 0 ? k + 2 : k + 1];
                                w00 = fma(t, x0, w00);
                                w01 = fma(t, x1, w01);
                            }
                            if (p >= 1) {
                                const int k = p - 3;
                                const T t = k == 0 ? cen[rr][1] : rt[1][k < 0 ? k + 2 : k + 1];
                                w10 = fma(t, x0, w10);
                                w11 = fma(t, x1, w11);
                            }
                        }
                        T *u3 = U3 + b * C::TE + (r * T3 + 2 * op) * FP + 2 * m;
                        T *rb = RB + b * C::TE + (r * T3 + 2 * op) * FP + 2 * m;
                        st2(u3, u00, u01);
                        st2(u3 + FP, u10, u11);
                        st2(rb, w00, w01);
                        st2(rb + FP, w10, w11);
                    }
                }
                B2_PROF(2);
                nb_arrive(BAR_FULL_BC + b, NB + NC);
            }
        }
        B2_PROF_DONE(16)
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 160;\n" ::: "memory");
        // =========================== C: mode 4, mode-1 ring, emission
        const int tc = tid - NA - NB;
        const int wc = tc >> 5;
        const int seg = __shfl_sync(0xffffffffu, wc >> 1, 0);   // warp-uniform segment of i4
        const int f = (wc & 1) * 32 + lane;                      // fibre (r, o) of the tile
        const int r = f >> 4, o = f & 15;
        T acc[6][4];
        unsigned nemit = 0;
        B2_PROF_INIT
        Sched sc = sc0;
        int a2, a3, o0, o1, g = 0;
        while (sc.next(a2, a3, o0, o1)) {
#pragma unroll
            for (int k = 0; k < 6; ++k)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[k][e] = T(0);
            const int jb = max(o0 - 3, -a.xoff), je = min(o1 + 3, a.nin - a.xoff);
            // mode-1 taps of input slab j: G1[j+k, j], lambda R1[j+k, j] (uniform), one
            // step ahead so that their constant-cache latency hides behind a step
            T g1n[7], r1n[5];
            auto taps1 = [&](int jj) {
                const int b1 = __shfl_sync(0xffffffffu, a.off1 + jj, 0);
#pragma unroll
                for (int k = -3; k <= 3; ++k) g1n[k + 3] = tapG<1>(a, 0, b1 + k, -k);
#pragma unroll
                for (int k = -2; k <= 2; ++k) r1n[k + 2] = tapR<1>(a, 0, b1 + k, -k);
            };
            taps1(o0 - 3);
            for (int j = o0 - 3; j < o1 + 3; ++j, ++g) {
                const int b = g & 1;
                const bool live = j >= jb && j < je;
                const bool emit = j - 3 >= o0 && j - 3 < o1;
                T g1[7], r1[5];
#pragma unroll
                for (int k = 0; k < 7; ++k) g1[k] = g1n[k];
#pragma unroll
                for (int k = 0; k < 5; ++k) r1[k] = r1n[k];
                taps1(j + 1);
                if (emit && tc == 0 && !(dbg & 128)) band::bulk_wait_read<1>();   // OUT[nemit & 1] is free again
                B2_PROF(0);
                nb_sync(BAR_FULL_BC + b, NB + NC);
                B2_PROF(1);
                T s[4], q[4], pc[4];
                if (live && !(dbg & 4)) {
                    const T *u3 = U3 + b * C::TE + f * FP;
                    const T *rb = RB + b * C::TE + f * FP;
                    const T *xp = XP + b * C::XPE + (r * XW + o + 2) * FP;
                    mode4_dispatch<T, N4, 0, PA>(seg, a, u3, rb, xp, s, q, pc);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) { s[e] = T(0); q[e] = T(0); pc[e] = T(0); }
                }
                B2_PROF(2);
                if (g + 2 < gtot) {
                    nb_arrive(BAR_EMPTY_XP + b, NA + NC);
                    nb_arrive(BAR_EMPTY_U3 + b, NB + NC);
                }
                T ov[4];
                const bool dot = a.pq_part != nullptr && j >= o0 && j < o1;
                if (!(dbg & 8)) band::ring_step<T, 4>(acc, s, q, pc, g1, r1, ov, dot, pq);
                else for (int e = 0; e < 4; ++e) ov[e] = s[e] + g1[e];
                B2_PROF(3);
                if (emit && !(dbg & 16)) {
                    T *out = OUT + (nemit & 1) * C::OUTE + r * (T3 * N4) + o * N4 + 4 * seg;
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (4 * seg + e < N4) out[e] = ov[e];
                    B2_PROF(4);
                    band::fence_proxy_async();
                    B2_PROF(5);
                    nb_sync(BAR_C, NC);
                    if (tc == 0) {
                        band::tma_store_3d(ymp, OUT + (nemit & 1) * C::OUTE, a3 * N4, a2, j - 3);
                        band::bulk_commit();
                    }
                    ++nemit;
                    B2_PROF(6);
                }
            }
        }
        if (tc == 0) band::bulk_wait<0>();
        B2_PROF_DONE(32)
    }
    (void)F;
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
    TCA_TRY(set_max_dynamic_smem((const void *)band2_kernel<T, N4, PA>, C::smem_bytes));
    count_launch();
    band2_kernel<T, N4, PA><<<(unsigned)op->band_grid, NTHR, C::smem_bytes, s>>>(xm, ym, prm);
    TCA_CUDA_TRY(cudaGetLastError());
#ifdef TCA_BAND2_PROF
    {   // per-phase cycles of block 0 (sums over the warps of each group, then per warp)
        unsigned long long h[64];
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(h, g_b2prof, sizeof(h));
        const char *nm[3] = {"A", "B", "C"};
        const int nw[3] = {NA / 32, NB / 32, NC / 32};
        for (int gr = 0; gr < 3; ++gr) {
            fprintf(stderr, "band2 prof %s:", nm[gr]);
            for (int k = 0; k < 8; ++k) fprintf(stderr, " %llu", h[16 * gr + k] / nw[gr]);
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
    switch ((int)op->n[3]) {
#define TCA_CASE(n) \
    case n: return launch_n4<T, n, PA>(op, prm, s, xm, ym);
        TCA_BAND2_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return fail(TCA_ERR_INVALID_ARG, "band apply v2: unsupported n4");
}

}  // namespace band2
}  // namespace tca
