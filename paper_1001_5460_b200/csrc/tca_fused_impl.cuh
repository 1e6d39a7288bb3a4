// tca_fused_impl.cuh -- fused banded operator apply, one HBM pass.
// Instantiated per (dtype, staging path) in tca_fused_*.cu.
//
//   q = (G_1 (x) G_2 (x) G_3 (x) G_4) p + sum_d (mode-d lambda R_d) p
//
// Eq. 4 applies the separable operator as successive
// one-dimensional transformations; Eq. 5 lets us pick their
// order; Eq. 9 is the Kronecker-sum regulariser.  Every
// G_d has half-bandwidth <= 3 and every R_d <= 2 (checked at create).
//
// Design (B200, fp64/fp32):
//   * A CTA owns a tile of T2=8 mode-2 rows x T3 mode-3 columns x all n4 and
//     STREAMS mode 1: slab j (all points with i1 = j) passes through shared
//     memory once; mode 1 is applied as a 7-slot register ring (each thread
//     keeps 7 partial outputs for each of its 8 points), so no slab is ever
//     re-read for mode 1.
//   * In-slice modes are applied in the order 2 -> 3 -> 4 (mode 2 first
//     shrinks the halo), each phase with its own register-blocked mapping and
//     TWO independent vectors per thread, so each tap row loaded from shared
//     memory feeds two outputs:
//       A: columns along i2 of the halo-extended tile (14 in, 8 out): G2
//       B: 4-output segments along i3 (10 in): G3, and R3 on p
//       C: 4-output segments along i4 (10 in): G4, and R4 on p
//       D: ring owner: R2 on its p column, ring update (G1, R1) and emission
//          of the finished slab j-3.
//     Three CTA barriers per slab (A|B, B|C, C|D); U2 is double-buffered by
//     slab parity and the next slab's staging is issued after A|B, which
//     makes an end-of-slab barrier unnecessary.
//   * n4 is a template parameter, so all shared-memory indexing is static;
//     phases A-C exist once in the code, only the ring update is specialised
//     for its 7 slot rotations.
//   * Slabs are staged three deep.  TMA path: warp 0 issues
//     cp.async.bulk.tensor boxes (one per row and column block) completing on
//     a per-stage mbarrier; out-of-domain boxes are zero-filled by the TMA
//     unit (the truncated band of reading Z15).  cp.async path (shapes whose
//     strides TMA cannot describe): per-element copies.
//   * Persistent grid: one CTA per SM, each owns a contiguous range of
//     (tile, i1) units; a range that crosses a tile boundary restarts the
//     ring (6 ramp slabs).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "tca_fused.cuh"

namespace tca {
namespace fused {

constexpr int T2 = 8;          // mode-2 rows per tile (register pencil)
constexpr int PR = T2 + 6;     // halo-extended rows in a slab stage
constexpr int NSTAGE = 3;      // slab stages
constexpr int TP = 16;         // tap row: G taps at 0..6, lambda*R taps at 8..12 (zero padded)
constexpr int TR = 8;          // offset of the R taps in a tap row

template <typename T, int N4>
struct Shape {
    static constexpr int T3 = (N4 >= 16) ? (N4 > 16 ? 8 : 16)
                              : ((8 * (32 / N4)) > 64 ? 64 : 8 * (32 / N4));
    static constexpr int NTHR = T3 * N4;
    static constexpr int T3N4 = T3 * N4;
    static constexpr int W = (T3 + 6) * N4;           // halo-extended flat columns
    static constexpr int VEC = 16 / (int)sizeof(T);   // TMA inner coordinate granularity (16 B)
    static constexpr int UNIT = 128 / (int)sizeof(T); // TMA smem destination granularity (128 B)
    // NB boxes of BOXW columns cover W columns starting at a VEC-aligned
    // coordinate (up to VEC-1 extra columns); each box lands 128-byte aligned.
    static constexpr int NEED = W + VEC - 1;
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
    static constexpr int PP = NB * BOXW;              // slab stage row pitch
    static constexpr int NS3 = T3 / 4;                // 4-output segments along i3
    static constexpr int NS4 = (N4 + 3) / 4;          // 4-output segments along i4
    static constexpr int NPA = (W + 1) / 2;           // phase A work items (2 columns each)
    static constexpr int NPB = 4 * N4 * NS3;          // phase B work items (2 rows each)
    static constexpr int NPC = 4 * T3 * NS4;          // phase C work items (2 rows each)
    static constexpr size_t smem_elems = (size_t)NSTAGE * PR * PP + 2 * (size_t)T2 * W + 2 * (size_t)T2 * T3N4 +
                                         (size_t)(T2 + T3 + N4) * TP;
    static constexpr size_t smem_bytes = smem_elems * sizeof(T) + 128;  // + mbarriers
    static_assert(NPA <= NTHR && NPB == NTHR, "phase sizes");
    static_assert((PR * PP * sizeof(T)) % 128 == 0 && (BOXW * sizeof(T)) % 128 == 0, "TMA alignment");
};

template <typename T>
struct FusedArgs {
    const T *x;
    T *y;
    int n1, n2, n3;
    int tiles3;
    long long total;       // ntiles * n1 units
    const T *tg[4];        // [n_d][7]  G_d[r, r+k-3]
    const T *tr[4];        // [n_d][5]  lambda R_d[r, r+k-2]
    const int32_t *done;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void *p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async_elem(void *smem, const void *gmem, int bytes, bool valid)
{
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                     "r"(valid ? 8 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                     "r"(valid ? 4 : 0));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

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

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// 8 taps starting at a 16-byte aligned row offset -> registers
template <typename T>
__device__ __forceinline__ void load8(const T *p, T (&t)[8])
{
    if constexpr (sizeof(T) == 8) {
        const double2 *q = reinterpret_cast<const double2 *>(p);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double2 v = q[i];
            t[2 * i] = v.x;
            t[2 * i + 1] = v.y;
        }
    } else {
        const float4 *q = reinterpret_cast<const float4 *>(p);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float4 v = q[i];
            t[4 * i] = v.x;
            t[4 * i + 1] = v.y;
            t[4 * i + 2] = v.z;
            t[4 * i + 3] = v.w;
        }
    }
}

template <typename T>
__device__ __forceinline__ T dot7(const T (&t)[8], const T *v)
{
    T u = t[0] * v[0];
#pragma unroll
    for (int k = 1; k < 7; ++k) u = fma(t[k], v[k], u);
    return u;
}

template <typename T>
__device__ __forceinline__ T dot5(const T (&t)[8], const T *v)
{
    T u = t[0] * v[0];
#pragma unroll
    for (int k = 1; k < 5; ++k) u = fma(t[k], v[k], u);
    return u;
}

// ---------------------------------------------------------------- slab staging
// Offset (elements) between a TMA-staged slab row and the tile's first column.
template <typename T, int N4>
__device__ __forceinline__ int slab_delta(int a3)
{
    constexpr int V = Shape<T, N4>::VEC;
    const int c0 = (a3 - 3) * N4;
    return ((c0 % V) + V) % V;
}

// Stage slab j of x (rows a2-3 .. a2+10, flat (i3,i4) columns of the
// halo-extended tile) into dst[r*PP + c].  TMA: issued by warp 0.
template <typename T, int N4, bool TMA>
__device__ __forceinline__ void load_slab(T *dst, uint64_t *bar, const CUtensorMap *map,
                                          const FusedArgs<T> &a, int j, int a2, int a3)
{
    using S = Shape<T, N4>;
    const int tid = threadIdx.x;
    const int c0 = (a3 - 3) * N4;   // flat column of local column 0
    if constexpr (TMA) {
        // boxes start at the aligned column c0 - delta; consumers read dst + delta
        const int ca = c0 - slab_delta<T, N4>(a3);
        if (tid < 32) {
            if (tid == 0) mbar_arrive_expect_tx(bar, (unsigned)(S::NB * PR * S::BOXW * sizeof(T)));
            __syncwarp();
#pragma unroll 1
            for (int b = tid; b < S::NB * PR; b += 32) {
                const int r = b / S::NB, h = b % S::NB;
                tma_load_3d(dst + r * S::PP + h * S::BOXW, map, bar, ca + h * S::BOXW, a2 - 3 + r, j);
            }
        }
    } else {
        const int n3n4 = a.n3 * N4;
        const bool jv = j >= 0 && j < a.n1;
#pragma unroll 1
        for (int r = 0; r < PR; ++r) {
            const int g2 = a2 - 3 + r;
            const bool rv = jv && g2 >= 0 && g2 < a.n2;
            const T *src = a.x + ((long long)(rv ? j : 0) * a.n2 + (rv ? g2 : 0)) * n3n4;
            for (int c = tid; c < S::PP; c += S::NTHR) {
                const int f = c0 + c;
                const bool v = rv && f >= 0 && f < n3n4;
                cp_async_elem(dst + r * S::PP + c, v ? (const void *)(src + f) : (const void *)a.x,
                              (int)sizeof(T), v);
            }
        }
        cp_async_commit();
    }
}

template <typename T>
struct Smem {
    T *P, *U2[2], *U3, *REG, *tap2, *tap3, *tap4;
    uint64_t *bar;
};

// Ring update for rotation U (compile-time slots: output slab j+o lives in
// slot (U+o) mod 7), then emission of the finished slab j-3 (slot (U+4) mod 7).
template <typename T, int U>
__device__ __forceinline__ void ring_emit(T (&acc)[7][T2], const T (&sv)[T2], const T (&pc)[T2],
                                          const T (&rg)[T2], const T (&g1)[7], const T (&r1)[5], T *dst,
                                          int n3n4, int nrow, bool emit)
{
#pragma unroll
    for (int o = -3; o <= 3; ++o) {
#pragma unroll
        for (int i = 0; i < T2; ++i) {
            T v = acc[(U + o + 7) % 7][i];
            v = fma(g1[o + 3], sv[i], v);
            if (o >= -2 && o <= 2) v = fma(r1[o + 2], pc[i], v);
            if (o == 0) v += rg[i];
            acc[(U + o + 7) % 7][i] = v;
        }
    }
    constexpr int ES = (U + 4) % 7;
    if (emit) {
#pragma unroll
        for (int i = 0; i < T2; ++i)
            if (i < nrow) dst[i * n3n4] = acc[ES][i];
    }
#pragma unroll
    for (int i = 0; i < T2; ++i) acc[ES][i] = T(0);
}

template <typename T, int N4, bool TMA>
__global__ void __launch_bounds__(Shape<T, N4>::NTHR, 1)
fused_apply_kernel(const FusedArgs<T> a, const __grid_constant__ CUtensorMap map)
{
    using S = Shape<T, N4>;
    constexpr int W = S::W, T3N4 = S::T3N4, T3 = S::T3, PP = S::PP;
    if (a.done && *a.done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem<T> sm;
    sm.bar = reinterpret_cast<uint64_t *>(smem_raw);
    sm.P = reinterpret_cast<T *>(smem_raw + 128);  // TMA destinations: 128-byte aligned
    sm.U2[0] = sm.P + NSTAGE * PR * PP;
    sm.U2[1] = sm.U2[0] + T2 * W;
    sm.U3 = sm.U2[1] + T2 * W;
    sm.REG = sm.U3 + T2 * T3N4;
    sm.tap2 = sm.REG + T2 * T3N4;
    sm.tap3 = sm.tap2 + T2 * TP;
    sm.tap4 = sm.tap3 + T3 * TP;
    const int tid = threadIdx.x;
    const CUtensorMap *mp = &map;
    if constexpr (TMA) {
        if (tid == 0) {
            for (int s = 0; s < NSTAGE; ++s) mbar_init(sm.bar + s, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
    }
    // mode-4 taps (same for every tile)
    for (int e = tid; e < N4 * TP; e += S::NTHR) {
        const int r = e / TP, k = e % TP;
        sm.tap4[e] = k < 7 ? a.tg[3][r * 7 + k] : (k >= TR && k < TR + 5 ? a.tr[3][r * 5 + k - TR] : T(0));
    }
    __syncthreads();

    long long u0 = a.total * blockIdx.x / gridDim.x;
    const long long u1 = a.total * (blockIdx.x + 1) / gridDim.x;
    unsigned g = 0;  // CTA-lifetime slab counter: stage g % 3, mbarrier parity (g / 3) & 1
    T acc[7][T2];
    const int n3n4 = a.n3 * N4;
    while (u0 < u1) {
        const int tile = (int)(u0 / a.n1);
        const int o0 = (int)(u0 % a.n1);
        const long long rem = u1 - u0;
        const int o1 = (int)((long long)a.n1 < o0 + rem ? (long long)a.n1 : o0 + rem);
        u0 += o1 - o0;
        const int a2 = (tile / a.tiles3) * T2;
        const int a3 = (tile % a.tiles3) * T3;
        const int delta = TMA ? slab_delta<T, N4>(a3) : 0;
        // tile taps for modes 2 and 3 (zero rows outside the domain)
        for (int e = tid; e < T2 * TP; e += S::NTHR) {
            const int r = a2 + e / TP, k = e % TP;
            sm.tap2[e] = r >= a.n2 ? T(0)
                                   : (k < 7 ? a.tg[1][r * 7 + k] : (k >= TR && k < TR + 5 ? a.tr[1][r * 5 + k - TR] : T(0)));
        }
        for (int e = tid; e < T3 * TP; e += S::NTHR) {
            const int r = a3 + e / TP, k = e % TP;
            sm.tap3[e] = r >= a.n3 ? T(0)
                                   : (k < 7 ? a.tg[2][r * 7 + k] : (k >= TR && k < TR + 5 ? a.tr[2][r * 5 + k - TR] : T(0)));
        }
#pragma unroll
        for (int s = 0; s < 7; ++s)
#pragma unroll
            for (int i = 0; i < T2; ++i) acc[s][i] = T(0);
        const int j0 = o0 - 3, j1 = o1 + 3;
        load_slab<T, N4, TMA>(sm.P + (g % NSTAGE) * PR * PP, sm.bar + g % NSTAGE, mp, a, j0, a2, a3);
        load_slab<T, N4, TMA>(sm.P + ((g + 1) % NSTAGE) * PR * PP, sm.bar + (g + 1) % NSTAGE, mp, a, j0 + 1, a2,
                              a3);
        __syncthreads();  // tap tables visible

        int rot = 0;  // ring rotation: (j - j0) mod 7
#pragma unroll 1
        for (int j = j0; j < j1; ++j, ++g) {
            // ---- wait for slab j
            if constexpr (TMA) {
                mbar_wait(sm.bar + g % NSTAGE, (g / NSTAGE) & 1);
            } else {
                cp_async_wait<1>();
                __syncthreads();
            }
            const T *P = sm.P + (g % NSTAGE) * PR * PP + delta;
            T *U2 = sm.U2[g & 1];

            // ---- phase A: G2 on the halo-extended columns (2 per thread)
            if (tid < S::NPA) {
                const int c0 = tid, c1 = tid + S::NPA;   // c1 <= W, inside the staged row
                T v0[PR], v1[PR];
#pragma unroll
                for (int k = 0; k < PR; ++k) {
                    v0[k] = P[k * PP + c0];
                    v1[k] = P[k * PP + c1];
                }
#pragma unroll
                for (int i = 0; i < T2; ++i) {
                    T t[8];
                    load8(sm.tap2 + i * TP, t);
                    U2[i * W + c0] = dot7(t, v0 + i);
                    if (c1 < W) U2[i * W + c1] = dot7(t, v1 + i);
                }
            }
            __syncthreads();  // A | B

            // ---- stage slab j+2 (its stage was last read in slab j-1, finished by all threads)
            if (j + 2 < j1)
                load_slab<T, N4, TMA>(sm.P + ((g + 2) % NSTAGE) * PR * PP, sm.bar + (g + 2) % NSTAGE, mp, a, j + 2,
                                      a2, a3);
            else if constexpr (!TMA)
                cp_async_commit();

            // ---- phase B: G3 on U2 rows, R3 on p rows (4 outputs along i3, rows 2a and 2a+1)
            {
                const int i4 = tid % N4;
                const int rest = tid / N4;
                const int seg = rest % S::NS3;
                const int i2 = 2 * (rest / S::NS3);
                const int b3 = seg * 4;
                const T *u2 = U2 + i2 * W + b3 * N4 + i4;
                const T *pp = P + (i2 + 3) * PP + (b3 + 1) * N4 + i4;
                T v0[10], v1[10], p0[8], p1[8];
#pragma unroll
                for (int m = 0; m < 10; ++m) {
                    v0[m] = u2[m * N4];
                    v1[m] = u2[W + m * N4];
                }
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    p0[m] = pp[m * N4];
                    p1[m] = pp[PP + m * N4];
                }
                const int ob = i2 * T3N4 + b3 * N4 + i4;
#pragma unroll
                for (int mo = 0; mo < 4; ++mo) {
                    T t[8], tr[8];
                    load8(sm.tap3 + (b3 + mo) * TP, t);
                    load8(sm.tap3 + (b3 + mo) * TP + TR, tr);
                    const int o = ob + mo * N4;
                    sm.U3[o] = dot7(t, v0 + mo);
                    sm.U3[o + T3N4] = dot7(t, v1 + mo);
                    sm.REG[o] = dot5(tr, p0 + mo);
                    sm.REG[o + T3N4] = dot5(tr, p1 + mo);
                }
            }
            __syncthreads();  // B | C

            // ---- phase C: G4 on U3 lines, R4 on p lines (4 outputs along i4, rows 2a and 2a+1)
            T *Sb = U2;  // this slab's U2 is dead after B
#pragma unroll 1
            for (int it = tid; it < S::NPC; it += S::NTHR) {
                const int i3 = it % T3;
                const int rest = it / T3;
                const int seg = rest % S::NS4;
                const int i2 = 2 * (rest / S::NS4);
                const int b4 = seg * 4;
                const T *u0 = sm.U3 + i2 * T3N4 + i3 * N4;
                const T *pl0 = P + (i2 + 3) * PP + (i3 + 3) * N4;
                T v0[10], v1[10], p0[8], p1[8];
#pragma unroll
                for (int m = 0; m < 10; ++m) {
                    const int i4 = b4 - 3 + m;
                    const bool ok = i4 >= 0 && i4 < N4;
                    v0[m] = ok ? u0[i4] : T(0);
                    v1[m] = ok ? u0[T3N4 + i4] : T(0);
                }
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int i4 = b4 - 2 + m;
                    const bool ok = i4 >= 0 && i4 < N4;
                    p0[m] = ok ? pl0[i4] : T(0);
                    p1[m] = ok ? pl0[PP + i4] : T(0);
                }
                const int ob = i2 * T3N4 + i3 * N4 + b4;
#pragma unroll
                for (int mo = 0; mo < 4; ++mo) {
                    if (b4 + mo < N4) {
                        T t[8], tr[8];
                        load8(sm.tap4 + (b4 + mo) * TP, t);
                        load8(sm.tap4 + (b4 + mo) * TP + TR, tr);
                        const int o = ob + mo;
                        Sb[o] = dot7(t, v0 + mo);
                        Sb[o + T3N4] = dot7(t, v1 + mo);
                        sm.REG[o] += dot5(tr, p0 + mo);
                        sm.REG[o + T3N4] += dot5(tr, p1 + mo);
                    }
                }
            }
            __syncthreads();  // C | D

            // ---- phase D: R2 on the own p column, mode-1 ring (G1, R1), emission of slab j-3
            {
                T sv[T2], pc[T2], rg[T2];
                T col[T2 + 4];
#pragma unroll
                for (int k = 0; k < T2 + 4; ++k) col[k] = P[(k + 1) * PP + tid + 3 * N4];
#pragma unroll
                for (int i = 0; i < T2; ++i) {
                    T tr[8];
                    load8(sm.tap2 + i * TP + TR, tr);
                    sv[i] = Sb[i * T3N4 + tid];
                    rg[i] = sm.REG[i * T3N4 + tid] + dot5(tr, col + i);
                    pc[i] = col[i + 2];
                }
                T g1[7], r1[5];
#pragma unroll
                for (int o = -3; o <= 3; ++o) {
                    const int row = j + o;
                    const bool ok = row >= 0 && row < a.n1;
                    g1[o + 3] = ok ? __ldg(a.tg[0] + row * 7 + (3 - o)) : T(0);
                    if (o >= -2 && o <= 2) r1[o + 2] = ok ? __ldg(a.tr[0] + row * 5 + (2 - o)) : T(0);
                }
                const int oj = j - 3;
                const bool emit = oj >= o0 && oj < o1 && (a3 + tid / N4 < a.n3);
                T *dst = a.y + ((long long)(emit ? oj : 0) * a.n2 + a2) * n3n4 + a3 * N4 + tid;
                const int nrow = a.n2 - a2;
                switch (rot) {
                case 0: ring_emit<T, 0>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                case 1: ring_emit<T, 1>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                case 2: ring_emit<T, 2>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                case 3: ring_emit<T, 3>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                case 4: ring_emit<T, 4>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                case 5: ring_emit<T, 5>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                default: ring_emit<T, 6>(acc, sv, pc, rg, g1, r1, dst, n3n4, nrow, emit); break;
                }
                rot = rot == 6 ? 0 : rot + 1;
            }
            // no end-of-slab barrier: the next slab writes U2[g+1 & 1], and its
            // B/C/D buffers only after its A|B barrier
        }
        if constexpr (!TMA) cp_async_wait<0>();
        __syncthreads();  // segment end: tap tables and stages are rewritten next
    }
}

// ---------------------------------------------------------------- host side
template <typename T, int N4, bool TMA>
tca_status launch_n4(const tca_operator *op, const T *x, T *y, const int32_t *done, cudaStream_t s,
                     const CUtensorMap *map)
{
    using S = Shape<T, N4>;
    FusedArgs<T> a{};
    a.x = x;
    a.y = y;
    a.n1 = (int)op->nloc1;
    a.n2 = (int)op->n[1];
    a.n3 = (int)op->n[2];
    a.tiles3 = (a.n3 + S::T3 - 1) / S::T3;
    const int tiles2 = (a.n2 + T2 - 1) / T2;
    a.total = (long long)tiles2 * a.tiles3 * a.n1;
    for (int d = 0; d < kD; ++d) {
        a.tg[d] = (const T *)op->tapG[d];
        a.tr[d] = (const T *)op->tapR[d];
    }
    a.done = done;
    static bool attr_set = false;
    if (!attr_set) {
        TCA_CUDA_TRY(cudaFuncSetAttribute(fused_apply_kernel<T, N4, TMA>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::smem_bytes));
        attr_set = true;
    }
    long long grid = op->num_sms;
    if (grid > a.total) grid = a.total;
    if (grid < 1) grid = 1;
    CUtensorMap m{};
    if (map) m = *map;
    count_launch();
    fused_apply_kernel<T, N4, TMA><<<(unsigned)grid, S::NTHR, S::smem_bytes, s>>>(a, m);
    TCA_CUDA_TRY(cudaGetLastError());
    return TCA_OK;
}

#define TCA_FUSED_N4_LIST(X) X(1) X(2) X(4) X(7) X(8) X(15) X(16) X(32)

template <typename T, bool TMA>
tca_status launch_dispatch(const tca_operator *op, const T *x, T *y, const int32_t *done, cudaStream_t s,
                           const CUtensorMap *map)
{
    switch ((int)op->n[3]) {
#define TCA_CASE(n) \
    case n: return launch_n4<T, n, TMA>(op, x, y, done, s, map);
        TCA_FUSED_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return fail(TCA_ERR_INVALID_ARG, "fused apply: unsupported n4");
}

template <typename T>
size_t smem_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Shape<T, n>::smem_bytes;
        TCA_FUSED_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

template <typename T>
int boxw_for(int n4)
{
    switch (n4) {
#define TCA_CASE(n) \
    case n: return Shape<T, n>::BOXW;
        TCA_FUSED_N4_LIST(TCA_CASE)
#undef TCA_CASE
    }
    return 0;
}

}  // namespace fused
}  // namespace tca
