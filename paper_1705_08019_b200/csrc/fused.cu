// fused.cu -- TMA-staged, z-marching fused kernels for sm_100a.
//
//  K1  leapfrog step (rows a2 + a3 in ONE pass):  e' = e + bE.*(C^T h) - q ;  h' = h - bH.*(C e')
//  K2  Newton pair (row a6, two A-applications in ONE pass):
//        u = X w ;  y <- y + a w + b u ;  w' = X u + e2 w      (HALF: no w')
//
// Each CTA owns a BX x BY tile of (i, j) columns and marches a chunk [kb, ke) of z-planes.
// Plane k of the input state (6 components, plus coefficient arrays in ARRAY mode) is
// brought into shared memory by ONE 4-D TMA load of a (WX x (BY+2) x 1 x NC) box that
// starts at (x0-1, y0-1, k, 0); out-of-range coordinates (the PEC box, z = -1 or nz) are
// zero-filled by the TMA unit, which is exactly the "virtual DOF reads 0" rule.  An
// S-stage mbarrier ring keeps S-1 planes in flight per CTA.  The first curl half is
// evaluated on the tile plus a one-cell halo (recomputed, never exchanged), kept in a
// 2-plane shared ring, and the second half consumes it for the tile:
//   leapfrog:  e'(k+1) on [x0, x0+BX] x [y0, y0+BY], then h'(k) on the tile
//   pair:      u_e(k+1) on the +1 halo, u_h(k) on the -1 halo, then w'(k), y(k)
// Input and output states are different buffers (ping-pong): the halos read the input.
// HBM traffic per cell-update: leapfrog reads e,h and writes e,h (12 values);
// pair reads w, y and writes w', y (24 values per two A-applications) -- DESIGN.md.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "internal.h"
#include "kernels_common.cuh"

namespace pe {

// ---------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---------------------------------------------------------------------------------------
// geometry
// ---------------------------------------------------------------------------------------
template <typename T, int BX_, int BY_>
struct Geo {
    static constexpr int BX = BX_, BY = BY_;
    static constexpr int NT = BX * BY;                              // tile points (phase B)
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int OX = VEC;                                  // tile origin inside the box (the TMA x start must be 16 B aligned)
    static constexpr int WX = ((OX + BX + 1 + VEC - 1) / VEC) * VEC; // TMA box width (16 B multiple)
    static constexpr int HY = BY + 2;
    static constexpr int PL = WX * HY;                              // one component of a stage
    static constexpr int EX = BX + 1, EY = BY + 1;                 // halo-extended ring plane
    static constexpr int RP = EX * EY;                              // one component of a ring plane
    static constexpr int NTHR = ((RP + 31) / 32) * 32;               // threads: phase A in one pass
};

struct Sched {
    int tiles_x, tiles_y, ntiles, chunk, nchunks, units;
};

struct SrcList {
    int n;
    int c[16], i[16], j[16], k[16];
};

template <typename T, int EM, bool HA>
struct NComp {
    static constexpr int value = 6 + (EM == 2 ? 3 : 0) + (HA ? 3 : 0);
};

// Stage layout: [state box 6*PL | cE box 3*PL (ARRAY) | cH box 3*PL (HA)], each region
// padded to 128 B because every TMA destination must be 128-byte aligned.
template <typename T, int EM, bool HA, typename G>
struct StageL {
    static constexpr int A = 128 / (int)sizeof(T);
    static constexpr int ST = ((6 * G::PL + A - 1) / A) * A;
    static constexpr int CE = EM == 2 ? ((3 * G::PL + A - 1) / A) * A : 0;
    static constexpr int CH = HA ? ((3 * G::PL + A - 1) / A) * A : 0;
    static constexpr int SZ = ST + CE + CH;
};

template <typename T, int EM, bool HA, typename G>
__device__ __forceinline__ T stage_bE(const Coef<T, EM, HA> &cf, const T *st, int c, int kk, int sidx) {
    if (EM == 2) return st[StageL<T, EM, HA, G>::ST + c * G::PL + sidx] * cf.sig;
    if (EM == 1) return __ldg(cf.tab + c * cf.nz + kk) * cf.sig;
    return cf.cEs[c] * cf.sig;
}
template <typename T, int EM, bool HA, typename G>
__device__ __forceinline__ T stage_bH(const Coef<T, EM, HA> &cf, const T *st, int c, int sidx) {
    using SL = StageL<T, EM, HA, G>;
    if (HA) return st[SL::ST + SL::CE + c * G::PL + sidx] * cf.sig;
    return cf.cHs[c] * cf.sig;
}

// issue the TMA loads of plane `kz` into stage buffer `dst` (state + coefficient maps)
template <typename T, int EM, bool HA, typename G>
__device__ __forceinline__ void issue_plane(T *dst, uint64_t *bar, const CUtensorMap *tm_state,
                                            const CUtensorMap *tm_cE, const CUtensorMap *tm_cH, int x0,
                                            int y0, int kz) {
    using SL = StageL<T, EM, HA, G>;
    constexpr uint32_t bytes = (uint32_t)(NComp<T, EM, HA>::value * G::PL * sizeof(T));
    mbar_expect_tx(bar, bytes);
    tma_load_4d(dst, tm_state, bar, x0 - G::OX, y0 - 1, kz, 0);
    if (EM == 2) tma_load_4d(dst + SL::ST, tm_cE, bar, x0 - G::OX, y0 - 1, kz, 0);
    if (HA) tma_load_4d(dst + SL::ST + SL::CE, tm_cH, bar, x0 - G::OX, y0 - 1, kz, 0);
}

// (C^T h) at stage coords (xx, yy) from planes H1 = k+1 (this plane) and H0 = k (below)
template <typename T, typename G>
__device__ __forceinline__ void curlT_stage(const T *H1, const T *H0, int s, T &c0, T &c1, T &c2) {
    const T *hx = H1 + 3 * G::PL, *hy = H1 + 4 * G::PL, *hz = H1 + 5 * G::PL;
    const T hz0 = hz[s], hz_jm = hz[s - G::WX], hy0 = hy[s], hy_km = H0[4 * G::PL + s];
    const T hx0 = hx[s], hx_km = H0[3 * G::PL + s], hz_im = hz[s - 1], hy_im = hy[s - 1];
    const T hx_jm = hx[s - G::WX];
    c0 = ((hz0 - hz_jm) - hy0) + hy_km;
    c1 = ((hx0 - hx_km) - hz0) + hz_im;
    c2 = ((hy0 - hy_im) - hx0) + hx_jm;
}
// (C e) at stage coords from planes E0 = k (this plane) and E1 = k+1 (above)
template <typename T, typename G>
__device__ __forceinline__ void curl_stage(const T *E0, const T *E1, int s, T &c0, T &c1, T &c2) {
    const T *ex = E0, *ey = E0 + G::PL, *ez = E0 + 2 * G::PL;
    const T ex0 = ex[s], ey0 = ey[s], ez0 = ez[s];
    const T ez_jp = ez[s + G::WX], ex_jp = ex[s + G::WX];
    const T ey_kp = E1[G::PL + s], ex_kp = E1[s];
    const T ez_ip = ez[s + 1], ey_ip = ey[s + 1];
    c0 = ((ey0 + ez_jp) - ey_kp) - ez0;
    c1 = ((ez0 + ex_kp) - ez_ip) - ex0;
    c2 = ((ex0 + ey_ip) - ex_jp) - ey0;
}

// ---------------------------------------------------------------------------------------
// K1: fused leapfrog step
// ---------------------------------------------------------------------------------------
template <typename T, int EM, bool HA, int BX, int BY, int S>
__global__ void __launch_bounds__(Geo<T, BX, BY>::NTHR) leapfrog_fused_kernel(
    const __grid_constant__ CUtensorMap tm_state, const __grid_constant__ CUtensorMap tm_cE,
    const __grid_constant__ CUtensorMap tm_cH, Dev<T> D, Coef<T, EM, HA> cf, T *__restrict__ out,
    Sched sch, SrcList src, const T *__restrict__ q) {
    using G = Geo<T, BX, BY>;
    constexpr int NC = NComp<T, EM, HA>::value;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *stages = reinterpret_cast<T *>(smem_raw);
    T *ring = stages + S * StageL<T, EM, HA, G>::SZ;                   // [2][3][EY][EX] e' planes
    uint64_t *bars = reinterpret_cast<uint64_t *>(ring + 2 * 3 * G::RP);
    const int tid = threadIdx.x;
    const int tx = tid % BX, ty = tid / BX;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint32_t lcount = 0;   // planes loaded by this CTA so far (ring position)
    for (int unit = blockIdx.x; unit < sch.units; unit += gridDim.x) {
        const int tile = unit % sch.ntiles, chunk = unit / sch.ntiles;
        const int x0 = (tile % sch.tiles_x) * BX, y0 = (tile / sch.tiles_x) * BY;
        const int kb = chunk * sch.chunk, ke = min(kb + sch.chunk, D.nz);
        const int nplanes = ke - kb + 2;                 // planes kb-1 .. ke
        if (tid == 0)
            for (int p = 0; p < min(S, nplanes); ++p) {
                const uint32_t L = lcount + p;
                issue_plane<T, EM, HA, G>(stages + (L % S) * StageL<T, EM, HA, G>::SZ, &bars[L % S], &tm_state, &tm_cE,
                                          &tm_cH, x0, y0, kb - 1 + p);
            }
        for (int p = 0; p + 1 < nplanes; ++p) {         // iteration on planes k = kb-1+p, k+1
            const int k = kb - 1 + p;
            const uint32_t L0 = lcount + p, L1 = L0 + 1;
            if (p == 0) mbar_wait(&bars[L0 % S], (L0 / S) & 1);
            mbar_wait(&bars[L1 % S], (L1 / S) & 1);
            const T *P0 = stages + (L0 % S) * StageL<T, EM, HA, G>::SZ;   // plane k
            const T *P1 = stages + (L1 % S) * StageL<T, EM, HA, G>::SZ;   // plane k+1
            T *R1 = ring + ((k + 1) & 1) * 3 * G::RP;
            const int kk = k + 1;
            // ---- e'(k+1) on the tile and its +1 halo ----
            for (int q2 = tid; q2 < G::RP; q2 += G::NTHR) {
                const int ii = q2 % G::EX, jj = q2 / G::EX;
                const int i = x0 + ii, j = y0 + jj;
                const int s = (jj + 1) * G::WX + (ii + G::OX);
                T c0, c1, c2;
                curlT_stage<T, G>(P1, P0, s, c0, c1, c2);
                const bool valid = i < D.nx && j < D.ny && kk < D.nz && kk >= 0;
                T en[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const T cc = c == 0 ? c0 : (c == 1 ? c1 : c2);
                    en[c] = (valid && D.e_live(c, i, j, kk))
                                ? P1[c * G::PL + s] + stage_bE<T, EM, HA, G>(cf, P1, c, kk, s) * cc
                                : T(0);
                }
                if (valid)
                    for (int r = 0; r < src.n; ++r)
                        if (src.k[r] == kk && src.i[r] == i && src.j[r] == j) {
                            const int sc = src.c[r];
                            const T qv = q[r];
                            if (sc == 0) en[0] = en[0] - qv;
                            if (sc == 1) en[1] = en[1] - qv;
                            if (sc == 2) en[2] = en[2] - qv;
                        }
#pragma unroll
                for (int c = 0; c < 3; ++c) R1[c * G::RP + q2] = en[c];
                if (ii < BX && jj < BY && valid && kk >= kb && kk < ke) {
                    const int64_t gi = D.idx(i, j, kk);
#pragma unroll
                    for (int c = 0; c < 3; ++c) out[c * D.cs + gi] = en[c];
                }
            }
            __syncthreads();
            // ---- h'(k) on the tile ----
            if (k >= kb && tid < G::NT) {
                const T *R0 = ring + (k & 1) * 3 * G::RP;
                const int i = x0 + tx, j = y0 + ty;
                const int r = ty * G::EX + tx;
                const T ex0 = R0[r], ey0 = R0[G::RP + r], ez0 = R0[2 * G::RP + r];
                const T ez_jp = R0[2 * G::RP + r + G::EX], ex_jp = R0[r + G::EX];
                const T ez_ip = R0[2 * G::RP + r + 1], ey_ip = R0[G::RP + r + 1];
                const T ex_kp = R1[r], ey_kp = R1[G::RP + r];
                const T c0 = ((ey0 + ez_jp) - ey_kp) - ez0;
                const T c1 = ((ez0 + ex_kp) - ez_ip) - ex0;
                const T c2 = ((ex0 + ey_ip) - ex_jp) - ey0;
                const int s = (ty + 1) * G::WX + (tx + G::OX);
                if (i < D.nx && j < D.ny) {
                    const int64_t gi = D.idx(i, j, k);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const T cc = c == 0 ? c0 : (c == 1 ? c1 : c2);
                        const T hv = P0[(3 + c) * G::PL + s];
                        out[(3 + c) * D.cs + gi] =
                            D.h_live(c, i, j, k) ? hv - stage_bH<T, EM, HA, G>(cf, P0, c, s) * cc : hv;
                    }
                }
            }
            __syncthreads();
            // plane k is consumed: refill its slot with plane k + S
            if (tid == 0 && p + S < nplanes) {
                const uint32_t L = lcount + p + S;
                issue_plane<T, EM, HA, G>(stages + (L % S) * StageL<T, EM, HA, G>::SZ, &bars[L % S], &tm_state, &tm_cE,
                                          &tm_cH, x0, y0, kb - 1 + p + S);
            }
        }
        lcount += nplanes;
    }
}

// ---------------------------------------------------------------------------------------
// K2: fused Newton pair  u = X w ; y <- (init?0:y) + a w + b u ; [w' = X u + e2 w]
// ---------------------------------------------------------------------------------------
template <typename T, int EM, bool HA, int BX, int BY, int S>
__global__ void __launch_bounds__(Geo<T, BX, BY>::NTHR) pair_fused_kernel(
    const __grid_constant__ CUtensorMap tm_state, const __grid_constant__ CUtensorMap tm_cE,
    const __grid_constant__ CUtensorMap tm_cH, Dev<T> D, Coef<T, EM, HA> cf, T *__restrict__ wout,
    T *__restrict__ y, Sched sch, T a, T b, T e2, int init, int do_w) {
    using G = Geo<T, BX, BY>;
    constexpr int NC = NComp<T, EM, HA>::value;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *stages = reinterpret_cast<T *>(smem_raw);
    T *UE = stages + S * StageL<T, EM, HA, G>::SZ;                    // [2][3][EY][EX]: u_e at (ii, jj) in [0,BX]x[0,BY]
    T *UH = UE + 2 * 3 * G::RP;                         // [2][3][EY][EX]: u_h at (ii-1, jj-1)
    uint64_t *bars = reinterpret_cast<uint64_t *>(UH + 2 * 3 * G::RP);
    const int tid = threadIdx.x;
    const int tx = tid % BX, ty = tid / BX;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint32_t lcount = 0;
    for (int unit = blockIdx.x; unit < sch.units; unit += gridDim.x) {
        const int tile = unit % sch.ntiles, chunk = unit / sch.ntiles;
        const int x0 = (tile % sch.tiles_x) * BX, y0 = (tile / sch.tiles_x) * BY;
        const int kb = chunk * sch.chunk, ke = min(kb + sch.chunk, D.nz);
        const int nplanes = ke - kb + 2;
        if (tid == 0)
            for (int p = 0; p < min(S, nplanes); ++p) {
                const uint32_t L = lcount + p;
                issue_plane<T, EM, HA, G>(stages + (L % S) * StageL<T, EM, HA, G>::SZ, &bars[L % S], &tm_state, &tm_cE,
                                          &tm_cH, x0, y0, kb - 1 + p);
            }
        const int i_own = x0 + tx, j_own = y0 + ty;
        const bool own_in = tid < G::NT && i_own < D.nx && j_own < D.ny;
        for (int p = 0; p + 1 < nplanes; ++p) {
            const int k = kb - 1 + p;
            const uint32_t L0 = lcount + p, L1 = L0 + 1;
            // prefetch y(k) for the own point (consumed after the halo phase)
            T yv[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
            if (k >= kb && own_in && !init) {
                const int64_t gi = D.idx(i_own, j_own, k);
#pragma unroll
                for (int c = 0; c < 6; ++c) yv[c] = y[c * D.cs + gi];
            }
            if (p == 0) mbar_wait(&bars[L0 % S], (L0 / S) & 1);
            mbar_wait(&bars[L1 % S], (L1 / S) & 1);
            const T *P0 = stages + (L0 % S) * StageL<T, EM, HA, G>::SZ;   // w plane k
            const T *P1 = stages + (L1 % S) * StageL<T, EM, HA, G>::SZ;   // w plane k+1
            T *UE1 = UE + ((k + 1) & 1) * 3 * G::RP;         // u_e(k+1)
            T *UH0 = UH + (k & 1) * 3 * G::RP;               // u_h(k)
            const int kk = k + 1;
            for (int q2 = tid; q2 < G::RP; q2 += G::NTHR) {
                const int ii = q2 % G::EX, jj = q2 / G::EX;
                // u_e(k+1) at (x0+ii, y0+jj)
                {
                    const int i = x0 + ii, j = y0 + jj;
                    const int s = (jj + 1) * G::WX + (ii + G::OX);
                    T c0, c1, c2;
                    curlT_stage<T, G>(P1, P0, s, c0, c1, c2);
                    const bool valid = i < D.nx && j < D.ny && kk < D.nz;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const T cc = c == 0 ? c0 : (c == 1 ? c1 : c2);
                        UE1[c * G::RP + q2] = (valid && D.e_live(c, i, j, kk))
                                                  ? stage_bE<T, EM, HA, G>(cf, P1, c, kk, s) * cc
                                                  : T(0);
                    }
                }
                // u_h(k) at (x0+ii-1, y0+jj-1)
                {
                    const int i = x0 + ii - 1, j = y0 + jj - 1;
                    const int s = jj * G::WX + (ii - 1 + G::OX);
                    T c0, c1, c2;
                    curl_stage<T, G>(P0, P1, s, c0, c1, c2);
                    const bool valid = i >= 0 && j >= 0 && i < D.nx && j < D.ny && k >= 0 && k < D.nz;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const T cc = c == 0 ? c0 : (c == 1 ? c1 : c2);
                        UH0[c * G::RP + q2] = (valid && D.h_live(c, i, j, k))
                                                  ? -(stage_bH<T, EM, HA, G>(cf, P0, c, s) * cc)
                                                  : T(0);
                    }
                }
            }
            __syncthreads();
            if (k >= kb && own_in) {
                const T *UE0 = UE + (k & 1) * 3 * G::RP;     // u_e(k)
                const T *UHm = UH + ((k - 1) & 1) * 3 * G::RP; // u_h(k-1)
                const int re = ty * G::EX + tx;              // u_e ring index of the own point
                const int rh = (ty + 1) * G::EX + (tx + 1);  // u_h ring index of the own point
                const int s = (ty + 1) * G::WX + (tx + G::OX);   // stage index of the own point
                const int64_t gi = D.idx(i_own, j_own, k);
                T un[6], wn[6];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    un[c] = UE0[c * G::RP + re];
                    un[3 + c] = UH0[c * G::RP + rh];
                }
                if (do_w) {
                    // w'_h(k) = -bH C u_e + e2 w_h
                    const T ux0 = un[0], uy0 = un[1], uz0 = un[2];
                    const T uz_jp = UE0[2 * G::RP + re + G::EX], ux_jp = UE0[re + G::EX];
                    const T uz_ip = UE0[2 * G::RP + re + 1], uy_ip = UE0[G::RP + re + 1];
                    const T ux_kp = UE1[re], uy_kp = UE1[G::RP + re];
                    const T c0 = ((uy0 + uz_jp) - uy_kp) - uz0;
                    const T c1 = ((uz0 + ux_kp) - uz_ip) - ux0;
                    const T c2 = ((ux0 + uy_ip) - ux_jp) - uy0;
                    // w'_e(k) = bE C^T u_h + e2 w_e
                    const T hx0 = un[3], hy0 = un[4], hz0 = un[5];
                    const T hz_jm = UH0[2 * G::RP + rh - G::EX], hx_jm = UH0[rh - G::EX];
                    const T hz_im = UH0[2 * G::RP + rh - 1], hy_im = UH0[G::RP + rh - 1];
                    const T hy_km = UHm[G::RP + rh], hx_km = UHm[rh];
                    const T d0 = ((hz0 - hz_jm) - hy0) + hy_km;
                    const T d1 = ((hx0 - hx_km) - hz0) + hz_im;
                    const T d2 = ((hy0 - hy_im) - hx0) + hx_jm;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const T ce = c == 0 ? d0 : (c == 1 ? d1 : d2);
                        const T ch = c == 0 ? c0 : (c == 1 ? c1 : c2);
                        const T xe = D.e_live(c, i_own, j_own, k) ? stage_bE<T, EM, HA, G>(cf, P0, c, k, s) * ce : T(0);
                        const T xh = D.h_live(c, i_own, j_own, k) ? -(stage_bH<T, EM, HA, G>(cf, P0, c, s) * ch) : T(0);
                        wn[c] = xe + e2 * P0[c * G::PL + s];
                        wn[3 + c] = xh + e2 * P0[(3 + c) * G::PL + s];
                    }
#pragma unroll
                    for (int c = 0; c < 6; ++c) wout[c * D.cs + gi] = wn[c];
                }
#pragma unroll
                for (int c = 0; c < 6; ++c) y[c * D.cs + gi] = (yv[c] + a * P0[c * G::PL + s]) + b * un[c];
            }
            __syncthreads();
            if (tid == 0 && p + S < nplanes) {
                const uint32_t L = lcount + p + S;
                issue_plane<T, EM, HA, G>(stages + (L % S) * StageL<T, EM, HA, G>::SZ, &bars[L % S], &tm_state, &tm_cE,
                                          &tm_cH, x0, y0, kb - 1 + p + S);
            }
        }
        lcount += nplanes;
    }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

bool fused_supported(const Grid &g) {
    if (getenv("PARAEXP_FORCE_UNFUSED")) return false;
    if (g.nx < 16 || g.ny < 8) return false;   // tiny grids: unfused kernels
    return get_encode() != nullptr;
}

template <typename T>
static int make_map(CUtensorMap *m, const Grid &g, const void *base, int ncomp, int wx, int hy) {
    auto enc = get_encode();
    if (!enc) return fail(PARAEXP_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz, (cuuint64_t)ncomp};
    const cuuint64_t strides[3] = {(cuuint64_t)(g.L.px * sizeof(T)), (cuuint64_t)(g.L.plane * sizeof(T)),
                                   (cuuint64_t)(g.L.cs * sizeof(T))};
    const cuuint32_t box[4] = {(cuuint32_t)wx, (cuuint32_t)hy, 1u, (cuuint32_t)ncomp};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                     const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PARAEXP_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return PARAEXP_OK;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// choose the z-chunk so that units / resident CTAs is close to an integer and halo planes
// (2 per chunk) stay a small fraction
static Sched make_sched(const Grid &g, int BX, int BY, int resident) {
    Sched s;
    s.tiles_x = (g.nx + BX - 1) / BX;
    s.tiles_y = (g.ny + BY - 1) / BY;
    s.ntiles = s.tiles_x * s.tiles_y;
    double best = 1e300;
    int bc = g.nz;
    for (int ch = 1; ch <= g.nz; ++ch) {
        const int nch = (g.nz + ch - 1) / ch;
        if (ch < std::min(g.nz, 8) && nch > 1) continue;
        const double units = (double)s.ntiles * nch;
        const double waves = units / resident;
        const double eff_waves = std::ceil(waves);
        // cost ~ rounds * (chunk + 2 halo planes)
        const double cost = eff_waves * (double)(ch + 2);
        if (cost < best - 1e-9) {
            best = cost;
            bc = ch;
        }
    }
    if (const char *ev = getenv("PARAEXP_ZCHUNK")) bc = std::max(1, std::min(g.nz, atoi(ev)));
    s.chunk = bc;
    s.nchunks = (g.nz + bc - 1) / bc;
    s.units = s.ntiles * s.nchunks;
    return s;
}

template <typename T, int EM, bool HA, int BX, int BY, int S>
struct FusedCfg {
    using G = Geo<T, BX, BY>;
    static constexpr int NC = NComp<T, EM, HA>::value;
    static constexpr size_t lf_smem = (size_t)(S * StageL<T, EM, HA, G>::SZ + 2 * 3 * G::RP) * sizeof(T) + 8 * S + 16;
    static constexpr size_t pair_smem = (size_t)(S * StageL<T, EM, HA, G>::SZ + 4 * 3 * G::RP) * sizeof(T) + 8 * S + 16;
};

template <typename T, int EM, bool HA>
static int leapfrog_fused_T(const KernelArgs &ka, void *bufs[2], int64_t nsteps, const SrcDev *,
                            int nsrc, const void *q_dev, const std::vector<SrcDev> &hsrc) {
    constexpr int BX = 32, BY = 8, S = 3;
    using Cfg = FusedCfg<T, EM, HA, BX, BY, S>;
    using G = Geo<T, BX, BY>;
    const Grid &g = *ka.g;
    auto kern = leapfrog_fused_kernel<T, EM, HA, BX, BY, S>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::lf_smem);
        attr_set = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NTHR, Cfg::lf_smem);
    if (per_sm < 1) return fail(PARAEXP_ECUDA, "fused leapfrog kernel does not fit on an SM");
    const Sched sch = make_sched(g, BX, BY, per_sm * num_sms());
    const int grid = std::min(sch.units, per_sm * num_sms());
    auto D = make_dev<T>(g);
    auto cf = make_coef<T, EM, HA>(g, 1.0);
    CUtensorMap tmE, tmH, tmA, tmB;
    int rc;
    if (EM == 2 && (rc = make_map<T>(&tmE, g, g.d_cE_arr, 3, G::WX, G::HY))) return rc;
    if (HA && (rc = make_map<T>(&tmH, g, g.d_cH_arr, 3, G::WX, G::HY))) return rc;
    if ((rc = make_map<T>(&tmA, g, bufs[0], 6, G::WX, G::HY))) return rc;
    if ((rc = make_map<T>(&tmB, g, bufs[1], 6, G::WX, G::HY))) return rc;
    SrcList sl;
    sl.n = nsrc;
    for (int r = 0; r < nsrc && r < 16; ++r) {
        sl.c[r] = hsrc[r].comp;
        sl.i[r] = hsrc[r].i;
        sl.j[r] = hsrc[r].j;
        sl.k[r] = hsrc[r].k;
    }
    cudaStream_t s = (cudaStream_t)ka.stream;
    for (int64_t m = 0; m < nsteps; ++m) {
        const bool even = (m % 2) == 0;
        kern<<<grid, G::NTHR, Cfg::lf_smem, s>>>(even ? tmA : tmB, tmE, tmH, D, cf,
                                                 (T *)(even ? bufs[1] : bufs[0]), sch, sl,
                                                 nsrc ? (const T *)q_dev + m * nsrc : nullptr);
        ++*ka.launches;
    }
    if (nsteps % 2) std::swap(bufs[0], bufs[1]);
    return check_cuda("leapfrog fused");
}

int k_leapfrog_fused(const KernelArgs &ka, void *bufs[2], int64_t nsteps, const SrcDev *src_dev,
                     int nsrc, const void *q_dev) {
    if (nsrc > 16) return k_leapfrog_unfused(ka, bufs[0], nsteps, src_dev, nsrc, q_dev);
    const std::vector<SrcDev> &hsrc = ka.g->h_src;
    return with_types(*ka.g, 1.0, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        return leapfrog_fused_T<T, EM, HA>(ka, bufs, nsteps, src_dev, nsrc, q_dev, hsrc);
    });
}

int zero_node_launch(const KernelArgs &ka, const Plan &plan, const void *w, void *wn, void *y,
                     double c, int init, int do_w);

template <typename T, int EM, bool HA>
static int poly_fused_T(const KernelArgs &ka, const Plan &plan, void *bufs[4]) {
    constexpr int BX = 32, BY = 8, S = 3;
    using Cfg = FusedCfg<T, EM, HA, BX, BY, S>;
    using G = Geo<T, BX, BY>;
    const Grid &g = *ka.g;
    auto kern = pair_fused_kernel<T, EM, HA, BX, BY, S>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::pair_smem);
        attr_set = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NTHR, Cfg::pair_smem);
    if (per_sm < 1) return fail(PARAEXP_ECUDA, "fused pair kernel does not fit on an SM");
    const Sched sch = make_sched(g, BX, BY, per_sm * num_sms());
    const int grid = std::min(sch.units, per_sm * num_sms());
    auto D = make_dev<T>(g);
    auto cf = make_coef<T, EM, HA>(g, plan.sigma);
    CUtensorMap tmE, tmH;
    int rc;
    if (EM == 2 && (rc = make_map<T>(&tmE, g, g.d_cE_arr, 3, G::WX, G::HY))) return rc;
    if (HA && (rc = make_map<T>(&tmH, g, g.d_cH_arr, 3, G::WX, G::HY))) return rc;
    cudaStream_t s = (cudaStream_t)ka.stream;
    T *w = (T *)bufs[0], *yy = (T *)bufs[1], *sp = (T *)bufs[2], *sp2 = (T *)bufs[3];
    int init = 1;
    for (const Op &op : plan.ops) {
        if (op.kind == 0 || op.kind == 1) {
            CUtensorMap tmW;
            if ((rc = make_map<T>(&tmW, g, w, 6, G::WX, G::HY))) return rc;
            const int do_w = op.kind == 0;
            kern<<<grid, G::NTHR, Cfg::pair_smem, s>>>(tmW, tmE, tmH, D, cf, sp, yy, sch, T(op.a), T(op.b),
                                                       T(op.e2), init, do_w);
            ++*ka.launches;
            if (do_w) std::swap(w, sp);
        } else {
            const int do_w = op.kind == 2;
            if ((rc = zero_node_launch(ka, plan, w, sp, yy, op.a, init, do_w))) return rc;
            if (do_w) std::swap(w, sp);
        }
        init = 0;
    }
    bufs[0] = yy;
    bufs[1] = w;
    bufs[2] = sp;
    bufs[3] = sp2;
    return check_cuda("poly fused");
}

int k_poly_substep_fused(const KernelArgs &ka, const Plan &plan, void *bufs[4]) {
    return with_types(*ka.g, plan.sigma, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        return poly_fused_T<T, EM, HA>(ka, plan, bufs);
    });
}

}  // namespace pe
