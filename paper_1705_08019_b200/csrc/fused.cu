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
#include <type_traits>
#include <map>
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
#ifdef PARAEXP_DEBUG_CHECKS
    uint64_t spins = 0;
#endif
    while (!done) {
#ifdef PARAEXP_DEBUG_CHECKS
        PE_CHECK(++spins < (1ull << 28), "mbarrier wait never completed (TMA byte count / phase)");
#endif
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


// Programmatic dependent launch (PDL): the fused kernels are launched with programmatic stream
// serialisation, so a kernel's launch and CTA setup overlap the tail of the previous one; every
// fused kernel first waits for its predecessor grid to complete (griddepcontrol.wait, which also
// makes that grid's memory visible) before touching global memory, so semantics are unchanged.
__device__ __forceinline__ void pdl_sync() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("PARAEXP_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
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
    // dynamic unit order (ctr != nullptr): CTAs grab units from a grid-owned monotone counter,
    // so the units in flight are always a contiguous window of the chunk-major sequence and
    // x/y-neighbour tiles run within a fraction of a unit of each other (their halo planes
    // stay in L2 however many waves a launch has).  Each launch advances the counter by
    // exactly units + gridDim (every CTA ends with one failing grab); base is its start.
    unsigned long long *ctr;
    unsigned long long base;
    int lookahead;   // cross-unit prefetch of the next unit's first planes (PARAEXP_NO_LOOKAHEAD=1: off)
};

// unit loop: static stride (ctr == nullptr) or dynamic grabs; uniform per CTA
__device__ __forceinline__ int grab_unit(const Sched &sch, int prev) {
    if (!sch.ctr) return prev < 0 ? (int)blockIdx.x : prev + (int)gridDim.x;
    __shared__ int s_unit;
    __syncthreads();                                      // previous s_unit consumed
    if (threadIdx.x == 0) {
        const long long d = (long long)(atomicAdd(sch.ctr, 1ull) - sch.base);
        s_unit = (d < 0 || d > 0x7fffffffLL) ? 0x7fffffff : (int)d;   // never loop on a bad count
    }
    __syncthreads();
    return s_unit;
}

// Lookahead grab of the NEXT unit by thread 0 alone (no barrier), used by the kernels that
// prefetch the next unit's first planes while the current unit drains (cross-unit pipelining):
// the same counter as grab_unit (each CTA still ends with exactly one failing grab) or the
// static stride.
__device__ __forceinline__ int grab_next_t0(const Sched &sch, int cur) {
    if (!sch.ctr) return cur + (int)gridDim.x;
    const long long d = (long long)(atomicAdd(sch.ctr, 1ull) - sch.base);
    return (d < 0 || d > 0x7fffffffLL) ? 0x7fffffff : (int)d;
}

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

// z-table coefficients (EM == 1, layered materials) of a unit's planes kb-1 .. kb+nplanes-2,
// scaled by sigma, staged in shared memory once per unit: a per-plane __ldg of the table from
// global memory sat on the critical path of every plane iteration (ncu: ~8-11% of the warp
// stall samples of K1r / K2 waited on it -- the streaming y / state traffic evicts the table's
// lines from L1).  zt[c * ZT_ROW + q] = bE_c at plane kb - 1 + q (0 outside [0, nz)).
constexpr int ZT_ROW = 132;      // >= max z-chunk (130, make_sched) + 2
template <typename T, int EM>
struct ZtL {
    static constexpr int N = EM == 1 ? 3 * ZT_ROW : 0;
};
template <typename T, int EM, bool HA>
__device__ __forceinline__ void stage_ztab(T *zt, const Coef<T, EM, HA> &cf, int kb, int nplanes, int nz) {
    if constexpr (EM == 1) {
        for (int q = threadIdx.x; q < 3 * nplanes; q += blockDim.x) {
            const int c = q / nplanes, r = q - c * nplanes, kz = kb - 1 + r;
            zt[c * ZT_ROW + r] = (kz >= 0 && kz < nz) ? __ldg(cf.tab + c * nz + kz) * cf.sig : T(0);
        }
        __syncthreads();
    }
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
// K1r: fused leapfrog step, row-aligned warps and register-carried own values
// ---------------------------------------------------------------------------------------
// Per-CTA pipeline (S stages, ring depth 2, two barriers per plane).  Iteration p works on
// planes k = kb-1+p and k+1:
//   phase A: e'(k+1) on the tile + halo  -> ring slot (k+1) % 2 (and global for tile points)
//   barrier
//   phase B: h'(k) on the tile           -> global
//   barrier, refill the stage of plane k
// TR: also accumulate the step's energy E_{m+1} = dt [sum e'^2/cE + sum h h'/cH] (eq:energy)
// and write the probe values e' (f1; paraexp.h trace).
// ---------------------------------------------------------------------------------------
// K1r: the leapfrog step with row-aligned warps and register-carried own values
// ---------------------------------------------------------------------------------------
// Mapping:
//  * phase-A points are mapped so that warps 0..BY cover whole 32-wide rows (the +1 halo
//    column x0+BX is handled by the last warp): no warp straddles two rows;
//  * the thread of tile point (tx, ty) is the phase-A thread of the same point, so phase B
//    takes e'(k), e'(k+1) and h(k) at its own point from registers (only the four i+1 / j+1
//    neighbours of e'(k) are read from shared memory), and phase A carries h(k) at its own
//    point from the previous plane (only h(k+1) and its i-1 / j-1 neighbours are read).
template <typename T, int EM, bool HA, int BX, int BY, int S, bool TR>
__global__ void __launch_bounds__(Geo<T, BX, BY>::NTHR, 3) leapfrog_r_kernel(
    const __grid_constant__ CUtensorMap tm_state, const __grid_constant__ CUtensorMap tm_cE,
    const __grid_constant__ CUtensorMap tm_cH, Dev<T> D, Coef<T, EM, HA> cf, T *__restrict__ out,
    Sched sch, SrcList src, const T *__restrict__ q, const __grid_constant__ TraceDev tr) {
    pdl_sync();
    using G = Geo<T, BX, BY>;
    using SL = StageL<T, EM, HA, G>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *stages = reinterpret_cast<T *>(smem_raw);
    T *ring = stages + S * SL::SZ;                       // [2][3][EY][EX] e' planes
    T *zt = ring + 2 * 3 * G::RP;                         // [3][ZT_ROW] z-table (EM == 1)
    uint64_t *bars = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(zt + ZtL<T, EM>::N) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x;
    constexpr int MAIN = BX * G::EY;                      // row-aligned phase-A points
    const bool hasA = tid < G::RP;
    const int ii = tid < MAIN ? tid % BX : BX, jj = tid < MAIN ? tid / BX : tid - MAIN;
    const int rA = jj * G::EX + ii;                       // ring index of the phase-A point
    const int sA = (jj + 1) * G::WX + ii + G::OX;         // stage index of the phase-A point
    const bool tileA = ii < BX && jj < BY;                // == phase-B thread of the same point
    T bE0 = cf.cEs[0] * cf.sig, bE1 = cf.cEs[1] * cf.sig, bE2 = cf.cEs[2] * cf.sig;
    const T bH0 = cf.cHs[0] * cf.sig, bH1 = cf.cHs[1] * cf.sig, bH2 = cf.cHs[2] * cf.sig;
    if (tid == 0) {
        for (int s2 = 0; s2 < S; ++s2) mbar_init(&bars[s2], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint32_t lcount = 0;
    double eacc = 0.0;
    // cross-unit pipelining (as in K2): thread 0 issues the next unit's first planes into the
    // stage slots the draining unit frees
    __shared__ int s_next;
    int pre = 0;
    int unit = grab_unit(sch, -1);
    while (unit < sch.units) {
        const int tile = unit % sch.ntiles, chunk = unit / sch.ntiles;
        const int x0 = (tile % sch.tiles_x) * BX, y0 = (tile / sch.tiles_x) * BY;
        const int kb = chunk * sch.chunk, ke = min(kb + sch.chunk, D.nz);
        const int nplanes = ke - kb + 2;
        const int pre_cur = pre;
        pre = 0;
        int nxt = 0x7fffffff, nx0 = 0, ny0 = 0, nkb = 0, nke = 0;
        stage_ztab<T, EM, HA>(zt, cf, kb, nplanes, D.nz);
        const int iA = x0 + ii, jA = y0 + jj;
        const bool inA = hasA && iA < D.nx && jA < D.ny;
        const bool lxA = inA && jA > 0, lyA = inA && iA > 0, lzA = inA && iA > 0 && jA > 0;
        const bool wrA = inA && tileA;
        uint32_t smask = 0, pmask = 0;
        for (int r = 0; r < src.n; ++r)
            if (inA && src.i[r] == iA && src.j[r] == jA) smask |= 1u << r;
        if (TR)
            for (int r = 0; r < tr.np; ++r)
                if (wrA && tr.i[r] == iA && tr.j[r] == jA) pmask |= 1u << r;
        T *oA = out + D.idx(wrA ? iA : 0, wrA ? jA : 0, 0);
        // carried own-point values: h(k) (x, y, z) and e'(k) (x, y, z) of the previous plane
        T hxk = T(0), hyk = T(0), hzk = T(0), ek0 = T(0), ek1 = T(0), ek2 = T(0);
        T g0 = bH0, g1 = bH1, g2 = bH2;                    // cH at the own point, plane k (HA)
        if (tid == 0)
            for (int p = pre_cur; p < min(S, nplanes); ++p) {
                const uint32_t L = lcount + p;
                issue_plane<T, EM, HA, G>(stages + (L % S) * SL::SZ, &bars[L % S], &tm_state, &tm_cE,
                                          &tm_cH, x0, y0, kb - 1 + p);
            }
        for (int p = 0; p + 1 < nplanes; ++p) {
            const int k = kb - 1 + p, kk = k + 1;
            const uint32_t L0 = lcount + p, L1 = L0 + 1;
            if (p == 0) mbar_wait(&bars[L0 % S], (L0 / S) & 1);
            mbar_wait(&bars[L1 % S], (L1 / S) & 1);
            const T *P0 = stages + (L0 % S) * SL::SZ;
            const T *P1 = stages + (L1 % S) * SL::SZ;
            T *R1 = ring + (kk & 1) * 3 * G::RP;
            const T *R0 = ring + (k & 1) * 3 * G::RP;
            if (EM == 1) {
                bE0 = zt[p + 1];
                bE1 = zt[ZT_ROW + p + 1];
                bE2 = zt[2 * ZT_ROW + p + 1];
            }
            if (p == 0 && hasA) {                         // h(kb-1) at the own point
                hxk = P0[3 * G::PL + sA];
                hyk = P0[4 * G::PL + sA];
            }
            T e0 = T(0), e1 = T(0), e2 = T(0), hx1 = T(0), hy1 = T(0), hz1 = T(0);
            // ---- phase A: e'(k+1) on the tile and its +1 halo ----
            if (hasA) {
                const T *hx = P1 + 3 * G::PL, *hy = P1 + 4 * G::PL, *hz = P1 + 5 * G::PL;
                hx1 = hx[sA];
                hy1 = hy[sA];
                hz1 = hz[sA];
                const T hz_jm = hz[sA - G::WX], hx_jm = hx[sA - G::WX];
                const T hz_im = hz[sA - 1], hy_im = hy[sA - 1];
                const T c0 = ((hz1 - hz_jm) - hy1) + hyk;
                const T c1 = ((hx1 - hxk) - hz1) + hz_im;
                const T c2 = ((hy1 - hy_im) - hx1) + hx_jm;
                const bool vk = kk < D.nz, kp = kk > 0;
                T w0 = bE0, w1 = bE1, w2 = bE2;
                if (EM == 2) {
                    w0 = P1[SL::ST + sA] * cf.sig;
                    w1 = P1[SL::ST + G::PL + sA] * cf.sig;
                    w2 = P1[SL::ST + 2 * G::PL + sA] * cf.sig;
                }
                e0 = (lxA && vk && kp) ? P1[sA] + w0 * c0 : T(0);
                e1 = (lyA && vk && kp) ? P1[G::PL + sA] + w1 * c1 : T(0);
                e2 = (lzA && vk) ? P1[2 * G::PL + sA] + w2 * c2 : T(0);
                if (smask && vk)
                    for (int r = 0; r < src.n; ++r)
                        if (((smask >> r) & 1u) && src.k[r] == kk) {
                            const int sc = src.c[r];
                            const T qv = q[r];
                            if (sc == 0) e0 = e0 - qv;
                            if (sc == 1) e1 = e1 - qv;
                            if (sc == 2) e2 = e2 - qv;
                        }
                PE_CHECK(rA >= 0 && rA < G::RP && sA >= G::WX && sA + 1 < G::PL, "K1r ring / stage index");
                R1[rA] = e0;
                R1[G::RP + rA] = e1;
                R1[2 * G::RP + rA] = e2;
                if (wrA && vk && kk >= kb && kk < ke) {
                    T *o = oA + (int64_t)kk * D.plane;
                    PE_CHECK(D.in_state((o - out) + 2 * D.cs), "K1r e store");
                    o[0] = e0;
                    o[D.cs] = e1;
                    o[2 * D.cs] = e2;
                    if (TR) {
                        if (w0 != T(0)) eacc += (double)e0 * (double)e0 / (double)w0;
                        if (w1 != T(0)) eacc += (double)e1 * (double)e1 / (double)w1;
                        if (w2 != T(0)) eacc += (double)e2 * (double)e2 / (double)w2;
                        if (pmask)
                            for (int r = 0; r < tr.np; ++r)
                                if (((pmask >> r) & 1u) && tr.k[r] == kk)
                                    tr.probe[r] = (double)(tr.c[r] == 0 ? e0 : (tr.c[r] == 1 ? e1 : e2));
                    }
                }
            }
            __syncthreads();
            // ---- phase B: h'(k) on the tile (own e'(k), e'(k+1), h(k) from registers) ----
            if (k >= kb && wrA) {
                const T ez_jp = R0[2 * G::RP + rA + G::EX], ex_jp = R0[rA + G::EX];
                const T ez_ip = R0[2 * G::RP + rA + 1], ey_ip = R0[G::RP + rA + 1];
                const T c0 = ((ek1 + ez_jp) - e1) - ek2;
                const T c1 = ((ek2 + e0) - ez_ip) - ek0;
                const T c2 = ((ek0 + ey_ip) - ex_jp) - ek1;
                if (HA) {
                    const int ch = SL::ST + SL::CE;
                    g0 = P0[ch + sA] * cf.sig;
                    g1 = P0[ch + G::PL + sA] * cf.sig;
                    g2 = P0[ch + 2 * G::PL + sA] * cf.sig;
                }
                const bool lxB = iA > 0, lyB = jA > 0;
                const T n0 = lxB ? hxk - g0 * c0 : hxk;
                const T n1 = lyB ? hyk - g1 * c1 : hyk;
                const T n2 = k > 0 ? hzk - g2 * c2 : hzk;
                T *o = oA + (int64_t)k * D.plane + 3 * D.cs;
                PE_CHECK(D.in_state((o - out) + 2 * D.cs) && iA < D.nx, "K1r h store");
                o[0] = n0;
                o[D.cs] = n1;
                o[2 * D.cs] = n2;
                if (TR) {
                    if (lxB && g0 != T(0)) eacc += (double)hxk * (double)n0 / (double)g0;
                    if (lyB && g1 != T(0)) eacc += (double)hyk * (double)n1 / (double)g1;
                    if (k > 0 && g2 != T(0)) eacc += (double)hzk * (double)n2 / (double)g2;
                }
            }
            // carry plane k+1 -> k
            hxk = hx1;
            hyk = hy1;
            hzk = hz1;
            ek0 = e0;
            ek1 = e1;
            ek2 = e2;
            __syncthreads();
            if (tid == 0) {
                const uint32_t L = lcount + p + S;
                if (p + S < nplanes) {
                    const int kz = kb - 1 + p + S;
                    issue_plane<T, EM, HA, G>(stages + (L % S) * SL::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                                x0, y0, kz);
                } else {
                    if (p + S == nplanes) {                   // the slots start to free: next unit
                        nxt = grab_next_t0(sch, unit);
                        s_next = nxt;
                        if (nxt < sch.units) {
                            const int nt = nxt % sch.ntiles, nc = nxt / sch.ntiles;
                            nx0 = (nt % sch.tiles_x) * BX;
                            ny0 = (nt / sch.tiles_x) * BY;
                            nkb = nc * sch.chunk;
                            nke = min(nkb + sch.chunk, D.nz);
                        }
                    }
                    const int q = p + S - nplanes;            // plane q of the next unit
                    if (sch.lookahead && nxt < sch.units && q < nke - nkb + 2) {
                        const int kz = nkb - 1 + q;
                        issue_plane<T, EM, HA, G>(stages + (L % S) * SL::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                                    nx0, ny0, kz);
                        pre = q + 1;
                    }
                }
            }
        }
        lcount += nplanes;
        if (S == 2) __syncthreads();                          // s_next written in the last iteration
        unit = s_next;
    }
    if (TR && tr.energy) {
        const double sum = block_sum(eacc);
        if (tid == 0 && sum != 0.0) atomicAdd(tr.energy, sum * tr.dt);
    }
}

// ---------------------------------------------------------------------------------------
// K1v: fp32 leapfrog step, two x-adjacent points per thread (float2 shared/global accesses)
// ---------------------------------------------------------------------------------------
// fp32 moves half the bytes of fp64 through the same per-point instruction stream, so K1r
// is issue/latency-bound there.  K1v is K1r with a 64 x 8 tile and each thread owning the
// pair (i, i+1): own values, j-neighbours and stores are float2; the i-1 neighbour of the
// left point is one scalar load and the i-1 neighbour of the right point is the left own
// value (phase A), the i+1 neighbour of the left point is the right own value (phase B).
// Phase-A points: 32 pair-threads per row for rows y0 .. y0+BY (the +1 halo row) and one
// single-point thread per row for the +1 halo column x0+64.  Ring rows have an even pitch so
// float2 accesses stay 8-byte aligned.
template <int BY>
struct GeoV {
    static constexpr int BX = 64;                          // points per tile row
    static constexpr int OX = 4;                           // TMA x start = x0 - 4 (16 B aligned)
    static constexpr int WX = 72;                          // box width (>= OX + BX + 1, 16 B multiple)
    static constexpr int HY = BY + 2;
    static constexpr int PL = WX * HY;
    static constexpr int EY = BY + 1;
    static constexpr int RX = 66;                          // ring row pitch (>= 65, even)
    static constexpr int RP = RX * EY;
    static constexpr int MAIN = 32 * EY;                   // pair threads (tile + halo row)
    static constexpr int NA = MAIN + EY;                   // + halo-column threads
    static constexpr int NTHR = ((NA + 31) / 32) * 32;
    static constexpr int NT = 32 * BY;                     // phase-B pair threads
};

template <int EM, bool HA, int BY, int S, bool TR>
__global__ void __launch_bounds__(GeoV<BY>::NTHR, 3) leapfrog_v_kernel(
    const __grid_constant__ CUtensorMap tm_state, const __grid_constant__ CUtensorMap tm_cE,
    const __grid_constant__ CUtensorMap tm_cH, Dev<float> D, Coef<float, EM, HA> cf, float *__restrict__ out,
    Sched sch, SrcList src, const float *__restrict__ q, const __grid_constant__ TraceDev tr) {
    pdl_sync();
    using G = GeoV<BY>;
    using SL = StageL<float, EM, HA, G>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *stages = reinterpret_cast<float *>(smem_raw);
    float *ring = stages + S * SL::SZ;                     // [2][3][RP]
    float *zt = ring + 2 * 3 * G::RP;                      // [3][ZT_ROW] z-table (EM == 1)
    uint64_t *bars = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(zt + ZtL<float, EM>::N) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x;
    const bool hasA = tid < G::NA;
    const bool pair = tid < G::MAIN;
    const int ii = pair ? 2 * (tid % 32) : G::BX;          // local x of the (left) point
    const int jj = pair ? tid / 32 : tid - G::MAIN;
    const int rA = jj * G::RX + ii;
    const int sA = (jj + 1) * G::WX + ii + G::OX;
    const bool tileA = pair && jj < BY;                    // == phase-B thread of the same pair
    float bE0 = cf.cEs[0] * cf.sig, bE1 = cf.cEs[1] * cf.sig, bE2 = cf.cEs[2] * cf.sig;
    const float bH0 = cf.cHs[0] * cf.sig, bH1 = cf.cHs[1] * cf.sig, bH2 = cf.cHs[2] * cf.sig;
    if (tid == 0) {
        for (int s2 = 0; s2 < S; ++s2) mbar_init(&bars[s2], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto ld2 = [](const float *p) { return *reinterpret_cast<const float2 *>(p); };
    auto st2 = [](float *p, float a, float b) { *reinterpret_cast<float2 *>(p) = make_float2(a, b); };
    uint32_t lcount = 0;
    double eacc = 0.0;
    // cross-unit pipelining (as in K2): thread 0 issues the next unit's first planes into the
    // stage slots the draining unit frees
    __shared__ int s_next;
    int pre = 0;
    int unit = grab_unit(sch, -1);
    while (unit < sch.units) {
        const int tile = unit % sch.ntiles, chunk = unit / sch.ntiles;
        const int x0 = (tile % sch.tiles_x) * G::BX, y0 = (tile / sch.tiles_x) * BY;
        const int kb = chunk * sch.chunk, ke = min(kb + sch.chunk, D.nz);
        const int nplanes = ke - kb + 2;
        const int pre_cur = pre;
        pre = 0;
        int nxt = 0x7fffffff, nx0 = 0, ny0 = 0, nkb = 0, nke = 0;
        stage_ztab<float, EM, HA>(zt, cf, kb, nplanes, D.nz);
        const int ia = x0 + ii, jA = y0 + jj, ib = ia + 1;
        const bool rowA = hasA && jA < D.ny;
        const bool inA = rowA && ia < D.nx, inB = pair && rowA && ib < D.nx;
        // liveness (reading 5): e_x: j>0 (k>0); e_y: i>0 (k>0); e_z: i>0 && j>0
        const bool lxa = inA && jA > 0, lya = inA && ia > 0, lza = inA && ia > 0 && jA > 0;
        const bool lxb = inB && jA > 0, lyb = inB, lzb = inB && jA > 0;
        const bool wrA = inA && tileA;
        uint32_t sma = 0, smb = 0, pma = 0, pmb = 0;
        for (int r = 0; r < src.n; ++r) {
            if (inA && src.i[r] == ia && src.j[r] == jA) sma |= 1u << r;
            if (inB && src.i[r] == ib && src.j[r] == jA) smb |= 1u << r;
        }
        if (TR)
            for (int r = 0; r < tr.np; ++r) {
                if (wrA && tr.i[r] == ia && tr.j[r] == jA) pma |= 1u << r;
                if (wrA && inB && tr.i[r] == ib && tr.j[r] == jA) pmb |= 1u << r;
            }
        float *oA = out + D.idx(wrA ? ia : 0, wrA ? jA : 0, 0);
        // carried own values of plane k: h (x, y, z) and e' (x, y, z), left (a) and right (b)
        float hxa = 0.f, hxb = 0.f, hya = 0.f, hyb = 0.f, hza = 0.f, hzb = 0.f;
        float ea0 = 0.f, eb0 = 0.f, ea1 = 0.f, eb1 = 0.f, ea2 = 0.f, eb2 = 0.f;
        float g0a = bH0, g1a = bH1, g2a = bH2, g0b = bH0, g1b = bH1, g2b = bH2;
        if (tid == 0)
            for (int p = pre_cur; p < min(S, nplanes); ++p) {
                const uint32_t L = lcount + p;
                issue_plane<float, EM, HA, G>(stages + (L % S) * SL::SZ, &bars[L % S], &tm_state, &tm_cE,
                                              &tm_cH, x0, y0, kb - 1 + p);
            }
        for (int p = 0; p + 1 < nplanes; ++p) {
            const int k = kb - 1 + p, kk = k + 1;
            const uint32_t L0 = lcount + p, L1 = L0 + 1;
            if (p == 0) mbar_wait(&bars[L0 % S], (L0 / S) & 1);
            mbar_wait(&bars[L1 % S], (L1 / S) & 1);
            const float *P0 = stages + (L0 % S) * SL::SZ;
            const float *P1 = stages + (L1 % S) * SL::SZ;
            float *R1 = ring + (kk & 1) * 3 * G::RP;
            const float *R0 = ring + (k & 1) * 3 * G::RP;
            if (EM == 1) {
                bE0 = zt[p + 1];
                bE1 = zt[ZT_ROW + p + 1];
                bE2 = zt[2 * ZT_ROW + p + 1];
            }
            if (p == 0 && hasA) {                           // h(kb-1) at the own points
                if (pair) {
                    const float2 x = ld2(P0 + 3 * G::PL + sA), y = ld2(P0 + 4 * G::PL + sA);
                    hxa = x.x; hxb = x.y; hya = y.x; hyb = y.y;
                } else {
                    hxa = P0[3 * G::PL + sA];
                    hya = P0[4 * G::PL + sA];
                }
            }
            float na0 = 0.f, nb0 = 0.f, na1 = 0.f, nb1 = 0.f, na2 = 0.f, nb2 = 0.f;   // e'(k+1)
            float h1xa = 0.f, h1xb = 0.f, h1ya = 0.f, h1yb = 0.f, h1za = 0.f, h1zb = 0.f;
            // ---- phase A: e'(k+1) ----
            if (hasA) {
                const float *hx = P1 + 3 * G::PL, *hy = P1 + 4 * G::PL, *hz = P1 + 5 * G::PL;
                const bool vk = kk < D.nz, kp = kk > 0;
                float wa0 = bE0, wa1 = bE1, wa2 = bE2, wb0 = bE0, wb1 = bE1, wb2 = bE2;
                if (pair) {
                    const float2 X = ld2(hx + sA), Y = ld2(hy + sA), Z = ld2(hz + sA);
                    const float2 Zjm = ld2(hz + sA - G::WX), Xjm = ld2(hx + sA - G::WX);
                    const float zim = hz[sA - 1], yim = hy[sA - 1];
                    h1xa = X.x; h1xb = X.y; h1ya = Y.x; h1yb = Y.y; h1za = Z.x; h1zb = Z.y;
                    const float c0a = ((Z.x - Zjm.x) - Y.x) + hya, c0b = ((Z.y - Zjm.y) - Y.y) + hyb;
                    const float c1a = ((X.x - hxa) - Z.x) + zim, c1b = ((X.y - hxb) - Z.y) + Z.x;
                    const float c2a = ((Y.x - yim) - X.x) + Xjm.x, c2b = ((Y.y - Y.x) - X.y) + Xjm.y;
                    if (EM == 2) {
                        const float2 A0 = ld2(P1 + SL::ST + sA), A1 = ld2(P1 + SL::ST + G::PL + sA);
                        const float2 A2 = ld2(P1 + SL::ST + 2 * G::PL + sA);
                        wa0 = A0.x * cf.sig; wb0 = A0.y * cf.sig;
                        wa1 = A1.x * cf.sig; wb1 = A1.y * cf.sig;
                        wa2 = A2.x * cf.sig; wb2 = A2.y * cf.sig;
                    }
                    const float2 E0 = ld2(P1 + sA), E1 = ld2(P1 + G::PL + sA), E2 = ld2(P1 + 2 * G::PL + sA);
                    na0 = (lxa && vk && kp) ? E0.x + wa0 * c0a : 0.f;
                    nb0 = (lxb && vk && kp) ? E0.y + wb0 * c0b : 0.f;
                    na1 = (lya && vk && kp) ? E1.x + wa1 * c1a : 0.f;
                    nb1 = (lyb && vk && kp) ? E1.y + wb1 * c1b : 0.f;
                    na2 = (lza && vk) ? E2.x + wa2 * c2a : 0.f;
                    nb2 = (lzb && vk) ? E2.y + wb2 * c2b : 0.f;
                } else {
                    const float X = hx[sA], Y = hy[sA], Z = hz[sA];
                    h1xa = X; h1ya = Y; h1za = Z;
                    const float c0 = ((Z - hz[sA - G::WX]) - Y) + hya;
                    const float c1 = ((X - hxa) - Z) + hz[sA - 1];
                    const float c2 = ((Y - hy[sA - 1]) - X) + hx[sA - G::WX];
                    if (EM == 2) {
                        wa0 = P1[SL::ST + sA] * cf.sig;
                        wa1 = P1[SL::ST + G::PL + sA] * cf.sig;
                        wa2 = P1[SL::ST + 2 * G::PL + sA] * cf.sig;
                    }
                    na0 = (lxa && vk && kp) ? P1[sA] + wa0 * c0 : 0.f;
                    na1 = (lya && vk && kp) ? P1[G::PL + sA] + wa1 * c1 : 0.f;
                    na2 = (lza && vk) ? P1[2 * G::PL + sA] + wa2 * c2 : 0.f;
                }
                if ((sma | smb) && vk)
                    for (int r = 0; r < src.n; ++r) {
                        if (src.k[r] != kk) continue;
                        const int sc = src.c[r];
                        const float qv = q[r];
                        if ((sma >> r) & 1u) {
                            if (sc == 0) na0 -= qv;
                            if (sc == 1) na1 -= qv;
                            if (sc == 2) na2 -= qv;
                        }
                        if ((smb >> r) & 1u) {
                            if (sc == 0) nb0 -= qv;
                            if (sc == 1) nb1 -= qv;
                            if (sc == 2) nb2 -= qv;
                        }
                    }
                if (pair) {
                    st2(R1 + rA, na0, nb0);
                    st2(R1 + G::RP + rA, na1, nb1);
                    st2(R1 + 2 * G::RP + rA, na2, nb2);
                } else {
                    R1[rA] = na0;
                    R1[G::RP + rA] = na1;
                    R1[2 * G::RP + rA] = na2;
                }
                if (wrA && vk && kk >= kb && kk < ke) {
                    float *o = oA + (int64_t)kk * D.plane;
                    PE_CHECK(D.in_state((o - out) + 2 * D.cs + 1) && ((o - out) & 1) == 0, "K1v e store");
                    st2(o, na0, nb0);                     // b beyond nx lands in the zero x-padding
                    st2(o + D.cs, na1, nb1);
                    st2(o + 2 * D.cs, na2, nb2);
                    if (TR) {
                        if (wa0 != 0.f) eacc += (double)na0 * na0 / (double)wa0;
                        if (wa1 != 0.f) eacc += (double)na1 * na1 / (double)wa1;
                        if (wa2 != 0.f) eacc += (double)na2 * na2 / (double)wa2;
                        if (inB) {
                            if (wb0 != 0.f) eacc += (double)nb0 * nb0 / (double)wb0;
                            if (wb1 != 0.f) eacc += (double)nb1 * nb1 / (double)wb1;
                            if (wb2 != 0.f) eacc += (double)nb2 * nb2 / (double)wb2;
                        }
                        if (pma | pmb)
                            for (int r = 0; r < tr.np; ++r) {
                                if (tr.k[r] != kk) continue;
                                const int c = tr.c[r];
                                if ((pma >> r) & 1u) tr.probe[r] = (double)(c == 0 ? na0 : (c == 1 ? na1 : na2));
                                if ((pmb >> r) & 1u) tr.probe[r] = (double)(c == 0 ? nb0 : (c == 1 ? nb1 : nb2));
                            }
                    }
                }
            }
            __syncthreads();
            // ---- phase B: h'(k) on the tile pair ----
            if (k >= kb && wrA) {
                const float2 Zj = ld2(R0 + 2 * G::RP + rA + G::RX), Xj = ld2(R0 + rA + G::RX);
                const float zip = R0[2 * G::RP + rA + 2], yip = R0[G::RP + rA + 2];
                // point a: i+1 neighbours are the own right values; point b: from the ring
                const float c0a = ((ea1 + Zj.x) - na1) - ea2, c0b = ((eb1 + Zj.y) - nb1) - eb2;
                const float c1a = ((ea2 + na0) - eb2) - ea0, c1b = ((eb2 + nb0) - zip) - eb0;
                const float c2a = ((ea0 + eb1) - Xj.x) - ea1, c2b = ((eb0 + yip) - Xj.y) - eb1;
                if (HA) {
                    const int ch = SL::ST + SL::CE;
                    const float2 A0 = ld2(P0 + ch + sA), A1 = ld2(P0 + ch + G::PL + sA), A2 = ld2(P0 + ch + 2 * G::PL + sA);
                    g0a = A0.x * cf.sig; g0b = A0.y * cf.sig;
                    g1a = A1.x * cf.sig; g1b = A1.y * cf.sig;
                    g2a = A2.x * cf.sig; g2b = A2.y * cf.sig;
                }
                const bool lxA2 = ia > 0, lyA2 = jA > 0, kp = k > 0;
                const float nxa = lxA2 ? hxa - g0a * c0a : hxa, nxb = hxb - g0b * c0b;
                const float nya = lyA2 ? hya - g1a * c1a : hya, nyb = lyA2 ? hyb - g1b * c1b : hyb;
                const float nza = kp ? hza - g2a * c2a : hza, nzb = kp ? hzb - g2b * c2b : hzb;
                float *o = oA + (int64_t)k * D.plane + 3 * D.cs;
                PE_CHECK(D.in_state((o - out) + 2 * D.cs + 1), "K1v h store");
                st2(o, nxa, inB ? nxb : 0.f);
                st2(o + D.cs, nya, inB ? nyb : 0.f);
                st2(o + 2 * D.cs, nza, inB ? nzb : 0.f);
                if (TR) {
                    if (lxA2 && g0a != 0.f) eacc += (double)hxa * nxa / (double)g0a;
                    if (lyA2 && g1a != 0.f) eacc += (double)hya * nya / (double)g1a;
                    if (kp && g2a != 0.f) eacc += (double)hza * nza / (double)g2a;
                    if (inB) {
                        if (g0b != 0.f) eacc += (double)hxb * nxb / (double)g0b;
                        if (lyA2 && g1b != 0.f) eacc += (double)hyb * nyb / (double)g1b;
                        if (kp && g2b != 0.f) eacc += (double)hzb * nzb / (double)g2b;
                    }
                }
            }
            hxa = h1xa; hxb = h1xb; hya = h1ya; hyb = h1yb; hza = h1za; hzb = h1zb;
            ea0 = na0; eb0 = nb0; ea1 = na1; eb1 = nb1; ea2 = na2; eb2 = nb2;
            __syncthreads();
            if (tid == 0) {
                const uint32_t L = lcount + p + S;
                if (p + S < nplanes) {
                    const int kz = kb - 1 + p + S;
                    issue_plane<float, EM, HA, G>(stages + (L % S) * SL::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                                x0, y0, kz);
                } else {
                    if (p + S == nplanes) {                   // the slots start to free: next unit
                        nxt = grab_next_t0(sch, unit);
                        s_next = nxt;
                        if (nxt < sch.units) {
                            const int nt = nxt % sch.ntiles, nc = nxt / sch.ntiles;
                            nx0 = (nt % sch.tiles_x) * G::BX;
                            ny0 = (nt / sch.tiles_x) * BY;
                            nkb = nc * sch.chunk;
                            nke = min(nkb + sch.chunk, D.nz);
                        }
                    }
                    const int q = p + S - nplanes;            // plane q of the next unit
                    if (sch.lookahead && nxt < sch.units && q < nke - nkb + 2) {
                        const int kz = nkb - 1 + q;
                        issue_plane<float, EM, HA, G>(stages + (L % S) * SL::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                                    nx0, ny0, kz);
                        pre = q + 1;
                    }
                }
            }
        }
        lcount += nplanes;
        if (S == 2) __syncthreads();                          // s_next written in the last iteration
        unit = s_next;
    }
    if (TR && tr.energy) {
        const double sum = block_sum(eacc);
        if (tid == 0 && sum != 0.0) atomicAdd(tr.energy, sum * tr.dt);
    }
}

// K2 stage: the w box of StageL plus the y tile (6 x BY x BX, no halo) of the same plane, so
// that the Newton sum y(k) arrives by TMA with w(k), S - 1 planes ahead of its use.  (Loaded
// by the threads themselves, y(k) was on the critical path: ncu put 23% of K2's warp-stall
// samples on the first use of y, and 28% on the barrier that waited for those warps.)
// Only for the scalar / z-table materials: with per-edge coefficient boxes in the stage as well
// (EM == 2, HA) the y tile would cost the second resident CTA per SM, so there the threads keep
// loading y(k) themselves at the top of the plane iteration.
template <typename T, int EM, bool HA, typename G>
struct StageP {
    static constexpr bool Y = EM != 2 && !HA;               // y staged by TMA
    static constexpr int YOFF = StageL<T, EM, HA, G>::SZ;
    static constexpr int YT = Y ? 6 * G::BX * G::BY : 0;    // multiple of 128 B for 32 x 8 / 64 x 8 tiles
    static constexpr int SZ = YOFF + YT;
};
template <typename T, int EM, bool HA, typename G>
__device__ __forceinline__ void issue_plane_y(T *dst, uint64_t *bar, const CUtensorMap *tm_state,
                                              const CUtensorMap *tm_cE, const CUtensorMap *tm_cH,
                                              const CUtensorMap *tm_y, int x0, int y0, int kz, bool with_y) {
    using SL = StageL<T, EM, HA, G>;
    constexpr uint32_t wbytes = (uint32_t)(NComp<T, EM, HA>::value * G::PL * sizeof(T));
    constexpr uint32_t ybytes = (uint32_t)(StageP<T, EM, HA, G>::YT * sizeof(T));
    mbar_expect_tx(bar, wbytes + ((StageP<T, EM, HA, G>::Y && with_y) ? ybytes : 0u));
    tma_load_4d(dst, tm_state, bar, x0 - G::OX, y0 - 1, kz, 0);
    if (EM == 2) tma_load_4d(dst + SL::ST, tm_cE, bar, x0 - G::OX, y0 - 1, kz, 0);
    if (HA) tma_load_4d(dst + SL::ST + SL::CE, tm_cH, bar, x0 - G::OX, y0 - 1, kz, 0);
    if (StageP<T, EM, HA, G>::Y && with_y) tma_load_4d(dst + StageP<T, EM, HA, G>::YOFF, tm_y, bar, x0, y0, kz, 0);
}

// ---------------------------------------------------------------------------------------
// K2: fused Newton pair  u = X w ; y <- (init?0:y) + a w + b u ; [w' = X u + e2 w]
// ---------------------------------------------------------------------------------------
// Phase A of iteration k: u_e(k+1) on the +1 halo and u_h(k) on the -1 halo; phase B: the
// tile's w'(k) and y(k).  Ring depth 2 (two barriers per plane).
// min 2 CTAs/SM: the measured K2 rate depends on two resident CTAs per SM (a register
// growth to > 102 per thread halves the occupancy: 376 vs 288 us per A-application)
template <typename T, int EM, bool HA, int BX, int BY, int S>
__global__ void __launch_bounds__(Geo<T, BX, BY>::NTHR, sizeof(T) == 8 ? 2 : 3) pair_fused_kernel(
    const __grid_constant__ CUtensorMap tm_state, const __grid_constant__ CUtensorMap tm_cE,
    const __grid_constant__ CUtensorMap tm_cH, const __grid_constant__ CUtensorMap tm_y, Dev<T> D,
    Coef<T, EM, HA> cf, T *__restrict__ wout, T *__restrict__ y, Sched sch, T a, T b, T e2, T cl, int init,
    int mode, EtDev et) {
    pdl_sync();
    using G = Geo<T, BX, BY>;
    if (et.norms && et_skip(et)) {                        // early termination (f2)
        // a skipped launch still advances the dynamic-schedule counter by units + gridDim,
        // the amount the host's shadow base assumed
        if (sch.ctr && blockIdx.x == 0 && threadIdx.x == 0)
            atomicAdd(sch.ctr, (unsigned long long)sch.units + gridDim.x);
        return;
    }
    double dacc = 0.0, yacc = 0.0;                        // ||delta y||^2, ||y||^2 (energy norm)
    using SP = StageP<T, EM, HA, G>;
    using SL = StageL<T, EM, HA, G>;
    constexpr int NR = 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *stages = reinterpret_cast<T *>(smem_raw);
    T *UE = stages + S * SP::SZ;                         // [NR][3][EY][EX]: u_e at (ii, jj)
    T *UH = UE + NR * 3 * G::RP;                         // [3][EY][EX]: u_h(k) at (ii-1, jj-1), one plane
    T *zt = UH + 3 * G::RP;                              // [3][ZT_ROW] z-table (EM == 1)
    uint64_t *bars = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(zt + ZtL<T, EM>::N) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x;
    const bool hasA = tid < G::RP;
    // row-aligned phase-A mapping: warps cover whole 32-wide rows, the +1 halo column last
    constexpr int MAIN = BX * G::EY;
    const int ii = tid < MAIN ? tid % BX : BX, jj = tid < MAIN ? tid / BX : tid - MAIN;
    const int rA = jj * G::EX + ii;                       // ring index of the phase-A point
    const int sE = (jj + 1) * G::WX + ii + G::OX;         // stage index of the u_e point
    const int sH = jj * G::WX + ii - 1 + G::OX;           // stage index of the u_h point
    const bool hasB = tid < G::NT;
    const int tx = tid % BX, ty = tid / BX;
    const int re = ty * G::EX + tx;                       // u_e ring index of the own point
    const int rh = (ty + 1) * G::EX + (tx + 1);           // u_h ring index of the own point
    const int sB = (ty + 1) * G::WX + tx + G::OX;         // stage index of the own point
    T bE0 = cf.cEs[0] * cf.sig, bE1 = cf.cEs[1] * cf.sig, bE2 = cf.cEs[2] * cf.sig;
    const T bH0 = cf.cHs[0] * cf.sig, bH1 = cf.cHs[1] * cf.sig, bH2 = cf.cHs[2] * cf.sig;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint32_t lcount = 0;
    // cross-unit pipelining: while a unit drains (its last S - 1 plane iterations issue no
    // refills), thread 0 grabs the next unit and issues that unit's first planes into the
    // freed stage slots, so the next unit starts on planes already in flight
    __shared__ int s_next;
    int pre = 0;                                          // (thread 0) planes of `unit` already issued
    int unit = grab_unit(sch, -1);
    while (unit < sch.units) {
        const int tile = unit % sch.ntiles, chunk = unit / sch.ntiles;
        const int x0 = (tile % sch.tiles_x) * BX, y0 = (tile / sch.tiles_x) * BY;
        const int kb = chunk * sch.chunk, ke = min(kb + sch.chunk, D.nz);
        const int nplanes = ke - kb + 2;
        const int pre_cur = pre;
        pre = 0;
        int nxt = 0x7fffffff, nx0 = 0, ny0 = 0, nkb = 0, nke = 0;   // (thread 0) the next unit
        stage_ztab<T, EM, HA>(zt, cf, kb, nplanes, D.nz);
        // phase-A validity (k-independent parts)
        const int iE = x0 + ii, jE = y0 + jj;             // u_e point
        const bool inE = hasA && iE < D.nx && jE < D.ny;
        const bool lxE = inE && jE > 0, lyE = inE && iE > 0, lzE = inE && iE > 0 && jE > 0;
        const int iH = iE - 1, jH = jE - 1;               // u_h point
        const bool inH = hasA && iH >= 0 && jH >= 0 && iH < D.nx && jH < D.ny;
        const bool lxH = inH && iH > 0, lyH = inH && jH > 0;
        // own point
        const int iB = x0 + tx, jB = y0 + ty;
        const bool inB = hasB && iB < D.nx && jB < D.ny;
        const bool lxBe = jB > 0, lyBe = iB > 0, lzBe = iB > 0 && jB > 0;
        const bool lxBh = iB > 0, lyBh = jB > 0;
        const int64_t gB = D.idx(inB ? iB : 0, inB ? jB : 0, 0);
        // own-point u_h(k-1) (x, y) carried from the previous plane (the u_h ring holds one plane)
        T hxm = T(0), hym = T(0);
        if (tid == 0)
            for (int p = pre_cur; p < min(S, nplanes); ++p) {
                const uint32_t L = lcount + p, kz = kb - 1 + p;
                issue_plane_y<T, EM, HA, G>(stages + (L % S) * SP::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                            &tm_y, x0, y0, kz, !init && kz >= kb && kz < ke);
            }
        for (int p = 0; p + 1 < nplanes; ++p) {
            const int k = kb - 1 + p, kk = k + 1;
            const uint32_t L0 = lcount + p, L1 = L0 + 1;
            const bool doB = k >= kb && inB;
            // y(k) of the own point: staged by TMA (SP::Y), else loaded here, consumed in phase B
            T yv0 = T(0), yv1 = T(0), yv2 = T(0), yv3 = T(0), yv4 = T(0), yv5 = T(0);
            if (!SP::Y && doB && !init) {
                const T *yp = y + gB + (int64_t)k * D.plane;
                yv0 = yp[0];
                yv1 = yp[D.cs];
                yv2 = yp[2 * D.cs];
                yv3 = yp[3 * D.cs];
                yv4 = yp[4 * D.cs];
                yv5 = yp[5 * D.cs];
            }
            if (p == 0) mbar_wait(&bars[L0 % S], (L0 / S) & 1);
            mbar_wait(&bars[L1 % S], (L1 / S) & 1);
            const T *P0 = stages + (L0 % S) * SP::SZ;    // w plane k (+ y(k))
            const T *P1 = stages + (L1 % S) * SP::SZ;    // w plane k+1
            T *UE1 = UE + (kk % NR) * 3 * G::RP;           // u_e(k+1)
            T *UH0 = UH;                                   // u_h(k)
            T bEk0 = bE0, bEk1 = bE1, bEk2 = bE2;         // coefficients at plane k (phase B)
            if (EM == 1) {
                bE0 = zt[p + 1];
                bE1 = zt[ZT_ROW + p + 1];
                bE2 = zt[2 * ZT_ROW + p + 1];
                bEk0 = zt[p];
                bEk1 = zt[ZT_ROW + p];
                bEk2 = zt[2 * ZT_ROW + p];
            }
            if (hasA) {
                // u_e(k+1) = bE .* C^T w_h
                {
                    T c0, c1, c2;
                    curlT_stage<T, G>(P1, P0, sE, c0, c1, c2);
                    const bool vk = kk < D.nz, kp = kk > 0;
                    T u0, u1, u2;
                    if (EM == 2) {
                        u0 = (lxE && vk && kp) ? (P1[SL::ST + sE] * cf.sig) * c0 : T(0);
                        u1 = (lyE && vk && kp) ? (P1[SL::ST + G::PL + sE] * cf.sig) * c1 : T(0);
                        u2 = (lzE && vk) ? (P1[SL::ST + 2 * G::PL + sE] * cf.sig) * c2 : T(0);
                    } else {
                        u0 = (lxE && vk && kp) ? bE0 * c0 : T(0);
                        u1 = (lyE && vk && kp) ? bE1 * c1 : T(0);
                        u2 = (lzE && vk) ? bE2 * c2 : T(0);
                    }
                    PE_CHECK(rA >= 0 && rA < G::RP && sE >= G::WX + 1 && sE < G::PL && sH >= 0 && sH + G::WX + 1 < G::PL,
                             "K2 ring / stage index");
                    UE1[rA] = u0;
                    UE1[G::RP + rA] = u1;
                    UE1[2 * G::RP + rA] = u2;
                }
                // u_h(k) = -bH .* C w_e
                {
                    T c0, c1, c2;
                    curl_stage<T, G>(P0, P1, sH, c0, c1, c2);
                    const bool vk = k >= 0 && k < D.nz;
                    T u0, u1, u2;
                    if (HA) {
                        const int ch = SL::ST + SL::CE;
                        u0 = (lxH && vk) ? -((P0[ch + sH] * cf.sig) * c0) : T(0);
                        u1 = (lyH && vk) ? -((P0[ch + G::PL + sH] * cf.sig) * c1) : T(0);
                        u2 = (inH && vk && k > 0) ? -((P0[ch + 2 * G::PL + sH] * cf.sig) * c2) : T(0);
                    } else {
                        u0 = (lxH && vk) ? -(bH0 * c0) : T(0);
                        u1 = (lyH && vk) ? -(bH1 * c1) : T(0);
                        u2 = (inH && vk && k > 0) ? -(bH2 * c2) : T(0);
                    }
                    UH0[rA] = u0;
                    UH0[G::RP + rA] = u1;
                    UH0[2 * G::RP + rA] = u2;
                }
            }
            __syncthreads();
            T hx0 = T(0), hy0 = T(0);
            if (hasB) {                                          // own u_h(k) (x, y)
                hx0 = UH0[rh];
                hy0 = UH0[G::RP + rh];
            }
            if (doB) {
                const T *UE0 = UE + (k % NR) * 3 * G::RP;        // u_e(k)
                const T ux0 = UE0[re], uy0 = UE0[G::RP + re], uz0 = UE0[2 * G::RP + re];
                const T hz0 = UH0[2 * G::RP + rh];
                if (SP::Y && !init) {      // y(k) at the own point, staged with w(k) by TMA
                    const T *YS = P0 + SP::YOFF;
                    yv0 = YS[tid];
                    yv1 = YS[G::NT + tid];
                    yv2 = YS[2 * G::NT + tid];
                    yv3 = YS[3 * G::NT + tid];
                    yv4 = YS[4 * G::NT + tid];
                    yv5 = YS[5 * G::NT + tid];
                }
                const T w0 = P0[sB], w1 = P0[G::PL + sB], w2 = P0[2 * G::PL + sB];
                const T w3 = P0[3 * G::PL + sB], w4 = P0[4 * G::PL + sB], w5 = P0[5 * G::PL + sB];
                const int64_t go = gB + (int64_t)k * D.plane;
                T wn0 = T(0), wn1 = T(0), wn2 = T(0), wn3 = T(0), wn4 = T(0), wn5 = T(0);
                if (mode != 1) {
                    // w'_h(k) = -bH C u_e + e2 w_h
                    const T uz_jp = UE0[2 * G::RP + re + G::EX], ux_jp = UE0[re + G::EX];
                    const T uz_ip = UE0[2 * G::RP + re + 1], uy_ip = UE0[G::RP + re + 1];
                    const T ux_kp = UE1[re], uy_kp = UE1[G::RP + re];
                    const T c0 = ((uy0 + uz_jp) - uy_kp) - uz0;
                    const T c1 = ((uz0 + ux_kp) - uz_ip) - ux0;
                    const T c2 = ((ux0 + uy_ip) - ux_jp) - uy0;
                    // w'_e(k) = bE C^T u_h + e2 w_e
                    const T hz_jm = UH0[2 * G::RP + rh - G::EX], hx_jm = UH0[rh - G::EX];
                    const T hz_im = UH0[2 * G::RP + rh - 1], hy_im = UH0[G::RP + rh - 1];
                    const T hy_km = hym, hx_km = hxm;
                    const T d0 = ((hz0 - hz_jm) - hy0) + hy_km;
                    const T d1 = ((hx0 - hx_km) - hz0) + hz_im;
                    const T d2 = ((hy0 - hy_im) - hx0) + hx_jm;
                    T be0 = bEk0, be1 = bEk1, be2 = bEk2, bh0 = bH0, bh1 = bH1, bh2 = bH2;
                    if (EM == 2) {
                        be0 = P0[SL::ST + sB] * cf.sig;
                        be1 = P0[SL::ST + G::PL + sB] * cf.sig;
                        be2 = P0[SL::ST + 2 * G::PL + sB] * cf.sig;
                    }
                    if (HA) {
                        const int ch = SL::ST + SL::CE;
                        bh0 = P0[ch + sB] * cf.sig;
                        bh1 = P0[ch + G::PL + sB] * cf.sig;
                        bh2 = P0[ch + 2 * G::PL + sB] * cf.sig;
                    }
                    const bool kp = k > 0;
                    wn0 = ((lxBe && kp) ? be0 * d0 : T(0)) + e2 * w0;
                    wn1 = ((lyBe && kp) ? be1 * d1 : T(0)) + e2 * w1;
                    wn2 = (lzBe ? be2 * d2 : T(0)) + e2 * w2;
                    wn3 = (lxBh ? -(bh0 * c0) : T(0)) + e2 * w3;
                    wn4 = (lyBh ? -(bh1 * c1) : T(0)) + e2 * w4;
                    wn5 = (kp ? -(bh2 * c2) : T(0)) + e2 * w5;
                    if (mode == 0) {
                        T *wo = wout + go;
                        PE_CHECK(D.in_state(go + 5 * D.cs) && iB < D.nx && jB < D.ny, "K2 w' store");
                        wo[0] = wn0;
                        wo[D.cs] = wn1;
                        wo[2 * D.cs] = wn2;
                        wo[3 * D.cs] = wn3;
                        wo[4 * D.cs] = wn4;
                        wo[5 * D.cs] = wn5;
                    }
                }
                T y0 = (yv0 + a * w0) + b * ux0, y1 = (yv1 + a * w1) + b * uy0;
                T y2 = (yv2 + a * w2) + b * uz0, y3 = (yv3 + a * w3) + b * hx0;
                T y4 = (yv4 + a * w4) + b * hy0, y5 = (yv5 + a * w5) + b * hz0;
                if (mode == 2) {
                    y0 = y0 + cl * wn0;
                    y1 = y1 + cl * wn1;
                    y2 = y2 + cl * wn2;
                    y3 = y3 + cl * wn3;
                    y4 = y4 + cl * wn4;
                    y5 = y5 + cl * wn5;
                }
                if (et.norms) {   // energy weights 1/(cE sigma), 1/(cH sigma) at the own point
                    T g[6] = {bEk0, bEk1, bEk2, bH0, bH1, bH2};
                    if (EM == 2) {
                        g[0] = P0[SL::ST + sB] * cf.sig;
                        g[1] = P0[SL::ST + G::PL + sB] * cf.sig;
                        g[2] = P0[SL::ST + 2 * G::PL + sB] * cf.sig;
                    }
                    if (HA) {
                        const int ch = SL::ST + SL::CE;
                        g[3] = P0[ch + sB] * cf.sig;
                        g[4] = P0[ch + G::PL + sB] * cf.sig;
                        g[5] = P0[ch + 2 * G::PL + sB] * cf.sig;
                    }
                    const T yn[6] = {y0, y1, y2, y3, y4, y5}, yo6[6] = {yv0, yv1, yv2, yv3, yv4, yv5};
#pragma unroll
                    for (int c = 0; c < 6; ++c)
                        if (g[c] != T(0)) {
                            const double d = (double)yn[c] - (double)yo6[c], v = (double)yn[c];
                            dacc += d * d / (double)g[c];
                            yacc += v * v / (double)g[c];
                        }
                }
                T *yo = y + go;
                PE_CHECK(D.in_state(go + 5 * D.cs), "K2 y store");
                yo[0] = y0;
                yo[D.cs] = y1;
                yo[2 * D.cs] = y2;
                yo[3 * D.cs] = y3;
                yo[4 * D.cs] = y4;
                yo[5 * D.cs] = y5;
            }
            hxm = hx0;
            hym = hy0;
            __syncthreads();
            if (tid == 0) {
                const uint32_t L = lcount + p + S;
                if (p + S < nplanes) {
                    const int kz = kb - 1 + p + S;
                    issue_plane_y<T, EM, HA, G>(stages + (L % S) * SP::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                                &tm_y, x0, y0, kz, !init && kz >= kb && kz < ke);
                } else {
                    if (p + S == nplanes) {                   // the slots start to free: next unit
                        nxt = grab_next_t0(sch, unit);
                        s_next = nxt;
                        if (nxt < sch.units) {
                            const int nt = nxt % sch.ntiles, nc = nxt / sch.ntiles;
                            nx0 = (nt % sch.tiles_x) * BX;
                            ny0 = (nt / sch.tiles_x) * BY;
                            nkb = nc * sch.chunk;
                            nke = min(nkb + sch.chunk, D.nz);
                        }
                    }
                    const int q = p + S - nplanes;            // plane q of the next unit
                    if (sch.lookahead && nxt < sch.units && q < nke - nkb + 2) {
                        const int kz = nkb - 1 + q;
                        issue_plane_y<T, EM, HA, G>(stages + (L % S) * SP::SZ, &bars[L % S], &tm_state, &tm_cE,
                                                    &tm_cH, &tm_y, nx0, ny0, kz, !init && kz >= nkb && kz < nke);
                        pre = q + 1;
                    }
                }
            }
        }
        lcount += nplanes;
        if (S == 2) __syncthreads();                          // s_next written in the last iteration
        unit = s_next;
    }
    if (et.norms) {
        const double ds = block_sum(dacc);
        __syncthreads();
        const double ys = block_sum(yacc);
        if (tid == 0) {
            atomicAdd(et.norms + 2 * et.op, ds);
            atomicAdd(et.norms + 2 * et.op + 1, ys);
        }
    }
}

// Tile 64 x 8.  Phase A: thread (pi, jj < BY) computes u_e(k+1) AND u_h(k) on the pair
// (x0+2pi, x0+2pi+1) of row y0+jj -- the same pair whose w'(k), y(k) it updates in phase B, so
// its own w(k), u_e(k), u_e(k+1), u_h(k), u_h(k-1) never leave registers.  The halo rows are
// done by the 32 threads jj = BY (u_e on row y0+BY, u_h on row y0-1) and the halo columns by 9
// single-point threads (u_e on column x0+64, rows y0..y0+BY; u_h on column x0-1, rows
// y0-1..y0+BY-1).  Rings (column c stored at c - x0 + 2, even pitch): u_e 2 planes (rows
// y0..y0+BY), u_h 1 plane (rows y0-1..y0+BY-1, stored at row + 1).  Phase B reads only the
// j+1 / i+2 neighbours of u_e(k) and the j-1 / i-1 neighbours of u_h(k).
// geometry of the two-points-per-thread pair kernel for T = float / double (64 x BY tiles)
template <typename T, int BY_>
struct GeoW {
    static constexpr int BX = 64, BY = BY_;
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int OX = VEC;                          // TMA x start x0 - OX (16 B aligned)
    static constexpr int WX = ((OX + BX + 1 + VEC - 1) / VEC) * VEC;   // covers x0-1 .. x0+64
    static constexpr int HY = BY_ + 2;
    static constexpr int PL = WX * HY;
    static constexpr int NTHR = ((32 * (BY_ + 1) + (BY_ + 1) + 31) / 32) * 32;
};
template <typename T> struct Vec2;
template <> struct Vec2<float> {
    using type = float2;
    static __device__ __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};
template <> struct Vec2<double> {
    using type = double2;
    static __device__ __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};

template <typename T, int EM, bool HA, int BY, int S, bool ET>
__global__ void __launch_bounds__(GeoW<T, BY>::NTHR, sizeof(T) == 8 ? 1 : 2) pair_v_kernel(
    const __grid_constant__ CUtensorMap tm_state, const __grid_constant__ CUtensorMap tm_cE,
    const __grid_constant__ CUtensorMap tm_cH, const __grid_constant__ CUtensorMap tm_y, Dev<T> D,
    Coef<T, EM, HA> cf, T *__restrict__ wout, T *__restrict__ y, Sched sch, T a, T b, T e2, T cl, int init,
    int mode, EtDev et) {
    pdl_sync();
    using G = GeoW<T, BY>;
    using V2 = typename Vec2<T>::type;
    using SL = StageL<T, EM, HA, G>;
    using SP = StageP<T, EM, HA, G>;                        // + the y tile of the plane (TMA)
    constexpr int RX = 68, RR = RX * (BY + 1);              // ring row pitch, ring plane
    if (ET && et.norms && et_skip(et)) {                          // early termination (f2)
        if (sch.ctr && blockIdx.x == 0 && threadIdx.x == 0)
            atomicAdd(sch.ctr, (unsigned long long)sch.units + gridDim.x);
        return;
    }
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *stages = reinterpret_cast<T *>(smem_raw);
    T *UE = stages + S * SP::SZ;                        // [2][3][RR]
    T *UH = UE + 2 * 3 * RR;                            // [3][RR]
    T *zt = UH + 3 * RR;                                  // [3][ZT_ROW] z-table (EM == 1)
    uint64_t *bars = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(zt + ZtL<T, EM>::N) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x;
    const bool pair = tid < 32 * (BY + 1);
    const bool single = !pair && tid < 32 * (BY + 1) + (BY + 1);
    const bool own = tid < 32 * BY;                         // tile pair thread (phase B)
    const int pi = tid % 32;
    const int jr = pair ? tid / 32 : tid - 32 * (BY + 1);   // row selector
    // local x of the E point / H point, local row of each (relative to x0, y0)
    const int xE = pair ? 2 * pi : 64, xH = pair ? 2 * pi : -1;
    const int yE = pair ? jr : jr;                          // E rows 0..BY
    const int yH = pair ? (jr < BY ? jr : -1) : jr - 1;     // H rows -1..BY-1
    const int sE = (yE + 1) * G::WX + xE + G::OX, sH = (yH + 1) * G::WX + xH + G::OX;
    const int rE = yE * RX + xE + 2, rH = (yH + 1) * RX + xH + 2;
    T bE0 = cf.cEs[0] * cf.sig, bE1 = cf.cEs[1] * cf.sig, bE2 = cf.cEs[2] * cf.sig;
    const T bH0 = cf.cHs[0] * cf.sig, bH1 = cf.cHs[1] * cf.sig, bH2 = cf.cHs[2] * cf.sig;
    if (tid == 0) {
        for (int s2 = 0; s2 < S; ++s2) mbar_init(&bars[s2], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto ld2 = [](const T *p) { return *reinterpret_cast<const V2 *>(p); };
    auto st2 = [](T *p, T u, T v) { *reinterpret_cast<V2 *>(p) = Vec2<T>::make(u, v); };
    double dacc = 0.0, yacc = 0.0;
    uint32_t lcount = 0;
    // cross-unit pipelining (as in K2): thread 0 issues the next unit's first planes into the
    // stage slots the draining unit frees
    __shared__ int s_next;
    int pre = 0;
    int unit = grab_unit(sch, -1);
    while (unit < sch.units) {
        const int tile = unit % sch.ntiles, chunk = unit / sch.ntiles;
        const int x0 = (tile % sch.tiles_x) * G::BX, y0 = (tile / sch.tiles_x) * BY;
        const int kb = chunk * sch.chunk, ke = min(kb + sch.chunk, D.nz);
        const int nplanes = ke - kb + 2;
        const int pre_cur = pre;
        pre = 0;
        int nxt = 0x7fffffff, nx0 = 0, ny0 = 0, nkb = 0, nke = 0;
        stage_ztab<T, EM, HA>(zt, cf, kb, nplanes, D.nz);
        // global coordinates and validity of the E / H points (a = left, b = right)
        const int iEa = x0 + xE, jE = y0 + yE, iHa = x0 + xH, jH = y0 + yH;
        const bool act = pair || single;
        const bool eRow = act && jE >= 0 && jE < D.ny, hRow = act && jH >= 0 && jH < D.ny;
        const bool inEa = eRow && iEa < D.nx, inEb = pair && eRow && iEa + 1 < D.nx;
        const bool inHa = hRow && iHa >= 0 && iHa < D.nx, inHb = pair && hRow && iHa + 1 < D.nx;
        const bool doT = own && inEa;                       // tile pair (E point == H point == own)
        const int64_t gB = D.idx(doT ? iEa : 0, doT ? jE : 0, 0);
        // carried own values of plane k
        T hxa = T(0), hxb = T(0), hya = T(0), hyb = T(0), hza = T(0), hzb = T(0);   // w_h at E point
        T exa = T(0), exb = T(0), eya = T(0), eyb = T(0);                         // w_e at H point
        T uea0 = T(0), ueb0 = T(0), uea1 = T(0), ueb1 = T(0), uea2 = T(0), ueb2 = T(0);   // u_e(k)
        T uma0 = T(0), umb0 = T(0), uma1 = T(0), umb1 = T(0), uma2 = T(0), umb2 = T(0);   // u_h(k-1)
        if (tid == 0)
            for (int p = pre_cur; p < min(S, nplanes); ++p) {
                const uint32_t L = lcount + p, kz = kb - 1 + p;
                issue_plane_y<T, EM, HA, G>(stages + (L % S) * SP::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                            &tm_y, x0, y0, kz, !init && kz >= kb && kz < ke);
            }
        for (int p = 0; p + 1 < nplanes; ++p) {
            const int k = kb - 1 + p, kk = k + 1;
            const uint32_t L0 = lcount + p, L1 = L0 + 1;
            const bool doB = doT && k >= kb;
            V2 yv[6];                                   // y(k) of the own pair
#pragma unroll
            for (int c = 0; c < 6; ++c) yv[c] = Vec2<T>::make(T(0), T(0));
            if (!SP::Y && doB && !init) {               // else staged with w(k) by TMA
                const T *yp = y + gB + (int64_t)k * D.plane;
#pragma unroll
                for (int c = 0; c < 6; ++c) yv[c] = ld2(yp + c * D.cs);
            }
            if (p == 0) mbar_wait(&bars[L0 % S], (L0 / S) & 1);
            mbar_wait(&bars[L1 % S], (L1 / S) & 1);
            const T *P0 = stages + (L0 % S) * SP::SZ;   // plane k (+ y(k))
            const T *P1 = stages + (L1 % S) * SP::SZ;   // plane k+1
            T *UE1 = UE + (kk & 1) * 3 * RR;
            const T *UE0 = UE + (k & 1) * 3 * RR;
            T bEk0 = bE0, bEk1 = bE1, bEk2 = bE2;
            if (EM == 1) {
                bE0 = zt[p + 1];
                bE1 = zt[ZT_ROW + p + 1];
                bE2 = zt[2 * ZT_ROW + p + 1];
                bEk0 = zt[p];
                bEk1 = zt[ZT_ROW + p];
                bEk2 = zt[2 * ZT_ROW + p];
            }
            if (p == 0 && act) {                            // w(kb-1) own values
                if (pair) {
                    V2 t = ld2(P0 + 3 * G::PL + sE); hxa = t.x; hxb = t.y;
                    t = ld2(P0 + 4 * G::PL + sE); hya = t.x; hyb = t.y;
                    t = ld2(P0 + 5 * G::PL + sE); hza = t.x; hzb = t.y;
                    t = ld2(P0 + sH); exa = t.x; exb = t.y;
                    t = ld2(P0 + G::PL + sH); eya = t.x; eyb = t.y;
                } else {
                    hxa = P0[3 * G::PL + sE]; hya = P0[4 * G::PL + sE]; hza = P0[5 * G::PL + sE];
                    exa = P0[sH]; eya = P0[G::PL + sH];
                }
            }
            // ---- phase A ----
            T ua0 = T(0), ub0 = T(0), ua1 = T(0), ub1 = T(0), ua2 = T(0), ub2 = T(0);   // u_e(k+1)
            T va0 = T(0), vb0 = T(0), va1 = T(0), vb1 = T(0), va2 = T(0), vb2 = T(0);   // u_h(k)
            T h1xa = T(0), h1xb = T(0), h1ya = T(0), h1yb = T(0), h1za = T(0), h1zb = T(0);
            T e1xa = T(0), e1xb = T(0), e1ya = T(0), e1yb = T(0), ezka = T(0), ezkb = T(0);
            if (act) {
                // u_e(k+1) = bE .* C^T w_h(k+1), w_h(k) own carried
                {
                    const T *hx = P1 + 3 * G::PL, *hy = P1 + 4 * G::PL, *hz = P1 + 5 * G::PL;
                    const bool vk = kk < D.nz, kp = kk > 0;
                    T wa0 = bE0, wa1 = bE1, wa2 = bE2, wb0 = bE0, wb1 = bE1, wb2 = bE2;
                    if (pair) {
                        const V2 X = ld2(hx + sE), Y = ld2(hy + sE), Z = ld2(hz + sE);
                        const V2 Zjm = ld2(hz + sE - G::WX), Xjm = ld2(hx + sE - G::WX);
                        const T zim = hz[sE - 1], yim = hy[sE - 1];
                        h1xa = X.x; h1xb = X.y; h1ya = Y.x; h1yb = Y.y; h1za = Z.x; h1zb = Z.y;
                        if (EM == 2) {
                            const V2 A0 = ld2(P1 + SL::ST + sE), A1 = ld2(P1 + SL::ST + G::PL + sE);
                            const V2 A2 = ld2(P1 + SL::ST + 2 * G::PL + sE);
                            wa0 = A0.x * cf.sig; wb0 = A0.y * cf.sig;
                            wa1 = A1.x * cf.sig; wb1 = A1.y * cf.sig;
                            wa2 = A2.x * cf.sig; wb2 = A2.y * cf.sig;
                        }
                        const T c0a = ((Z.x - Zjm.x) - Y.x) + hya, c0b = ((Z.y - Zjm.y) - Y.y) + hyb;
                        const T c1a = ((X.x - hxa) - Z.x) + zim, c1b = ((X.y - hxb) - Z.y) + Z.x;
                        const T c2a = ((Y.x - yim) - X.x) + Xjm.x, c2b = ((Y.y - Y.x) - X.y) + Xjm.y;
                        ua0 = (inEa && jE > 0 && vk && kp) ? wa0 * c0a : T(0);
                        ub0 = (inEb && jE > 0 && vk && kp) ? wb0 * c0b : T(0);
                        ua1 = (inEa && iEa > 0 && vk && kp) ? wa1 * c1a : T(0);
                        ub1 = (inEb && vk && kp) ? wb1 * c1b : T(0);
                        ua2 = (inEa && iEa > 0 && jE > 0 && vk) ? wa2 * c2a : T(0);
                        ub2 = (inEb && jE > 0 && vk) ? wb2 * c2b : T(0);
                        st2(UE1 + rE, ua0, ub0);
                        st2(UE1 + RR + rE, ua1, ub1);
                        st2(UE1 + 2 * RR + rE, ua2, ub2);
                    } else {
                        const T X = hx[sE], Y = hy[sE], Z = hz[sE];
                        h1xa = X; h1ya = Y; h1za = Z;
                        if (EM == 2) {
                            wa0 = P1[SL::ST + sE] * cf.sig;
                            wa1 = P1[SL::ST + G::PL + sE] * cf.sig;
                            wa2 = P1[SL::ST + 2 * G::PL + sE] * cf.sig;
                        }
                        const T c0 = ((Z - hz[sE - G::WX]) - Y) + hya;
                        const T c1 = ((X - hxa) - Z) + hz[sE - 1];
                        const T c2 = ((Y - hy[sE - 1]) - X) + hx[sE - G::WX];
                        ua0 = (inEa && jE > 0 && vk && kp) ? wa0 * c0 : T(0);
                        ua1 = (inEa && iEa > 0 && vk && kp) ? wa1 * c1 : T(0);
                        ua2 = (inEa && iEa > 0 && jE > 0 && vk) ? wa2 * c2 : T(0);
                        UE1[rE] = ua0;
                        UE1[RR + rE] = ua1;
                        UE1[2 * RR + rE] = ua2;
                    }
                }
                // u_h(k) = -bH .* C w_e(k), w_e(k) x, y own carried
                {
                    const T *ex = P0, *ey = P0 + G::PL, *ez = P0 + 2 * G::PL;
                    const bool vk = k >= 0 && k < D.nz;
                    T ga0 = bH0, ga1 = bH1, ga2 = bH2, gb0 = bH0, gb1 = bH1, gb2 = bH2;
                    if (pair) {
                        const V2 EZ = ld2(ez + sH), EX1 = ld2(P1 + sH), EY1 = ld2(P1 + G::PL + sH);
                        const V2 Zjp = ld2(ez + sH + G::WX), Xjp = ld2(ex + sH + G::WX);
                        const T zip = ez[sH + 2], yip = ey[sH + 2];
                        ezka = EZ.x; ezkb = EZ.y;
                        e1xa = EX1.x; e1xb = EX1.y; e1ya = EY1.x; e1yb = EY1.y;
                        if (HA) {
                            const int ch = SL::ST + SL::CE;
                            const V2 A0 = ld2(P0 + ch + sH), A1 = ld2(P0 + ch + G::PL + sH), A2 = ld2(P0 + ch + 2 * G::PL + sH);
                            ga0 = A0.x * cf.sig; gb0 = A0.y * cf.sig;
                            ga1 = A1.x * cf.sig; gb1 = A1.y * cf.sig;
                            ga2 = A2.x * cf.sig; gb2 = A2.y * cf.sig;
                        }
                        const T c0a = ((eya + Zjp.x) - EY1.x) - EZ.x, c0b = ((eyb + Zjp.y) - EY1.y) - EZ.y;
                        const T c1a = ((EZ.x + EX1.x) - EZ.y) - exa, c1b = ((EZ.y + EX1.y) - zip) - exb;
                        const T c2a = ((exa + eyb) - Xjp.x) - eya, c2b = ((exb + yip) - Xjp.y) - eyb;
                        va0 = (inHa && iHa > 0 && vk) ? -(ga0 * c0a) : T(0);
                        vb0 = (inHb && vk) ? -(gb0 * c0b) : T(0);
                        va1 = (inHa && jH > 0 && vk) ? -(ga1 * c1a) : T(0);
                        vb1 = (inHb && jH > 0 && vk) ? -(gb1 * c1b) : T(0);
                        va2 = (inHa && vk && k > 0) ? -(ga2 * c2a) : T(0);
                        vb2 = (inHb && vk && k > 0) ? -(gb2 * c2b) : T(0);
                        st2(UH + rH, va0, vb0);
                        st2(UH + RR + rH, va1, vb1);
                        st2(UH + 2 * RR + rH, va2, vb2);
                    } else {
                        const T EZv = ez[sH], EX1v = P1[sH], EY1v = P1[G::PL + sH];
                        ezka = EZv;
                        e1xa = EX1v;
                        e1ya = EY1v;
                        if (HA) {
                            const int ch = SL::ST + SL::CE;
                            ga0 = P0[ch + sH] * cf.sig;
                            ga1 = P0[ch + G::PL + sH] * cf.sig;
                            ga2 = P0[ch + 2 * G::PL + sH] * cf.sig;
                        }
                        const T c0 = ((eya + ez[sH + G::WX]) - EY1v) - EZv;
                        const T c1 = ((EZv + EX1v) - ez[sH + 1]) - exa;
                        const T c2 = ((exa + ey[sH + 1]) - ex[sH + G::WX]) - eya;
                        va0 = (inHa && iHa > 0 && vk) ? -(ga0 * c0) : T(0);
                        va1 = (inHa && jH > 0 && vk) ? -(ga1 * c1) : T(0);
                        va2 = (inHa && vk && k > 0) ? -(ga2 * c2) : T(0);
                        UH[rH] = va0;
                        UH[RR + rH] = va1;
                        UH[2 * RR + rH] = va2;
                    }
                }
            }
            __syncthreads();
            // ---- phase B: w'(k), y(k) on the own tile pair ----
            if (doB) {
                const bool inB = inEb;                      // right point inside the grid
                if (SP::Y && !init) {                       // y(k), staged with w(k) by TMA
#pragma unroll
                    for (int c = 0; c < 6; ++c) yv[c] = ld2(P0 + SP::YOFF + c * (G::BX * BY) + yE * G::BX + xE);
                }
                T wn[12];
#pragma unroll
                for (int c = 0; c < 12; ++c) wn[c] = T(0);
                const T w_a[6] = {exa, eya, ezka, hxa, hya, hza};
                const T w_b[6] = {exb, eyb, ezkb, hxb, hyb, hzb};
                T be[6] = {bEk0, bEk1, bEk2, bEk0, bEk1, bEk2};   // a: 0..2, b: 3..5
                T bh[6] = {bH0, bH1, bH2, bH0, bH1, bH2};
                if (EM == 2) {
                    const V2 A0 = ld2(P0 + SL::ST + sE), A1 = ld2(P0 + SL::ST + G::PL + sE);
                    const V2 A2 = ld2(P0 + SL::ST + 2 * G::PL + sE);
                    be[0] = A0.x * cf.sig; be[3] = A0.y * cf.sig;
                    be[1] = A1.x * cf.sig; be[4] = A1.y * cf.sig;
                    be[2] = A2.x * cf.sig; be[5] = A2.y * cf.sig;
                }
                if (HA) {
                    const int ch = SL::ST + SL::CE;
                    const V2 A0 = ld2(P0 + ch + sE), A1 = ld2(P0 + ch + G::PL + sE), A2 = ld2(P0 + ch + 2 * G::PL + sE);
                    bh[0] = A0.x * cf.sig; bh[3] = A0.y * cf.sig;
                    bh[1] = A1.x * cf.sig; bh[4] = A1.y * cf.sig;
                    bh[2] = A2.x * cf.sig; bh[5] = A2.y * cf.sig;
                }
                if (mode != 1) {
                    // C u_e(k): j+1 from the ring (float2), i+1 = own right (a) / ring i+2 (b)
                    const V2 UZj = ld2(UE0 + 2 * RR + rE + RX), UXj = ld2(UE0 + rE + RX);
                    const T uzi = UE0[2 * RR + rE + 2], uyi = UE0[RR + rE + 2];
                    const T c0a = ((uea1 + UZj.x) - ua1) - uea2, c0b = ((ueb1 + UZj.y) - ub1) - ueb2;
                    const T c1a = ((uea2 + ua0) - ueb2) - uea0, c1b = ((ueb2 + ub0) - uzi) - ueb0;
                    const T c2a = ((uea0 + ueb1) - UXj.x) - uea1, c2b = ((ueb0 + uyi) - UXj.y) - ueb1;
                    // C^T u_h(k): j-1 from the ring (float2), i-1 = ring (a) / own left (b)
                    const V2 HZj = ld2(UH + 2 * RR + rH - RX), HXj = ld2(UH + rH - RX);
                    const T hzi = UH[2 * RR + rH - 1], hyi = UH[RR + rH - 1];
                    const T d0a = ((va2 - HZj.x) - va1) + uma1, d0b = ((vb2 - HZj.y) - vb1) + umb1;
                    const T d1a = ((va0 - uma0) - va2) + hzi, d1b = ((vb0 - umb0) - vb2) + va2;
                    const T d2a = ((va1 - hyi) - va0) + HXj.x, d2b = ((vb1 - va1) - vb0) + HXj.y;
                    const bool kp = k > 0, jp = jE > 0, ip = iEa > 0;
                    wn[0] = ((jp && kp) ? be[0] * d0a : T(0)) + e2 * w_a[0];
                    wn[1] = ((ip && kp) ? be[1] * d1a : T(0)) + e2 * w_a[1];
                    wn[2] = ((ip && jp) ? be[2] * d2a : T(0)) + e2 * w_a[2];
                    wn[3] = (ip ? -(bh[0] * c0a) : T(0)) + e2 * w_a[3];
                    wn[4] = (jp ? -(bh[1] * c1a) : T(0)) + e2 * w_a[4];
                    wn[5] = (kp ? -(bh[2] * c2a) : T(0)) + e2 * w_a[5];
                    if (inB) {
                        wn[6] = ((jp && kp) ? be[3] * d0b : T(0)) + e2 * w_b[0];
                        wn[7] = (kp ? be[4] * d1b : T(0)) + e2 * w_b[1];
                        wn[8] = (jp ? be[5] * d2b : T(0)) + e2 * w_b[2];
                        wn[9] = -(bh[3] * c0b) + e2 * w_b[3];
                        wn[10] = (jp ? -(bh[4] * c1b) : T(0)) + e2 * w_b[4];
                        wn[11] = (kp ? -(bh[5] * c2b) : T(0)) + e2 * w_b[5];
                    }
                }
                const int64_t go = gB + (int64_t)k * D.plane;
                PE_CHECK(D.in_state(go + 5 * D.cs + 1) && (go & 1) == 0, "K2v w' / y store");
                if (mode == 0) {
#pragma unroll
                    for (int c = 0; c < 6; ++c) st2(wout + go + c * D.cs, wn[c], wn[6 + c]);
                }
                const T u_a[6] = {uea0, uea1, uea2, va0, va1, va2};
                const T u_b[6] = {ueb0, ueb1, ueb2, vb0, vb1, vb2};
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    T qa = (yv[c].x + a * w_a[c]) + b * u_a[c];
                    T qb = (yv[c].y + a * w_b[c]) + b * u_b[c];
                    if (mode == 2) {
                        qa = qa + cl * wn[c];
                        qb = qb + cl * wn[6 + c];
                    }
                    if (!inB) qb = T(0);
                    st2(y + go + c * D.cs, qa, qb);
                    if (ET && et.norms) {
                        const T ga = c < 3 ? be[c] : bh[c - 3], gb = c < 3 ? be[3 + c] : bh[c];
                        if (ga != T(0)) {
                            const double d = (double)qa - (double)yv[c].x;
                            dacc += d * d / (double)ga;
                            yacc += (double)qa * qa / (double)ga;
                        }
                        if (inB && gb != T(0)) {
                            const double d = (double)qb - (double)yv[c].y;
                            dacc += d * d / (double)gb;
                            yacc += (double)qb * qb / (double)gb;
                        }
                    }
                }
            }
            // carry plane k+1 -> k
            hxa = h1xa; hxb = h1xb; hya = h1ya; hyb = h1yb; hza = h1za; hzb = h1zb;
            exa = e1xa; exb = e1xb; eya = e1ya; eyb = e1yb;
            uea0 = ua0; ueb0 = ub0; uea1 = ua1; ueb1 = ub1; uea2 = ua2; ueb2 = ub2;
            uma0 = va0; umb0 = vb0; uma1 = va1; umb1 = vb1; uma2 = va2; umb2 = vb2;
            __syncthreads();
            if (tid == 0) {
                const uint32_t L = lcount + p + S;
                if (p + S < nplanes) {
                    const int kz = kb - 1 + p + S;
                    issue_plane_y<T, EM, HA, G>(stages + (L % S) * SP::SZ, &bars[L % S], &tm_state, &tm_cE, &tm_cH,
                                                &tm_y, x0, y0, kz, !init && kz >= kb && kz < ke);
                } else {
                    if (p + S == nplanes) {                   // the slots start to free: next unit
                        nxt = grab_next_t0(sch, unit);
                        s_next = nxt;
                        if (nxt < sch.units) {
                            const int nt = nxt % sch.ntiles, nc = nxt / sch.ntiles;
                            nx0 = (nt % sch.tiles_x) * G::BX;
                            ny0 = (nt / sch.tiles_x) * BY;
                            nkb = nc * sch.chunk;
                            nke = min(nkb + sch.chunk, D.nz);
                        }
                    }
                    const int q = p + S - nplanes;            // plane q of the next unit
                    if (sch.lookahead && nxt < sch.units && q < nke - nkb + 2) {
                        const int kz = nkb - 1 + q;
                        issue_plane_y<T, EM, HA, G>(stages + (L % S) * SP::SZ, &bars[L % S], &tm_state, &tm_cE,
                                                    &tm_cH, &tm_y, nx0, ny0, kz, !init && kz >= nkb && kz < nke);
                        pre = q + 1;
                    }
                }
            }
        }
        lcount += nplanes;
        if (S == 2) __syncthreads();                          // s_next written in the last iteration
        unit = s_next;
    }
    if (ET && et.norms) {
        const double ds = block_sum(dacc);
        __syncthreads();
        const double ys = block_sum(yacc);
        if (tid == 0) {
            atomicAdd(et.norms + 2 * et.op, ds);
            atomicAdd(et.norms + 2 * et.op + 1, ys);
        }
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

static int num_sms() {   // of the current device (cached per device)
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev] = n;
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
    int bc = std::min(g.nz, ZT_ROW - 2);
    // L2 reuse: in the dynamic unit order a y-neighbour tile (tiles_x units later) starts
    // about tiles_x * chunk / resident planes later; keep that within ~4 planes so its halo
    // rows are still in L2 (measured at 768^3 fp64: chunk 48-64 beats the unconstrained 154
    // by 4%)
    // and at most 32 planes: measured with the dynamic order (C5 vacuum, K1r fp64): 640^3 chunk
    // 32-48 4.27 ms vs the cost model's pick (88) 5.01 ms; 384^3 0.87 vs 0.99 ms; at 768^3 ncu
    // read 1.5x the algorithmic bytes with chunks 48-74 and 1.15x with 24 (L2 hit rate 35 -> 45%)
    const int cap = std::min(32, std::max(8, (int)(4.0 * resident / std::max(1, s.tiles_x))));
    for (int ch = 1; ch <= g.nz; ++ch) {
        const int nch = (g.nz + ch - 1) / ch;
        const double units = (double)s.ntiles * nch;
        // chunks below 8 planes only while every unit still gets its own CTA (mid-size,
        // L2-resident grids, where a unit's time is latency: measured at 64^3 fp64 chunk 4
        // 10.3 us vs chunk 8 12.3 us per leapfrog step, 32^3 chunk 1 6.2 vs 12.3 us)
        if (ch < std::min(g.nz, 8) && nch > 1 && units > resident) continue;
        if (ch > cap) continue;
        if (ch > ZT_ROW - 2) continue;       // the staged z-table holds chunk + 2 planes
        const double waves = units / resident;
        const double eff_waves = std::ceil(waves);
        // cost ~ rounds * (chunk + 2 halo planes)
        const double cost = eff_waves * (double)(ch + 2);
        if (cost < best - 1e-9) {
            best = cost;
            bc = ch;
        }
    }
    if (const char *ev = getenv("PARAEXP_ZCHUNK")) bc = std::max(1, std::min(std::min(g.nz, ZT_ROW - 2), atoi(ev)));
    s.chunk = bc;
    s.nchunks = (g.nz + bc - 1) / bc;
    s.units = s.ntiles * s.nchunks;
    s.ctr = nullptr;
    s.lookahead = 1;
    if (const char *ev = getenv("PARAEXP_NO_LOOKAHEAD")) s.lookahead = atoi(ev) == 0;
    s.base = 0;
    return s;
}

// dynamic scheduling (default; PARAEXP_STATIC_SCHED=1 keeps the static stride)
static bool dynamic_sched() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("PARAEXP_STATIC_SCHED");
        v = (e && atoi(e) != 0) ? 0 : 1;
    }
    return v == 1;
}
// per-launch Sched with the grid's unit counter; advances the host shadow of the counter
static Sched launch_sched(const Grid &g, Sched sch, int grid) {
    Grid &G = const_cast<Grid &>(g);
    if (!dynamic_sched() || !G.d_sched) return sch;
    if (grid >= sch.units) return sch;   // one wave: unit = blockIdx.x, no counter round trips
    sch.ctr = (unsigned long long *)G.d_sched;
    sch.base = G.sched_base;
    G.sched_base += (unsigned long long)sch.units + (unsigned long long)grid;
    return sch;
}

// occupancy per SM of a kernel at its shared-memory size, cached per (device, kernel): the
// dynamic shared-memory opt-in (cudaFuncSetAttribute) is per device context, so a grid on a
// second device gets its own attribute call
template <typename K>
static int resident_per_sm(K kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(dev, (const void *)kern);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    cache[key] = per_sm;
    return per_sm;
}

// K1r launcher (same schedule and maps as K1)
template <typename T, int EM, bool HA, int S, bool TR>
static int leapfrog_r_V(const KernelArgs &ka, void *bufs[2], int64_t nsteps, int nsrc, const void *q_dev,
                        const std::vector<SrcDev> &hsrc, const TraceDev *tr) {
    constexpr int BX = 32, BY = 8;
    using G = Geo<T, BX, BY>;
    constexpr size_t smem = (size_t)(S * StageL<T, EM, HA, G>::SZ + 2 * 3 * G::RP + ZtL<T, EM>::N) * sizeof(T) + 8 * S + 16;
    const Grid &g = *ka.g;
    auto kern = leapfrog_r_kernel<T, EM, HA, BX, BY, S, TR>;
    const int per_sm = resident_per_sm(kern, G::NTHR, smem);
    if (per_sm < 1) return fail(PARAEXP_ECUDA, "leapfrog_r kernel does not fit on an SM");
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
    TraceDev trm;
    if (TR) trm = *tr;
    for (int64_t m = 0; m < nsteps; ++m) {
        const bool even = (m % 2) == 0;
        if (TR) {
            trm.energy = tr->energy ? tr->energy + m : nullptr;
            trm.probe = tr->probe ? tr->probe + m * tr->np : nullptr;
            if (!trm.probe) trm.np = 0;
        }
        launch_k(kern, grid, G::NTHR, smem, s, even ? tmA : tmB, tmE, tmH, D, cf, (T *)(even ? bufs[1] : bufs[0]),
                                          ka.static_sched ? sch : launch_sched(g, sch, grid),
                                          sl, nsrc ? (const T *)q_dev + m * nsrc : nullptr, trm);
        ++*ka.launches;
    }
    if (nsteps % 2) std::swap(bufs[0], bufs[1]);
    return check_cuda("leapfrog_r");
}

// K1v launcher (fp32, 64 x 8 tiles, two points per thread)
template <int EM, bool HA, int S, bool TR>
static int leapfrog_v_V(const KernelArgs &ka, void *bufs[2], int64_t nsteps, int nsrc, const void *q_dev,
                        const std::vector<SrcDev> &hsrc, const TraceDev *tr) {
    constexpr int BY = 8;
    using G = GeoV<BY>;
    constexpr size_t smem = (size_t)(S * StageL<float, EM, HA, G>::SZ + 2 * 3 * G::RP + ZtL<float, EM>::N) * sizeof(float) + 8 * S + 16;
    const Grid &g = *ka.g;
    auto kern = leapfrog_v_kernel<EM, HA, BY, S, TR>;
    const int per_sm = resident_per_sm(kern, G::NTHR, smem);
    if (per_sm < 1) return fail(PARAEXP_ECUDA, "leapfrog_v kernel does not fit on an SM");
    const Sched sch = make_sched(g, G::BX, BY, per_sm * num_sms());
    const int grid = std::min(sch.units, per_sm * num_sms());
    auto D = make_dev<float>(g);
    auto cf = make_coef<float, EM, HA>(g, 1.0);
    CUtensorMap tmE, tmH, tmA, tmB;
    int rc;
    if (EM == 2 && (rc = make_map<float>(&tmE, g, g.d_cE_arr, 3, G::WX, G::HY))) return rc;
    if (HA && (rc = make_map<float>(&tmH, g, g.d_cH_arr, 3, G::WX, G::HY))) return rc;
    if ((rc = make_map<float>(&tmA, g, bufs[0], 6, G::WX, G::HY))) return rc;
    if ((rc = make_map<float>(&tmB, g, bufs[1], 6, G::WX, G::HY))) return rc;
    SrcList sl;
    sl.n = nsrc;
    for (int r = 0; r < nsrc && r < 16; ++r) {
        sl.c[r] = hsrc[r].comp;
        sl.i[r] = hsrc[r].i;
        sl.j[r] = hsrc[r].j;
        sl.k[r] = hsrc[r].k;
    }
    cudaStream_t s = (cudaStream_t)ka.stream;
    TraceDev trm;
    if (TR) trm = *tr;
    for (int64_t m = 0; m < nsteps; ++m) {
        const bool even = (m % 2) == 0;
        if (TR) {
            trm.energy = tr->energy ? tr->energy + m : nullptr;
            trm.probe = tr->probe ? tr->probe + m * tr->np : nullptr;
            if (!trm.probe) trm.np = 0;
        }
        launch_k(kern, grid, G::NTHR, smem, s, even ? tmA : tmB, tmE, tmH, D, cf, (float *)(even ? bufs[1] : bufs[0]),
                                          ka.static_sched ? sch : launch_sched(g, sch, grid), sl,
                                          nsrc ? (const float *)q_dev + m * nsrc : nullptr, trm);
        ++*ka.launches;
    }
    if (nsteps % 2) std::swap(bufs[0], bufs[1]);
    return check_cuda("leapfrog_v");
}

int k_leapfrog_fused(const KernelArgs &ka, void *bufs[2], int64_t nsteps, const SrcDev *src_dev,
                     int nsrc, const void *q_dev, const TraceDev *tr) {
    if (nsrc > 16) return k_leapfrog_unfused(ka, bufs[0], nsteps, src_dev, nsrc, q_dev, tr);
    const std::vector<SrcDev> &hsrc = ka.g->h_src;
    const bool trace = tr && (tr->energy || (tr->probe && tr->np > 0));
    return with_types(*ka.g, 1.0, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        if constexpr (std::is_same<T, float>::value) {   // K1v: fp32, two points per thread
            if (trace) return leapfrog_v_V<EM, HA, 3, true>(ka, bufs, nsteps, nsrc, q_dev, hsrc, tr);
            return leapfrog_v_V<EM, HA, 3, false>(ka, bufs, nsteps, nsrc, q_dev, hsrc, tr);
        } else {                                            // K1r: fp64
            if (trace) return leapfrog_r_V<T, EM, HA, 3, true>(ka, bufs, nsteps, nsrc, q_dev, hsrc, tr);
            return leapfrog_r_V<T, EM, HA, 3, false>(ka, bufs, nsteps, nsrc, q_dev, hsrc, tr);
        }
    });
}

// K2 launcher (fp64): one launch per pair op; w ping-pongs between bufs[0] and bufs[2]
template <typename T, int EM, bool HA, int S>
static int poly_fused_V(const KernelArgs &ka, const Plan &plan, void *bufs[4]) {
    constexpr int BX = 32, BY = 8;
    using G = Geo<T, BX, BY>;
    constexpr size_t smem = (size_t)(S * StageP<T, EM, HA, G>::SZ + 3 * 3 * G::RP + ZtL<T, EM>::N) * sizeof(T) + 8 * S + 16;
    const Grid &g = *ka.g;
    auto kern = pair_fused_kernel<T, EM, HA, BX, BY, S>;
    const int per_sm = resident_per_sm(kern, G::NTHR, smem);
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
    CUtensorMap tmW, tmS, tmY;   // maps of the two ping-pong w buffers and of y (tile box)
    if ((rc = make_map<T>(&tmW, g, w, 6, G::WX, G::HY))) return rc;
    if ((rc = make_map<T>(&tmS, g, sp, 6, G::WX, G::HY))) return rc;
    if ((rc = make_map<T>(&tmY, g, yy, 6, BX, BY))) return rc;
    int init = 1;
    EtDev et;
    if (ka.et) et = *ka.et;
    int opi = 0;
    for (const Op &op : plan.ops) {
        et.op = opi++;
        et.apps = op.kind == 1 ? 1 : 2;
        launch_k(kern, grid, G::NTHR, smem, s, tmW, tmE, tmH, tmY, D, cf, sp, yy, launch_sched(g, sch, grid),
                 T(op.a), T(op.b), T(op.e2), T(op.c), init, op.kind, et);
        ++*ka.launches;
        if (op.kind == 0) {
            std::swap(w, sp);
            std::swap(tmW, tmS);
        }
        init = 0;
    }
    bufs[0] = yy;
    bufs[1] = w;
    bufs[2] = sp;
    bufs[3] = sp2;
    return check_cuda("poly fused");
}

// K2v launcher (64 x BY tiles, two points per thread; same buffer protocol as K2)
template <typename T, int EM, bool HA, int BY, int S>
static int poly_v_V(const KernelArgs &ka, const Plan &plan, void *bufs[4]) {
    using G = GeoW<T, BY>;
    constexpr int RR = 68 * (BY + 1);
    constexpr size_t smem = (size_t)(S * StageP<T, EM, HA, G>::SZ + 3 * 3 * RR + ZtL<T, EM>::N) * sizeof(T) + 8 * S + 16;
    const Grid &g = *ka.g;
    auto kern = ka.et ? pair_v_kernel<T, EM, HA, BY, S, true> : pair_v_kernel<T, EM, HA, BY, S, false>;
    const int per_sm = resident_per_sm(pair_v_kernel<T, EM, HA, BY, S, true>, G::NTHR, smem);
    const int per_sm2 = resident_per_sm(pair_v_kernel<T, EM, HA, BY, S, false>, G::NTHR, smem);
    if (per_sm2 < per_sm) return fail(PARAEXP_ECUDA, "pair_v variants differ in occupancy");
    if (per_sm < 1) return fail(PARAEXP_ECUDA, "pair_v kernel does not fit on an SM");
    const Sched sch = make_sched(g, G::BX, BY, per_sm * num_sms());
    const int grid = std::min(sch.units, per_sm * num_sms());
    auto D = make_dev<T>(g);
    auto cf = make_coef<T, EM, HA>(g, plan.sigma);
    CUtensorMap tmE, tmH;
    int rc;
    if (EM == 2 && (rc = make_map<T>(&tmE, g, g.d_cE_arr, 3, G::WX, G::HY))) return rc;
    if (HA && (rc = make_map<T>(&tmH, g, g.d_cH_arr, 3, G::WX, G::HY))) return rc;
    cudaStream_t s = (cudaStream_t)ka.stream;
    T *w = (T *)bufs[0], *yy = (T *)bufs[1], *sp = (T *)bufs[2], *sp2 = (T *)bufs[3];
    CUtensorMap tmW, tmS, tmY;
    if ((rc = make_map<T>(&tmW, g, w, 6, G::WX, G::HY))) return rc;
    if ((rc = make_map<T>(&tmS, g, sp, 6, G::WX, G::HY))) return rc;
    if ((rc = make_map<T>(&tmY, g, yy, 6, G::BX, BY))) return rc;
    int init = 1;
    EtDev et;
    if (ka.et) et = *ka.et;
    int opi = 0;
    for (const Op &op : plan.ops) {
        et.op = opi++;
        et.apps = op.kind == 1 ? 1 : 2;
        launch_k(kern, grid, G::NTHR, smem, s, tmW, tmE, tmH, tmY, D, cf, sp, yy, launch_sched(g, sch, grid), (T)op.a,
                                          (T)op.b, (T)op.e2, (T)op.c, init, op.kind, et);
        ++*ka.launches;
        if (op.kind == 0) {
            std::swap(w, sp);
            std::swap(tmW, tmS);
        }
        init = 0;
    }
    bufs[0] = yy;
    bufs[1] = w;
    bufs[2] = sp;
    bufs[3] = sp2;
    return check_cuda("poly_v");
}

int k_poly_substep_fused(const KernelArgs &ka, const Plan &plan, void *bufs[4]) {
    return with_types(*ka.g, plan.sigma, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        if constexpr (std::is_same<T, float>::value)
            return poly_v_V<float, EM, HA, 8, 3>(ka, plan, bufs);   // K2v: fp32, two points per thread
        else
            return poly_fused_V<T, EM, HA, 3>(ka, plan, bufs);      // K2: fp64
    });
}

}  // namespace pe
