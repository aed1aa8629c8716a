// small.cu -- single-CTA, shared-memory-resident kernels for small grids (sm_100a).
//
// A grid of up to ~2k cells (fp64) / ~4k cells (fp32) -- the paper's 2-D wave (40 x 40 x 1 cells),
// C1 (8^3) -- fits one CTA's shared memory.  Stepping it with one kernel launch per time step
// (or per Newton pair) is launch-bound (~4-6 us per launch for microseconds of work), so here ONE
// CTA keeps the state in shared memory and runs a whole leapfrog sequence (rows a2/a3) or a whole
// polynomial propagator p(X)^s (row a6) in a single launch, with __syncthreads between the curl
// half-sweeps.  Arithmetic, operation order and liveness are those of the unfused kernels in
// kernels.cu (the curl helpers' operand order, on a compact copy of the layout), so results match
// them and the oracle at the north_star tolerances.  Per-cell indices, liveness and neighbour flags
// are computed once per launch, so the time loops do no index arithmetic.  Independent problems (ParaExp's sub-interval sweeps)
// run as independent single-CTA launches on separate streams, i.e. concurrently on separate SMs.
#include <cuda_runtime.h>

#include "internal.h"
#include "kernels_common.cuh"

namespace pe {

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxOps = 80;
constexpr size_t kSmallSmemMax = 232448;   // 227 KB opt-in shared memory per CTA   // pair ops per substep (m <= 150 -> 75)

template <typename T>
static constexpr int64_t small_max_cells() {
    return sizeof(T) == 8 ? 2048 : 4096;   // two 6-component vectors in <= 196 KB of shared memory
}

bool small_supported(const Grid &g) {
    static const bool off = [] {
        const char *e = getenv("PARAEXP_NO_SMALL");
        return e && atoi(e) != 0;
    }();
    if (off) return false;
    const int64_t cells = (int64_t)g.nx * g.ny * g.nz;
    return g.dtype == PARAEXP_F64 ? cells <= small_max_cells<double>() : cells <= small_max_cells<float>();
}

struct SmallSrc {
    int n;
    int c[16], i[16], j[16], k[16];
};

constexpr int kQChunk = 256;   // leapfrog steps of source values staged in shared memory at a time

// Per owned cell, computed once per launch: the compact index x, the padded (global) index g
// (per-edge / per-face coefficient arrays) and a flag word -- bits 0-5: the -1/+1 neighbours
// exist (i>0, j>0, k>0, i+1<nx, j+1<ny, k+1<nz), bits 6-8: e_c live, bits 9-11: h_c live,
// bits 12-31: k (z-table coefficients).  The time loops then do no index arithmetic.
struct SmallCell {
    int x, g;
    unsigned f;
};

template <typename T>
__device__ __forceinline__ SmallCell small_cell(const Dev<T> &D, int x) {
    SmallCell c;
    c.x = x;
    const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
    c.g = (int)D.idx(i, j, k);
    c.f = (unsigned)(i > 0) | ((unsigned)(j > 0) << 1) | ((unsigned)(k > 0) << 2) |
          ((unsigned)(i + 1 < D.nx) << 3) | ((unsigned)(j + 1 < D.ny) << 4) | ((unsigned)(k + 1 < D.nz) << 5);
    for (int q = 0; q < 3; ++q) {
        c.f |= (unsigned)D.e_live(q, i, j, k) << (6 + q);
        c.f |= (unsigned)D.h_live(q, i, j, k) << (9 + q);
    }
    c.f |= (unsigned)k << 12;
    return c;
}

// (C e) and (C^T h) at a cell of the compact layout (px = nx, plane = nx*ny) from its flag word;
// the same operands and operation order as curl_at / curlT_at (kernels_common.cuh).
template <typename T>
__device__ __forceinline__ void curl_f(const T *ex, const T *ey, const T *ez, int x, unsigned f, int px,
                                       int plane, T &c0, T &c1, T &c2) {
    const T ex0 = ex[x], ey0 = ey[x], ez0 = ez[x];
    const T ez_jp = (f & 16u) ? ez[x + px] : T(0);
    const T ex_jp = (f & 16u) ? ex[x + px] : T(0);
    const T ey_kp = (f & 32u) ? ey[x + plane] : T(0);
    const T ex_kp = (f & 32u) ? ex[x + plane] : T(0);
    const T ez_ip = (f & 8u) ? ez[x + 1] : T(0);
    const T ey_ip = (f & 8u) ? ey[x + 1] : T(0);
    c0 = ((ey0 + ez_jp) - ey_kp) - ez0;
    c1 = ((ez0 + ex_kp) - ez_ip) - ex0;
    c2 = ((ex0 + ey_ip) - ex_jp) - ey0;
}

template <typename T>
__device__ __forceinline__ void curlT_f(const T *hx, const T *hy, const T *hz, int x, unsigned f, int px,
                                        int plane, T &c0, T &c1, T &c2) {
    const T hx0 = hx[x], hy0 = hy[x], hz0 = hz[x];
    const T hz_jm = (f & 2u) ? hz[x - px] : T(0);
    const T hx_jm = (f & 2u) ? hx[x - px] : T(0);
    const T hy_km = (f & 4u) ? hy[x - plane] : T(0);
    const T hx_km = (f & 4u) ? hx[x - plane] : T(0);
    const T hz_im = (f & 1u) ? hz[x - 1] : T(0);
    const T hy_im = (f & 1u) ? hy[x - 1] : T(0);
    c0 = ((hz0 - hz_jm) - hy0) + hy_km;
    c1 = ((hx0 - hx_km) - hz0) + hz_im;
    c2 = ((hy0 - hy_im) - hx0) + hx_jm;
}

template <typename T>
__device__ __forceinline__ void load_state(const Dev<T> &D, const T *st, T *S, int cells) {
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            S[c * cells + x] = st[c * D.cs + D.idx(i, j, k)];
        }
}

template <typename T>
__device__ __forceinline__ void store_state(const Dev<T> &D, T *st, const T *S, int cells) {
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            st[c * D.cs + D.idx(i, j, k)] = S[c * cells + x];
        }
}

// ---------------------------------------------------------------------------------------
// leapfrog: nsteps steps on the state (device layout) in place.  Thread t owns cells
// t, t + 1024, ... (R of them).  The source values of kQChunk steps are staged in shared memory;
// the owner of a source's cell subtracts it right after its own e-update (e_s <- e_s - q[m][s],
// in s order for sources on the same edge), so a step takes two barriers.
// ---------------------------------------------------------------------------------------
template <typename T, int EM, bool HA, int R>
__global__ void __launch_bounds__(kSmallThreads, 1) leapfrog_small_kernel(Dev<T> D, Coef<T, EM, HA> cf,
                                                                          T *__restrict__ st, int64_t nsteps,
                                                                          SmallSrc src, const T *__restrict__ q) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *S = reinterpret_cast<T *>(smem_raw);
    const int cells = D.nx * D.ny * D.nz, px = D.nx, plane = D.nx * D.ny;
    // per-edge / per-face coefficients (EM 2, HA) are staged once as beta values in shared
    // memory [bE0 bE1 bE2 bH0 bH1 bH2][cells]: read from global every step they miss L1
    constexpr bool CS = (EM == 2 || HA);
    T *CF = S + 6 * cells;
    T *Q = S + (CS ? 12 : 6) * cells;
    load_state(D, st, S, cells);
    SmallCell cl[R];
    unsigned smask[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int x = threadIdx.x + r * kSmallThreads;
        cl[r] = small_cell(D, x < cells ? x : 0);
        cl[r].x = x;
        smask[r] = 0;
        for (int s = 0; s < src.n; ++s)
            if (src.i[s] + D.nx * (src.j[s] + D.ny * src.k[s]) == x) smask[r] |= 1u << s;
        if (CS && x < cells) {
            const int k = (int)(cl[r].f >> 12);
            for (int c = 0; c < 3; ++c) {
                CF[c * cells + x] = cf.bE(c, k, cl[r].g);
                CF[(3 + c) * cells + x] = T(1) * cf.bH(c, cl[r].g);
            }
        }
    }
    auto bEx = [&](int c, int k, const SmallCell &q) -> T { return CS ? CF[c * cells + q.x] : cf.bE(c, k, q.g); };
    auto bHx = [&](int c, const SmallCell &q) -> T {
        return CS ? CF[(3 + c) * cells + q.x] : T(1) * cf.bH(c, q.g);
    };
    T *ex = S, *ey = S + cells, *ez = S + 2 * cells, *hx = S + 3 * cells, *hy = S + 4 * cells, *hz = S + 5 * cells;
    for (int64_t m = 0; m < nsteps; ++m) {
        const int mq = (int)(m % kQChunk);
        if (src.n > 0 && mq == 0) {
            const int64_t n = min((int64_t)kQChunk, nsteps - m) * src.n;
            for (int t = threadIdx.x; t < n; t += blockDim.x) Q[t] = q[m * src.n + t];
        }
        __syncthreads();                    // h (and Q) complete
        // e <- e + bE .* (C^T h); then the owned sources
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int x = cl[r].x;
            if (x >= cells) continue;
            const unsigned f = cl[r].f;
            const int k = (int)(f >> 12);
            T c0, c1, c2;
            curlT_f(hx, hy, hz, x, f, px, plane, c0, c1, c2);
            if (f & 64u) ex[x] = ex[x] + bEx(0, k, cl[r]) * c0;
            if (f & 128u) ey[x] = ey[x] + bEx(1, k, cl[r]) * c1;
            if (f & 256u) ez[x] = ez[x] + bEx(2, k, cl[r]) * c2;
            for (unsigned sm = smask[r]; sm; sm &= sm - 1) {
                const int s = __ffs(sm) - 1;
                S[src.c[s] * cells + x] = S[src.c[s] * cells + x] - Q[mq * src.n + s];
            }
        }
        __syncthreads();
        // h <- h - bH .* (C e)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int x = cl[r].x;
            if (x >= cells) continue;
            const unsigned f = cl[r].f;
            T c0, c1, c2;
            curl_f(ex, ey, ez, x, f, px, plane, c0, c1, c2);
            if (f & 512u) hx[x] = hx[x] - bHx(0, cl[r]) * c0;
            if (f & 1024u) hy[x] = hy[x] - bHx(1, cl[r]) * c1;
            if (f & 2048u) hz[x] = hz[x] - bHx(2, cl[r]) * c2;
        }
    }
    __syncthreads();
    store_state(D, st, S, cells);
}

// ---------------------------------------------------------------------------------------
// polynomial propagator: b <- p(X)^s b (all substeps, all pair ops) in one launch
// ---------------------------------------------------------------------------------------
struct SmallOps {
    int n;
    int kind[kSmallMaxOps];
    double a[kSmallMaxOps], b[kSmallMaxOps], e2[kSmallMaxOps], c[kSmallMaxOps];
};

// out = X in at an owned cell (e rows: bE C^T h, h rows: -bH C e; dead DOFs 0)
// CF (optional): the beta values staged in shared memory [bE0 bE1 bE2 bH0 bH1 bH2][cells]
template <typename T, int EM, bool HA, bool STG>
__device__ __forceinline__ void small_applyX(const Coef<T, EM, HA> &cf, const T *CF, const T *in, int cells,
                                             const SmallCell &c, int px, int plane, T o[6]) {
    const int x = c.x, k = (int)(c.f >> 12);
    T a0, a1, a2, b0, b1, b2;
    curlT_f(in + 3 * cells, in + 4 * cells, in + 5 * cells, x, c.f, px, plane, a0, a1, a2);
    curl_f(in, in + cells, in + 2 * cells, x, c.f, px, plane, b0, b1, b2);
    auto be = [&](int q) -> T { return STG ? CF[q * cells + x] : cf.bE(q, k, c.g); };
    auto bh = [&](int q) -> T { return STG ? CF[(3 + q) * cells + x] : cf.bH(q, c.g); };
    o[0] = (c.f & 64u) ? be(0) * a0 : T(0);
    o[1] = (c.f & 128u) ? be(1) * a1 : T(0);
    o[2] = (c.f & 256u) ? be(2) * a2 : T(0);
    o[3] = (c.f & 512u) ? -(bh(0) * b0) : T(0);
    o[4] = (c.f & 1024u) ? -(bh(1) * b1) : T(0);
    o[5] = (c.f & 2048u) ? -(bh(2) * b2) : T(0);
}

// y (the Newton sum) stays in registers: thread t owns cells t, t + 1024, ... (R of them)
template <typename T, int EM, bool HA, int R, bool STG>
__global__ void __launch_bounds__(kSmallThreads, 1) poly_small_kernel(Dev<T> D, Coef<T, EM, HA> cf,
                                                                      T *__restrict__ st, int s,
                                                                      const __grid_constant__ SmallOps ops) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *W = reinterpret_cast<T *>(smem_raw);
    const int cells = D.nx * D.ny * D.nz, px = D.nx, plane = D.nx * D.ny;
    T *U = W + 6 * cells;
    T *CF = U + 6 * cells;                         // staged betas (STG: EM 2 / HA, when they fit)
    load_state(D, st, W, cells);
    SmallCell cl[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int x = threadIdx.x + r * kSmallThreads;
        cl[r] = small_cell(D, x < cells ? x : 0);
        cl[r].x = x;
        if (STG && x < cells) {
            const int k = (int)(cl[r].f >> 12);
            for (int c = 0; c < 3; ++c) {
                CF[c * cells + x] = cf.bE(c, k, cl[r].g);
                CF[(3 + c) * cells + x] = cf.bH(c, cl[r].g);
            }
        }
    }
    __syncthreads();
    T y[R][6];
    for (int q = 0; q < s; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < 6; ++c) y[r][c] = T(0);
        for (int o = 0; o < ops.n; ++o) {
            const T a = (T)ops.a[o], b = (T)ops.b[o], e2 = (T)ops.e2[o], cc = (T)ops.c[o];
            const int kind = ops.kind[o];
#pragma unroll
            for (int r = 0; r < R; ++r) {                 // U = X W
                if (cl[r].x >= cells) continue;
                T u[6];
                small_applyX<T, EM, HA, STG>(cf, CF, W, cells, cl[r], px, plane, u);
#pragma unroll
                for (int c = 0; c < 6; ++c) U[c * cells + cl[r].x] = u[c];
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int x = cl[r].x;
                if (x >= cells) continue;
                T xu[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
                if (kind != 1) small_applyX<T, EM, HA, STG>(cf, CF, U, cells, cl[r], px, plane, xu);   // X U (U neighbours)
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    const T wv = W[c * cells + x], uv = U[c * cells + x];
                    T yn = (y[r][c] + a * wv) + b * uv;
                    if (kind == 2) yn = yn + cc * (xu[c] + e2 * wv);
                    y[r][c] = yn;
                    if (kind == 0) W[c * cells + x] = xu[c] + e2 * wv;   // own cell only: safe in place
                }
            }
            __syncthreads();
        }
        // b <- y (the next substep's start vector)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int x = cl[r].x;
            if (x >= cells) continue;
#pragma unroll
            for (int c = 0; c < 6; ++c) W[c * cells + x] = y[r][c];
        }
        __syncthreads();
    }
    store_state(D, st, W, cells);
}

// ---------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------
int k_leapfrog_small(const KernelArgs &ka, void *state, int64_t nsteps, int nsrc, const void *q_dev) {
    if (nsteps <= 0) return PARAEXP_OK;
    const Grid &g = *ka.g;
    if (nsrc > 16) return fail(PARAEXP_EINVAL, "small leapfrog: at most 16 sources");
    SmallSrc sl;
    sl.n = nsrc;
    for (int r = 0; r < nsrc; ++r) {
        sl.c[r] = g.h_src[r].comp;
        sl.i[r] = g.h_src[r].i;
        sl.j[r] = g.h_src[r].j;
        sl.k[r] = g.h_src[r].k;
    }
    return with_types(g, 1.0, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        constexpr int R = (int)(small_max_cells<T>() / kSmallThreads);
        constexpr size_t nv = (EM == 2 || HA) ? 12 : 6;   // state (+ staged coefficients)
        const size_t smem = (nv * g.nx * g.ny * g.nz + (size_t)kQChunk * nsrc) * sizeof(T);
        auto kern = leapfrog_small_kernel<T, EM, HA, R>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, kSmallThreads, smem, (cudaStream_t)ka.stream>>>(make_dev<T>(g), make_coef<T, EM, HA>(g, 1.0),
                                                                   (T *)state, nsteps, sl, (const T *)q_dev);
        ++*ka.launches;
        return check_cuda("leapfrog small");
    });
}

int k_poly_small(const KernelArgs &ka, const Plan &plan, void *state) {
    if (plan.s <= 0) return PARAEXP_OK;
    if ((int)plan.ops.size() > kSmallMaxOps) return fail(PARAEXP_EINVAL, "small poly: too many ops");
    SmallOps ops;
    ops.n = (int)plan.ops.size();
    for (int o = 0; o < ops.n; ++o) {
        ops.kind[o] = plan.ops[o].kind;
        ops.a[o] = plan.ops[o].a;
        ops.b[o] = plan.ops[o].b;
        ops.e2[o] = plan.ops[o].e2;
        ops.c[o] = plan.ops[o].c;
    }
    const Grid &g = *ka.g;
    return with_types(g, plan.sigma, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        constexpr int R = (int)(small_max_cells<T>() / kSmallThreads);
        const size_t cells = (size_t)g.nx * g.ny * g.nz;
        const bool stage = (EM == 2 || HA) && 18 * cells * sizeof(T) <= kSmallSmemMax;
        const size_t smem = (stage ? 18 : 12) * cells * sizeof(T);
        auto kern = stage ? poly_small_kernel<T, EM, HA, R, (EM == 2 || HA)> : poly_small_kernel<T, EM, HA, R, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmemMax);
        kern<<<1, kSmallThreads, smem, (cudaStream_t)ka.stream>>>(make_dev<T>(g), make_coef<T, EM, HA>(g, plan.sigma),
                                                                   (T *)state, plan.s, ops);
        ++*ka.launches;
        return check_cuda("poly small");
    });
}

}  // namespace pe
