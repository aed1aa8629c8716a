// small.cu -- single-CTA, shared-memory-resident kernels for small grids (sm_100a).
//
// A grid of up to ~2k cells (fp64) / ~4k cells (fp32) -- the paper's 2-D wave (40 x 40 x 1 cells),
// C1 (8^3) -- fits one CTA's shared memory.  Stepping it with one kernel launch per time step
// (or per Newton pair) is launch-bound (~4-6 us per launch for microseconds of work), so here ONE
// CTA keeps the state in shared memory and runs a whole leapfrog sequence (rows a2/a3) or a whole
// polynomial propagator p(X)^s (row a6) in a single launch, with __syncthreads between the curl
// half-sweeps.  Arithmetic, operation order and liveness are those of the unfused kernels in
// kernels.cu (the same curl helpers on a compact view of the layout), so results match them and
// the oracle at the north_star tolerances.  Independent problems (ParaExp's sub-interval sweeps)
// run as independent single-CTA launches on separate streams, i.e. concurrently on separate SMs.
#include <cuda_runtime.h>

#include "internal.h"
#include "kernels_common.cuh"

namespace pe {

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxOps = 80;   // pair ops per substep (m <= 150 -> 75)

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

// compact (shared-memory) view of the stored box: px = nx, plane = nx*ny, cs = cells
template <typename T>
__device__ __forceinline__ Dev<T> compact(const Dev<T> &D) {
    Dev<T> C = D;
    C.px = D.nx;
    C.plane = (int64_t)D.nx * D.ny;
    C.cs = C.plane * D.nz;
    return C;
}

// ---------------------------------------------------------------------------------------
// leapfrog: nsteps steps on the state (device layout) in place
// ---------------------------------------------------------------------------------------
template <typename T, int EM, bool HA>
__global__ void __launch_bounds__(kSmallThreads, 1) leapfrog_small_kernel(Dev<T> D, Coef<T, EM, HA> cf,
                                                                          T *__restrict__ st, int64_t nsteps,
                                                                          SmallSrc src, const T *__restrict__ q) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *S = reinterpret_cast<T *>(smem_raw);
    const Dev<T> C = compact(D);
    const int cells = (int)C.cs;
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            S[c * cells + x] = st[c * D.cs + D.idx(i, j, k)];
        }
    __syncthreads();
    T *ex = S, *ey = S + cells, *ez = S + 2 * cells, *hx = S + 3 * cells, *hy = S + 4 * cells, *hz = S + 5 * cells;
    for (int64_t m = 0; m < nsteps; ++m) {
        // e <- e + bE .* (C^T h)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            const int64_t g = D.idx(i, j, k);
            T c0, c1, c2;
            curlT_at(C, hx, hy, hz, i, j, k, (int64_t)x, c0, c1, c2);
            if (D.e_live(0, i, j, k)) ex[x] = ex[x] + cf.bE(0, k, g) * c0;
            if (D.e_live(1, i, j, k)) ey[x] = ey[x] + cf.bE(1, k, g) * c1;
            if (D.e_live(2, i, j, k)) ez[x] = ez[x] + cf.bE(2, k, g) * c2;
        }
        __syncthreads();
        if (threadIdx.x == 0)       // e_s <- e_s - q[m][s], sequentially in s
            for (int r = 0; r < src.n; ++r) {
                const int x = src.i[r] + D.nx * (src.j[r] + D.ny * src.k[r]);
                S[src.c[r] * cells + x] = S[src.c[r] * cells + x] - q[m * src.n + r];
            }
        __syncthreads();
        // h <- h - bH .* (C e)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            const int64_t g = D.idx(i, j, k);
            T c0, c1, c2;
            curl_at(C, ex, ey, ez, i, j, k, (int64_t)x, c0, c1, c2);
            if (D.h_live(0, i, j, k)) hx[x] = hx[x] - (T(1) * cf.bH(0, g)) * c0;
            if (D.h_live(1, i, j, k)) hy[x] = hy[x] - (T(1) * cf.bH(1, g)) * c1;
            if (D.h_live(2, i, j, k)) hz[x] = hz[x] - (T(1) * cf.bH(2, g)) * c2;
        }
        __syncthreads();
    }
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            st[c * D.cs + D.idx(i, j, k)] = S[c * cells + x];
        }
}

// ---------------------------------------------------------------------------------------
// polynomial propagator: b <- p(X)^s b (all substeps, all pair ops) in one launch
// ---------------------------------------------------------------------------------------
struct SmallOps {
    int n;
    int kind[kSmallMaxOps];
    double a[kSmallMaxOps], b[kSmallMaxOps], e2[kSmallMaxOps], c[kSmallMaxOps];
};

// y (the Newton sum) stays in registers: thread t owns cells t, t + 1024, ... (R of them)
template <typename T, int EM, bool HA, int R>
__global__ void __launch_bounds__(kSmallThreads, 1) poly_small_kernel(Dev<T> D, Coef<T, EM, HA> cf,
                                                                      T *__restrict__ st, int s,
                                                                      const __grid_constant__ SmallOps ops) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *W = reinterpret_cast<T *>(smem_raw);
    const Dev<T> C = compact(D);
    const int cells = (int)C.cs;
    T *U = W + 6 * cells;
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            W[c * cells + x] = st[c * D.cs + D.idx(i, j, k)];
        }
    __syncthreads();
    auto applyX = [&](const T *in, T *out, int x) {       // out(x) = X in at cell x
        const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
        const int64_t g = D.idx(i, j, k);
        T a0, a1, a2, b0, b1, b2;
        curlT_at(C, in + 3 * cells, in + 4 * cells, in + 5 * cells, i, j, k, (int64_t)x, a0, a1, a2);
        curl_at(C, in, in + cells, in + 2 * cells, i, j, k, (int64_t)x, b0, b1, b2);
        out[x] = D.e_live(0, i, j, k) ? cf.bE(0, k, g) * a0 : T(0);
        out[cells + x] = D.e_live(1, i, j, k) ? cf.bE(1, k, g) * a1 : T(0);
        out[2 * cells + x] = D.e_live(2, i, j, k) ? cf.bE(2, k, g) * a2 : T(0);
        out[3 * cells + x] = D.h_live(0, i, j, k) ? -(cf.bH(0, g) * b0) : T(0);
        out[4 * cells + x] = D.h_live(1, i, j, k) ? -(cf.bH(1, g) * b1) : T(0);
        out[5 * cells + x] = D.h_live(2, i, j, k) ? -(cf.bH(2, g) * b2) : T(0);
    };
    T y[R][6];
    for (int q = 0; q < s; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < 6; ++c) y[r][c] = T(0);
        for (int o = 0; o < ops.n; ++o) {
            const T a = (T)ops.a[o], b = (T)ops.b[o], e2 = (T)ops.e2[o], cl = (T)ops.c[o];
            const int kind = ops.kind[o];
            for (int x = threadIdx.x; x < cells; x += blockDim.x) applyX(W, U, x);   // U = X W
            __syncthreads();
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int x = threadIdx.x + r * kSmallThreads;
                if (x >= cells) continue;
                T xu[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
                if (kind != 1) {                          // X U at the own cell (U neighbours)
                    const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
                    const int64_t g = D.idx(i, j, k);
                    T a0, a1, a2, b0, b1, b2;
                    curlT_at(C, U + 3 * cells, U + 4 * cells, U + 5 * cells, i, j, k, (int64_t)x, a0, a1, a2);
                    curl_at(C, U, U + cells, U + 2 * cells, i, j, k, (int64_t)x, b0, b1, b2);
                    xu[0] = D.e_live(0, i, j, k) ? cf.bE(0, k, g) * a0 : T(0);
                    xu[1] = D.e_live(1, i, j, k) ? cf.bE(1, k, g) * a1 : T(0);
                    xu[2] = D.e_live(2, i, j, k) ? cf.bE(2, k, g) * a2 : T(0);
                    xu[3] = D.h_live(0, i, j, k) ? -(cf.bH(0, g) * b0) : T(0);
                    xu[4] = D.h_live(1, i, j, k) ? -(cf.bH(1, g) * b1) : T(0);
                    xu[5] = D.h_live(2, i, j, k) ? -(cf.bH(2, g) * b2) : T(0);
                }
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    const T wv = W[c * cells + x], uv = U[c * cells + x];
                    T yn = (y[r][c] + a * wv) + b * uv;
                    if (kind == 2) yn = yn + cl * (xu[c] + e2 * wv);
                    y[r][c] = yn;
                    if (kind == 0) W[c * cells + x] = xu[c] + e2 * wv;   // own cell only: safe in place
                }
            }
            __syncthreads();
        }
        // b <- y (the next substep's start vector)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int x = threadIdx.x + r * kSmallThreads;
            if (x >= cells) continue;
#pragma unroll
            for (int c = 0; c < 6; ++c) W[c * cells + x] = y[r][c];
        }
        __syncthreads();
    }
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x % D.nx, j = (x / D.nx) % D.ny, k = x / (D.nx * D.ny);
            st[c * D.cs + D.idx(i, j, k)] = W[c * cells + x];
        }
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
        const size_t smem = (size_t)6 * g.nx * g.ny * g.nz * sizeof(T);
        auto kern = leapfrog_small_kernel<T, EM, HA>;
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
        const size_t smem = (size_t)12 * g.nx * g.ny * g.nz * sizeof(T);
        auto kern = poly_small_kernel<T, EM, HA, R>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, kSmallThreads, smem, (cudaStream_t)ka.stream>>>(make_dev<T>(g), make_coef<T, EM, HA>(g, plan.sigma),
                                                                   (T *)state, plan.s, ops);
        ++*ka.launches;
        return check_cuda("poly small");
    });
}

}  // namespace pe
