// kernels_common.cuh -- device-side views of the grid (layout, liveness, coefficients),
// curl helpers and the (dtype, material mode) dispatcher shared by kernels.cu / fused.cu.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>
#include <utility>

#include "internal.h"

namespace pe {

// Layout view.  Liveness rules (reading 5) inside the stored box i<nx, j<ny, k<nz:
//   e_x live iff j>0 && k>0;  e_y iff i>0 && k>0;  e_z iff i>0 && j>0   (PEC box walls)
//   h_x live iff i>0;  h_y iff j>0;  h_z iff k>0                         (box-normal faces)
// Interior PEC cells are encoded by cE = 0 (material mode ARRAY only).
template <typename T>
// ---- debug checks: built into libparaexp_debug.so (python paper_1705_08019_b200/build.py --debug,
// -DPARAEXP_DEBUG_CHECKS); compute-sanitizer is closed on this GPU pool, so out-of-range global
// stores, ring / stage indices out of their shared-memory planes and mbarrier waits that never
// complete trap with a message instead.  Compiled out of the product library.
#ifdef PARAEXP_DEBUG_CHECKS
#include <cstdio>
#define PE_CHECK(cond, what)                                                                        \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("paraexp debug check failed: %s at %s:%d (block %d, thread %d)\n", what, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                   \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define PE_CHECK(cond, what) \
    do {                     \
    } while (0)
#endif

struct Dev {
    int nx, ny, nz;
    int64_t px, plane, cs;
    // a store of components [c0, c0 + n) at element offset `off` of a state vector stays inside it
    __host__ __device__ __forceinline__ bool in_state(int64_t off) const { return off >= 0 && off < 6 * cs; }
    __host__ __device__ __forceinline__ int64_t idx(int i, int j, int k) const {
        return (int64_t)i + px * ((int64_t)j + (int64_t)ny * k);
    }
    __host__ __device__ __forceinline__ bool e_live(int c, int i, int j, int k) const {
        return c == 0 ? (j > 0 && k > 0) : (c == 1 ? (i > 0 && k > 0) : (i > 0 && j > 0));
    }
    __host__ __device__ __forceinline__ bool h_live(int c, int i, int j, int k) const {
        return c == 0 ? (i > 0) : (c == 1 ? (j > 0) : (k > 0));
    }
};

template <typename T>
inline Dev<T> make_dev(const Grid &g) {
    Dev<T> D;
    D.nx = g.nx;
    D.ny = g.ny;
    D.nz = g.nz;
    D.px = g.L.px;
    D.plane = g.L.plane;
    D.cs = g.L.cs;
    return D;
}

// Coefficients of X = sigma*dt*A_orig: beta_E = fl_T(cE_T * sigma_T), beta_H likewise
// (DESIGN reading 24: one documented multiplication order, mirrored by the oracle).
// EM: 0 scalar per component, 1 per (component, k) table, 2 per-edge array.
// HA: per-face cH array.
template <typename T, int EM, bool HA>
struct Coef {
    T sig;
    T cEs[3], cHs[3];
    const T *__restrict__ tab;
    const T *__restrict__ cEa;
    const T *__restrict__ cHa;
    int64_t cs;
    int nz;
    __device__ __forceinline__ T cE(int c, int k, int64_t idx) const {
        if (EM == 0) return cEs[c];
        if (EM == 1) return __ldg(tab + c * nz + k);
        return __ldg(cEa + c * cs + idx);
    }
    __device__ __forceinline__ T cH(int c, int64_t idx) const {
        if (!HA) return cHs[c];
        return __ldg(cHa + c * cs + idx);
    }
    __device__ __forceinline__ T bE(int c, int k, int64_t idx) const { return cE(c, k, idx) * sig; }
    __device__ __forceinline__ T bH(int c, int64_t idx) const { return cH(c, idx) * sig; }
    __device__ __forceinline__ bool e_alive(int c, int64_t idx) const {
        if (EM == 2) return __ldg(cEa + c * cs + idx) != T(0);
        return true;
    }
};

template <typename T, int EM, bool HA>
inline Coef<T, EM, HA> make_coef(const Grid &g, double sigma) {
    Coef<T, EM, HA> c;
    c.sig = (T)sigma;
    for (int q = 0; q < 3; ++q) {
        c.cEs[q] = (T)g.cE_scalar[q];
        c.cHs[q] = (T)g.cH_scalar[q];
    }
    c.tab = (const T *)g.d_cE_tab;
    c.cEa = (const T *)g.d_cE_arr;
    c.cHa = (const T *)g.d_cH_arr;
    c.cs = g.L.cs;
    c.nz = g.nz;
    return c;
}

// (C e) at (i,j,k): +1 neighbours, 0 outside the box.
template <typename T>
__device__ __forceinline__ void curl_at(const Dev<T> &D, const T *__restrict__ ex,
                                        const T *__restrict__ ey, const T *__restrict__ ez,
                                        int i, int j, int k, int64_t idx, T &c0, T &c1, T &c2) {
    const T ex0 = ex[idx], ey0 = ey[idx], ez0 = ez[idx];
    const bool ip = i + 1 < D.nx, jp = j + 1 < D.ny, kp = k + 1 < D.nz;
    const T ez_jp = jp ? ez[idx + D.px] : T(0);
    const T ex_jp = jp ? ex[idx + D.px] : T(0);
    const T ey_kp = kp ? ey[idx + D.plane] : T(0);
    const T ex_kp = kp ? ex[idx + D.plane] : T(0);
    const T ez_ip = ip ? ez[idx + 1] : T(0);
    const T ey_ip = ip ? ey[idx + 1] : T(0);
    c0 = ((ey0 + ez_jp) - ey_kp) - ez0;
    c1 = ((ez0 + ex_kp) - ez_ip) - ex0;
    c2 = ((ex0 + ey_ip) - ex_jp) - ey0;
}

// (C^T h) at (i,j,k): -1 neighbours, 0 outside the box.
template <typename T>
__device__ __forceinline__ void curlT_at(const Dev<T> &D, const T *__restrict__ hx,
                                         const T *__restrict__ hy, const T *__restrict__ hz,
                                         int i, int j, int k, int64_t idx, T &c0, T &c1,
                                         T &c2) {
    const T hx0 = hx[idx], hy0 = hy[idx], hz0 = hz[idx];
    const T hz_jm = j > 0 ? hz[idx - D.px] : T(0);
    const T hx_jm = j > 0 ? hx[idx - D.px] : T(0);
    const T hy_km = k > 0 ? hy[idx - D.plane] : T(0);
    const T hx_km = k > 0 ? hx[idx - D.plane] : T(0);
    const T hz_im = i > 0 ? hz[idx - 1] : T(0);
    const T hy_im = i > 0 ? hy[idx - 1] : T(0);
    c0 = ((hz0 - hz_jm) - hy0) + hy_km;
    c1 = ((hx0 - hx_km) - hz0) + hz_im;
    c2 = ((hy0 - hy_im) - hx0) + hx_jm;
}

// block-wide sum for blocks of up to 1024 threads (any 1-3D shape)
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) sh[tid >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (tid < 32) {
        r = tid < (nthr + 31) / 32 ? sh[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    return r;   // valid in thread 0
}

// Early termination (f2): called by every thread at kernel start; true => return at once.
// Thread 0 of each block evaluates the criterion on the norms of the two previous ops (all
// blocks see the same values, so they agree); block 0 records the decision / the count.
__device__ __forceinline__ bool et_skip(const EtDev &et) {
    __shared__ int s_skip;
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        int skip = *(volatile int *)et.done;
        if (!skip && et.op >= 2) {
            const double d1 = et.norms[2 * (et.op - 1)], y1 = et.norms[2 * (et.op - 1) + 1];
            const double d2 = et.norms[2 * (et.op - 2)], y2 = et.norms[2 * (et.op - 2) + 1];
            if (d1 <= et.eps2 * y1 && d2 <= et.eps2 * y2) skip = 1;
        }
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
            if (skip) *et.done = 1;
            else atomicAdd(et.count, et.apps);
        }
        s_skip = skip;
    }
    __syncthreads();
    return s_skip != 0;
}

// Dispatch on (dtype, material mode, h-array):  fn(T{}, integral_constant<EM>, bool_constant<HA>)
template <typename Fn>
int with_types(const Grid &g, double /*sigma*/, Fn &&fn) {
    auto by_mode = [&](auto tT) -> int {
        switch (g.mat_mode * 2 + (g.h_array ? 1 : 0)) {
            case 0: return fn(tT, std::integral_constant<int, 0>{}, std::false_type{});
            case 1: return fn(tT, std::integral_constant<int, 0>{}, std::true_type{});
            case 2: return fn(tT, std::integral_constant<int, 1>{}, std::false_type{});
            case 3: return fn(tT, std::integral_constant<int, 1>{}, std::true_type{});
            case 4: return fn(tT, std::integral_constant<int, 2>{}, std::false_type{});
            default: return fn(tT, std::integral_constant<int, 2>{}, std::true_type{});
        }
    };
    if (g.dtype == PARAEXP_F64) return by_mode(double{});
    return by_mode(float{});
}

}  // namespace pe
