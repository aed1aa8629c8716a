// mid.cu -- multi-CTA, shared-memory-resident leapfrog for mid-size grids (sm_100a).
//
// Grids of ~2k .. ~280k cells (fp64; ~450k fp32) -- C2 (64^3), the L2-resident end of the C5
// sweep -- are too small for the z-marching TMA kernels to reach HBM speed (a launch per leapfrog
// step costs ~4-8 us of latency for ~1 us of traffic) and too large for one CTA's shared memory
// (small.cu).  But the whole state fits the AGGREGATE shared memory of the 148 SMs (64^3 fp64:
// 12.6 MB of 33 MB).  So ONE cooperative launch runs a whole leapfrog sequence (rows a2/a3):
//
//  * CTA c (one per SM, at most #SMs) owns a box of whole x-rows: i in [0, nx), j in
//    [j0, j0 + by), k in [k0, k0 + bz); the box's 6-component state lives in its shared memory
//    for the whole launch, per-edge / per-face coefficients in registers;
//  * the curls need one neighbour across each y / z box face: C^T h reads h_x, h_z at j - 1 and
//    h_x, h_y at k - 1; C e reads e_x, e_z at j + 1 and e_x, e_y at k + 1.  After every curl
//    half a CTA writes just those face values of its box to a global exchange buffer (L2) as
//    tagged 16-byte lines (value bits + epoch tag in every 8-byte half, NCCL's LL idea), and
//    before its next half it polls its neighbours' lines until their tags show the epoch,
//    staging them into shared-memory halos.  No flags, fences or grid barriers: the data
//    carries its own readiness, and only neighbours synchronise;
//  * a CTA computes its face rows first and publishes each face cell straight from registers,
//    then its interior rows while those faces travel;
//  * exchange slots alternate by epoch parity.  Every CTA reads all the faces it needs of epoch
//    t - 1 (staging ends at a __syncthreads before any face store of epoch t), and the cells
//    that publish towards a neighbour are the cells that read that neighbour's faces, so a
//    neighbour has read the slot epoch t overwrites (epoch t - 2's) before it published the
//    epoch t - 1 faces this CTA just read: a slot is never overwritten while still needed.
//
// Measured (B200, tools/mid_bench.py): 64^3 fp64 5.1 us per leapfrog step against 8.2 us with
// the TMA kernels (48^3 3.2 vs 6.6, 32^3 2.3 vs 4.6).  A polynomial (Newton pair) variant with
// W, U in shared memory and the Newton sum in registers was built and measured slower than the
// TMA pair kernel (64^3 fp64 12 vs 6 us per A-application: the per-edge betas and the Newton
// sum do not fit the registers left beside 5 cells per thread, and a stage of L2 round trips
// per epoch remains), so the propagators stay on the TMA kernels.
//
// Arithmetic, operand order and liveness are those of small.cu / the unfused kernels (the same
// curl expressions), so results match the oracle at the north_star tolerances.  Cooperative
// launch guarantees that all CTAs are co-resident (a requirement of the neighbour polls); a
// poll that does not complete within ~2^24 tries traps instead of hanging the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <type_traits>

#include "internal.h"
#include "kernels_common.cuh"

namespace pe {

constexpr int kMidThreads = 384;   // 12 warps: 3 per SM sub-partition -> up to 168 registers
constexpr size_t kMidSmemMax = 232448;   // 227 KB opt-in shared memory per CTA

template <typename T>
constexpr int mid_R() {                  // owned cells per thread
    return sizeof(T) == 8 ? 5 : 8;
}
template <typename T>
constexpr int mid_cap() {                // cells per CTA (fp64 1920, fp32 3072)
    return kMidThreads * mid_R<T>();
}

// flag bits of an owned cell: neighbours exist (i-1, j-1, k-1, i+1, j+1, k+1), e / h live
// (bits 6-8 / 9-11), neighbour across a box face (remote: read from the halo of that CTA's
// face), the cell lies in a face row (bit 16), k in bits 17-31 (so nz < 2^15)
enum : unsigned {
    F_IM = 1u, F_JM = 2u, F_KM = 4u, F_IP = 8u, F_JP = 16u, F_KP = 32u,
    F_RJM = 1u << 12, F_RKM = 1u << 13, F_RJP = 1u << 14, F_RKP = 1u << 15, F_FACE = 1u << 16
};
constexpr int kKShift = 17;   // k in bits 17-31

struct MidGeo {
    int by, bz, nby, nbz, ncta;
    int fj, fk;          // face cells: nx*bz (y faces), nx*by (z faces)
    int slot, xstride;   // 16-byte lines per exchange slot and per CTA (2 slots)
    int nlmax;           // cells of the largest box (nx*by*bz)
};

// Exchange lines (NCCL's "LL" idea): a face cell's two values travel in 16-byte lines whose
// 32-bit halves each carry the epoch tag next to 32 data bits -- {v0, tag, v1, tag} (fp32) or
// {lo v0, tag, hi v0, tag}, {lo v1, tag, hi v1, tag} (fp64).  A 16-byte store is seen whole or
// not at all per 8-byte half, so a reader that finds the tag in both halves has the data: no
// separate flag, fence or flag round trip.  Tags are unique per launch (a per-grid counter).
template <typename T>
constexpr int mid_lines() {
    return sizeof(T) == 8 ? 2 : 1;
}
// regions of a slot (in lines): JM = (e_x, e_z) of row j0 (read by the j-1 neighbour), KM =
// (e_x, e_y) of plane k0, JP = (h_x, h_z) of row j0+by-1, KP = (h_x, h_y) of plane k0+bz-1
template <typename T>
__host__ __device__ __forceinline__ int region_off(const MidGeo &g, int r) {
    const int L = mid_lines<T>();
    return r == 0 ? 0 : r == 1 ? g.fj * L : r == 2 ? (g.fj + g.fk) * L : (2 * g.fj + g.fk) * L;
}

struct MidBox {
    int c, j0, k0, byc, bzc, nl, plane;
    int nb[4];   // CTA ids of the j-1, k-1, j+1, k+1 neighbours, -1 at the domain boundary
};

template <typename T>
__device__ __forceinline__ MidBox mid_box(const MidGeo &mg, const Dev<T> &D) {
    MidBox b;
    b.c = blockIdx.x;
    const int cy = b.c % mg.nby, cz = b.c / mg.nby;
    b.j0 = cy * mg.by;
    b.k0 = cz * mg.bz;
    b.byc = min(mg.by, D.ny - b.j0);
    b.bzc = min(mg.bz, D.nz - b.k0);
    b.plane = D.nx * b.byc;
    b.nl = b.plane * b.bzc;
    b.nb[0] = cy > 0 ? b.c - 1 : -1;
    b.nb[1] = cz > 0 ? b.c - mg.nby : -1;
    b.nb[2] = cy + 1 < mg.nby ? b.c + 1 : -1;
    b.nb[3] = cz + 1 < mg.nbz ? b.c + mg.nby : -1;
    return b;
}

// per owned cell, computed once per launch: local index x, flags, face indices
// (i + nx*kk for the y faces in bits 0-15, i + nx*jj for the z faces in bits 16-31)
struct MidCell {
    int x;
    unsigned f, fi;
};

// Cell of the box assigned to slot `sl` (= threadIdx.x + r * kMidThreads): slots enumerate the
// box's rows (whole x-rows) FACE ROWS FIRST -- the rows on the box's y / z boundary, whose cells
// read the halos and are published to the neighbours -- then the interior rows, so that a CTA
// computes and publishes its faces at the start of an epoch and its interior while those faces
// travel (x = the cell's natural local index, i + nx*(jj + byc*kk)).
template <typename T>
__device__ __forceinline__ MidCell mid_cell(const Dev<T> &D, const MidBox &b, int sl, int &g) {
    const int i = sl % D.nx, rho = sl / D.nx;
    const int by = b.byc, bz = b.bzc;
    int jj, kk;
    if (bz == 1) {
        jj = rho;
        kk = 0;
    } else if (rho < by) {
        jj = rho;
        kk = 0;
    } else if (rho < 2 * by) {
        jj = rho - by;
        kk = bz - 1;
    } else {
        const int w = by > 1 ? 2 : 1;                 // face rows per interior plane: jj = 0, by - 1
        const int r2 = rho - 2 * by;
        if (r2 < (bz - 2) * w) {
            kk = 1 + r2 / w;
            jj = (r2 % w == 0) ? 0 : by - 1;
        } else {
            const int r3 = r2 - (bz - 2) * w;          // interior rows (by > 2 here)
            kk = 1 + r3 / (by - 2);
            jj = 1 + r3 % (by - 2);
        }
    }
    MidCell c;
    c.x = i + D.nx * (jj + by * kk);
    PE_CHECK(jj >= 0 && jj < by && kk >= 0 && kk < bz && c.x < b.nl, "mid cell slot");
    const int j = b.j0 + jj, k = b.k0 + kk;
    g = (int)D.idx(i, j, k);
    c.f = (unsigned)(i > 0) | ((unsigned)(j > 0) << 1) | ((unsigned)(k > 0) << 2) |
          ((unsigned)(i + 1 < D.nx) << 3) | ((unsigned)(j + 1 < D.ny) << 4) | ((unsigned)(k + 1 < D.nz) << 5);
    for (int q = 0; q < 3; ++q) {
        c.f |= (unsigned)D.e_live(q, i, j, k) << (6 + q);
        c.f |= (unsigned)D.h_live(q, i, j, k) << (9 + q);
    }
    if (jj == 0 && j > 0) c.f |= F_RJM;
    if (kk == 0 && k > 0) c.f |= F_RKM;
    if (jj == by - 1 && j + 1 < D.ny) c.f |= F_RJP;
    if (kk == bz - 1 && k + 1 < D.nz) c.f |= F_RKP;
    if (jj == 0 || jj == by - 1 || kk == 0 || kk == bz - 1) c.f |= F_FACE;
    c.f |= (unsigned)k << kKShift;
    c.fi = (unsigned)(i + D.nx * kk) | ((unsigned)(i + D.nx * jj) << 16);
    return c;
}

// Values made opaque to the compiler once per epoch: otherwise it hoists every owned cell's
// shared-memory addresses out of the time loop and spills them (measured: 300 B per thread)
__device__ __forceinline__ unsigned opaque(unsigned v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}
// a cell record whose flags the compiler cannot precompute (it would keep every flag bit of
// every owned cell in its own register across the time loop)
__device__ __forceinline__ MidCell opaque(const MidCell &c) {
    MidCell o;
    o.x = c.x;
    o.f = opaque(c.f);
    o.fi = opaque(c.fi);
    return o;
}

// ---- line exchange ----------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_line(const uint4 *p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_line(uint4 *p, unsigned a, unsigned tag, unsigned b) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(tag), "r"(b), "r"(tag)
                 : "memory");
}

// Publish this CTA's faces of the 6-component vector V (shared memory, component stride NL) into
// its slot `sl` with `tag`: lo = the e faces towards the j-1 / k-1 neighbours (JM: e_x, e_z of
// row j0; KM: e_x, e_y of plane k0), hi = the h faces towards j+1 / k+1 (JP: h_x, h_z of the
// last row; KP: h_x, h_y of the last plane).  One 16-byte line per thread and iteration.
template <typename T>
__device__ __forceinline__ void mid_publish(uint4 *sl, const MidGeo &mg, const MidBox &b, int nx, const T *V,
                                            bool lo, bool hi, unsigned tag) {
    constexpr int L = mid_lines<T>();
    const int NL = b.nl, pl = b.plane;
    const int nj = nx * b.bzc * L, nk = nx * b.byc * L;
    const int e0 = (lo && b.nb[0] >= 0) ? nj : 0;
    const int e1 = e0 + ((lo && b.nb[1] >= 0) ? nk : 0);
    const int e2 = e1 + ((hi && b.nb[2] >= 0) ? nj : 0);
    const int e3 = e2 + ((hi && b.nb[3] >= 0) ? nk : 0);
    for (int l = threadIdx.x; l < e3; l += kMidThreads) {
        const int r = l < e0 ? 0 : l < e1 ? 1 : l < e2 ? 2 : 3;
        PE_CHECK(l - (r == 0 ? 0 : r == 1 ? e0 : r == 2 ? e1 : e2) < ((r & 1) ? mg.fk : mg.fj) * L, "mid publish index");
        const int ll = l - (r == 0 ? 0 : r == 1 ? e0 : r == 2 ? e1 : e2);
        const int q = ll / L, part = ll - q * L;
        int x;
        if (r == 0) x = (q % nx) + pl * (q / nx);                              // row jj = 0
        else if (r == 1) x = q;                                                 // plane kk = 0
        else if (r == 2) x = (q % nx) + nx * (b.byc - 1) + pl * (q / nx);      // row jj = byc - 1
        else x = q + pl * (b.bzc - 1);                                          // plane kk = bzc - 1
        // component pair of the region: JM (0, 2), KM (0, 1), JP (3, 5), KP (3, 4)
        const int c0 = r < 2 ? 0 : 3, c1 = c0 + ((r & 1) ? 1 : 2);
        uint4 *p = sl + region_off<T>(mg, r) + ll;
        if (L == 1) {
            st_line(p, __float_as_uint((float)V[c0 * NL + x]), tag, __float_as_uint((float)V[c1 * NL + x]));
        } else {
            const unsigned long long a =
                (unsigned long long)__double_as_longlong((double)V[(part ? c1 : c0) * NL + x]);
            st_line(p, (unsigned)a, tag, (unsigned)(a >> 32));
        }
    }
}

// A face cell's values straight from registers into this CTA's slot `sl`: e values towards the
// j-1 / k-1 neighbours (JM: e_x, e_z; KM: e_x, e_y), h values towards j+1 / k+1 (JP: h_x, h_z;
// KP: h_x, h_y).  Safe right after the cell is computed: every halo read of the epoch ended at
// the barrier that followed the staging.
__device__ __forceinline__ void put_pair(uint4 *p, float v0, float v1, unsigned tag) {
    st_line(p, __float_as_uint(v0), tag, __float_as_uint(v1));
}
__device__ __forceinline__ void put_pair(uint4 *p, double v0, double v1, unsigned tag) {
    const unsigned long long a = (unsigned long long)__double_as_longlong(v0);
    const unsigned long long c = (unsigned long long)__double_as_longlong(v1);
    st_line(p, (unsigned)a, tag, (unsigned)(a >> 32));
    st_line(p + 1, (unsigned)c, tag, (unsigned)(c >> 32));
}
template <typename T>
__device__ __forceinline__ void put_e_faces(uint4 *sl, const MidGeo &mg, const MidCell &c, T e0, T e1, T e2,
                                            unsigned tag) {
    constexpr int L = mid_lines<T>();
    PE_CHECK((int)(c.fi & 0xffffu) < mg.fj && (int)(c.fi >> 16) < mg.fk, "mid face index");
    if (c.f & F_RJM) put_pair(sl + region_off<T>(mg, 0) + (int)(c.fi & 0xffffu) * L, e0, e2, tag);
    if (c.f & F_RKM) put_pair(sl + region_off<T>(mg, 1) + (int)(c.fi >> 16) * L, e0, e1, tag);
}
template <typename T>
__device__ __forceinline__ void put_h_faces(uint4 *sl, const MidGeo &mg, const MidCell &c, T h0, T h1, T h2,
                                            unsigned tag) {
    constexpr int L = mid_lines<T>();
    if (c.f & F_RJP) put_pair(sl + region_off<T>(mg, 2) + (int)(c.fi & 0xffffu) * L, h0, h2, tag);
    if (c.f & F_RKP) put_pair(sl + region_off<T>(mg, 3) + (int)(c.fi >> 16) * L, h0, h1, tag);
}

// Halo buffers in shared memory: H[0] = the j-1 neighbour's (h_x, h_z), H[1] = the k-1
// neighbour's (h_x, h_y), H[2] = the j+1 neighbour's (e_x, e_z), H[3] = the k+1 neighbour's
// (e_x, e_y); component 0 at [q], component 1 at [stride + q] (stride fj for 0/2, fk for 1/3).
template <typename T>
struct Halo {
    T *h[4];
};

// Stage the neighbours' faces of epoch `tag` (slot `sidx`) into the halos: every thread issues
// up to 4 line loads at a time, then re-polls those whose tags are not there yet.  lo: the j-1 / k-1
// neighbours' faces, hi: the j+1 / k+1 neighbours'.  A poll that never completes traps.
template <typename T>
__device__ __forceinline__ void mid_stage(const uint4 *xb, const MidGeo &mg, const MidBox &b, int nx, unsigned sidx,
                                          unsigned tag, bool lo, bool hi, const Halo<T> &H) {
    constexpr int L = mid_lines<T>();
    constexpr int B = 4;
    const int nj = nx * b.bzc * L, nk = nx * b.byc * L;   // lines per y / z face of this box
    // segment ends (cumulative): j-1, k-1, j+1, k+1 neighbours
    const int e0 = (lo && b.nb[0] >= 0) ? nj : 0;
    const int e1 = e0 + ((lo && b.nb[1] >= 0) ? nk : 0);
    const int e2 = e1 + ((hi && b.nb[2] >= 0) ? nj : 0);
    const int e3 = e2 + ((hi && b.nb[3] >= 0) ? nk : 0);
    // the neighbour's region facing us: JP of j-1, KP of k-1, JM of j+1, KM of k+1
    const size_t so = (size_t)sidx * mg.slot;
    const uint4 *src0 = xb + (size_t)max(b.nb[0], 0) * mg.xstride + so + region_off<T>(mg, 2);
    const uint4 *src1 = xb + (size_t)max(b.nb[1], 0) * mg.xstride + so + region_off<T>(mg, 3) - e0;
    const uint4 *src2 = xb + (size_t)max(b.nb[2], 0) * mg.xstride + so + region_off<T>(mg, 0) - e1;
    const uint4 *src3 = xb + (size_t)max(b.nb[3], 0) * mg.xstride + so + region_off<T>(mg, 1) - e2;
    for (int base = threadIdx.x; base < e3; base += kMidThreads * B) {
        uint4 v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int l = base + u * kMidThreads;
            if (l < e3) {
                const uint4 *p = l < e0 ? src0 + l : l < e1 ? src1 + l : l < e2 ? src2 + l : src3 + l;
                v[u] = ld_line(p);
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int l = base + u * kMidThreads;
            if (l >= e3) continue;
            const int r = l < e0 ? 0 : l < e1 ? 1 : l < e2 ? 2 : 3;
            unsigned polls = 0;
            while (v[u].y != tag || v[u].w != tag) {
                if (++polls > (1u << 24)) {
                    printf("paraexp mid kernel: block %d: face line of neighbour %d never reached tag %u\n",
                           (int)blockIdx.x, r, tag);
                    __trap();
                }
                const uint4 *p = r == 0 ? src0 + l : r == 1 ? src1 + l : r == 2 ? src2 + l : src3 + l;
                v[u] = ld_line(p);
            }
            const int ll = l - (r == 0 ? 0 : r == 1 ? e0 : r == 2 ? e1 : e2);
            const int stride = (r & 1) ? mg.fk : mg.fj;
            PE_CHECK(ll >= 0 && ll < stride * L, "mid halo index");
            T *h = r == 0 ? H.h[0] : r == 1 ? H.h[1] : r == 2 ? H.h[2] : H.h[3];
            if (L == 1) {
                h[ll] = (T)__uint_as_float(v[u].x);
                h[stride + ll] = (T)__uint_as_float(v[u].z);
            } else {
                const double d = __longlong_as_double((long long)(((unsigned long long)v[u].z << 32) | v[u].x));
                h[(ll & 1) * stride + (ll >> 1)] = (T)d;
            }
        }
    }
}

// ---- curls with halo neighbours ---------------------------------------------------------------
// (C^T h) at an owned cell: the j-1 / k-1 neighbours of box-face cells come from the halos;
// same operands and order as curlT_at
template <typename T, bool REMOTE = true>
__device__ __forceinline__ void curlT_mid(const T *hx, const T *hy, const T *hz, const MidCell &c, int nx, int pl,
                                          const Halo<T> &H, int fj, int fk, T &c0, T &c1, T &c2) {
    const int x = c.x;
    const unsigned f = c.f;
    const T hx0 = hx[x], hy0 = hy[x], hz0 = hz[x];
    T hz_jm = T(0), hx_jm = T(0), hy_km = T(0), hx_km = T(0), hz_im = T(0), hy_im = T(0);
    if (REMOTE && (f & F_RJM)) {
        const int q = (int)(c.fi & 0xffffu);
        hx_jm = H.h[0][q];
        hz_jm = H.h[0][fj + q];
    } else if (f & F_JM) {
        hz_jm = hz[x - nx];
        hx_jm = hx[x - nx];
    }
    if (REMOTE && (f & F_RKM)) {
        const int q = (int)(c.fi >> 16);
        hx_km = H.h[1][q];
        hy_km = H.h[1][fk + q];
    } else if (f & F_KM) {
        hy_km = hy[x - pl];
        hx_km = hx[x - pl];
    }
    if (f & F_IM) {
        hz_im = hz[x - 1];
        hy_im = hy[x - 1];
    }
    c0 = ((hz0 - hz_jm) - hy0) + hy_km;
    c1 = ((hx0 - hx_km) - hz0) + hz_im;
    c2 = ((hy0 - hy_im) - hx0) + hx_jm;
}

// (C e) at an owned cell: the j+1 / k+1 neighbours of box-face cells come from the halos;
// same operands and order as curl_at
template <typename T, bool REMOTE = true>
__device__ __forceinline__ void curl_mid(const T *ex, const T *ey, const T *ez, const MidCell &c, int nx, int pl,
                                         const Halo<T> &H, int fj, int fk, T &c0, T &c1, T &c2) {
    const int x = c.x;
    const unsigned f = c.f;
    const T ex0 = ex[x], ey0 = ey[x], ez0 = ez[x];
    T ez_jp = T(0), ex_jp = T(0), ey_kp = T(0), ex_kp = T(0), ez_ip = T(0), ey_ip = T(0);
    if (REMOTE && (f & F_RJP)) {
        const int q = (int)(c.fi & 0xffffu);
        ex_jp = H.h[2][q];
        ez_jp = H.h[2][fj + q];
    } else if (f & F_JP) {
        ez_jp = ez[x + nx];
        ex_jp = ex[x + nx];
    }
    if (REMOTE && (f & F_RKP)) {
        const int q = (int)(c.fi >> 16);
        ex_kp = H.h[3][q];
        ey_kp = H.h[3][fk + q];
    } else if (f & F_KP) {
        ey_kp = ey[x + pl];
        ex_kp = ex[x + pl];
    }
    if (f & F_IP) {
        ez_ip = ez[x + 1];
        ey_ip = ey[x + 1];
    }
    c0 = ((ey0 + ez_jp) - ey_kp) - ez0;
    c1 = ((ez0 + ex_kp) - ez_ip) - ex0;
    c2 = ((ex0 + ey_ip) - ex_jp) - ey0;
}

template <typename T>
__device__ __forceinline__ void mid_load(const Dev<T> &D, const MidBox &b, const T *st, T *S, int stride) {
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < b.nl; x += blockDim.x) {
            const int i = x % D.nx, jj = (x / D.nx) % b.byc, kk = x / b.plane;
            S[c * stride + x] = st[c * D.cs + D.idx(i, b.j0 + jj, b.k0 + kk)];
        }
}
template <typename T>
__device__ __forceinline__ void mid_store(const Dev<T> &D, const MidBox &b, T *st, const T *S, int stride) {
    for (int c = 0; c < 6; ++c)
        for (int x = threadIdx.x; x < b.nl; x += blockDim.x) {
            const int i = x % D.nx, jj = (x / D.nx) % b.byc, kk = x / b.plane;
            st[c * D.cs + D.idx(i, b.j0 + jj, b.k0 + kk)] = S[c * stride + x];
        }
}

// halos after `used` values of T in shared memory
template <typename T>
__device__ __forceinline__ Halo<T> mid_halo(T *S, size_t used, const MidGeo &mg) {
    Halo<T> H;
    H.h[0] = S + used;
    H.h[1] = H.h[0] + 2 * mg.fj;
    H.h[2] = H.h[1] + 2 * mg.fk;
    H.h[3] = H.h[2] + 2 * mg.fj;
    return H;
}

struct MidSrc {
    int n;
    int c[16], i[16], j[16], k[16];
};

// Coefficient registers of the leapfrog kernel: per-edge betas (EM 2) and per-face betas (HA)
// are loaded once per launch; scalar / z-table betas are formed on the fly as in Coef
template <typename T, int EM, bool HA, int R>
struct MidCoef {
    T e[EM == 2 ? R : 1][3];
    T h[HA ? R : 1][3];
};

// ---------------------------------------------------------------------------------------
// leapfrog: nsteps steps on the state (device layout) in place.  Epoch 2m+1: stage the lower
// neighbours' h faces, e <- e + bE C^T h (then the owned sources), publish the e faces; epoch
// 2m+2: stage the upper neighbours' e faces, h <- h - bH C e, publish the h faces.  Epoch 0
// publishes the initial h faces.  Epoch t's faces go to slot t & 1 with tag tag0 + t.
// ---------------------------------------------------------------------------------------
// TR: also the f1 trace per step (paraexp.h): energy E_{m+1} = dt [sum e'^2 / cE + sum h h' / cH]
// over the live DOFs (per-thread fp64 partials, one block reduction and one atomicAdd per CTA
// per step, as K1r-TR) and the probe values e^(m+1) written by the owning thread.
template <typename T, int EM, bool HA, int R, bool TR>
__global__ void __launch_bounds__(kMidThreads, 1)
    leapfrog_mid_kernel(Dev<T> D, Coef<T, EM, HA> cf, MidGeo mg, T *__restrict__ st, int64_t nsteps, MidSrc src,
                        const T *__restrict__ q, uint4 *xb, unsigned tag0, TraceDev tr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *S = reinterpret_cast<T *>(smem_raw);
    const MidBox b = mid_box(mg, D);
    const int NL = b.nl, nx = D.nx, pl = b.plane;
    T *ex = S, *ey = S + NL, *ez = S + 2 * NL, *hx = S + 3 * NL, *hy = S + 4 * NL, *hz = S + 5 * NL;
    const Halo<T> H = mid_halo(S, (size_t)6 * mg.nlmax, mg);
    uint4 *mine = xb + (size_t)b.c * mg.xstride;
    mid_load(D, b, st, S, NL);
    MidCell cl[R];
    MidCoef<T, EM, HA, R> co;
    unsigned smask[R];
    unsigned pmask[TR ? R : 1];   // probes at the cell (TR)
    double eacc = 0.0;            // this step's energy partial (TR)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int sl = threadIdx.x + r * kMidThreads;
        int g = 0;
        cl[r] = mid_cell(D, b, sl < NL ? sl : 0, g);
        if (sl >= NL) cl[r].x = NL;   // no cell
        const int x = cl[r].x;
        smask[r] = 0;
        if (TR) pmask[TR ? r : 0] = 0;
        if (x < NL) {
            const int i = x % nx, j = b.j0 + (x / nx) % b.byc, k = b.k0 + x / pl;
            for (int s = 0; s < src.n; ++s)
                if (src.i[s] == i && src.j[s] == j && src.k[s] == k) smask[r] |= 1u << s;
            if (TR)
                for (int s = 0; s < tr.np; ++s)
                    if (tr.i[s] == i && tr.j[s] == j && tr.k[s] == k) pmask[TR ? r : 0] |= 1u << s;
        }
        if (EM == 2)
            for (int c = 0; c < 3; ++c) co.e[EM == 2 ? r : 0][c] = cf.bE(c, 0, g);
        if (HA)
            for (int c = 0; c < 3; ++c) co.h[HA ? r : 0][c] = T(1) * cf.bH(c, g);
    }
    __syncthreads();
    mid_publish(mine, mg, b, nx, S, false, true, tag0);   // epoch 0: the initial h faces
    // per-cell updates; `pub` = publish the cell's faces from registers (face pass)
    auto e_cell = [&](int r, int64_t m, uint4 *sl, unsigned tag, auto remote) {
        const MidCell c = opaque(cl[r]);
        const int x = c.x;
        const unsigned f = c.f;
        T c0, c1, c2;
        curlT_mid<T, decltype(remote)::value>(hx, hy, hz, c, nx, pl, H, mg.fj, mg.fk, c0, c1, c2);
        T e[3] = {ex[x], ey[x], ez[x]};
        const T cc[3] = {c0, c1, c2};
#pragma unroll
        for (int q3 = 0; q3 < 3; ++q3) {
            const T be = EM == 2 ? co.e[EM == 2 ? r : 0][q3] : cf.bE(q3, (int)(f >> kKShift), 0);
            if (f & (64u << q3)) e[q3] = e[q3] + be * cc[q3];
        }
        for (unsigned sm = smask[r]; sm; sm &= sm - 1) {
            const int s = __ffs(sm) - 1;
            const T qv = __ldg(q + m * src.n + s);
            const int sc = src.c[s];
            if (sc == 0) e[0] = e[0] - qv;
            else if (sc == 1) e[1] = e[1] - qv;
            else e[2] = e[2] - qv;
        }
        ex[x] = e[0];
        ey[x] = e[1];
        ez[x] = e[2];
        if (sl) put_e_faces(sl, mg, c, e[0], e[1], e[2], tag);
        if (TR) {
#pragma unroll
            for (int q3 = 0; q3 < 3; ++q3) {
                const T be = EM == 2 ? co.e[EM == 2 ? r : 0][q3] : cf.bE(q3, (int)(f >> kKShift), 0);
                if (be != T(0)) eacc += (double)e[q3] * (double)e[q3] / (double)be;
            }
            for (unsigned pm = pmask[TR ? r : 0]; pm; pm &= pm - 1) {
                const int s = __ffs(pm) - 1;
                tr.probe[m * tr.np + s] = (double)e[tr.c[s]];
            }
        }
    };
    auto h_cell = [&](int r, uint4 *sl, unsigned tag, auto remote) {
        const MidCell c = opaque(cl[r]);
        const int x = c.x;
        const unsigned f = c.f;
        T c0, c1, c2;
        curl_mid<T, decltype(remote)::value>(ex, ey, ez, c, nx, pl, H, mg.fj, mg.fk, c0, c1, c2);
        T h[3] = {hx[x], hy[x], hz[x]};
        const T cc[3] = {c0, c1, c2};
#pragma unroll
        for (int q3 = 0; q3 < 3; ++q3) {
            const T bh = HA ? co.h[HA ? r : 0][q3] : T(1) * cf.bH(q3, 0);
            if (f & (512u << q3)) {
                const T hn = h[q3] - bh * cc[q3];
                if (TR && bh != T(0)) eacc += (double)h[q3] * (double)hn / (double)bh;
                h[q3] = hn;
            }
        }
        hx[x] = h[0];
        hy[x] = h[1];
        hz[x] = h[2];
        if (sl) put_h_faces(sl, mg, c, h[0], h[1], h[2], tag);
    };
    unsigned t = 1;
#pragma unroll 1
    for (int64_t m = 0; m < nsteps; ++m, t += 2) {
        // ---- e half (epoch t): stage the lower neighbours' h faces; face rows first (computed
        // and published at once), then the interior while the faces travel
        mid_stage(xb, mg, b, nx, (t - 1) & 1u, tag0 + t - 1, true, false, H);
        __syncthreads();
        {
            uint4 *sl = mine + (size_t)(t & 1u) * mg.slot;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (cl[r].x < NL && (cl[r].f & F_FACE)) e_cell(r, m, sl, tag0 + t, std::true_type{});
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (cl[r].x < NL && !(cl[r].f & F_FACE)) e_cell(r, m, nullptr, 0u, std::false_type{});
        }
        __syncthreads();
        // ---- h half (epoch t + 1): the upper neighbours' e faces
        mid_stage(xb, mg, b, nx, t & 1u, tag0 + t, false, true, H);
        __syncthreads();
        {
            uint4 *sl = mine + (size_t)((t + 1) & 1u) * mg.slot;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (cl[r].x < NL && (cl[r].f & F_FACE)) h_cell(r, sl, tag0 + t + 1, std::true_type{});
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (cl[r].x < NL && !(cl[r].f & F_FACE)) h_cell(r, nullptr, 0u, std::false_type{});
        }
        if (TR && tr.energy) {   // this step's energy: one block reduction, one atomic per CTA
            const double sum = block_sum(eacc);
            if (threadIdx.x == 0 && sum != 0.0) atomicAdd(tr.energy + m, sum * tr.dt);
            eacc = 0.0;
        }
        __syncthreads();
    }
    mid_store(D, b, st, S, NL);
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
int device_sm_count() {   // of the current device (cached per device)
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

// shared memory of the kernel: the 6-component state of the box and the four halos
static size_t mid_smem(const MidGeo &mg, size_t esize) {
    return ((size_t)6 * mg.nlmax + 4 * (size_t)(mg.fj + mg.fk)) * esize;
}

// Box partition of the (y, z) rows: at most one CTA per SM, at most mid_cap cells per box, the
// shared memory within the opt-in limit; among those, the least cells per
// box plus face cells (the per-epoch work), ties -> fewer CTAs.
static bool mid_partition(int nx, int ny, int nz, int cap, int nsm, size_t esize, MidGeo &mg) {
    if (nx > cap) return false;
    double best = 1e300;
    bool ok = false;
    for (int by = 1; by <= ny; ++by) {
        if ((int64_t)nx * by > cap) break;
        for (int bz = 1; bz <= nz; ++bz) {
            const int64_t cells = (int64_t)nx * by * bz;
            if (cells > cap) break;
            const int nby = (ny + by - 1) / by, nbz = (nz + bz - 1) / bz;
            if ((int64_t)nby * nbz > nsm) continue;
            MidGeo t;
            t.nlmax = (int)cells;
            t.fj = nx * bz;
            t.fk = nx * by;
            if (mid_smem(t, esize) > kMidSmemMax) continue;
            const double cost = (double)cells + (double)nx * (by + bz) + 1e-3 * nby * nbz;
            if (cost < best) {
                best = cost;
                ok = true;
                mg.by = by;
                mg.bz = bz;
                mg.nby = nby;
                mg.nbz = nbz;
            }
        }
    }
    if (!ok) return false;
    mg.ncta = mg.nby * mg.nbz;
    mg.fj = nx * mg.bz;
    mg.fk = nx * mg.by;
    mg.nlmax = nx * mg.by * mg.bz;
    return true;
}

static bool mid_geo(const Grid &g, MidGeo &mg, int max_cta) {
    const bool f64 = g.dtype == PARAEXP_F64;
    const int cap = f64 ? mid_cap<double>() : mid_cap<float>();
    const int64_t cells = (int64_t)g.nx * g.ny * g.nz;
    const int nsm = max_cta > 0 ? std::min(max_cta, device_sm_count()) : device_sm_count();
    if (cells > (int64_t)cap * nsm || g.nz >= (1 << 15)) return false;   // k in 15 flag bits
    if (!mid_partition(g.nx, g.ny, g.nz, cap, nsm, g.esize(), mg)) return false;
    const int L = f64 ? mid_lines<double>() : mid_lines<float>();
    mg.slot = 2 * (mg.fj + mg.fk) * L;
    mg.xstride = 2 * mg.slot;
    return true;
}

bool mid_supported(const Grid &g, int max_cta) {
    static const bool off = [] {
        const char *e = getenv("PARAEXP_NO_MID");
        return e && atoi(e) != 0;
    }();
    if (off || g.kernels != PARAEXP_KERNELS_FUSED || small_supported(g)) return false;
    int coop = 0, dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess || !coop) return false;
    MidGeo mg;
    return mid_geo(g, mg, max_cta);
}

// exchange lines (2 slots per CTA), grid-owned, grown on demand and zeroed (tag 0 is never
// used); the launch's tag base comes from a per-grid counter so that lines left by earlier
// launches never match -- on wrap-around the buffer is zeroed again
static int mid_buffers(Grid &G, int slot, const MidGeo &mg, int64_t epochs, void *stream, uint4 **xb,
                       unsigned *tag0) {
    if (slot < 0 || slot >= Grid::kMidSlots) return fail(PARAEXP_EINVAL, "mid kernels: bad buffer slot");
    const size_t need = (size_t)mg.ncta * mg.xstride * sizeof(uint4);
    int rc;
    bool zero = false;
    if ((size_t)G.mid_bytes[slot] < need) {
        dev_free(G.d_mid[slot]);
        G.d_mid[slot] = nullptr;
        G.device_bytes -= G.mid_bytes[slot];
        G.mid_bytes[slot] = 0;
        if ((rc = dev_alloc(&G.d_mid[slot], need))) return rc;
        G.mid_bytes[slot] = (int64_t)need;
        G.device_bytes += (int64_t)need;
        zero = true;
    }
    uint32_t &tag = G.mid_tag[slot];
    if (tag == 0 || (uint64_t)tag + (uint64_t)epochs + 2 > 0x7fffffffull) zero = true;
    if (zero) {
        if ((rc = dev_memset_async(G.d_mid[slot], 0, (size_t)G.mid_bytes[slot], stream))) return rc;
        tag = 1;
    }
    if ((uint64_t)epochs + 2 > 0x7ffffff0ull) return fail(PARAEXP_EINVAL, "mid kernels: too many epochs in one launch");
    *tag0 = (unsigned)tag;
    tag += (uint32_t)(epochs + 2);
    *xb = (uint4 *)G.d_mid[slot];
    return PARAEXP_OK;
}

int k_leapfrog_mid(const KernelArgs &ka, void *state, int64_t nsteps, int nsrc, const void *q_dev,
                   const TraceDev *tr) {
    if (nsteps <= 0) return PARAEXP_OK;
    Grid &g = *const_cast<Grid *>(ka.g);
    if (nsrc > 16) return fail(PARAEXP_EINVAL, "mid leapfrog: at most 16 sources");
    MidGeo mg;
    if (!mid_geo(g, mg, ka.mid_max_cta)) return fail(PARAEXP_EINVAL, "mid leapfrog: grid does not fit");
    MidSrc sl;
    sl.n = nsrc;
    for (int r = 0; r < nsrc; ++r) {
        sl.c[r] = g.h_src[r].comp;
        sl.i[r] = g.h_src[r].i;
        sl.j[r] = g.h_src[r].j;
        sl.k[r] = g.h_src[r].k;
    }
    uint4 *xb = nullptr;
    unsigned tag0 = 0;
    int rc = mid_buffers(g, ka.mid_slot, mg, 2 * nsteps + 1, ka.stream, &xb, &tag0);
    if (rc) return rc;
    return with_types(g, 1.0, [&](auto tT, auto tEM, auto tHA) {
        using T = decltype(tT);
        constexpr int EM = decltype(tEM)::value;
        constexpr bool HA = decltype(tHA)::value;
        constexpr int R = mid_R<T>();
        const size_t smem = mid_smem(mg, sizeof(T));
        const bool trace = tr && (tr->energy || (tr->probe && tr->np > 0));
        auto kern = trace ? leapfrog_mid_kernel<T, EM, HA, R, true> : leapfrog_mid_kernel<T, EM, HA, R, false>;
        TraceDev trm;
        if (trace) {
            trm = *tr;
            if (!trm.probe) trm.np = 0;
        }
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        Dev<T> D = make_dev<T>(g);
        Coef<T, EM, HA> cf = make_coef<T, EM, HA>(g, 1.0);
        T *st = (T *)state;
        const T *q = (const T *)q_dev;
        void *args[] = {&D, &cf, &mg, &st, &nsteps, &sl, &q, &xb, &tag0, &trm};
        if (cudaLaunchCooperativeKernel((const void *)kern, dim3(mg.ncta), dim3(kMidThreads), args, smem,
                                        (cudaStream_t)ka.stream) != cudaSuccess)
            return check_cuda("leapfrog mid (cooperative launch)");
        ++*ka.launches;
        return check_cuda("leapfrog mid");
    });
}

}  // namespace pe
