// internal.h -- shared declarations of the paraexp-b200 library (not part of the ABI).
//
// Device layout:
//   Every live DOF of the canonical layout lies in i < nx, j < ny, k < nz (each component's
//   live range per axis is [0,n) or [1,n)), so the device stores exactly one cell-indexed
//   array per component:  idx(i,j,k) = i + px*(j + ny*k),  px = nx rounded up to 128 B.
//   A state vector is 6 components [ex, ey, ez, hx, hy, hz], component stride `cs`.
//   Entries with i >= nx (x padding) and every dead DOF are kept at exactly 0.
#pragma once
#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>

#include "../../include/paraexp.h"

typedef struct CUstream_st *cudaStream_t_;

namespace pe {

struct Layout {
    int nx, ny, nz;
    int64_t px;     // x pitch in elements
    int64_t plane;  // px*ny
    int64_t cs;     // component stride = plane*nz
    int64_t state_elems() const { return 6 * cs; }
};

struct SrcDev {       // one source edge in device layout
    int64_t off;      // element offset into the state vector (component + idx)
    int32_t comp, i, j, k;
};

struct Grid {
    int nx, ny, nz;
    int dtype;          // PARAEXP_F64 / F32
    int device;         // -1 host only
    int kernels;        // resolved PARAEXP_KERNELS_*
    int mat_mode;       // PARAEXP_MAT_*
    bool h_array;       // per-face cH array
    double dt, dt_cfl, rho_cfl, rho_pow;
    int warnings;
    Layout L;
    int64_t npts;
    // host fp64 coefficients, canonical layout (3*npts each)
    std::vector<double> cE64, cH64;
    // compact host tables (fp64): scalar per comp, or per (comp, k)
    double cE_scalar[3], cH_scalar[3];
    std::vector<double> cE_ztab;   // 3*nz
    // device buffers
    void *d_cE_tab = nullptr;   // 3*nz of T (ztable)
    void *d_cE_arr = nullptr;   // 3*cs of T (array)
    void *d_cH_arr = nullptr;   // 3*cs of T (array-H)
    // workspace (state vectors)
    std::vector<void *> ws;     // each 6*cs elements of T
    int64_t ws_bytes = 0;
    void *d_flag = nullptr;     // int device flag (non-finite)
    void *d_red = nullptr;      // double reduction scratch
    void *d_src = nullptr;      // source descriptors
    std::vector<SrcDev> h_src;  // host copy of the current source descriptors
    void *d_q = nullptr;        // source amplitude table
    void *d_canon[2] = {nullptr, nullptr};   // canonical-layout staging of host-pointer fields
    std::vector<void *> kry;    // Krylov basis vectors (f3), allocated on first use
    void *d_et = nullptr;       // early-termination norms / flags (f2)
    std::vector<void *> conc;   // state buffers of concurrently swept sub-intervals
    std::vector<void *> streams; // their cudaStream_t / cudaEvent_t handles (created on demand)
    std::vector<void *> events;
    void *d_norms = nullptr;    // per-propagator energy norms of a solve (rho safety net, f. intervals)
    void *call_event = nullptr; // recorded at the end of every call (stream order across calls)
    void *call_stream = nullptr;
    // mid.cu: tagged face-exchange lines of the resident leapfrog, one set per slot (slot 0:
    // the caller's stream; slots 1..8: concurrently swept sub-intervals), and per slot the next
    // epoch-tag base of a launch (0: the buffer is not zeroed yet)
    static constexpr int kMidSlots = 9;
    void *d_mid[kMidSlots] = {};
    int64_t mid_bytes[kMidSlots] = {};
    uint32_t mid_tag[kMidSlots] = {};
    void *d_sched = nullptr;    // monotone unit counter of the fused kernels' dynamic schedule
    unsigned long long sched_base = 0;   // host shadow: value of *d_sched before the next launch
    int64_t d_q_cap = 0;
    int64_t device_bytes = 0;
    size_t esize() const { return dtype == PARAEXP_F64 ? 8 : 4; }
};

// ---- errors ----
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
void grid_free_device(Grid &G);
int grid_create(const paraexp_grid_desc *d, paraexp_grid **out);

// ---- plan ----
struct Op {              // one conjugate pair of the real Newton schedule (readings 28-29)
    int kind;            // 0 pair: u = Xw; y += a w + b u; w <- Xu + e2 w
                         // 1 half (m = 1): u = Xw; y += a w + b u
                         // 2 last pair: u = Xw; y += a w + b u + c (Xu + e2 w)
    double a, b, e2, c;
};
struct Plan {
    int method, m, s;
    double tau, rho, a, gamma, sigma;
    std::vector<double> xi;        // Leja sequence on [-1,1]
    std::vector<double> node_im;   // Im of capacity-scaled nodes 2*xi (Leja), empty (Taylor)
    std::vector<double> d_re, d_im;
    std::vector<Op> ops;
    bool early_term = false;       // f2: stop a substep on two small consecutive increments
    double eps_A = 0;
};
int make_plan(int method, int m, int s, double eps_A, double tau, double rho, double dt,
              Plan &out);
void leja_sequence(int count, std::vector<double> &xi);
double theta_m(int method, int m, double tol);
void plan_to_info(const Plan &p, paraexp_plan_info *out);

// ---- device entry points (kernels.cu) ----
int dev_alloc(void **p, size_t bytes);
void dev_free(void *p);
int dev_memset_async(void *p, int v, size_t bytes, void *stream);
int dev_memcpy_h2d_async(void *dst, const void *src, size_t bytes, void *stream);
int dev_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream);
int dev_memcpy_d2d_async(void *dst, const void *src, size_t bytes, void *stream);
int dev_set_device(int device);
int dev_sync(void *stream);
int dev_stream_create(void **s);
void dev_stream_destroy(void *s);
int dev_event_create(void **e);
void dev_event_destroy(void *e);
int dev_stream_after(void *waiter, void *from, void *ev);
int check_cuda(const char *what);

// early termination of the Newton sum (f2; reading 18): per op the kernels accumulate the
// energy norms ||delta y||^2 and ||y||^2 into norms[2 op], norms[2 op + 1]; a launch whose two
// predecessors both had ||delta|| <= eps ||y|| sets *done and returns, as do all later launches
// of the substep; *count accumulates the A-applications actually performed.
struct EtDev {
    double *norms = nullptr;   // nullptr = early termination off
    int *done = nullptr;
    int *count = nullptr;
    double eps2 = 0;
    int op = 0, apps = 0;
};

struct KernelArgs {
    const Grid *g;
    void *stream;
    int64_t *launches;
    const EtDev *et = nullptr;   // per-call early-termination buffers (op/apps set per launch)
    bool static_sched = false;   // launches that run concurrently with others: no shared counter
    int mid_slot = 0;            // mid.cu exchange-buffer slot (> 0: a concurrent sweep's own)
    int mid_max_cta = 0;         // mid.cu CTA budget (0: one per SM) for concurrent sweeps
};

// per-step trace outputs of a leapfrog sequence (f1): device pointers at the row of the
// first step; probes are e components at state offsets (comp*cs + idx).
struct TraceDev {
    double *energy = nullptr;   // one double per step (accumulated: zeroed by the caller)
    double *probe = nullptr;    // np doubles per step
    int np = 0;
    int c[PARAEXP_MAX_PROBES], i[PARAEXP_MAX_PROBES], j[PARAEXP_MAX_PROBES], k[PARAEXP_MAX_PROBES];
    int64_t off[PARAEXP_MAX_PROBES];
    double dt = 0;
};

// pack canonical (e, h) -> device state (zeroing dead DOFs); unpack the reverse.
int k_pack(const KernelArgs &ka, const void *e, const void *h, void *state);
int k_unpack(const KernelArgs &ka, const void *state, void *e, void *h);
// leapfrog: `nsteps` steps; bufs[0] = state in/out, bufs[1] = spare (fused kernels
// ping-pong; on return bufs[0] names the buffer holding the result).  q_dev points at the
// amplitude row of the first step (nsrc values per step).
// tr (optional): energy E_{m+1} and probe values e^(m+1) per step (paraexp.h trace).
int k_leapfrog(const KernelArgs &ka, void *bufs[2], int64_t nsteps, const SrcDev *src_dev,
               int nsrc, const void *q_dev, const TraceDev *tr = nullptr);
int k_leapfrog_unfused(const KernelArgs &ka, void *state, int64_t nsteps, const SrcDev *src_dev,
                       int nsrc, const void *q_dev, const TraceDev *tr = nullptr);
// h <- h + 0.5 cH (C e)  (seed sync, a4)
int k_sync(const KernelArgs &ka, void *state);
// h <- h - 0.5 cH (C e)  (staggered start, reading 11)
int k_half_start(const KernelArgs &ka, void *state);
// one substep of the polynomial: b <- p(X) b.  bufs[0] = b in/out, bufs[1..3] scratch; on
// return bufs[0] names the result and bufs[1..3] the free buffers.
int k_poly_substep(const KernelArgs &ka, const Plan &plan, void *bufs[4]);
int k_poly_substep_unfused(const KernelArgs &ka, const Plan &plan, void *bufs[4]);
// small grids (small.cu): one CTA, state in shared memory, whole sequences per launch
bool small_supported(const Grid &g);
int k_leapfrog_small(const KernelArgs &ka, void *state, int64_t nsteps, int nsrc, const void *q_dev);
int k_poly_small(const KernelArgs &ka, const Plan &plan, void *state);
// mid-size grids (mid.cu): one cooperative launch per leapfrog sequence, the state resident in
// the shared memory of up to one CTA per SM, neighbour-only face exchange through L2
bool mid_supported(const Grid &g, int max_cta = 0);
int device_sm_count();
int k_leapfrog_mid(const KernelArgs &ka, void *state, int64_t nsteps, int nsrc, const void *q_dev,
                   const TraceDev *tr = nullptr);
// the TMA z-marching kernels serve this grid (kernels FUSED = auto choice, or TMA only)
inline bool zmarch_kernels(const Grid &g) {
    return g.kernels == PARAEXP_KERNELS_FUSED || g.kernels == PARAEXP_KERNELS_TMA;
}
// x <- x + alpha y (state-sized), or over components [c0, c1)
int k_axpy(const KernelArgs &ka, void *x, const void *y, double alpha);
int k_axpy_comps(const KernelArgs &ka, void *x, const void *y, double alpha, int c0, int c1);
int k_check_finite_async(const KernelArgs &ka, const void *state, int *dflag);
// non-finite check over the state; sets *flag (device int) if any
int k_check_finite(const KernelArgs &ka, const void *state, int *host_flag);
// energy-weighted dot products for K5 Lanczos: out[0] = <x,y>_M (host, synchronous)
int k_dot_M(const KernelArgs &ka, const void *x, const void *y, double *out);
// *dout += scale * <x,y>_M / dt  (device accumulator, stream-ordered; energy with scale = dt)
int k_dot_M_async(const KernelArgs &ka, const void *x, const void *y, double *dout, double scale);
// dout[r] = state[off[r]] (as double), r < np; or 0 if zero != 0
int k_gather(const KernelArgs &ka, const void *state, const TraceDev &tr, double *dout, int zero);
// y <- sigma*dt*A_orig x  (one A-application, unfused)
int k_apply_A(const KernelArgs &ka, const void *x, void *y, double sigma);
// z <- alpha x + beta y + gamma z
int k_lincomb(const KernelArgs &ka, void *z, const void *x, const void *y, double alpha,
              double beta, double gamma);
// fill a live-masked pseudo-random state (counter-based hash, seed)
int k_fill_random(const KernelArgs &ka, void *state, uint64_t seed);

}  // namespace pe

struct paraexp_grid {
    pe::Grid g;
};
