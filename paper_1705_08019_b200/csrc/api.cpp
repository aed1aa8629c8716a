// api.cpp -- C ABI entry points: leapfrog (a2/a3), expmv (a5/a6), ParaExp solve (a4, a7-a9),
// K5 norm estimate, communicator (a8), host helpers and error handling.
// See include/paraexp.h for the contract of every function.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace pe {

// ---- errors ------------------------------------------------------------------------------
static thread_local std::string t_last_error;
void set_error(const std::string &msg) { t_last_error = msg; }
int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

// ---- workspace ---------------------------------------------------------------------------
static int ensure_ws(Grid &G, int n) {
    const size_t bytes = (size_t)G.L.state_elems() * G.esize();
    while ((int)G.ws.size() < n) {
        void *p = nullptr;
        int rc = dev_alloc(&p, bytes);
        if (rc) return rc;
        // padding entries (i >= nx) are never written by the kernels: start from zero
        if ((rc = dev_memset_async(p, 0, bytes, nullptr)) || (rc = dev_sync(nullptr))) return rc;
        G.ws.push_back(p);
        G.device_bytes += bytes;
        G.ws_bytes += bytes;
    }
    return PARAEXP_OK;
}

// ---- stream order across calls -----------------------------------------------------------
// Calls on one grid share its workspaces (ws, the source table, the schedule counter), so a
// call enqueued on another stream than the previous call first waits for the previous call's
// work (an event recorded at the end of every call).
struct CallScope {
    Grid &G;
    void *stream;
    CallScope(Grid &g, void *s) : G(g), stream(s) {
        if (G.call_event && G.call_stream != stream)
            cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)G.call_event, 0);
    }
    ~CallScope() {
        if (!G.call_event) dev_event_create(&G.call_event);
        if (G.call_event) cudaEventRecord((cudaEvent_t)G.call_event, (cudaStream_t)stream);
        G.call_stream = stream;
    }
};

// the driver's view of a communicator (rho broadcast); empty for one rank / no comm
struct CommView {
    void *ctx = nullptr;
    int (*bcast_rho)(void *ctx, double *rho, void *stream) = nullptr;
};
typedef CommView paraexp_comm_view;

// ---- concurrent particular sweeps ------------------------------------------------------------
// On by default for grids of at most 2^19 cells (64^3: one fused sweep covers ~128 (tile, chunk)
// units, far fewer than the ~444 resident CTAs); PARAEXP_CONCURRENT=0/1 forces it off/on.
static bool concurrent_sweeps(const Grid &G) {
    const char *e = getenv("PARAEXP_CONCURRENT");
    if (e) return atoi(e) != 0;
    return (int64_t)G.nx * G.ny * G.nz <= (1 << 19);
}

// ---- dynamic-schedule counter check ---------------------------------------------------------
// The fused kernels take their units from a grid-owned monotone counter whose expected value
// the host tracks (fused.cu Sched).  At points where a call synchronises anyway, verify it;
// on a mismatch (an aborted launch) reset both and report the error instead of letting later
// launches work on a shifted unit sequence.
static int sched_check(Grid &G, void *stream) {
    if (!G.d_sched) return PARAEXP_OK;
    unsigned long long v = 0;
    int rc = dev_memcpy_d2h(&v, G.d_sched, sizeof(v), stream);
    if (rc) return rc;
    if (v == G.sched_base) return PARAEXP_OK;
    dev_memset_async(G.d_sched, 0, sizeof(v), stream);
    dev_sync(stream);
    G.sched_base = 0;
    return fail(PARAEXP_ECUDA, "fused-kernel schedule counter out of step (aborted launch?); reset");
}

// ---- host or device field pointers ---------------------------------------------------------
// Field arguments may be device pointers (stream-ordered, no copy) or host pointers (pinned or
// pageable): host fields are staged through canonical-layout device buffers with
// cudaMemcpyAsync and the call synchronises its stream before returning.
static bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static int ensure_canon(Grid &G) {
    const size_t bytes = (size_t)3 * G.npts * G.esize();
    for (int q = 0; q < 2; ++q)
        if (!G.d_canon[q]) {
            int rc = dev_alloc(&G.d_canon[q], bytes);
            if (rc) return rc;
            G.device_bytes += bytes;
        }
    return PARAEXP_OK;
}

// pack (e, h) from host or device into the device state; *host_io |= any host pointer
static int pack_any(const KernelArgs &ka, Grid &G, const void *e, const void *h, void *state, bool *host_io) {
    const bool de = is_device_ptr(e), dh = is_device_ptr(h);
    if (de && dh) return k_pack(ka, e, h, state);
    int rc = ensure_canon(G);
    if (rc) return rc;
    const size_t bytes = (size_t)3 * G.npts * G.esize();
    if (!de && (rc = dev_memcpy_h2d_async(G.d_canon[0], e, bytes, ka.stream))) return rc;
    if (!dh && (rc = dev_memcpy_h2d_async(G.d_canon[1], h, bytes, ka.stream))) return rc;
    *host_io = true;
    return k_pack(ka, de ? e : G.d_canon[0], dh ? h : G.d_canon[1], state);
}

// unpack the device state into (e, h) on host or device
static int unpack_any(const KernelArgs &ka, Grid &G, const void *state, void *e, void *h, bool *host_io) {
    const bool de = is_device_ptr(e), dh = is_device_ptr(h);
    if (de && dh) return k_unpack(ka, state, e, h);
    int rc = ensure_canon(G);
    if (rc) return rc;
    const size_t bytes = (size_t)3 * G.npts * G.esize();
    if ((rc = k_unpack(ka, state, de ? e : G.d_canon[0], dh ? h : G.d_canon[1]))) return rc;
    *host_io = true;
    if (!de && cudaMemcpyAsync(e, G.d_canon[0], bytes, cudaMemcpyDeviceToHost, (cudaStream_t)ka.stream) != cudaSuccess)
        return check_cuda("memcpy d2h");
    if (!dh && cudaMemcpyAsync(h, G.d_canon[1], bytes, cudaMemcpyDeviceToHost, (cudaStream_t)ka.stream) != cudaSuccess)
        return check_cuda("memcpy d2h");
    return PARAEXP_OK;
}

// ---- sources (reading 6, 24) ---------------------------------------------------------------
static double waveform(const paraexp_source &s, double t) {
    switch (s.kind) {
        case PARAEXP_SRC_ZERO: return 0.0;
        case PARAEXP_SRC_GAUSS_PAPER: {
            const double x = (t - s.t_param) / s.t_param;
            return s.amp * std::exp(-4.0 * x * x);
        }
        case PARAEXP_SRC_GAUSS_SINE: {
            const double x = t - s.t_delay;
            const double r = x / s.t_param;
            return s.amp * std::sin(2.0 * M_PI * s.f0 * x) * std::exp(-(r * r));
        }
        case PARAEXP_SRC_SINE: return s.amp * std::sin(2.0 * M_PI * s.f0 * t);
    }
    return 0.0;
}

// validate sources and upload descriptors + the amplitude table q[m][s] for global steps
// m0 .. m0+nsteps-1:  q = fl_T(cE64_s * weight_s * i_s(t0 + (m + 1/2) dt)).
static int prepare_sources(Grid &G, const paraexp_source *src, int nsrc, double t0, int64_t m0,
                           int64_t nsteps, void *stream, std::vector<SrcDev> &sd) {
    if (nsrc < 0 || nsrc > PARAEXP_MAX_SOURCES) return fail(PARAEXP_EINVAL, "nsrc out of range");
    if (nsrc > 0 && !src) return fail(PARAEXP_EINVAL, "null sources");
    sd.resize(nsrc);
    std::vector<double> ce(nsrc);
    const int64_t NX = G.nx + 1, NY = G.ny + 1;
    for (int s = 0; s < nsrc; ++s) {
        const paraexp_source &S = src[s];
        if (S.comp < 0 || S.comp > 2 || S.i < 0 || S.j < 0 || S.k < 0 || S.i > G.nx || S.j > G.ny || S.k > G.nz)
            return fail(PARAEXP_EINVAL, "source edge out of range");
        if (S.kind < 0 || S.kind > 3) return fail(PARAEXP_EINVAL, "bad source kind");
        if ((S.kind == PARAEXP_SRC_GAUSS_PAPER || S.kind == PARAEXP_SRC_GAUSS_SINE) && !(S.t_param > 0))
            return fail(PARAEXP_EINVAL, "source t_param must be > 0");
        const double c = G.cE64[S.comp * G.npts + S.i + NX * (S.j + NY * (int64_t)S.k)];
        if (c == 0.0) return fail(PARAEXP_EINVAL, "source on a dead (PEC/virtual) edge");
        ce[s] = c;
        sd[s].comp = S.comp;
        sd[s].i = S.i;
        sd[s].j = S.j;
        sd[s].k = S.k;
        sd[s].off = S.comp * G.L.cs + S.i + G.L.px * (S.j + (int64_t)G.ny * S.k);
    }
    if (nsrc == 0 || nsteps <= 0) return PARAEXP_OK;
    const size_t es = G.esize();
    const int64_t n = nsteps * nsrc;
    std::vector<char> host(n * es);
    for (int64_t m = 0; m < nsteps; ++m)
        for (int s = 0; s < nsrc; ++s) {
            const double t = t0 + ((double)(m0 + m) + 0.5) * G.dt;
            const double q = ce[s] * (src[s].weight * waveform(src[s], t));
            if (G.dtype == PARAEXP_F64)
                reinterpret_cast<double *>(host.data())[m * nsrc + s] = q;
            else
                reinterpret_cast<float *>(host.data())[m * nsrc + s] = (float)q;
        }
    if ((int64_t)(n * es) > G.d_q_cap) {
        dev_free(G.d_q);
        G.d_q = nullptr;
        int rc = dev_alloc(&G.d_q, n * es);
        if (rc) return rc;
        G.device_bytes += n * es - G.d_q_cap;
        G.d_q_cap = n * es;
    }
    int rc = dev_memcpy_h2d_async(G.d_q, host.data(), n * es, stream);
    if (rc) return rc;
    rc = dev_memcpy_h2d_async(G.d_src, sd.data(), sizeof(SrcDev) * nsrc, stream);
    if (rc) return rc;
    G.h_src = sd;
    return dev_sync(stream);   // host staging buffers go out of scope
}

// ---- K5: Lanczos estimate of ||A||_2 -----------------------------------------------------
// Lanczos on B = -(dt A_orig)^2, self-adjoint and PSD in the energy inner product
// <x,y>_M (A = T A_orig T^-1 normal with imaginary spectrum), 60 steps
// without reorthogonalisation; rho_pow = sqrt(largest Ritz value) / dt.
static double tridiag_max_eig(const std::vector<double> &a, const std::vector<double> &b) {
    const int n = (int)a.size();
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? std::fabs(b[i - 1]) : 0) + (i + 1 < n ? std::fabs(b[i]) : 0);
        lo = std::min(lo, a[i] - r);
        hi = std::max(hi, a[i] + r);
    }
    auto count_below = [&](double x) {   // Sturm count of eigenvalues < x
        int c = 0;
        double d = 1;
        for (int i = 0; i < n; ++i) {
            d = a[i] - x - (i > 0 ? b[i - 1] * b[i - 1] / d : 0);
            if (d == 0) d = 1e-300;
            if (d < 0) ++c;
        }
        return c;
    };
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (count_below(mid) >= n) hi = mid; else lo = mid;
    }
    return hi;
}

static int compute_rho_pow(Grid &G, void *stream, int64_t *launches) {
    int rc = ensure_ws(G, 4);
    if (rc) return rc;
    KernelArgs ka{&G, stream, launches};
    void *q = G.ws[0], *qp = G.ws[1], *t = G.ws[2], *w = G.ws[3];
    if ((rc = k_fill_random(ka, q, 0x5eed1234ull))) return rc;
    if ((rc = dev_memset_async(qp, 0, G.L.state_elems() * G.esize(), stream))) return rc;
    double nn;
    if ((rc = k_dot_M(ka, q, q, &nn))) return rc;
    if (!(nn > 0)) {
        G.rho_pow = 0;
        return PARAEXP_OK;
    }
    if ((rc = k_lincomb(ka, q, q, q, 1.0 / std::sqrt(nn), 0.0, 0.0))) return rc;
    std::vector<double> al, be;
    double beta_prev = 0;
    const int K = 60;
    for (int it = 0; it < K; ++it) {
        if ((rc = k_apply_A(ka, q, t, 1.0))) return rc;   // t = dt A q
        if ((rc = k_apply_A(ka, t, w, 1.0))) return rc;   // w = (dt A)^2 q
        double alpha;
        if ((rc = k_dot_M(ka, q, w, &alpha))) return rc;
        alpha = -alpha;                                  // <q, B q>, B = -(dt A)^2
        // w <- -w - alpha q - beta_prev qp
        if ((rc = k_lincomb(ka, w, q, qp, -alpha, -beta_prev, -1.0))) return rc;
        double bb;
        if ((rc = k_dot_M(ka, w, w, &bb))) return rc;
        al.push_back(alpha);
        const double beta = std::sqrt(std::max(bb, 0.0));
        if (!(beta > 1e-14 * std::fabs(alpha)) || it == K - 1) break;
        be.push_back(beta);
        std::swap(q, qp);                                // qp <- q
        if ((rc = k_lincomb(ka, q, w, w, 1.0 / beta, 0.0, 0.0))) return rc;   // q <- w / beta
        beta_prev = beta;
    }
    be.resize(al.size() > 0 ? al.size() - 1 : 0);
    const double lmax = tridiag_max_eig(al, be);
    G.rho_pow = std::sqrt(std::max(lmax, 0.0)) / G.dt;
    return PARAEXP_OK;
}

static double default_rho(Grid &G, const paraexp_expmv_opts *o, void *stream, int64_t *launches,
                          int *rc) {
    *rc = PARAEXP_OK;
    if (o && o->rho > 0) return o->rho;
    if (G.device < 0) return G.rho_cfl;
    if (G.rho_pow == 0) {
        *rc = compute_rho_pow(G, stream, launches);
        if (*rc) return 0;
    }
    return G.rho_pow > 0 ? std::min(G.rho_cfl, 1.05 * G.rho_pow) : G.rho_cfl;
}

// ---- dispatch fused / unfused -------------------------------------------------------------
int k_leapfrog_fused(const KernelArgs &ka, void *bufs[2], int64_t nsteps, const SrcDev *src_dev,
                     int nsrc, const void *q_dev, const TraceDev *tr);
int k_poly_substep_fused(const KernelArgs &ka, const Plan &plan, void *bufs[4]);
bool fused_supported(const Grid &g);

int k_leapfrog(const KernelArgs &ka, void *bufs[2], int64_t nsteps, const SrcDev *src_dev,
               int nsrc, const void *q_dev, const TraceDev *tr) {
    const bool tracing = tr && (tr->energy || (tr->probe && tr->np > 0));
    if (ka.g->kernels == PARAEXP_KERNELS_FUSED && !tracing && nsrc <= 16 && small_supported(*ka.g))
        return k_leapfrog_small(ka, bufs[0], nsteps, nsrc, q_dev);
    // mid-size grids: one cooperative launch per sequence (mid.cu) -- over all SMs, or, for a
    // concurrently swept sub-interval, over its CTA budget with its own exchange-buffer slot
    if (ka.g->kernels == PARAEXP_KERNELS_FUSED && nsrc <= 16 && (!ka.static_sched || ka.mid_slot > 0) &&
        mid_supported(*ka.g, ka.mid_max_cta))
        return k_leapfrog_mid(ka, bufs[0], nsteps, nsrc, q_dev, tracing ? tr : nullptr);
    if (zmarch_kernels(*ka.g) && fused_supported(*ka.g))
        return k_leapfrog_fused(ka, bufs, nsteps, src_dev, nsrc, q_dev, tr);
    return k_leapfrog_unfused(ka, bufs[0], nsteps, src_dev, nsrc, q_dev, tr);
}

// validate a paraexp_trace and build its device view (probe offsets in the device layout)
static int prepare_trace(const Grid &G, const paraexp_trace *t, TraceDev &tr) {
    tr = TraceDev();
    tr.dt = G.dt;
    if (!t) return PARAEXP_OK;
    if (t->nprobe < 0 || t->nprobe > PARAEXP_MAX_PROBES) return fail(PARAEXP_EINVAL, "nprobe out of range");
    const int64_t NX = G.nx + 1, NY = G.ny + 1;
    for (int r = 0; r < t->nprobe; ++r) {
        const int c = t->comp[r], i = t->i[r], j = t->j[r], k = t->k[r];
        if (c < 0 || c > 2 || i < 0 || j < 0 || k < 0 || i > G.nx || j > G.ny || k > G.nz)
            return fail(PARAEXP_EINVAL, "probe edge out of range");
        if (G.cE64[c * G.npts + i + NX * (j + NY * (int64_t)k)] == 0.0)
            return fail(PARAEXP_EINVAL, "probe on a dead (PEC/virtual) edge");
        tr.c[r] = c;
        tr.i[r] = i;
        tr.j[r] = j;
        tr.k[r] = k;
        tr.off[r] = c * G.L.cs + i + G.L.px * (j + (int64_t)G.ny * k);
    }
    tr.np = t->probe ? t->nprobe : 0;
    tr.energy = t->energy;
    tr.probe = t->probe;
    return PARAEXP_OK;
}
int k_poly_substep(const KernelArgs &ka, const Plan &plan, void *bufs[4]) {
    if (zmarch_kernels(*ka.g) && fused_supported(*ka.g))
        return k_poly_substep_fused(ka, plan, bufs);
    return k_poly_substep_unfused(ka, plan, bufs);
}

struct Events {
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    cudaStream_t s;
    explicit Events(void *stream) : s((cudaStream_t)stream) {}
    int open(int phase) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        ev.push_back({phase, {a, b}});
        return (int)ev.size() - 1;
    }
    void close(int id) { cudaEventRecord(ev[id].second.second, s); }
    void sum(double out[7]) {
        for (auto &e : ev) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e.second.first, e.second.second);
            out[e.first] += ms;
        }
    }
    ~Events() {
        for (auto &e : ev) {
            cudaEventDestroy(e.second.first);
            cudaEventDestroy(e.second.second);
        }
    }
};

// ---- f3: Krylov (Arnoldi, sigma = infinity) ---------------------------------
// exp(H) e_1 of a small real matrix (l <= 100): scaling and squaring of a Taylor series in
// long double.
static void expm_first_column(const std::vector<long double> &H, int l, std::vector<double> &c) {
    long double nrm = 0;
    for (int i = 0; i < l; ++i) {
        long double r = 0;
        for (int j = 0; j < l; ++j) r += std::fabs(H[i * l + j]);
        nrm = std::max(nrm, r);
    }
    int sq = 0;
    while (nrm > 0.25L) {
        nrm *= 0.5L;
        ++sq;
    }
    const long double scale = std::ldexp(1.0L, -sq);
    std::vector<long double> A(l * l), E(l * l, 0.0L), T(l * l), N(l * l);
    for (int q = 0; q < l * l; ++q) A[q] = H[q] * scale;
    for (int i = 0; i < l; ++i) E[i * l + i] = 1.0L;
    T = E;
    for (int k = 1; k <= 30; ++k) {           // T <- T A / k ; E += T
        for (int i = 0; i < l; ++i)
            for (int j = 0; j < l; ++j) {
                long double acc = 0;
                for (int q = 0; q < l; ++q) acc += T[i * l + q] * A[q * l + j];
                N[i * l + j] = acc / k;
            }
        T = N;
        for (int q = 0; q < l * l; ++q) E[q] += T[q];
    }
    for (int r = 0; r < sq; ++r) {            // E <- E^2
        for (int i = 0; i < l; ++i)
            for (int j = 0; j < l; ++j) {
                long double acc = 0;
                for (int q = 0; q < l; ++q) acc += E[i * l + q] * E[q * l + j];
                N[i * l + j] = acc;
            }
        E = N;
    }
    c.resize(l);
    for (int i = 0; i < l; ++i) c[i] = (double)E[i * l + 0];
}

// One Krylov substep in place on bufs[0]: b <- ||b|| V_l exp(H_l) e_1, Arnoldi in the energy
// inner product <x,y> = sum x y / cE + sum x y / cH (k_dot_M), modified Gram-Schmidt applied
// twice.  Returns the realised dimension (happy breakdown stops early).
static int krylov_substep(const KernelArgs &ka, Grid &G, const Plan &plan, void *b, int *l_out) {
    const int l = plan.m;
    const size_t bytes = (size_t)G.L.state_elems() * G.esize();
    while ((int)G.kry.size() < l + 1) {
        void *q = nullptr;
        int rc = dev_alloc(&q, bytes);
        if (rc) return rc;
        if ((rc = dev_memset_async(q, 0, bytes, nullptr)) || (rc = dev_sync(nullptr))) return rc;
        G.kry.push_back(q);
        G.device_bytes += bytes;
    }
    int rc;
    double bb;
    if ((rc = k_dot_M(ka, b, b, &bb))) return rc;
    const double beta0 = std::sqrt(std::max(bb, 0.0));
    *l_out = 0;
    if (!(beta0 > 0)) return PARAEXP_OK;              // exp(X) 0 = 0
    std::vector<void *> V(G.kry.begin(), G.kry.begin() + l + 1);
    if ((rc = k_lincomb(ka, V[0], b, b, 1.0 / beta0, 0.0, 0.0))) return rc;
    std::vector<long double> H((size_t)l * l, 0.0L);
    int lr = l;
    double hmax = 0;
    for (int j = 0; j < l; ++j) {
        void *w = V[j + 1];
        if ((rc = k_apply_A(ka, V[j], w, plan.sigma))) return rc;     // w = X v_j
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i <= j; ++i) {
                double hij;
                if ((rc = k_dot_M(ka, V[i], w, &hij))) return rc;
                H[(size_t)i * l + j] += hij;
                hmax = std::max(hmax, std::fabs(hij));
                if ((rc = k_lincomb(ka, w, V[i], V[i], -hij, 0.0, 1.0))) return rc;
            }
        if (j + 1 == l) break;                                        // h_{l+1,l} unused
        double ww;
        if ((rc = k_dot_M(ka, w, w, &ww))) return rc;
        const double hn = std::sqrt(std::max(ww, 0.0));
        hmax = std::max(hmax, hn);
        if (!(hn > 1e-12 * hmax)) {                                   // happy breakdown:
            lr = j + 1;                                               // K_{j+1} is invariant
            break;
        }
        H[(size_t)(j + 1) * l + j] = hn;
        if ((rc = k_lincomb(ka, w, w, w, 1.0 / hn, 0.0, 0.0))) return rc;
    }
    std::vector<long double> Hr((size_t)lr * lr);
    for (int i = 0; i < lr; ++i)
        for (int j = 0; j < lr; ++j) Hr[(size_t)i * lr + j] = H[(size_t)i * l + j];
    std::vector<double> c;
    expm_first_column(Hr, lr, c);
    if ((rc = k_lincomb(ka, b, V[0], V[0], beta0 * c[0], 0.0, 0.0))) return rc;
    for (int i = 1; i < lr; ++i)
        if ((rc = k_lincomb(ka, b, V[i], V[i], beta0 * c[i], 0.0, 1.0))) return rc;
    *l_out = lr;
    return PARAEXP_OK;
}

// apply the propagator p(X)^s in place: bufs[0] in/out.  Kernel time is attributed to
// phase 6 (ms_poly_kernels) when an Events recorder is given.
static int run_plan(const KernelArgs &ka, const Plan &plan, void *bufs[4], paraexp_stats *st,
                    Events *ev = nullptr) {
    if (plan.method == PARAEXP_KRYLOV) {
        const int id = ev && plan.s > 0 ? ev->open(6) : -1;
        int64_t apps = 0;
        for (int q = 0; q < plan.s; ++q) {
            int lr = 0;
            int rc = krylov_substep(ka, *const_cast<Grid *>(ka.g), plan, bufs[0], &lr);
            if (rc) return rc;
            apps += lr;
        }
        if (id >= 0) ev->close(id);
        if (st) {
            st->a_applications += apps;
            st->substeps += plan.s;
        }
        return PARAEXP_OK;
    }
    const int id = ev && plan.s > 0 ? ev->open(6) : -1;
    if (!plan.early_term && plan.s > 0 && ka.g->kernels == PARAEXP_KERNELS_FUSED && small_supported(*ka.g) &&
        plan.ops.size() <= 80) {
        // small grid: every substep of the propagator in one single-CTA launch (small.cu)
        int rc = k_poly_small(ka, plan, bufs[0]);
        if (rc) return rc;
        if (id >= 0) ev->close(id);
        if (st) {
            st->a_applications += (int64_t)plan.s * plan.m;
            st->substeps += plan.s;
        }
        return PARAEXP_OK;
    }
    if (plan.early_term && plan.s > 0) {
        // f2: per substep the op norms and the done flag are reset; the kernels count the
        // A-applications they actually perform (reading 18)
        Grid &G = *const_cast<Grid *>(ka.g);
        const size_t nops = plan.ops.size();
        if (!G.d_et) {
            int rc = dev_alloc(&G.d_et, (2 * (PARAEXP_MAX_DEGREE + 2)) * sizeof(double) + 64);
            if (rc) return rc;
        }
        EtDev et;
        et.norms = (double *)G.d_et;
        et.done = (int *)((char *)G.d_et + 2 * (PARAEXP_MAX_DEGREE + 2) * sizeof(double));
        et.count = et.done + 1;
        et.eps2 = plan.eps_A * plan.eps_A;
        KernelArgs kb = ka;
        kb.et = &et;
        int rc = dev_memset_async(et.count, 0, sizeof(int), ka.stream);
        for (int q = 0; q < plan.s && !rc; ++q) {
            if ((rc = dev_memset_async(et.norms, 0, 2 * nops * sizeof(double), ka.stream))) break;
            if ((rc = dev_memset_async(et.done, 0, sizeof(int), ka.stream))) break;
            rc = k_poly_substep(kb, plan, bufs);
        }
        if (rc) return rc;
        if (id >= 0) ev->close(id);
        int count = 0;
        if ((rc = dev_memcpy_d2h(&count, et.count, sizeof(int), ka.stream))) return rc;
        if (st) {
            st->a_applications += count;
            st->substeps += plan.s;
        }
        return PARAEXP_OK;
    }
    for (int q = 0; q < plan.s; ++q) {
        int rc = k_poly_substep(ka, plan, bufs);
        if (rc) return rc;
    }
    if (id >= 0) ev->close(id);
    if (st) {
        st->a_applications += (int64_t)plan.s * plan.m;
        st->substeps += plan.s;
    }
    return PARAEXP_OK;
}

static int opts_plan(Grid &G, double tau, const paraexp_expmv_opts *o, double rho, Plan &plan) {
    paraexp_expmv_opts def{PARAEXP_LEJA, 0, 0, 1e-12, 0.0, 0, 0.0, 0};
    if (!o) o = &def;
    double eps = o->eps_A;
    if (eps == 0.0 && o->beta > 0) {   // eq:tolerance_leja_2 (f2, reading 30)
        int clamped = 0;
        eps = paraexp_optimal_tolerance(G.dt, o->beta, rho, &clamped);
    }
    if (o->early_term && !(eps >= 1e-14 && eps < 1)) return fail(PARAEXP_EINVAL, "early termination needs eps_A in [1e-14, 1)");
    if (o->early_term && o->method == PARAEXP_KRYLOV) return fail(PARAEXP_EINVAL, "early termination applies to Taylor/Leja");
    int rc = make_plan(o->method, o->m, o->s, eps, tau, rho, G.dt, plan);
    if (rc) return rc;
    plan.early_term = o->early_term != 0;
    plan.eps_A = eps;
    return PARAEXP_OK;
}

// rho safety net (SURVEY finding 8): on when rho came from the K5 estimate (or opts->rho_check
// > 0), never for Krylov (norm-preserving by construction) or when rho is already rho_cfl.
static void schedule_blocks(int p, int world, double ratio, bool u0, std::vector<int> &F,
                            std::vector<int> &L, int &root);
static void schedule_lpt(int p, int world, double ratio, bool u0, std::vector<int> &owner, int &root);
static int ensure_norms(Grid &G);

static bool rho_check_on(const Grid &G, const paraexp_expmv_opts *o, double rho) {
    const int mode = o ? o->rho_check : 0;
    const bool explicit_rho = o && o->rho > 0;
    if (o && o->method == PARAEXP_KRYLOV) return false;
    return (mode > 0 || (mode == 0 && !explicit_rho)) && rho < G.rho_cfl;
}
// tolerance on | ||p(X)^s b||_M / ||b||_M - 1 |: the planner bounds the forward error per
// substep by eps_A theta (reading 16), i.e. eps_A rho tau over the propagator; fixed plans
// and fp32 rounding get a floor.  A rho that misses the spectrum makes the polynomial grow
// exponentially outside the Leja interval, far beyond either bound.
static double norm_tol(const Grid &G, const Plan &P, bool auto_plan) {
    const double floor_tol = G.dtype == PARAEXP_F64 ? 1e-9 : 1e-3;
    return auto_plan ? std::max(floor_tol, 10.0 * P.eps_A * P.rho * P.tau) : std::max(floor_tol, 1e-3);
}

}  // namespace pe

// =====================================================================================
// NCCL (a8), loaded at run time
// =====================================================================================
namespace {
typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    // optional (checked at use): async error polling, abort, symmetric windows (NCCL >= 2.27)
    ncclResult_t (*GetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*MemAlloc)(void **, size_t) = nullptr;
    ncclResult_t (*MemFree)(void *) = nullptr;
    ncclResult_t (*WindowRegister)(ncclComm_t, void *, size_t, void **, int) = nullptr;
    ncclResult_t (*WindowDeregister)(ncclComm_t, void *) = nullptr;
};
NcclApi g_nccl;
const int kNcclSum = 0, kNcclF32 = 7, kNcclF64 = 8;

int load_nccl() {
    if (g_nccl.ok) return PARAEXP_OK;
    void *h = nullptr;
    const char *env = getenv("PARAEXP_NCCL_LIBRARY");
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return pe::fail(PARAEXP_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.Reduce = (decltype(g_nccl.Reduce))dlsym(h, "ncclReduce");
    g_nccl.Broadcast = (decltype(g_nccl.Broadcast))dlsym(h, "ncclBroadcast");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.GetAsyncError = (decltype(g_nccl.GetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    g_nccl.CommAbort = (decltype(g_nccl.CommAbort))dlsym(h, "ncclCommAbort");
    g_nccl.MemAlloc = (decltype(g_nccl.MemAlloc))dlsym(h, "ncclMemAlloc");
    g_nccl.MemFree = (decltype(g_nccl.MemFree))dlsym(h, "ncclMemFree");
    g_nccl.WindowRegister = (decltype(g_nccl.WindowRegister))dlsym(h, "ncclCommWindowRegister");
    g_nccl.WindowDeregister = (decltype(g_nccl.WindowDeregister))dlsym(h, "ncclCommWindowDeregister");
    if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.CommDestroy || !g_nccl.Reduce ||
        !g_nccl.Broadcast || !g_nccl.AllReduce || !g_nccl.GetErrorString)
        return pe::fail(PARAEXP_ENCCL, "libnccl.so.2 lacks required symbols");
    g_nccl.ok = true;
    return PARAEXP_OK;
}
int nccl_check(ncclResult_t r, const char *what) {
    if (r == 0) return PARAEXP_OK;
    return pe::fail(PARAEXP_ENCCL, std::string(what) + ": " + g_nccl.GetErrorString(r));
}
}  // namespace

struct paraexp_comm {
    ncclComm_t comm;
    int rank, world, device;
    bool aborted = false;
    void *win_buf = nullptr;    // ncclMemAlloc'd reduce buffer registered as a symmetric window
    size_t win_bytes = 0;
    void *win = nullptr;
};

namespace {
// Wait for `stream` while polling NCCL's asynchronous error state: a failed peer would
// otherwise leave cudaStreamSynchronize blocked forever.  On an error the communicator is
// aborted (it must then only be destroyed) and ENCCL returned.
int comm_wait(paraexp_comm *comm, void *stream) {
    for (;;) {
        const cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
        if (q == cudaSuccess) return PARAEXP_OK;
        if (q != cudaErrorNotReady) return pe::check_cuda("stream query");
        if (g_nccl.GetAsyncError && !comm->aborted) {
            ncclResult_t ae = 0;
            g_nccl.GetAsyncError(comm->comm, &ae);
            if (ae != 0 && ae != 7 /* ncclInProgress */) {
                if (g_nccl.CommAbort) g_nccl.CommAbort(comm->comm);
                comm->aborted = true;
                return pe::fail(PARAEXP_ENCCL, std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(ae));
            }
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

struct CommCtx {
    paraexp_comm *comm;
    pe::Grid *G;
};

// every rank takes rank 0's rho (the K5 estimate uses atomics and can differ in the last bits)
int bcast_rho_nccl(void *ctx, double *rho, void *stream) {
    CommCtx *c = (CommCtx *)ctx;
    double *d = (double *)c->G->d_red;
    int rc = pe::dev_memcpy_h2d_async(d, rho, sizeof(double), stream);
    if (rc) return rc;
    if ((rc = nccl_check(g_nccl.Broadcast(d, d, 1, kNcclF64, 0, c->comm->comm, (cudaStream_t)stream),
                         "ncclBroadcast(rho)"))) return rc;
    if ((rc = comm_wait(c->comm, stream))) return rc;
    return pe::dev_memcpy_d2h(rho, d, sizeof(double), stream);
}

// a8: W summed onto the root.  With PARAEXP_NCCL_WINDOW=1 the reduction runs on an
// ncclMemAlloc'd buffer registered as a symmetric window (NCCL_WIN_COLL_SYMMETRIC: lets NCCL
// use NVLS / symmetric kernels); W is staged through it with two device copies.
int comm_reduce_W(paraexp_comm *comm, const pe::Grid &G, void *W, size_t bytes, int root, void *stream) {
    const int dt = G.dtype == PARAEXP_F64 ? kNcclF64 : kNcclF32;
    const size_t n = bytes / G.esize();
    const char *w = getenv("PARAEXP_NCCL_WINDOW");
    if (w && atoi(w) != 0) {
        if (!g_nccl.MemAlloc || !g_nccl.WindowRegister)
            return pe::fail(PARAEXP_ENCCL, "PARAEXP_NCCL_WINDOW: NCCL lacks ncclMemAlloc / ncclCommWindowRegister");
        if (comm->win_bytes < bytes) {
            if (comm->win && g_nccl.WindowDeregister) g_nccl.WindowDeregister(comm->comm, comm->win);
            if (comm->win_buf && g_nccl.MemFree) g_nccl.MemFree(comm->win_buf);
            comm->win = comm->win_buf = nullptr;
            comm->win_bytes = 0;
            int rc = nccl_check(g_nccl.MemAlloc(&comm->win_buf, bytes), "ncclMemAlloc");
            if (rc) return rc;
            if ((rc = nccl_check(g_nccl.WindowRegister(comm->comm, comm->win_buf, bytes, &comm->win, 1),
                                 "ncclCommWindowRegister"))) return rc;
            comm->win_bytes = bytes;
        }
        if (cudaMemcpyAsync(comm->win_buf, W, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
            return pe::check_cuda("window stage");
        int rc = nccl_check(g_nccl.Reduce(comm->win_buf, comm->win_buf, n, dt, kNcclSum, root, comm->comm,
                                          (cudaStream_t)stream), "ncclReduce");
        if (rc) return rc;
        if (comm->rank == root &&
            cudaMemcpyAsync(W, comm->win_buf, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
            return pe::check_cuda("window unstage");
        return PARAEXP_OK;
    }
    return nccl_check(g_nccl.Reduce(W, W, n, dt, kNcclSum, root, comm->comm, (cudaStream_t)stream), "ncclReduce");
}

int comm_allreduce_trace(paraexp_comm *comm, const pe::TraceDev &tr, int p, void *stream) {
    int rc = PARAEXP_OK;
    if (tr.np > 0)
        rc = nccl_check(g_nccl.AllReduce(tr.probe, tr.probe, (size_t)p * tr.np, kNcclF64, kNcclSum, comm->comm,
                                         (cudaStream_t)stream), "ncclAllReduce");
    if (!rc && tr.energy)
        rc = nccl_check(g_nccl.AllReduce(tr.energy, tr.energy, (size_t)p, kNcclF64, kNcclSum, comm->comm,
                                         (cudaStream_t)stream), "ncclAllReduce");
    return rc;
}

// max over ranks of a local failure flag (one int, ncclAllReduce max): returns 1 if any rank
// failed, 0 if none, or a negative error code if the collective itself failed
int comm_status_any(paraexp_comm *comm, const pe::Grid &G, bool failed, void *stream) {
    const int kNcclInt32 = 2, kNcclMax = 2;
    int *d = (int *)G.d_flag + 1020;               // past the per-sub-interval flags (p <= 1000)
    const int v = failed ? 1 : 0;
    int rc = pe::dev_memcpy_h2d_async(d, &v, sizeof(int), stream);
    if (rc) return rc;
    if ((rc = nccl_check(g_nccl.AllReduce(d, d, 1, kNcclInt32, kNcclMax, comm->comm, (cudaStream_t)stream),
                         "ncclAllReduce(status)"))) return rc;
    if ((rc = comm_wait(comm, stream))) return rc;
    int any = 0;
    if ((rc = pe::dev_memcpy_d2h(&any, d, sizeof(int), stream))) return rc;
    return any;
}

int comm_bcast_state(paraexp_comm *comm, const pe::Grid &G, void *P, int root, void *stream) {
    const int dt = G.dtype == PARAEXP_F64 ? kNcclF64 : kNcclF32;
    return nccl_check(g_nccl.Broadcast(P, P, (size_t)G.L.state_elems(), dt, root, comm->comm,
                                       (cudaStream_t)stream), "ncclBroadcast");
}
}  // namespace

extern "C" {

const char *paraexp_version(void) { return "paraexp-b200 0.1 (sm_100a)"; }

const char *paraexp_strerror(int code) {
    switch (code) {
        case PARAEXP_OK: return "ok";
        case PARAEXP_EINVAL: return "invalid argument";
        case PARAEXP_ENOMEM: return "out of memory";
        case PARAEXP_ECUDA: return "CUDA error";
        case PARAEXP_ENCCL: return "NCCL error";
        case PARAEXP_EDIVERGED: return "integration diverged (non-finite field)";
        case PARAEXP_EOVERFLOW: return "exp(tA)v overflow (non-finite result; use more substeps)";
        case PARAEXP_ENOTSUP: return "not supported";
        case PARAEXP_WCFL: return "warning: dt exceeds the CFL bound";
    }
    return "unknown status";
}

const char *paraexp_last_error(void) { return pe::t_last_error.c_str(); }

int paraexp_host_alloc(size_t bytes, void **out) {
    if (!out || bytes == 0) return pe::fail(PARAEXP_EINVAL, "paraexp_host_alloc: need bytes > 0 and out != NULL");
    *out = nullptr;
    const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
    if (e == cudaSuccess) return PARAEXP_OK;
    *out = nullptr;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) return pe::fail(PARAEXP_ENOMEM, "paraexp_host_alloc: cannot pin that much host memory");
    return pe::fail(PARAEXP_ECUDA, std::string("paraexp_host_alloc: ") + cudaGetErrorString(e));
}

void paraexp_host_free(void *p) {
    if (p && cudaFreeHost(p) != cudaSuccess) cudaGetLastError();
}

int paraexp_partition(int64_t nsteps, int32_t p, int64_t *bounds) {
    if (p < 1 || nsteps < p || !bounds) return pe::fail(PARAEXP_EINVAL, "need p >= 1 and nsteps >= p");
    const int64_t M = nsteps / p;
    for (int j = 0; j < p; ++j) bounds[j] = j * M;
    bounds[p] = nsteps;
    return PARAEXP_OK;
}

int paraexp_schedule(int32_t p, int32_t world, int32_t rank, double tail_ratio, int32_t has_u0,
                     int32_t *first, int32_t *last, int32_t *root) {
    if (p < 1 || world < 1 || rank < 0 || rank >= world) return pe::fail(PARAEXP_EINVAL, "bad schedule arguments");
    std::vector<int> F, L;
    int r = 0;
    pe::schedule_blocks(p, world, tail_ratio, has_u0 != 0, F, L, r);
    if (first) *first = F[rank];
    if (last) *last = L[rank];
    if (root) *root = r;
    return PARAEXP_OK;
}

int paraexp_schedule_lpt(int32_t p, int32_t world, double tail_ratio, int32_t has_u0, int32_t *owner,
                         int32_t *root) {
    if (p < 1 || world < 1 || !owner) return pe::fail(PARAEXP_EINVAL, "bad schedule arguments");
    std::vector<int> o;
    int r = 0;
    pe::schedule_lpt(p, world, tail_ratio, has_u0 != 0, o, r);
    for (int j = 0; j <= p; ++j) owner[j] = o[j];
    if (root) *root = r;
    return PARAEXP_OK;
}

int paraexp_grid_info(paraexp_grid *grid, int32_t compute_rho_pow, void *stream,
                      paraexp_grid_info_t *o) {
    if (!grid || !o) return pe::fail(PARAEXP_EINVAL, "null argument");
    pe::Grid &G = grid->g;
    if (compute_rho_pow && G.device >= 0 && G.rho_pow == 0) {
        int64_t launches = 0;
        pe::dev_set_device(G.device);
        pe::CallScope scope(G, stream);
        int rc = pe::compute_rho_pow(G, stream, &launches);
        if (rc) return rc;
    }
    *o = paraexp_grid_info_t();
    o->nx = G.nx;
    o->ny = G.ny;
    o->nz = G.nz;
    o->dtype = G.dtype;
    o->npts = G.npts;
    o->ndof_field = 3 * G.npts;
    o->cells = (int64_t)G.nx * G.ny * G.nz;
    o->dt = G.dt;
    o->dt_cfl = G.dt_cfl;
    o->rho_cfl = G.rho_cfl;
    o->rho_pow = G.rho_pow;
    o->material_mode = G.mat_mode;
    o->kernels = G.kernels;
    o->pitch_x = G.L.px;
    o->device_bytes = G.device_bytes;
    o->device = G.device;
    o->warnings = G.warnings;
    o->leapfrog_path = -1;
    if (G.device >= 0) {
        pe::dev_set_device(G.device);
        o->leapfrog_path = G.kernels == PARAEXP_KERNELS_UNFUSED                      ? PARAEXP_PATH_UNFUSED
                           : G.kernels == PARAEXP_KERNELS_FUSED && pe::small_supported(G) ? PARAEXP_PATH_SMALL
                           : G.kernels == PARAEXP_KERNELS_FUSED && pe::mid_supported(G)   ? PARAEXP_PATH_MID
                           : pe::fused_supported(G)                                     ? PARAEXP_PATH_TMA
                                                                                        : PARAEXP_PATH_UNFUSED;
    }
    return PARAEXP_OK;
}

static int leapfrog_impl(paraexp_grid *grid, const paraexp_source *src, int32_t nsrc, double t0,
                         int64_t nsteps, void *e, void *h, int32_t check_finite,
                         const paraexp_trace *trace, void *stream, paraexp_stats *st);

int paraexp_leapfrog(paraexp_grid *grid, const paraexp_source *src, int32_t nsrc, double t0,
                     int64_t nsteps, void *e, void *h, int32_t check_finite, void *stream,
                     paraexp_stats *st) {
    return leapfrog_impl(grid, src, nsrc, t0, nsteps, e, h, check_finite, nullptr, stream, st);
}

int paraexp_leapfrog_trace(paraexp_grid *grid, const paraexp_source *src, int32_t nsrc, double t0,
                           int64_t nsteps, void *e, void *h, const paraexp_trace *trace, void *stream,
                           paraexp_stats *st) {
    return leapfrog_impl(grid, src, nsrc, t0, nsteps, e, h, 0, trace, stream, st);
}

static int leapfrog_impl(paraexp_grid *grid, const paraexp_source *src, int32_t nsrc, double t0,
                         int64_t nsteps, void *e, void *h, int32_t check_finite,
                         const paraexp_trace *trace, void *stream, paraexp_stats *st) {
    using namespace pe;
    if (!grid) return fail(PARAEXP_EINVAL, "null grid");
    Grid &G = grid->g;
    if (G.device < 0) return fail(PARAEXP_ENOTSUP, "host-only grid");
    if (nsteps < 0) return fail(PARAEXP_EINVAL, "nsteps < 0");
    if (!e || !h) return fail(PARAEXP_EINVAL, "null field pointer");
    paraexp_stats local{};
    paraexp_stats &S = st ? *st : local;
    S = paraexp_stats();
    int rc = dev_set_device(G.device);
    if (rc) return rc;
    CallScope scope(G, stream);
    nvtxRangePushA("paraexp_leapfrog");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    std::vector<SrcDev> sd;
    if ((rc = prepare_sources(G, src, nsrc, t0, 0, nsteps, stream, sd))) return rc;
    TraceDev tr;
    if ((rc = prepare_trace(G, trace, tr))) return rc;
    const bool tracing = tr.energy || tr.np > 0;
    if (tr.energy && nsteps > 0 && (rc = dev_memset_async(tr.energy, 0, sizeof(double) * nsteps, stream))) return rc;
    if ((rc = ensure_ws(G, 2))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    Events ev(stream);
    const int id = ev.open(4);
    void *bufs[2] = {G.ws[0], G.ws[1]};
    bool host_io = false;
    if ((rc = pack_any(ka, G, e, h, bufs[0], &host_io))) return rc;
    const int id5 = ev.open(5);
    if ((rc = k_leapfrog(ka, bufs, nsteps, (const SrcDev *)G.d_src, nsrc, G.d_q, tracing ? &tr : nullptr))) return rc;
    ev.close(id5);
    if ((rc = unpack_any(ka, G, bufs[0], e, h, &host_io))) return rc;
    ev.close(id);
    if (host_io && (rc = dev_sync(stream))) return rc;
    S.leapfrog_steps = nsteps;
    S.curl_applications = 2 * nsteps;
    S.cell_updates = nsteps * (int64_t)G.nx * G.ny * G.nz;
    if (check_finite) {
        int flag = 0;
        if ((rc = k_check_finite(ka, bufs[0], &flag))) return rc;
        if (flag) return fail(PARAEXP_EDIVERGED, "leapfrog produced non-finite values");
    }
    if (st) {
        dev_sync(stream);
        double ms[7] = {0, 0, 0, 0, 0, 0, 0};
        ev.sum(ms);
        S.ms_total = ms[4];
        S.ms_leapfrog_kernels = ms[5];
        if ((rc = sched_check(G, stream))) return rc;
    }
    return PARAEXP_OK;
}

int paraexp_expmv_plan(paraexp_grid *grid, double tau, const paraexp_expmv_opts *opts,
                       paraexp_plan_info *out) {
    using namespace pe;
    if (!grid || !out) return fail(PARAEXP_EINVAL, "null argument");
    Grid &G = grid->g;
    int rc;
    int64_t launches = 0;
    if (G.device >= 0) dev_set_device(G.device);
    const double rho = default_rho(G, opts, nullptr, &launches, &rc);
    if (rc) return rc;
    Plan plan;
    if ((rc = opts_plan(G, tau, opts, rho, plan))) return rc;
    plan_to_info(plan, out);
    return PARAEXP_OK;
}

int paraexp_expmv(paraexp_grid *grid, double tau, const paraexp_expmv_opts *opts, void *e,
                  void *h, void *stream, paraexp_stats *st) {
    using namespace pe;
    if (!grid) return fail(PARAEXP_EINVAL, "null grid");
    Grid &G = grid->g;
    if (G.device < 0) return fail(PARAEXP_ENOTSUP, "host-only grid");
    if (!e || !h) return fail(PARAEXP_EINVAL, "null field pointer");
    if (!(tau >= 0) || !std::isfinite(tau)) return fail(PARAEXP_EINVAL, "tau must be >= 0");
    paraexp_stats local{};
    paraexp_stats &S = st ? *st : local;
    S = paraexp_stats();
    int rc = dev_set_device(G.device);
    if (rc) return rc;
    CallScope scope(G, stream);
    nvtxRangePushA("paraexp_expmv");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    double rho = default_rho(G, opts, stream, &S.kernel_launches, &rc);
    if (rc) return rc;
    Plan plan;
    if ((rc = opts_plan(G, tau, opts, rho, plan))) return rc;
    const bool chk = tau > 0 && rho_check_on(G, opts, rho);
    if ((rc = ensure_ws(G, chk ? 5 : 4)) || (rc = ensure_norms(G))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    Events ev(stream);
    const int id = ev.open(4);
    void *bufs[4] = {G.ws[0], G.ws[1], G.ws[2], G.ws[3]};
    bool host_io = false;
    if ((rc = pack_any(ka, G, e, h, bufs[0], &host_io))) return rc;
    double *nrm = (double *)G.d_norms;
    const size_t sbytes = (size_t)G.L.state_elems() * G.esize();
    if (chk) {   // rho safety net: keep the input, compare energy norms before / after
        if ((rc = dev_memset_async(nrm, 0, 2 * sizeof(double), stream)) ||
            (rc = k_dot_M_async(ka, bufs[0], bufs[0], nrm, G.dt)) ||
            (rc = dev_memcpy_d2d_async(G.ws[4], bufs[0], sbytes, stream))) return rc;
    }
    if ((rc = run_plan(ka, plan, bufs, &S, &ev))) return rc;
    if (chk) {
        double n2[2];
        if ((rc = k_dot_M_async(ka, bufs[0], bufs[0], nrm + 1, G.dt)) ||
            (rc = dev_memcpy_d2h(n2, nrm, 2 * sizeof(double), stream))) return rc;
        const double dev = n2[0] > 0 ? std::fabs(std::sqrt(n2[1] / n2[0]) - 1.0) : 0.0;
        S.norm_deviation = dev;
        if (!(dev <= norm_tol(G, plan, !(opts && opts->m > 0)))) {
            S.rho_fallback = 1;
            rho = G.rho_cfl;
            if ((rc = opts_plan(G, tau, opts, rho, plan))) return rc;
            if ((rc = dev_memcpy_d2d_async(bufs[0], G.ws[4], sbytes, stream))) return rc;
            S.a_applications = 0;
            S.substeps = 0;
            if ((rc = run_plan(ka, plan, bufs, &S, &ev))) return rc;
        }
    }
    if ((rc = unpack_any(ka, G, bufs[0], e, h, &host_io))) return rc;
    ev.close(id);
    S.rho = rho;
    S.method = plan.method;
    S.m = plan.m;
    S.s_first = S.s_last = plan.s;
    S.curl_applications = 2 * S.a_applications;
    S.cell_updates = S.a_applications * (int64_t)G.nx * G.ny * G.nz;
    int flag = 0;
    if ((rc = k_check_finite(ka, bufs[0], &flag))) return rc;
    if (flag) return fail(PARAEXP_EOVERFLOW, "exp(tA)v produced non-finite values (use larger s)");
    if ((rc = sched_check(G, stream))) return rc;
    double ms[7] = {0, 0, 0, 0, 0, 0, 0};
    ev.sum(ms);
    S.ms_total = ms[4];
    S.ms_poly_kernels = ms[6];
    return PARAEXP_OK;
}

int paraexp_comm_unique_id(uint8_t id[128]) {
    int rc = load_nccl();
    if (rc) return rc;
    ncclUniqueId u;
    if ((rc = nccl_check(g_nccl.GetUniqueId(&u), "ncclGetUniqueId"))) return rc;
    std::memcpy(id, u.internal, 128);
    return PARAEXP_OK;
}

int paraexp_comm_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device,
                        paraexp_comm **out) {
    if (!id || !out || world < 1 || rank < 0 || rank >= world) return pe::fail(PARAEXP_EINVAL, "bad comm arguments");
    int rc = load_nccl();
    if (rc) return rc;
    if ((rc = pe::dev_set_device(device))) return rc;
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    ncclComm_t c;
    if ((rc = nccl_check(g_nccl.CommInitRank(&c, world, u, rank), "ncclCommInitRank"))) return rc;
    *out = new paraexp_comm{c, rank, world, device};
    return PARAEXP_OK;
}

void paraexp_comm_destroy(paraexp_comm *comm) {
    if (!comm) return;
    if (g_nccl.ok && !comm->aborted) {
        if (comm->win && g_nccl.WindowDeregister) g_nccl.WindowDeregister(comm->comm, comm->win);
        g_nccl.CommDestroy(comm->comm);
    }
    if (comm->win_buf && g_nccl.MemFree) g_nccl.MemFree(comm->win_buf);
    delete comm;
}

}  // extern "C"

// =====================================================================================
// ParaExp driver (Algorithm 1): block (a4, a7) -> reduce (a8) -> finish (a9)
// =====================================================================================
namespace pe {

struct SolveCtx {
    int64_t nsteps = 0;
    int p = 0, rank = 0, world = 1, first = 0, last = -1, root = 0;
    int tail_mode = PARAEXP_TAIL_EXP;
    bool has_u0 = false;
    bool rho_check = false;     // norm-preservation check of every propagator (SURVEY finding 8)
    bool auto_plan = true;      // (m, s) chosen by the planner (eps_A meaningful for the check)
    double rho = 0, ratio = 0;
    std::vector<int64_t> B;
    std::map<int64_t, Plan> plans;
    Plan half;
    const paraexp_expmv_opts *opts = nullptr;
    // tail_mode EXP_LPT: the sub-intervals this rank owns (ascending) and whether it owns the
    // u0 tail (job 0)
    std::vector<int> owned;
    bool owns_u0 = false;
    bool exp_tails() const { return tail_mode != PARAEXP_TAIL_LEAPFROG; }
};

struct SolveBufs {
    void *P = nullptr;          // particular state of the current / last sub-interval
    void *W = nullptr;          // Horner accumulator of the tails
    void *X[3] = {nullptr, nullptr, nullptr};
};

// one plan per distinct sub-interval length plus the dt/2 shift plan (reading 10)
static int build_plans(Grid &G, SolveCtx &c) {
    c.plans.clear();
    for (int i = 1; i <= c.p; ++i) {
        const int64_t M = c.B[i] - c.B[i - 1];
        if (!c.plans.count(M)) {
            Plan pl;
            int rc = opts_plan(G, M * G.dt, c.opts, c.rho, pl);
            if (rc) return rc;
            c.plans[M] = pl;
        }
    }
    const double theta = c.rho * G.dt * 0.5;
    const int sh = std::max(1, (int)std::ceil(theta));
    return make_plan(PARAEXP_TAYLOR, 24, sh, 0.0, 0.5 * G.dt, c.rho, G.dt, c.half);
}

// Cost of one propagator E_i relative to one sub-interval's leapfrog sweep.  The fused pair
// kernel streams the same bytes per A-application as the leapfrog kernel per step,
// so the ratio is A-applications of E_i over steps of sub-interval i.
static double tail_ratio(const SolveCtx &c) {
    if (c.tail_mode == PARAEXP_TAIL_LEAPFROG) return 1.0;
    const Plan &P = c.plans.at(c.B[1] - c.B[0]);
    return (double)P.m * P.s / (double)(c.B[1] - c.B[0]);
}

// Contiguous blocks of sub-intervals, cost-balanced: rank r owning [f, l] costs
// (l - f + 1) sweeps + (p - f) propagators (+ one more for the u0 tail if f = 1), in units of a
// sweep with propagator/sweep = ratio.  The smallest makespan C is found by bisection; the
// forward greedy at C (each rank takes as many sub-intervals as fit) realises it and uses the
// fewest ranks -- with Horner tails that is also the least total work.  ratio <= 0: equal
// shares, the remainder to the later ranks (earlier blocks carry the longer tails).
static void schedule_blocks(int p, int world, double ratio, bool u0, std::vector<int> &F,
                            std::vector<int> &L, int &root) {
    F.assign(world, 0);
    L.assign(world, -1);
    const int active = std::min(p, world);
    if (!(ratio > 0) || active == 1) {
        const int base = p / active, rem = p % active;
        int start = 1;
        for (int r = 0; r < active; ++r) {
            const int n = base + (r >= active - rem ? 1 : 0);
            F[r] = start;
            L[r] = start + n - 1;
            start += n;
        }
        root = active - 1;
        return;
    }
    auto greedy = [&](double C, bool assign) -> bool {
        int f = 1;
        for (int r = 0; r < active && f <= p; ++r) {
            const double tail = (p - f) * ratio + (f == 1 && u0 ? ratio : 0.0);
            int n = (int)std::floor(C - tail + 1e-9);
            if (n < 1) return false;
            n = std::min(n, p - f + 1);
            if (assign) {
                F[r] = f;
                L[r] = f + n - 1;
            }
            f += n;
        }
        return f > p;
    };
    double lo = (p - 1) * ratio + (u0 ? ratio : 0.0), hi = lo + p;   // lo infeasible, hi feasible
    for (int it = 0; it < 200 && hi - lo > 1e-9 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (greedy(mid, false)) hi = mid; else lo = mid;
    }
    greedy(hi, true);
    root = 0;
    for (int r = 0; r < world; ++r)
        if (L[r] == p) root = r;
}

// Schedule (B) of SURVEY 8(e), kept as a comparison: the paper's literal structure, one
// independent tail per sub-interval, longest-processing-time-first.  Job j
// (1..p) costs one sweep + (p - j) propagators; job 0 (the u0 tail, if present) p propagators.
// Jobs in decreasing cost (ties: lower j first) go to the least-loaded rank (ties: lower
// rank).  owner[j] = rank of job j (owner[0] = -1 without u0); root = owner[p].
static void schedule_lpt(int p, int world, double ratio, bool u0, std::vector<int> &owner, int &root) {
    owner.assign(p + 1, -1);
    std::vector<std::pair<double, int>> jobs;
    if (u0) jobs.push_back({p * std::max(ratio, 0.0), 0});
    for (int j = 1; j <= p; ++j) jobs.push_back({1.0 + (p - j) * std::max(ratio, 0.0), j});
    std::stable_sort(jobs.begin(), jobs.end(), [](const std::pair<double, int> &a, const std::pair<double, int> &b) {
        return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    std::vector<double> load(world, 0.0);
    for (const auto &jb : jobs) {
        int r = 0;
        for (int q = 1; q < world; ++q)
            if (load[q] < load[r]) r = q;
        owner[jb.second] = r;
        load[r] += jb.first;
    }
    root = owner[p];
}

// ---- debug fault injection (PARAEXP_DEBUG_NAN=particular:<i> | tail:<i>) --
// Writes one NaN into a live interior e_x entry after sub-interval i's particular sweep or
// after propagator E_i, so the tests can check that EDIVERGED / EOVERFLOW name interval i.
struct NanHook {
    int particular = 0, tail = 0;
    NanHook() {
        const char *e = getenv("PARAEXP_DEBUG_NAN");
        if (!e) return;
        if (!strncmp(e, "particular:", 11)) particular = atoi(e + 11);
        if (!strncmp(e, "tail:", 5)) tail = atoi(e + 5);
    }
};
static int inject_nan(const Grid &G, void *state, void *stream) {
    static const double nan64 = std::nan("");
    static const float nan32 = std::nanf("");
    const int64_t off = G.nx / 2 + G.L.px * (G.ny / 2 + (int64_t)G.ny * (G.nz / 2));
    char *dst = (char *)state + off * G.esize();
    const void *src = G.dtype == PARAEXP_F64 ? (const void *)&nan64 : (const void *)&nan32;
    return dev_memcpy_h2d_async(dst, src, G.esize(), stream) ? PARAEXP_ECUDA : dev_sync(stream);
}

static int ensure_norms(Grid &G) {
    if (G.d_norms) return PARAEXP_OK;
    int rc = dev_alloc(&G.d_norms, sizeof(double) * 2 * 1002);
    if (!rc) G.device_bytes += sizeof(double) * 2 * 1002;
    return rc;
}

// Resolve the plans, rho and this rank's block.  rho: opts->rho, else min(rho_cfl,
// 1.05 rho_pow) (reading 17), broadcast from rank 0 when a communicator spans several ranks so
// that every rank builds the same plans.
static int solve_prepare(Grid &G, paraexp_comm_view comm, int rank, int world,
                         const paraexp_expmv_opts *opts, int64_t nsteps, int p, int tail_mode,
                         bool has_u0, void *stream, paraexp_stats &S, SolveCtx &c) {
    if (p < 1 || nsteps < p) return fail(PARAEXP_EINVAL, "need p >= 1 and nsteps >= p");
    if (p > 1000) return fail(PARAEXP_EINVAL, "p > 1000 not supported");
    if (tail_mode != PARAEXP_TAIL_EXP && tail_mode != PARAEXP_TAIL_LEAPFROG && tail_mode != PARAEXP_TAIL_EXP_LPT)
        return fail(PARAEXP_EINVAL, "bad tail mode");
    if (world < 1 || rank < 0 || rank >= world) return fail(PARAEXP_EINVAL, "bad rank / world");
    c.nsteps = nsteps;
    c.p = p;
    c.rank = rank;
    c.world = world;
    c.tail_mode = tail_mode;
    c.has_u0 = has_u0;
    c.opts = opts;
    c.B.assign(p + 1, 0);
    paraexp_partition(nsteps, p, c.B.data());
    int rc;
    c.rho = default_rho(G, opts, stream, &S.kernel_launches, &rc);
    if (rc) return rc;
    if (comm.bcast_rho && (rc = comm.bcast_rho(comm.ctx, &c.rho, stream))) return rc;
    const int mode = opts ? opts->rho_check : 0;
    const bool explicit_rho = opts && opts->rho > 0;
    c.rho_check = c.exp_tails() && !(opts && opts->method == PARAEXP_KRYLOV) &&
                  (mode > 0 || (mode == 0 && !explicit_rho)) && c.rho < G.rho_cfl;
    c.auto_plan = !(opts && opts->m > 0);
    if ((rc = build_plans(G, c))) return rc;
    c.ratio = tail_ratio(c);
    if (tail_mode == PARAEXP_TAIL_EXP_LPT) {
        std::vector<int> owner;
        schedule_lpt(p, world, c.ratio, has_u0, owner, c.root);
        c.owned.clear();
        for (int j = 1; j <= p; ++j)
            if (owner[j] == rank) c.owned.push_back(j);
        c.owns_u0 = has_u0 && owner[0] == rank;
        c.first = c.owned.empty() ? 0 : c.owned.front();
        c.last = c.owned.empty() ? -1 : c.owned.back();
    } else {
        std::vector<int> F, L;
        schedule_blocks(p, world, c.ratio, has_u0, F, L, c.root);
        c.first = F[rank];
        c.last = L[rank];
    }
    S.first_interval = c.first;
    S.last_interval = c.last;
    S.root = c.root;
    return PARAEXP_OK;
}

static void plan_stats(const SolveCtx &c, paraexp_stats &S) {
    const Plan &P1 = c.plans.at(c.B[1] - c.B[0]);
    const Plan &Pp = c.plans.at(c.B[c.p] - c.B[c.p - 1]);
    S.rho = c.rho;
    S.method = P1.method;
    S.m = P1.m;
    S.s_first = P1.s;
    S.s_last = Pp.s;
    S.m_half = c.half.m;
    S.s_half = c.half.s;
}

// This rank's share of the parfor for its block [first, last]: particular
// sweeps from zero with global source times (a2/a3), seeds (a4) and the Horner accumulation
// of the tails to T_p (a7, SURVEY finding 9).  Leaves W (zero if the rank owns nothing) and,
// on the owner of p, its particular state P.  Device flags: dflag[i] non-finite particular i,
// norms[2i] / norms[2i+1] = energy of W before / after propagator E_i.
static int solve_block_dev(Grid &G, const SolveCtx &c, int nsrc, const void *e0, const void *h0,
                           const TraceDev &tr, const KernelArgs &ka, Events &ev, paraexp_stats &S,
                           SolveBufs &b, bool &host_io) {
    const NanHook hook;
    const int p = c.p, first = c.first, last = c.last;
    void *stream = ka.stream;
    const size_t sbytes = (size_t)G.L.state_elems() * G.esize();
    int rc;
    b.P = G.ws[0];
    b.W = G.ws[1];
    b.X[0] = G.ws[2];
    b.X[1] = G.ws[3];
    b.X[2] = G.ws[4];
    bool W_valid = false;
    int *dflag = (int *)G.d_flag;
    double *norms = (double *)G.d_norms;
    if ((rc = dev_memset_async(dflag, 0, sizeof(int) * (p + 2), stream))) return rc;
    if ((rc = dev_memset_async(norms, 0, sizeof(double) * 2 * (p + 1), stream))) return rc;
    const bool tracing = tr.energy || tr.np > 0;
    if (tracing) {
        // rows i < p of the energy need the summed field: NaN with several ranks (paraexp.h)
        std::vector<double> init(p, c.world > 1 ? std::nan("") : 0.0);
        init[p - 1] = 0.0;
        if (tr.energy && (rc = dev_memcpy_h2d_async(tr.energy, init.data(), sizeof(double) * p, stream))) return rc;
        if (tr.np > 0 && (rc = dev_memset_async(tr.probe, 0, sizeof(double) * p * tr.np, stream))) return rc;
        if ((rc = dev_sync(stream))) return rc;
    }

    auto propagate = [&](int i) -> int {   // W <- E_i W
        const int64_t M = c.B[i] - c.B[i - 1];
        nvtxRangePushA("propagate");
        int r = PARAEXP_OK;
        if (c.rho_check) r = k_dot_M_async(ka, b.W, b.W, norms + 2 * i, G.dt);
        if (!r && c.tail_mode == PARAEXP_TAIL_EXP) {
            void *bufs[4] = {b.W, b.X[0], b.X[1], b.X[2]};
            r = run_plan(ka, c.plans.at(M), bufs, &S, &ev);
            b.W = bufs[0];
            b.X[0] = bufs[1];
            b.X[1] = bufs[2];
            b.X[2] = bufs[3];
        } else if (!r) {
            void *bufs[2] = {b.W, b.X[0]};
            const int id5 = ev.open(5);
            r = k_leapfrog(ka, bufs, M, nullptr, 0, nullptr);
            ev.close(id5);
            if (bufs[0] != b.W) std::swap(b.W, b.X[0]);
            S.leapfrog_steps += M;
            S.curl_applications += 2 * M;
        }
        if (!r && hook.tail == i) r = inject_nan(G, b.W, stream);
        if (!r) r = k_dot_M_async(ka, b.W, b.W, norms + 2 * i + 1, G.dt);   // energy after E_i
        nvtxRangePop();
        return r;
    };

    // f1: the Horner accumulator after sub-interval i (seed added) is this rank's share of the
    // same-time solution u(T_i) = v_i(T_i) + sum_{j<i} w_j(T_i)
    auto trace_row = [&](int i) -> int {
        int r = PARAEXP_OK;
        if (tr.np > 0) r = k_gather(ka, b.W, tr, tr.probe + (int64_t)(i - 1) * tr.np, 0);
        if (!r && tr.energy && c.world == 1) r = k_dot_M_async(ka, b.W, b.W, tr.energy + (i - 1), G.dt);
        return r;
    };

    // Concurrent particular sweeps (small grids): the sub-intervals of this rank's block are
    // independent leapfrog problems from zero (the parfor of PAPER:358-361).  When one sweep
    // cannot fill the GPU they run concurrently on side streams, each into its own buffer, and
    // the Horner chain on `stream` consumes them in order as they complete.
    const int nb = first >= 1 ? last - first + 1 : 0;
    int nstr = std::min(nb, 8);
    bool conc = nb >= 2 && nb <= 64 && concurrent_sweeps(G);
    // Mid-size grids (mid.cu): a sweep is ONE resident launch instead of one TMA launch per step
    // (at 32^3 those per-step launches bound the solve by the host's launch rate).  The sweeps
    // run concurrently on SM partitions -- as many streams (<= 8) as leave each sweep the CTAs
    // it needs, each stream with its own exchange-buffer slot -- or, if not even two fit,
    // serially over the whole GPU (unless PARAEXP_CONCURRENT forces the concurrent TMA sweeps).
    int mid_budget = 0;
    if (conc && G.kernels == PARAEXP_KERNELS_FUSED && nsrc <= 16 && mid_supported(G)) {
        const int nsm = device_sm_count();
        for (int ns = nstr; ns >= 2 && !mid_budget; --ns)
            if (mid_supported(G, nsm / ns)) {
                mid_budget = nsm / ns;
                nstr = ns;
            }
        if (!mid_budget && !getenv("PARAEXP_CONCURRENT")) conc = false;
    }
    std::vector<void *> Pc;
    if (conc) {
        while ((int)G.conc.size() < nb + nstr) {
            void *q = nullptr;
            if ((rc = dev_alloc(&q, sbytes))) return rc;
            if ((rc = dev_memset_async(q, 0, sbytes, nullptr)) || (rc = dev_sync(nullptr))) return rc;
            G.conc.push_back(q);
            G.device_bytes += sbytes;
        }
        while ((int)G.streams.size() < nstr) {
            void *q = nullptr;
            if ((rc = dev_stream_create(&q))) return rc;
            G.streams.push_back(q);
        }
        while ((int)G.events.size() < nb + 1) {
            void *q = nullptr;
            if ((rc = dev_event_create(&q))) return rc;
            G.events.push_back(q);
        }
        Pc.assign(G.conc.begin(), G.conc.begin() + nb);
        std::vector<void *> scratch(G.conc.begin() + nb, G.conc.begin() + nb + nstr);
        for (int q = 0; q < nstr; ++q)   // side streams start after the work already on `stream`
            if ((rc = dev_stream_after(G.streams[q], stream, G.events[nb]))) return rc;
        for (int q = 0; q < nb; ++q) {
            const int i = first + q, sq = q % nstr;
            KernelArgs kq = ka;
            kq.stream = G.streams[sq];
            kq.static_sched = true;                        // concurrent launches: no shared counter
            if (mid_budget) {                              // resident sweep on its SM partition
                kq.mid_slot = 1 + sq;
                kq.mid_max_cta = mid_budget;
            }
            if ((rc = dev_memset_async(Pc[q], 0, sbytes, kq.stream))) return rc;
            void *bufs[2] = {Pc[q], scratch[sq]};
            const size_t qoff = (size_t)c.B[i - 1] * nsrc * G.esize();
            if ((rc = k_leapfrog(kq, bufs, c.B[i] - c.B[i - 1], (const SrcDev *)G.d_src, nsrc,
                                 (const char *)G.d_q + qoff))) return rc;
            if (bufs[0] != Pc[q]) std::swap(Pc[q], scratch[sq]);   // result buffer <-> scratch
            if (hook.particular == i && (rc = inject_nan(G, Pc[q], kq.stream))) return rc;
            if ((rc = k_check_finite_async(kq, Pc[q], dflag + i))) return rc;
            if (cudaEventRecord((cudaEvent_t)G.events[q], (cudaStream_t)kq.stream) != cudaSuccess)
                return check_cuda("event record");
            S.leapfrog_steps += c.B[i] - c.B[i - 1];
            S.curl_applications += 2 * (c.B[i] - c.B[i - 1]);
        }
        // keep the buffer roles for the next call (results may now live in former scratch)
        for (int q = 0; q < nb; ++q) G.conc[q] = Pc[q];
        for (int q = 0; q < nstr; ++q) G.conc[nb + q] = scratch[q];
    }

    if (first >= 1) {
        if (first == 1 && c.has_u0) {
            if ((rc = pack_any(ka, G, e0, h0, b.W, &host_io))) return rc;
            if (c.tail_mode == PARAEXP_TAIL_LEAPFROG && (rc = k_half_start(ka, b.W))) return rc;
            W_valid = true;
        }
        for (int i = first; i <= last; ++i) {
            const int64_t M = c.B[i] - c.B[i - 1];
            int id = ev.open(0);
            nvtxRangePushA("particular");
            if (conc) {
                if (cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)G.events[i - first], 0) != cudaSuccess)
                    return check_cuda("stream wait");
                b.P = Pc[i - first];
            } else {
                if ((rc = dev_memset_async(b.P, 0, sbytes, stream))) return rc;
                void *bufs[2] = {b.P, b.X[0]};
                const size_t qoff = (size_t)c.B[i - 1] * nsrc * G.esize();
                const int id5 = ev.open(5);
                if ((rc = k_leapfrog(ka, bufs, M, (const SrcDev *)G.d_src, nsrc, (const char *)G.d_q + qoff))) return rc;
                ev.close(id5);
                if (bufs[0] != b.P) std::swap(b.P, b.X[0]);
                S.leapfrog_steps += M;
                S.curl_applications += 2 * M;
                if (hook.particular == i && (rc = inject_nan(G, b.P, stream))) return rc;
                if ((rc = k_check_finite_async(ka, b.P, dflag + i))) return rc;
            }
            nvtxRangePop();
            ev.close(id);
            id = ev.open(1);
            if (W_valid && (rc = propagate(i))) return rc;
            if (i < p) {
                if (c.tail_mode == PARAEXP_TAIL_EXP && (rc = k_sync(ka, b.P))) return rc;
                if (W_valid) {
                    if ((rc = k_axpy(ka, b.W, b.P, 1.0))) return rc;
                } else {
                    if ((rc = dev_memcpy_d2d_async(b.W, b.P, sbytes, stream))) return rc;
                    W_valid = true;
                }
                if (tracing && (rc = trace_row(i))) return rc;
            }
            ev.close(id);
        }
        const int id = ev.open(1);
        for (int i = last + 1; i <= p; ++i) {
            if (W_valid && (rc = propagate(i))) return rc;
            if (tracing && i < p && W_valid && (rc = trace_row(i))) return rc;
        }
        ev.close(id);
    }
    if (!W_valid && (rc = dev_memset_async(b.W, 0, sbytes, stream))) return rc;
    return k_check_finite_async(ka, b.W, dflag + p + 1);
}

// tail_mode EXP_LPT (schedule B, reading 34): this rank's jobs of the paper's literal parfor --
// for each owned j, v_j by leapfrog from zero, its seed s_j and its OWN tail E_p..E_{j+1} s_j
// (PAPER:358-365), summed into W; the u0 tail E_p..E_1 u0 if the rank owns job 0.  Same flags
// and norms as solve_block_dev (the propagator norms accumulate over the rank's tails).
static int solve_block_lpt_dev(Grid &G, const SolveCtx &c, int nsrc, const void *e0, const void *h0,
                               const KernelArgs &ka, Events &ev, paraexp_stats &S, SolveBufs &b,
                               bool &host_io) {
    const NanHook hook;
    const int p = c.p;
    void *stream = ka.stream;
    const size_t sbytes = (size_t)G.L.state_elems() * G.esize();
    int rc;
    b.P = G.ws[0];
    b.W = G.ws[1];
    b.X[0] = G.ws[2];
    b.X[1] = G.ws[3];
    b.X[2] = G.ws[4];
    int *dflag = (int *)G.d_flag;
    double *norms = (double *)G.d_norms;
    if ((rc = dev_memset_async(dflag, 0, sizeof(int) * (p + 2), stream))) return rc;
    if ((rc = dev_memset_async(norms, 0, sizeof(double) * 2 * (p + 1), stream))) return rc;
    bool W_valid = false;
    auto propagate = [&](int i) -> int {              // P <- E_i P
        nvtxRangePushA("propagate");
        int r = PARAEXP_OK;
        if (c.rho_check) r = k_dot_M_async(ka, b.P, b.P, norms + 2 * i, G.dt);
        if (!r) {
            void *bufs[4] = {b.P, b.X[0], b.X[1], b.X[2]};
            r = run_plan(ka, c.plans.at(c.B[i] - c.B[i - 1]), bufs, &S, &ev);
            b.P = bufs[0];
            b.X[0] = bufs[1];
            b.X[1] = bufs[2];
            b.X[2] = bufs[3];
        }
        if (!r && hook.tail == i) r = inject_nan(G, b.P, stream);
        if (!r) r = k_dot_M_async(ka, b.P, b.P, norms + 2 * i + 1, G.dt);
        nvtxRangePop();
        return r;
    };
    auto add_to_W = [&]() -> int {
        if (W_valid) return k_axpy(ka, b.W, b.P, 1.0);
        W_valid = true;
        return dev_memcpy_d2d_async(b.W, b.P, sbytes, stream);
    };
    if (c.owns_u0) {                                   // job 0: E_p..E_1 u0
        const int id = ev.open(1);
        if ((rc = pack_any(ka, G, e0, h0, b.P, &host_io))) return rc;
        for (int i = 1; i <= p; ++i)
            if ((rc = propagate(i))) return rc;
        if ((rc = add_to_W())) return rc;
        ev.close(id);
    }
    for (int j : c.owned) {
        const int64_t M = c.B[j] - c.B[j - 1];
        int id = ev.open(0);
        if ((rc = dev_memset_async(b.P, 0, sbytes, stream))) return rc;
        void *bufs[2] = {b.P, b.X[0]};
        const size_t qoff = (size_t)c.B[j - 1] * nsrc * G.esize();
        const int id5 = ev.open(5);
        if ((rc = k_leapfrog(ka, bufs, M, (const SrcDev *)G.d_src, nsrc, (const char *)G.d_q + qoff))) return rc;
        ev.close(id5);
        if (bufs[0] != b.P) std::swap(b.P, b.X[0]);
        S.leapfrog_steps += M;
        S.curl_applications += 2 * M;
        if (hook.particular == j && (rc = inject_nan(G, b.P, stream))) return rc;
        if ((rc = k_check_finite_async(ka, b.P, dflag + j))) return rc;
        ev.close(id);
        if (j < p) {                                   // seed and its own tail to T_p
            id = ev.open(1);
            if ((rc = k_sync(ka, b.P))) return rc;
            for (int i = j + 1; i <= p; ++i)
                if ((rc = propagate(i))) return rc;
            if ((rc = add_to_W())) return rc;
            ev.close(id);
        }
    }
    if (!W_valid && (rc = dev_memset_async(b.W, 0, sbytes, stream))) return rc;
    return k_check_finite_async(ka, b.W, dflag + p + 1);
}

// Read back the block's device flags and propagator norms (synchronises `stream`).
// Returns EDIVERGED / EOVERFLOW naming the first failing sub-interval, or sets *violation when
// a propagator changed the energy norm by more than its tolerance (rho too small: the
// spectrum leaves the Leja interval and the polynomial grows there -- SURVEY finding 8).
static int block_status(const Grid &G, const SolveCtx &c, void *stream, paraexp_stats &S, bool *violation,
                        double *max_dev) {
    const int p = c.p;
    std::vector<int> flags(p + 2, 0);
    std::vector<double> nrm(2 * (p + 1), 0.0);
    int rc = dev_memcpy_d2h(flags.data(), G.d_flag, sizeof(int) * (p + 2), stream);
    if (!rc) rc = dev_memcpy_d2h(nrm.data(), G.d_norms, sizeof(double) * 2 * (p + 1), stream);
    if (rc) return rc;
    for (int i = 1; i <= p; ++i)
        if (flags[i]) {
            S.fail_interval = i;
            return fail(PARAEXP_EDIVERGED, "leapfrog diverged in sub-interval " + std::to_string(i));
        }
    *violation = false;
    *max_dev = 0;
    // first propagator this rank applied (Horner: from its block's start; LPT: its first tail)
    int fprop = c.first >= 1 ? (c.first == 1 && c.has_u0 ? 1 : c.first + 1) : p + 1;
    if (c.tail_mode == PARAEXP_TAIL_EXP_LPT) fprop = c.owns_u0 ? 1 : (c.first >= 1 ? c.first + 1 : p + 1);
    for (int i = fprop; i <= p; ++i) {
        const double after = nrm[2 * i + 1];
        if (!std::isfinite(after)) {
            S.fail_interval = i;
            return fail(PARAEXP_EOVERFLOW, "exp(tA)v tail produced non-finite values in propagator " + std::to_string(i));
        }
        if (c.rho_check && nrm[2 * i] > 0) {
            const double dev = std::fabs(std::sqrt(after / nrm[2 * i]) - 1.0);
            const Plan &P = c.plans.at(c.B[i] - c.B[i - 1]);
            const double floor_tol = G.dtype == PARAEXP_F64 ? 1e-9 : 1e-3;
            const double tol = c.auto_plan ? std::max(floor_tol, 10.0 * P.eps_A * P.rho * P.tau)
                                           : std::max(floor_tol, 1e-3);
            *max_dev = std::max(*max_dev, dev);
            if (!(dev <= tol)) *violation = true;
        }
    }
    if (flags[p + 1]) {
        S.fail_interval = c.first;
        return fail(PARAEXP_EOVERFLOW, "exp(tA)v tails produced non-finite values");
    }
    return PARAEXP_OK;
}

// solve_block_dev + block_status, with the rho safety net: when a propagator violated norm
// preservation and rho < rho_cfl, the block is recomputed with rho = rho_cfl (an upper bound of
// ||A||_2, SURVEY finding 7).  The schedule is kept, so the ranks' partial sums still add up.
static int solve_block_checked(Grid &G, SolveCtx &c, int nsrc, const void *e0, const void *h0,
                               const TraceDev &tr, const KernelArgs &ka, Events &ev, paraexp_stats &S,
                               SolveBufs &b, bool &host_io) {
    int rc;
    nvtxRangePushA("paraexp_block");
    for (int attempt = 0; attempt < 2; ++attempt) {
        rc = c.tail_mode == PARAEXP_TAIL_EXP_LPT ? solve_block_lpt_dev(G, c, nsrc, e0, h0, ka, ev, S, b, host_io)
                                                 : solve_block_dev(G, c, nsrc, e0, h0, tr, ka, ev, S, b, host_io);
        if (rc) break;
        bool viol = false;
        double dev = 0;
        if ((rc = block_status(G, c, ka.stream, S, &viol, &dev))) break;
        S.norm_deviation = dev;
        if (!viol) break;
        if (attempt == 1 || !(c.rho < G.rho_cfl)) {
            rc = fail(PARAEXP_EOVERFLOW, "exp(tA)v tails violate norm preservation even with rho_cfl");
            break;
        }
        S.rho_fallback = 1;
        c.rho = G.rho_cfl;
        c.rho_check = false;
        if ((rc = build_plans(G, c))) break;
        plan_stats(c, S);
    }
    nvtxRangePop();
    return rc;
}

// a9 on the owner of p: e_out = e_p + W_e, h_out = h_p + [exp(dt/2 A) W]_h (eq:averaging1/2,
// reading 10), in place in b.P.
static int solve_finish_dev(Grid &G, const SolveCtx &c, const KernelArgs &ka, Events &ev,
                            paraexp_stats &S, SolveBufs &b) {
    int rc;
    nvtxRangePushA("paraexp_finish");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    if (c.exp_tails()) {
        if ((rc = k_axpy_comps(ka, b.P, b.W, 1.0, 0, 3))) return rc;       // e_out = e_p + W_e
        void *bufs[4] = {b.W, b.X[0], b.X[1], b.X[2]};
        if ((rc = run_plan(ka, c.half, bufs, nullptr, &ev))) return rc;     // exp(dt/2 A) W
        S.a_applications += (int64_t)c.half.s * c.half.m;
        b.W = bufs[0];
        b.X[0] = bufs[1];
        b.X[1] = bufs[2];
        b.X[2] = bufs[3];
        if ((rc = k_axpy_comps(ka, b.P, b.W, 1.0, 3, 6))) return rc;       // h_out = h_p + [.]_h
    } else {
        if ((rc = k_axpy(ka, b.P, b.W, 1.0))) return rc;
    }
    return PARAEXP_OK;
}

static void finish_stats(const Grid &G, Events &ev, paraexp_stats &S) {
    const int64_t cells = (int64_t)G.nx * G.ny * G.nz;
    S.curl_applications = 2 * (S.leapfrog_steps + S.a_applications);
    S.cell_updates = (S.leapfrog_steps + S.a_applications) * cells;
    double ms[7] = {0, 0, 0, 0, 0, 0, 0};
    ev.sum(ms);
    S.ms_particular = ms[0];
    S.ms_tails = ms[1];
    S.ms_reduce = ms[2];
    S.ms_finish = ms[3];
    S.ms_total = ms[4];
    S.ms_leapfrog_kernels = ms[5];
    S.ms_poly_kernels = ms[6];
}

}  // namespace pe

extern "C" {

static int solve_impl(paraexp_grid *grid, paraexp_comm *comm, const paraexp_source *src,
                      int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                      const paraexp_expmv_opts *opts, int32_t tail_mode, int32_t broadcast_out,
                      const void *e0, const void *h0, void *e_out, void *h_out,
                      const paraexp_trace *trace, void *stream, paraexp_stats *st);

int paraexp_solve(paraexp_grid *grid, paraexp_comm *comm, const paraexp_source *src,
                  int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                  const paraexp_expmv_opts *opts, int32_t tail_mode, int32_t broadcast_out,
                  const void *e0, const void *h0, void *e_out, void *h_out, void *stream,
                  paraexp_stats *st) {
    return solve_impl(grid, comm, src, nsrc, t0, nsteps, p, opts, tail_mode, broadcast_out, e0, h0, e_out,
                      h_out, nullptr, stream, st);
}

int paraexp_solve_trace(paraexp_grid *grid, paraexp_comm *comm, const paraexp_source *src,
                        int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                        const paraexp_expmv_opts *opts, int32_t broadcast_out, const void *e0,
                        const void *h0, void *e_out, void *h_out, const paraexp_trace *trace,
                        void *stream, paraexp_stats *st) {
    return solve_impl(grid, comm, src, nsrc, t0, nsteps, p, opts, PARAEXP_TAIL_EXP, broadcast_out, e0, h0,
                      e_out, h_out, trace, stream, st);
}

static int solve_impl(paraexp_grid *grid, paraexp_comm *comm, const paraexp_source *src,
                      int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                      const paraexp_expmv_opts *opts, int32_t tail_mode, int32_t broadcast_out,
                      const void *e0, const void *h0, void *e_out, void *h_out,
                      const paraexp_trace *trace, void *stream, paraexp_stats *st) {
    using namespace pe;
    if (!grid) return fail(PARAEXP_EINVAL, "null grid");
    Grid &G = grid->g;
    if (G.device < 0) return fail(PARAEXP_ENOTSUP, "host-only grid");
    if ((e0 == nullptr) != (h0 == nullptr)) return fail(PARAEXP_EINVAL, "e0 and h0 must both be given or both NULL");
    if (trace && tail_mode != PARAEXP_TAIL_EXP) return fail(PARAEXP_EINVAL, "trace needs tail_mode EXP");
    const int rank = comm ? comm->rank : 0, world = comm ? comm->world : 1;
    paraexp_stats local{};
    paraexp_stats &S = st ? *st : local;
    S = paraexp_stats();
    int rc = dev_set_device(G.device);
    if (rc) return rc;
    CallScope scope(G, stream);
    nvtxRangePushA("paraexp_solve");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    // the collectives also run for a one-rank communicator when PARAEXP_FORCE_COLLECTIVES is
    // set, so the NCCL code path can be exercised on a single GPU (tests)
    const bool coll = comm && (world > 1 || getenv("PARAEXP_FORCE_COLLECTIVES"));
    CommCtx cctx{comm, &G};
    paraexp_comm_view view;
    if (coll && !(opts && opts->rho > 0)) {      // also for a forced one-rank communicator (tests)
        view.ctx = &cctx;
        view.bcast_rho = bcast_rho_nccl;
    }
    SolveCtx c;
    if ((rc = solve_prepare(G, view, rank, world, opts, nsteps, p, tail_mode, e0 != nullptr, stream, S, c))) return rc;
    plan_stats(c, S);

    std::vector<SrcDev> sd;
    if ((rc = prepare_sources(G, src, nsrc, t0, 0, nsteps, stream, sd))) return rc;
    TraceDev tr;
    if ((rc = prepare_trace(G, trace, tr))) return rc;
    const bool tracing = tr.energy || tr.np > 0;
    if ((rc = ensure_ws(G, 5)) || (rc = ensure_norms(G))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    const size_t sbytes = (size_t)G.L.state_elems() * G.esize();
    Events ev(stream);
    const int idt = ev.open(4);
    bool host_io = false;       // host-pointer fields (staged copies; the call syncs anyway)
    SolveBufs b;
    rc = solve_block_checked(G, c, nsrc, e0, h0, tr, ka, ev, S, b, host_io);
    // the ranks agree on the blocks' status before the reduce: a rank whose block failed
    // (divergence, overflow, allocation) would otherwise leave its peers waiting in ncclReduce
    if (coll) {
        const int rc2 = comm_status_any(comm, G, rc != PARAEXP_OK, stream);
        if (rc) return rc;
        if (rc2 < 0) return rc2;
        if (rc2 > 0) return fail(PARAEXP_EDIVERGED, "another rank's block failed (status all-reduce)");
    } else if (rc) {
        return rc;
    }

    // a8: sum the tails onto the root
    if (coll) {
        const int id = ev.open(2);
        nvtxRangePushA("paraexp_reduce");
        rc = comm_reduce_W(comm, G, b.W, sbytes, c.root, stream);
        nvtxRangePop();
        if (rc) return rc;
        ev.close(id);
    }
    const int idf = ev.open(3);
    if (rank == c.root && tracing) {
        // row p: u(T_p) = sync(v_p) + W, same-time (reading 9)
        if ((rc = dev_memcpy_d2d_async(b.X[0], b.P, sbytes, stream))) return rc;
        if ((rc = k_sync(ka, b.X[0]))) return rc;
        if ((rc = k_axpy(ka, b.X[0], b.W, 1.0))) return rc;
        if (tr.np > 0 && (rc = k_gather(ka, b.X[0], tr, tr.probe + (int64_t)(p - 1) * tr.np, 0))) return rc;
        if (tr.energy && (rc = k_dot_M_async(ka, b.X[0], b.X[0], tr.energy + (p - 1), G.dt))) return rc;
    }
    if (tracing && coll && (rc = comm_allreduce_trace(comm, tr, p, stream))) return rc;
    // a9: reconstruction on the root (eq:averaging1/2, reading 10)
    if (rank == c.root && (rc = solve_finish_dev(G, c, ka, ev, S, b))) return rc;
    if (broadcast_out && coll && (rc = comm_bcast_state(comm, G, b.P, c.root, stream))) return rc;
    if ((rank == c.root || broadcast_out) && e_out && h_out) {
        if ((rc = unpack_any(ka, G, b.P, e_out, h_out, &host_io))) return rc;
    }
    ev.close(idf);
    ev.close(idt);
    if (coll && (rc = comm_wait(comm, stream))) return rc;
    if ((rc = dev_sync(stream))) return rc;
    if ((rc = sched_check(G, stream))) return rc;
    finish_stats(G, ev, S);
    return PARAEXP_OK;
}

int paraexp_solve_block(paraexp_grid *grid, int32_t rank, int32_t world, const paraexp_source *src,
                        int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                        const paraexp_expmv_opts *opts, int32_t tail_mode, const void *e0,
                        const void *h0, void *w_e, void *w_h, void *v_e, void *v_h, void *stream,
                        paraexp_stats *st) {
    using namespace pe;
    if (!grid) return fail(PARAEXP_EINVAL, "null grid");
    Grid &G = grid->g;
    if (G.device < 0) return fail(PARAEXP_ENOTSUP, "host-only grid");
    if ((e0 == nullptr) != (h0 == nullptr)) return fail(PARAEXP_EINVAL, "e0 and h0 must both be given or both NULL");
    if (!w_e || !w_h) return fail(PARAEXP_EINVAL, "null w_e / w_h");
    paraexp_stats local{};
    paraexp_stats &S = st ? *st : local;
    S = paraexp_stats();
    int rc = dev_set_device(G.device);
    if (rc) return rc;
    CallScope scope(G, stream);
    SolveCtx c;
    if ((rc = solve_prepare(G, paraexp_comm_view(), rank, world, opts, nsteps, p, tail_mode, e0 != nullptr,
                            stream, S, c))) return rc;
    plan_stats(c, S);
    std::vector<SrcDev> sd;
    if ((rc = prepare_sources(G, src, nsrc, t0, 0, nsteps, stream, sd))) return rc;
    if ((rc = ensure_ws(G, 5)) || (rc = ensure_norms(G))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    Events ev(stream);
    const int idt = ev.open(4);
    bool host_io = false;
    SolveBufs b;
    if ((rc = solve_block_checked(G, c, nsrc, e0, h0, TraceDev(), ka, ev, S, b, host_io))) return rc;
    if ((rc = unpack_any(ka, G, b.W, w_e, w_h, &host_io))) return rc;
    if (rank == c.root && v_e && v_h && (rc = unpack_any(ka, G, b.P, v_e, v_h, &host_io))) return rc;
    ev.close(idt);
    if ((rc = dev_sync(stream))) return rc;
    if ((rc = sched_check(G, stream))) return rc;
    finish_stats(G, ev, S);
    return PARAEXP_OK;
}

int paraexp_solve_finish(paraexp_grid *grid, const paraexp_expmv_opts *opts, int32_t tail_mode,
                         const void *w_e, const void *w_h, const void *v_e, const void *v_h,
                         void *e_out, void *h_out, void *stream, paraexp_stats *st) {
    using namespace pe;
    if (!grid) return fail(PARAEXP_EINVAL, "null grid");
    Grid &G = grid->g;
    if (G.device < 0) return fail(PARAEXP_ENOTSUP, "host-only grid");
    if (!w_e || !w_h || !v_e || !v_h || !e_out || !h_out) return fail(PARAEXP_EINVAL, "null field pointer");
    if (tail_mode != PARAEXP_TAIL_EXP && tail_mode != PARAEXP_TAIL_LEAPFROG && tail_mode != PARAEXP_TAIL_EXP_LPT)
        return fail(PARAEXP_EINVAL, "bad tail mode");
    paraexp_stats local{};
    paraexp_stats &S = st ? *st : local;
    S = paraexp_stats();
    int rc = dev_set_device(G.device);
    if (rc) return rc;
    CallScope scope(G, stream);
    SolveCtx c;
    c.tail_mode = tail_mode;
    c.rho = default_rho(G, opts, stream, &S.kernel_launches, &rc);
    if (rc) return rc;
    {
        const double theta = c.rho * G.dt * 0.5;
        if ((rc = make_plan(PARAEXP_TAYLOR, 24, std::max(1, (int)std::ceil(theta)), 0.0, 0.5 * G.dt, c.rho, G.dt,
                            c.half))) return rc;
    }
    S.rho = c.rho;
    S.m_half = c.half.m;
    S.s_half = c.half.s;
    if ((rc = ensure_ws(G, 5))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    Events ev(stream);
    const int idt = ev.open(4);
    bool host_io = false;
    SolveBufs b;
    b.P = G.ws[0];
    b.W = G.ws[1];
    b.X[0] = G.ws[2];
    b.X[1] = G.ws[3];
    b.X[2] = G.ws[4];
    if ((rc = pack_any(ka, G, w_e, w_h, b.W, &host_io))) return rc;
    if ((rc = pack_any(ka, G, v_e, v_h, b.P, &host_io))) return rc;
    if ((rc = solve_finish_dev(G, c, ka, ev, S, b))) return rc;
    if ((rc = unpack_any(ka, G, b.P, e_out, h_out, &host_io))) return rc;
    ev.close(idt);
    if ((rc = dev_sync(stream))) return rc;
    finish_stats(G, ev, S);
    return PARAEXP_OK;
}

}  // extern "C"
