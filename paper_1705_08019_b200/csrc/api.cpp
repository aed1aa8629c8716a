// api.cpp -- C ABI entry points: leapfrog (a2/a3), expmv (a5/a6), ParaExp solve (a4, a7-a9),
// K5 norm estimate, communicator (a8), host helpers and error handling.
// See include/paraexp.h for the contract of every function.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
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
    if (ka.g->kernels == PARAEXP_KERNELS_FUSED && fused_supported(*ka.g))
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
    if (ka.g->kernels == PARAEXP_KERNELS_FUSED && fused_supported(*ka.g))
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
    paraexp_expmv_opts def{PARAEXP_LEJA, 0, 0, 1e-12, 0.0, 0, 0.0};
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
};

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

int paraexp_partition(int64_t nsteps, int32_t p, int64_t *bounds) {
    if (p < 1 || nsteps < p || !bounds) return pe::fail(PARAEXP_EINVAL, "need p >= 1 and nsteps >= p");
    const int64_t M = nsteps / p;
    for (int j = 0; j < p; ++j) bounds[j] = j * M;
    bounds[p] = nsteps;
    return PARAEXP_OK;
}

int paraexp_schedule(int32_t p, int32_t world, int32_t rank, int32_t *first, int32_t *last,
                     int32_t *root) {
    if (p < 1 || world < 1 || rank < 0 || rank >= world) return pe::fail(PARAEXP_EINVAL, "bad schedule arguments");
    // contiguous blocks; ranks with longer tails (earlier blocks) get the smaller share
    const int active = std::min(p, world);
    const int base = p / active, rem = p % active;
    int f = 0, l = -1;
    if (rank < active) {
        // ranks active-rem .. active-1 get base+1
        int start = 1;
        for (int r = 0; r < rank; ++r) start += base + (r >= active - rem ? 1 : 0);
        f = start;
        l = start + base + (rank >= active - rem ? 1 : 0) - 1;
    }
    if (first) *first = f;
    if (last) *last = l;
    if (root) *root = active - 1;
    return PARAEXP_OK;
}

int paraexp_grid_info(paraexp_grid *grid, int32_t compute_rho_pow, void *stream,
                      paraexp_grid_info_t *o) {
    if (!grid || !o) return pe::fail(PARAEXP_EINVAL, "null argument");
    pe::Grid &G = grid->g;
    if (compute_rho_pow && G.device >= 0 && G.rho_pow == 0) {
        int64_t launches = 0;
        pe::dev_set_device(G.device);
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
    const double rho = default_rho(G, opts, stream, &S.kernel_launches, &rc);
    if (rc) return rc;
    Plan plan;
    if ((rc = opts_plan(G, tau, opts, rho, plan))) return rc;
    if ((rc = ensure_ws(G, 4))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    Events ev(stream);
    const int id = ev.open(4);
    void *bufs[4] = {G.ws[0], G.ws[1], G.ws[2], G.ws[3]};
    bool host_io = false;
    if ((rc = pack_any(ka, G, e, h, bufs[0], &host_io))) return rc;
    if ((rc = run_plan(ka, plan, bufs, &S, &ev))) return rc;
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
    if (g_nccl.ok) g_nccl.CommDestroy(comm->comm);
    delete comm;
}

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
    if (p < 1 || nsteps < p) return fail(PARAEXP_EINVAL, "need p >= 1 and nsteps >= p");
    if (p > 1000) return fail(PARAEXP_EINVAL, "p > 1000 not supported");
    if (tail_mode != PARAEXP_TAIL_EXP && tail_mode != PARAEXP_TAIL_LEAPFROG) return fail(PARAEXP_EINVAL, "bad tail mode");
    if ((e0 == nullptr) != (h0 == nullptr)) return fail(PARAEXP_EINVAL, "e0 and h0 must both be given or both NULL");
    if (trace && tail_mode != PARAEXP_TAIL_EXP) return fail(PARAEXP_EINVAL, "trace needs tail_mode EXP");
    const int rank = comm ? comm->rank : 0, world = comm ? comm->world : 1;
    paraexp_stats local{};
    paraexp_stats &S = st ? *st : local;
    S = paraexp_stats();
    int rc = dev_set_device(G.device);
    if (rc) return rc;
    std::vector<int64_t> B(p + 1);
    paraexp_partition(nsteps, p, B.data());
    int first, last, root;
    paraexp_schedule(p, world, rank, &first, &last, &root);
    S.first_interval = first;
    S.last_interval = last;
    S.root = root;
    const bool has_u0 = e0 != nullptr;

    double rho = default_rho(G, opts, stream, &S.kernel_launches, &rc);
    if (rc) return rc;
    if (comm && world > 1 && !(opts && opts->rho > 0)) {
        // every rank must build the same plans: the K5 estimate (atomics) can differ in the
        // last bits between ranks, so all ranks take rank 0's value
        double *d = (double *)G.d_red;
        if ((rc = dev_memcpy_h2d_async(d, &rho, sizeof(double), stream))) return rc;
        if ((rc = nccl_check(g_nccl.Broadcast(d, d, 1, kNcclF64, 0, comm->comm, (cudaStream_t)stream),
                             "ncclBroadcast(rho)"))) return rc;
        if ((rc = dev_memcpy_d2h(&rho, d, sizeof(double), stream))) return rc;
    }
    S.rho = rho;
    // one plan per distinct sub-interval length, plus the dt/2 shift plan
    std::map<int64_t, Plan> plans;
    for (int i = 1; i <= p; ++i) {
        const int64_t M = B[i] - B[i - 1];
        if (!plans.count(M)) {
            Plan pl;
            if ((rc = opts_plan(G, M * G.dt, opts, rho, pl))) return rc;
            plans[M] = pl;
        }
    }
    Plan half;
    {
        const double theta = rho * G.dt * 0.5;
        const int sh = std::max(1, (int)std::ceil(theta));
        if ((rc = make_plan(PARAEXP_TAYLOR, 24, sh, 0.0, 0.5 * G.dt, rho, G.dt, half))) return rc;
    }
    const Plan &P1 = plans[B[1] - B[0]];
    const Plan &Pp = plans[B[p] - B[p - 1]];
    S.method = P1.method;
    S.m = P1.m;
    S.s_first = P1.s;
    S.s_last = Pp.s;
    S.m_half = half.m;
    S.s_half = half.s;

    std::vector<SrcDev> sd;
    if ((rc = prepare_sources(G, src, nsrc, t0, 0, nsteps, stream, sd))) return rc;
    TraceDev tr;
    if ((rc = prepare_trace(G, trace, tr))) return rc;
    const bool tracing = tr.energy || tr.np > 0;
    if (tracing) {
        // rows i < p of the energy need the summed field: NaN with several ranks (paraexp.h)
        std::vector<double> init(p, world > 1 ? std::nan("") : 0.0);
        init[p - 1] = 0.0;
        if (tr.energy && (rc = dev_memcpy_h2d_async(tr.energy, init.data(), sizeof(double) * p, stream))) return rc;
        if (tr.np > 0 && (rc = dev_memset_async(tr.probe, 0, sizeof(double) * p * tr.np, stream))) return rc;
        if ((rc = dev_sync(stream))) return rc;
    }
    if ((rc = ensure_ws(G, 5))) return rc;
    KernelArgs ka{&G, stream, &S.kernel_launches};
    const size_t sbytes = (size_t)G.L.state_elems() * G.esize();
    const int64_t cells = (int64_t)G.nx * G.ny * G.nz;
    Events ev(stream);
    const int idt = ev.open(4);

    bool host_io = false;       // host-pointer fields (staged copies; the call syncs anyway)
    void *P = G.ws[0];          // particular state of the current sub-interval
    void *W = G.ws[1];          // Horner accumulator of the tails
    void *X[3] = {G.ws[2], G.ws[3], G.ws[4]};
    bool W_valid = false;
    int *dflag = (int *)G.d_flag;
    if ((rc = dev_memset_async(dflag, 0, sizeof(int) * (p + 2), stream))) return rc;

    auto propagate = [&](int i) -> int {   // W <- E_i W
        const int64_t M = B[i] - B[i - 1];
        if (tail_mode == PARAEXP_TAIL_EXP) {
            void *bufs[4] = {W, X[0], X[1], X[2]};
            int r = run_plan(ka, plans[M], bufs, &S, &ev);
            W = bufs[0];
            X[0] = bufs[1];
            X[1] = bufs[2];
            X[2] = bufs[3];
            return r;
        }
        void *bufs[2] = {W, X[0]};
        const int id5 = ev.open(5);
        int r = k_leapfrog(ka, bufs, M, nullptr, 0, nullptr);
        ev.close(id5);
        if (bufs[0] != W) std::swap(W, X[0]);
        S.leapfrog_steps += M;
        S.curl_applications += 2 * M;
        return r;
    };

    // f1: the Horner accumulator after sub-interval i (seed added) is this rank's share of the
    // same-time solution u(T_i) = v_i(T_i) + sum_{j<i} w_j(T_i)
    auto trace_row = [&](int i) -> int {
        int r = PARAEXP_OK;
        if (tr.np > 0) r = k_gather(ka, W, tr, tr.probe + (int64_t)(i - 1) * tr.np, 0);
        if (!r && tr.energy && world == 1) r = k_dot_M_async(ka, W, W, tr.energy + (i - 1), G.dt);
        return r;
    };

    // Concurrent particular sweeps (small grids): the sub-intervals of this rank's block are
    // independent leapfrog problems from zero (the parfor of PAPER:358-361).  When one sweep
    // cannot fill the GPU they run concurrently on side streams, each into its own buffer, and
    // the Horner chain on `stream` consumes them in order as they complete.
    const int nb = first >= 1 ? last - first + 1 : 0;
    const int nstr = std::min(nb, 8);
    const bool conc = nb >= 2 && nb <= 64 && concurrent_sweeps(G);
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
            if ((rc = dev_memset_async(Pc[q], 0, sbytes, kq.stream))) return rc;
            void *bufs[2] = {Pc[q], scratch[sq]};
            const size_t qoff = (size_t)B[i - 1] * nsrc * G.esize();
            if ((rc = k_leapfrog(kq, bufs, B[i] - B[i - 1], (const SrcDev *)G.d_src, nsrc,
                                 (const char *)G.d_q + qoff))) return rc;
            if (bufs[0] != Pc[q]) std::swap(Pc[q], scratch[sq]);   // result buffer <-> scratch
            if ((rc = k_check_finite_async(kq, Pc[q], dflag + i))) return rc;
            if (cudaEventRecord((cudaEvent_t)G.events[q], (cudaStream_t)kq.stream) != cudaSuccess)
                return check_cuda("event record");
            S.leapfrog_steps += B[i] - B[i - 1];
            S.curl_applications += 2 * (B[i] - B[i - 1]);
        }
        // keep the buffer roles for the next call (results may now live in former scratch)
        for (int q = 0; q < nb; ++q) G.conc[q] = Pc[q];
        for (int q = 0; q < nstr; ++q) G.conc[nb + q] = scratch[q];
    }

    if (first >= 1) {
        if (first == 1 && has_u0) {
            if ((rc = pack_any(ka, G, e0, h0, W, &host_io))) return rc;
            if (tail_mode == PARAEXP_TAIL_LEAPFROG && (rc = k_half_start(ka, W))) return rc;
            W_valid = true;
        }
        for (int i = first; i <= last; ++i) {
            const int64_t M = B[i] - B[i - 1];
            int id = ev.open(0);
            if (conc) {
                if (cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)G.events[i - first], 0) != cudaSuccess)
                    return check_cuda("stream wait");
                P = Pc[i - first];
            } else {
                if ((rc = dev_memset_async(P, 0, sbytes, stream))) return rc;
                void *bufs[2] = {P, X[0]};
                const size_t qoff = (size_t)B[i - 1] * nsrc * G.esize();
                const int id5 = ev.open(5);
                if ((rc = k_leapfrog(ka, bufs, M, (const SrcDev *)G.d_src, nsrc, (const char *)G.d_q + qoff))) return rc;
                ev.close(id5);
                if (bufs[0] != P) std::swap(P, X[0]);
                S.leapfrog_steps += M;
                S.curl_applications += 2 * M;
                if ((rc = k_check_finite_async(ka, P, dflag + i))) return rc;
            }
            ev.close(id);
            id = ev.open(1);
            if (W_valid && (rc = propagate(i))) return rc;
            if (i < p) {
                if (tail_mode == PARAEXP_TAIL_EXP && (rc = k_sync(ka, P))) return rc;
                if (W_valid) {
                    if ((rc = k_axpy(ka, W, P, 1.0))) return rc;
                } else {
                    if ((rc = dev_memcpy_d2d_async(W, P, sbytes, stream))) return rc;
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
    if (!W_valid && (rc = dev_memset_async(W, 0, sbytes, stream))) return rc;
    if ((rc = k_check_finite_async(ka, W, dflag + p + 1))) return rc;

    // a8: sum the tails onto the root
    // the collectives also run for a one-rank communicator when PARAEXP_FORCE_COLLECTIVES is
    // set, so the NCCL code path can be exercised on a single GPU (tests)
    const bool coll = comm && (world > 1 || getenv("PARAEXP_FORCE_COLLECTIVES"));
    if (coll) {
        const int id = ev.open(2);
        const int dt = G.dtype == PARAEXP_F64 ? kNcclF64 : kNcclF32;
        if ((rc = nccl_check(g_nccl.Reduce(W, W, (size_t)G.L.state_elems(), dt, kNcclSum, root,
                                          comm->comm, (cudaStream_t)stream), "ncclReduce"))) return rc;
        ev.close(id);
    }
    // a9: reconstruction on the root (eq:averaging1/2, reading 10)
    const int idf = ev.open(3);
    if (rank == root && tracing) {
        // row p: u(T_p) = sync(v_p) + W, same-time (reading 9)
        if ((rc = dev_memcpy_d2d_async(X[0], P, sbytes, stream))) return rc;
        if ((rc = k_sync(ka, X[0]))) return rc;
        if ((rc = k_axpy(ka, X[0], W, 1.0))) return rc;
        if (tr.np > 0 && (rc = k_gather(ka, X[0], tr, tr.probe + (int64_t)(p - 1) * tr.np, 0))) return rc;
        if (tr.energy && (rc = k_dot_M_async(ka, X[0], X[0], tr.energy + (p - 1), G.dt))) return rc;
    }
    if (tracing && coll) {
        if (tr.np > 0 && (rc = nccl_check(g_nccl.AllReduce(tr.probe, tr.probe, (size_t)p * tr.np, kNcclF64, kNcclSum,
                                                          comm->comm, (cudaStream_t)stream), "ncclAllReduce"))) return rc;
        if (tr.energy && (rc = nccl_check(g_nccl.AllReduce(tr.energy, tr.energy, (size_t)p, kNcclF64, kNcclSum,
                                                           comm->comm, (cudaStream_t)stream), "ncclAllReduce"))) return rc;
    }
    if (rank == root) {
        if (tail_mode == PARAEXP_TAIL_EXP) {
            if ((rc = k_axpy_comps(ka, P, W, 1.0, 0, 3))) return rc;       // e_out = e_p + W_e
            void *bufs[4] = {W, X[0], X[1], X[2]};
            if ((rc = run_plan(ka, half, bufs, nullptr))) return rc;       // exp(dt/2 A) W
            S.a_applications += (int64_t)half.s * half.m;
            if ((rc = k_axpy_comps(ka, P, bufs[0], 1.0, 3, 6))) return rc;  // h_out = h_p + [.]_h
        } else {
            if ((rc = k_axpy(ka, P, W, 1.0))) return rc;
        }
    }
    if (broadcast_out && coll) {
        const int dt = G.dtype == PARAEXP_F64 ? kNcclF64 : kNcclF32;
        if ((rc = nccl_check(g_nccl.Broadcast(P, P, (size_t)G.L.state_elems(), dt, root, comm->comm,
                                             (cudaStream_t)stream), "ncclBroadcast"))) return rc;
    }
    if ((rank == root || broadcast_out) && e_out && h_out) {
        if ((rc = unpack_any(ka, G, P, e_out, h_out, &host_io))) return rc;
    }
    ev.close(idf);
    ev.close(idt);
    S.curl_applications = 2 * (S.leapfrog_steps + S.a_applications);
    S.cell_updates = (S.leapfrog_steps + S.a_applications) * cells;
    std::vector<int> flags(p + 2, 0);
    if ((rc = dev_memcpy_d2h(flags.data(), dflag, sizeof(int) * (p + 2), stream))) return rc;
    if ((rc = sched_check(G, stream))) return rc;
    double ms[7] = {0, 0, 0, 0, 0, 0, 0};
    ev.sum(ms);
    S.ms_particular = ms[0];
    S.ms_tails = ms[1];
    S.ms_reduce = ms[2];
    S.ms_finish = ms[3];
    S.ms_total = ms[4];
    S.ms_leapfrog_kernels = ms[5];
    S.ms_poly_kernels = ms[6];
    for (int i = 1; i <= p; ++i)
        if (flags[i]) {
            S.fail_interval = i;
            return fail(PARAEXP_EDIVERGED, "leapfrog diverged in sub-interval " + std::to_string(i));
        }
    if (flags[p + 1]) {
        S.fail_interval = first;
        return fail(PARAEXP_EOVERFLOW, "exp(tA)v tails produced non-finite values");
    }
    return PARAEXP_OK;
}

}  // extern "C"
