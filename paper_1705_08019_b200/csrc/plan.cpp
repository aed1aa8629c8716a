// plan.cpp -- host planner for exp(tau A) v (row a5): Leja sequence, scaled Newton
// coefficients, theta_m criterion, (m, s) selection and the real conjugate-pair schedule.
//
// PAPER:404-448 (scaling + polynomial recurrence; Leja's method on an imaginary interval),
// DESIGN readings 14-16.  Written independently of oracle/ (which uses an mpmath
// divided-difference table; here: first column of exp(gamma Z) for the bidiagonal node
// matrix Z, Taylor-stepped in __float128).
#include <algorithm>
#include <cmath>
#include <complex>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.h"

namespace pe {

// ---- Leja sequence (reading 14) -------------------------------------------------------
// xi = (1, -1, 0, +eta_1, -eta_1, ...), eta_l maximising
//   log|c| + sum_{p in {1, eta_1..eta_{l-1}}} log|c^2 - p^2|   over c = k/5000, k = 1..5000
// (first maximum wins: ties -> smallest eta).
static std::mutex g_leja_mu;
static std::vector<double> g_leja;

void leja_sequence(int count, std::vector<double> &xi) {
    std::lock_guard<std::mutex> lk(g_leja_mu);
    if ((int)g_leja.size() < count) {
        std::vector<double> seq = {1.0, -1.0, 0.0};
        std::vector<double> pos = {1.0};
        const int need = std::max(count, PARAEXP_MAX_DEGREE + 1);
        std::vector<double> cand(5000), base(5000);
        for (int k = 1; k <= 5000; ++k) {
            cand[k - 1] = k / 5000.0;
            base[k - 1] = std::log(std::fabs(cand[k - 1]));
        }
        // accumulated objective, updated incrementally in selection order
        std::vector<double> obj = base;
        for (int k = 0; k < 5000; ++k) obj[k] = obj[k] + std::log(std::fabs(cand[k] * cand[k] - 1.0 * 1.0));
        while ((int)seq.size() < need) {
            int best = 0;
            for (int k = 1; k < 5000; ++k)
                if (obj[k] > obj[best]) best = k;
            const double eta = cand[best];
            pos.push_back(eta);
            seq.push_back(eta);
            seq.push_back(-eta);
            for (int k = 0; k < 5000; ++k) obj[k] = obj[k] + std::log(std::fabs(cand[k] * cand[k] - eta * eta));
        }
        g_leja = seq;
    }
    xi.assign(g_leja.begin(), g_leja.begin() + count);
}

// ---- divided differences of exp(gamma*xi) on imaginary nodes i*y_k ----------------------
// d_k = g[xi_0..xi_k] is the first column of g(Z), Z = diag(xi_k) + subdiag(1) (Opitz).
// exp(gamma Z) e_0 = (exp(gamma Z / S))^S e_0, each factor a Taylor series to full
// precision; ||gamma Z / S|| <= 1/2.
template <typename R>
static void divdiff_exp_imag(const std::vector<double> &y, double gamma, std::vector<R> &vr,
                             std::vector<R> &vi, R eps) {
    const int n = (int)y.size();
    double ymax = 0;
    for (double v : y) ymax = std::max(ymax, std::fabs(v));
    const int S = std::max(1, (int)std::ceil(2.0 * gamma * (ymax + 1.0)));
    const R g = (R)gamma / (R)S;
    vr.assign(n, (R)0);
    vi.assign(n, (R)0);
    vr[0] = 1;
    std::vector<R> tr(n), ti(n), nr(n), ni(n), ar(n), ai(n);
    for (int st = 0; st < S; ++st) {
        tr = vr;
        ti = vi;
        ar = vr;
        ai = vi;
        for (int it = 1; it < 200; ++it) {
            // t <- (g / it) * Z t ;  (Z t)_k = i y_k t_k + t_{k-1}
            R amax = 0, tmax = 0;
            for (int k = n - 1; k >= 0; --k) {
                R zr = -(R)y[k] * ti[k];
                R zi = (R)y[k] * tr[k];
                if (k > 0) {
                    zr += tr[k - 1];
                    zi += ti[k - 1];
                }
                nr[k] = zr * g / (R)it;
                ni[k] = zi * g / (R)it;
            }
            for (int k = 0; k < n; ++k) {
                tr[k] = nr[k];
                ti[k] = ni[k];
                ar[k] += tr[k];
                ai[k] += ti[k];
                R ta = tr[k] < 0 ? -tr[k] : tr[k];
                R tb = ti[k] < 0 ? -ti[k] : ti[k];
                R aa = ar[k] < 0 ? -ar[k] : ar[k];
                R ab = ai[k] < 0 ? -ai[k] : ai[k];
                tmax = std::max(tmax, std::max(ta, tb));
                amax = std::max(amax, std::max(aa, ab));
            }
            if (tmax <= eps * amax) break;
        }
        vr = ar;
        vi = ai;
    }
}

// Evaluation order of the degree-m node set (DESIGN reading 29): the greedy prefix
// (1, -1, 0, +eta_1, -eta_1, ..., +eta_L, -eta_L) with the zero node moved last, so that every
// conjugate pair is closed and the zero-node term folds into the final pair.
static void newton_order(int m, std::vector<double> &xi) {
    std::vector<double> g;
    leja_sequence(m + 1, g);
    xi.clear();
    if (m == 1) {
        xi = {g[0], g[1]};
        return;
    }
    xi.push_back(g[0]);
    xi.push_back(g[1]);
    for (int k = 3; k <= m; ++k) xi.push_back(g[k]);
    xi.push_back(g[2]);
}

static void leja_coefficients(int m, double gamma, std::vector<double> &xi,
                              std::vector<double> &dre, std::vector<double> &dim,
                              bool quad) {
    newton_order(m, xi);
    std::vector<double> y(m + 1);
    for (int k = 0; k <= m; ++k) y[k] = 2.0 * xi[k];   // capacity-scaled nodes 2i*xi'_k
    dre.resize(m + 1);
    dim.resize(m + 1);
    if (quad) {
        std::vector<__float128> vr, vi;
        divdiff_exp_imag<__float128>(y, gamma, vr, vi, (__float128)1e-36);
        for (int k = 0; k <= m; ++k) {
            dre[k] = (double)vr[k];
            dim[k] = (double)vi[k];
        }
    } else {
        std::vector<long double> vr, vi;
        divdiff_exp_imag<long double>(y, gamma, vr, vi, 1e-21L);
        for (int k = 0; k <= m; ++k) {
            dre[k] = (double)vr[k];
            dim[k] = (double)vi[k];
        }
    }
}

static void taylor_coefficients(int m, std::vector<double> &dre, std::vector<double> &dim) {
    dre.resize(m + 1);
    dim.assign(m + 1, 0.0);
    __float128 f = 1;
    for (int k = 0; k <= m; ++k) {
        if (k > 0) f *= k;
        dre[k] = (double)((__float128)1 / f);
    }
}

// ---- theta_m (reading 16; the oracle side is pinned in tests/test_oracle_theta.py) -----------
// max over x = j*theta/800, j = 0..800, of |p(ix) - e^{ix}|; p interpolates exp on
// i[-a, a], a = 1.05 theta (Leja), or is the degree-m Taylor polynomial.
static double poly_error(int method, int m, double theta) {
    std::vector<double> xi, dre, dim;
    double gamma = 1.0;
    std::vector<double> ny(m + 1, 0.0);
    if (method == PARAEXP_LEJA) {
        gamma = 1.05 * theta / 2.0;
        leja_coefficients(m, gamma, xi, dre, dim, false);
        for (int k = 0; k <= m; ++k) ny[k] = 2.0 * xi[k];
    } else {
        taylor_coefficients(m, dre, dim);
    }
    double err = 0;
    const double step = theta / 800.0;
    for (int jx = 0; jx <= 800; ++jx) {
        const double x = jx * step;
        const std::complex<double> lam(0.0, x / gamma);
        std::complex<double> yv(0, 0), w(1, 0);
        for (int k = 0; k <= m; ++k) {
            yv += std::complex<double>(dre[k], dim[k]) * w;
            w = w * (lam - std::complex<double>(0.0, ny[k]));
        }
        err = std::max(err, std::abs(yv - std::complex<double>(std::cos(x), std::sin(x))));
    }
    return err;
}

static std::mutex g_theta_mu;
static std::map<std::tuple<int, int, double>, double> g_theta;

double theta_m(int method, int m, double tol) {
    auto key = std::make_tuple(method, m, tol);
    {
        std::lock_guard<std::mutex> lk(g_theta_mu);
        auto it = g_theta.find(key);
        if (it != g_theta.end()) return it->second;
    }
    double lo = 0.0, hi = (double)(2 * m + 4);
    for (int it = 0; it < 40; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid > 0 && poly_error(method, m, mid) <= tol * mid)
            lo = mid;
        else
            hi = mid;
    }
    std::lock_guard<std::mutex> lk(g_theta_mu);
    g_theta[key] = lo;
    return lo;
}

// ---- schedule of one substep (DESIGN a6) ------------------------------------------------
static void build_ops(Plan &p) {
    // conjugate pairs (k, k+1), k = 0, 2, ..., m-2; the last one also adds Re d_m * w_m
    p.ops.clear();
    const int m = p.m;
    auto eta_at = [&](int k) { return p.node_im.empty() ? 0.0 : std::fabs(p.node_im[k]); };
    for (int k = 0; k < std::max(m, 1); k += 2) {
        Op o;
        const double eta = eta_at(k);
        o.kind = m == 1 ? 1 : (k == m - 2 ? 2 : 0);
        o.a = p.d_re[k] + eta * p.d_im[k + 1];
        o.b = p.d_re[k + 1];
        o.e2 = eta * eta;
        o.c = o.kind == 2 ? p.d_re[k + 2] : 0.0;
        p.ops.push_back(o);
    }
}

static int make_plan_uncached(int method, int m, int s, double eps_A, double tau, double rho, double dt,
                              Plan &out);

// Plans are pure functions of their arguments; building the Newton coefficients (quad
// precision, m up to 100) costs up to ~0.3 s on the host, which a ParaExp solve would
// otherwise pay on every call while the GPU idles.  Memoise them (bounded).
int make_plan(int method, int m, int s, double eps_A, double tau, double rho, double dt, Plan &out) {
    using Key = std::tuple<int, int, int, double, double, double, double>;
    static std::mutex mu;
    static std::map<Key, Plan> cache;
    const Key key{method, m, s, eps_A, tau, rho, dt};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            out = it->second;
            return PARAEXP_OK;
        }
    }
    int rc = make_plan_uncached(method, m, s, eps_A, tau, rho, dt, out);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 512) cache.clear();
    cache.emplace(key, out);
    return PARAEXP_OK;
}

static int make_plan_uncached(int method, int m, int s, double eps_A, double tau, double rho, double dt,
                              Plan &out) {
    if (method == PARAEXP_KRYLOV) {
        // f3: Krylov plan = subspace dimension l = m and substeps s (reading 31)
        if (!(tau >= 0) || !std::isfinite(tau)) return fail(PARAEXP_EINVAL, "tau must be >= 0");
        if (!(rho >= 0) || !std::isfinite(rho)) return fail(PARAEXP_EINVAL, "rho must be >= 0");
        if (m < 1 || m > PARAEXP_MAX_DEGREE) return fail(PARAEXP_EINVAL, "Krylov dimension m must be in 1..150");
        if (s < 0) return fail(PARAEXP_EINVAL, "s must be >= 0");
        out = Plan();
        out.method = method;
        out.tau = tau;
        out.rho = rho;
        out.m = m;
        out.gamma = 1.0;
        if (tau == 0.0) {
            out.s = 0;
            out.sigma = 0;
            return PARAEXP_OK;
        }
        out.s = s > 0 ? s : (int)std::max(1.0, std::ceil(2.0 * rho * tau / m));
        out.sigma = (tau / out.s) / dt;      // X = h A_orig through the stencil scale sigma*dt
        return PARAEXP_OK;
    }
    if (method != PARAEXP_LEJA && method != PARAEXP_TAYLOR) return fail(PARAEXP_EINVAL, "bad method");
    if (!(tau >= 0) || !std::isfinite(tau)) return fail(PARAEXP_EINVAL, "tau must be >= 0");
    if (!(rho >= 0) || !std::isfinite(rho)) return fail(PARAEXP_EINVAL, "rho must be >= 0");
    if (m < 0 || m > PARAEXP_MAX_DEGREE || (m > 1 && m % 2)) return fail(PARAEXP_EINVAL, "degree m must be 1 or even and <= 150");
    if (s < 0) return fail(PARAEXP_EINVAL, "s must be >= 0");
    if ((m == 0 || s == 0) && !(eps_A >= 1e-14 && eps_A < 1)) return fail(PARAEXP_EINVAL, "eps_A must lie in [1e-14, 1)");
    out = Plan();
    out.method = method;
    out.tau = tau;
    out.rho = rho;
    if (tau == 0.0) {   // identity: no substeps
        out.m = m > 0 ? m : 1;
        out.s = 0;
        out.gamma = 1;
        out.sigma = 0;
        return PARAEXP_OK;
    }
    const double tr = tau * rho;
    if (m == 0) {
        if (method == PARAEXP_LEJA) {
            // every admissible degree (even m in [8, 150], reading 16): for each substep count s
            // from the fewest possible (theta_150) upwards, the smallest m whose per-substep
            // criterion holds at theta = tau rho / s (bisection over m on poly_error, one
            // polynomial per probe); keep the least m * s (the A-applications of the plan)
            const int mmax = PARAEXP_MAX_DEGREE;
            const double thmax = theta_m(method, mmax, eps_A);
            if (!(thmax > 0)) return fail(PARAEXP_EINVAL, "no degree satisfies eps_A");
            const long s0 = s > 0 ? s : std::max(1L, (long)std::ceil(tr / thmax));
            if (s > 0 && s0 * thmax < tr) return fail(PARAEXP_EINVAL, "no degree satisfies eps_A at the given s");
            long best = -1;
            for (long sq = s0; sq <= (s > 0 ? s0 : s0 + 4); ++sq) {
                const double th = tr / (double)sq;
                auto ok = [&](int mm) { return poly_error(method, mm, th) <= eps_A * th; };
                int lo = 4, hi = mmax / 2;                       // m = 2 * half
                if (!ok(2 * hi)) continue;
                while (lo < hi) {
                    const int mid = (lo + hi) / 2;
                    if (ok(2 * mid)) hi = mid; else lo = mid + 1;
                }
                const long cost = sq * 2 * lo;
                if (best < 0 || cost < best) {
                    best = cost;
                    out.m = 2 * lo;
                    out.s = (int)sq;
                }
            }
            if (best < 0) return fail(PARAEXP_EINVAL, "no degree satisfies eps_A at the given s");
        } else {
            static const int tay_c[] = {4, 8, 12, 16, 20, 24, 32, 40, 48};
            long best = -1;
            for (int q = 0; q < 9; ++q) {
                const double th = theta_m(method, tay_c[q], eps_A);
                if (!(th > 0)) continue;
                const long sq = s > 0 ? s : std::max(1L, (long)std::ceil(tr / th));
                if (s > 0 && sq * th < tr) continue;
                const long cost = sq * tay_c[q];
                if (best < 0 || cost < best) {
                    best = cost;
                    out.m = tay_c[q];
                    out.s = (int)sq;
                }
            }
            if (best < 0) return fail(PARAEXP_EINVAL, "no degree satisfies eps_A at the given s");
        }
    } else {
        out.m = m;
        if (s > 0) {
            out.s = s;
        } else {
            const double th = theta_m(method, m, eps_A);
            if (!(th > 0)) return fail(PARAEXP_EINVAL, "degree too low for eps_A");
            out.s = (int)std::max(1L, (long)std::ceil(tr / th));
        }
    }
    const double h = tau / out.s;
    if (method == PARAEXP_LEJA && rho > 0) {
        out.a = 1.05 * h * rho;
        out.gamma = out.a / 2.0;
        leja_coefficients(out.m, out.gamma, out.xi, out.d_re, out.d_im, true);
        out.node_im.resize(out.m + 1);
        for (int k = 0; k <= out.m; ++k) out.node_im[k] = 2.0 * out.xi[k];
    } else {   // Taylor (c = 0), also Leja with a degenerate interval
        out.a = 0;
        out.gamma = 1.0;
        taylor_coefficients(out.m, out.d_re, out.d_im);
        if (method == PARAEXP_LEJA) newton_order(out.m, out.xi);
    }
    out.sigma = h / (out.gamma * dt);
    build_ops(out);
    return PARAEXP_OK;
}

void plan_to_info(const Plan &p, paraexp_plan_info *o) {
    *o = paraexp_plan_info();
    o->method = p.method;
    o->m = p.m;
    o->s = p.s;
    o->n_ops = (int)p.ops.size();
    o->tau = p.tau;
    o->rho = p.rho;
    o->a = p.a;
    o->gamma = p.gamma;
    o->sigma = p.sigma;
    for (size_t k = 0; k < p.xi.size() && k <= PARAEXP_MAX_DEGREE; ++k) o->xi[k] = p.xi[k];
    for (size_t k = 0; k < p.d_re.size() && k <= PARAEXP_MAX_DEGREE; ++k) {
        o->d_re[k] = p.d_re[k];
        o->d_im[k] = p.d_im[k];
    }
}

}  // namespace pe

extern "C" {

int paraexp_leja_points(int32_t count, double *xi) {
    if (count < 1 || count > 4 * PARAEXP_MAX_DEGREE || !xi) return pe::fail(PARAEXP_EINVAL, "bad count");
    std::vector<double> v;
    pe::leja_sequence(count, v);
    std::copy(v.begin(), v.end(), xi);
    return PARAEXP_OK;
}

double paraexp_optimal_tolerance(double dt, double beta, double norm_A, int32_t *clamped) {
    if (clamped) *clamped = 0;
    const double v = beta * dt * dt / norm_A;
    if (!(dt > 0) || !(beta > 0) || !(norm_A > 0) || !std::isfinite(v)) {
        if (clamped) *clamped = 1;
        return 0.1;
    }
    if (v < 1e-14 || v > 0.1) {
        if (clamped) *clamped = 1;
        return v < 1e-14 ? 1e-14 : 0.1;
    }
    return v;
}

double paraexp_theta(int32_t method, int32_t m, double eps_A) {
    if (m < 1 || m > PARAEXP_MAX_DEGREE || !(eps_A > 0)) return -1.0;
    return pe::theta_m(method, m, eps_A);
}

int paraexp_plan_host(int32_t method, int32_t m, int32_t s, double eps_A, double tau,
                      double rho, double dt, paraexp_plan_info *out) {
    if (!out || !(dt > 0)) return pe::fail(PARAEXP_EINVAL, "bad arguments");
    pe::Plan p;
    int rc = pe::make_plan(method, m, s, eps_A, tau, rho, dt, p);
    if (rc) return rc;
    pe::plan_to_info(p, out);
    return PARAEXP_OK;
}

}  // extern "C"
