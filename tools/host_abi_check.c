/* host_abi_check.c -- exercises every host-side entry point of the C ABI (no GPU needed): grid
 * creation on a HOST-ONLY grid (device -1) with uniform / non-uniform spacings, random eps/mu,
 * PEC cells and bad arguments; grid info and coefficient export; the planner (Taylor / Leja,
 * fixed and auto degrees, eps_A extremes); theta; Leja points; partition and the cost-balanced
 * schedule over many (p, world, ratio); eq:tolerance_leja_2; error strings.  Built by
 * tools/asan_host.sh with -fsanitize=address,undefined over the library's host sources so the
 * planner's and the grid assembly's memory accesses are checked (ASan/UBSan on the
 * host planner).  Exit status 0 = every call behaved as documented. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/paraexp.h"

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            fprintf(stderr, "check failed: %s (line %d): %s\n", #c, __LINE__, \
                    paraexp_last_error());                                    \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

static unsigned long long rng = 88172645463325252ull;
static double urand(void) {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return (double)(rng >> 11) / 9007199254740992.0;
}

static void grid_cases(void) {
    for (int t = 0; t < 24; ++t) {
        const int nx = 1 + (int)(urand() * 9), ny = 1 + (int)(urand() * 7), nz = 1 + (int)(urand() * 6);
        const long cells = (long)nx * ny * nz;
        double *dx = malloc(sizeof(double) * nx), *dy = malloc(sizeof(double) * ny);
        double *dz = malloc(sizeof(double) * nz), *eps = malloc(sizeof(double) * cells);
        double *mu = malloc(sizeof(double) * cells);
        unsigned char *pec = malloc(cells);
        for (int i = 0; i < nx; ++i) dx[i] = 1e-3 * (0.2 + urand());
        for (int i = 0; i < ny; ++i) dy[i] = 1e-3 * (0.2 + urand());
        for (int i = 0; i < nz; ++i) dz[i] = 1e-3 * (0.2 + urand());
        for (long c = 0; c < cells; ++c) {
            eps[c] = 1 + 10 * urand();
            mu[c] = 1 + urand();
            pec[c] = urand() < 0.15;
        }
        paraexp_grid_desc d;
        memset(&d, 0, sizeof d);
        d.nx = nx;
        d.ny = ny;
        d.nz = nz;
        d.dx = (t & 1) ? dx : NULL;
        d.dy = (t & 2) ? dy : NULL;
        d.dz = (t & 4) ? dz : NULL;
        d.d0 = 1e-3;
        d.eps_r = (t & 8) ? eps : NULL;
        d.mu_r = (t & 16) ? mu : NULL;
        d.pec_cell = (t % 3 == 0) ? pec : NULL;
        d.dtype = t % 2 ? PARAEXP_F32 : PARAEXP_F64;
        d.device = -1;
        d.dt_frac = 0.9;
        paraexp_grid *g = NULL;
        CHECK(paraexp_grid_create(&d, &g) >= 0 && g);
        if (g) {
            paraexp_grid_info_t info;
            CHECK(paraexp_grid_info(g, 0, NULL, &info) == PARAEXP_OK);
            CHECK(info.npts == (long)(nx + 1) * (ny + 1) * (nz + 1) && info.dt > 0 && info.dt < info.dt_cfl);
            double *cE = malloc(sizeof(double) * 3 * info.npts), *cH = malloc(sizeof(double) * 3 * info.npts);
            CHECK(paraexp_grid_coefficients(g, cE, cH) == PARAEXP_OK);
            for (long q = 0; q < 3 * info.npts; ++q) CHECK(cE[q] >= 0 && cH[q] >= 0 && isfinite(cE[q]));
            paraexp_plan_info pl;
            paraexp_expmv_opts o = {PARAEXP_LEJA, 0, 0, 1e-8, info.rho_cfl, 0, 0.0, 0};
            CHECK(paraexp_expmv_plan(g, 37 * info.dt, &o, &pl) == PARAEXP_OK && pl.m >= 8 && pl.s >= 1);
            free(cE);
            free(cH);
            paraexp_grid_destroy(g);
        }
        free(dx);
        free(dy);
        free(dz);
        free(eps);
        free(mu);
        free(pec);
    }
    /* invalid descriptors */
    paraexp_grid_desc d;
    memset(&d, 0, sizeof d);
    d.nx = 0;
    d.ny = 4;
    d.nz = 4;
    d.d0 = 1e-3;
    d.device = -1;
    d.dt_frac = 0.9;
    paraexp_grid *g = NULL;
    CHECK(paraexp_grid_create(&d, &g) == PARAEXP_EINVAL);
    d.nx = 4;
    d.dt = 1e-12;            /* both dt and dt_frac */
    CHECK(paraexp_grid_create(&d, &g) == PARAEXP_EINVAL);
    d.dt = 0;
    double bad[64];
    for (int i = 0; i < 64; ++i) bad[i] = i == 7 ? -1.0 : 1.0;
    d.eps_r = bad;
    CHECK(paraexp_grid_create(&d, &g) == PARAEXP_EINVAL);
}

static void planner_cases(void) {
    const double taus[] = {0.0, 0.3, 1.0, 7.5, 64.0, 500.0, 3790.0};
    const double eps[] = {1e-14, 1e-12, 1e-10, 1e-6, 1e-2, 0.5};
    for (int a = 0; a < 7; ++a)
        for (int b = 0; b < 6; ++b)
            for (int meth = 0; meth < 2; ++meth) {
                paraexp_plan_info p;
                const int rc = paraexp_plan_host(meth, 0, 0, eps[b], taus[a], 1.0, 1.0, &p);
                CHECK(rc == PARAEXP_OK || rc == PARAEXP_EINVAL);
                if (rc == PARAEXP_OK && taus[a] > 0) {
                    CHECK(p.s >= 1 && p.m >= 1 && p.m <= PARAEXP_MAX_DEGREE);
                    for (int k = 0; k <= p.m; ++k) CHECK(isfinite(p.d_re[k]) && isfinite(p.d_im[k]));
                }
            }
    const int ms[] = {1, 2, 8, 40, 98, 150};
    for (int q = 0; q < 6; ++q)
        for (int s = 1; s <= 3; ++s) {
            paraexp_plan_info p;
            CHECK(paraexp_plan_host(PARAEXP_LEJA, ms[q], s, 1e-10, 3.0 * ms[q], 1.0, 1.0, &p) == PARAEXP_OK);
            CHECK(paraexp_plan_host(PARAEXP_TAYLOR, ms[q], s, 1e-10, 0.5 * ms[q], 1.0, 1.0, &p) == PARAEXP_OK);
        }
    paraexp_plan_info p;
    CHECK(paraexp_plan_host(PARAEXP_LEJA, 3, 1, 1e-10, 1.0, 1.0, 1.0, &p) == PARAEXP_EINVAL);   /* odd m */
    CHECK(paraexp_plan_host(PARAEXP_LEJA, 152, 1, 1e-10, 1.0, 1.0, 1.0, &p) == PARAEXP_EINVAL);
    CHECK(paraexp_theta(PARAEXP_LEJA, 64, 1e-10) > 30 && paraexp_theta(PARAEXP_TAYLOR, 16, 1e-13) > 1);
    double xi[151];
    CHECK(paraexp_leja_points(151, xi) == PARAEXP_OK && xi[0] == 1.0 && xi[1] == -1.0 && xi[2] == 0.0);
    int32_t clamped = 0;
    CHECK(paraexp_optimal_tolerance(1e-12, 1.0, 1e12, &clamped) == 1e-14 && clamped == 1);
    CHECK(paraexp_optimal_tolerance(-1.0, 1.0, 1.0, NULL) == 0.1);
}

static void schedule_cases(void) {
    const double ratios[] = {0.0, 0.4, 1.0, 2.64, 16.0};
    for (int p = 1; p <= 70; p += 3)
        for (int world = 1; world <= 9; ++world)
            for (int q = 0; q < 5; ++q)
                for (int u0 = 0; u0 < 2; ++u0) {
                    int next = 1, roots = -1, ok = 1;
                    for (int r = 0; r < world; ++r) {
                        int32_t f, l, root;
                        CHECK(paraexp_schedule(p, world, r, ratios[q], u0, &f, &l, &root) == PARAEXP_OK);
                        if (roots < 0) roots = root;
                        ok &= root == roots;
                        if (f >= 1) {
                            ok &= f == next && l >= f;
                            next = l + 1;
                            if (l == p) ok &= root == r;
                        } else {
                            ok &= l == -1;
                        }
                    }
                    ok &= next == p + 1;
                    CHECK(ok);
                }
    int32_t f, l, root;
    CHECK(paraexp_schedule(0, 2, 0, 1.0, 0, &f, &l, &root) == PARAEXP_EINVAL);
    CHECK(paraexp_schedule(4, 2, 2, 1.0, 0, &f, &l, &root) == PARAEXP_EINVAL);
    int64_t b[9];
    CHECK(paraexp_partition(103, 4, b) == PARAEXP_OK && b[4] == 103 && b[3] - b[2] == 25 && b[4] - b[3] == 28);
    CHECK(paraexp_partition(3, 4, b) == PARAEXP_EINVAL);
}

int main(void) {
    grid_cases();
    planner_cases();
    schedule_cases();
    for (int c = -8; c <= 1; ++c) CHECK(paraexp_strerror(c) != NULL);
    printf("%s (%s): %d failed checks\n", paraexp_version(), failures ? "FAIL" : "ok", failures);
    return failures ? 1 : 0;
}
