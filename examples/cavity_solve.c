/* cavity_solve.c -- the C ABI used from plain C (no Python, no CUDA API calls): an 8^3 PEC
 * cavity (BASELINE config C1: 1 mm cells, vacuum, 0.9 dt_CFL, Gaussian-modulated sine on
 * z-edge (3,5,4)) solved by ParaExp with p = 2 sub-intervals and by serial leapfrog, both with
 * HOST field buffers (the library stages them).  Prints the relative difference, the
 * discretisation gap between the exponential tails and leapfrog (O(dt^2), small but not 0).
 *
 *   gcc -std=c11 -O2 -I include examples/cavity_solve.c -L paper_1705_08019_b200 \
 *       -l:libparaexp.so -Wl,-rpath,$PWD/paper_1705_08019_b200 -lm -o cavity_solve && ./cavity_solve */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "paraexp.h"

#define CHECK(x)                                                                       \
    do {                                                                               \
        int rc_ = (x);                                                                 \
        if (rc_ < 0) {                                                                 \
            fprintf(stderr, "%s failed: %s (%s)\n", #x, paraexp_strerror(rc_),        \
                    paraexp_last_error());                                             \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(void) {
    paraexp_grid_desc d = {0};
    d.nx = d.ny = d.nz = 8;
    d.d0 = 1e-3;
    d.dtype = PARAEXP_F64;
    d.device = 0;
    d.dt_frac = 0.9;
    d.kernels = PARAEXP_KERNELS_AUTO;
    paraexp_grid *g = NULL;
    CHECK(paraexp_grid_create(&d, &g));
    paraexp_grid_info_t info;
    CHECK(paraexp_grid_info(g, 0, NULL, &info));

    const double pi = 3.14159265358979323846, bw = 50e9, tau = 2.0 / (pi * bw);
    paraexp_source src = {2, 3, 5, 4, PARAEXP_SRC_GAUSS_SINE, 1.0, 1.0, tau, 100e9, 4.0 * tau};
    const int64_t n = 3 * info.npts, nsteps = 2000;
    /* ParaExp outputs in pinned host memory from the library (fast copy-out), the leapfrog
     * state in ordinary pageable memory: both are valid host field arguments */
    double *e = NULL, *h = NULL;
    CHECK(paraexp_host_alloc(n * sizeof(double), (void **)&e));
    CHECK(paraexp_host_alloc(n * sizeof(double), (void **)&h));
    memset(e, 0, n * sizeof(double));
    memset(h, 0, n * sizeof(double));
    double *el = calloc(n, sizeof(double)), *hl = calloc(n, sizeof(double));

    paraexp_expmv_opts o = {PARAEXP_LEJA, 0, 0, 1e-12, 0.0, 0, 0.0};
    paraexp_stats st;
    CHECK(paraexp_solve(g, NULL, &src, 1, 0.0, nsteps, 2, &o, PARAEXP_TAIL_EXP, 0, NULL, NULL, e, h,
                        NULL, &st));
    CHECK(paraexp_leapfrog(g, &src, 1, 0.0, nsteps, el, hl, 0, NULL, NULL));
    double num = 0, den = 0;
    for (int64_t q = 0; q < n; ++q) {
        num += (e[q] - el[q]) * (e[q] - el[q]);
        den += el[q] * el[q];
    }
    printf("%s: %dx%dx%d cells, dt = %.6e s, %lld steps, p = 2: %lld A-applications (m = %d, s = %d), "
           "%lld kernel launches; ||e_paraexp - e_leapfrog|| / ||e_leapfrog|| = %.3e\n",
           paraexp_version(), info.nx, info.ny, info.nz, info.dt, (long long)nsteps,
           (long long)st.a_applications, st.m, st.s_first, (long long)st.kernel_launches,
           sqrt(num / den));
    paraexp_host_free(e);
    paraexp_host_free(h);
    free(el);
    free(hl);
    paraexp_grid_destroy(g);
    return 0;
}
