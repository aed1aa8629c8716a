/* ranks_solve.c -- ParaExp's parfor through the C ABI's building blocks, from plain C: the
 * C3-shaped layered cavity (48x24x16 cells, Gaussian line current) split into p = 8
 * sub-intervals over `world` ranks that are simulated one after the other in this process --
 * each rank's paraexp_solve_block writes its tails W_r to HOST buffers, the host sums them (what
 * an MPI_Reduce would do), and paraexp_solve_finish reconstructs on the root.  The result is
 * compared with the one-call paraexp_solve (same plan, explicit rho): they differ only by
 * summation order.  Usage: ranks_solve [world] (default 3).
 *
 *   gcc -std=c11 -O2 -I include examples/ranks_solve.c -L paper_1705_08019_b200 \
 *       -l:libparaexp.so -Wl,-rpath,$PWD/paper_1705_08019_b200 -lm -o ranks_solve && ./ranks_solve 3 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

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

int main(int argc, char **argv) {
    const int world = argc > 1 ? atoi(argv[1]) : 3, p = 8;
    const int nx = 48, ny = 24, nz = 16;
    double *eps = malloc(sizeof(double) * nx * ny * nz);
    for (int k = 0; k < nz; ++k)                      /* four z-slabs, as C3 */
        for (int q = 0; q < nx * ny; ++q) eps[k * nx * ny + q] = (double[]){1.0, 2.2, 4.4, 9.8}[k / 4];
    paraexp_grid_desc d = {0};
    d.nx = nx;
    d.ny = ny;
    d.nz = nz;
    d.d0 = 1e-3;
    d.eps_r = eps;
    d.dtype = PARAEXP_F64;
    d.device = 0;
    d.dt_frac = 0.95;
    paraexp_grid *g = NULL;
    CHECK(paraexp_grid_create(&d, &g));
    paraexp_grid_info_t info;
    CHECK(paraexp_grid_info(g, 0, NULL, &info));
    paraexp_source src = {2, 24, 12, 4, PARAEXP_SRC_GAUSS_PAPER, 1.0, 1.0, 20e-12, 0.0, 0.0};
    const int64_t n = 3 * info.npts, nsteps = 160;
    paraexp_expmv_opts o = {PARAEXP_LEJA, 0, 0, 1e-10, info.rho_cfl, 0, 0.0, 0};

    double *we = malloc(sizeof(double) * n), *wh = malloc(sizeof(double) * n);
    double *se = calloc(n, sizeof(double)), *sh = calloc(n, sizeof(double));   /* sum of W_r */
    double *ve = calloc(n, sizeof(double)), *vh = calloc(n, sizeof(double));   /* root's v_p */
    int root = -1;
    for (int r = 0; r < world; ++r) {
        paraexp_stats st;
        CHECK(paraexp_solve_block(g, r, world, &src, 1, 0.0, nsteps, p, &o, PARAEXP_TAIL_EXP, NULL, NULL, we, wh,
                                  ve, vh, NULL, &st));
        for (int64_t q = 0; q < n; ++q) {
            se[q] += we[q];
            sh[q] += wh[q];
        }
        root = st.root;
        printf("rank %d/%d: sub-intervals [%d, %d], %lld leapfrog steps, %lld A-applications, %.2f ms\n", r, world,
               st.first_interval, st.last_interval, (long long)st.leapfrog_steps, (long long)st.a_applications,
               st.ms_total);
    }
    double *eo = malloc(sizeof(double) * n), *ho = malloc(sizeof(double) * n);
    CHECK(paraexp_solve_finish(g, &o, PARAEXP_TAIL_EXP, se, sh, ve, vh, eo, ho, NULL, NULL));
    double *e1 = malloc(sizeof(double) * n), *h1 = malloc(sizeof(double) * n);
    CHECK(paraexp_solve(g, NULL, &src, 1, 0.0, nsteps, p, &o, PARAEXP_TAIL_EXP, 0, NULL, NULL, e1, h1, NULL, NULL));
    double ne = 0, de = 0, nh = 0, dh = 0;
    for (int64_t q = 0; q < n; ++q) {
        ne += (eo[q] - e1[q]) * (eo[q] - e1[q]);
        de += e1[q] * e1[q];
        nh += (ho[q] - h1[q]) * (ho[q] - h1[q]);
        dh += h1[q] * h1[q];
    }
    printf("root %d; blocks + host sum + finish vs paraexp_solve: rel-L2 e = %.3e, h = %.3e\n", root,
           sqrt(ne / de), sqrt(nh / dh));
    paraexp_grid_destroy(g);
    free(eps);
    free(we);
    free(wh);
    free(se);
    free(sh);
    free(ve);
    free(vh);
    free(eo);
    free(ho);
    free(e1);
    free(h1);
    return (sqrt(ne / de) < 1e-12 && sqrt(nh / dh) < 1e-12) ? 0 : 2;
}
