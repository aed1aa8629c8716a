/*
 * fit_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU definitions of the FIT operators and the
 * leapfrog iteration of arXiv:1705.08019.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file.  It
 * shares no code, header, table or constant generator with the CUDA library
 * (paper_1705_08019_b200/csrc); it is written independently from the paper.
 *
 * Citations: PAPER:n = /root/reference/PAPER.md line n (not needed at run time).
 *
 * Layout ("canonical"): every field component is an array of
 *   Np = (nx+1)(ny+1)(nz+1) primal points, index P(i,j,k) = i + (nx+1)(j + (ny+1)k),
 * x fastest.  A vector of one field is 3*Np doubles: comp 0 (x), 1 (y), 2 (z).
 *   e_x(i,j,k): primal edge (i,j,k)->(i+1,j,k)        (virtual at i = nx)
 *   h_z(i,j,k): dual edge through the primal z-face spanned by e_x(i,j,k), e_y(i,j,k)
 * Out-of-range neighbours (index > n or < 0) read as 0 (virtual entries).
 *
 * All arithmetic is fp64.  Loops are plain; OpenMP only splits the outer k loop
 * (no blocking, no fusion, no reordering of the per-entry arithmetic).  Every entry is
 * computed independently, so the thread count never changes a result; grids below
 * OR_OMP_MIN points per component run on one thread (a fork/join per half-step costs more
 * than the loop there, and oversubscribes the host when tests run in parallel).
 */
#include <math.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>

#define OR_OMP_MIN 32768L

typedef struct {
    int nx, ny, nz;
} dims_t;

static inline long P(const dims_t *d, long i, long j, long k) {
    return i + (long)(d->nx + 1) * (j + (long)(d->ny + 1) * k);
}

/* read component array a at (i,j,k); 0 outside the point lattice */
static inline double rd(const dims_t *d, const double *a, long i, long j, long k) {
    if (i < 0 || j < 0 || k < 0 || i > d->nx || j > d->ny || k > d->nz) return 0.0;
    return a[P(d, i, j, k)];
}

/* ------------------------------------------------------------------------ */
/* FIT material matrices (eq:maxwell_grid3; DESIGN reading 4/5)
 *
 *  M_eps(x-edge i,j,k) = sum_{cells (i,jj,kk), jj in {j-1,j}, kk in {k-1,k}, existing}
 *                        eps0*eps_r(cell) * (dy_jj/2)*(dz_kk/2)  /  dx_i
 *  (y-, z-edges by cyclic permutation).  Edges with i = nx (x) etc. are virtual: 0.
 *
 *  M_nu(z-face i,j,k) = [ sum_{kk in {k-1,k}, existing} (dz_kk/2)/(mu0*mu_r(i,j,kk)) ] / (dx_i*dy_j)
 *  Faces with i = nx or j = ny (z) are virtual: 0.
 *
 *  live_e = 1 for an edge that is neither virtual, nor tangential to the PEC box
 *  boundary, nor an edge of a PEC cell (DESIGN reading 5).
 *  live_h = 1 for a face that is neither virtual nor normal to the box boundary.
 */
void or_fit_matrices(int nx, int ny, int nz, const double *dx, const double *dy, const double *dz,
                     const double *eps_r, const double *mu_r, const unsigned char *pec_cell,
                     double eps0, double mu0,
                     double *Meps, double *Mnu, unsigned char *live_e, unsigned char *live_h) {
    dims_t D = {nx, ny, nz};
    const dims_t *d = &D;
    long Np = (long)(nx + 1) * (ny + 1) * (nz + 1);
    int n[3] = {nx, ny, nz};
    const double *sp[3] = {dx, dy, dz};
#define CELL(ci, cj, ck) ((ci) + (long)nx * ((cj) + (long)ny * (ck)))
    for (int c = 0; c < 3; ++c) {
        int a = c, b = (c + 1) % 3, g = (c + 2) % 3; /* edge axis a, transverse b, g */
        for (long k = 0; k <= nz; ++k)
            for (long j = 0; j <= ny; ++j)
                for (long i = 0; i <= nx; ++i) {
                    long idx[3] = {i, j, k};
                    long p = (long)c * Np + P(d, i, j, k);
                    /* ---- edge along axis a starting at point idx ---- */
                    double me = 0.0;
                    int edge_exists = idx[a] < n[a];
                    int on_wall = (idx[b] == 0 || idx[b] == n[b] || idx[g] == 0 || idx[g] == n[g]);
                    int touches_pec = 0;
                    if (edge_exists) {
                        for (int ob = -1; ob <= 0; ++ob)
                            for (int og = -1; og <= 0; ++og) {
                                long cidx[3];
                                cidx[a] = idx[a];
                                cidx[b] = idx[b] + ob;
                                cidx[g] = idx[g] + og;
                                if (cidx[b] < 0 || cidx[b] >= n[b] || cidx[g] < 0 || cidx[g] >= n[g]) continue;
                                long cell = CELL(cidx[0], cidx[1], cidx[2]);
                                double er = eps_r ? eps_r[cell] : 1.0;
                                me += eps0 * er * (sp[b][cidx[b]] * 0.5) * (sp[g][cidx[g]] * 0.5);
                                if (pec_cell && pec_cell[cell]) touches_pec = 1;
                            }
                        me /= sp[a][idx[a]];
                    }
                    Meps[p] = me;
                    live_e[p] = (unsigned char)(edge_exists && !on_wall && !touches_pec);
                    /* ---- face with normal axis a at point idx (spanned by b,g edges) ---- */
                    double mn = 0.0;
                    int face_exists = idx[b] < n[b] && idx[g] < n[g];
                    int normal_wall = (idx[a] == 0 || idx[a] == n[a]);
                    if (face_exists) {
                        for (int oa = -1; oa <= 0; ++oa) {
                            long cidx[3];
                            cidx[a] = idx[a] + oa;
                            cidx[b] = idx[b];
                            cidx[g] = idx[g];
                            if (cidx[a] < 0 || cidx[a] >= n[a]) continue;
                            long cell = CELL(cidx[0], cidx[1], cidx[2]);
                            double mr = mu_r ? mu_r[cell] : 1.0;
                            mn += (sp[a][cidx[a]] * 0.5) / (mu0 * mr);
                        }
                        mn /= (sp[b][idx[b]] * sp[g][idx[g]]);
                    }
                    Mnu[p] = mn;
                    live_h[p] = (unsigned char)(face_exists && !normal_wall);
                }
    }
#undef CELL
}

/* ------------------------------------------------------------------------ */
/* Discrete curls (eq:maxwell_grid1; SURVEY 8a stencils).
 * out = C e   (faces)      out = C^T h  (edges).  Right-handed, topological. */
static inline double curl_x(const dims_t *d, const double *ex, const double *ey, const double *ez,
                            long i, long j, long k) {
    (void)ex;
    return rd(d, ey, i, j, k) + rd(d, ez, i, j + 1, k) - rd(d, ey, i, j, k + 1) - rd(d, ez, i, j, k);
}
static inline double curl_y(const dims_t *d, const double *ex, const double *ey, const double *ez,
                            long i, long j, long k) {
    (void)ey;
    return rd(d, ez, i, j, k) + rd(d, ex, i, j, k + 1) - rd(d, ez, i + 1, j, k) - rd(d, ex, i, j, k);
}
static inline double curl_z(const dims_t *d, const double *ex, const double *ey, const double *ez,
                            long i, long j, long k) {
    (void)ez;
    return rd(d, ex, i, j, k) + rd(d, ey, i + 1, j, k) - rd(d, ex, i, j + 1, k) - rd(d, ey, i, j, k);
}
static inline double curlT_x(const dims_t *d, const double *hx, const double *hy, const double *hz,
                             long i, long j, long k) {
    (void)hx;
    return rd(d, hz, i, j, k) - rd(d, hz, i, j - 1, k) - rd(d, hy, i, j, k) + rd(d, hy, i, j, k - 1);
}
static inline double curlT_y(const dims_t *d, const double *hx, const double *hy, const double *hz,
                             long i, long j, long k) {
    (void)hy;
    return rd(d, hx, i, j, k) - rd(d, hx, i, j, k - 1) - rd(d, hz, i, j, k) + rd(d, hz, i - 1, j, k);
}
static inline double curlT_z(const dims_t *d, const double *hx, const double *hy, const double *hz,
                             long i, long j, long k) {
    (void)hz;
    return rd(d, hy, i, j, k) - rd(d, hy, i - 1, j, k) - rd(d, hx, i, j, k) + rd(d, hx, i, j - 1, k);
}

void or_curl(int nx, int ny, int nz, const double *e, double *out) {
    dims_t D = {nx, ny, nz};
    long Np = (long)(nx + 1) * (ny + 1) * (nz + 1);
    const double *ex = e, *ey = e + Np, *ez = e + 2 * Np;
#pragma omp parallel for schedule(static) if(Np >= OR_OMP_MIN)
    for (long k = 0; k <= nz; ++k)
        for (long j = 0; j <= ny; ++j)
            for (long i = 0; i <= nx; ++i) {
                long p = P(&D, i, j, k);
                out[p] = curl_x(&D, ex, ey, ez, i, j, k);
                out[Np + p] = curl_y(&D, ex, ey, ez, i, j, k);
                out[2 * Np + p] = curl_z(&D, ex, ey, ez, i, j, k);
            }
}

void or_curlT(int nx, int ny, int nz, const double *h, double *out) {
    dims_t D = {nx, ny, nz};
    long Np = (long)(nx + 1) * (ny + 1) * (nz + 1);
    const double *hx = h, *hy = h + Np, *hz = h + 2 * Np;
#pragma omp parallel for schedule(static) if(Np >= OR_OMP_MIN)
    for (long k = 0; k <= nz; ++k)
        for (long j = 0; j <= ny; ++j)
            for (long i = 0; i <= nx; ++i) {
                long p = P(&D, i, j, k);
                out[p] = curlT_x(&D, hx, hy, hz, i, j, k);
                out[Np + p] = curlT_y(&D, hx, hy, hz, i, j, k);
                out[2 * Np + p] = curlT_z(&D, hx, hy, hz, i, j, k);
            }
}

/* ------------------------------------------------------------------------ */
/* Leapfrog (with C on e in the h-update: DESIGN reading 1).
 *   for m = 0..nsteps-1:
 *     e <- e + cE .* (C^T h)            ;  e[src_s] <- e[src_s] - q[m][s]
 *     h <- h - cH .* (C e)
 * q[m][s] = cE_s * jhat_s(t0 + (m+1/2) dt) is supplied by the caller (fp64, or
 * fp32-rounded values for fp32 parity, DESIGN reading 24).
 * src_dof[s] is an index into the 3*Np e-vector.                                */
void or_leapfrog(int nx, int ny, int nz, const double *cE, const double *cH, long nsteps,
                 int nsrc, const long *src_dof, const double *q, double *e, double *h) {
    dims_t D = {nx, ny, nz};
    long Np = (long)(nx + 1) * (ny + 1) * (nz + 1);
    double *ex = e, *ey = e + Np, *ez = e + 2 * Np;
    double *hx = h, *hy = h + Np, *hz = h + 2 * Np;
    for (long m = 0; m < nsteps; ++m) {
        /* e-half-step: reads h only, so the update may be done in place */
#pragma omp parallel for schedule(static) if(Np >= OR_OMP_MIN)
        for (long k = 0; k <= nz; ++k)
            for (long j = 0; j <= ny; ++j)
                for (long i = 0; i <= nx; ++i) {
                    long p = P(&D, i, j, k);
                    ex[p] = ex[p] + cE[p] * curlT_x(&D, hx, hy, hz, i, j, k);
                    ey[p] = ey[p] + cE[Np + p] * curlT_y(&D, hx, hy, hz, i, j, k);
                    ez[p] = ez[p] + cE[2 * Np + p] * curlT_z(&D, hx, hy, hz, i, j, k);
                }
        for (int s = 0; s < nsrc; ++s) e[src_dof[s]] = e[src_dof[s]] - q[m * nsrc + s];
        /* h-half-step: reads e only */
#pragma omp parallel for schedule(static) if(Np >= OR_OMP_MIN)
        for (long k = 0; k <= nz; ++k)
            for (long j = 0; j <= ny; ++j)
                for (long i = 0; i <= nx; ++i) {
                    long p = P(&D, i, j, k);
                    hx[p] = hx[p] - cH[p] * curl_x(&D, ex, ey, ez, i, j, k);
                    hy[p] = hy[p] - cH[Np + p] * curl_y(&D, ex, ey, ez, i, j, k);
                    hz[p] = hz[p] - cH[2 * Np + p] * curl_z(&D, ex, ey, ez, i, j, k);
                }
    }
}

/* ------------------------------------------------------------------------ */
/* One application of the scaled FIT operator in original variables
 * (PAPER:204-215 with T^-1 A T, SURVEY finding 1):
 *      y_h = - sH .* (C x_e)        y_e = sE .* (C^T x_h)
 * sE = cE * sigma, sH = cH * sigma (the caller forms the scale).             */
void or_apply_A(int nx, int ny, int nz, const double *sE, const double *sH,
                const double *xe, const double *xh, double *ye, double *yh) {
    dims_t D = {nx, ny, nz};
    long Np = (long)(nx + 1) * (ny + 1) * (nz + 1);
    const double *ex = xe, *ey = xe + Np, *ez = xe + 2 * Np;
    const double *hx = xh, *hy = xh + Np, *hz = xh + 2 * Np;
#pragma omp parallel for schedule(static) if(Np >= OR_OMP_MIN)
    for (long k = 0; k <= nz; ++k)
        for (long j = 0; j <= ny; ++j)
            for (long i = 0; i <= nx; ++i) {
                long p = P(&D, i, j, k);
                yh[p] = -sH[p] * curl_x(&D, ex, ey, ez, i, j, k);
                yh[Np + p] = -sH[Np + p] * curl_y(&D, ex, ey, ez, i, j, k);
                yh[2 * Np + p] = -sH[2 * Np + p] * curl_z(&D, ex, ey, ez, i, j, k);
                ye[p] = sE[p] * curlT_x(&D, hx, hy, hz, i, j, k);
                ye[Np + p] = sE[Np + p] * curlT_y(&D, hx, hy, hz, i, j, k);
                ye[2 * Np + p] = sE[2 * Np + p] * curlT_z(&D, hx, hy, hz, i, j, k);
            }
}

/* y <- y + a*x  and  x <- b*x + c*z  helpers are done in numpy by the caller. */

int or_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* The real conjugate-pair Newton recurrence (DESIGN readings 28-29),
 * s substeps of the same op list, step by step exactly as fit.expmv_pairs states it:
 *   substep: w = b; y = 0; for each op:
 *     u = X w;  y = (y + a w) + b u;
 *     pair: w = X u + e2 w        last: y = y + c (X u + e2 w)        half: (nothing)
 *   b = y
 * X is or_apply_A with the caller's scaled coefficients sE, sH.  kind: 0 pair, 1 half,
 * 2 last.  Elementwise updates are plain loops (OpenMP splits the index range only); the
 * association of each update is the one written above.                                  */
static void axpy2(long n, double *y, double a, const double *w, double b, const double *u) {
#pragma omp parallel for schedule(static) if(n >= OR_OMP_MIN)
    for (long i = 0; i < n; ++i) y[i] = (y[i] + a * w[i]) + b * u[i];
}
static void xpay(long n, double *out, const double *x, double e2, const double *w) {
#pragma omp parallel for schedule(static) if(n >= OR_OMP_MIN)
    for (long i = 0; i < n; ++i) out[i] = x[i] + e2 * w[i];
}
static void axpy1(long n, double *y, double c, const double *x) {
#pragma omp parallel for schedule(static) if(n >= OR_OMP_MIN)
    for (long i = 0; i < n; ++i) y[i] = y[i] + c * x[i];
}

int or_expmv_pairs(int nx, int ny, int nz, const double *sE, const double *sH, int nops,
                   const int *kind, const double *a, const double *b, const double *e2,
                   const double *c, int s, double *e, double *h) {
    long Np = (long)(nx + 1) * (ny + 1) * (nz + 1);
    long n = 3 * Np;
    /* workspace of 10 vectors, kept between calls (the Python side calls one at a time) */
    static double *buf = NULL;
    static long buf_n = 0;
    if (n > buf_n) {
        free(buf);
        buf = (double *)malloc(sizeof(double) * 10 * n);
        buf_n = buf ? n : 0;
    }
    if (!buf) return -1;
    /* vectors are (e, h) pairs of n doubles each */
    double *we = buf, *wh = buf + n, *ue = buf + 2 * n, *uh = buf + 3 * n;
    double *xe = buf + 4 * n, *xh = buf + 5 * n, *ye = buf + 6 * n, *yh = buf + 7 * n;
    double *te = buf + 8 * n, *th = buf + 9 * n;
    for (int q = 0; q < s; ++q) {
        memcpy(we, e, sizeof(double) * n);
        memcpy(wh, h, sizeof(double) * n);
        memset(ye, 0, sizeof(double) * n);
        memset(yh, 0, sizeof(double) * n);
        for (int o = 0; o < nops; ++o) {
            or_apply_A(nx, ny, nz, sE, sH, we, wh, ue, uh);          /* u = X w */
            axpy2(n, ye, a[o], we, b[o], ue);                          /* y = (y + a w) + b u */
            axpy2(n, yh, a[o], wh, b[o], uh);
            if (kind[o] == 1) continue;                                /* half */
            or_apply_A(nx, ny, nz, sE, sH, ue, uh, xe, xh);          /* X u */
            xpay(n, te, xe, e2[o], we);                                /* X u + e2 w */
            xpay(n, th, xh, e2[o], wh);
            if (kind[o] == 2) {                                        /* last */
                axpy1(n, ye, c[o], te);
                axpy1(n, yh, c[o], th);
            } else {                                                   /* pair: w = X u + e2 w */
                double *t = we; we = te; te = t;
                t = wh; wh = th; th = t;
            }
        }
        memcpy(e, ye, sizeof(double) * n);
        memcpy(h, yh, sizeof(double) * n);
    }
    return 0;
}

/* thread count of the OpenMP loops (1 = the single-thread oracle rate of bench.py) */
void or_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}
