/*
 * paraexp.h -- C ABI of the B200-native ParaExp + Leapfrog library for FIT-discretised
 * Maxwell equations (Merkel, Niyonzima, Schoeps, arXiv:1705.08019).
 *
 * Citations: PAPER:n = line n of the paper text; SPEC:n = line n of the
 * CPU-program spec; "reading n" = DESIGN.md "Readings of the paper" item n.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Grid       nx, ny, nz primal cells; (nx+1)(ny+1)(nz+1) = npts primal points.
 *  Fields     "canonical layout" (PAPER:164-167 with n_dof = 3 npts, reading 3):
 *             e = [e_x | e_y | e_z], h = [h_x | h_y | h_z], each component an array of
 *             npts values indexed i + (nx+1)*(j + (ny+1)*k), x fastest.
 *             e_x(i,j,k) is the primal edge (i,j,k)->(i+1,j,k); h_z(i,j,k) the dual edge
 *             through the primal z-face spanned by e_x(i,j,k) and e_y(i,j,k).
 *             Values are grid voltages: e in volts, h in amperes.
 *             Element type = the grid dtype (double for PARAEXP_F64, float for F32).
 *  Dead DOFs  PEC edges (tangential on the box, edges of PEC cells), virtual edges/faces
 *             and boundary-normal faces are ZEROED by the library on input and are
 *             always written as 0 (reading 5).
 *  Pointers   Field pointers passed to leapfrog/expmv/solve are caller-owned pointers
 *             to DEVICE memory on the grid's device (e.g. torch tensors) or to HOST memory
 *             (pinned or pageable; told apart with cudaPointerGetAttributes).  Host fields
 *             are copied through library-owned canonical-layout device buffers
 *             (cudaMemcpyAsync on `stream`) and the call synchronises `stream` before it
 *             returns.  The library never frees caller memory.  `stream` is a
 *             cudaStream_t (NULL = legacy default stream); all device work is
 *             stream-ordered on it and, with device fields, the call returns after
 *             enqueue unless it must read back a status flag (then it synchronises).
 *             Trace outputs (paraexp_trace) are device pointers.
 *  Errors     0 = PARAEXP_OK, negative = error (see codes), positive = warning bits.
 *             paraexp_last_error() returns a thread-local message for the last failure.
 *             On error the output buffers are unspecified.
 *  Threads    A grid owns a device workspace: calls on one grid must not run
 *             concurrently from several host threads.  Calls on one grid from one
 *             thread may use different streams: each call records an event at its end
 *             and the next call's stream waits for it before touching the grid's
 *             workspaces, so the device work of consecutive calls never overlaps.
 */
#ifndef PARAEXP_H
#define PARAEXP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------ */
#define PARAEXP_OK 0
#define PARAEXP_EINVAL (-1)     /* invalid argument                                      */
#define PARAEXP_ENOMEM (-2)     /* host or device allocation failed                     */
#define PARAEXP_ECUDA (-3)      /* CUDA runtime / driver error                          */
#define PARAEXP_ENCCL (-4)      /* NCCL error or NCCL library not loadable              */
#define PARAEXP_EDIVERGED (-5)  /* non-finite field in leapfrog              */
#define PARAEXP_EOVERFLOW (-6)  /* non-finite result of exp(tA)v             */
#define PARAEXP_ENOTSUP (-7)    /* valid but unsupported request (e.g. host-only grid)  */
#define PARAEXP_WCFL 1          /* warning bit: dt > dt_CFL (SPEC:189 warn, not forbid) */

/* ---- enums ----------------------------------------------------------------------- */
enum { PARAEXP_F64 = 0, PARAEXP_F32 = 1 };
enum { PARAEXP_SRC_ZERO = 0, PARAEXP_SRC_GAUSS_PAPER = 1, PARAEXP_SRC_GAUSS_SINE = 2,
       PARAEXP_SRC_SINE = 3 };
enum { PARAEXP_TAYLOR = 0, PARAEXP_LEJA = 1, PARAEXP_KRYLOV = 2 };
enum { PARAEXP_TAIL_EXP = 0, PARAEXP_TAIL_LEAPFROG = 1, PARAEXP_TAIL_EXP_LPT = 2 };
enum { PARAEXP_MAT_SCALAR = 0, PARAEXP_MAT_ZTABLE = 1, PARAEXP_MAT_ARRAY = 2 };
enum { PARAEXP_KERNELS_AUTO = 0, PARAEXP_KERNELS_UNFUSED = 1, PARAEXP_KERNELS_FUSED = 2,
       PARAEXP_KERNELS_TMA = 3 };
/* leapfrog kernel path of a grid (paraexp_grid_info_t.leapfrog_path): one kernel per curl half,
 * the TMA z-marching kernels (one launch per step), the single-CTA small-grid kernel or the
 * cooperative mid-size resident kernel (one launch per sequence) */
enum { PARAEXP_PATH_UNFUSED = 0, PARAEXP_PATH_TMA = 1, PARAEXP_PATH_SMALL = 2, PARAEXP_PATH_MID = 3 };

#define PARAEXP_MAX_DEGREE 150
#define PARAEXP_MAX_SOURCES 64

/* ---- grid ------------------------------------------------------------------------ */
/* Grid description (SPEC:30-35 grid, SPEC:63-67 materials).
 *   nx, ny, nz  cells per axis, each >= 1 ("< 2 points" rejected)
 *   dx, dy, dz  per-cell spacings in metres (length nx / ny / nz), or NULL => uniform d0
 *   eps_r, mu_r per-cell relative permittivity / permeability, length nx*ny*nz, x fastest,
 *               strictly positive and finite, or NULL => 1 (vacuum)
 *   pec_cell    per-cell PEC flag (nonzero = PEC), or NULL => none (reading 5)
 *   dtype       PARAEXP_F64 or PARAEXP_F32: storage and arithmetic type of every kernel
 *   device      CUDA device ordinal, or -1 for a HOST-ONLY grid (coefficients, CFL and
 *               plans only; every compute call on it returns PARAEXP_ENOTSUP)
 *   dt, dt_frac exactly one > 0: explicit time step in seconds, or a fraction of the
 *               eq:cfl bound dt_CFL.  dt is a grid property: it is baked
 *               into cE = dt*M_eps^-1 and cH = dt*M_nu (reading 24)
 *   kernels     PARAEXP_KERNELS_AUTO = _FUSED: the fused kernels chosen by size -- one CTA
 *               with the state in shared memory (<= 2048 cells fp64 / 4096 fp32), one
 *               cooperative launch with the state resident in the shared memory of up to
 *               one CTA per SM (mid-size grids, <= #SMs x 2048 / 4096 cells), else the TMA
 *               z-marching kernels; _TMA: the TMA z-marching kernels at every size;
 *               _UNFUSED: one kernel per curl half (debugging / parity baseline)
 * All input arrays are host pointers, read during the call only. */
typedef struct {
    int32_t nx, ny, nz;
    const double *dx, *dy, *dz;
    double d0;
    const double *eps_r, *mu_r;
    const uint8_t *pec_cell;
    int32_t dtype;
    int32_t device;
    double dt;
    double dt_frac;
    int32_t kernels;
} paraexp_grid_desc;

typedef struct paraexp_grid paraexp_grid;
typedef struct paraexp_comm paraexp_comm;

typedef struct {
    int32_t nx, ny, nz, dtype;
    int64_t npts;          /* (nx+1)(ny+1)(nz+1)                                        */
    int64_t ndof_field;    /* 3*npts per field; the paper's n_dof counts e+h = 6*npts   */
    int64_t cells;         /* nx*ny*nz                                                  */
    double dt, dt_cfl;     /* seconds; dt_cfl per eq:cfl                                 */
    double rho_cfl;        /* 2/dt_cfl, an upper bound of ||A||_2 (SURVEY finding 7)     */
    double rho_pow;        /* Lanczos estimate of ||A||_2 (K5), 0 if not yet computed    */
    int32_t material_mode; /* PARAEXP_MAT_*                                              */
    int32_t kernels;       /* resolved kernel family                                     */
    int64_t pitch_x;       /* device layout x pitch (elements)                           */
    int64_t device_bytes;  /* bytes of device memory currently owned by the grid         */
    int32_t device;
    int32_t warnings;      /* PARAEXP_WCFL if dt > dt_cfl                                */
    int32_t leapfrog_path; /* PARAEXP_PATH_*: the kernels a leapfrog call on this grid    *
                            * runs (<= 16 sources; a traced call on a single-CTA grid     *
                            * runs the TMA kernels); -1 for a host-only grid              */
} paraexp_grid_info_t;

/* Create a grid: validates, assembles fp64 FIT coefficients on the host (standard FIT
 * dual-facet averaging, reading 4), rounds them once to dtype and uploads them.
 * *out receives a new grid owned by the caller (free with paraexp_grid_destroy).
 * Returns PARAEXP_OK, PARAEXP_WCFL (created, dt > dt_CFL), or an error code. */
int paraexp_grid_create(const paraexp_grid_desc *desc, paraexp_grid **out);
void paraexp_grid_destroy(paraexp_grid *grid);
/* Fill *out.  If compute_rho_pow != 0 and the grid is on a device, runs the Lanczos
 * norm estimate K5 (60 steps, stream-synchronous on `stream`) and caches it. */
int paraexp_grid_info(paraexp_grid *grid, int32_t compute_rho_pow, void *stream,
                      paraexp_grid_info_t *out);
/* Export the fp64 coefficients the library assembled, canonical layout, host pointers of
 * 3*npts doubles each: cE = dt*M_eps^-1 (0 on dead edges), cH = dt*M_nu (0 on dead faces).
 * Host-side; works on host-only grids.  (Used to check the host assembly.) */
int paraexp_grid_coefficients(const paraexp_grid *grid, double *cE, double *cH);

/* ---- sources ---------------------------------------------------------------------- */
/* An edge current (eq:line_current; reading 6): primal edge (comp, i,j,k),
 * comp 0/1/2 = x/y/z.  The edge must be live.  The injected current at global step m is
 * jhat = weight * i(t0 + (m + 1/2) dt) amperes, subtracted in the e-update:
 *   e_s <- e_s - fl_T(cE64_s * jhat)       (PAPER:232 '-j'; PAPER:647 g = -[0, j]).
 * Waveforms i(t):
 *   ZERO         0
 *   GAUSS_PAPER  amp * exp(-4 ((t - t_param)/t_param)^2)                 (eq:line_current)
 *   GAUSS_SINE   amp * sin(2 pi f0 (t - t_delay)) * exp(-((t - t_delay)/t_param)^2)
 *   SINE         amp * sin(2 pi f0 t)                                                    */
typedef struct {
    int32_t comp, i, j, k;
    int32_t kind;
    double weight, amp, t_param, f0, t_delay;
} paraexp_source;

/* ---- statistics / SMVP ledger ------------------------------------ */
typedef struct {
    int64_t curl_applications; /* SMVPs: leapfrog counts 2 per step (eq:cost_LF), an
                                  A-application counts 2 curl halves                    */
    int64_t a_applications;    /* A-applications of exp(tA)v polynomials (n_Leja)       */
    int64_t leapfrog_steps;
    int64_t substeps;          /* polynomial substeps (sum of s)                         */
    int64_t kernel_launches;   /* device kernels launched by the call                    */
    int64_t cell_updates;      /* (leapfrog steps + A-applications) * cells              */
    double rho;                /* spectral bound used by the plans                        */
    int32_t method, m, s_first, s_last, m_half, s_half; /* plans used (solve: E_1 / E_p)  */
    int32_t root;              /* solve: rank owning sub-interval p (holds the output)    */
    int32_t first_interval, last_interval; /* solve: block owned by this rank (1-based)   */
    int32_t fail_interval;     /* solve: sub-interval index of a divergence, else 0       */
    double ms_particular, ms_tails, ms_reduce, ms_finish, ms_total; /* device-event times */
    double ms_leapfrog_kernels;  /* device time of the leapfrog kernel sequences (a2/a3)      */
    double ms_poly_kernels;      /* device time of the polynomial substep kernels (a6, incl.
                                    solve's dt/2 reconstruction propagator)                   */
    int32_t rho_fallback;        /* 1 if the rho safety net re-ran with rho = rho_cfl        */
    double norm_deviation;       /* max | ||E_i b||_M / ||b||_M - 1 | seen by the safety net  */
} paraexp_stats;

/* ---- leapfrog (a2, a3) ----------------------------------------------------------- */
/* nsteps leapfrog steps (with C on e in the h-update: reading 1):
 *   e <- e + cE.*(C^T h) - q(m);   h <- h - cH.*(C e)      m = 0..nsteps-1
 * In/out (e, h) = (e^(0), h^(1/2)) -> (e^(n), h^(n+1/2)), device pointers, canonical
 * layout, 3*npts elements each of the grid dtype.  Source times t0 + (m + 1/2) dt.
 * Returns after enqueue; the non-finite check (EDIVERGED) is performed only if
 * check_finite != 0 (then the call synchronises `stream`).
 * Errors: EINVAL (nsteps < 0, nsrc out of range, dead/out-of-range source edge),
 *         ENOTSUP (host-only grid), EDIVERGED, ECUDA. */
int paraexp_leapfrog(paraexp_grid *grid, const paraexp_source *src, int32_t nsrc, double t0,
                     int64_t nsteps, void *e, void *h, int32_t check_finite, void *stream,
                     paraexp_stats *stats);

/* ---- trace: energy and probe outputs (Fig. 7) ------- */
/* Probes are e-field edges (comp, i, j, k) (the paper's probe is a grid voltage, Fig. 3).
 * All output pointers are caller-owned DEVICE pointers of doubles (stream-ordered), or
 * NULL to skip that output.
 *   leapfrog: energy[m] = E_{m+1} = e^(m+1)' M_eps e^(m+1) + h^(m+1/2)' M_mu h^(m+3/2)
 *             (eq:energy; conserved exactly by leapfrog without source),
 *             probe[m*nprobe + r] = e_r^(m+1), for m = 0 .. nsteps-1.  The energy
 *             weights are M_eps = dt/cE_T and M_mu = dt/cH_T, evaluated in fp64 from the
 *             run-dtype coefficients (joules with volts/amperes as grid voltages).
 *   solve:    one row per sub-interval boundary T_i = t0 + S_i dt, i = 1 .. p:
 *             energy[i-1] = <e,e>_eps + <h,h>_mu of the reconstructed same-time solution
 *             u(T_i) = v_i(T_i) + sum_{j<i} w_j(T_i) (E(t) of PAPER:742-747, with h at
 *             T_i from reading 9) and probe[(i-1)*nprobe + r] = e_r(T_i).  With more
 *             than one rank the probe rows are summed over ranks (a few doubles) and
 *             delivered on every rank; the energy rows need the whole summed field and are
 *             delivered for i = p only (others NaN) -- the root computes E(T_p).
 * Errors: EINVAL (nprobe out of range, probe edge out of range or dead). */
#define PARAEXP_MAX_PROBES 16
typedef struct {
    int32_t nprobe;
    int32_t comp[PARAEXP_MAX_PROBES], i[PARAEXP_MAX_PROBES], j[PARAEXP_MAX_PROBES],
        k[PARAEXP_MAX_PROBES];
    double *energy;  /* device, nsteps (leapfrog) or p (solve) doubles, or NULL        */
    double *probe;   /* device, rows x nprobe doubles, or NULL                        */
} paraexp_trace;

/* paraexp_leapfrog with a trace (trace == NULL is paraexp_leapfrog). */
int paraexp_leapfrog_trace(paraexp_grid *grid, const paraexp_source *src, int32_t nsrc,
                           double t0, int64_t nsteps, void *e, void *h,
                           const paraexp_trace *trace, void *stream, paraexp_stats *stats);

/* ---- exp(tau A) v (a5, a6) -------------------------------------------------------- */
/* Options:
 *   method   PARAEXP_LEJA (Newton form on Leja points of i[-a,a], a = 1.05 h rho,
 *            reading 14), PARAEXP_TAYLOR (truncated Taylor) or
 *            PARAEXP_KRYLOV (Arnoldi with sigma = infinity, SURVEY 8(f) f3:
 *            per substep h = tau/s an l = m dimensional Krylov space of X = hA in the
 *            energy inner product, modified Gram-Schmidt applied twice, result
 *            ||b|| V_l exp(H_l) e_1; m = l in 1..150 any parity; s = 0 => s = ceil(2 rho tau / l)
 *            (rho h <= l/2, reading 31); eps_A unused; stops early on a happy breakdown)
 *   m, s     fixed degree (1 or even, <= 150, reading 16) and substep count; m = 0 => choose (m, s)
 *            minimising m*s subject to the per-substep criterion of reading 16 at eps_A;
 *            m > 0 with s = 0 => s from the criterion at that m
 *   eps_A    relative backward-error tolerance in (1e-14, 1)
 *   rho      spectral bound of A; 0 => min(rho_cfl, 1.05*rho_pow) (reading 17)
 *   early_term  Taylor/Leja: != 0 ends a substep's Newton sum once two consecutive increments
 *            satisfy ||delta y|| <= eps_A ||y|| in the energy norm ("early
 *            termination", reading 18); the skipped ops launch and return at once;
 *            stats.a_applications reports the A-applications actually performed
 *   beta     with eps_A == 0 and beta > 0: eps_A = eps_A* = beta dt^2 / rho
 *            (eq:tolerance_leja_2; see paraexp_optimal_tolerance)
 *   rho_check  rho safety net (SURVEY finding 8): exp(tau A) preserves the energy norm
 *            (A skew in <.,.>_M), so every propagator's energy norm is
 *            compared before and after (one fused dot each); a deviation above
 *            max(1e-9 (f64) / 1e-3 (f32), 10 eps_A rho tau) (fixed (m, s): 1e-3) means rho
 *            missed the spectrum, and the propagator (expmv) / the rank's block (solve) is
 *            recomputed with rho = rho_cfl (stats.rho_fallback = 1).
 *            0 = on when rho is the K5 estimate (opts rho == 0), off for an explicit rho;
 *            > 0 = on; < 0 = off.  Never for Krylov (norm-preserving by construction).      */
typedef struct {
    int32_t method;
    int32_t m, s;
    double eps_A;
    double rho;
    int32_t early_term;
    double beta;
    int32_t rho_check;
} paraexp_expmv_opts;

/* Plan export (reading 25: parity is defined at a fixed plan). */
typedef struct {
    int32_t method, m, s, n_ops;
    double tau, rho, a, gamma;
    double sigma;              /* (tau/s) / (gamma dt): scale of cE, cH in X = h/gamma A  */
    double xi[PARAEXP_MAX_DEGREE + 1];    /* Leja sequence on [-1,1] (k <= m)             */
    double d_re[PARAEXP_MAX_DEGREE + 1];  /* d-hat_k = gamma^k exp[z_0..z_k], fp64       */
    double d_im[PARAEXP_MAX_DEGREE + 1];
} paraexp_plan_info;

/* In place (h, e) <- exp(tau A_orig)(h, e), A_orig = [[0, -M_nu C], [M_eps^-1 C^T, 0]]
 * (original variables; PAPER:204-215 via SURVEY finding 1), same time level.
 * e, h: device pointers, canonical layout.  tau >= 0 seconds.
 * Errors: EINVAL (tau < 0, bad opts), ENOTSUP, EOVERFLOW (non-finite, synchronises). */
int paraexp_expmv(paraexp_grid *grid, double tau, const paraexp_expmv_opts *opts, void *e,
                  void *h, void *stream, paraexp_stats *stats);
/* Compute the plan paraexp_expmv would use (host only; no device work unless rho = 0
 * requires the K5 estimate). */
int paraexp_expmv_plan(paraexp_grid *grid, double tau, const paraexp_expmv_opts *opts,
                       paraexp_plan_info *out);

/* ---- communicator (a8) ------------------------------------------------------------ */
/* NCCL is loaded at run time (dlopen "libnccl.so.2"); the library owns the ncclComm_t.
 * The caller broadcasts the 128-byte id (e.g. with torch.distributed) and every rank
 * calls paraexp_comm_create with the same id.  Errors: ENCCL. */
int paraexp_comm_unique_id(uint8_t id[128]);
int paraexp_comm_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device,
                        paraexp_comm **out);
void paraexp_comm_destroy(paraexp_comm *comm);

/* ---- ParaExp solve (a4, a7, a8, a9; Algorithm 1) -------------------- */
/* COLLECTIVE over `comm` (NULL => single GPU, world 1): every rank calls with identical
 * arguments.  Time interval (t0, t0 + nsteps dt] is split into p sub-intervals of
 * nsteps/p steps, residual steps to the last.  Sub-intervals are assigned
 * to ranks in contiguous blocks, cost-balanced (paraexp_schedule with tail_ratio = the
 * A-applications of one propagator over the steps of one sub-interval); a rank computes,
 * for each owned j, the particular solution v_j by leapfrog from zero with global source
 * times, the seed s_j = (e_j, h_j + cH/2 C e_j) (reading 9) and accumulates its tails to
 * T_p by Horner over the per-sub-interval propagators E_i (SURVEY finding 9):
 * W <- E_i W + s_i.  The rank owning sub-interval 1 also carries u0 (reading 12).  W is
 * summed with ncclReduce onto the root = owner of sub-interval p, which reconstructs
 * (eq:averaging1/2, reading 10):
 *      e_out = e_p + W_e,   h_out = h_p + [exp(dt/2 A) W]_h.
 * = paraexp_solve_block on every rank, a sum of the blocks' W, paraexp_solve_finish on the
 * root.  tail_mode PARAEXP_TAIL_LEAPFROG propagates the staggered seeds with leapfrog
 * instead (debug identity: equals serial leapfrog).  tail_mode
 * PARAEXP_TAIL_EXP_LPT is schedule (B) of SURVEY 8(e), kept as a comparison: the paper's
 * literal structure, one independent exp tail per sub-interval (E_p..E_{j+1} s_j, and
 * E_p..E_1 u0 as a job of its own), jobs assigned longest-processing-time-first
 * (paraexp_schedule_lpt); the result equals EXP's up to summation order, with
 * sum_j (p - j) propagators of work instead of Horner's at most p per rank.  Traces need
 * tail_mode EXP.
 *   e0, h0   same-time initial value u0 at t0 (device, canonical) or NULL => 0
 *   e_out, h_out  device, canonical; written on the root, or on every rank when
 *            broadcast_out != 0 (one ncclBroadcast).  Output convention equals
 *            paraexp_leapfrog from (e0, h0 - cH/2 C e0): (e^(n), h^(n+1/2)).
 * With a communicator the ranks all-reduce their blocks' status before the reduce (a rank
 * whose block failed makes every rank return: EDIVERGED "another rank's block failed" on
 * the others), and the call waits for its stream while polling ncclCommGetAsyncError (a
 * failed peer => the communicator is aborted, ENCCL).
 * Errors: EINVAL (p < 1, nsteps < p), ENOTSUP, EDIVERGED (particular sweep of
 *         stats.fail_interval non-finite) / EOVERFLOW (propagator E_{fail_interval}
 *         produced a non-finite field), ENCCL, ECUDA.  Synchronises `stream` before
 *         returning. */
int paraexp_solve(paraexp_grid *grid, paraexp_comm *comm, const paraexp_source *src,
                  int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                  const paraexp_expmv_opts *opts, int32_t tail_mode, int32_t broadcast_out,
                  const void *e0, const void *h0, void *e_out, void *h_out, void *stream,
                  paraexp_stats *stats);

/* One rank's share of paraexp_solve without any communication (the parfor body of
 * PAPER:358-365 for the block paraexp_schedule gives `rank` of `world`), for callers that
 * sum the blocks themselves (MPI, gloo, or several virtual ranks on one GPU).
 *   w_e, w_h  out (device or host, canonical): this rank's tails carried to T_p,
 *            W_rank = sum_{owned j < p} E_p..E_{j+1} s_j (+ E_p..E_1 u0 if it owns j = 1,
 *            or job 0 under PARAEXP_TAIL_EXP_LPT);
 *            zero if the rank owns no sub-interval.  The sum of W_rank over ranks is the
 *            W that paraexp_solve reduces.
 *   v_e, v_h  out on the root only (stats.root == rank; may be NULL elsewhere): the
 *            particular state (e_p^(M), h_p^(M+1/2)) of sub-interval p.
 * All ranks must use the same rho: pass opts->rho > 0 (e.g. rank 0's stats.rho) unless
 * the grids are identical (the K5 estimate is then cached per grid).  The rho safety net
 * acts per rank.  Synchronises `stream`.  Errors as paraexp_solve (no ENCCL). */
int paraexp_solve_block(paraexp_grid *grid, int32_t rank, int32_t world,
                        const paraexp_source *src, int32_t nsrc, double t0, int64_t nsteps,
                        int32_t p, const paraexp_expmv_opts *opts, int32_t tail_mode,
                        const void *e0, const void *h0, void *w_e, void *w_h, void *v_e,
                        void *v_h, void *stream, paraexp_stats *stats);

/* Reconstruction on the root (a9, eq:averaging1/2, reading 10) from the summed W = (w_e,
 * w_h) and the root's particular state (v_e, v_h):  e_out = v_e + w_e,
 * h_out = v_h + [exp(dt/2 A) W]_h (tail_mode EXP; a degree-24 Taylor propagator with
 * rho from opts as in paraexp_expmv), or (e_out, h_out) = v + W (tail_mode LEAPFROG).
 * All pointers canonical, device or host; the outputs may alias v.  Synchronises. */
int paraexp_solve_finish(paraexp_grid *grid, const paraexp_expmv_opts *opts, int32_t tail_mode,
                         const void *w_e, const void *w_h, const void *v_e, const void *v_h,
                         void *e_out, void *h_out, void *stream, paraexp_stats *stats);

/* paraexp_solve (tail_mode EXP) with a trace of the reconstructed solution at the
 * sub-interval boundaries T_1 .. T_p (see paraexp_trace above; f1).  Collective. */
int paraexp_solve_trace(paraexp_grid *grid, paraexp_comm *comm, const paraexp_source *src,
                        int32_t nsrc, double t0, int64_t nsteps, int32_t p,
                        const paraexp_expmv_opts *opts, int32_t broadcast_out, const void *e0,
                        const void *h0, void *e_out, void *h_out, const paraexp_trace *trace,
                        void *stream, paraexp_stats *stats);

/* ---- host-only helpers (no GPU needed) -------------------------------------------- */
/* Partition of nsteps into p sub-intervals: bounds[0..p], bounds[0] = 0, bounds[p] = nsteps
 * (SPEC:345-353).  EINVAL if p < 1 or nsteps < p. */
int paraexp_partition(int64_t nsteps, int32_t p, int64_t *bounds);
/* Contiguous block [first, last] (1-based sub-interval indices) owned by `rank` of `world`
 * for p sub-intervals; first = 0, last = -1 if the rank owns none; root = owner of p.
 * Cost-balanced: with a block [f, l] costing (l - f + 1) sweeps plus
 * (p - f) propagators (one more if f = 1 and has_u0), a propagator costing tail_ratio
 * sweeps, the blocks minimise the largest rank cost (bisection on the makespan, then each
 * rank in order takes as many sub-intervals as fit -- the fewest ranks, hence the least
 * Horner work, at that makespan).  tail_ratio <= 0: equal shares, the remainder to the
 * later ranks.  Host-only. */
int paraexp_schedule(int32_t p, int32_t world, int32_t rank, double tail_ratio, int32_t has_u0,
                     int32_t *first, int32_t *last, int32_t *root);
/* Schedule (B), tail_mode PARAEXP_TAIL_EXP_LPT: owner[j] (j = 1..p) = rank of sub-interval j
 * and its independent tail, owner[0] = rank of the u0 tail (-1 if has_u0 == 0); job j costs
 * one sweep + (p - j) propagators, job 0 p propagators (propagator = tail_ratio sweeps); jobs
 * in decreasing cost (ties: lower j) go to the least-loaded rank (ties: lower rank).
 * *root = owner[p].  Host-only. */
int paraexp_schedule_lpt(int32_t p, int32_t world, double tail_ratio, int32_t has_u0, int32_t *owner,
                         int32_t *root);
/* Symmetrised Leja sequence xi'_0..xi'_{count-1} on [-1,1] (reading 14). */
int paraexp_leja_points(int32_t count, double *xi);
/* Plan without a grid: tau and rho given, dt used only for sigma (may be 1). */
int paraexp_plan_host(int32_t method, int32_t m, int32_t s, double eps_A, double tau,
                      double rho, double dt, paraexp_plan_info *out);
/* eq:tolerance_leja_2: eps_A* = beta dt^2 / ||A||_2, the Leja
 * tolerance that balances the exponential's backward error against the leapfrog truncation
 * error eps_B = beta dt^2 (kappa_exp(A) = ||A||_2 for normal A).  Taken literally (reading 30:
 * the paper gives neither beta's value nor its units; beta carries s^-3 for SI dt and ||A||),
 * clamped to [1e-14, 0.1]; *clamped (may be NULL) is set to 1 if the clamp applied.
 * Returns 0.1 for non-positive or non-finite input. */
double paraexp_optimal_tolerance(double dt, double beta, double norm_A, int32_t *clamped);
/* theta_m(eps_A): largest theta with max_{|x|<=theta} |p(ix) - e^{ix}| <= eps_A theta
 * (reading 16), method TAYLOR or LEJA.  Cached. */
double paraexp_theta(int32_t method, int32_t m, double eps_A);

/* Page-locked (pinned) host memory for field arguments passed as HOST pointers: the library
 * copies host fields with cudaMemcpyAsync, which reaches the link's bandwidth only from pinned
 * memory (pageable buffers go through the driver's staging path, several times slower for the
 * 815 MB of a C3 fp64 output).  *out is owned by the caller until paraexp_host_free; usable
 * from any device (portable).  The memory is not initialised.
 * Errors: EINVAL (bytes == 0, out == NULL), ENOMEM / ECUDA (no driver, pinning failed). */
int paraexp_host_alloc(size_t bytes, void **out);
/* Release memory from paraexp_host_alloc (NULL is a no-op). */
void paraexp_host_free(void *p);

const char *paraexp_strerror(int code);
const char *paraexp_last_error(void);
/* library version string, e.g. "paraexp-b200 0.1 (sm_100a)" */
const char *paraexp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARAEXP_H */
