// grid.cpp -- host grid builder (row a1): validation, fp64 FIT coefficients, eq:cfl,
// material-mode detection and device upload.
//
// PAPER:150-180 (FIT grid, M_eps, M_mu), PAPER:246-254 (eq:cfl); DESIGN readings 3-5.
// Coefficients (per live DOF, fp64):
//   cE(edge) = dt / M_eps(edge),  M_eps(x-edge i,j,k) = (1/dx_i) * sum over the <= 4 cells
//              (i, j-1..j, k-1..k) of eps0*eps_r * dy_jj*dz_kk/4         (y, z cyclic)
//   cH(face) = dt * M_nu(face),  M_nu(x-face i,j,k) = (1/(dy_j dz_k)) * sum over the <= 2
//              cells (i-1..i, j, k) of dx_ii / (2 mu0 mu_r)               (y, z cyclic)
// Live edges: not virtual, not tangential to the box, not an edge of a PEC cell.
// Live faces: not virtual, not normal to the box.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace {
const double kEps0 = 8.8541878128e-12;  // CODATA 2018
const double kMu0 = 1.25663706212e-6;
}  // namespace

namespace pe {

static int build_coefficients(Grid &G, const paraexp_grid_desc &d) {
    const int nx = G.nx, ny = G.ny, nz = G.nz;
    std::vector<double> dx(nx), dy(ny), dz(nz);
    for (int i = 0; i < nx; ++i) dx[i] = d.dx ? d.dx[i] : d.d0;
    for (int j = 0; j < ny; ++j) dy[j] = d.dy ? d.dy[j] : d.d0;
    for (int k = 0; k < nz; ++k) dz[k] = d.dz ? d.dz[k] : d.d0;
    for (double v : dx) if (!(v > 0) || !std::isfinite(v)) return fail(PARAEXP_EINVAL, "spacing must be positive and finite");
    for (double v : dy) if (!(v > 0) || !std::isfinite(v)) return fail(PARAEXP_EINVAL, "spacing must be positive and finite");
    for (double v : dz) if (!(v > 0) || !std::isfinite(v)) return fail(PARAEXP_EINVAL, "spacing must be positive and finite");
    const int64_t ncell = (int64_t)nx * ny * nz;
    auto cid = [&](int64_t i, int64_t j, int64_t k) { return i + (int64_t)nx * (j + (int64_t)ny * k); };
    auto eps = [&](int64_t c) { return d.eps_r ? d.eps_r[c] : 1.0; };
    auto mu = [&](int64_t c) { return d.mu_r ? d.mu_r[c] : 1.0; };
    auto pec = [&](int64_t c) { return d.pec_cell ? d.pec_cell[c] != 0 : false; };
    if (d.eps_r)
        for (int64_t c = 0; c < ncell; ++c)
            if (!(d.eps_r[c] > 0) || !std::isfinite(d.eps_r[c])) return fail(PARAEXP_EINVAL, "eps_r must be positive and finite");
    if (d.mu_r)
        for (int64_t c = 0; c < ncell; ++c)
            if (!(d.mu_r[c] > 0) || !std::isfinite(d.mu_r[c])) return fail(PARAEXP_EINVAL, "mu_r must be positive and finite");

    // eq:cfl
    double cfl = INFINITY;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const double inv = 1.0 / (dx[i] * dx[i]) + 1.0 / (dy[j] * dy[j]) + 1.0 / (dz[k] * dz[k]);
                const int64_t c = cid(i, j, k);
                cfl = std::min(cfl, std::sqrt(kEps0 * eps(c) * kMu0 * mu(c) / inv));
            }
    G.dt_cfl = cfl;
    G.rho_cfl = 2.0 / cfl;
    const bool has_dt = d.dt > 0, has_frac = d.dt_frac > 0;
    if (has_dt == has_frac) return fail(PARAEXP_EINVAL, "exactly one of dt, dt_frac must be > 0");
    G.dt = has_dt ? d.dt : d.dt_frac * cfl;
    if (!std::isfinite(G.dt)) return fail(PARAEXP_EINVAL, "dt not finite");
    G.warnings = G.dt > cfl ? PARAEXP_WCFL : 0;

    const int64_t NX = nx + 1, NY = ny + 1;
    const int64_t np = NX * NY * (nz + 1);
    G.npts = np;
    G.cE64.assign(3 * np, 0.0);
    G.cH64.assign(3 * np, 0.0);
    const int64_t n3[3] = {nx, ny, nz};
    const std::vector<double> *sp[3] = {&dx, &dy, &dz};
    for (int64_t k = 0; k <= nz; ++k)
        for (int64_t j = 0; j <= ny; ++j)
            for (int64_t i = 0; i <= nx; ++i) {
                const int64_t p = i + NX * (j + NY * k);
                const int64_t P3[3] = {i, j, k};
                for (int c = 0; c < 3; ++c) {
                    const int b = (c + 1) % 3, g = (c + 2) % 3;
                    // edge along c from point P3
                    const bool e_in = P3[c] < n3[c];
                    const bool e_wall = P3[b] == 0 || P3[b] == n3[b] || P3[g] == 0 || P3[g] == n3[g];
                    if (e_in && !e_wall) {
                        double area_eps = 0.0;
                        bool touches_pec = false;
                        for (int ob = 0; ob < 2; ++ob)
                            for (int og = 0; og < 2; ++og) {
                                int64_t C3[3];
                                C3[c] = P3[c];
                                C3[b] = P3[b] - 1 + ob;
                                C3[g] = P3[g] - 1 + og;
                                const int64_t cc = cid(C3[0], C3[1], C3[2]);
                                area_eps += kEps0 * eps(cc) * ((*sp[b])[C3[b]] * (*sp[g])[C3[g]] * 0.25);
                                touches_pec = touches_pec || pec(cc);
                            }
                        if (!touches_pec) {
                            const double Meps = area_eps / (*sp[c])[P3[c]];
                            G.cE64[c * np + p] = G.dt / Meps;
                        }
                    }
                    // face normal to c at P3 (spanned by b, g edges)
                    const bool f_in = P3[b] < n3[b] && P3[g] < n3[g];
                    const bool f_wall = P3[c] == 0 || P3[c] == n3[c];
                    if (f_in && !f_wall) {
                        double len_nu = 0.0;
                        for (int oc = 0; oc < 2; ++oc) {
                            int64_t C3[3];
                            C3[c] = P3[c] - 1 + oc;
                            C3[b] = P3[b];
                            C3[g] = P3[g];
                            len_nu += (*sp[c])[C3[c]] * 0.5 / (kMu0 * mu(cid(C3[0], C3[1], C3[2])));
                        }
                        const double Mnu = len_nu / ((*sp[b])[P3[b]] * (*sp[g])[P3[g]]);
                        G.cH64[c * np + p] = G.dt * Mnu;
                    }
                }
            }

    // ---- material mode (DESIGN "kernels"): SCALAR if all live cE of a component agree,
    // ZTABLE if they agree per z-plane, else ARRAY.  cH: scalar per component or ARRAY.
    bool scalar = true, ztab = true, hscalar = true;
    double es[3] = {0, 0, 0}, hs[3] = {0, 0, 0};
    bool es_set[3] = {false, false, false}, hs_set[3] = {false, false, false};
    std::vector<double> zt(3 * nz, 0.0);
    std::vector<char> zt_set(3 * nz, 0);
    for (int c = 0; c < 3; ++c)
        for (int64_t k = 0; k <= nz; ++k)
            for (int64_t j = 0; j <= ny; ++j)
                for (int64_t i = 0; i <= nx; ++i) {
                    const int64_t p = i + NX * (j + NY * k);
                    const double ce = G.cE64[c * np + p];
                    const int64_t P3[3] = {i, j, k};
                    const int b = (c + 1) % 3, g = (c + 2) % 3;
                    const bool e_box_live = P3[c] < n3[c] && P3[b] > 0 && P3[b] < n3[b] && P3[g] > 0 && P3[g] < n3[g];
                    if (e_box_live) {
                        if (ce == 0.0) { scalar = false; ztab = false; }   // interior PEC edge
                        if (!es_set[c]) { es[c] = ce; es_set[c] = true; }
                        else if (ce != es[c]) scalar = false;
                        if (k < nz) {
                            if (!zt_set[c * nz + k]) { zt[c * nz + k] = ce; zt_set[c * nz + k] = 1; }
                            else if (ce != zt[c * nz + k]) ztab = false;
                        }
                    }
                    const double ch = G.cH64[c * np + p];
                    if (ch != 0.0) {
                        if (!hs_set[c]) { hs[c] = ch; hs_set[c] = true; }
                        else if (ch != hs[c]) hscalar = false;
                    }
                }
    G.mat_mode = scalar ? PARAEXP_MAT_SCALAR : (ztab ? PARAEXP_MAT_ZTABLE : PARAEXP_MAT_ARRAY);
    G.h_array = !hscalar;
    for (int c = 0; c < 3; ++c) {
        G.cE_scalar[c] = es[c];
        G.cH_scalar[c] = hs[c];
    }
    G.cE_ztab = zt;
    return PARAEXP_OK;
}

static int upload(Grid &G) {
    const int nx = G.nx, ny = G.ny, nz = G.nz;
    const Layout &L = G.L;
    const size_t es = G.esize();
    const int64_t NX = nx + 1, NY = ny + 1, np = G.npts;
    auto to_dev_layout = [&](const std::vector<double> &src, void **dst) -> int {
        const size_t bytes = 3 * L.cs * es;
        std::vector<char> host(bytes, 0);
        for (int c = 0; c < 3; ++c)
            for (int64_t k = 0; k < nz; ++k)
                for (int64_t j = 0; j < ny; ++j)
                    for (int64_t i = 0; i < nx; ++i) {
                        const double v = src[c * np + i + NX * (j + NY * k)];
                        const int64_t q = c * L.cs + i + L.px * (j + (int64_t)ny * k);
                        if (G.dtype == PARAEXP_F64)
                            reinterpret_cast<double *>(host.data())[q] = v;
                        else
                            reinterpret_cast<float *>(host.data())[q] = (float)v;
                    }
        int rc = dev_alloc(dst, bytes);
        if (rc) return rc;
        G.device_bytes += bytes;
        rc = dev_memcpy_h2d_async(*dst, host.data(), bytes, nullptr);
        if (rc) return rc;
        return dev_sync(nullptr);
    };
    if (G.mat_mode == PARAEXP_MAT_ZTABLE) {
        const size_t bytes = 3 * nz * es;
        std::vector<char> host(bytes, 0);
        for (int q = 0; q < 3 * nz; ++q) {
            if (G.dtype == PARAEXP_F64)
                reinterpret_cast<double *>(host.data())[q] = G.cE_ztab[q];
            else
                reinterpret_cast<float *>(host.data())[q] = (float)G.cE_ztab[q];
        }
        int rc = dev_alloc(&G.d_cE_tab, bytes);
        if (rc) return rc;
        G.device_bytes += bytes;
        rc = dev_memcpy_h2d_async(G.d_cE_tab, host.data(), bytes, nullptr);
        if (rc) return rc;
        if ((rc = dev_sync(nullptr))) return rc;
    }
    if (G.mat_mode == PARAEXP_MAT_ARRAY) {
        int rc = to_dev_layout(G.cE64, &G.d_cE_arr);
        if (rc) return rc;
    }
    if (G.h_array) {
        int rc = to_dev_layout(G.cH64, &G.d_cH_arr);
        if (rc) return rc;
    }
    int rc = dev_alloc(&G.d_flag, 4096);
    if (rc) return rc;
    rc = dev_alloc(&G.d_red, 4096);
    if (rc) return rc;
    rc = dev_alloc(&G.d_src, sizeof(SrcDev) * PARAEXP_MAX_SOURCES);
    if (rc) return rc;
    // dynamic-schedule unit counter of the fused kernels (starts at 0; see fused.cu Sched)
    if ((rc = dev_alloc(&G.d_sched, 256))) return rc;
    if ((rc = dev_memset_async(G.d_sched, 0, 256, nullptr)) || (rc = dev_sync(nullptr))) return rc;
    G.sched_base = 0;
    G.device_bytes += 8192 + 256 + sizeof(SrcDev) * PARAEXP_MAX_SOURCES;
    return PARAEXP_OK;
}

void grid_free_device(Grid &G) {
    for (void *p : G.ws) dev_free(p);
    G.ws.clear();
    dev_free(G.d_cE_tab);
    dev_free(G.d_cE_arr);
    dev_free(G.d_cH_arr);
    dev_free(G.d_flag);
    dev_free(G.d_red);
    dev_free(G.d_src);
    dev_free(G.d_q);
    dev_free(G.d_et);
    G.d_et = nullptr;
    for (void *q : G.conc) dev_free(q);
    G.conc.clear();
    for (void *q : G.streams) dev_stream_destroy(q);
    G.streams.clear();
    for (void *q : G.events) dev_event_destroy(q);
    G.events.clear();
    dev_free(G.d_sched);
    G.d_sched = nullptr;
    for (int q = 0; q < Grid::kMidSlots; ++q) {
        dev_free(G.d_mid[q]);
        G.d_mid[q] = nullptr;
        G.mid_bytes[q] = 0;
        G.mid_tag[q] = 0;
    }
    dev_free(G.d_norms);
    G.d_norms = nullptr;
    if (G.call_event) dev_event_destroy(G.call_event);
    G.call_event = G.call_stream = nullptr;
    G.sched_base = 0;
    for (void *q : G.kry) dev_free(q);
    G.kry.clear();
    dev_free(G.d_canon[0]);
    dev_free(G.d_canon[1]);
    G.d_canon[0] = G.d_canon[1] = nullptr;
    G.d_cE_tab = G.d_cE_arr = G.d_cH_arr = G.d_flag = G.d_red = G.d_src = G.d_q = nullptr;
    G.device_bytes = 0;
    G.ws_bytes = 0;
}

int grid_create(const paraexp_grid_desc *d, paraexp_grid **out) {
    if (!d || !out) return fail(PARAEXP_EINVAL, "null argument");
    *out = nullptr;
    if (d->nx < 1 || d->ny < 1 || d->nz < 1) return fail(PARAEXP_EINVAL, "nx, ny, nz must be >= 1 cell");
    if (d->dtype != PARAEXP_F64 && d->dtype != PARAEXP_F32) return fail(PARAEXP_EINVAL, "bad dtype");
    if (!d->dx || !d->dy || !d->dz)
        if (!(d->d0 > 0) || !std::isfinite(d->d0)) return fail(PARAEXP_EINVAL, "d0 must be > 0 when spacings are NULL");
    if (d->kernels < 0 || d->kernels > 3) return fail(PARAEXP_EINVAL, "bad kernels selector");
    const int64_t cells = (int64_t)d->nx * d->ny * d->nz;
    if (cells > (int64_t)1 << 33) return fail(PARAEXP_EINVAL, "grid too large");
    paraexp_grid *pg = new (std::nothrow) paraexp_grid();
    if (!pg) return fail(PARAEXP_ENOMEM, "host allocation");
    Grid &G = pg->g;
    G.nx = d->nx;
    G.ny = d->ny;
    G.nz = d->nz;
    G.dtype = d->dtype;
    G.device = d->device;
    G.rho_pow = 0;
    int rc = build_coefficients(G, *d);
    if (rc < 0) {
        delete pg;
        return rc;
    }
    const int64_t align = 128 / (int64_t)G.esize();
    G.L.nx = G.nx;
    G.L.ny = G.ny;
    G.L.nz = G.nz;
    G.L.px = (G.nx + align - 1) / align * align;
    G.L.plane = G.L.px * G.ny;
    G.L.cs = G.L.plane * G.nz;
    G.kernels = d->kernels == PARAEXP_KERNELS_UNFUSED ? PARAEXP_KERNELS_UNFUSED
                : d->kernels == PARAEXP_KERNELS_TMA     ? PARAEXP_KERNELS_TMA
                                                        : PARAEXP_KERNELS_FUSED;
    if (G.device >= 0) {
        if ((rc = dev_set_device(G.device))) {
            delete pg;
            return rc;
        }
        if ((rc = upload(G))) {
            grid_free_device(G);
            delete pg;
            return rc;
        }
    }
    *out = pg;
    return G.warnings;
}

}  // namespace pe

extern "C" {

int paraexp_grid_create(const paraexp_grid_desc *desc, paraexp_grid **out) {
    return pe::grid_create(desc, out);
}

void paraexp_grid_destroy(paraexp_grid *grid) {
    if (!grid) return;
    if (grid->g.device >= 0) {
        pe::dev_set_device(grid->g.device);
        pe::grid_free_device(grid->g);
    }
    delete grid;
}

int paraexp_grid_coefficients(const paraexp_grid *grid, double *cE, double *cH) {
    if (!grid) return pe::fail(PARAEXP_EINVAL, "null grid");
    if (cE) std::memcpy(cE, grid->g.cE64.data(), grid->g.cE64.size() * sizeof(double));
    if (cH) std::memcpy(cH, grid->g.cH64.data(), grid->g.cH64.size() * sizeof(double));
    return PARAEXP_OK;
}

}  // extern "C"
