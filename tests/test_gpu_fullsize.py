"""GPU parity at BASELINE.json's full grid sizes, in the launch configuration bench.py times
(fused TMA kernels, persistent grid over the whole field), on SAMPLED outputs.

The oracle cannot run every full-size case on the whole grid in seconds, but every output
value depends only on inputs inside its domain of dependence: one leapfrog step or one
A-application reaches one cell further along each axis (the curls couple nearest neighbours
only).  So for a sample box B of output points, the oracle runs on a SUB-GRID
that contains B plus a margin R >= (leapfrog steps + A-applications + 2) cells on every side
that is not a real boundary of the grid, with the same materials, the same dt and the
sources inside it.  The sub-grid's artificial PEC walls are more than R cells from B, so its
values on B are the full grid's values (exact, not approximate) -- compared element by
element with the CUDA result at the north_star tolerances.

Inputs are seeded random fields generated on the device with torch's Philox generator
(plumbing: 768^3 fields do not fit comfortably in host memory); the oracle gets the sub-box
of those inputs, the CUDA path the whole grid.  dt comes from the oracle's own eq:cfl over
the full grid (fit.cfl_dt)."""
import math

import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from gpu_util import TOL, max_abs_rel, rel_l2
from oracle import fit
from synth import config_c3, config_c4, config_c5

pytestmark = pytest.mark.gpu


def _dev_fields(w, seed, dtype):
    """e ~ U[-1,1] V, h ~ U[-1,1]/Z0 A (reading 26) on cuda:0, canonical layout."""
    import torch
    from synth.configs import Z0
    g = torch.Generator(device="cuda:0")
    g.manual_seed(seed)
    td = torch.float64 if dtype == "f64" else torch.float32
    n = 3 * w.npts
    e = torch.rand(n, generator=g, dtype=td, device="cuda:0").mul_(2).sub_(1)
    h = torch.rand(n, generator=g, dtype=td, device="cuda:0").mul_(2).sub_(1).div_(Z0)
    return e, h


def _box(w, center, half, R):
    """cell ranges [lo, hi) of the sub-grid per axis, and the sample range of points"""
    lo, hi, slo, shi = [], [], [], []
    for c, n in zip(center, (w.nx, w.ny, w.nz)):
        a, b = max(0, c - half), min(n, c + half)
        lo.append(max(0, a - R))
        hi.append(min(n, b + R))
        slo.append(a)
        shi.append(b)
    return lo, hi, slo, shi


def _extract(t, w, lo, hi):
    """canonical field (3 * npts) -> sub-grid canonical field (host fp64) of cells [lo, hi)"""
    v = t.view(3, w.nz + 1, w.ny + 1, w.nx + 1)
    sub = v[:, lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
    return sub.double().cpu().numpy().reshape(-1)


def _sub_grid(w, lo, hi, dt, dtype):
    def cut(a, dt_):
        if a is None:
            return None
        return np.ascontiguousarray(np.asarray(a).reshape(w.nz, w.ny, w.nx)[
            lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].reshape(-1), dtype=dt_)
    sx, sy, sz = hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]
    return fit.Grid(sx, sy, sz, d0=w.d0, eps_r=cut(w.eps_r, float), pec_cell=cut(w.pec_cell, np.uint8),
                    dt=dt, dtype=dtype)


def _sub_sources(og, w, lo, hi):
    out = []
    for s in w.sources:
        i, j, k = s.i - lo[0], s.j - lo[1], s.k - lo[2]
        if not (0 <= i < og.nx + 1 and 0 <= j < og.ny + 1 and 0 <= k < og.nz + 1):
            continue
        if og.cE[og.edge_dof(s.comp, i, j, k)] == 0:     # on the sub-grid's artificial wall
            continue
        out.append(type(s)(s.comp, i, j, k, s.kind, s.amp, s.t_param, s.f0, s.t_delay, s.weight))
    return out


def _compare(got_e, got_h, ref, og, w, lo, slo, shi, dtype, what):
    """compare the sample box (points slo..shi) of the sub-grid result with the GPU result"""
    def sample_full(t):
        v = t.view(3, w.nz + 1, w.ny + 1, w.nx + 1)
        return v[:, slo[2]:shi[2] + 1, slo[1]:shi[1] + 1, slo[0]:shi[0] + 1].double().cpu().numpy()

    def sample_sub(a):
        v = a.reshape(3, og.nz + 1, og.ny + 1, og.nx + 1)
        return v[:, slo[2] - lo[2]:shi[2] - lo[2] + 1, slo[1] - lo[1]:shi[1] - lo[1] + 1,
                 slo[0] - lo[0]:shi[0] - lo[0] + 1]

    ge, gh = sample_full(got_e), sample_full(got_h)
    re, rh = sample_sub(ref[0]), sample_sub(ref[1])
    ee, eh = rel_l2(ge, re), rel_l2(gh, rh)
    tol = TOL[dtype]
    assert np.linalg.norm(re) > 0 and np.linalg.norm(rh) > 0, what
    assert ee <= tol and eh <= tol, f"{what}: rel-L2 e={ee:.3e} h={eh:.3e} (tol {tol})"
    me, mh = max_abs_rel(ge, re), max_abs_rel(gh, rh)
    assert me <= 100 * tol and mh <= 100 * tol, f"{what}: max-abs e={me:.3e} h={mh:.3e}"
    return ee, eh


def _full_dt(w):
    n = (w.nx, w.ny, w.nz)
    d = [np.full(k, w.d0) for k in n]
    return w.dt_frac * fit.cfl_dt(*n, *d, w.eps_r)


def _run_leapfrog_expmv(w, dtype, nlf, m, centers, half=6, seed=11, t0=0.0):
    """full-grid CUDA: nlf leapfrog steps (with the workload's sources) then exp(tau A) with a
    fixed degree-m Leja plan (s = 1); oracle on sub-grids around each sample centre"""
    import torch
    dt = _full_dt(w)
    rho = 2.0 / (dt / w.dt_frac)                              # rho_CFL of the full grid
    lg = pe.Grid.from_workload(w, dtype=dtype)
    assert abs(lg.dt - dt) <= 1e-14 * dt
    e, h = _dev_fields(w, seed, dtype)
    e_in, h_in = e.clone(), h.clone()
    tau = 3.0 * dt
    pe.leapfrog(lg, e, h, nlf, w.sources, t0)
    pe.expmv(lg, tau, e, h, method="leja", m=m, s=1, rho=rho)
    torch.cuda.synchronize()
    R = nlf + m + 2
    for c in centers:
        lo, hi, slo, shi = _box(w, c, half, R)
        og = _sub_grid(w, lo, hi, dt, dtype)
        se, sh = og.clean(_extract(e_in, w, lo, hi), _extract(h_in, w, lo, hi))
        src = _sub_sources(og, w, lo, hi)
        ref = fit.leapfrog(og, se, sh, nlf, src, t0)
        plan = fit.make_plan("leja", m, 1, tau, rho)
        ref = fit.expmv(og, plan, *ref, mode="pairs", dtype=dtype)
        _compare(e, h, ref, og, w, lo, slo, shi, dtype, f"{w.name} {dtype} centre {c}")
    del e, h, e_in, h_in
    lg.close()
    torch.cuda.empty_cache()


def _run_solve(w, dtype, nsteps, p, m, centers, half=5, seed=13, t0=0.0, host_io=False):
    """full-grid CUDA paraexp_solve (random u0 + the workload's sources, fixed Leja plan
    (m, s = 1) per sub-interval) vs the oracle's sequential Algorithm 1 on sub-grids"""
    import torch
    dt = _full_dt(w)
    rho = 2.0 / (dt / w.dt_frac)
    lg = pe.Grid.from_workload(w, dtype=dtype)
    e0, h0 = _dev_fields(w, seed, dtype)
    eo, ho = torch.zeros_like(e0), torch.zeros_like(h0)
    st = pe.solve(lg, nsteps, p, w.sources, t0=t0, u0=(e0, h0), method="leja", m=m, s=1, rho=rho,
                  e_out=eo, h_out=ho)
    torch.cuda.synchronize()
    assert st["leapfrog_steps"] == nsteps
    if host_io:
        # bench.py's e2e path at full size: u0 and the outputs as pinned HOST fields from
        # paraexp_host_alloc, staged by the library -- the bits of the device-buffer solve
        hf = [pe.HostField(lg) for _ in range(4)]
        hf[0].tensor.copy_(e0)
        hf[1].tensor.copy_(h0)
        hf[2].tensor.fill_(float("nan"))
        hf[3].tensor.fill_(float("nan"))
        pe.solve(lg, nsteps, p, w.sources, t0=t0, u0=(hf[0].tensor, hf[1].tensor), method="leja", m=m,
                 s=1, rho=rho, e_out=hf[2].tensor, h_out=hf[3].tensor)
        assert torch.equal(hf[2].tensor, eo.cpu()) and torch.equal(hf[3].tensor, ho.cpu())
        for f in hf:
            f.close()
    # domain of dependence: all leapfrog steps + p propagators of m + the dt/2 Taylor (24 s)
    half_plan = fit.half_step_plan(fit.Grid(1, 1, 1, d0=w.d0, dt=dt), rho)
    R = nsteps + p * m + half_plan.m * half_plan.s + 2
    for c in centers:
        lo, hi, slo, shi = _box(w, c, half, R)
        og = _sub_grid(w, lo, hi, dt, dtype)
        u0 = (_extract(e0, w, lo, hi), _extract(h0, w, lo, hi))
        src = _sub_sources(og, w, lo, hi)
        ref = fit.paraexp(og, src, t0, nsteps, p, lambda tau: fit.make_plan("leja", m, 1, tau, rho),
                          u0=u0, rho=rho, dtype=dtype)
        _compare(eo, ho, ref, og, w, lo, slo, shi, dtype, f"{w.name} solve {dtype} centre {c}")
    del e0, h0, eo, ho
    lg.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c3_fullsize_leapfrog_expmv_m150(dtype):
    """C3 256^3 layered: 8 steps + one degree-150 Leja substep (the bench planner's degree);
    samples at the source and at a corner."""
    w = config_c3(dtype)
    _run_leapfrog_expmv(w, dtype, 8, 150, [(128, 128, 32), (0, 255, 255)], half=4, t0=200e-12)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c3_fullsize_solve(dtype):
    """C3 256^3: paraexp_solve with p = 8 sub-intervals at full size (random u0 + source)."""
    w = config_c3(dtype)
    _run_solve(w, dtype, 16, 8, 4, [(128, 128, 32), (250, 3, 190)], host_io=dtype == "f64")


def test_c4_fullsize_spiral():
    """C4 512x512x64 spiral (per-edge eps, PEC trace + via, port sources): leapfrog + expmv and
    a p = 8 solve, sampled at the port and on the trace."""
    w = config_c4(nsteps=64)
    port = (w.sources[0].i, w.sources[0].j, 5)
    _run_leapfrog_expmv(w, "f64", 40, 16, [port, (256, 256, 10)], t0=150e-12)
    _run_solve(w, "f64", 16, 8, 4, [port])


def test_c4_fullsize_longer_horizon():
    """C4 with the port current at its peak (t0 = 200 ps, GAUSS_SINE delay 254.6 ps): 180
    leapfrog steps + a degree-16 substep, and a p = 8 solve over 120 steps (every sub-interval
    and tail), sampled at the port -- a domain of dependence of ~200 cells in x and y, the
    whole height in z."""
    w = config_c4(nsteps=200)
    port = (w.sources[0].i, w.sources[0].j, 5)
    _run_leapfrog_expmv(w, "f64", 180, 16, [port], half=4, t0=200e-12)
    _run_solve(w, "f64", 120, 8, 8, [port], half=4, t0=200e-12)


@pytest.mark.parametrize("n,dtype", [(768, "f32"), (512, "f64")])
def test_c5_max_sizes(n, dtype):
    """C5 vacuum at the largest sizes: 768^3 fp32 (5.5 GB per field) and 512^3 fp64; 20 leapfrog
    steps + the bench's degree-64 Leja substep; p = 8 solve on 768^3 fp32."""
    w = config_c5(n=n, dtype=dtype)
    _run_leapfrog_expmv(w, dtype, 20, 64, [(n // 2, n // 3, n - 10), (5, n - 3, 7)], half=4)
    if n == 768:
        _run_solve(w, dtype, 16, 8, 4, [(n // 2, n // 2, n // 2)], half=4)
