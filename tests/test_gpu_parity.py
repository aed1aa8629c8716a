"""GPU parity: the CUDA path (through the C ABI) vs the oracle on the same seeded inputs.

Tolerances (north_star): rel-L2 <= 1e-10 (fp64), <= 1e-4 (fp32, oracle fed the fp32-rounded
constants, DESIGN reading 24), separately for e (volts) and h (amperes)."""
import math

import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from gpu_util import (TOL, assert_parity, inputs, lib_expmv, lib_leapfrog, lib_solve, rel_l2)
from oracle import fit
from synth import (Source, config_c1, config_c2, config_c3, gauss_sine, layered_eps, random_fields,
                   spiral_pec_cells)

pytestmark = pytest.mark.gpu
KERNELS = ["unfused", "fused", "tma"]   # fused = auto choice (small / mid / TMA by size)


def _material(kind, n, seed=3):
    nx, ny, nz = n
    if kind == "vacuum":
        return None, None
    if kind == "layered":
        return layered_eps(nx, ny, nz, (1.0, 2.2, 4.4, 9.8)[:max(1, min(4, nz))]), None
    rng = np.random.default_rng(seed)
    eps = rng.uniform(1.0, 4.0, nx * ny * nz)
    pec = (rng.uniform(size=nx * ny * nz) < 0.03).astype(np.uint8)
    return eps, pec


def _grids(n, kind, dtype, kernels, frac=0.95):
    eps, pec = _material(kind, n)
    og = fit.Grid(*n, d0=1e-3, eps_r=eps, pec_cell=pec, dt_frac=frac, dtype=dtype)
    lg = pe.Grid(*n, d0=1e-3, eps_r=eps, pec_cell=pec, dt_frac=frac, dtype=dtype, kernels=kernels)
    return og, lg


def _sources(og, n):
    nx, ny, nz = n
    cands = [gauss_sine(2, nx // 2, ny // 3, nz // 2, f0=40e9, bw=40e9),
             Source(0, nx // 3, ny // 2, max(1, nz // 3), "gauss_paper", 0.7, 6e-12),
             Source(1, max(1, nx - 2), 1, max(1, nz - 2), "sine", 0.3, 0.0, 25e9, 0.0, 2.0)]
    return [s for s in cands if og.cE[og.edge_dof(s.comp, s.i, s.j, s.k)] != 0]


@pytest.mark.parametrize("kernels", KERNELS)
def test_leapfrog_c1(kernels):
    w = config_c1()
    og = fit.Grid.from_workload(w)
    lg = pe.Grid.from_workload(w, kernels=kernels)
    assert lg.info()["material_mode"] == pe.abi.MAT_SCALAR
    e, h = og.zeros()
    ref = fit.leapfrog(og, e, h, w.nsteps, w.sources)
    ge, gh, st = lib_leapfrog(lg, e, h, w.nsteps, w.sources)
    assert_parity((ge, gh), ref, "f64", "C1 leapfrog")
    assert st["curl_applications"] == 2 * w.nsteps          # eq:cost_LF
    assert np.linalg.norm(ref[0]) > 0


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["vacuum", "layered", "random"])
@pytest.mark.parametrize("kernels", KERNELS)
def test_leapfrog_ragged(dtype, kind, kernels):
    n = (37, 23, 11)
    og, lg = _grids(n, kind, dtype, kernels)
    e, h = inputs(og, *random_fields(*n, seed=41))
    src = _sources(og, n)
    t0 = 3.5e-12
    ref = fit.leapfrog(og, e, h, 300, src, t0=t0)
    ge, gh, _ = lib_leapfrog(lg, e, h, 300, src, t0=t0)
    assert_parity((ge, gh), ref, dtype, f"leapfrog {kind} {dtype}")
    # dead DOFs stay exactly zero
    assert not ge[~og.live_e].any() and not gh[~og.live_h].any()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("method,m,s", [("leja", 40, 3), ("leja", 1, 7), ("leja", 2, 5),
                                         ("leja", 64, 1), ("taylor", 16, 6), ("leja", 6, 2),
                                         ("leja", 10, 1), ("leja", 4, 3), ("leja", 150, 1)])
@pytest.mark.parametrize("kind", ["vacuum", "layered", "random"])
@pytest.mark.parametrize("kernels", KERNELS)
def test_expmv_fixed_plan(dtype, method, m, s, kind, kernels):
    n = (21, 19, 13)
    og, lg = _grids(n, kind, dtype, kernels)
    e, h = inputs(og, *random_fields(*n, seed=7))
    rho = og.rho_cfl
    tau = 30 * og.dt if method == "leja" else 6 * og.dt
    plan = fit.make_plan(method, m, s, tau, rho)
    ref = fit.expmv(og, plan, e, h, mode="pairs", dtype=dtype)
    ge, gh, st = lib_expmv(lg, tau, e, h, method=method, m=m, s=s, rho=rho)
    assert_parity((ge, gh), ref, dtype, f"expmv {method} m={m} s={s} {kind}")
    assert st["a_applications"] == m * s
    # plan equality (reading 25): m, s, nodes exactly; d-hat to 1e-14
    lp = pe.expmv_plan(lg, tau, method, m, s, rho=rho)
    assert (lp["m"], lp["s"]) == (plan.m, plan.s)
    assert abs(lp["gamma"] - plan.gamma) <= 1e-15 * plan.gamma
    assert max(abs(a - b) for a, b in zip(lp["d"], plan.d)) <= 1e-14


def test_expmv_vs_complex_newton_fp64():
    n = (16, 16, 12)
    og, lg = _grids(n, "random", "f64", "auto")
    e, h = inputs(og, *random_fields(*n, seed=9))
    plan = fit.make_plan("leja", 30, 4, 40 * og.dt, og.rho_cfl)
    ref = fit.expmv(og, plan, e, h, mode="complex")
    ge, gh, _ = lib_expmv(lg, 40 * og.dt, e, h, method="leja", m=30, s=4, rho=og.rho_cfl)
    assert_parity((ge, gh), ref, "f64", "expmv vs complex Newton")


def _fixed_s(method, m, tol, tau, rho):
    return max(1, math.ceil(tau * rho / fit.theta_m(method, m, tol)))


def test_solve_c1():
    """C1: 8^3 vacuum, 2000 steps, p = 2, Leja fixed plan (m = 40 at eps_A 1e-12)."""
    w = config_c1()
    og = fit.Grid.from_workload(w)
    lg = pe.Grid.from_workload(w)
    rho = og.rho_cfl
    S = fit.partition(w.nsteps, w.p)
    s = _fixed_s("leja", 40, 1e-12, (S[1] - S[0]) * og.dt, rho)
    ref = fit.paraexp(og, w.sources, 0.0, w.nsteps, w.p,
                      lambda tau: fit.make_plan("leja", 40, s, tau, rho), rho=rho)
    ge, gh, st = lib_solve(lg, w.nsteps, w.p, w.sources, method="leja", m=40, s=s, rho=rho)
    assert_parity((ge, gh), ref, "f64", "C1 solve")
    assert st["root"] == 0 and st["first_interval"] == 1 and st["last_interval"] == 2


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("p", [1, 3, 4, 61])
@pytest.mark.parametrize("kernels", KERNELS)
def test_solve_random_u0(dtype, p, kernels):
    n = (19, 17, 9)
    og, lg = _grids(n, "random", dtype, kernels)
    u0 = inputs(og, *random_fields(*n, seed=77))
    src = _sources(og, n)
    nsteps = 61
    rho = og.rho_cfl
    s = 6
    ref = fit.paraexp(og, src, 1e-12, nsteps, p, lambda tau: fit.make_plan("leja", 24, s, tau, rho),
                      u0=u0, rho=rho, dtype=dtype)
    ge, gh, _ = lib_solve(lg, nsteps, p, src, u0=u0, t0=1e-12, method="leja", m=24, s=s, rho=rho)
    assert_parity((ge, gh), ref, dtype, f"solve p={p} {dtype}")


def test_solve_leapfrog_tails_equal_serial():
    """tail = LEAPFROG reproduces serial leapfrog on the GPU path."""
    n = (19, 17, 9)
    og, lg = _grids(n, "random", "f64", "auto")
    u0 = inputs(og, *random_fields(*n, seed=5))
    src = _sources(og, n)
    ref = fit.leapfrog(og, u0[0], fit.half_step_start(og, *u0), 50, src)
    ge, gh, _ = lib_solve(lg, 50, 4, src, u0=u0, tail_mode="leapfrog", rho=og.rho_cfl, m=8, s=1)
    assert_parity((ge, gh), ref, "f64", "leapfrog tails")


def test_solve_c2_reduced():
    """C2 grid at full size (64^3, random eps), 400 of its 20000 steps, p = 8."""
    w = config_c2(nsteps=400)
    og = fit.Grid.from_workload(w)
    lg = pe.Grid.from_workload(w)
    assert lg.info()["material_mode"] == pe.abi.MAT_ARRAY
    rho = og.rho_cfl
    s = _fixed_s("leja", 40, 1e-10, 50 * og.dt, rho)
    ref = fit.paraexp(og, w.sources, 0.0, w.nsteps, w.p,
                      lambda tau: fit.make_plan("leja", 40, s, tau, rho), rho=rho)
    ge, gh, _ = lib_solve(lg, w.nsteps, w.p, w.sources, method="leja", m=40, s=s, rho=rho)
    assert_parity((ge, gh), ref, "f64", "C2 reduced solve")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c3_full_grid_short(dtype):
    """C3 at full size (256^3, layered): 12 leapfrog steps from random fields with the C3
    source, then exp(tau A) with a fixed degree-8 Leja plan."""
    w = config_c3(dtype=dtype)
    og = fit.Grid.from_workload(w)
    lg = pe.Grid.from_workload(w)
    assert lg.info()["material_mode"] == pe.abi.MAT_ZTABLE
    e, h = inputs(og, *random_fields(w.nx, w.ny, w.nz, seed=3))
    ref = fit.leapfrog(og, e, h, 12, w.sources, t0=100e-12)
    ge, gh, _ = lib_leapfrog(lg, e, h, 12, w.sources, t0=100e-12)
    assert_parity((ge, gh), ref, dtype, "C3 leapfrog")
    plan = fit.make_plan("leja", 8, 1, 3 * og.dt, og.rho_cfl)
    ref2 = fit.expmv(og, plan, *ref, mode="pairs", dtype=dtype)
    ge2, gh2, _ = lib_expmv(lg, 3 * og.dt, *ref, method="leja", m=8, s=1, rho=og.rho_cfl)
    assert_parity((ge2, gh2), ref2, dtype, "C3 expmv")


def test_spiral_pec_small():
    """C4-like structure on a small grid: PEC spiral + via + substrate, port sources."""
    nx, ny, nz = 64, 64, 16
    pec, port, _ = spiral_pec_cells(nx, ny, nz, k_trace=5, turns=3, width=2, gap=1, outer=40, k_sub=5)
    eps = np.ones((nz, ny, nx))
    eps[:5] = 11.9
    og = fit.Grid(nx, ny, nz, d0=25e-6, eps_r=eps.reshape(-1), pec_cell=pec, dt_frac=0.95)
    lg = pe.Grid(nx, ny, nz, d0=25e-6, eps_r=eps.reshape(-1), pec_cell=pec, dt_frac=0.95)
    src = [gauss_sine(2, port[0], port[1], k, f0=5e9, bw=10e9) for k in range(5)]
    e, h = og.zeros()
    ref = fit.leapfrog(og, e, h, 400, src)
    ge, gh, _ = lib_leapfrog(lg, e, h, 400, src)
    assert_parity((ge, gh), ref, "f64", "spiral leapfrog")
    assert np.linalg.norm(ref[0]) > 0


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["layered", "random"])
@pytest.mark.parametrize("kernels", KERNELS)
def test_leapfrog_trace(dtype, kind, kernels):
    """f1: per-step energy E_{m+1} (eq:energy) and probe values, fused (in-kernel block
    reductions) and unfused (trace kernel between the halves), vs the oracle."""
    n = (37, 23, 11)
    og, lg = _grids(n, kind, dtype, kernels)
    e, h = inputs(og, *random_fields(*n, seed=43))
    src = _sources(og, n)
    probes = [(s.comp, s.i, s.j, s.k) for s in src] + [(0, 5, 7, 3), (2, 36, 22, 10)]
    probes = [q for q in probes if og.cE[og.edge_dof(*q)] != 0]
    ref_e, ref_h, ref_en, ref_pr = fit.leapfrog_trace(og, e, h, 120, src, t0=1e-12, probes=probes)
    import torch
    from gpu_util import to_dev, to_host
    te, th = to_dev(e, lg), to_dev(h, lg)
    st, en, pr = pe.leapfrog_trace(lg, te, th, 120, src, 1e-12, probes=probes)
    torch.cuda.synchronize()
    assert_parity((to_host(te), to_host(th)), (ref_e, ref_h), dtype, "trace fields")
    tol = TOL[dtype]
    assert rel_l2(en.cpu().numpy(), ref_en) <= tol
    assert rel_l2(pr.cpu().numpy(), ref_pr) <= tol


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_solve_trace(dtype):
    """f1: energy / probes of the reconstructed solution at every sub-interval boundary vs
    the oracle's independent-tail boundary states."""
    n = (19, 17, 9)
    og, lg = _grids(n, "random", dtype, "auto")
    u0 = inputs(og, *random_fields(*n, seed=78))
    src = _sources(og, n)
    probes = [(s.comp, s.i, s.j, s.k) for s in src] + [(1, 3, 4, 5)]
    nsteps, p, m, s = 61, 4, 24, 6
    rho = og.rho_cfl
    states = fit.paraexp_boundary_states(og, src, 1e-12, nsteps, p,
                                         lambda tau: fit.make_plan("leja", m, s, tau, rho), u0=u0,
                                         rho=rho, dtype=dtype)
    ref_en = np.array([og.energy_norm2(ue, uh) for ue, uh in states])
    ref_pr = np.array([[ue[og.edge_dof(*q)] for q in probes] for ue, _ in states])
    import torch
    from gpu_util import to_dev
    eo = torch.zeros(3 * lg.npts, dtype=lg.torch_dtype(), device="cuda:0")
    ho = torch.zeros_like(eo)
    st, en, pr = pe.solve_trace(lg, nsteps, p, src, 1e-12, method="leja", m=m, s=s, rho=rho,
                                u0=(to_dev(u0[0], lg), to_dev(u0[1], lg)), e_out=eo, h_out=ho,
                                probes=probes)
    torch.cuda.synchronize()
    tol = TOL[dtype]
    assert rel_l2(en.cpu().numpy(), ref_en) <= tol
    assert rel_l2(pr.cpu().numpy(), ref_pr) <= tol
    ref = fit.paraexp(og, src, 1e-12, nsteps, p, lambda tau: fit.make_plan("leja", m, s, tau, rho),
                      u0=u0, rho=rho, dtype=dtype)
    assert_parity((eo.double().cpu().numpy(), ho.double().cpu().numpy()), ref, dtype, "solve_trace output")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["vacuum", "random"])
@pytest.mark.parametrize("l,s", [(12, 2), (30, 1), (5, 3)])
def test_expmv_krylov(dtype, kind, l, s):
    """f3: Krylov (Arnoldi, sigma = infinity) on the GPU vs the oracle's step-by-step Arnoldi
    in the same energy inner product."""
    n = (21, 19, 13)
    og, lg = _grids(n, kind, dtype, "auto")
    e, h = inputs(og, *random_fields(*n, seed=17))
    tau = 9 * og.dt
    ref_e, ref_h, apps = fit.expmv_krylov(og, l, s, tau, e, h, dtype=dtype)
    ge, gh, st = lib_expmv(lg, tau, e, h, method="krylov", m=l, s=s, rho=og.rho_cfl)
    assert_parity((ge, gh), (ref_e, ref_h), dtype, f"krylov l={l} s={s} {kind}")
    assert st["a_applications"] == apps


def test_solve_krylov_tails():
    """ParaExp with Krylov tails (the paper's third propagator) vs the oracle."""
    n = (19, 17, 9)
    og, lg = _grids(n, "random", "f64", "auto")
    u0 = inputs(og, *random_fields(*n, seed=79))
    src = _sources(og, n)
    rho = og.rho_cfl
    # oracle: Algorithm 1 sequentially with Krylov propagators E_i (Horner over the
    # sub-intervals, as paraexp() does for polynomial plans), then the dt/2 Taylor shift
    S = fit.partition(40, 4)
    We, Wh = og.clean(*u0)
    parts = []
    for i in range(1, 5):
        z = og.zeros()
        parts.append(fit.leapfrog(og, z[0], z[1], S[i] - S[i - 1], src, 0.0, S[i - 1]))
    for i in range(1, 5):
        We, Wh, _ = fit.expmv_krylov(og, 16, 2, (S[i] - S[i - 1]) * og.dt, We, Wh)
        if i < 4:
            ei, hi = parts[i - 1]
            We, Wh = We + ei, Wh + fit.sync_h(og, ei, hi)
    ref = fit.paraexp_finish(og, parts[-1], (We, Wh), rho)
    ge, gh, st = lib_solve(lg, 40, 4, src, u0=u0, method="krylov", m=16, s=2, rho=rho)
    assert_parity((ge, gh), ref, "f64", "solve krylov")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["layered", "random"])
@pytest.mark.parametrize("kernels", KERNELS)
def test_expmv_early_termination(dtype, kind, kernels):
    """f2: the device-side early termination (fused block-reduced energy norms + skip flag)
    makes the same stop decisions as the oracle and gives the same result."""
    n = (21, 19, 13)
    og, lg = _grids(n, kind, dtype, kernels)
    e, h = inputs(og, *random_fields(*n, seed=19))
    rho = og.rho_cfl
    tau = 1.0 * og.dt
    eps = 1e-6 if dtype == "f32" else 1e-9
    plan = fit.make_plan("leja", 60, 2, tau, rho)
    ref_e, ref_h, apps = fit.expmv_pairs_et(og, plan, e, h, eps, dtype=dtype)
    assert apps < 120
    ge, gh, st = lib_expmv(lg, tau, e, h, method="leja", m=60, s=2, rho=rho, eps_A=eps,
                           early_term=True)
    assert st["a_applications"] == apps
    assert_parity((ge, gh), (ref_e, ref_h), dtype, f"expmv early-term {kind}")


@pytest.mark.parametrize("kernels", KERNELS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_nonuniform_mesh(kernels, dtype):
    """f4: non-uniform spacings dx, dy, dz (per-edge cE and per-face cH arrays) -- leapfrog
    and expmv vs the oracle."""
    n = (23, 17, 9)
    rng = np.random.default_rng(8)
    dx, dy, dz = (rng.uniform(0.3e-3, 1.5e-3, k) for k in n)
    kw = dict(dx=dx, dy=dy, dz=dz, dt_frac=0.95, dtype=dtype)
    og = fit.Grid(*n, **kw)
    lg = pe.Grid(*n, kernels=kernels, **kw)
    assert lg.info()["material_mode"] == pe.abi.MAT_ARRAY
    e, h = inputs(og, *random_fields(*n, seed=23))
    src = _sources(og, n)
    ref = fit.leapfrog(og, e, h, 200, src)
    ge, gh, _ = lib_leapfrog(lg, e, h, 200, src)
    assert_parity((ge, gh), ref, dtype, "non-uniform leapfrog")
    plan = fit.make_plan("leja", 32, 3, 20 * og.dt, og.rho_cfl)
    ref2 = fit.expmv(og, plan, *ref, dtype=dtype)
    ge2, gh2, _ = lib_expmv(lg, 20 * og.dt, *ref, m=32, s=3, rho=og.rho_cfl)
    assert_parity((ge2, gh2), ref2, dtype, "non-uniform expmv")


@pytest.mark.parametrize("k", [1, 10])
def test_wave2d_solve(k):
    """The paper's 2-D cylindrical wave (41 x 41 x 2) over its full interval
    T = 2e-7 s, with one small element of ratio k (the R(k) study mesh): ParaExp p = 8 vs the
    oracle at a fixed Leja plan."""
    from synth import config_wave2d
    w = config_wave2d(41, k)
    og = fit.Grid.from_workload(w)
    lg = pe.Grid.from_workload(w)
    nt = math.ceil(w.t_end / og.dt)
    nt += (-nt) % 8
    rho = 1.05 * fit.norm_A(og)
    S = fit.partition(nt, 8)
    s = _fixed_s("leja", 40, 1e-10, (S[1] - S[0]) * og.dt, rho)
    ref = fit.paraexp(og, w.sources, 0.0, nt, 8, lambda tau: fit.make_plan("leja", 40, s, tau, rho),
                      rho=rho)
    ge, gh, st = lib_solve(lg, nt, 8, w.sources, method="leja", m=40, s=s, rho=rho)
    assert_parity((ge, gh), ref, "f64", f"wave2d k={k}")
    assert np.linalg.norm(ref[0]) > 0


@pytest.mark.parametrize("k", [1, 5, 20])
def test_rho_pow_vs_oracle_norm(k):
    """K5 (library Lanczos) vs the oracle's ARPACK ||A||_2 on the R(k) meshes (SPEC: 1e-3)."""
    from synth import config_wave2d
    w = config_wave2d(41, k)
    og = fit.Grid.from_workload(w)
    lg = pe.Grid.from_workload(w)
    rp = lg.info(compute_rho_pow=True)["rho_pow"]
    ref = fit.norm_A(og)
    assert abs(rp - ref) <= 1e-3 * ref, (rp, ref)
