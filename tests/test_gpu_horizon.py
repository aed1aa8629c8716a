"""GPU parity at the configs' stated runs and with the bench's own (auto) plan (north_star:
"GPU fields match the oracle ... on all five configs"; PAPER:309-316 partition, PAPER:436-448
planner).

* C2 (64^3, per-edge eps, 3 sources): the full 20000 steps, p = 8, on the AUTO plan the bench
  uses (rho = 0 -> the K5 estimate, (m, s) from the planner at eps_A = 1e-10).  The library's
  plan (rho, m, s) is read from the stats and the oracle runs Algorithm 1 with exactly that
  plan (reading 25) on the whole grid -- fp64, and the same run in fp32 (reading 24's constant
  recipe) for the fp32 drift over a long horizon (20000 steps + ~37000 A-applications).
* C3 256^3 with p = 64 (BASELINE configs[2]: "8 and 64 sub-intervals"): the WHOLE grid against
  the oracle, 64 steps (one per sub-interval), 63 Horner propagators -- every sub-interval,
  tail and the reduction order of the bench's launch configuration.
* C5 768^3 fp64 (the largest fp64 sweep size), sampled domains of dependence.
Each comparison is rel-L2 per field plus a max-abs check (a localised error on a few edges
would be diluted in the rel-L2 of a large box)."""
import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from gpu_util import TOL, assert_parity, inputs, lib_solve, rel_l2, to_host
from oracle import fit
from synth import config_c2, config_c3, config_c5, random_fields

pytestmark = pytest.mark.gpu


def assert_maxabs(got, ref, dtype, what, factor=20.0):
    for g, r, name in zip(got, ref, "eh"):
        err = np.abs(np.asarray(g) - np.asarray(r)).max() / np.abs(r).max()
        assert err <= factor * TOL[dtype], f"{what}: max-abs {name} {err:.3e}"


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c2_full_horizon_auto_plan(dtype):
    w = config_c2()
    og = fit.Grid.from_workload(w, dtype=dtype)
    lg = pe.Grid.from_workload(w, dtype=dtype)
    got = lib_solve(lg, w.nsteps, w.p, w.sources, eps_A=1e-10)          # auto rho, m, s
    st = got[2]
    assert w.nsteps % w.p == 0 and st["s_first"] == st["s_last"]
    assert st["rho_fallback"] == 0 and st["rho"] < og.rho_cfl            # K5's tight rho (finding 8)
    assert st["leapfrog_steps"] == w.nsteps
    m, s, rho = st["m"], st["s_first"], st["rho"]
    ref = fit.paraexp(og, w.sources, 0.0, w.nsteps, w.p, lambda tau: fit.make_plan("leja", m, s, tau, rho),
                      rho=rho, dtype=dtype)
    assert_parity(got[:2], ref, dtype, f"C2 {dtype} 20000 steps auto plan m={m} s={s}")
    assert_maxabs(got[:2], ref, dtype, f"C2 {dtype}")


def test_c3_p64_whole_grid():
    """C3 256^3 fp64, p = 64: one step per sub-interval, degree-8 Leja propagators, random u0
    plus the C3 source; the whole 2 x 50.9 M-value output against the oracle."""
    import torch
    w = config_c3("f64")
    nsteps, p, m = 64, 64, 8
    og = fit.Grid.from_workload(w, dtype="f64")
    lg = pe.Grid.from_workload(w, dtype="f64")
    assert abs(lg.dt - og.dt) <= 1e-15 * og.dt
    rho = og.rho_cfl
    u0 = og.clean(*random_fields(w.nx, w.ny, w.nz, seed=64))
    got = lib_solve(lg, nsteps, p, w.sources, u0=u0, m=m, s=1, rho=rho)
    st = got[2]
    assert st["root"] == 0 and st["last_interval"] == p
    plan_for = lambda tau: fit.make_plan("leja", m, 1, tau, rho)           # noqa: E731
    W, P = fit.paraexp_block(og, w.sources, 0.0, nsteps, p, plan_for, 1, p, u0=u0)
    ref = fit.paraexp_finish(og, P, W, rho)
    assert_parity(got[:2], ref, "f64", "C3 p=64 whole grid")
    assert_maxabs(got[:2], ref, "f64", "C3 p=64 whole grid")
    lg.close()
    torch.cuda.empty_cache()


def test_c5_768_fp64_sampled():
    """C5 768^3 fp64 (21.8 GB per state): 20 leapfrog steps + the sweep's degree-64 Leja substep,
    sampled domains of dependence (the method of tests/test_gpu_fullsize.py)."""
    from test_gpu_fullsize import _run_leapfrog_expmv
    n = 768
    w = config_c5(n=n, dtype="f64")
    _run_leapfrog_expmv(w, "f64", 20, 64, [(n // 2, n // 3, n - 10), (5, n - 3, 7)], half=4)


def test_c3r_refined_full_interval_auto_plan():
    """C3r (C3 with the centre cell column and row refined to Delta/k; reading 32 in 3-D) at
    24^3 and k = 10: the whole interval T = 7.49 ns (n_t from T, ~33500 steps at the refined
    mesh's eq:cfl step), p = 8, on the AUTO plan (K5's rho, planner (m, s)) -- the per-edge /
    per-face coefficient kernels of the G = 1..8 refined-mesh model, against
    Algorithm 1 in the oracle with the library's plan."""
    import math
    from synth import config_c3r
    w = config_c3r(k=10.0, n=24)
    og = fit.Grid.from_workload(w, dtype="f64")
    lg = pe.Grid.from_workload(w, dtype="f64")
    nsteps = int(math.ceil(w.t_end / lg.dt))
    nsteps -= nsteps % w.p
    # random initial fields beside the source: driven from zero, the PEC cavity ends with the
    # pulse's large static e (charge) and a ringing h ~1e-6 of it in Z0 units, whose rel-L2
    # would measure rounding against a near-zero norm (h 2e-10 there, e 2e-13)
    u0 = og.clean(*random_fields(w.nx, w.ny, w.nz, seed=10))
    got = lib_solve(lg, nsteps, w.p, w.sources, u0=u0, eps_A=1e-10)
    st = got[2]
    assert st["rho_fallback"] == 0 and st["rho"] < 0.5 * og.rho_cfl     # ||A|| far below the CFL bound
    m, s, rho = st["m"], st["s_first"], st["rho"]
    ref = fit.paraexp(og, w.sources, 0.0, nsteps, w.p, lambda tau: fit.make_plan("leja", m, s, tau, rho),
                      u0=u0, rho=rho, dtype="f64")
    assert_parity(got[:2], ref, "f64", f"C3r k=10 24^3 {nsteps} steps m={m} s={s}")
    assert_maxabs(got[:2], ref, "f64", "C3r k=10")
    lg.close()
