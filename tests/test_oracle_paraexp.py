"""Pins of the oracle's ParaExp: exact identities, paper/SPEC
worked examples, convergence to serial leapfrog."""
import json
import math
import os

import numpy as np
import pytest

from oracle import dense, fit
from synth import Source, gauss_sine, random_fields

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_partition_example():
    ex = GOLD["partition_example"]
    S = fit.partition(ex["nsteps"], ex["p"])
    assert [b - a for a, b in zip(S[:-1], S[1:])] == ex["steps"]
    assert fit.partition(10, 1) == [0, 10]
    with pytest.raises(ValueError):
        fit.partition(3, 4)


def test_cost_proc_example():
    ex = GOLD["cost_proc_example"]
    assert fit.cost_proc(ex["nt"], ex["p"], ex["n_leja"]) == ex["C_proc"]


def _setup(n=(4, 4, 3), eps_seed=None, frac=0.9):
    eps = None if eps_seed is None else np.random.default_rng(eps_seed).uniform(1, 4, np.prod(n))
    g = fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=frac)
    src = [gauss_sine(2, n[0] // 2, n[1] // 2, 1, f0=60e9, bw=60e9),
           Source(0, 1, 1, 1, "gauss_paper", 0.5, 8e-12)]
    return g, src


def _plan_for(g, rho, m=40, tol=1e-14, method="leja"):
    th = fit.theta_m(method, m, tol)

    def pf(tau):
        return fit.make_plan(method, m, max(1, math.ceil(tau * rho / th)), tau, rho)
    return pf


def test_p1_equals_serial_leapfrog():
    g, src = _setup()
    ref = fit.leapfrog(g, *g.zeros(), 60, src)
    out = fit.paraexp(g, src, 0.0, 60, 1, _plan_for(g, g.rho_cfl))
    assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])


@pytest.mark.parametrize("p", [2, 3, 5])
def test_leapfrog_tails_equal_serial(p):
    """Propagating the staggered seeds with leapfrog reproduces serial leapfrog to roundoff
    (SURVEY finding 2), with sources and a nonzero u0."""
    g, src = _setup(eps_seed=4)
    u0 = g.clean(*random_fields(g.nx, g.ny, g.nz, 17))
    n = 61
    out = fit.paraexp(g, src, 1e-12, n, p, None, u0=u0, tail="leapfrog")
    e0, h0 = u0
    ref = fit.leapfrog(g, e0, fit.half_step_start(g, e0, h0), n, src, t0=1e-12)
    for a, b in zip(out, ref):
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)


def test_source_free_is_pure_expmv():
    """g = 0 => every v_j = 0 and the result is exp(T A) u0: e at T, h at T+dt/2,
    checked against the dense exponential."""
    g, _ = _setup(n=(3, 3, 2))
    A, ie, ih, T = dense.dense_A(g)
    u0 = g.clean(*random_fields(g.nx, g.ny, g.nz, 2))
    n, p = 40, 4
    out = fit.paraexp(g, [], 0.0, n, p, _plan_for(g, g.rho_cfl), u0=u0)
    u = np.concatenate([u0[1][ih], u0[0][ie]])
    nh = len(ih)
    ref_e = dense.expm_dense_apply(A, T, n * g.dt, u)[nh:]
    ref_h = dense.expm_dense_apply(A, T, (n + 0.5) * g.dt, u)[:nh]
    assert np.linalg.norm(out[0][ie] - ref_e) <= 1e-12 * np.linalg.norm(ref_e)
    assert np.linalg.norm(out[1][ih] - ref_h) <= 1e-12 * np.linalg.norm(ref_h)


def test_horner_equals_independent_tails():
    """W by Horner == W by independent tails summed in order (SURVEY finding 9)."""
    g, src = _setup(eps_seed=6)
    u0 = g.clean(*random_fields(g.nx, g.ny, g.nz, 5))
    pf = _plan_for(g, g.rho_cfl, m=30, tol=1e-12)
    a = fit.paraexp(g, src, 0.0, 48, 4, pf, u0=u0, sum_mode="horner")
    b = fit.paraexp(g, src, 0.0, 48, 4, pf, u0=u0, sum_mode="independent")
    for x, y in zip(a, b):
        assert np.linalg.norm(x - y) <= 1e-12 * np.linalg.norm(y)


def test_exp_tails_converge_to_leapfrog_second_order():
    """ParaExp with (accurate) exponential tails differs from serial leapfrog by leapfrog's
    own O(dt^2) error: the gap drops ~4x when dt halves (SURVEY finding 2)."""
    n = (4, 4, 3)
    g0 = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    T_end = 24 * g0.dt
    src = [Source(2, 2, 2, 1, "gauss_paper", 1.0, 6 * g0.dt)]
    gaps = []
    for div in [1, 2, 4]:
        nsteps = 24 * div
        g = fit.Grid(*n, d0=1e-3, dt=T_end / nsteps)
        out = fit.paraexp(g, src, 0.0, nsteps, 3, _plan_for(g, g.rho_cfl))
        ref = fit.leapfrog(g, *g.zeros(), nsteps, src)
        gaps.append(np.linalg.norm(out[0] - ref[0]) / np.linalg.norm(ref[0]))
    r1, r2 = gaps[0] / gaps[1], gaps[1] / gaps[2]
    assert 3.0 < r1 < 5.0 and 3.0 < r2 < 5.0, gaps


def test_fp32_constants_paraexp_close():
    g, src = _setup()
    g32 = fit.Grid(g.nx, g.ny, g.nz, d0=1e-3, dt_frac=0.9, dtype="f32")
    a = fit.paraexp(g, src, 0.0, 40, 2, _plan_for(g, g.rho_cfl, m=20, tol=1e-10))
    b = fit.paraexp(g32, src, 0.0, 40, 2, _plan_for(g, g.rho_cfl, m=20, tol=1e-10))
    for x, y in zip(a, b):
        assert np.linalg.norm(x - y) / np.linalg.norm(x) < 1e-5
