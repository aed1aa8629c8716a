"""Pins of the oracle's trace outputs: the leapfrog energy
trace (eq:energy) and the ParaExp boundary states u(T_i)."""
import math

import numpy as np

from oracle import fit
from synth import Source, gauss_sine, random_fields


def _grid(n=(5, 4, 4), eps_seed=3):
    eps = np.random.default_rng(eps_seed).uniform(1, 4, int(np.prod(n)))
    return fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.9)


def test_leapfrog_trace_energy_constant_without_source():
    """without excitation the leapfrog energy E_m is conserved exactly."""
    g = _grid()
    e, h = g.clean(*random_fields(g.nx, g.ny, g.nz, 5))
    _, _, en, _ = fit.leapfrog_trace(g, e, h, 200)
    assert np.ptp(en) <= 1e-12 * en[0] and en[0] > 0


def test_leapfrog_trace_energy_after_pulse():
    """Energy rises while the pulse acts and stays constant once i_L(t) = 0
    (Fig. 7)."""
    g = _grid()
    src = [Source(2, 2, 2, 1, "gauss_paper", 1.0, 4 * g.dt)]     # i_L ~ 0 after ~3 sigma_t
    e, h = g.zeros()
    _, _, en, _ = fit.leapfrog_trace(g, e, h, 120, src)
    assert en[0] >= 0 and en[40] > 0
    tail = en[60:]
    assert np.ptp(tail) <= 1e-10 * tail.mean()


def test_leapfrog_trace_matches_plain_run_and_probes():
    g = _grid()
    src = [gauss_sine(1, 2, 1, 2, f0=50e9, bw=50e9)]
    e, h = g.clean(*random_fields(g.nx, g.ny, g.nz, 9))
    probes = [(1, 2, 1, 2), (0, 1, 2, 3), (2, 4, 3, 1)]
    e1, h1, en, pr = fit.leapfrog_trace(g, e, h, 30, src, t0=2e-12, probes=probes)
    e2, h2 = fit.leapfrog(g, e, h, 30, src, t0=2e-12)
    assert np.array_equal(e1, e2) and np.array_equal(h1, h2)
    assert np.array_equal(pr[-1], [e2[g.edge_dof(*q)] for q in probes])
    e3, h3 = fit.leapfrog(g, e, h, 17, src, t0=2e-12)
    assert np.array_equal(pr[16], [e3[g.edge_dof(*q)] for q in probes])


def _accurate(g, rho, m=40, tol=1e-15):
    th = fit.theta_m("leja", m, 1e-14)

    def pf(tau):
        return fit.make_plan("leja", m, max(1, math.ceil(tau * rho / th)), tau, rho)
    return pf


def test_boundary_states_energy_conserved_by_exp():
    """g = 0: u(T_i) = exp((T_i - t0) A) u0, and exp of the skew operator preserves the energy
    norm <e,e>_eps + <h,h>_mu -- to the Leja tolerance."""
    g = _grid()
    u0 = g.clean(*random_fields(g.nx, g.ny, g.nz, 21))
    states = fit.paraexp_boundary_states(g, [], 0.0, 40, 4, _accurate(g, g.rho_cfl), u0=u0)
    E0 = g.energy_norm2(*u0)
    for ue, uh in states:
        assert abs(g.energy_norm2(ue, uh) - E0) <= 1e-11 * E0


def test_boundary_state_p_equals_solution_output():
    """u(T_p) (independent tails) has the e of the paraexp output (eq:averaging1, Horner)."""
    g = _grid()
    src = [gauss_sine(2, 2, 2, 1, f0=60e9, bw=60e9)]
    u0 = g.clean(*random_fields(g.nx, g.ny, g.nz, 4))
    pf = _accurate(g, g.rho_cfl)
    states = fit.paraexp_boundary_states(g, src, 0.0, 30, 3, pf, u0=u0)
    eo, ho = fit.paraexp(g, src, 0.0, 30, 3, pf, u0=u0)
    ue, uh = states[-1]
    np.testing.assert_allclose(ue, eo, rtol=0, atol=1e-12 * np.abs(eo).max())


def test_boundary_states_converge_to_serial_leapfrog():
    """u(T_i) (e part) approaches the serial leapfrog e at step S_i as O(dt^2) (the
    leapfrog-vs-exact error of the tails)."""
    n = (4, 4, 3)
    errs = []
    for frac in (0.4, 0.2):
        g = fit.Grid(*n, d0=1e-3, dt_frac=frac)
        u0 = g.clean(*random_fields(*n, 8))
        T = 40 * 1.0e-12
        nsteps = int(round(T / g.dt))
        nsteps -= nsteps % 4
        g = fit.Grid(*n, d0=1e-3, dt=T / nsteps)
        u0 = g.clean(*random_fields(*n, 8))
        states = fit.paraexp_boundary_states(g, [], 0.0, nsteps, 4, _accurate(g, g.rho_cfl), u0=u0)
        e_ref, _ = fit.leapfrog(g, u0[0], fit.half_step_start(g, *u0), nsteps // 2)
        errs.append(np.linalg.norm(states[1][0] - e_ref) / np.linalg.norm(e_ref))
    assert 2.5 < errs[0] / errs[1] < 6.0
