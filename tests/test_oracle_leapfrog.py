"""Pins of the oracle's leapfrog: invariants and closed forms."""
import math

import numpy as np
import pytest

from oracle import dense, fit
from synth import Source, config_c1, gauss_sine, random_fields

C_LIGHT = 1.0 / math.sqrt(fit.EPS0 * fit.MU0)


def _rand_state(g, seed):
    e, h = random_fields(g.nx, g.ny, g.nz, seed)
    return g.clean(e, h)


def test_zero_in_zero_out():
    g = fit.Grid(4, 4, 3, d0=1e-3, dt_frac=0.9)
    e, h = fit.leapfrog(g, *g.zeros(), 50)
    assert not e.any() and not h.any()


@pytest.mark.parametrize("eps_seed", [None, 3])
def test_energy_conserved_source_free(eps_seed):
    """E_m = e^m' M_eps e^m + h^(m-1/2)' M_mu h^(m+1/2) is constant and so
    is the paper's interpolated form (eq:energy)."""
    n = (5, 4, 4)
    eps = None if eps_seed is None else np.random.default_rng(eps_seed).uniform(1, 4, 80)
    g = fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.9)
    e, h = _rand_state(g, 7)                 # (e^0, h^{1/2})
    vals = []
    for m in range(2000):
        hprev = h                            # h^{m+1/2}
        e, h = fit.leapfrog(g, e, h, 1)      # (e^{m+1}, h^{m+3/2})
        vals.append(fit.energy_staggered(g, e, hprev, h))
    E0 = vals[0]
    drift = max(abs(v - E0) for v in vals) / E0
    assert drift < 1e-12


def test_energy_paper_interpolated_form():
    g = fit.Grid(4, 4, 4, d0=1e-3, dt_frac=0.95)
    e, h = _rand_state(g, 11)
    Me, Mm = g.M_eps_w(), g.M_mu_w()

    def paper_energy(e_m, e_m1, h_mmh, h_mph):
        # W_e^{m,m+1/2} + W_h^{m,m+1/2} with e^{m+1/2} = (e^m+e^{m+1})/2, h^m = (h^{m-1/2}+h^{m+1/2})/2
        return float(e_m @ (Me * 0.5 * (e_m + e_m1)) + (0.5 * (h_mmh + h_mph)) @ (Mm * h_mph))

    traj = [(e, h)]
    for _ in range(300):
        traj.append(fit.leapfrog(g, *traj[-1], 1))
    vals = [paper_energy(traj[m][0], traj[m + 1][0], traj[m - 1][1], traj[m][1])
            for m in range(1, 299)]
    assert (max(vals) - min(vals)) / abs(vals[0]) < 1e-12


def test_charge_identity_with_source():
    """S M_eps e^{m+1} = S M_eps e^m - dt S j^{m+1/2} at interior points:
    a +z source edge leaves -dt*j at its start point and +dt*j at its end point."""
    n = (4, 4, 4)
    g = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    src = Source(2, 2, 2, 1, "gauss_paper", 1.0, 2e-12)
    S = dense.divergence_primal(*n).astype(float)
    e, h = _rand_state(g, 5)
    Me = g.M_eps_w()
    m0 = 3
    e1, h1 = fit.leapfrog(g, e, h, 1, [src], t0=0.0, m0=m0)
    dq = S @ (Me * e1) - S @ (Me * e)
    t = (m0 + 0.5) * g.dt
    j = fit.waveform(src, t)
    start = 2 + 5 * (2 + 5 * 1)
    end = 2 + 5 * (2 + 5 * 2)
    scale = g.dt * abs(j)
    idx = np.indices((5, 5, 5)).reshape(3, -1)[::-1]
    interior = np.all((idx >= 1) & (idx <= 3), axis=0)
    expect = np.zeros(g.Np)
    expect[start] = -g.dt * j
    expect[end] = +g.dt * j
    assert np.abs(dq[interior] - expect[interior]).max() < 1e-10 * scale


def test_one_step_map_eigenvalues():
    """|lambda| = 1 and arg lambda = dt*omega_LF, omega_LF = (2/dt) asin(dt omega/2)
    (SURVEY finding 7)."""
    n = (3, 3, 2)
    g = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    ie = np.flatnonzero(g.live_e)
    ih = np.flatnonzero(g.live_h)
    N = len(ie) + len(ih)
    Mmap = np.zeros((N, N))
    for c in range(N):
        e, h = g.zeros()
        if c < len(ie):
            e[ie[c]] = 1.0
        else:
            h[ih[c - len(ie)]] = 1.0
        e1, h1 = fit.leapfrog(g, e, h, 1)
        Mmap[:, c] = np.concatenate([e1[ie], h1[ih]])
    lam = np.linalg.eigvals(Mmap)
    assert np.abs(np.abs(lam) - 1.0).max() < 1e-9
    ang = np.sort(np.abs(np.angle(lam)))
    ang = ang[ang > 1e-8]
    om = dense.cavity_frequencies(*n, 1e-3, C_LIGHT)
    ref = np.sort(np.concatenate([2 * np.arcsin(g.dt * om / 2)] * 2))
    assert len(ang) == len(ref)
    assert np.abs(ang - ref).max() < 1e-9


def test_cfl_stability_boundary():
    """0.99 CFL bounded, 1.05 CFL grows >= 1e3 in 2000 steps."""
    for frac, grows in [(0.99, False), (1.05, True)]:
        g = fit.Grid(8, 8, 8, d0=1e-3, dt_frac=frac)
        e, h = _rand_state(g, 3)
        E0 = g.energy_norm2(e, h)
        e, h = fit.leapfrog(g, e, h, 2000)
        E1 = g.energy_norm2(e, h)
        grew = (not np.isfinite(E1)) or E1 / E0 >= 1e3
        assert grew == grows


def test_second_order_convergence_vs_dense_exp():
    """Leapfrog -> exact exp(tA)u0 as O(dt^2): error ratio 4 +- 20% when dt halves."""
    n = (3, 3, 2)
    g0 = fit.Grid(*n, d0=1e-3, dt_frac=0.5)
    A, ie, ih, T = dense.dense_A(g0)
    # smooth initial data: the two lowest cavity modes
    w, V = np.linalg.eig(A)
    order = np.argsort(np.abs(w.imag) + (np.abs(w.imag) < 1e-3 * np.abs(w).max()) * 1e30)
    u = (V[:, order[0]] + V[:, order[2]]).real / T   # original variables
    T_end = 40 * g0.dt_cfl
    errs = []
    for frac in [0.4, 0.2, 0.1]:
        nsteps = int(round(T_end / (frac * g0.dt_cfl)))
        g = fit.Grid(*n, d0=1e-3, dt=T_end / nsteps)
        nh = len(ih)
        e0, h0 = g.zeros()
        h0[ih] = u[:nh]
        e0[ie] = u[nh:]
        # exact staggered start h(dt/2)
        uh = dense.expm_dense_apply(A, T, 0.5 * g.dt, u)
        h_half = np.zeros_like(h0)
        h_half[ih] = uh[:nh]
        e, h = fit.leapfrog(g, e0, h_half, nsteps)
        ex = dense.expm_dense_apply(A, T, T_end, u)
        errs.append(np.linalg.norm(e[ie] - ex[nh:]) / np.linalg.norm(ex[nh:]))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.2 < r1 < 4.8 and 3.2 < r2 < 4.8, errs


def test_cavity_resonances_dft():
    """C1 grid (8^3, 1 mm, 0.9 CFL): the probe spectrum peaks at the leapfrog frequencies
    f_LF = asin(dt*omega_sd/2)/(pi dt) of the closed-form cavity modes (north_star pin)."""
    w = config_c1()
    g = fit.Grid.from_workload(w)
    e, h = _rand_state(g, 123)
    nsteps = 1 << 15
    # record a few probe edges each step (plain loop over chunks of 1 step is slow; use
    # 16-step chunks and subsample is not allowed for a DFT -> record every step)
    probes = [g.edge_dof(2, 3, 5, 4), g.edge_dof(0, 2, 1, 3), g.edge_dof(1, 6, 3, 2)]
    sig = np.zeros((nsteps, len(probes)))
    for m in range(nsteps):
        e, h = fit.leapfrog(g, e, h, 1)
        sig[m] = e[probes]
    spec = np.sum(np.abs(np.fft.rfft(sig - sig.mean(0), axis=0)) ** 2, axis=1)
    freqs = np.fft.rfftfreq(nsteps, g.dt)
    om = np.unique(np.round(dense.cavity_frequencies(8, 8, 8, 1e-3, C_LIGHT), 3))
    f_lf = np.arcsin(g.dt * om / 2) / (math.pi * g.dt)
    f_sd = om / (2 * math.pi)
    binw = freqs[1]
    for fl, fs in zip(f_lf[:6], f_sd[:6]):
        b = int(round(fl / binw))
        window = spec[max(b - 40, 1):b + 41]
        peak = max(b - 40, 1) + int(np.argmax(window))
        assert abs(freqs[peak] - fl) <= 1.01 * binw, (fl, freqs[peak])
    # third mode up: f_LF and f_sd are more than one bin apart
    assert abs(f_lf[2] - f_sd[2]) > binw
