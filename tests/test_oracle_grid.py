"""Pins of the oracle's grid, curls, materials, CFL and spectrum (CPU only).

Each pin checks the oracle against something other than itself: paper-printed
values (tests/golden), integer identities of the FIT complex, closed forms, and a
dense incidence matrix enumerated from face geometry (oracle/dense.py)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import dense, fit

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
C_LIGHT = 1.0 / math.sqrt(fit.EPS0 * fit.MU0)


@pytest.mark.parametrize("case", GOLD["dof_counts"])
def test_dof_counts_paper(case):
    # n_dof counts e and h with 3 entries per primal point each (reading 3)
    nxp, nyp, nzp = case["points"]
    g = fit.Grid(nxp - 1, nyp - 1, nzp - 1, d0=0.5, dt_frac=0.9)
    assert 6 * g.Np == case["n_dof"]


def test_spiral_dof_convention():
    v = GOLD["spiral_dofs_per_field"]["value"]
    assert v % 3 == 0 and v // 3 == 427680


@pytest.mark.parametrize("n", [(2, 2, 1), (3, 3, 2), (2, 3, 4)])
def test_curl_matches_geometric_incidence(n):
    """Stencil curls (fit_oracle.c) == incidence enumerated from face boundaries, exactly
    on integer data (SPEC:53 hand-assembled incidence)."""
    g = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    C = dense.incidence_curl(*n)
    rng = np.random.default_rng(1)
    Np = g.Np
    # integer data on non-virtual entries (virtual entries are 0 by the layout convention)
    e = rng.integers(-50, 50, size=3 * Np).astype(float)
    h = rng.integers(-50, 50, size=3 * Np).astype(float)
    nn = np.array(n)
    idx = np.indices((n[2] + 1, n[1] + 1, n[0] + 1)).reshape(3, -1)[::-1]  # i, j, k
    for c in range(3):
        virt_e = idx[c] == nn[c]                          # edge leaves the lattice
        e[c * Np:(c + 1) * Np][virt_e] = 0
        a, b = (c + 1) % 3, (c + 2) % 3
        virt_h = (idx[a] == nn[a]) | (idx[b] == nn[b])     # face leaves the lattice
        h[c * Np:(c + 1) * Np][virt_h] = 0
    assert np.array_equal(C @ e, g.curl(e))
    assert np.array_equal(C.T @ h, g.curlT(h))


@pytest.mark.parametrize("n", [(2, 2, 1), (3, 3, 2), (3, 2, 4)])
def test_div_curl_identities(n):
    """S-tilde C = 0 (cells) and C S^T = 0 on faces inside the lattice."""
    C = dense.incidence_curl(*n)
    St = dense.divergence_dual(*n)
    S = dense.divergence_primal(*n)
    assert not np.any(St @ C)
    nn = np.array(n)
    Np = np.prod(nn + 1)
    idx = np.indices((n[2] + 1, n[1] + 1, n[0] + 1)).reshape(3, -1)[::-1]
    rows = []
    for c in range(3):
        a, b = (c + 1) % 3, (c + 2) % 3
        inside = (idx[a] < nn[a]) & (idx[b] < nn[b])
        rows.append(c * Np + np.flatnonzero(inside))
    rows = np.concatenate(rows)
    assert not np.any(C[rows] @ S.T)


def test_skew_A_and_spectrum_closed_form():
    """A = T A_orig T^-1 is skew and its spectrum equals the closed-form
    discrete cavity frequencies (SURVEY finding 7); rho < 2/dt_CFL."""
    for n in [(3, 3, 2), (4, 4, 3), (4, 3, 4)]:
        g = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
        A, ie, ih, T = dense.dense_A(g)
        assert np.abs(A + A.T).max() <= 1e-15 * np.abs(A).max()
        w = np.linalg.eigvals(A)
        assert np.abs(w.real).max() < 1e-6 * np.abs(w).max()
        om = np.sort(np.abs(w.imag))
        om = om[om > 1e-6 * om.max()]
        ref = dense.cavity_frequencies(*n, 1e-3, C_LIGHT)
        ref2 = np.sort(np.concatenate([ref, ref]))   # +/- i omega
        assert len(om) == len(ref2)
        assert np.abs(om - ref2).max() <= 1e-12 * om.max()
        assert om.max() < g.rho_cfl


def test_rho_8cube_ratio():
    # closed form: rho/rho_CFL = sin(7 pi/16) on 8^3 (SURVEY finding 7)
    ref = dense.cavity_frequencies(8, 8, 8, 1e-3, C_LIGHT).max()
    g = fit.Grid(8, 8, 8, d0=1e-3, dt_frac=0.9)
    assert abs(ref / g.rho_cfl - math.sin(7 * math.pi / 16)) < 1e-12


def test_uniform_vacuum_material_values():
    """Interior M_eps = eps0*d, M_nu = 1/(mu0*d); doubling eps doubles M_eps."""
    d = 2e-3
    g = fit.Grid(4, 4, 4, d0=d, dt_frac=0.9)
    live = g.live_e
    assert np.allclose(g.Meps[live], fit.EPS0 * d, rtol=1e-14, atol=0)
    assert np.allclose(g.Mnu[g.live_h], 1.0 / (fit.MU0 * d), rtol=1e-14, atol=0)
    g2 = fit.Grid(4, 4, 4, d0=d, eps_r=np.full(64, 2.0), dt_frac=0.9)
    assert np.allclose(g2.Meps[live], 2 * g.Meps[live], rtol=1e-15, atol=0)
    # substrate eps_r = 12 -> 12x the vacuum metric
    g3 = fit.Grid(4, 4, 4, d0=d, eps_r=np.full(64, 12.0), dt_frac=0.9)
    assert np.allclose(g3.Meps[live], 12 * g.Meps[live], rtol=1e-14, atol=0)


def test_cfl_closed_form():
    """eq:cfl at uniform vacuum d = 0.5 m equals d/(c sqrt 3) = 9.6292e-10 s (finding 6)."""
    gold = GOLD["cfl_example"]
    g = fit.Grid(3, 3, 3, d0=gold["d"], dt_frac=1.0)
    assert abs(g.dt_cfl - gold["d"] / (C_LIGHT * math.sqrt(3))) < 1e-24
    assert f"{g.dt_cfl:.4e}" == f"{gold['dt_cfl']:.4e}"
    g2 = fit.Grid(3, 3, 3, d0=2 * gold["d"], dt_frac=1.0)
    assert abs(g2.dt_cfl / g.dt_cfl - 2.0) < 1e-14
    # one cell shrunk by k -> dt_CFL shrinks by k
    k = 5.0
    dx = np.array([0.5, 0.5 / k, 0.5])
    g3 = fit.Grid(3, 3, 3, dx=dx, dy=np.full(3, 0.5 / k), dz=np.full(3, 0.5 / k), dt_frac=1.0)
    assert abs(g3.dt_cfl - (0.5 / k) / (C_LIGHT * math.sqrt(3))) < 1e-12 * g3.dt_cfl


def test_pec_and_liveness():
    """PEC box: tangential boundary edges dead, boundary-normal faces dead; PEC cell kills
    its 12 edges (reading 5)."""
    g = fit.Grid(3, 3, 3, d0=1e-3, dt_frac=0.9)
    # live counts: ex live i<3, 1<=j<=2, 1<=k<=2 -> 3*2*2 per comp
    assert g.live_e.sum() == 3 * (3 * 2 * 2)
    assert g.live_h.sum() == 3 * (2 * 3 * 3)
    pec = np.zeros(27, np.uint8)
    pec[1 + 3 * (1 + 3 * 1)] = 1          # centre cell
    gp = fit.Grid(3, 3, 3, d0=1e-3, pec_cell=pec, dt_frac=0.9)
    assert g.live_e.sum() - gp.live_e.sum() == 12


def test_line_current_values():
    gl = GOLD["line_current"]
    from synth import Source
    s = Source(2, 0, 0, 0, "gauss_paper", gl["i_max"], gl["sigma_t"])
    assert abs(fit.waveform(s, 0.0) - gl["i_at_0"]) < 1e-15
    assert fit.waveform(s, gl["sigma_t"]) == gl["i_at_sigma"]
