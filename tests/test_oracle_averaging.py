"""Pins of the oracle's material averaging (DESIGN reading 4, eq:maxwell_grid3,
is silent on how M_eps and M_nu average cells and spacings).  CPU only.

(a) Exact pin, non-uniform spacings.  On a PEC box with arbitrary spacings along one axis
    (say x) and uniform ones along the other two, the field E = E_x(y, z) x-hat, uniform in x,
    is an exact eigenmode of the FIT operator: its grid voltages are e_x(i,j,k) = dx_i f(j,k)
    (e = integral of E along the edge), the dual voltages h = M_nu C e come out
    independent of i, so C^T h has no y/z part, and M_eps^-1 C^T M_nu C e = omega^2 e with
        omega = 2c sqrt(sin^2(m_y pi / 2N_y)/dy^2 + sin^2(m_z pi / 2N_z)/dz^2),
    the uniform-grid closed form (SURVEY finding 7) -- independent of every dx_i.  Any slip in
    which spacing divides which edge/face (a dx_{i-1}, an averaged dx, a transposed dy/dz)
    breaks the identity at round-off level.  Checked as an operator residual and in the dense
    spectrum of A (oracle/dense.py), cyclically for x, y and z.

(b) Convergence pin, heterogeneous material.  A PEC cavity with n_y = 1 (the e_y-only modes
    E_y(x, z), uniform in y) filled with two slabs whose interface lies on a grid plane
    z = d.  The continuum mode sin(pi x / L_x) Z(z) has Z'' + (omega^2 eps_i mu_i - k_x^2) Z = 0
    in each slab, Z(0) = Z(L_z) = 0, Z and Z'/mu continuous at z = d, i.e. the root of
        k_1 cot(k_1 d)/mu_1 + k_2 cot(k_2 (L_z - d))/mu_2 = 0.
    The FIT eigenfrequency must converge to it at second order (error ratio ~4 per halving of
    the cell).  The interface edges (tangential E) need the area-weighted ARITHMETIC mean of
    eps over the cells around them, the interface-crossing dual edges (normal B) the length-
    weighted mean of 1/mu along them -- reading 4; a wrong cell pair gives first order, which
    the test demonstrates on a deliberately mis-averaged M_eps.
"""
import math

import numpy as np
import pytest
from scipy.linalg import eigh
from scipy.optimize import brentq

from oracle import dense, fit

C_LIGHT = 1.0 / math.sqrt(fit.EPS0 * fit.MU0)


# ---------------------------------------------------------------------------------------
# (a) non-uniform spacings: m = 0 modes along the non-uniform axis
# ---------------------------------------------------------------------------------------
def _grid_axis_nonuniform(axis, rng):
    n = [4, 5, 3]
    n[axis], n[(axis + 1) % 3] = 5, 4                     # 5 cells along the random axis
    d_uni = [1.0e-3, 1.3e-3, 0.8e-3]                      # distinct, so a swapped axis shows
    sp = [np.full(n[a], d_uni[a]) for a in range(3)]
    sp[axis] = rng.uniform(0.3e-3, 2.0e-3, n[axis])
    g = fit.Grid(*n, dx=sp[0], dy=sp[1], dz=sp[2], dt_frac=0.9)
    return g, n, sp


def _mode(g, n, sp, axis, mb, mg):
    """e along `axis` = d_axis[i_axis] * sin(mb pi j_b / N_b) sin(mg pi j_g / N_g)."""
    b, c = (axis + 1) % 3, (axis + 2) % 3
    Np = g.Np
    idx = np.indices((n[2] + 1, n[1] + 1, n[0] + 1)).reshape(3, -1)[::-1]   # i, j, k
    e = np.zeros(3 * Np)
    ia = np.minimum(idx[axis], n[axis] - 1)
    val = sp[axis][ia] * np.sin(mb * math.pi * idx[b] / n[b]) * np.sin(mg * math.pi * idx[c] / n[c])
    val[idx[axis] == n[axis]] = 0.0                       # virtual edges
    e[axis * Np:(axis + 1) * Np] = val
    om = 2 * C_LIGHT * math.sqrt(math.sin(mb * math.pi / (2 * n[b])) ** 2 / sp[b][0] ** 2
                                 + math.sin(mg * math.pi / (2 * n[c])) ** 2 / sp[c][0] ** 2)
    return np.where(g.live_e, e, 0.0), om


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_nonuniform_spacing_m0_modes_exact(axis):
    rng = np.random.default_rng(10 + axis)
    g, n, sp = _grid_axis_nonuniform(axis, rng)
    b, c = (axis + 1) % 3, (axis + 2) % 3
    Meps = np.where(g.live_e, g.Meps, 1.0)
    Mnu = np.where(g.live_h, g.Mnu, 0.0)
    A, *_ = dense.dense_A(g)
    spec = np.sort(np.abs(np.linalg.eigvals(A).imag))
    for mb in range(1, n[b]):
        for mg in range(1, n[c]):
            e, om = _mode(g, n, sp, axis, mb, mg)
            h = Mnu * g.curl(e)                                     # dual voltages
            # h independent of the position along the non-uniform axis
            hv = h.reshape(3, n[2] + 1, n[1] + 1, n[0] + 1)
            ax_np = 2 - axis                                        # numpy axis of `axis`
            for comp in (b, c):
                blk = np.take(hv[comp], range(n[axis]), axis=ax_np)
                ref = np.take(blk, [0], axis=ax_np)
                assert np.abs(blk - ref).max() <= 1e-12 * np.abs(h).max()
            Ke = np.where(g.live_e, g.curlT(h) / Meps, 0.0)        # M_eps^-1 C^T M_nu C e
            res = np.linalg.norm(Ke - om ** 2 * e) / np.linalg.norm(om ** 2 * e)
            assert res <= 1e-12, (axis, mb, mg, res)
            # and the frequency is in A's spectrum (+-i omega)
            j = np.searchsorted(spec, om)
            near = min(abs(spec[max(j - 1, 0)] - om), abs(spec[min(j, len(spec) - 1)] - om))
            assert near <= 1e-12 * om


def test_nonuniform_spacing_spectrum_moves_with_dx():
    """Control: the x-varying modes DO depend on dx, so (a) is not vacuous."""
    rng = np.random.default_rng(3)
    g1, *_ = _grid_axis_nonuniform(0, rng)
    g2 = fit.Grid(g1.nx, g1.ny, g1.nz, dx=np.full(g1.nx, 1.0e-3), dy=g1.dy, dz=g1.dz, dt_frac=0.9)
    s1 = np.sort(np.abs(np.linalg.eigvals(dense.dense_A(g1)[0]).imag))
    s2 = np.sort(np.abs(np.linalg.eigvals(dense.dense_A(g2)[0]).imag))
    assert len(s1) == len(s2) and np.abs(s1 - s2).max() > 1e-3 * s1.max()


# ---------------------------------------------------------------------------------------
# (b) dielectric / magnetic slab: second-order convergence to the transcendental root
# ---------------------------------------------------------------------------------------
LX, LZ = 1.0, 1.0
D_IF = 0.375 * LZ           # interface plane z = 3/8 L_z (a grid plane for N = 8, 16, 32)


def _kcot(q, L):
    """k cot(k L) for k^2 = q (continued to imaginary k)."""
    if q > 0:
        k = math.sqrt(q)
        return k / math.tan(k * L)
    if q < 0:
        k = math.sqrt(-q)
        return k / math.tanh(k * L)
    return 1.0 / L


def _exact_omega(eps1, eps2, mu1, mu2, guess):
    kx = math.pi / LX

    def F(om):
        q1 = om ** 2 * eps1 * mu1 / C_LIGHT ** 2 - kx ** 2
        q2 = om ** 2 * eps2 * mu2 / C_LIGHT ** 2 - kx ** 2
        return _kcot(q1, D_IF) / mu1 + _kcot(q2, LZ - D_IF) / mu2

    # the root near the discrete guess: a sign change of F without a pole in between
    grid = np.linspace(0.9 * guess, 1.1 * guess, 4001)
    vals = np.array([F(x) for x in grid])
    best = None
    for a, b, fa, fb in zip(grid[:-1], grid[1:], vals[:-1], vals[1:]):
        if fa * fb < 0 and abs(fa) + abs(fb) < 1e3 * (abs(vals).min() + 1.0):
            r = brentq(F, a, b, xtol=1e-14 * guess, rtol=1e-15)
            if abs(F(0.5 * (r + a))) < 1e6 and (best is None or abs(r - guess) < abs(best - guess)):
                best = r
    assert best is not None
    return best


def _slab_grid(N, eps1, eps2, mu1, mu2):
    nx, ny, nz = N, 1, N
    d = LZ / N
    kint = int(round(D_IF / d))
    cells_k = np.repeat(np.arange(nz), nx * ny)            # x fastest, then y, then z
    eps = np.where(cells_k < kint, eps1, eps2).astype(float)
    mu = np.where(cells_k < kint, mu1, mu2).astype(float)
    return fit.Grid(nx, ny, nz, dx=np.full(nx, LX / nx), dy=np.full(ny, d), dz=np.full(nz, d),
                    eps_r=eps, mu_r=mu, dt_frac=0.9), kint


def _lowest_ey_omega(g, Meps):
    """Lowest eigenfrequency of C^T M_nu C x = omega^2 M_eps x on the live e_y DOFs (an
    invariant subspace for n_y = 1), assembled column by column through the oracle's curls."""
    Np = g.Np
    live = np.flatnonzero(g.live_e[Np:2 * Np]) + Np
    Mnu = np.where(g.live_h, g.Mnu, 0.0)
    K = np.empty((len(live), len(live)))
    for col, dof in enumerate(live):
        e = np.zeros(3 * Np)
        e[dof] = 1.0
        y = g.curlT(Mnu * g.curl(e))
        other = g.live_e.copy()
        other[live] = False
        assert not other.any() or np.abs(y[other]).max() <= 1e-12 * np.abs(y).max()
        K[:, col] = y[live]
    w = eigh(K, np.diag(Meps[live]), eigvals_only=True, subset_by_index=[0, 0])
    return math.sqrt(w[0])


def _errors(eps1, eps2, mu1, mu2, wrong=False):
    Ns = (8, 16, 32)
    oms = []
    for N in Ns:
        g, kint = _slab_grid(N, eps1, eps2, mu1, mu2)
        Meps = g.Meps.copy()
        if wrong:
            # deliberately mis-averaged: interface y-edges take only the upper cell's eps
            Np = g.Np
            d = LZ / N
            idx = np.indices((g.nz + 1, g.ny + 1, g.nx + 1)).reshape(3, -1)[::-1]
            on_if = (idx[2] == kint)
            Meps[Np:2 * Np][on_if] = fit.EPS0 * eps2 * (LX / N) * d / d
        oms.append(_lowest_ey_omega(g, np.where(g.live_e, Meps, 1.0)))
    ex = _exact_omega(eps1, eps2, mu1, mu2, oms[-1])
    err = [abs(o - ex) / ex for o in oms]
    return err, ex


@pytest.mark.parametrize("eps1,eps2,mu1,mu2", [(1.0, 4.4, 1.0, 1.0), (9.8, 2.2, 1.0, 1.0),
                                               (1.0, 1.0, 1.0, 3.0)])
def test_slab_cavity_second_order(eps1, eps2, mu1, mu2):
    err, ex = _errors(eps1, eps2, mu1, mu2)
    r1, r2 = err[0] / err[1], err[1] / err[2]
    assert 3.7 < r1 < 4.3 and 3.8 < r2 < 4.2, (err, r1, r2)
    assert err[-1] < 5e-3


def test_slab_cavity_wrong_average_is_first_order():
    """The pin discriminates: taking one cell's eps at the interface edges degrades the
    convergence to first order (ratio ~2)."""
    err, _ = _errors(1.0, 4.4, 1.0, 1.0, wrong=True)
    assert err[1] / err[2] < 2.6, err
