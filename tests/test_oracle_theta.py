"""Pins of the planner's theta_m (reading 16: theta_m = the largest theta with
max_{x in [0, theta]} |p(ix) - e^{ix}| <= eps_A * theta, the error sampled on 801 points, found by
40 bisections on [0, 2m + 4]; PAPER:436-448 give no table) against computations that share
nothing with the oracle's plan machinery (make_plan, the mpmath divided-difference table, the
Newton evaluation, poly_error):

* Taylor (the c -> 0 case): p is the truncated exponential series, so the error
  is the series tail |e^{ix} - sum_{k<=m} (ix)^k / k!|, evaluated here at 40 digits in mpmath
  (monotone in x on [0, theta], so the sampled max is the value at theta), and theta_m is the
  root of tail(theta) = eps_A theta; to leading order ((m+1)! eps_A)^(1/m).
* Leja: the interpolant at the node set of reading 29 (i a xi_k, a = 1.05 theta, xi the greedy
  Leja prefix -- itself pinned by brute force in test_oracle_expmv.py) is unique, so it is
  evaluated here in the barycentric Lagrange form (numpy, double), not the Newton form; same
  801-point criterion, same bisection.
The oracle evaluates the error in double (|p - e^{ix}| ~ eps_A theta next to values ~1: a relative
rounding of ~1e-16 / (eps_A theta) in the error, 1/m of that in theta), hence 1e-6 here; a wrong
divided difference, node order, capacity scaling, interval margin or criterion moves theta_m by
percents."""
import math

import numpy as np
import pytest

from oracle import fit


def _bisect(ok, m):
    lo, hi = 0.0, float(2 * m + 4)
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        if mid > 0 and ok(mid):
            lo = mid
        else:
            hi = mid
    return lo


def _taylor_tail(m, x):
    import mpmath as mp
    with mp.workdps(40):
        z = mp.mpc(0, x)
        part = mp.fsum(z ** k / mp.factorial(k) for k in range(m + 1))
        return float(abs(mp.exp(z) - part))


@pytest.mark.parametrize("m,tol", [(8, 1e-10), (16, 1e-10), (32, 1e-10), (12, 1e-6)])
def test_taylor_theta_is_the_series_tail_root(m, tol):
    xs = np.linspace(0.0, 1.0, 9)
    th = _bisect(lambda t: _taylor_tail(m, t) <= tol * t, m)
    # the tail grows monotonically on [0, theta], so the 801-point max is the value at theta
    vals = [_taylor_tail(m, th * u) for u in xs]
    assert all(b >= a for a, b in zip(vals, vals[1:]))
    assert abs(fit.theta_m("taylor", m, tol) - th) <= 1e-6 * th
    lead = (math.factorial(m + 1) * tol) ** (1.0 / m)             # leading-order closed form
    assert abs(th / lead - 1) < 0.5 * th / (m + 2) + 1e-3


def _leja_error(m, theta, npts=801):
    xi = np.array(fit.leja_points(m + 1), dtype=np.float64)           # the node set (reading 29)
    a = 1.05 * theta
    f = np.exp(1j * a * xi)
    diff = xi[:, None] - xi[None, :]
    np.fill_diagonal(diff, 1.0)
    w = 1.0 / np.prod(diff, axis=1)                                   # barycentric weights
    x = np.linspace(0.0, theta, npts)
    t = x / a
    d = t[:, None] - xi[None, :]
    hit = np.isclose(d, 0.0, atol=0.0, rtol=0.0)
    d[hit] = 1.0
    p = (w * f / d).sum(axis=1) / (w / d).sum(axis=1)
    rows, cols = np.nonzero(hit)
    p[rows] = f[cols]
    return float(np.abs(p - np.exp(1j * x)).max())


@pytest.mark.parametrize("m,tol", [(8, 1e-10), (32, 1e-10), (64, 1e-10), (150, 1e-10), (16, 1e-6)])
def test_leja_theta_from_barycentric_interpolant(m, tol):
    th = _bisect(lambda t: _leja_error(m, t) <= tol * t, m)
    assert abs(fit.theta_m("leja", m, tol) - th) <= 1e-6 * th
    # the efficiency the planner relies on (reading 16): theta_m / m grows with m at 1e-10
    if tol == 1e-10 and m >= 64:
        assert th / m > fit.theta_m("leja", 32, tol) / 32
