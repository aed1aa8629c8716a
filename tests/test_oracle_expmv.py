"""Pins of the oracle's exp(tA)v: dense eigendecomposition, closed forms,
interpolation identities, brute-force Leja property, Taylor degeneracy."""
import math

import numpy as np
import pytest

from oracle import dense, fit
from synth import random_fields


def _state(g, seed):
    e, h = random_fields(g.nx, g.ny, g.nz, seed)
    return g.clean(e, h)


def test_leja_points_greedy_bruteforce():
    """Each eta_l maximises prod |z - xi_j| over the 10^4-point symmetric candidate set
    {+-k/5000} among points not yet chosen (reading 14)."""
    xs = fit.leja_points(41)
    assert xs[:3] == (1.0, -1.0, 0.0)
    cand = np.concatenate([np.arange(1, 5001), -np.arange(1, 5001)]) / 5000.0
    for l in range(3, 41, 2):
        prev = np.array(xs[:l])
        with np.errstate(divide="ignore"):
            obj = np.sum(np.log(np.abs(cand[:, None] - prev[None, :])), axis=1)
        best = obj.max()
        k = int(round(abs(xs[l]) * 5000))
        assert xs[l] == k / 5000.0 and xs[l + 1] == -xs[l]
        # the chosen +eta attains the maximum (within fp64 rounding of the log sums)
        assert obj[k - 1] >= best - 1e-12 * abs(best)


def test_divided_differences_closed_forms():
    gamma = 3.7
    # coincident nodes at 0: g[0,...,0] = gamma^k / k!  (Taylor)
    d = fit.divided_differences([0j] * 8, gamma)
    assert all(abs(d[k] - gamma ** k / math.factorial(k)) < 1e-15 * gamma ** k for k in range(8))
    # two nodes: (g(z1) - g(z0)) / (z1 - z0)
    z = [0.3j, -1.1j]
    d = fit.divided_differences(z, gamma)
    ref = (np.exp(gamma * z[1]) - np.exp(gamma * z[0])) / (z[1] - z[0])
    assert abs(d[1] - ref) < 1e-15


def test_newton_interpolates_at_nodes_and_precision_stable():
    plan = fit.make_plan("leja", 40, 1, 30.0, 1.0)
    for k, z in enumerate(plan.nodes):
        val = fit.newton_eval_scalar(plan, z)
        assert abs(val - np.exp(plan.gamma * z)) < 1e-11
    d100 = fit.divided_differences(plan.nodes, plan.gamma, dps=100)
    assert max(abs(a - b) for a, b in zip(plan.d, d100)) < 1e-15


def test_rotation_2x2():
    """2-DOF rotation block [[0,-w],[w,0]], w t = pi/2, b = (1,0) -> (0,1)."""
    w = 2.0
    t = math.pi / 4
    plan = fit.make_plan("leja", 30, 1, t, w)
    # eigenvalues +-i w: p(X) on X = (h/gamma)(+-i w)
    lam_p = fit.newton_eval_scalar(plan, 1j * w * t / plan.gamma)
    lam_m = fit.newton_eval_scalar(plan, -1j * w * t / plan.gamma)
    # b = (1,0) = (v+ + v-)/2 with v+- = (1, -+i)
    y = 0.5 * (lam_p * np.array([1, -1j]) + lam_m * np.array([1, 1j]))
    assert np.allclose(y, [0, 1], atol=1e-14)


@pytest.mark.parametrize("method,tol", [("leja", 1e-8), ("taylor", 1e-8), ("leja", 1e-4)])
def test_random_skew_50_vs_dense(method, tol):
    """Random 50x50 skew: polynomial action vs dense eigendecomposition <= 100 eps_A,
    norm preserved within 10 eps_A."""
    rng = np.random.default_rng(4)
    for trial in range(5):
        B = rng.standard_normal((50, 50))
        A = B - B.T
        rho = np.abs(np.linalg.eigvals(A)).max()
        t = 1.3
        m = 32
        th = fit.theta_m(method, m, tol)
        s = max(1, math.ceil(t * rho / th))
        plan = fit.make_plan(method, m, s, t, rho)
        v = rng.standard_normal(50)
        # generic complex Newton with a matrix (same recurrence as the stencil version)
        X = A * (t / s) / plan.gamma
        b = v.astype(complex)
        for _ in range(s):
            w = b.copy()
            y = plan.d[0] * w
            for k in range(1, m + 1):
                w = X @ w - plan.nodes[k - 1] * w
                y = y + plan.d[k] * w
            b = y.real.astype(complex)
        lam, V = np.linalg.eigh(1j * A)
        ref = (V @ (np.exp(-1j * t * lam) * (V.conj().T @ v))).real
        assert np.linalg.norm(b.real - ref) / np.linalg.norm(ref) <= 100 * tol
        assert abs(np.linalg.norm(b.real) / np.linalg.norm(v) - 1) <= 10 * tol


def _tight_plan(method, tau, rho, m=40, tol=1e-14):
    th = fit.theta_m(method, m, tol)
    s = max(1, math.ceil(tau * rho / th))
    return fit.make_plan(method, m, s, tau, rho)


@pytest.mark.parametrize("n,eps_seed", [((3, 3, 2), None), ((4, 3, 3), 9), ((4, 4, 4), None)])
def test_stencil_expmv_vs_dense_eig(n, eps_seed):
    """exp(tau A_orig) v through the C stencil == dense eigh exponential (<= 4^3 cells)."""
    eps = None if eps_seed is None else np.random.default_rng(eps_seed).uniform(1, 4, np.prod(n))
    g = fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.9)
    A, ie, ih, T = dense.dense_A(g)
    rho = np.abs(np.linalg.eigvals(A)).max()
    e, h = _state(g, 21)
    tau = 37.3 * g.dt
    for method in ["leja", "taylor"]:
        plan = _tight_plan(method, tau, rho)
        ye, yh = fit.expmv(g, plan, e, h, mode="complex")
        u = np.concatenate([h[ih], e[ie]])
        ref = dense.expm_dense_apply(A, T, tau, u)
        nh = len(ih)
        assert np.linalg.norm(ye[ie] - ref[nh:]) / np.linalg.norm(ref[nh:]) < 1e-12
        assert np.linalg.norm(yh[ih] - ref[:nh]) / np.linalg.norm(ref[:nh]) < 1e-12
        # dead entries stay exactly zero
        assert not ye[~g.live_e].any() and not yh[~g.live_h].any()


def test_pairs_equal_complex_newton():
    """Real conjugate-pair recurrence == plain complex Newton form (fp64, 1e-13)."""
    g = fit.Grid(5, 4, 4, d0=1e-3, eps_r=np.random.default_rng(2).uniform(1, 4, 80), dt_frac=0.95)
    e, h = _state(g, 8)
    for method, m in [("leja", 1), ("leja", 2), ("leja", 4), ("leja", 30), ("taylor", 18)]:
        plan = fit.make_plan(method, m, 3, 20 * g.dt, g.rho_cfl)
        a_e, a_h = fit.expmv(g, plan, e, h, mode="complex")
        b_e, b_h = fit.expmv(g, plan, e, h, mode="pairs", dtype="f64")
        assert np.linalg.norm(a_e - b_e) <= 1e-13 * np.linalg.norm(a_e)
        assert np.linalg.norm(a_h - b_h) <= 1e-13 * np.linalg.norm(a_h)


def test_leja_reduces_to_taylor_as_c_to_0():
    """L_{m,c} -> Taylor for c -> 0: 1e-13."""
    g = fit.Grid(4, 4, 3, d0=1e-3, dt_frac=0.9)
    e, h = _state(g, 3)
    tau = 0.3 * g.dt
    # Leja nodes on i[-c, c] with c -> 0, written unscaled (gamma = 1, X = tau A)
    c = 1e-9
    nodes = [1j * c * x for x in fit.leja_points(17)]
    lj = fit.Plan("leja", 16, 1, tau, g.rho_cfl, c, 1.0, nodes,
                  fit.divided_differences(nodes, 1.0, dps=300))
    ty = fit.make_plan("taylor", 16, 1, tau, g.rho_cfl)
    a = fit.expmv(g, lj, e, h, mode="complex")
    b = fit.expmv(g, ty, e, h, mode="complex")
    for x, y in zip(a, b):
        assert np.linalg.norm(x - y) <= 1e-13 * np.linalg.norm(y)


def test_identity_group_norm():
    g = fit.Grid(6, 5, 4, d0=1e-3, dt_frac=0.9)
    e, h = _state(g, 12)
    rho = g.rho_cfl
    # t = 0 -> identity
    z = fit.expmv(g, fit.make_plan("leja", 8, 1, 0.0, rho), e, h)
    assert np.array_equal(z[0], e) and np.array_equal(z[1], h)
    t1, t2 = 11.5 * g.dt, 23.25 * g.dt
    x = fit.expmv(g, _tight_plan("leja", t1, rho), e, h)
    x = fit.expmv(g, _tight_plan("leja", t2, rho), *x)
    y = fit.expmv(g, _tight_plan("leja", t1 + t2, rho), e, h)
    for a, b in zip(x, y):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    n0 = g.energy_norm2(e, h)
    assert abs(g.energy_norm2(*y) / n0 - 1) < 1e-12


def test_leja_vs_taylor_factor_two():
    """Leja needs about half the SMVPs of Taylor at equal tolerance (PAPER:653-654 'factor
    of 2', qualitative): best m/theta_m over the degree candidates, tol 1e-8, ratio in
    [1.5, 3.5] (SURVEY finding 5)."""
    tol = 1e-8
    bt = min(m / fit.theta_m("taylor", m, tol) for m in [16, 24, 32, 48])
    bl = min(m / fit.theta_m("leja", m, tol) for m in [32, 64, 100])
    assert 1.5 < bt / bl < 3.5, (bt, bl)


def test_fp32_constant_recipe_close_to_fp64():
    """fp32-rounded constants (reading 24) change the result only at fp32 level."""
    g = fit.Grid(5, 4, 4, d0=1e-3, dt_frac=0.95)
    g32 = fit.Grid(5, 4, 4, d0=1e-3, dt_frac=0.95, dtype="f32")
    e, h = _state(g, 8)
    plan = fit.make_plan("leja", 30, 2, 25 * g.dt, g.rho_cfl)
    a = fit.expmv(g, plan, e, h, dtype="f64")
    b = fit.expmv(g32, plan, e, h, dtype="f32")
    for x, y in zip(a, b):
        r = np.linalg.norm(x - y) / np.linalg.norm(x)
        assert 1e-10 < r < 1e-5


def test_early_termination_oracle():
    """f2 (reading 18): with a degree much larger than the substep needs, the
    early-terminated Newton sum stops after fewer A-applications and stays within ~eps of the
    full sum (and of the dense exponential)."""
    n = (4, 4, 3)
    g = fit.Grid(*n, d0=1e-3, eps_r=np.random.default_rng(5).uniform(1, 4, 48), dt_frac=0.9)
    e, h = _state(g, 3)
    tau = 1.0 * g.dt
    rho = g.rho_cfl
    plan = fit.make_plan("leja", 60, 2, tau, rho)
    fe, fh = fit.expmv(g, plan, e, h)
    for eps in (1e-6, 1e-10):
        te, th, apps = fit.expmv_pairs_et(g, plan, e, h, eps)
        assert apps < 60 * 2
        full = np.concatenate([fe, fh])
        err = np.linalg.norm(np.concatenate([te, th]) - full) / np.linalg.norm(full)
        assert err <= 10 * eps
    # eps tiny: no early stop possible before the end -> identical to the plain sum
    te, th, apps = fit.expmv_pairs_et(g, fit.make_plan("leja", 8, 3, 10 * g.dt, rho), e, h, 1e-15)
    pe_, ph_ = fit.expmv(g, fit.make_plan("leja", 8, 3, 10 * g.dt, rho), e, h)
    assert apps == 24 and np.array_equal(te, pe_) and np.array_equal(th, ph_)


@pytest.mark.parametrize("method,m,s", [("leja", 40, 3), ("leja", 1, 5), ("leja", 2, 4), ("leja", 64, 1),
                                         ("taylor", 16, 6), ("leja", 6, 2)])
def test_horner_equals_forward_and_complex(method, m, s):
    """Reading 33: the nested (Horner) evaluation of the real pair-block polynomial equals the
    forward pair recurrence and the plain complex Newton form (fp64, 1e-12)."""
    g = fit.Grid(5, 4, 4, d0=1e-3, eps_r=np.random.default_rng(2).uniform(1, 4, 80), dt_frac=0.95)
    e, h = _state(g, 8)
    tau = (30 if method == "leja" else 6) * g.dt
    plan = fit.make_plan(method, m, s, tau, g.rho_cfl)
    he, hh = fit.expmv(g, plan, e, h, mode="horner")
    fe, fh = fit.expmv(g, plan, e, h, mode="pairs")
    ce, ch = fit.expmv(g, plan, e, h, mode="complex")
    ref = np.concatenate([ce, ch])
    for got in (np.concatenate([he, hh]), np.concatenate([fe, fh])):
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("method,m,s", [("leja", 16, 3), ("leja", 1, 2), ("taylor", 12, 2), ("leja", 40, 1)])
def test_pairs_c_loops_equal_numpy(dtype, method, m, s):
    """The C loops of or_expmv_pairs run expmv_pairs_numpy's recurrence step for step: the
    same fields (no contraction in the oracle build, so bit-equal up to OpenMP-free order)."""
    n = (7, 5, 6)
    g = fit.Grid(*n, d0=1e-3, eps_r=np.random.default_rng(2).uniform(1, 4, 210), dt_frac=0.9,
                 dtype=dtype)
    e, h = g.clean(*random_fields(*n, seed=4))
    plan = fit.make_plan(method, m, s, 12 * g.dt, g.rho_cfl)
    a = fit.expmv_pairs_numpy(g, plan, e, h, dtype)
    b = fit.expmv_pairs(g, plan, e, h, dtype)
    for x, y in zip(a, b):
        assert np.abs(x - y).max() <= 1e-15 * np.abs(x).max()
