"""Pins for the non-uniform-mesh study: the oracle's
||A||_2 (ARPACK on -A^2 through the oracle stencil), the paper's 2-D wave DOF counts, and the
R(k) = C_Leja / C_LF trend of Fig. 6 (ParaExp's exponential gains on meshes with one small
element because eq:cfl is pessimistic while ||A||_2 grows slowly)."""
import math

import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from oracle import dense, fit
from synth import config_wave2d


def test_norm_A_closed_form_and_dense():
    g = fit.Grid(8, 8, 8, d0=1e-3, dt_frac=0.9)
    assert abs(fit.norm_A(g) / g.rho_cfl - math.sin(7 * math.pi / 16)) < 1e-10   # finding 7
    g2 = fit.Grid(4, 3, 3, d0=1e-3, dx=[1e-3, 0.3e-3, 1e-3, 2e-3], dt_frac=0.9,
                  eps_r=np.random.default_rng(4).uniform(1, 4, 36))
    A, *_ = dense.dense_A(g2)
    assert abs(fit.norm_A(g2) - np.abs(np.linalg.eigvals(A)).max()) < 1e-9 * fit.norm_A(g2)


def test_wave2d_dofs():
    """n_dof = 20172 (41x41x2) and 175692 (121x121x2), e and h together."""
    for n, dof in ((41, 20172), (121, 175692)):
        g = fit.Grid.from_workload(config_wave2d(n))
        assert 6 * g.Np == dof


def _R(k, eps_A=1e-2):
    w = config_wave2d(41, k)
    g = fit.Grid.from_workload(w)
    nt = math.ceil(w.t_end / g.dt)
    c_lf = 2 * nt                                        # eq:cost_LF
    rho = 1.05 * fit.norm_A(g)
    plan = pe.plan_host("leja", 0, 0, eps_A, w.t_end, rho, g.dt)
    return plan["m"] * plan["s"] / c_lf


def test_rk_decreases_with_k():
    """Fig. 6: R(k) decreases as the smallest element shrinks (k = max/min element size)."""
    ks = (1, 2, 5, 10, 20)
    R = [_R(k) for k in ks]
    assert all(a > b for a, b in zip(R[:-1], R[1:])), R
    assert R[-1] < 0.5 * R[0]
