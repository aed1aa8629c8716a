"""Pins of the oracle's Krylov exp(tA)v (Arnoldi, sigma = infinity; SURVEY 8(f)
f3): exactness on a full / invariant Krylov space against the dense eigendecomposition,
energy-norm preservation and convergence in l.  (The paper's "factor 10" against Leja,
PAPER:653-654, is a run-time comparison on its workloads, not an SMVP identity: not pinned.)"""
import math

import numpy as np
import pytest

from oracle import dense, fit
from synth import random_fields


def _grid(n, eps_seed=None):
    eps = None if eps_seed is None else np.random.default_rng(eps_seed).uniform(1, 4, int(np.prod(n)))
    return fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.9)


def _dense_ref(g, tau, e, h):
    A, ie, ih, T = dense.dense_A(g)
    u = np.concatenate([h[ih], e[ie]])
    ref = dense.expm_dense_apply(A, T, tau, u)
    nh = len(ih)
    re, rh = np.zeros_like(e), np.zeros_like(h)
    re[ie], rh[ih] = ref[nh:], ref[:nh]
    return re, rh, len(u)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,eps_seed", [((2, 2, 1), None), ((2, 2, 2), 4)])
def test_full_space_is_exact(n, eps_seed):
    """l >= dim: the Krylov space is the whole (invariant) space -> the exact exponential."""
    g = _grid(n, eps_seed)
    e, h = g.clean(*random_fields(*n, seed=3))
    tau = 13.7 * g.dt
    re, rh, dim = _dense_ref(g, tau, e, h)
    assert dim <= 100
    ke, kh, apps = fit.expmv_krylov(g, 100, 1, tau, e, h)
    assert apps <= dim                      # happy breakdown at the invariant subspace
    assert _rel(ke, re) < 1e-10 and _rel(kh, rh) < 1e-10


def test_invariant_two_dim_subspace():
    """b in the real span of one eigenpair +-i omega: l = 2 is exact (a rotation)."""
    g = _grid((3, 2, 2))
    A, ie, ih, T = dense.dense_A(g)
    w, V = np.linalg.eigh(1j * A)
    k = int(np.argmax(w))
    v = V[:, k].real * 1.0                  # Re of an eigenvector of the skew A
    u = v / T                               # back to original variables
    nh = len(ih)
    e, h = np.zeros(3 * g.Np), np.zeros(3 * g.Np)
    e[ie], h[ih] = u[nh:], u[:nh]
    tau = 2.1 * g.dt
    re, rh, _ = _dense_ref(g, tau, e, h)
    ke, kh, apps = fit.expmv_krylov(g, 2, 1, tau, e, h)
    assert _rel(np.concatenate([ke, kh]), np.concatenate([re, rh])) < 1e-12


def test_energy_norm_preserved_and_convergence():
    """V orthonormal and exp(H) orthogonal (H skew): the energy norm is preserved for any l;
    the error falls fast with l (super-linear Krylov convergence)."""
    n = (4, 4, 3)
    g = _grid(n, 7)
    e, h = g.clean(*random_fields(*n, seed=5))
    tau = 12.0 * g.dt
    E0 = g.energy_norm2(e, h)
    re, rh, _ = _dense_ref(g, tau, e, h)
    errs = []
    for l in (10, 20, 30):
        ke, kh, _ = fit.expmv_krylov(g, l, 1, tau, e, h)
        assert abs(g.energy_norm2(ke, kh) - E0) <= 1e-12 * E0
        errs.append(_rel(np.concatenate([ke, kh]), np.concatenate([re, rh])))
    assert errs[1] < 0.1 * errs[0] and errs[2] < 0.1 * errs[1]
