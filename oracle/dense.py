"""Dense reference objects for tiny grids (<= 4^3 cells) -- TEST INFRASTRUCTURE ONLY.

Independent of the C stencil formulas: the curl incidence is enumerated from the
geometry of each face (boundary loop oriented by the right-hand rule), divergences
from edge/face endpoints.  Used to pin the oracle's C loops and the exponential
(numpy eigh of the Hermitian i*A, PAPER:217-219 'all eigenvalues are imaginary').
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def _P(n, i, j, k):
    nx, ny, nz = n
    return i + (nx + 1) * (j + (ny + 1) * k)


def incidence_curl(nx, ny, nz):
    """C (faces x edges) in the canonical layout: face (normal axis c, corner point P)
    spanned by axes a = c+1, b = c+2 (cyclic).  Its boundary, counter-clockwise seen from
    +c:  (P, a, +1), (P+e_a, b, +1), (P+e_b, a, -1), (P, b, -1).  Edges leaving the point
    lattice (virtual) are dropped."""
    n = (nx, ny, nz)
    Np = (nx + 1) * (ny + 1) * (nz + 1)
    C = np.zeros((3 * Np, 3 * Np), dtype=np.int64)
    unit = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
    for c in range(3):
        a, b = (c + 1) % 3, (c + 2) % 3
        for k, j, i in itertools.product(range(nz + 1), range(ny + 1), range(nx + 1)):
            P = (i, j, k)
            row = c * Np + _P(n, *P)
            loop = [(P, a, +1),
                    (tuple(P[d] + unit[a][d] for d in range(3)), b, +1),
                    (tuple(P[d] + unit[b][d] for d in range(3)), a, -1),
                    (P, b, -1)]
            for (Q, ax, sgn) in loop:
                if any(Q[d] < 0 or Q[d] > n[d] for d in range(3)):
                    continue
                if Q[ax] + 1 > n[ax]:          # edge would leave the lattice: virtual
                    continue
                C[row, ax * Np + _P(n, *Q)] += sgn
    return C


def divergence_primal(nx, ny, nz):
    """S (points x edges): +1 for an edge leaving the point, -1 for an edge arriving."""
    n = (nx, ny, nz)
    Np = (nx + 1) * (ny + 1) * (nz + 1)
    S = np.zeros((Np, 3 * Np), dtype=np.int64)
    for a in range(3):
        for k, j, i in itertools.product(range(nz + 1), range(ny + 1), range(nx + 1)):
            P = (i, j, k)
            if P[a] + 1 > n[a]:
                continue
            Q = list(P)
            Q[a] += 1
            col = a * Np + _P(n, *P)
            S[_P(n, *P), col] += 1
            S[_P(n, *Q), col] -= 1
    return S


def divergence_dual(nx, ny, nz):
    """S-tilde (cells x faces): outward normal sign of the 6 faces of each cell."""
    n = (nx, ny, nz)
    Np = (nx + 1) * (ny + 1) * (nz + 1)
    cells = nx * ny * nz
    St = np.zeros((cells, 3 * Np), dtype=np.int64)
    for k, j, i in itertools.product(range(nz), range(ny), range(nx)):
        cell = i + nx * (j + ny * k)
        for c in range(3):
            P = [i, j, k]
            St[cell, c * Np + _P(n, *P)] -= 1
            P[c] += 1
            St[cell, c * Np + _P(n, *P)] += 1
    return St


def dense_A(g):
    """Skew A = T A_orig T^-1 on the live DOFs.  Returns (A, idx_e, idx_h,
    Tdiag) with the state ordered [h_live; e_live]."""
    C = incidence_curl(g.nx, g.ny, g.nz).astype(float)
    ie = np.flatnonzero(g.live_e)
    ih = np.flatnonzero(g.live_h)
    Ceh = C[np.ix_(ih, ie)]                  # faces(live) x edges(live)
    Mnu = g.Mnu[ih]
    Meps = g.Meps[ie]
    nh, ne = len(ih), len(ie)
    Aorig = np.zeros((nh + ne, nh + ne))
    Aorig[:nh, nh:] = -(Mnu[:, None] * Ceh)
    Aorig[nh:, :nh] = (1.0 / Meps)[:, None] * Ceh.T
    T = np.concatenate([np.sqrt(1.0 / Mnu), np.sqrt(Meps)])
    A = (T[:, None] * Aorig) / T[None, :]
    return A, ie, ih, T


def expm_dense_apply(A, T, t, v):
    """exp(t A_orig) v via the eigendecomposition of the Hermitian matrix iA (A skew)."""
    H = 1j * A
    w, V = np.linalg.eigh(H)
    u = T * v
    # exp(tA) = exp(-i t H)
    y = V @ (np.exp(-1j * t * w) * (V.conj().T @ u))
    return (y / T).real


def cavity_frequencies(nx, ny, nz, d, c):
    """Closed-form angular frequencies of the FIT PEC cavity on a uniform grid (SURVEY
    finding 7): omega = (2c/d) sqrt(sum_d sin^2(m_d pi / (2 N_d))), 0 <= m_d <= N_d - 1,
    at most one m_d = 0; multiplicity 2 if all m_d >= 1 (two polarisations) else 1."""
    out = []
    for mx in range(nx):
        for my in range(ny):
            for mz in range(nz):
                zeros = (mx == 0) + (my == 0) + (mz == 0)
                if zeros > 1:
                    continue
                s = (math.sin(mx * math.pi / (2 * nx)) ** 2 + math.sin(my * math.pi / (2 * ny)) ** 2
                     + math.sin(mz * math.pi / (2 * nz)) ** 2)
                w = 2.0 * c / d * math.sqrt(s)
                out += [w] * (2 if zeros == 0 else 1)
    return np.sort(np.array(out))
