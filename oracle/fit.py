"""Oracle: FIT grid, leapfrog, exp(tA)v and ParaExp -- plain CPU definitions.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Heavy loops run in the plain C
file ``fit_oracle.c`` (compiled with gcc -O2 -fopenmp, no intrinsics); everything
else is numpy / mpmath written in the paper's order and notation.

Citations: PAPER:n = line n of the paper text; SURVEY/DESIGN readings are numbered
as in DESIGN.md "Readings of the paper".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from functools import lru_cache
from typing import List, Optional, Sequence

import numpy as np

# Own copies of the physical constants (CODATA 2018).
EPS0 = 8.8541878128e-12
MU0 = 1.25663706212e-6

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_fit_oracle.so")
_SRC = os.path.join(_HERE, "fit_oracle.c")


def build(force: bool = False) -> str:
    """Compile the plain C oracle (gcc -O2 -fopenmp; default FP contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        # ORACLE_SO: an alternative build of the same C file (tools/asan_host.sh: ASan/UBSan)
        _lib = ctypes.CDLL(os.environ.get("ORACLE_SO") or build())
        dp = ctypes.POINTER(ctypes.c_double)
        up = ctypes.POINTER(ctypes.c_ubyte)
        lp = ctypes.POINTER(ctypes.c_long)
        i = ctypes.c_int
        _lib.or_fit_matrices.argtypes = [i, i, i, dp, dp, dp, dp, dp, up, ctypes.c_double,
                                         ctypes.c_double, dp, dp, up, up]
        _lib.or_curl.argtypes = [i, i, i, dp, dp]
        _lib.or_curlT.argtypes = [i, i, i, dp, dp]
        _lib.or_leapfrog.argtypes = [i, i, i, dp, dp, ctypes.c_long, i, lp, dp, dp, dp]
        _lib.or_apply_A.argtypes = [i, i, i, dp, dp, dp, dp, dp, dp]
        ip = ctypes.POINTER(ctypes.c_int)
        _lib.or_expmv_pairs.argtypes = [i, i, i, dp, dp, i, ip, dp, dp, dp, dp, i, dp, dp]
        _lib.or_expmv_pairs.restype = ctypes.c_int
        _lib.or_num_threads.restype = ctypes.c_int
        _lib.or_set_threads.argtypes = [i]
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _up(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte))


def num_threads() -> int:
    return lib().or_num_threads()


def set_threads(n: int) -> None:
    """OpenMP thread count of the C loops (timing only; results do not depend on it)."""
    lib().or_set_threads(int(n))


def _round(x, dtype):
    """Round fp64 values once to the run dtype, returned as fp64 (DESIGN reading 24)."""
    if dtype == "f32":
        return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
    return np.asarray(x, dtype=np.float64)


# eq:cfl: min over cells of sqrt(eps mu / (dx^-2 + dy^-2 + dz^-2))
def cfl_dt(nx, ny, nz, dx, dy, dz, eps_r=None, mu_r=None):
    """dt_CFL of a grid; dx/dy/dz per-cell spacing arrays, eps_r/mu_r per cell (None = 1).
    Needs no FIT matrices, so it also serves grids too large to assemble here."""
    dx, dy, dz = (np.asarray(a, float) for a in (dx, dy, dz))
    best = math.inf
    eps = None if eps_r is None else np.asarray(eps_r, float).reshape(nz, ny, nx)
    mu = None if mu_r is None else np.asarray(mu_r, float).reshape(nz, ny, nx)
    for k in range(nz):                      # one z-layer of cells (ny x nx) at a time
        inv = 1.0 / dx[None, :] ** 2 + 1.0 / dy[:, None] ** 2 + 1.0 / dz[k] ** 2
        er = 1.0 if eps is None else eps[k]
        mr = 1.0 if mu is None else mu[k]
        v = np.sqrt(EPS0 * er * MU0 * mr / inv)
        best = min(best, float(np.min(v)))
    return best


# ---------------------------------------------------------------------------
# Grid
# ---------------------------------------------------------------------------
class Grid:
    """FIT grid with fp64 material matrices and the eq:cfl time step.

    cE = dt * M_eps^-1 on live edges (0 on PEC / virtual edges),
    cH = dt * M_nu on live faces (0 on boundary-normal / virtual faces).
    ``cE_T``/``cH_T`` are those values rounded once to the run dtype.
    """

    def __init__(self, nx, ny, nz, d0=None, dx=None, dy=None, dz=None, eps_r=None, mu_r=None,
                 pec_cell=None, dt=None, dt_frac=None, dtype="f64"):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.dtype = dtype
        self.dx = np.full(nx, d0, float) if dx is None else np.asarray(dx, float).copy()
        self.dy = np.full(ny, d0, float) if dy is None else np.asarray(dy, float).copy()
        self.dz = np.full(nz, d0, float) if dz is None else np.asarray(dz, float).copy()
        ncell = nx * ny * nz
        self.eps_r = np.ones(ncell) if eps_r is None else np.asarray(eps_r, float).copy()
        self.mu_r = np.ones(ncell) if mu_r is None else np.asarray(mu_r, float).copy()
        self.pec = (np.zeros(ncell, np.uint8) if pec_cell is None
                    else np.ascontiguousarray(pec_cell, dtype=np.uint8))
        self.Np = (nx + 1) * (ny + 1) * (nz + 1)
        Np = self.Np
        self.Meps = np.zeros(3 * Np)
        self.Mnu = np.zeros(3 * Np)
        live_e = np.zeros(3 * Np, np.uint8)
        live_h = np.zeros(3 * Np, np.uint8)
        lib().or_fit_matrices(nx, ny, nz, _dp(self.dx), _dp(self.dy), _dp(self.dz),
                              _dp(self.eps_r), _dp(self.mu_r), _up(self.pec), EPS0, MU0,
                              _dp(self.Meps), _dp(self.Mnu), _up(live_e), _up(live_h))
        self.live_e = live_e.astype(bool)
        self.live_h = live_h.astype(bool)
        self.dt_cfl = self.cfl()
        if dt is None:
            dt = dt_frac * self.dt_cfl
        self.dt = float(dt)
        self.rho_cfl = 2.0 / self.dt_cfl            # SURVEY finding 7 / reading 17
        self.cE = np.where(self.live_e, self.dt / np.where(self.Meps > 0, self.Meps, 1.0), 0.0)
        self.cH = np.where(self.live_h, self.dt * self.Mnu, 0.0)
        self.cE_T = _round(self.cE, dtype)
        self.cH_T = _round(self.cH, dtype)

    @classmethod
    def from_workload(cls, w, dtype=None):
        return cls(w.nx, w.ny, w.nz, d0=w.d0, dx=getattr(w, "dx", None), dy=getattr(w, "dy", None),
                   dz=getattr(w, "dz", None), eps_r=w.eps_r, pec_cell=w.pec_cell,
                   dt_frac=w.dt_frac, dtype=dtype or w.dtype)

    def cfl(self):
        return cfl_dt(self.nx, self.ny, self.nz, self.dx, self.dy, self.dz, self.eps_r, self.mu_r)

    # --- vectors -----------------------------------------------------------
    def zeros(self):
        return np.zeros(3 * self.Np), np.zeros(3 * self.Np)

    def clean(self, e, h):
        """Zero PEC/virtual entries of input fields (DESIGN reading 5); round to dtype."""
        e = _round(np.where(self.live_e, e, 0.0), self.dtype)
        h = _round(np.where(self.live_h, h, 0.0), self.dtype)
        return e, h

    def curl(self, e):
        out = np.empty(3 * self.Np)
        lib().or_curl(self.nx, self.ny, self.nz, _dp(np.ascontiguousarray(e)), _dp(out))
        return out

    def curlT(self, h):
        out = np.empty(3 * self.Np)
        lib().or_curlT(self.nx, self.ny, self.nz, _dp(np.ascontiguousarray(h)), _dp(out))
        return out

    def edge_dof(self, comp, i, j, k):
        return comp * self.Np + i + (self.nx + 1) * (j + (self.ny + 1) * k)

    # --- energy -----------------------------------------------
    def M_eps_w(self):
        """M_eps on live edges (0 elsewhere) -- weights of the electric energy."""
        return np.where(self.live_e, self.Meps, 0.0)

    def M_mu_w(self):
        """M_mu = M_nu^-1 on live faces (0 elsewhere)."""
        return np.where(self.live_h, 1.0 / np.where(self.Mnu > 0, self.Mnu, 1.0), 0.0)

    def energy_norm2(self, e, h):
        """<h,h>_mu + <e,e>_eps."""
        return float(np.dot(e * self.M_eps_w(), e) + np.dot(h * self.M_mu_w(), h))


# ---------------------------------------------------------------------------
# Sources (PAPER:640-648 eq:line_current; reading 6)
# ---------------------------------------------------------------------------
def waveform(src, t):
    kind = src.kind
    if kind == "zero":
        return 0.0
    if kind == "gauss_paper":
        s = src.t_param
        return src.amp * math.exp(-4.0 * ((t - s) / s) ** 2)
    if kind == "gauss_sine":
        x = t - src.t_delay
        return src.amp * math.sin(2.0 * math.pi * src.f0 * x) * math.exp(-(x / src.t_param) ** 2)
    if kind == "sine":
        return src.amp * math.sin(2.0 * math.pi * src.f0 * t)
    raise ValueError(kind)


def source_table(g: Grid, sources, t0, m0, nsteps):
    """q[m][s] = fl_T( cE64_s * (weight_s * i_s(t0 + (m0+m+1/2) dt)) ), global step index
    (PAPER:232 '-j', PAPER:647 g = -[0,j]; readings 6, 24)."""
    ns = len(sources)
    q = np.zeros((max(nsteps, 0), ns))
    dofs = np.array([g.edge_dof(s.comp, s.i, s.j, s.k) for s in sources], dtype=np.int64)
    for si, s in enumerate(sources):
        c = g.cE[dofs[si]]
        for m in range(nsteps):
            t = t0 + (float(m0 + m) + 0.5) * g.dt
            q[m, si] = c * (s.weight * waveform(s, t))
    return _round(q, g.dtype), dofs


# ---------------------------------------------------------------------------
# Leapfrog (PAPER:227-234 with C on e: reading 1)
# ---------------------------------------------------------------------------
def leapfrog(g: Grid, e, h, nsteps, sources=(), t0=0.0, m0=0):
    """(e^(0), h^(1/2)) -> (e^(n), h^(n+1/2)) with the grid's dt; sources at global
    times t0 + (m0+m+1/2) dt.  Returns new arrays (fp64; fp32-rounded constants when the
    grid dtype is f32)."""
    e = np.array(e, dtype=np.float64, copy=True)
    h = np.array(h, dtype=np.float64, copy=True)
    sources = list(sources)
    q, dofs = source_table(g, sources, t0, m0, nsteps)
    if nsteps <= 0:
        return e, h
    q = np.ascontiguousarray(q)
    lib().or_leapfrog(g.nx, g.ny, g.nz, _dp(g.cE_T), _dp(g.cH_T), int(nsteps), len(sources),
                      dofs.ctypes.data_as(ctypes.POINTER(ctypes.c_long)),
                      _dp(q) if len(sources) else ctypes.POINTER(ctypes.c_double)(),
                      _dp(e), _dp(h))
    return e, h


def half_step_start(g: Grid, e0, h0):
    """h^(1/2) = h^0 - 1/2 cH (C e^0) for a same-time initial value (reading 11)."""
    return h0 - 0.5 * g.cH_T * g.curl(e0)


def sync_h(g: Grid, e, h):
    """h(T_j) = h^(M+1/2) + 1/2 cH (C e^(M))  ==  (h^(M-1/2) + h^(M+1/2))/2 (
    reading 9)."""
    return h + (0.5 * g.cH_T) * g.curl(e)


def energy_staggered(g: Grid, e_m, h_mmh, h_mph):
    """E_m = e^m' M_eps e^m + h^(m-1/2)' M_mu h^(m+1/2) (eq:energy)."""
    return float(np.dot(e_m * g.M_eps_w(), e_m) + np.dot(h_mmh * g.M_mu_w(), h_mph))


def leapfrog_trace(g: Grid, e, h, nsteps, sources=(), t0=0.0, probes=()):
    """Leapfrog with per-step outputs: one step at a time,
    energy[m] = E_{m+1} = e^(m+1)' M_eps e^(m+1) + h^(m+1/2)' M_mu h^(m+3/2) (eq:energy,
    PAPER:256-275) and probe[m, r] = e^(m+1) at the probe edges (comp, i, j, k).
    Returns (e^(n), h^(n+1/2), energy, probe)."""
    e = np.array(e, dtype=np.float64, copy=True)
    h = np.array(h, dtype=np.float64, copy=True)
    dofs = [g.edge_dof(*pr) for pr in probes]
    energy = np.zeros(nsteps)
    probe = np.zeros((nsteps, len(dofs)))
    for m in range(nsteps):
        e1, h1 = leapfrog(g, e, h, 1, sources, t0, m)
        energy[m] = energy_staggered(g, e1, h, h1)
        probe[m] = [e1[d] for d in dofs]
        e, h = e1, h1
    return e, h, energy, probe


# ---------------------------------------------------------------------------
# Leja points and divided differences (readings 14, 15)
# ---------------------------------------------------------------------------
@lru_cache(maxsize=None)
def leja_points(count: int) -> tuple:
    """Symmetrised greedy Leja sequence on [-1,1]: xi = (1, -1, 0, +eta1, -eta1, ...),
    eta_l = argmax over candidates {k/5000} of log|eta| + sum_prev log|eta^2 - xi^2|
    (prev = 1, eta_1..eta_{l-1}); ties -> smallest eta (reading 14)."""
    xs = [1.0, -1.0, 0.0]
    pos = [1.0]
    cand = np.arange(1, 5001, dtype=np.float64) / 5000.0
    while len(xs) < count:
        obj = np.log(np.abs(cand))
        for p in pos:
            with np.errstate(divide="ignore"):
                obj = obj + np.log(np.abs(cand * cand - p * p))
        best = int(np.argmax(obj))            # first maximum = smallest eta on ties
        eta = float(cand[best])
        pos.append(eta)
        xs += [eta, -eta]
    return tuple(xs[:count])


def divided_differences(nodes: Sequence[complex], gamma: float, dps: int = 60) -> List[complex]:
    """Newton divided differences of g(xi) = exp(gamma*xi) on `nodes`, i.e.
    d_k = g[xi_0, ..., xi_k], by the textbook recursive table in mpmath at `dps`
    digits (d-hat_k = gamma^k exp[z_0..z_k] with xi = z/gamma; reading 15)."""
    import mpmath as mp
    with mp.workdps(dps):
        z = [mp.mpc(complex(x).real, complex(x).imag) for x in nodes]
        col = [mp.exp(gamma * x) for x in z]
        out = [col[0]]
        n = len(z)
        for lev in range(1, n):
            new = []
            for r in range(n - lev):
                if z[r + lev] == z[r]:
                    # confluent (all nodes r..r+lev equal): g^(lev)(z)/lev!
                    if any(z[q] != z[r] for q in range(r, r + lev + 1)):
                        raise ValueError("mixed confluent nodes not supported")
                    new.append(mp.mpf(gamma) ** lev * mp.exp(gamma * z[r]) / mp.factorial(lev))
                else:
                    new.append((col[r + 1] - col[r]) / (z[r + lev] - z[r]))
            col = new
            out.append(col[0])
        return [complex(v) for v in out]


@dataclass
class Plan:
    """One polynomial propagator p(X)^s for exp(tau A): X = (h/gamma) A_orig, h = tau/s.

    method 'leja': nodes xi_k = 2i*xi'_k (capacity-scaled), a = 1.05*h*rho, gamma = a/2;
    method 'taylor': all nodes 0, gamma = 1, d_k = 1/k!."""
    method: str
    m: int
    s: int
    tau: float
    rho: float
    a: float
    gamma: float
    nodes: list
    d: list


def make_plan(method: str, m: int, s: int, tau: float, rho: float) -> Plan:
    if m < 1 or (m > 1 and m % 2):
        raise ValueError("degree must be 1 or even (conjugate-closed node prefix)")
    h = tau / s
    if method == "taylor":
        nodes = [0j] * (m + 1)
        d = [1.0 / math.factorial(k) + 0j for k in range(m + 1)]
        return Plan("taylor", m, s, tau, rho, 0.0, 1.0, nodes, d)
    a = 1.05 * h * rho
    gamma = a / 2.0
    if gamma == 0:       # degenerate interval: the c -> 0 limit is Taylor
        nodes = [0j] * (m + 1)
        d = [1.0 / math.factorial(k) + 0j for k in range(m + 1)]
        return Plan("leja", m, s, tau, rho, 0.0, 1.0, nodes, d)
    xi = newton_order(m)
    nodes = [2j * x for x in xi]
    d = divided_differences(nodes, gamma)
    return Plan("leja", m, s, tau, rho, a, gamma, nodes, d)


def newton_order(m: int) -> tuple:
    """Evaluation order of the degree-m Leja node set (DESIGN reading 29): the same set as the
    greedy prefix (1, -1, 0, +eta_1, -eta_1, ..., +eta_L, -eta_L), L = (m-2)/2, with the zero
    node moved last:  (1, -1, +eta_1, -eta_1, ..., +eta_L, -eta_L, 0).  The interpolation
    polynomial depends only on the node set, so L_{m,c} is unchanged; m = 1 uses (1, -1)."""
    if m == 1:
        return (1.0, -1.0)
    xs = leja_points(m + 1)
    return tuple([xs[0], xs[1]] + list(xs[3:m + 1]) + [xs[2]])


def newton_eval_scalar(plan: Plan, lam: complex) -> complex:
    """p(X) at a scalar X = lam (Newton form) -- used by pins."""
    y = 0j
    w = 1 + 0j
    for k in range(plan.m + 1):
        y += plan.d[k] * w
        w = w * (lam - plan.nodes[k])
    return y


# ---------------------------------------------------------------------------
# exp(tau A) v -- original variables, A_orig = [[0, -M_nu C], [M_eps^-1 C^T, 0]]
# ---------------------------------------------------------------------------
class ScaledOp:
    """X = sigma * dt * A_orig applied through the C stencil: y_h = -sH.*(C x_e),
    y_e = sE.*(C^T x_h), sE = cE*sigma, sH = cH*sigma (SURVEY finding 1).

    dtype f32: sE = fl32(fl32(cE64) * fl32(sigma)) -- the documented constant recipe the
    kernels use (reading 24), evaluated here in numpy float32 arithmetic."""

    def __init__(self, g: Grid, sigma: float, dtype: str = "f64"):
        self.g = g
        if dtype == "f32":
            s32 = np.float32(sigma)
            self.sE = (g.cE.astype(np.float32) * s32).astype(np.float64)
            self.sH = (g.cH.astype(np.float32) * s32).astype(np.float64)
        else:
            self.sE = g.cE * sigma
            self.sH = g.cH * sigma

    def __call__(self, xe, xh):
        g = self.g
        ye = np.empty(3 * g.Np)
        yh = np.empty(3 * g.Np)
        lib().or_apply_A(g.nx, g.ny, g.nz, _dp(self.sE), _dp(self.sH),
                         _dp(np.ascontiguousarray(xe)), _dp(np.ascontiguousarray(xh)),
                         _dp(ye), _dp(yh))
        return ye, yh


def expmv_newton_complex(g: Grid, plan: Plan, e, h, check_imag=True):
    """Plain definition: b_{i+1} = L_{m,c}(tau A/s) b_i, i = 0..s-1, each
    L evaluated in complex Newton form  sum_k d_k prod_{j<k} (X - xi_j) b.  fp64 only."""
    X = ScaledOp(g, (plan.tau / plan.s) / (plan.gamma * g.dt), "f64")
    be = np.array(e, dtype=np.complex128)
    bh = np.array(h, dtype=np.complex128)
    max_imag = 0.0
    for _ in range(plan.s):
        we, wh = be.copy(), bh.copy()
        ye = plan.d[0] * we
        yh = plan.d[0] * wh
        for k in range(1, plan.m + 1):
            xr_e, xr_h = X(we.real, wh.real)
            xi_e, xi_h = X(we.imag, wh.imag)
            xw_e = xr_e + 1j * xi_e
            xw_h = xr_h + 1j * xi_h
            we = xw_e - plan.nodes[k - 1] * we
            wh = xw_h - plan.nodes[k - 1] * wh
            ye = ye + plan.d[k] * we
            yh = yh + plan.d[k] * wh
        nrm = max(np.abs(ye).max(initial=0.0), np.abs(yh).max(initial=0.0), 1e-300)
        max_imag = max(max_imag, max(np.abs(ye.imag).max(initial=0.0),
                                     np.abs(yh.imag).max(initial=0.0)) / nrm)
        be, bh = ye.real.astype(np.complex128), yh.real.astype(np.complex128)
    if check_imag and max_imag > 1e-8:
        raise AssertionError(f"Newton sum not real: {max_imag}")
    return be.real.copy(), bh.real.copy()


def pair_schedule(plan: Plan):
    """Real conjugate-pair schedule of one substep (readings 28-29): nodes come
    in conjugate pairs (k, k+1) = (+i eta, -i eta); the zero node is last.  Entries:
    ('pair', k, eta) / ('last', k, eta) (the final pair, which also adds d_m w_m) /
    ('half', k, eta) (m = 1)."""
    m = plan.m
    if m == 1:
        return [("half", 0, abs(plan.nodes[0].imag))]
    return [("last" if k == m - 2 else "pair", k, abs(plan.nodes[k].imag)) for k in range(0, m, 2)]


def pair_constants(plan: Plan, dtype: str = "f64"):
    """Per-op constants, each computed in fp64 and rounded once to dtype (reading 24):
    a = Re d_k + eta Im d_{k+1}, b = Re d_{k+1}, e2 = eta^2 and, for 'last', c = Re d_m."""
    out = []
    for kind, k, eta in pair_schedule(plan):
        a = plan.d[k].real + eta * plan.d[k + 1].imag
        b = plan.d[k + 1].real
        c = plan.d[k + 2].real if kind == "last" else 0.0
        out.append((kind, float(_round(a, dtype)), float(_round(b, dtype)),
                    float(_round(eta * eta, dtype)), float(_round(c, dtype))))
    return out


def expmv_pairs_et(g: Grid, plan: Plan, e, h, eps: float, dtype: str = "f64"):
    """expmv_pairs with the early termination of the Newton sum (reading 18;
    SURVEY 8(f) f2): within a substep, before op k >= 2, stop if the two previous ops both
    had ||delta y|| <= eps ||y|| (delta y = the op's increment of y), norms in the energy
    inner product <x,y> = sum_e x y / cE_T + sum_h x y / cH_T.  Returns (e, h, A-applications
    performed)."""
    X = ScaledOp(g, (plan.tau / plan.s) / (plan.gamma * g.dt), dtype)
    consts = pair_constants(plan, dtype)
    we = np.where(g.cE_T != 0, 1.0 / np.where(g.cE_T != 0, g.cE_T, 1.0), 0.0)
    wh = np.where(g.cH_T != 0, 1.0 / np.where(g.cH_T != 0, g.cH_T, 1.0), 0.0)

    def n2(xe, xh):
        return float(np.dot(xe * we, xe) + np.dot(xh * wh, xh))

    be = np.array(e, dtype=np.float64, copy=True)
    bh = np.array(h, dtype=np.float64, copy=True)
    apps = 0
    for _ in range(plan.s):
        we_, wh_ = be, bh
        ye = np.zeros_like(be)
        yh = np.zeros_like(bh)
        small = []
        for k, (kind, a, b, e2, c) in enumerate(consts):
            if k >= 2 and small[k - 1] and small[k - 2]:
                break
            apps += 1 if kind == "half" else 2
            ue, uh = X(we_, wh_)
            ne = ye + a * we_ + b * ue
            nh = yh + a * wh_ + b * uh
            if kind != "half":
                xe, xh = X(ue, uh)
                we2 = xe + e2 * we_
                wh2 = xh + e2 * wh_
                if kind == "last":
                    ne = ne + c * we2
                    nh = nh + c * wh2
                else:
                    we_, wh_ = we2, wh2
            small.append(n2(ne - ye, nh - yh) <= eps * eps * n2(ne, nh))
            ye, yh = ne, nh
        be, bh = ye, yh
    return be, bh, apps


def expmv_pairs_numpy(g: Grid, plan: Plan, e, h, dtype: str = "f64"):
    """The same polynomial in real arithmetic, conjugate pairs folded (readings 28-29):
        pair: u = X w; y += a w + b u; w = X u + e2 w
        last: u = X w; y += a w + b u + c (X u + e2 w)      half (m = 1): u = X w; y += a w + b u
        substep: w = b; y = 0; ...; b = y
    Arithmetic fp64; constants rounded to `dtype` (reading 24).  Pinned against
    expmv_newton_complex in fp64."""
    X = ScaledOp(g, (plan.tau / plan.s) / (plan.gamma * g.dt), dtype)
    consts = pair_constants(plan, dtype)
    be = np.array(e, dtype=np.float64, copy=True)
    bh = np.array(h, dtype=np.float64, copy=True)
    for _ in range(plan.s):
        we, wh = be, bh
        ye = np.zeros_like(be)
        yh = np.zeros_like(bh)
        for kind, a, b, e2, c in consts:
            ue, uh = X(we, wh)
            ye = ye + a * we + b * ue
            yh = yh + a * wh + b * uh
            if kind != "half":
                xe, xh = X(ue, uh)
                we2 = xe + e2 * we
                wh2 = xh + e2 * wh
                if kind == "last":
                    ye = ye + c * we2
                    yh = yh + c * wh2
                else:
                    we, wh = we2, wh2
        be, bh = ye, yh
    return be, bh


def expmv_pairs(g: Grid, plan: Plan, e, h, dtype: str = "f64"):
    """expmv_pairs_numpy's recurrence, the same steps in the same order, run by the plain C
    loops of fit_oracle.c (or_expmv_pairs) -- fast enough for the full-horizon parity runs.
    Pinned to expmv_pairs_numpy (tests/test_oracle_expmv.py)."""
    X = ScaledOp(g, (plan.tau / plan.s) / (plan.gamma * g.dt), dtype)
    consts = pair_constants(plan, dtype)
    kinds = np.array([{"pair": 0, "half": 1, "last": 2}[k] for k, *_ in consts], dtype=np.intc)
    a, b, e2, c = (np.array([x[q] for x in consts], dtype=np.float64) for q in (1, 2, 3, 4))
    be = np.array(e, dtype=np.float64, copy=True)
    bh = np.array(h, dtype=np.float64, copy=True)
    rc = lib().or_expmv_pairs(g.nx, g.ny, g.nz, _dp(X.sE), _dp(X.sH), len(consts),
                              kinds.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _dp(a), _dp(b),
                              _dp(e2), _dp(c), int(plan.s), _dp(be), _dp(bh))
    if rc != 0:
        raise MemoryError("or_expmv_pairs: workspace allocation failed")
    return be, bh


def expmv_krylov(g: Grid, l: int, s: int, tau: float, e, h, dtype: Optional[str] = None):
    """Krylov approximation of exp(tau A) v (Arnoldi with sigma = infinity, PAPER:383-402;
    SURVEY 8(f) f3), step by step: for each of s substeps of h = tau/s,
        beta = ||b||, v_1 = b / beta; for j = 1..l: w = X v_j (X = h A_orig),
        h_ij = <v_i, w>, w -= h_ij v_i (i = 1..j, the sweep done twice: modified
        Gram-Schmidt with one reorthogonalisation), h_{j+1,j} = ||w||, v_{j+1} = w / h_{j+1,j},
        b <- beta V_l expm(H_l) e_1,
    in the energy inner product <x, y> = sum_e x y / cE_T + sum_h x y / cH_T over live DOFs
    (proportional to <e,e>_eps + <h,h>_mu).  A happy breakdown
    (h_{j+1,j} <= 1e-12 max|h|) ends the space early (reading 31).  Returns (e, h, A-applications)."""
    import scipy.linalg
    dtype = dtype or g.dtype
    n3 = 3 * g.Np
    we = np.where(g.cE_T != 0, 1.0 / np.where(g.cE_T != 0, g.cE_T, 1.0), 0.0)
    wh = np.where(g.cH_T != 0, 1.0 / np.where(g.cH_T != 0, g.cH_T, 1.0), 0.0)
    wgt = np.concatenate([we, wh])

    def dot(x, y):
        return float(np.dot(x * wgt, y))

    b = np.concatenate([np.asarray(e, float), np.asarray(h, float)])
    if tau == 0.0:
        return b[:n3].copy(), b[n3:].copy(), 0
    X = ScaledOp(g, (tau / s) / g.dt, dtype)
    apps = 0
    for _ in range(s):
        beta = math.sqrt(max(dot(b, b), 0.0))
        if beta == 0.0:
            break
        V = [b / beta]
        H = np.zeros((l, l))
        lr, hmax = l, 0.0
        for j in range(l):
            xe, xh = X(V[j][:n3], V[j][n3:])
            apps += 1
            w = np.concatenate([xe, xh])
            for _pass in range(2):
                for i in range(j + 1):
                    hij = dot(V[i], w)
                    H[i, j] += hij
                    hmax = max(hmax, abs(hij))
                    w = w - hij * V[i]
            if j + 1 == l:
                break
            hn = math.sqrt(max(dot(w, w), 0.0))
            hmax = max(hmax, hn)
            if not hn > 1e-12 * hmax:
                lr = j + 1
                break
            H[j + 1, j] = hn
            V.append(w / hn)
        c = scipy.linalg.expm(H[:lr, :lr])[:, 0]
        b = beta * sum(c[i] * V[i] for i in range(lr))
    return b[:n3].copy(), b[n3:].copy(), apps


def expmv_horner(g: Grid, plan: Plan, e, h, dtype: str = "f64"):
    """The same polynomial as expmv_pairs in nested (Horner) order (DESIGN reading 33):
    with the pair blocks (a_k + b_k X) and the factors (X^2 + e2_k) of pair_constants,
        p(X) b = sum_k (a_k + b_k X) prod_{j<k} (X^2 + e2_j) b  +  c prod_{j<K} (X^2 + e2_j) b,
    evaluated from the innermost block out:
        r = b, s = c;  for k = K-1 .. 0:  r <- (a_k b + b_k (X b)) + s (X (X r) + e2_k r),  s = 1
    ('half', m = 1: r = a b + b_k X b).  Arithmetic fp64, constants rounded to `dtype`."""
    X = ScaledOp(g, (plan.tau / plan.s) / (plan.gamma * g.dt), dtype)
    consts = pair_constants(plan, dtype)
    be = np.array(e, dtype=np.float64, copy=True)
    bh = np.array(h, dtype=np.float64, copy=True)
    for _ in range(plan.s):
        xbe, xbh = X(be, bh)
        re_, rh_ = be, bh
        scale = consts[-1][4]
        for k in range(len(consts) - 1, -1, -1):
            kind, a, bk, e2, _c = consts[k]
            ne = a * be + bk * xbe
            nh = a * bh + bk * xbh
            if kind != "half":
                ue, uh = X(re_, rh_)
                x2e, x2h = X(ue, uh)
                ne = ne + scale * (x2e + e2 * re_)
                nh = nh + scale * (x2h + e2 * rh_)
            re_, rh_ = ne, nh
            scale = 1.0
        be, bh = re_, rh_
    return be, bh


def expmv(g: Grid, plan: Plan, e, h, mode: str = "pairs", dtype: Optional[str] = None):
    if plan.tau == 0.0:
        return np.array(e, float), np.array(h, float)
    if mode == "complex":
        return expmv_newton_complex(g, plan, e, h)
    if mode == "horner":
        return expmv_horner(g, plan, e, h, dtype or g.dtype)
    return expmv_pairs(g, plan, e, h, dtype or g.dtype)


def half_step_plan(g: Grid, rho: float) -> Plan:
    """Propagator for the 1/2 dt reconstruction shift (reading 10): truncated Taylor of
    degree 24 with s = max(1, ceil(rho*dt/2)) substeps (error < 1e-24 per unit theta)."""
    theta = rho * g.dt * 0.5
    s = max(1, int(math.ceil(theta)))
    return make_plan("taylor", 24, s, 0.5 * g.dt, rho)


# ---------------------------------------------------------------------------
# ParaExp (Algorithm 1; 452-470 eq:averaging1/2)
# ---------------------------------------------------------------------------
def partition(nsteps: int, p: int):
    """Step boundaries S_0 = 0 < ... < S_p = nsteps, uniform M = nsteps // p, residual to the
    last interval (reading 8)."""
    if p < 1 or nsteps < p:
        raise ValueError("need p >= 1 and nsteps >= p")
    M = nsteps // p
    return [j * M for j in range(p)] + [nsteps]


def paraexp(g: Grid, sources, t0: float, nsteps: int, p: int, plan_for, u0=None,
            tail: str = "exp", mode: str = "pairs", sum_mode: str = "horner", rho=None,
            dtype: Optional[str] = None):
    """Algorithm 1 executed sequentially.  plan_for(tau) -> Plan for the propagator E_i of
    a sub-interval of length tau.  Returns (e^(n), h^(n+1/2)).

    tail='exp'     : W = sum_{j<p} E_p..E_{j+1} s_j (+ E_p..E_1 u0) with s_j = (e_j, h_sync_j)
                     (Horner or independent-tail sums); output e = e_p + W_e,
                     h = h_p + [exp(dt/2 A) W]_h  (eq:averaging1/2 at t^{n}, t^{n+1/2}).
    tail='leapfrog': tails propagated by source-free leapfrog from the staggered seeds;
                     equals serial leapfrog up to roundoff."""
    dtype = dtype or g.dtype
    S = partition(nsteps, p)
    rho = g.rho_cfl if rho is None else rho
    Ehalf = half_step_plan(g, rho)

    def E(i, we, wh):
        tau = (S[i] - S[i - 1]) * g.dt
        return expmv(g, plan_for(tau), we, wh, mode, dtype)

    def LF(i, we, wh):
        return leapfrog(g, we, wh, S[i] - S[i - 1])

    parts = []
    for i in range(1, p + 1):
        z_e, z_h = g.zeros()
        ei, hi = leapfrog(g, z_e, z_h, S[i] - S[i - 1], sources, t0, S[i - 1])
        parts.append((ei, hi))
    e_p, h_p = parts[-1]

    if tail == "leapfrog":
        We = Wh = None
        if u0 is not None:
            e0, h0 = g.clean(*u0)
            We, Wh = e0, half_step_start(g, e0, h0)
        for i in range(1, p + 1):
            if We is not None:
                We, Wh = LF(i, We, Wh)
            if i < p:
                ei, hi = parts[i - 1]
                We, Wh = (ei.copy(), hi.copy()) if We is None else (We + ei, Wh + hi)
        if We is None:
            return e_p.copy(), h_p.copy()
        return e_p + We, h_p + Wh

    seeds = []
    for i in range(1, p):
        ei, hi = parts[i - 1]
        seeds.append((ei, sync_h(g, ei, hi)))

    if sum_mode == "horner":
        We = Wh = None
        if u0 is not None:
            We, Wh = g.clean(*u0)
        for i in range(1, p + 1):
            if We is not None:
                We, Wh = E(i, We, Wh)
            if i < p:
                se, sh = seeds[i - 1]
                We, Wh = (se.copy(), sh.copy()) if We is None else (We + se, Wh + sh)
    else:  # independent tails, summed in order j = 1..p
        tails = []
        if u0 is not None:
            te, th = g.clean(*u0)
            for i in range(1, p + 1):
                te, th = E(i, te, th)
            tails.append((te, th))
        for j in range(1, p):
            te, th = seeds[j - 1]
            for i in range(j + 1, p + 1):
                te, th = E(i, te, th)
            tails.append((te, th))
        We = Wh = None
        for te, th in tails:
            We, Wh = (te.copy(), th.copy()) if We is None else (We + te, Wh + th)

    if We is None:
        return e_p.copy(), h_p.copy()
    _, Wh_half = expmv(g, Ehalf, We, Wh, mode, dtype)
    return e_p + We, h_p + Wh_half


def paraexp_boundary_states(g: Grid, sources, t0: float, nsteps: int, p: int, plan_for, u0=None,
                            rho=None, dtype: Optional[str] = None, mode: str = "pairs"):
    """The reconstructed same-time solution at every sub-interval boundary (f1; the E(t) of
    PAPER:742-747 sampled at T_i, i = 1..p), written as its plain definition with independent
    tails (a different association from the library's Horner accumulator):
        u(T_i) = s_i + sum_{j<i} E_i ... E_{j+1} s_j  (+ E_i ... E_1 u0),
    s_j = (e_j, h_sync_j) the seed of sub-interval j (reading 9).  Returns [(e, h)] * p."""
    dtype = dtype or g.dtype
    S = partition(nsteps, p)

    def E(i, we, wh):
        return expmv(g, plan_for((S[i] - S[i - 1]) * g.dt), we, wh, mode, dtype)

    seeds = []
    for i in range(1, p + 1):
        z_e, z_h = g.zeros()
        ei, hi = leapfrog(g, z_e, z_h, S[i] - S[i - 1], sources, t0, S[i - 1])
        seeds.append((ei, sync_h(g, ei, hi)))
    states = []
    for i in range(1, p + 1):
        ue, uh = seeds[i - 1][0].copy(), seeds[i - 1][1].copy()
        starts = [(j, seeds[j - 1]) for j in range(1, i)]
        if u0 is not None:
            starts.insert(0, (0, g.clean(*u0)))
        for j, (te, th) in starts:
            for q in range(j + 1, i + 1):
                te, th = E(q, te, th)
            ue, uh = ue + te, uh + th
        states.append((ue, uh))
    return states


def paraexp_block(g: Grid, sources, t0: float, nsteps: int, p: int, plan_for, first: int,
                  last: int, u0=None, mode: str = "pairs", dtype: Optional[str] = None):
    """One worker's share of Algorithm 1's parfor for the contiguous block of
    sub-intervals [first, last] (1-based; first = 0 => none): its tails carried to T_p,
        W_r = sum_{j in block, j < p} E_p..E_{j+1} s_j  (+ E_p..E_1 u0 if first == 1),
    and, if it owns p, the particular state (e_p, h_p).  The sum over workers of W_r is the
    W of paraexp() (superposition; SURVEY finding 9)."""
    dtype = dtype or g.dtype
    S = partition(nsteps, p)
    We = Wh = None
    P = None
    if first >= 1:
        if first == 1 and u0 is not None:
            We, Wh = g.clean(*u0)
        for i in range(first, last + 1):
            z_e, z_h = g.zeros()
            ei, hi = leapfrog(g, z_e, z_h, S[i] - S[i - 1], sources, t0, S[i - 1])
            if We is not None:
                We, Wh = expmv(g, plan_for((S[i] - S[i - 1]) * g.dt), We, Wh, mode, dtype)
            if i < p:
                se, sh = ei, sync_h(g, ei, hi)
                We, Wh = (se.copy(), sh.copy()) if We is None else (We + se, Wh + sh)
            else:
                P = (ei, hi)
        for i in range(last + 1, p + 1):
            if We is not None:
                We, Wh = expmv(g, plan_for((S[i] - S[i - 1]) * g.dt), We, Wh, mode, dtype)
    if We is None:
        We, Wh = g.zeros()
    return (We, Wh), P


def paraexp_finish(g: Grid, P, W, rho, mode: str = "pairs", dtype: Optional[str] = None):
    """Reconstruction on the owner of sub-interval p (eq:averaging1/2, reading 10)."""
    dtype = dtype or g.dtype
    _, Wh_half = expmv(g, half_step_plan(g, rho), W[0], W[1], mode, dtype)
    return P[0] + W[0], P[1] + Wh_half


def cost_proc(nt: int, p: int, n_leja: int) -> float:
    """eq:tot_cost: C_proc = (2/p) n_t + n_Leja + 2."""
    return 2.0 * nt / p + n_leja + 2


def norm_A(g: Grid, tol: float = 1e-10) -> float:
    """||A||_2 of the normal A = T A_orig T^-1 (lambda_max = ||A||_2), as the
    square root of the largest eigenvalue of the symmetric PSD operator -A^2 = A^T A on the
    live DOFs, from scipy's ARPACK (eigsh) on a LinearOperator that applies A_orig through the
    oracle's own stencil (X = dt A_orig, then / dt).  T = sqrt(M_eps) on e, sqrt(M_mu) on h."""
    from scipy.sparse.linalg import LinearOperator, eigsh
    n3 = 3 * g.Np
    X = ScaledOp(g, 1.0, "f64")
    Te = np.where(g.live_e, np.sqrt(np.where(g.live_e, g.Meps, 1.0)), 0.0)
    Mmu = g.M_mu_w()
    Th = np.where(g.live_h, np.sqrt(np.where(g.live_h, Mmu, 1.0)), 0.0)
    Ti = np.concatenate([np.where(Te > 0, 1.0 / np.where(Te > 0, Te, 1.0), 0.0),
                         np.where(Th > 0, 1.0 / np.where(Th > 0, Th, 1.0), 0.0)])
    T = np.concatenate([Te, Th])

    def mv(x):
        x = np.asarray(x, float).reshape(-1)
        u = Ti * x
        ae, ah = X(u[:n3], u[n3:])
        ae, ah = X(ae, ah)
        return -(T * np.concatenate([ae, ah]))

    op = LinearOperator((2 * n3, 2 * n3), matvec=mv, dtype=np.float64)
    # seeded random start on the live DOFs (a symmetric start can be orthogonal to the top mode)
    v0 = np.random.default_rng(12345).uniform(-1, 1, 2 * n3) * np.concatenate([g.live_e, g.live_h])
    lam = eigsh(op, k=1, which="LA", tol=tol, v0=v0, return_eigenvectors=False)[0]
    return math.sqrt(max(lam, 0.0)) / g.dt


# ---------------------------------------------------------------------------
# Planner (reading 16) -- no paper table; theta_m pinned by tests/test_oracle_theta.py
# (series-tail root for Taylor, barycentric interpolant for Leja)
# ---------------------------------------------------------------------------
def poly_error(method: str, m: int, theta: float, npts: int = 801) -> float:
    """max_{x in [-theta, theta]} |p(ix) - e^{ix}| for the degree-m interpolant of one
    substep of length theta (rho h = theta), interval margin a = 1.05 theta."""
    plan = make_plan(method, m, 1, theta, 1.0)
    xs = np.linspace(0.0, theta, npts)
    err = 0.0
    for x in xs:
        lam = 1j * x / plan.gamma
        err = max(err, abs(newton_eval_scalar(plan, lam) - complex(math.cos(x), math.sin(x))))
    return err


def theta_m(method: str, m: int, tol: float) -> float:
    """Largest theta with max error <= tol*theta (bisection, 40 halvings).  Pinned by
    tests/test_oracle_theta.py (Taylor: the series-tail root; Leja: the barycentric interpolant)."""
    lo, hi = 0.0, float(2 * m + 4)
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        if mid > 0 and poly_error(method, m, mid) <= tol * mid:
            lo = mid
        else:
            hi = mid
    return lo
