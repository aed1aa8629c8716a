"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI and the
oracle on the same seeded inputs, compare per field (e volts, h amperes)."""
from __future__ import annotations

import math

import numpy as np

from oracle import fit

TOL = {"f64": 1e-10, "f32": 1e-4}   # north_star: rel-L2 per field


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def to_dev(x, grid):
    import torch
    return torch.tensor(np.asarray(x), dtype=grid.torch_dtype(), device=f"cuda:{grid.device}")


def to_host(t):
    return t.detach().double().cpu().numpy()


def inputs(og, e, h):
    """Round inputs to the run dtype and zero dead DOFs (both sides zero them)."""
    return og.clean(e, h)


def lib_leapfrog(lg, e, h, nsteps, sources, t0=0.0, check_finite=False):
    import paper_1705_08019_b200 as pe
    te, th = to_dev(e, lg), to_dev(h, lg)
    st = pe.leapfrog(lg, te, th, nsteps, sources, t0, check_finite)
    return to_host(te), to_host(th), st


def lib_expmv(lg, tau, e, h, **kw):
    import paper_1705_08019_b200 as pe
    te, th = to_dev(e, lg), to_dev(h, lg)
    st = pe.expmv(lg, tau, te, th, **kw)
    return to_host(te), to_host(th), st


def lib_solve(lg, nsteps, p, sources, u0=None, **kw):
    import torch
    import paper_1705_08019_b200 as pe
    eo = torch.zeros(3 * lg.npts, dtype=lg.torch_dtype(), device=f"cuda:{lg.device}")
    ho = torch.zeros_like(eo)
    tu0 = None if u0 is None else (to_dev(u0[0], lg), to_dev(u0[1], lg))
    st = pe.solve(lg, nsteps, p, sources, u0=tu0, e_out=eo, h_out=ho, **kw)
    return to_host(eo), to_host(ho), st


def oracle_plan_for(method, m, s):
    def pf(tau, rho):
        return fit.make_plan(method, m, s, tau, rho)
    return pf


def max_abs_rel(a, b):
    """max |a - b| / max |b| (0 if b == 0 and a == b)"""
    a, b = np.asarray(a), np.asarray(b)
    nb = np.abs(b).max(initial=0.0)
    d = np.abs(a - b).max(initial=0.0)
    return float(d / nb) if nb > 0 else float(d)


def assert_parity(got, ref, dtype, what="", maxabs_factor=100.0):
    """rel-L2 per field (north_star) and, beside it, max-abs relative to the field's largest
    value within maxabs_factor x the tolerance: an error confined to a few edges (a source, a
    PEC corner) is diluted in the rel-L2 of a large box but not in the max-abs."""
    ge, gh = got
    re, rh = ref
    tol = TOL[dtype]
    ee, eh = rel_l2(ge, re), rel_l2(gh, rh)
    assert ee <= tol and eh <= tol, f"{what}: rel-L2 e={ee:.3e} h={eh:.3e} (tol {tol})"
    me, mh = max_abs_rel(ge, re), max_abs_rel(gh, rh)
    assert me <= maxabs_factor * tol and mh <= maxabs_factor * tol, \
        f"{what}: max-abs e={me:.3e} h={mh:.3e} (bound {maxabs_factor * tol})"
    return ee, eh
