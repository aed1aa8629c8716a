"""GPU parity of the single-CTA shared-memory kernels (csrc/small.cu) that run small grids (<= 2048
cells fp64, <= 4096 fp32): one launch per leapfrog sequence and one per polynomial propagator.
Every material mode (scalar eps, z-table, per-edge eps with interior PEC, non-uniform mesh =
per-face cH) at and below the size limit, against the oracle at the north_star tolerances; the
launch counts prove the small path ran.  The same cases with PARAEXP_NO_SMALL=1 (and
PARAEXP_NO_MID=1, else the mid-size resident leapfrog of mid.cu would take them) run the TMA
z-marching kernels on the same small grids (subprocess: the switch is read once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from oracle import fit
from synth import gauss_sine, layered_eps, random_fields
from gpu_util import assert_parity, inputs, lib_expmv, lib_leapfrog, lib_solve

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _grid_kw(mode, n, seed=3):
    rng = np.random.default_rng(seed)
    nx, ny, nz = n
    if mode == "scalar":
        return dict(d0=1e-3)
    if mode == "ztable":
        return dict(d0=1e-3, eps_r=layered_eps(nx, ny, nz, (1.0, 2.2, 4.4)))
    if mode == "edge":
        pec = np.zeros(nx * ny * nz, np.uint8)
        pec[rng.choice(nx * ny * nz, size=max(1, nx * ny * nz // 20), replace=False)] = 1
        return dict(d0=1e-3, eps_r=rng.uniform(1.0, 5.0, nx * ny * nz), pec_cell=pec)
    if mode == "nonuniform":
        return dict(dx=rng.uniform(0.5e-3, 1.5e-3, nx), dy=rng.uniform(0.5e-3, 1.5e-3, ny),
                    dz=rng.uniform(0.5e-3, 1.5e-3, nz), mu_r=rng.uniform(1.0, 2.0, nx * ny * nz))
    raise ValueError(mode)


CASES = [("scalar", (16, 16, 8), "f64"),        # 2048 cells: the fp64 limit
         ("ztable", (13, 9, 7), "f64"),
         ("edge", (11, 10, 9), "f64"),
         ("nonuniform", (12, 7, 5), "f64"),
         ("scalar", (40, 40, 1), "f64"),        # the paper's 2-D wave mesh
         ("ztable", (16, 16, 16), "f32"),       # 4096 cells: the fp32 limit
         ("edge", (17, 9, 6), "f32"),
         ("nonuniform", (9, 8, 7), "f32")]


def run_case(mode, n, dtype, expect_small):
    kw = _grid_kw(mode, n)
    og = fit.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
    lg = pe.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
    e, h = inputs(og, *random_fields(*n, seed=7))
    ci = (n[0] // 2, n[1] // 2, n[2] // 2)
    src = [gauss_sine(2, *ci, f0=40e9, bw=40e9),
           gauss_sine(0, max(0, ci[0] - 1), ci[1], ci[2], f0=30e9, bw=30e9, amp=0.5)]
    src = [s for s in src if og.cE[og.edge_dof(s.comp, s.i, s.j, s.k)] != 0]
    ref = fit.leapfrog(og, e, h, 60, src)
    ge, gh, st = lib_leapfrog(lg, e, h, 60, src)
    assert_parity((ge, gh), ref, dtype, f"{mode} {n} {dtype} leapfrog")
    assert (st["kernel_launches"] < 10) == expect_small, st
    rho = og.rho_cfl
    for m, s in ((150, 1), (40, 2), (1, 3)):
        plan = fit.make_plan("leja", m, s, 20 * og.dt, rho)
        r2 = fit.expmv(og, plan, e, h, dtype=dtype)
        ge, gh, st = lib_expmv(lg, 20 * og.dt, e, h, m=m, s=s, rho=rho)
        assert_parity((ge, gh), r2, dtype, f"{mode} {n} {dtype} expmv m={m} s={s}")
        if m > 1:
            assert (st["kernel_launches"] < 10) == expect_small, (m, s, st)
    r3 = fit.paraexp(og, src, 0.0, 48, 4, lambda tau: fit.make_plan("leja", 16, 2, tau, rho), u0=(e, h),
                     rho=rho, dtype=dtype)
    assert_parity(lib_solve(lg, 48, 4, src, u0=(e, h), m=16, s=2, rho=rho)[:2], r3, dtype,
                  f"{mode} {n} {dtype} solve")
    lg.close()


@pytest.mark.parametrize("mode,n,dtype", CASES)
def test_small_parity(mode, n, dtype):
    run_case(mode, n, dtype, expect_small=True)


def test_small_limits():
    """one cell over the limit (and more than 16 sources) takes the TMA kernels; still parity"""
    n = (16, 16, 8)
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.95)
    e, h = inputs(og, *random_fields(*n, seed=9))
    src = [gauss_sine(2, 1 + i % 14, 1 + (3 * i) % 14, i % 8, f0=40e9, bw=40e9) for i in range(17)]
    lg = pe.Grid(*n, d0=1e-3, dt_frac=0.95)
    ref = fit.leapfrog(og, e, h, 30, src)
    ge, gh, st = lib_leapfrog(lg, e, h, 30, src)
    assert_parity((ge, gh), ref, "f64", "17 sources")
    assert st["kernel_launches"] >= 30, st
    lg.close()
    n = (17, 11, 11)                               # 2057 cells > 2048: the mid kernel (mid.cu)
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.95)
    e, h = inputs(og, *random_fields(*n, seed=9))
    for kernels, many in (("auto", False), ("tma", True)):
        lg = pe.Grid(*n, d0=1e-3, dt_frac=0.95, kernels=kernels)
        ge, gh, st = lib_leapfrog(lg, e, h, 30, [])
        assert_parity((ge, gh), fit.leapfrog(og, e, h, 30, []), "f64", f"2057 cells {kernels}")
        assert (st["kernel_launches"] >= 30) == many, st
        lg.close()


SNIPPET = r'''
import sys
sys.path.insert(0, "{root}"); sys.path.insert(0, "{root}/tests")
from test_gpu_small import CASES, run_case
for c in CASES:
    run_case(*c, expect_small=False)
print("no-small ok")
'''


def test_no_small_parity():
    env = dict(os.environ, PARAEXP_NO_SMALL="1", PARAEXP_NO_MID="1")
    out = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT)], env=env,
                         capture_output=True, text=True, timeout=800)
    assert out.returncode == 0 and "no-small ok" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
