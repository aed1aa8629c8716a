"""GPU parity under the debug switches of the fused kernels' launch machinery (each read once
per process, so every variant runs in its own subprocess): the static unit order
(PARAEXP_STATIC_SCHED), a forced z-chunk (PARAEXP_ZCHUNK) and plain launches without
programmatic dependent launch (PARAEXP_PDL=0).  Each subprocess checks leapfrog, expmv and a
solve against the oracle at the north_star tolerances."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r'''
import sys, numpy as np, torch
sys.path.insert(0, "{root}"); sys.path.insert(0, "{root}/tests")
import paper_1705_08019_b200 as pe
from oracle import fit
from synth import layered_eps, random_fields, gauss_sine
from gpu_util import TOL, assert_parity, inputs, lib_leapfrog, lib_expmv, lib_solve
for dtype in ("f64", "f32"):
    n = (70, 23, 11)
    eps = layered_eps(*n, (1.0, 2.2, 4.4))
    og = fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.95, dtype=dtype)
    lg = pe.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.95, dtype=dtype)
    e, h = inputs(og, *random_fields(*n, seed=5))
    src = [gauss_sine(2, 30, 11, 5, f0=40e9, bw=40e9)]
    ref = fit.leapfrog(og, e, h, 60, src)
    assert_parity(lib_leapfrog(lg, e, h, 60, src)[:2], ref, dtype, "leapfrog")
    for m, s in ((40, 2), (6, 3)):
        plan = fit.make_plan("leja", m, s, 20 * og.dt, og.rho_cfl)
        r2 = fit.expmv(og, plan, e, h, dtype=dtype)
        assert_parity(lib_expmv(lg, 20 * og.dt, e, h, m=m, s=s, rho=og.rho_cfl)[:2], r2, dtype, "expmv")
    rho = og.rho_cfl
    r3 = fit.paraexp(og, src, 0.0, 48, 4, lambda tau: fit.make_plan("leja", 16, 2, tau, rho), u0=(e, h),
                     rho=rho, dtype=dtype)
    assert_parity(lib_solve(lg, 48, 4, src, u0=(e, h), m=16, s=2, rho=rho)[:2], r3, dtype, "solve")
print("variant ok")
'''


@pytest.mark.parametrize("env", [{"PARAEXP_STATIC_SCHED": "1"}, {"PARAEXP_ZCHUNK": "5"},
                                 {"PARAEXP_PDL": "0"}])
def test_variant_parity(env):
    full = dict(os.environ)
    full.update(env)
    out = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT)], env=full,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "variant ok" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
