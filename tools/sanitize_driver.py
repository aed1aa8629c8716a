"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):
every default kernel family of the library once, on grids of at most 32 x 16 x 12 cells.

  fused TMA kernels (32x16x12, fp64 and fp32):
    K1r / K1v leapfrog with a source, their TR (trace) variants, K2 / K2v Newton pairs, their
    ET (early-termination) variants, a ParaExp solve (sync, axpy, finite, dot, gather,
    pack/unpack, the dt/2 Taylor propagator) and a solve_block / solve_finish pair
  single-CTA small-grid kernels (12x10x8, fp64 and fp32): K0L leapfrog, K0P polynomial
  unfused kernels (kernels="unfused"): e/h halves, inject, applyX, pair update, lincomb
  K5 Lanczos (rho_pow) and the rho safety net (auto rho)
Usage: compute-sanitizer --tool <tool> python tools/sanitize_driver.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import Source, layered_eps  # noqa: E402


def fields(g, seed):
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(seed)
    e = torch.rand(3 * g.npts, generator=gen, dtype=g.torch_dtype(), device="cuda:0") - 0.5
    h = (torch.rand(3 * g.npts, generator=gen, dtype=g.torch_dtype(), device="cuda:0") - 0.5) * 1e-3
    return e, h


def run(n, dtype, kernels="auto"):
    eps = layered_eps(*n, (1.0, 2.2, 4.4))
    g = pe.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.95, dtype=dtype, kernels=kernels)
    src = [Source(2, n[0] // 2, n[1] // 2, n[2] // 2, "gauss_paper", 1.0, 20e-12)]
    e, h = fields(g, 1)
    pe.leapfrog(g, e, h, 4, src)
    pe.leapfrog_trace(g, e, h, 3, src, probes=[(2, n[0] // 2, n[1] // 2, n[2] // 2)])
    rho = g.info()["rho_cfl"]
    pe.expmv(g, 6 * g.dt, e, h, m=8, s=1, rho=rho)
    pe.expmv(g, 6 * g.dt, e, h, m=16, s=1, rho=rho, eps_A=1e-6, early_term=True)
    eo, ho = torch.zeros_like(e), torch.zeros_like(h)
    pe.solve(g, 16, 4, src, u0=(e, h), m=8, s=1, rho=rho, e_out=eo, h_out=ho)
    pe.solve_trace(g, 16, 4, src, u0=(e, h), m=8, s=1, rho=rho, e_out=eo, h_out=ho,
                   probes=[(2, n[0] // 2, n[1] // 2, n[2] // 2)])
    w = (torch.zeros_like(e), torch.zeros_like(h))
    v = (torch.zeros_like(e), torch.zeros_like(h))
    for r in range(2):
        st = pe.solve_block(g, r, 2, 16, 4, w, src, m=8, s=1, rho=rho, v=v)
    pe.solve_finish(g, w, v, eo, ho, rho=rho)
    pe.expmv(g, 6 * g.dt, e, h, eps_A=1e-8)          # auto rho: K5 Lanczos + the rho check
    torch.cuda.synchronize()
    g.close()
    print(f"ok {n} {dtype} {kernels}", flush=True)


if __name__ == "__main__":
    for dtype in ("f64", "f32"):
        run((32, 16, 12), dtype)                       # fused TMA kernels
        run((12, 10, 8), dtype)                        # single-CTA small kernels
        run((20, 9, 7), dtype, kernels="unfused")      # unfused kernels
    print("sanitize driver done")
