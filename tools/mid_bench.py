"""Mid-size grid timing (development aid): per-step / per-A-application time of the leapfrog
and polynomial kernels on C2-like grids, the cooperative shared-memory-resident kernels
(kernels="auto", csrc/mid.cu) against the TMA z-marching kernels (kernels="tma"), CUDA events
inside the library.  Usage: python tools/mid_bench.py [n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_c2  # noqa: E402


def run(n, dtype, kernels):
    w = config_c2()
    if n != 64:
        w.nx = w.ny = w.nz = n
        w.eps_r = np.random.default_rng(2).uniform(1.0, 4.0, size=n ** 3)
        w.sources = [s for s in w.sources if max(s.i, s.j, s.k) < n]
    g = pe.Grid.from_workload(w, dtype=dtype, kernels=kernels)
    td = g.torch_dtype()
    e = torch.rand(3 * g.npts, dtype=td, device="cuda:0")
    h = torch.rand(3 * g.npts, dtype=td, device="cuda:0") * 1e-3
    pe.leapfrog(g, e, h, 20, w.sources)
    nlf = 2000
    st = pe.leapfrog(g, e, h, nlf, w.sources)
    lf_us = st["ms_leapfrog_kernels"] / nlf * 1e3
    pe.expmv(g, 1e-11, e, h, method="leja", m=148, s=1, rho=g.rho_cfl)
    st2 = pe.expmv(g, 1e-10, e, h, method="leja", m=148, s=10, rho=g.rho_cfl)
    ex_us = st2["ms_poly_kernels"] / 1480 * 1e3
    cells = n ** 3
    print(f"n={n}^3 {dtype} {kernels:5s}: leapfrog {lf_us:6.2f} us/step ({cells / lf_us / 1e3:6.1f} G cell-upd/s, "
          f"{st['kernel_launches']} launches) | expmv {ex_us:6.2f} us/A-app ({cells / ex_us / 1e3:6.1f} G/s, "
          f"{st2['kernel_launches']} launches)", flush=True)
    g.close()


def main():
    ns = [int(a) for a in sys.argv[1:]] or [32, 48, 64]
    for n in ns:
        for dtype in ("f64", "f32"):
            for k in os.environ.get("MID_KERNELS", "auto,tma").split(","):
                run(n, dtype, k)


if __name__ == "__main__":
    main()
