"""Kernel micro-benchmark (development aid): per-step time and algorithmic GB/s of the
leapfrog and expmv-pair kernel families on a C3-like grid, timed with CUDA events.
Usage: python tools/kbench.py [n] [f64|f32] [kernels] [c3|c5]   (c5: uniform vacuum)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_c3, config_c5  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    dtype = sys.argv[2] if len(sys.argv) > 2 else "f64"
    kernels = sys.argv[3] if len(sys.argv) > 3 else "auto"
    which = sys.argv[4] if len(sys.argv) > 4 else "c3"
    w = config_c3(dtype, n=n) if which == "c3" else config_c5(n=n, dtype=dtype)
    g = pe.Grid.from_workload(w, kernels=kernels)
    td = g.torch_dtype()
    es = 8 if dtype == "f64" else 4
    e = torch.rand(3 * g.npts, dtype=td, device="cuda:0")
    h = torch.rand(3 * g.npts, dtype=td, device="cuda:0") * 1e-3
    pe.leapfrog(g, e, h, 10, w.sources)
    nlf = int(os.environ.get("KBENCH_STEPS", "100"))
    st = pe.leapfrog(g, e, h, nlf, w.sources)
    lf_ms = st["ms_leapfrog_kernels"] / nlf
    pe.expmv(g, 1e-11, e, h, method="leja", m=100, s=1, rho=g.rho_cfl)
    st2 = pe.expmv(g, 1e-10, e, h, method="leja", m=100, s=2, rho=g.rho_cfl)
    ex_ms = st2["ms_poly_kernels"] / 200
    cells = w.cells
    print(f"n={n} {which} {dtype} {kernels} chunk={os.environ.get('PARAEXP_ZCHUNK', 'auto')}: "
          f"leapfrog {lf_ms * 1e3:.1f} us/step {12 * es * cells / lf_ms / 1e6:.0f} GB/s | "
          f"expmv {ex_ms * 1e3:.1f} us/A-app {cells / ex_ms / 1e6:.2f} G A-app/s", flush=True)


if __name__ == "__main__":
    main()
