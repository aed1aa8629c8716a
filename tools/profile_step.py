"""Small driver for ncu captures: the bench workload's kernels (C3 256^3 layered fp64) on a
short run -- a few fused leapfrog steps and one degree-150 Leja substep (the planner's choice
for the bench's sub-intervals: m = 150, s = 9).  Usage: python tools/profile_step.py [f64|f32] [lf_steps] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_c3  # noqa: E402


def main():
    dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
    nlf = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    w = config_c3(dtype, n=n)
    g = pe.Grid.from_workload(w)
    td = g.torch_dtype()
    e = torch.rand(3 * g.npts, dtype=td, device="cuda:0")
    h = torch.rand(3 * g.npts, dtype=td, device="cuda:0") * 1e-3
    st = pe.leapfrog(g, e, h, nlf, w.sources)
    st2 = pe.expmv(g, 512 * g.dt / 9, e, h, method="leja", m=150, s=1, rho=g.rho_cfl)
    torch.cuda.synchronize()
    print("leapfrog ms", st["ms_leapfrog_kernels"], "expmv ms", st2["ms_poly_kernels"],
          "launches", st["kernel_launches"] + st2["kernel_launches"])


if __name__ == "__main__":
    main()
