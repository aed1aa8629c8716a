"""expmv on small grids: device and host time per pair launch over three calls of the same plan
(development aid; the measurement behind DESIGN's note on CUDA graphs).  Usage: pair_small.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from bench import workload  # noqa: E402

n = sys.argv[1] if len(sys.argv) > 1 else "32"
w = workload(f"c3r-20-{n}")
g = pe.Grid.from_workload(w)
td = g.torch_dtype()
e = torch.rand(3 * g.npts, dtype=td, device="cuda:0")
h = torch.rand(3 * g.npts, dtype=td, device="cuda:0")
pe.expmv(g, 1e-12, e, h, method="leja", m=148, s=2, rho=g.rho_cfl)   # warm-up (other plan)
for call in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = pe.expmv(g, 1e-12, e, h, method="leja", m=148, s=20, rho=g.rho_cfl)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"n={n} call {call}: {st['kernel_launches']} launches, device {st['ms_poly_kernels'] * 1e3 / st['kernel_launches']:.2f} "
          f"us/launch, host wall {(t1 - t0) * 1e6 / st['kernel_launches']:.2f} us/launch", flush=True)
