"""One leapfrog sequence and one propagator through the mid kernels on C2 (64^3, fp64 unless
argv[1] == f32) for an ncu capture (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_c2  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
w = config_c2()
g = pe.Grid.from_workload(w, dtype=dtype)
td = g.torch_dtype()
e = torch.rand(3 * g.npts, dtype=td, device="cuda:0")
h = torch.rand(3 * g.npts, dtype=td, device="cuda:0") * 1e-3
st = pe.leapfrog(g, e, h, 500, w.sources)

torch.cuda.synchronize()
print(f"leapfrog {st["ms_leapfrog_kernels"] / 500 * 1e3:.2f} us/step (first call, includes module load)")
