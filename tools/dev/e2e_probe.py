"""Where the e2e (host-buffer) solve loses time against the device-buffer solve (development
aid): per call host wall time and device event time, C3 fp64."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from bench import workload  # noqa: E402

w = workload("c3")
g = pe.Grid.from_workload(w)
g.info(compute_rho_pow=True)
td = g.torch_dtype()
ed = torch.zeros(3 * g.npts, dtype=td, device="cuda:0")
hd = torch.zeros_like(ed)
eh = torch.empty(3 * g.npts, dtype=td, pin_memory=True)
hh = torch.empty(3 * g.npts, dtype=td, pin_memory=True)
kw = dict(sources=w.sources, method=w.method, m=w.m, s=w.s, eps_A=w.eps_A)
for outs, name in (((ed, hd), "device"), ((eh, hh), "host"), ((ed, hd), "device"), ((eh, hh), "host")):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    st = pe.solve(g, w.nsteps, w.p, e_out=outs[0], h_out=outs[1], **kw)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: call returned after {1e3 * (t1 - t0):.1f} ms, done after {1e3 * (t2 - t0):.1f} ms, "
          f"device {a.elapsed_time(b):.1f} ms, library ms_total {st['ms_total']:.1f}", flush=True)
