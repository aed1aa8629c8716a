"""One-off whole-grid, full-horizon parity of the bench's own solve (too long for the test
suite): the library's paraexp_solve of the bench workload (C3 256^3 layered, n_t = 4096, p = 8,
auto plan at eps_A = 1e-10: rho from K5, (m, s) from the planner) against the oracle's
sequential Algorithm 1 (fit.paraexp) run with exactly the exported plan (reading 25) on the
box's host cores.  Prints one JSON line: rel-L2 and max-abs per field, plan, timings.
Usage: python tools/full_parity.py [c3|c3-f32]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from bench import workload  # noqa: E402
from oracle import fit  # noqa: E402

TOL = {"f64": 1e-10, "f32": 1e-4}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    w = workload(name)
    g = pe.Grid.from_workload(w)
    td = g.torch_dtype()
    eo = torch.zeros(3 * g.npts, dtype=td, device="cuda:0")
    ho = torch.zeros_like(eo)
    t0 = time.perf_counter()
    st = pe.solve(g, w.nsteps, w.p, w.sources, method=w.method, eps_A=w.eps_A, e_out=eo, h_out=ho)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    got_e, got_h = eo.double().cpu().numpy(), ho.double().cpu().numpy()
    m, s1, s2, rho = st["m"], st["s_first"], st["s_last"], st["rho"]
    assert s1 == s2, "sub-intervals of different lengths"
    og = fit.Grid.from_workload(w)
    t0 = time.perf_counter()
    ref_e, ref_h = fit.paraexp(og, w.sources, 0.0, w.nsteps, w.p,
                               lambda tau: fit.make_plan("leja", m, s1, tau, rho), rho=rho, dtype=w.dtype)
    t_or = time.perf_counter() - t0
    out = {"workload": w.name, "dtype": w.dtype, "cells": w.cells, "nsteps": w.nsteps, "p": w.p,
           "plan": {"m": m, "s": s1, "rho": rho, "a_applications": st["a_applications"]},
           "gpu_solve_s": t_gpu, "oracle_s": t_or, "oracle_cores": fit.num_threads(), "tol": TOL[w.dtype]}
    for nm, a, b in (("e", got_e, ref_e), ("h", got_h, ref_h)):
        out[f"rel_l2_{nm}"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
        out[f"max_abs_rel_{nm}"] = float(np.abs(a - b).max() / np.abs(b).max())
    out["pass"] = out["rel_l2_e"] <= TOL[w.dtype] and out["rel_l2_h"] <= TOL[w.dtype]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
