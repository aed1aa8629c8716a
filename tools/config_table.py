"""Measured table for BASELINE.md section 2: for each BASELINE config (C1-C4; C5 via
tools/sweep_c5.py) the leapfrog and expmv-pair kernel rates (cell-updates/s, CUDA events
inside the library), the full ParaExp solve wall time at G = 1 and the serial 1-GPU leapfrog
over the same interval.  Usage: python tools/config_table.py [c1 c2 c3 c3-f32 c4]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_c1, config_c2, config_c3, config_c4  # noqa: E402

CFG = {"c1": config_c1, "c2": config_c2, "c3": lambda: config_c3("f64"),
       "c3-f32": lambda: config_c3("f32"), "c4": config_c4}


def ev_time(fn):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    out = fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


def main():
    names = sys.argv[1:] or list(CFG)
    for name in names:
        w = CFG[name]()
        g = pe.Grid.from_workload(w)
        inf = g.info(compute_rho_pow=True)
        td = g.torch_dtype()
        dev = "cuda:0"
        e = torch.zeros(3 * g.npts, dtype=td, device=dev)
        h = torch.zeros_like(e)
        nlf = min(w.nsteps, 400)
        pe.leapfrog(g, e, h, 20, w.sources)
        st = pe.leapfrog(g, e, h, nlf, w.sources)
        lf_rate = nlf * w.cells / (st["ms_leapfrog_kernels"] * 1e-3)
        e.add_(1e-3)
        pe.expmv(g, 20 * g.dt, e, h, method="leja", m=40, s=1, rho=inf["rho_cfl"])
        st2 = pe.expmv(g, 200 * g.dt, e, h, method="leja", m=40, s=10, rho=inf["rho_cfl"])
        ex_rate = st2["a_applications"] * w.cells / (st2["ms_poly_kernels"] * 1e-3)
        eo = torch.zeros_like(e)
        ho = torch.zeros_like(e)
        kw = dict(sources=w.sources, method=w.method, m=w.m, s=w.s, eps_A=w.eps_A, e_out=eo, h_out=ho)
        pe.solve(g, w.nsteps, w.p, **kw)                        # warm-up (plans, workspace)
        ms_solve, sst = ev_time(lambda: pe.solve(g, w.nsteps, w.p, **kw))
        te = torch.zeros_like(e)
        th = torch.zeros_like(e)
        ms_lf, _ = ev_time(lambda: pe.leapfrog(g, te, th, w.nsteps, w.sources))
        print(json.dumps({
            "config": w.name, "dtype": w.dtype, "grid": [w.nx, w.ny, w.nz], "nsteps": w.nsteps, "p": w.p,
            "material_mode": inf["material_mode"], "rho_pow_over_rho_cfl": inf["rho_pow"] / inf["rho_cfl"],
            "leapfrog_cell_updates_s": lf_rate, "expmv_cell_updates_s": ex_rate,
            "paraexp_wall_ms_G1": ms_solve, "a_applications": sst["a_applications"],
            "plan_m": sst["m"], "plan_s": sst["s_first"], "serial_leapfrog_ms": ms_lf,
            "speedup_G1": ms_lf / ms_solve}), flush=True)
        g.close()
        del e, h, eo, ho, te, th
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
