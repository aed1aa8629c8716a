"""The oracle's own wall time for whole runs of the small BASELINE configs:
the sequential Algorithm 1 (fit.paraexp: particular sweeps + Horner tails + reconstruction)
with the plan the library chose (rho, m, s from paraexp_solve's stats), and the oracle's serial
leapfrog over the same interval, on all host cores and on one thread; beside them the GPU's
solve and serial-leapfrog times from the same process.  Prints JSON lines.
Usage: python tools/oracle_solve_time.py [c1 c2]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from oracle import fit  # noqa: E402
from synth import config_c1, config_c2  # noqa: E402

CFG = {"c1": config_c1, "c2": config_c2}


def main():
    for name in sys.argv[1:] or ["c1", "c2"]:
        w = CFG[name]()
        g = pe.Grid.from_workload(w)
        td = g.torch_dtype()
        eo = torch.zeros(3 * g.npts, dtype=td, device="cuda:0")
        ho = torch.zeros_like(eo)
        pe.solve(g, w.nsteps, w.p, w.sources, eps_A=w.eps_A, e_out=eo, h_out=ho)
        st = pe.solve(g, w.nsteps, w.p, w.sources, eps_A=w.eps_A, e_out=eo, h_out=ho)
        te, th = torch.zeros_like(eo), torch.zeros_like(eo)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pe.leapfrog(g, te, th, w.nsteps, w.sources)
        b.record()
        torch.cuda.synchronize()
        gpu_lf = a.elapsed_time(b)
        og = fit.Grid.from_workload(w)
        m, s, rho = st["m"], st["s_first"], st["rho"]
        cores = fit.num_threads()
        out = {"config": w.name, "cells": w.cells, "nsteps": w.nsteps, "p": w.p, "plan": {"m": m, "s": s, "rho": rho},
               "gpu_solve_ms": st["ms_total"], "gpu_serial_leapfrog_ms": gpu_lf}
        for threads in (cores, 1):
            fit.set_threads(threads)
            t0 = time.perf_counter()
            fit.paraexp(og, w.sources, 0.0, w.nsteps, w.p, lambda tau: fit.make_plan("leja", m, s, tau, rho), rho=rho)
            t1 = time.perf_counter()
            z = og.zeros()
            fit.leapfrog(og, *z, w.nsteps, w.sources)
            t2 = time.perf_counter()
            out[f"oracle_{threads}t"] = {"cores": threads, "paraexp_s": t1 - t0, "serial_leapfrog_s": t2 - t1}
            if w.cells > 100_000:
                break                              # one-thread C2 would take many minutes
        fit.set_threads(cores)
        print(json.dumps(out), flush=True)
        g.close()


if __name__ == "__main__":
    main()
