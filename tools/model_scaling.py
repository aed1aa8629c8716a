"""ParaExp wall time at G = 1, 2, 4, 8 GPUs as a MODEL from measured per-rank block times
(one B200; no multi-GPU box was available): for each G, every rank's paraexp_solve_block
(its cost-balanced contiguous block: particular sweeps + Horner tails to T_p) is run on cuda:0
and timed with CUDA events on the launching stream (after one warm-up call of the same block);
the modelled wall time is

    T_G = max_rank T_block(rank) + T_reduce + T_finish

with T_finish measured (paraexp_solve_finish on the root) and T_reduce = bytes of W / the
measured 8-rank all-reduce bus bandwidth of this pool (725 GB/s, B200_PROFILING.md; a reduce
moves at most that).  The G = 1 row is the measured single-GPU solve.  Both schedules of
SURVEY 8(e): (A) cost-balanced contiguous blocks with Horner tails (the default) and (B)
independent tails, longest-processing-time-first (tail_mode EXP_LPT).  Printed as JSON lines.
Usage: python tools/model_scaling.py [workload] [p ...]   (default c3 8 64)"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from bench import workload  # noqa: E402

BUS_GBS = 725.0


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    ps = [int(a) for a in sys.argv[2:]] or [8, 64]
    w = workload(name)
    g = pe.Grid.from_workload(w)
    info = g.info(compute_rho_pow=True)
    if not w.nsteps and w.t_end:            # interval given as T (refined meshes): n_t from dt
        w.nsteps = int(math.ceil(w.t_end / info["dt"]))
    td = g.torch_dtype()
    z = lambda: torch.zeros(3 * g.npts, dtype=td, device="cuda:0")   # noqa: E731
    kw = dict(sources=w.sources, method=w.method, m=w.m, s=w.s, eps_A=w.eps_A)
    es = 8 if w.dtype == "f64" else 4
    wbytes = 6 * w.cells * es
    for p in ps:
        eo, ho = z(), z()
        pe.solve(g, w.nsteps, p, e_out=eo, h_out=ho, **kw)                      # warm-up (plans)
        st1 = pe.solve(g, w.nsteps, p, e_out=eo, h_out=ho, **kw)
        rho = st1["rho"]
        serial = None
        te, th = z(), z()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        pe.leapfrog(g, te, th, w.nsteps, w.sources)
        s1.record()
        torch.cuda.synchronize()
        serial = s0.elapsed_time(s1)
        print(json.dumps({"workload": w.name, "p": p, "G": 1, "kind": "measured", "wall_ms": st1["ms_total"],
                          "serial_leapfrog_ms": serial, "speedup": serial / st1["ms_total"], "nsteps": w.nsteps,
                          "a_applications": st1["a_applications"], "rho": rho, "rho_cfl": info["rho_cfl"],
                          "rho_pow": info["rho_pow"]}), flush=True)
        for G, sched in [(g_, sc) for sc in ("blocks", "lpt") for g_ in (2, 4, 8)]:
            tm = "exp" if sched == "blocks" else "exp_lpt"
            blocks = []
            v = (z(), z())
            We, Wh = z(), z()
            for r in range(G):
                wv = (z(), z())
                # warm-up of this rank's block first (first-use allocations of its concurrent-
                # sweep buffers, exchange slots and streams are not part of a rank's time)
                pe.solve_block(g, r, G, w.nsteps, p, wv, rho=rho, v=(z(), z()), tail_mode=tm, **kw)
                wv = (z(), z())
                st = pe.solve_block(g, r, G, w.nsteps, p, wv, rho=rho, v=v, tail_mode=tm, **kw)
                blocks.append({"rank": r, "first": st["first_interval"], "last": st["last_interval"],
                               "ms": st["ms_total"], "leapfrog_steps": st["leapfrog_steps"],
                               "a_applications": st["a_applications"]})
                We += wv[0]
                Wh += wv[1]
            fin = pe.solve_finish(g, (We, Wh), v, eo, ho, rho=rho)
            t_red = wbytes / (BUS_GBS * 1e9) * 1e3
            crit = max(b["ms"] for b in blocks)
            wall = crit + t_red + fin["ms_total"]
            print(json.dumps({"workload": w.name, "p": p, "G": G, "kind": "model", "schedule": sched, "wall_ms": wall,
                              "critical_block_ms": crit, "reduce_ms_model": t_red, "finish_ms": fin["ms_total"],
                              "serial_leapfrog_ms": serial, "speedup": serial / wall, "blocks": blocks,
                              "rho": rho, "rho_pow": info["rho_pow"]}), flush=True)


if __name__ == "__main__":
    main()
