#!/usr/bin/env python
"""bench.py -- ParaExp + Leapfrog (arXiv:1705.08019) on B200: FIT curl cell-updates/s and
ParaExp wall time.

One "step" = one full ParaExp solve (Algorithm 1, every SURVEY 8(a) row: particular leapfrog
sweeps with the source, seed sync, Leja tails by Horner over the sub-interval propagators,
NCCL reduce for N > 1, dt/2 reconstruction) of the default workload C3 (256^3 layered PEC
cavity, fp64, n_t = 4096, p = 8) through the C ABI.  Inputs are resident in HBM when the timed
region starts; the working set (815 MB per state vector) exceeds the 126 MB L2, so no L2
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W]
                  [--workload c3|c3-f32|c3-p64|c2|c1|c4|c5-<n>[-f64]|c5s-<n>[-f64]|wave2d[-k]|c3r-<k>[-<n>]]
                  [--p P]
                  [--impl ours|reference] [--no-cpu-baseline]

Under torchrun (N > 1) every rank runs one process per GPU; sub-intervals are sharded in
contiguous blocks, tails summed with one ncclReduce (the library's own communicator).
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FIT curl cell-updates/s per GPU; ParaExp wall time & speedup at 1-8 B200"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0


def workload(name):
    from synth import config_c1, config_c2, config_c3, config_c3r, config_c4, config_c5, config_c5s, config_wave2d
    if name == "c3":
        return config_c3("f64", p=8, nsteps=4096)
    if name == "c3-f32":
        return config_c3("f32", p=8, nsteps=4096)
    if name == "c3-p64":
        return config_c3("f64", p=64, nsteps=4096)
    if name == "c2":
        return config_c2()
    if name == "c1":
        return config_c1()
    if name == "c4":
        return config_c4()
    if name.startswith("c3r-"):           # c3r-<k>[-<n>]: C3 with one refined element (an addition)
        parts = name.split("-")
        return config_c3r(k=float(parts[1]), n=int(parts[2]) if len(parts) > 2 else 128)
    if name.startswith("wave2d"):          # wave2d[-k]: the paper's 2-D wave, n_t from T = 2e-7 s
        k = float(name.split("-")[1]) if "-" in name else 1.0
        return config_wave2d(41, k)
    if name.startswith("c5s-"):           # c5s-<n>[-f64]: C5 + a centred source, ParaExp (addition)
        n = int(name.split("-")[1])
        return config_c5s(n=n, dtype="f64" if name.endswith("f64") else "f32")
    if name.startswith("c5-"):
        n = int(name.split("-")[1])
        return config_c5(n=n, dtype="f64" if name.endswith("f64") else "f32")
    raise SystemExit(f"unknown workload {name}")


def set_p(w, p):
    """--p: override the workload's sub-interval count (and the -p<k> suffix of its name)."""
    import re
    w.p = p
    w.name = re.sub(r"-p\d+$", "", w.name) + f"-p{p}"


def hbm_peak():
    try:
        d = json.load(open(PEAKS_FILE))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# ---------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region (200 ms)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# committed `ncu --set full` summaries (tools/ncu_kernels.sh + tools/ncu_summary.py) of the
# current kernels on the bench grids: (file, kernel-name substring); the pair entry is the
# non-initial op (the first op of a substep does not read y)
TRAFFIC_FILES = {("expmv_pair", "C3-f64-p8"): ("profiles/r2_ncu_full_f64_256.json", "pair_fused"),
                 ("leapfrog", "C3-f64-p8"): ("profiles/r2_ncu_full_f64_256.json", "leapfrog_r"),
                 ("expmv_pair", "C3-f32-p8"): ("profiles/r2_ncu_full_f32_256.json", "pair_v"),
                 ("leapfrog", "C3-f32-p8"): ("profiles/r2_ncu_full_f32_256.json", "leapfrog_v")}


def committed_traffic(kernel, w):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    committed `ncu --set full` summary of the same kernel on the same grid (or None)."""
    path, sub = TRAFFIC_FILES.get((kernel, w.name), (None, None))
    if not path or not os.path.exists(os.path.join(ROOT, path)):
        return None, None
    d = [x for x in json.load(open(os.path.join(ROOT, path))) if sub in x["kernel"]]
    if not d:
        return None, None
    return (max(x["dram_bytes"] for x in d) if kernel == "expmv_pair"
            else sum(x["dram_bytes"] for x in d) / len(d)), path


def _oracle_sample(fit, g, w, nlf):
    """nlf leapfrog steps + one degree-8 Leja substep of the oracle on the full grid; returns
    (leapfrog seconds, expmv seconds)."""
    e, h = g.zeros()
    t0 = time.perf_counter()
    e, h = fit.leapfrog(g, e, h, nlf, w.sources, t0=0.0)
    t1 = time.perf_counter()
    plan = fit.make_plan("leja", 8, 1, 3 * g.dt, g.rho_cfl)
    fit.expmv(g, plan, e + 1.0 * g.live_e, h, mode="pairs")
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def cpu_baseline(w, solve_stats=None, single_thread=True):
    """The oracle as it stands, on the host cores, on a bounded sample of the workload:
    20 leapfrog steps (4 above 20 M cells) + one degree-8 Leja substep (8 A-applications) on
    the full grid, cell-updates/s.  Also: the same rate on ONE thread (2 steps + the substep),
    and the oracle's ParaExp wall time for the whole solve extrapolated from the two measured
    rates and the solve's leapfrog steps / A-applications (an extrapolation, not a run)."""
    from oracle import fit
    g = fit.Grid.from_workload(w)
    nlf = 20 if w.cells <= 20_000_000 else 4
    cores = fit.num_threads()
    tl, te = _oracle_sample(fit, g, w, nlf)
    cu = (nlf + 8) * w.cells
    out = {"value": cu / (tl + te), "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
           "sample": f"{w.name} grid {w.nx}x{w.ny}x{w.nz} {w.dtype}: {nlf} leapfrog steps + one "
                     f"degree-8 Leja substep (8 A-applications), plain C/OpenMP oracle",
           "leapfrog_rate": nlf * w.cells / tl, "expmv_rate": 8 * w.cells / te, "seconds": tl + te}
    if single_thread:
        fit.set_threads(1)
        try:
            tl1, te1 = _oracle_sample(fit, g, w, 2)
        finally:
            fit.set_threads(cores)
        out["one_thread"] = {"value": 10 * w.cells / (tl1 + te1), "cores": 1,
                             "sample": "2 leapfrog steps + one degree-8 Leja substep",
                             "leapfrog_rate": 2 * w.cells / tl1, "expmv_rate": 8 * w.cells / te1}
    if solve_stats:
        lf, aa = solve_stats["leapfrog_steps"], solve_stats["a_applications"]
        sec = lf * w.cells / out["leapfrog_rate"] + aa * w.cells / out["expmv_rate"]
        out["paraexp_wall_s_extrapolated"] = sec
        out["paraexp_extrapolation"] = (f"{lf} leapfrog steps / leapfrog_rate + {aa} A-applications / "
                                        f"expmv_rate on {cores} cores (the oracle's own Horner sum does "
                                        f"the same work as one GPU)")
    return out


def run_reference(args, rank, world):
    """--impl reference: the oracle (the only reference this paper-only tier has)."""
    if rank != 0:
        return
    w = workload(args.workload)
    steps = []
    cb = None
    if args.p:
        set_p(w, args.p)
    for it in range(args.warmup + args.steps):
        r = cpu_baseline(w, single_thread=False)
        if it >= args.warmup:
            steps.append(r)
        cb = r
    value = statistics.median(s["value"] for s in steps)
    ms = statistics.median(s["seconds"] for s in steps) * 1e3
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "cell-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": w.dtype,
        "data": "synthetic", "config": {"workload": w.name, "cells": w.cells, "nsteps": w.nsteps,
                                        "p": w.p, "sample": cb["sample"]},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cb["cores"],
                         "kind": "oracle", "sample": cb["sample"]},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


# ---------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernels", default="auto", choices=["auto", "unfused", "fused", "tma"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-serial", action="store_true")
    ap.add_argument("--p", type=int, default=0, help="override the workload's sub-interval count")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e pass (secondary lines)")
    ap.add_argument("--tail-mode", default="exp", choices=["exp", "exp_lpt"],
                    help="schedule (A) blocks + Horner tails (default) or (B) independent tails, LPT")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1705_08019_b200 as pe

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args.workload)
    if args.p:
        set_p(w, args.p)
    grid = pe.Grid.from_workload(w, device=local, kernels=args.kernels)
    stream = torch.cuda.current_stream(local)
    info = grid.info(compute_rho_pow=True, stream=stream.cuda_stream)
    if not w.nsteps and w.t_end:            # interval given as T: n_t from the library's dt
        w.nsteps = int(math.ceil(w.t_end / info["dt"]))
        w.nsteps += (-w.nsteps) % w.p
    # BENCH_FORCE_COMM=1: create the library's NCCL communicator (and run its collectives via
    # PARAEXP_FORCE_COLLECTIVES) even at world size 1 -- exercises the multi-rank path on 1 GPU
    force_comm = os.environ.get("BENCH_FORCE_COMM") == "1"
    if force_comm:
        os.environ["PARAEXP_FORCE_COLLECTIVES"] = "1"
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
    comm = pe.Comm(rank, world, local) if (world > 1 or force_comm) else None
    tdt = grid.torch_dtype()
    e_out = torch.zeros(3 * grid.npts, dtype=tdt, device=f"cuda:{local}")
    h_out = torch.zeros_like(e_out)
    kw = dict(sources=w.sources, method=w.method, m=w.m, s=w.s, eps_A=w.eps_A, comm=comm,
              tail_mode=args.tail_mode)
    u0 = None
    if w.u0_seed is not None:
        import numpy as np
        e0, h0 = w.u0()
        u0 = (torch.tensor(e0, dtype=tdt, device=f"cuda:{local}"),
              torch.tensor(h0, dtype=tdt, device=f"cuda:{local}"))

    def step():
        return pe.solve(grid, w.nsteps, w.p, u0=u0, e_out=e_out, h_out=h_out, **kw)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device events on the launching stream, max over ranks) ----
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    stats = [step() for _ in range(args.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms_local = ev0.elapsed_time(ev1)

    cu_local = sum(s["cell_updates"] for s in stats)
    launches_local = sum(s["kernel_launches"] for s in stats)
    lf_ms = sum(s["ms_leapfrog_kernels"] for s in stats)
    poly_ms = sum(s["ms_poly_kernels"] for s in stats)
    lf_steps = sum(s["leapfrog_steps"] for s in stats)
    a_apps = sum(s["a_applications"] for s in stats)
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([cu_local, launches_local], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(c)
        cu, launches = float(c[0].item()), int(c[1].item())
    else:
        ms, cu, launches = ms_local, float(cu_local), launches_local
    value = cu / (ms * 1e-3)

    e2e_out = None
    if not args.no_e2e:
        # ---- e2e: the same C-ABI call with HOST buffers (pinned): the library copies u0 in and
        # (e_out, h_out) out inside the call, inside the timed region ----
        e_host = torch.empty(3 * grid.npts, dtype=tdt, pin_memory=True)
        h_host = torch.empty(3 * grid.npts, dtype=tdt, pin_memory=True)   # empty_like would not pin
        u0_host = None
        if u0 is not None:
            u0_host = (u0[0].cpu().pin_memory(), u0[1].cpu().pin_memory())
        barrier()
        torch.cuda.synchronize()
        e2e0 = torch.cuda.Event(enable_timing=True)
        e2e1 = torch.cuda.Event(enable_timing=True)
        e2e0.record(stream)
        cu_e2e = 0
        h2d = d2h = 0
        q_bytes = w.nsteps * len(w.sources) * (8 if w.dtype == "f64" else 4)
        for _ in range(args.steps):
            if u0_host is not None:
                h2d += 2 * u0_host[0].numel() * u0_host[0].element_size()
            st = pe.solve(grid, w.nsteps, w.p, u0=u0_host, e_out=e_host, h_out=h_host, **kw)
            h2d += q_bytes           # the library uploads the source amplitude table every call
            cu_e2e += st["cell_updates"]
            if rank == st["root"]:
                d2h += 2 * e_host.numel() * e_host.element_size()
        e2e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = e2e0.elapsed_time(e2e1)
        if world > 1:
            t = torch.tensor([ms_e2e, cu_e2e, h2d, d2h], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            s2 = t[1:].clone()
            dist.all_reduce(s2)
            ms_e2e, cu_e2e, h2d, d2h = float(t[0]), float(s2[0]), float(s2[1]), float(s2[2])
        e2e_out = {"value": cu_e2e / (ms_e2e * 1e-3), "unit": "cell-updates/s",
                   "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps)}

    # ---- serial leapfrog over the same interval on 1 GPU (speedup denominator) ----
    serial_ms = None
    if not args.no_serial and rank == 0:
        te = torch.zeros(3 * grid.npts, dtype=tdt, device=f"cuda:{local}")
        th = torch.zeros_like(te)
        if u0 is not None:
            te.copy_(u0[0])
            th.copy_(u0[1])
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        pe.leapfrog(grid, te, th, w.nsteps, w.sources)
        s1.record(stream)
        torch.cuda.synchronize()
        serial_ms = s0.elapsed_time(s1)
    barrier()

    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel family (HBM bound) ----
    es = 8 if w.dtype == "f64" else 4
    # values per cell-update: 12 state values; a per-edge material array adds 3
    # (leapfrog reads cE once per step) or 1.5 (a pair reads it once per 2 A-applications)
    peak, peak_kind = hbm_peak()
    fam = []
    if lf_ms > 0 and lf_steps > 0:
        fam.append(("leapfrog", lf_ms, lf_steps))
    if poly_ms > 0 and a_apps > 0:
        fam.append(("expmv_pair", poly_ms, a_apps))
    name, fam_ms, units = max(fam, key=lambda f: f[1])
    arr = info["material_mode"] == 2
    per_cell = 12 + ((3 if name == "leapfrog" else 1.5) if arr else 0)
    bytes_per_unit = int(per_cell * es * w.cells)
    achieved = bytes_per_unit * units / (fam_ms * 1e-3) / 1e9
    traffic, traffic_src = committed_traffic(name, w)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": bytes_per_unit * (2 if name == "expmv_pair" else 1),
                "kernel": name,
                "peak_kind": peak_kind,
                "algorithmic_bytes_per_cell_update": per_cell * es,
                "share_of_step": fam_ms / ms_local if ms_local else None,
                "leapfrog_ms": lf_ms, "expmv_ms": poly_ms}

    out = {
        "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": w.dtype,
        "data": "synthetic",
        "config": {"workload": w.name, "grid": [w.nx, w.ny, w.nz], "cells": w.cells,
                   "nsteps": w.nsteps, "p": w.p, "method": w.method, "eps_A": w.eps_A,
                   "rho": stats[-1]["rho"], "m": stats[-1]["m"], "s_per_subinterval": stats[-1]["s_first"],
                   "material_mode": info["material_mode"], "kernels": args.kernels,
                   "schedule": "blocks+horner" if args.tail_mode == "exp" else "independent tails, LPT",
                   "parallelism": f"paraexp time-parallel x{world}",
                   "l2": (f"inputs larger than L2 ({6 * w.cells * es / 1e6:.0f} MB per state vector "
                          f"vs 126 MB L2), no flush" if 6 * w.cells * es > 126e6 else
                          f"L2-resident working set ({6 * w.cells * es / 1e6:.1f} MB per state vector), "
                          f"not flushed: a small-config measurement, not the headline")},
        "per_gpu": value / world,
        "paraexp": {"wall_ms": ms / args.steps, "serial_leapfrog_ms": serial_ms,
                    "speedup_vs_serial_leapfrog": (serial_ms / (ms / args.steps)) if serial_ms else None,
                    "leapfrog_steps_per_solve": stats[-1]["leapfrog_steps"],
                    "a_applications_per_solve": stats[-1]["a_applications"]},
        "roofline": roofline,
        "e2e": e2e_out,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and world == 1:      # rank 0 at N = 1 only
        out["cpu_baseline"] = cpu_baseline(w, solve_stats=stats[-1])
    print(json.dumps(out), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
