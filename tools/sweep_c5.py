"""C5 throughput sweep (BASELINE.json configs[4]): uniform-vacuum n^3 grids,
fp32 and fp64, random e/h in [-1,1] (natural units, reading 26, seed 5+n, generated on the
device with torch's Philox), no source.  Per size and dtype: leapfrog (20 warm-up + 200 timed
steps) and exp(tau A)v at Leja degree 64, s = 1, tau rho = 32 (20 A-applications warm-up,
then 10 substeps timed = 640 A-applications), CUDA events on the launching stream.  Prints one
CSV row per (n, dtype): cell-updates/s and the fraction of the measured HBM copy bandwidth
at the algorithmic 12 values per cell-update.
Usage: python tools/sweep_c5.py [sizes...]   (default 128 256 384 512 640 768)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_c5  # noqa: E402
from synth.configs import Z0  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [128, 256, 384, 512, 640, 768]
    P = peak()
    print("n,dtype,cells,state_GB,leapfrog_Gcu_s,leapfrog_frac_hbm,expmv_Gcu_s,expmv_frac_hbm")
    for n in sizes:
        for dtype in ("f32", "f64"):
            w = config_c5(n=n, dtype=dtype)
            g = pe.Grid.from_workload(w)
            td = g.torch_dtype()
            gen = torch.Generator(device="cuda:0")
            gen.manual_seed(5 + n)
            e = torch.rand(3 * g.npts, generator=gen, dtype=td, device="cuda:0").mul_(2).sub_(1)
            h = torch.rand(3 * g.npts, generator=gen, dtype=td, device="cuda:0").mul_(2).sub_(1).div_(Z0)
            es = 8 if dtype == "f64" else 4
            pe.leapfrog(g, e, h, 20)
            st = pe.leapfrog(g, e, h, 200)
            lf = 200 * w.cells / (st["ms_leapfrog_kernels"] * 1e-3)
            tau = 32.0 / g.rho_cfl
            pe.expmv(g, tau, e, h, method="leja", m=64, s=1, rho=g.rho_cfl)
            st2 = pe.expmv(g, 10 * tau, e, h, method="leja", m=64, s=10, rho=g.rho_cfl)
            ex = st2["a_applications"] * w.cells / (st2["ms_poly_kernels"] * 1e-3)
            gb = 6 * w.cells * es / 1e9
            print(f"{n},{dtype},{w.cells},{gb:.2f},{lf / 1e9:.2f},{lf * 12 * es / 1e9 / P:.3f},"
                  f"{ex / 1e9:.2f},{ex * 12 * es / 1e9 / P:.3f}", flush=True)
            del e, h
            g.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
