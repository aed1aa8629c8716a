"""R(k) study (Fig. 6): SMVP cost of Leja's exponential over the
whole interval vs leapfrog, C_Leja(k) / C_LF(k), on the 2-D wave mesh with one element shrunk
by k.  C_LF = 2 n_t (eq:cost_LF) with dt = 0.99 dt_CFL(k); C_Leja = s*m of the library's
auto plan for exp(T A) at eps_A = 1e-2 (the paper's Fig. 5 tolerance) with rho = 1.05 ||A||_2.
||A||_2: the library's K5 Lanczos on the GPU (the oracle's ARPACK value of the same meshes is
checked against it in tests/test_gpu_parity.py; tools/ never run the oracle).
Usage: python tools/rk_study.py [--n 41]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1705_08019_b200 as pe  # noqa: E402
from synth import config_wave2d  # noqa: E402


def main():
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 41
    print("k,dt_cfl_s,n_t,C_LF,rho_cfl,norm_A,norm_source,m,s,C_Leja,R")
    for k in (1, 2, 3, 5, 7, 10, 15, 20):
        w = config_wave2d(n, k)
        lg = pe.Grid.from_workload(w, device=0)
        inf = lg.info(compute_rho_pow=True)
        nrm, src = inf["rho_pow"], "library K5 Lanczos"
        nt = math.ceil(w.t_end / inf["dt"])
        c_lf = 2 * nt
        plan = pe.plan_host("leja", 0, 0, 1e-2, w.t_end, 1.05 * nrm, inf["dt"])
        c_leja = plan["m"] * plan["s"]
        print(f"{k},{inf['dt_cfl']:.6e},{nt},{c_lf},{inf['rho_cfl']:.6e},{nrm:.6e},{src},"
              f"{plan['m']},{plan['s']},{c_leja},{c_leja / c_lf:.4f}")


if __name__ == "__main__":
    main()
