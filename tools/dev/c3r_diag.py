"""C3r 24^3 k=10 parity diagnostics (development aid): leapfrog-only and ParaExp errors per
component against the oracle."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np  # noqa: E402

import paper_1705_08019_b200 as pe  # noqa: E402
from gpu_util import lib_leapfrog, lib_solve  # noqa: E402
from oracle import fit  # noqa: E402
from synth import config_c3r  # noqa: E402

w = config_c3r(k=10.0, n=24)
og = fit.Grid.from_workload(w, dtype="f64")
lg = pe.Grid.from_workload(w, dtype="f64")
nsteps = int(math.ceil(w.t_end / lg.dt))
nsteps -= nsteps % w.p
z = np.zeros(3 * og.Np)
for kern in ("auto", "tma", "unfused"):
    lk = pe.Grid.from_workload(w, dtype="f64", kernels=kern)
    ge, gh, _ = lib_leapfrog(lk, z, z, nsteps, w.sources)
    re_, rh = fit.leapfrog(og, z, z, nsteps, w.sources)
    print(kern, "leapfrog rel e", np.linalg.norm(ge - re_) / np.linalg.norm(re_), "h", np.linalg.norm(gh - rh) / np.linalg.norm(rh),
          "|e|", np.linalg.norm(re_), "|h|", np.linalg.norm(rh), flush=True)
got = lib_solve(lg, nsteps, w.p, w.sources, eps_A=1e-10)
st = got[2]
m, s, rho = st["m"], st["s_first"], st["rho"]
ref = fit.paraexp(og, w.sources, 0.0, nsteps, w.p, lambda tau: fit.make_plan("leja", m, s, tau, rho), rho=rho,
                  dtype="f64")
n3 = og.Np
for name, g, r in (("e", got[0], ref[0]), ("h", got[1], ref[1])):
    for c in range(3):
        gc, rc = g[c * n3:(c + 1) * n3], r[c * n3:(c + 1) * n3]
        print(name, c, "rel", np.linalg.norm(gc - rc) / max(np.linalg.norm(rc), 1e-300), "norm", np.linalg.norm(rc),
              "maxerr at", int(np.argmax(np.abs(gc - rc))))
re_, rh = fit.leapfrog(og, z, z, nsteps, w.sources)
print("paraexp vs serial leapfrog (oracle): e", np.linalg.norm(ref[0] - re_) / np.linalg.norm(re_), "h",
      np.linalg.norm(ref[1] - rh) / np.linalg.norm(rh))
print("m s rho", m, s, rho, "rho_cfl", og.rho_cfl)
