"""Workload descriptions C1..C5 (BASELINE.json configs; SURVEY 8(d) concrete inputs).

Every random draw uses ``numpy.random.default_rng(seed)`` (PCG64) with the seed
stated here, in fp64, generated once on the host.  Values marked [P] in SURVEY 8(d)
are proposals adopted as stated there (recorded in DESIGN.md "input recipe").

Conventions (shared vocabulary only, no method arithmetic):
  * grid: nx, ny, nz cells; uniform spacing ``d0`` metres on every axis
    (per-axis spacing arrays are accepted by both sides but no config needs them);
  * eps_r: per-cell relative permittivity, length nx*ny*nz, x fastest (None = 1);
  * pec_cell: per-cell uint8 PEC flag (None = no interior PEC);
  * source: a current on one primal edge (comp 0/1/2 = x/y/z, start point i,j,k)
    with waveform kind and parameters (PAPER:640-648 eq:line_current and the
    Gaussian-modulated sine of BASELINE.json);
  * dt_frac: time step as a fraction of the eq:cfl bound (each side computes
    that bound itself);
  * fields are in the canonical point layout: 3 arrays of (nx+1)(ny+1)(nz+1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

# Physical constants (CODATA 2018), SI.
EPS0 = 8.8541878128e-12
MU0 = 1.25663706212e-6
C0 = 299792458.0
Z0 = math.sqrt(MU0 / EPS0)

SOURCE_KINDS = {"zero": 0, "gauss_paper": 1, "gauss_sine": 2, "sine": 3}


@dataclass
class Source:
    """Edge current i(t)*weight on primal edge (comp, i, j, k).

    kind 'gauss_paper': amp*exp(-4((t-t_param)/t_param)^2)
    kind 'gauss_sine' : amp*sin(2 pi f0 (t-t_delay))*exp(-((t-t_delay)/t_param)^2)
    kind 'sine'       : amp*sin(2 pi f0 t)
    kind 'zero'       : 0
    """
    comp: int
    i: int
    j: int
    k: int
    kind: str = "gauss_sine"
    amp: float = 1.0
    t_param: float = 0.0
    f0: float = 0.0
    t_delay: float = 0.0
    weight: float = 1.0


def gauss_sine(comp, i, j, k, f0, bw, amp=1.0, weight=1.0) -> Source:
    """Gaussian-modulated sine with amplitude-spectrum 1/e full width ``bw``:
    tau = 2/(pi*bw), delay t_d = 4*tau (SURVEY 8(d) waveforms)."""
    tau = 2.0 / (math.pi * bw)
    return Source(comp, i, j, k, "gauss_sine", amp, tau, f0, 4.0 * tau, weight)


@dataclass
class Workload:
    name: str
    nx: int
    ny: int
    nz: int
    d0: float
    dtype: str = "f64"
    dt_frac: float = 0.95
    nsteps: int = 100
    p: int = 2
    eps_r: Optional[np.ndarray] = None
    pec_cell: Optional[np.ndarray] = None
    sources: List[Source] = field(default_factory=list)
    u0_seed: Optional[int] = None       # random initial fields (C5) if not None
    method: str = "leja"
    m: int = 0                          # fixed Leja/Taylor degree (0 = from eps_A)
    s: int = 0                          # fixed substeps per propagator (0 = auto)
    eps_A: float = 1e-12
    note: str = ""
    dx: Optional[np.ndarray] = None     # per-cell spacings (non-uniform meshes); None = d0
    dy: Optional[np.ndarray] = None
    dz: Optional[np.ndarray] = None
    t_end: Optional[float] = None        # interval length T when nsteps follows from dt

    @property
    def cells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def npts(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    def u0(self):
        if self.u0_seed is None:
            return None, None
        return random_fields(self.nx, self.ny, self.nz, self.u0_seed)


def random_fields(nx, ny, nz, seed):
    """e ~ U[-1,1] V per edge, h ~ U[-1,1]/Z0 A per dual edge (DESIGN reading 26),
    canonical layout, fp64.  Dead (PEC / virtual) entries are NOT zeroed here:
    both the library and the oracle zero them on input."""
    rng = np.random.default_rng(seed)
    npts = (nx + 1) * (ny + 1) * (nz + 1)
    e = rng.uniform(-1.0, 1.0, size=3 * npts)
    h = rng.uniform(-1.0, 1.0, size=3 * npts) / Z0
    return e, h


# --------------------------------------------------------------------------
def small_cavity(n=(4, 4, 3), d0=1e-3, dt_frac=0.9, nsteps=200, p=2, seed=None,
                 eps_seed=None, src=True, dtype="f64") -> Workload:
    """Tiny test cavity (pins, dense checks).  Optional random eps (U[1,4))."""
    nx, ny, nz = n
    eps = None
    if eps_seed is not None:
        eps = np.random.default_rng(eps_seed).uniform(1.0, 4.0, size=nx * ny * nz)
    sources = []
    if src:
        sources = [gauss_sine(2, nx // 2, ny // 2, nz // 2 if nz > 1 else 0,
                              f0=100e9, bw=50e9)]
    return Workload(f"cavity{nx}x{ny}x{nz}", nx, ny, nz, d0, dtype, dt_frac, nsteps, p,
                    eps_r=eps, sources=sources, u0_seed=seed)


def config_c1() -> Workload:
    """C1: 8^3 PEC vacuum cavity, 1 mm, fp64, 0.9*CFL, 2000 steps, p = 2;
    GAUSS_SINE f0 = 100 GHz, BW = 50 GHz on z-edge (3,5,4) [P]; Leja from eps_A 1e-12 [P]."""
    return Workload("C1", 8, 8, 8, 1e-3, "f64", 0.9, 2000, 2,
                    sources=[gauss_sine(2, 3, 5, 4, f0=100e9, bw=50e9)],
                    method="leja", eps_A=1e-12)


def config_c2(nsteps=20000) -> Workload:
    """C2: 64^3, 1 mm [P], eps_r ~ U[1,4) per cell (seed 2, x-fastest) [P], fp64,
    3 z-edge GAUSS_SINE sources at seeded interior points, f0 ~ U[5,20] GHz, BW = f0,
    drawn from the same generator after eps [P]; 0.95*CFL(min eps), 20000 steps, p = 8."""
    n = 64
    rng = np.random.default_rng(2)
    eps = rng.uniform(1.0, 4.0, size=n * n * n)
    srcs = []
    for _ in range(3):
        i, j = (int(v) for v in rng.integers(8, 56, size=2))
        k = int(rng.integers(8, 56))
        f0 = float(rng.uniform(5e9, 20e9))
        srcs.append(gauss_sine(2, i, j, k, f0=f0, bw=f0))
    return Workload("C2", n, n, n, 1e-3, "f64", 0.95, nsteps, 8, eps_r=eps, sources=srcs,
                    method="leja", eps_A=1e-10)


def layered_eps(nx, ny, nz, layers=(1.0, 2.2, 4.4, 9.8)):
    """z-slabs of equal thickness with the given eps_r from the bottom (C3)."""
    eps = np.empty((nz, ny, nx))
    t = nz // len(layers)
    for li, er in enumerate(layers):
        hi = nz if li == len(layers) - 1 else (li + 1) * t
        eps[li * t:hi] = er
    return eps.reshape(-1)


def config_c3(dtype="f64", p=8, nsteps=4096, n=256) -> Workload:
    """C3: 256^3, 1 mm [P], 4 z-slabs eps_r = 1, 2.2, 4.4, 9.8 [P], fp32 and fp64,
    GAUSS_PAPER sigma_t = 128 ps [P] on z-edge (n/2, n/2, n/8) [P], 0.95*CFL [P],
    n_t = 4096 [P], p in {8, 64}."""
    eps = layered_eps(n, n, n)
    src = [Source(2, n // 2, n // 2, n // 8, "gauss_paper", 1.0, 128e-12)]
    return Workload(f"C3-{dtype}-p{p}", n, n, n, 1e-3, dtype, 0.95, nsteps, p, eps_r=eps,
                    sources=src, method="leja", eps_A=1e-10)


def config_c3r(k=10.0, n=128, dtype="f64", p=8) -> Workload:
    """C3 with one locally refined element (an addition, the paper's R(k) mechanism in 3-D,
    PAPER:708-737): n^3 cells of 1 mm with C3's four z-slabs, the centre column and row of
    cells refined to dx = dy = 1 mm / k (reading 32, as the 2-D wave), over C3's interval
    T = 4096 x 0.95 dt_CFL(1 mm) = 7.494 ns at 0.95 of the refined mesh's eq:cfl step (n_t from
    T, so it grows ~k-fold), GAUSS_PAPER sigma_t = 128 ps on a z-edge off the refined slabs,
    Leja at eps_A = 1e-10."""
    eps = layered_eps(n, n, n)
    d = 1e-3
    dx = np.full(n, d)
    dy = np.full(n, d)
    dz = np.full(n, d)
    c = n // 2
    if k != 1.0:
        dx[c] = d / k
        dy[c] = d / k
    t_end = 4096 * 0.95 * d / (C0 * math.sqrt(3.0))
    src = [Source(2, (5 * n) // 16, (5 * n) // 16, n // 8, "gauss_paper", 1.0, 128e-12)]
    return Workload(f"C3r-{n}-k{k:g}-{dtype}-p{p}", n, n, n, d, dtype, 0.95, 0, p, eps_r=eps,
                    sources=src, method="leja", eps_A=1e-10, dx=dx, dy=dy, dz=dz, t_end=t_end)


def spiral_pec_cells(nx, ny, nz, k_trace=10, turns=5, width=4, gap=2, outer=160, k_sub=10):
    """Synthetic planar rectangular spiral (C4, [P]): PEC cells in layer k_trace along a
    `turns`-turn rectangular spiral, `width` cells wide with `gap`-cell gaps, outer square
    `outer` cells centred; inner end shorted to the ground (k = 0 wall) by a PEC via
    column k in [0, k_sub).  Returns (pec uint8 array x-fastest, port (i, j), inner (i, j))."""
    pec = np.zeros((nz, ny, nx), dtype=np.uint8)
    pitch = width + gap
    x0 = (nx - outer) // 2
    y0 = (ny - outer) // 2
    # walk an inward rectangular spiral of segments; each segment is a width x L strip
    x, y = x0, y0                     # lower-left corner of the current strip head
    L = outer
    dirs = [(1, 0), (0, 1), (-1, 0), (0, -1)]
    seg = 0
    port = (x0, y0)
    lengths = []
    # segment lengths: L, L-width, L-width, L-width-pitch, L-width-pitch, ... (inward)
    lengths.append(outer)
    cur = outer - width
    for t in range(4 * turns - 1):
        lengths.append(cur)
        if t % 2 == 1:
            cur -= pitch
    lengths = [l for l in lengths if l > width]
    cx, cy = x0, y0
    for seg, Lseg in enumerate(lengths):
        dx, dy = dirs[seg % 4]
        if dx == 1:
            xs, xe, ys, ye = cx, cx + Lseg, cy, cy + width
            ncx, ncy = cx + Lseg - width, cy + width
        elif dy == 1:
            xs, xe, ys, ye = cx, cx + width, cy, cy + Lseg
            ncx, ncy = cx - width, cy + Lseg - width
        elif dx == -1:
            xs, xe, ys, ye = cx - Lseg + width, cx + width, cy, cy + width
            ncx, ncy = cx - Lseg + width, cy - width
        else:
            xs, xe, ys, ye = cx, cx + width, cy - Lseg + width, cy + width
            ncx, ncy = cx + width, cy - Lseg + width
        pec[k_trace, max(ys, 0):min(ye, ny), max(xs, 0):min(xe, nx)] = 1
        last = (xs, ys)
        cx, cy = ncx, ncy
    inner = last
    ix, iy = inner
    pec[0:k_sub, iy:iy + width, ix:ix + width] = 1   # via to ground
    return pec.reshape(-1), port, inner


def config_c4(nsteps=23176, p=8) -> Workload:
    """C4: 512x512x64 synthetic spiral inductor, 25 um [P], fp64, PEC box;
    substrate k in [0,10) eps_r = 11.9; PEC spiral in layer k = 10; PEC via;
    port = the 10 z-edges k = 0..9 under the outer terminal, each GAUSS_SINE
    f0 = 5 GHz, BW = 10 GHz; n_t = 23176 [P], p = 8."""
    nx, ny, nz = 512, 512, 64
    eps = np.ones((nz, ny, nx))
    eps[0:10] = 11.9
    pec, port, _ = spiral_pec_cells(nx, ny, nz)
    pi, pj = port
    srcs = [gauss_sine(2, pi, pj, k, f0=5e9, bw=10e9) for k in range(10)]
    return Workload("C4", nx, ny, nz, 25e-6, "f64", 0.95, nsteps, p, eps_r=eps.reshape(-1),
                    pec_cell=pec, sources=srcs, method="leja", eps_A=1e-10)


def config_c5(n=128, dtype="f32", nsteps=1024, p=8) -> Workload:
    """C5: uniform vacuum n^3, 1 mm, random e/h (seed 5+n, DESIGN reading 26), no source."""
    return Workload(f"C5-{n}-{dtype}", n, n, n, 1e-3, dtype, 0.95, nsteps, p,
                    u0_seed=5 + n, method="leja", m=64, s=1, eps_A=1e-12)


def config_c5s(n=768, dtype="f64", nsteps=1024, p=8) -> Workload:
    """C5s (an addition, SURVEY 8(d) C5 note): C5's vacuum n^3 with random u0 PLUS one centred
    GAUSS_PAPER z-edge source (sigma_t = 128 ps), so the particular sweeps are not identically
    zero and ParaExp does not degenerate to one exp(T A) u0.  Auto Leja plan at eps_A = 1e-10
    (as C2-C4), n_t = 1024 [P], p in {8, 16, 64}."""
    src = [Source(2, n // 2, n // 2, n // 2, "gauss_paper", 1.0, 128e-12)]
    return Workload(f"C5s-{n}-{dtype}-p{p}", n, n, n, 1e-3, dtype, 0.95, nsteps, p,
                    sources=src, u0_seed=5 + n, method="leja", eps_A=1e-10)


def config_wave2d(n_pts=41, k=1.0, nsteps=None, p=8, dt_frac=0.99, dtype="f64") -> Workload:
    """The paper's two-dimensional cylindrical wave (Fig. 2): vacuum PEC box
    L_x = L_y = 20 m, L_z = 1 m ("L_y = 1 m" read as L_z, reading 21), n_x = n_y =
    n_pts points (41: Leapfrog/Leja, 121: reference), n_z = 2 points (one cell layer), line
    current in z at the centre, eq:line_current with i_max = 1 A, sigma_t = 2e-8 s, T = 2e-7 s.
    k > 1: the R(k) study: one element shrunk so that biggest/smallest element
    size = k -- here the centre column and row of cells get dx = dy = Delta/k (reading 32;
    the rest of the mesh is unchanged).  nsteps = None leaves n_t to the consumer:
    n_t = ceil(T / dt) with its own dt (t_end = T)."""
    nc = n_pts - 1
    d = 20.0 / nc
    dx = np.full(nc, d)
    dy = np.full(nc, d)
    dz = np.full(1, 1.0)
    c = nc // 2
    if k != 1.0:
        dx[c] = d / k
        dy[c] = d / k
    src = [Source(2, c, c, 0, "gauss_paper", 1.0, 2e-8)]
    return Workload(f"wave2d-{n_pts}-k{k:g}", nc, nc, 1, d, dtype, dt_frac, nsteps or 0, p,
                    sources=src, method="leja", eps_A=1e-2, dx=dx, dy=dy, dz=dz, t_end=2e-7)
