"""paraexp-b200: B200-native ParaExp + Leapfrog for FIT-discretised Maxwell equations
(arXiv:1705.08019).  Python binding of the C ABI in include/paraexp.h.

The functions below only marshal arguments (torch tensors -> device pointers, streams,
ctypes structs); every step of the hot path runs in libparaexp.so.  Names follow the C ABI
(``paraexp_<name>`` -> ``<name>``).
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, Optional, Sequence

import numpy as np

from . import abi
from .abi import (EDIVERGED, EINVAL, ENOTSUP, EOVERFLOW, F32, F64, KERNELS_AUTO, KERNELS_FUSED, KERNELS_TMA,  # noqa
                  KERNELS_UNFUSED, KRYLOV, LEJA, TAIL_EXP, TAIL_EXP_LPT, TAIL_LEAPFROG, TAYLOR, ParaexpError,
                  check)

__all__ = ["Grid", "Comm", "leapfrog", "leapfrog_trace", "expmv", "expmv_plan", "solve", "solve_trace",
           "solve_block", "solve_finish",
           "optimal_tolerance",
           "partition", "schedule", "schedule_lpt",
           "leja_points", "plan_host", "theta", "version", "make_sources", "ParaexpError"]

_DT = {"f64": F64, "f32": F32}
_KER = {"auto": KERNELS_AUTO, "unfused": KERNELS_UNFUSED, "fused": KERNELS_FUSED, "tma": KERNELS_TMA}
_SRC_KIND = {"zero": 0, "gauss_paper": 1, "gauss_sine": 2, "sine": 3}
_METHOD = {"taylor": TAYLOR, "leja": LEJA, "krylov": KRYLOV}
_METHOD_NAME = {v: k for k, v in _METHOD.items()}


def version() -> str:
    return abi.lib.paraexp_version().decode()


def _arr(a, dtype):
    if a is None:
        return None, None
    x = np.ascontiguousarray(a, dtype=dtype)
    return x, x.ctypes.data_as(C.POINTER(C.c_double if dtype == np.float64 else C.c_uint8))


class Grid:
    """paraexp_grid_create / _destroy / _info / _coefficients.

    device=-1 builds a host-only grid (coefficients, CFL and plans; no compute)."""

    def __init__(self, nx, ny, nz, d0=None, dx=None, dy=None, dz=None, eps_r=None, mu_r=None,
                 pec_cell=None, dtype="f64", device=0, dt=None, dt_frac=None, kernels="auto"):
        keep = []
        d = abi.paraexp_grid_desc()
        d.nx, d.ny, d.nz = int(nx), int(ny), int(nz)
        for name, v in (("dx", dx), ("dy", dy), ("dz", dz), ("eps_r", eps_r), ("mu_r", mu_r)):
            arr, ptr = _arr(v, np.float64)
            keep.append(arr)
            setattr(d, name, ptr)
        arr, ptr = _arr(pec_cell, np.uint8)
        keep.append(arr)
        d.pec_cell = ptr
        d.d0 = float(d0 or 0.0)
        d.dtype = _DT[dtype]
        d.device = int(device)
        d.dt = float(dt or 0.0)
        d.dt_frac = float(dt_frac or 0.0)
        d.kernels = _KER[kernels]
        h = C.c_void_p()
        rc = abi.lib.paraexp_grid_create(C.byref(d), C.byref(h))
        check(rc, "paraexp_grid_create")
        self.warnings = rc
        self._h = h
        self.dtype = dtype
        self.device = int(device)
        self.nx, self.ny, self.nz = d.nx, d.ny, d.nz
        self.npts = (self.nx + 1) * (self.ny + 1) * (self.nz + 1)
        inf = self.info()
        self.dt, self.dt_cfl, self.rho_cfl = inf["dt"], inf["dt_cfl"], inf["rho_cfl"]

    @classmethod
    def from_workload(cls, w, device=0, dtype=None, kernels="auto"):
        return cls(w.nx, w.ny, w.nz, d0=w.d0, dx=getattr(w, "dx", None), dy=getattr(w, "dy", None),
                   dz=getattr(w, "dz", None), eps_r=w.eps_r, pec_cell=w.pec_cell,
                   dtype=dtype or w.dtype, device=device, dt_frac=w.dt_frac, kernels=kernels)

    @property
    def handle(self):
        return self._h

    def info(self, compute_rho_pow=False, stream=None):
        o = abi.paraexp_grid_info_t()
        check(abi.lib.paraexp_grid_info(self._h, int(bool(compute_rho_pow)), _stream(stream, self),
                                        C.byref(o)), "paraexp_grid_info")
        return {f[0]: getattr(o, f[0]) for f in o._fields_}

    def coefficients(self):
        cE = np.empty(3 * self.npts)
        cH = np.empty(3 * self.npts)
        check(abi.lib.paraexp_grid_coefficients(self._h, cE.ctypes.data_as(abi._dp),
                                                cH.ctypes.data_as(abi._dp)),
              "paraexp_grid_coefficients")
        return cE, cH

    def torch_dtype(self):
        import torch
        return torch.float64 if self.dtype == "f64" else torch.float32

    def close(self):
        if getattr(self, "_h", None):
            abi.lib.paraexp_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream(stream, grid):
    if stream is not None:
        return C.c_void_p(int(stream))
    if grid is None or grid.device < 0:
        return C.c_void_p(0)
    import torch
    return C.c_void_p(torch.cuda.current_stream(grid.device).cuda_stream)


def _field(t, grid, name, writable=True):
    """Validate a canonical-layout field tensor and return its pointer: a tensor on the
    grid's device, or a host (CPU, ideally pinned) tensor that the library stages itself."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if t.device.type != "cpu" and (t.device.type != "cuda" or t.device.index != grid.device):
        raise ValueError(f"{name} must live on cuda:{grid.device} or on the host")
    if t.dtype != grid.torch_dtype() or not t.is_contiguous() or t.numel() != 3 * grid.npts:
        raise ValueError(f"{name} must be a contiguous {grid.torch_dtype()} tensor of 3*npts elements")
    return C.c_void_p(t.data_ptr())


class HostField:
    """paraexp_host_alloc / paraexp_host_free: one canonical-layout field (3*npts values of the
    grid's dtype) in page-locked host memory, viewed as a torch CPU tensor (``.tensor``, no
    copy) that solve / leapfrog / expmv accept as a host buffer."""

    def __init__(self, grid: "Grid"):
        import numpy as np
        import torch
        dt = np.float64 if grid.dtype == "f64" else np.float32
        self.nbytes = 3 * grid.npts * np.dtype(dt).itemsize
        h = C.c_void_p()
        check(abi.lib.paraexp_host_alloc(self.nbytes, C.byref(h)), "paraexp_host_alloc")
        self._p = h
        buf = (C.c_uint8 * self.nbytes).from_address(h.value)
        self.tensor = torch.from_numpy(np.frombuffer(buf, dtype=dt))

    @property
    def ptr(self) -> int:
        return self._p.value

    def close(self):
        """Free the pinned memory; ``tensor`` must not be used afterwards."""
        if getattr(self, "_p", None):
            self.tensor = None
            abi.lib.paraexp_host_free(self._p)
            self._p = None


def make_sources(sources: Optional[Iterable]) -> tuple:
    """Sources as any objects with comp, i, j, k, kind, weight, amp, t_param, f0, t_delay."""
    srcs = list(sources or [])
    arr = (abi.paraexp_source * max(1, len(srcs)))()
    for q, s in enumerate(srcs):
        a = arr[q]
        a.comp, a.i, a.j, a.k = int(s.comp), int(s.i), int(s.j), int(s.k)
        a.kind = _SRC_KIND[s.kind] if isinstance(s.kind, str) else int(s.kind)
        a.weight = float(getattr(s, "weight", 1.0))
        a.amp = float(s.amp)
        a.t_param = float(s.t_param)
        a.f0 = float(s.f0)
        a.t_delay = float(s.t_delay)
    return arr, len(srcs)


def _opts(method="leja", m=0, s=0, eps_A=1e-12, rho=0.0, early_term=False, beta=0.0, rho_check=0):
    o = abi.paraexp_expmv_opts()
    o.method = _METHOD[method] if isinstance(method, str) else int(method)
    o.m, o.s, o.eps_A, o.rho = int(m), int(s), float(eps_A), float(rho or 0.0)
    o.early_term, o.beta = int(bool(early_term)), float(beta or 0.0)
    o.rho_check = int(rho_check)
    return o


def optimal_tolerance(dt: float, beta: float, norm_A: float) -> tuple:
    """paraexp_optimal_tolerance: eps_A* = beta dt^2 / ||A||_2 (eq:tolerance_leja_2), clamped
    to [1e-14, 0.1]; returns (eps_A*, clamped)."""
    c = C.c_int32()
    v = abi.lib.paraexp_optimal_tolerance(float(dt), float(beta), float(norm_A), C.byref(c))
    return v, bool(c.value)


def leapfrog(grid: Grid, e, h, nsteps: int, sources=None, t0: float = 0.0,
             check_finite: bool = False, stream=None) -> dict:
    """paraexp_leapfrog: (e^(0), h^(1/2)) -> (e^(n), h^(n+1/2)) in place on the tensors."""
    arr, n = make_sources(sources)
    st = abi.paraexp_stats()
    check(abi.lib.paraexp_leapfrog(grid.handle, arr, n, float(t0), int(nsteps), _field(e, grid, "e"),
                                   _field(h, grid, "h"), int(bool(check_finite)),
                                   _stream(stream, grid), C.byref(st)), "paraexp_leapfrog", st)
    return st.as_dict()


def _trace(grid, rows, probes, energy):
    """paraexp_trace with device output tensors (fp64) of `rows` energies / rows x nprobe probes."""
    import torch
    probes = list(probes or [])
    if len(probes) > abi.MAX_PROBES:
        raise ValueError(f"at most {abi.MAX_PROBES} probes")
    t = abi.paraexp_trace()
    t.nprobe = len(probes)
    for r, (c, i, j, k) in enumerate(probes):
        t.comp[r], t.i[r], t.j[r], t.k[r] = int(c), int(i), int(j), int(k)
    dev = f"cuda:{grid.device}"
    en = torch.zeros(max(rows, 1), dtype=torch.float64, device=dev) if energy else None
    pr = torch.zeros(max(rows, 1) * max(len(probes), 1), dtype=torch.float64, device=dev) if probes else None
    t.energy = en.data_ptr() if en is not None else None
    t.probe = pr.data_ptr() if pr is not None else None
    return t, en, pr


def leapfrog_trace(grid: Grid, e, h, nsteps: int, sources=None, t0: float = 0.0, probes=None,
                   energy: bool = True, stream=None):
    """paraexp_leapfrog_trace: leapfrog in place plus per-step outputs (f1).  Returns
    (stats, energy[nsteps] fp64 tensor or None, probe[nsteps, nprobe] fp64 tensor or None):
    energy[m] = E_{m+1} (eq:energy), probe[m, r] = e_r^(m+1); probes = [(comp, i, j, k), ...]."""
    arr, n = make_sources(sources)
    t, en, pr = _trace(grid, nsteps, probes, energy)
    st = abi.paraexp_stats()
    check(abi.lib.paraexp_leapfrog_trace(grid.handle, arr, n, float(t0), int(nsteps), _field(e, grid, "e"),
                                         _field(h, grid, "h"), C.byref(t), _stream(stream, grid),
                                         C.byref(st)), "paraexp_leapfrog_trace", st)
    if pr is not None:
        pr = pr[:nsteps * len(probes)].view(nsteps, len(probes))
    if en is not None:
        en = en[:nsteps]
    return st.as_dict(), en, pr


def expmv(grid: Grid, tau: float, e, h, method="leja", m=0, s=0, eps_A=1e-12, rho=0.0,
          stream=None, early_term=False, beta=0.0, rho_check=0) -> dict:
    """paraexp_expmv: (h, e) <- exp(tau A_orig)(h, e) in place."""
    o = _opts(method, m, s, eps_A, rho, early_term, beta, rho_check)
    st = abi.paraexp_stats()
    check(abi.lib.paraexp_expmv(grid.handle, float(tau), C.byref(o), _field(e, grid, "e"),
                                _field(h, grid, "h"), _stream(stream, grid), C.byref(st)),
          "paraexp_expmv", st)
    return st.as_dict()


def _plan_dict(p):
    m = p.m
    return {"method": _METHOD_NAME[p.method], "m": m, "s": p.s, "tau": p.tau,
            "rho": p.rho, "a": p.a, "gamma": p.gamma, "sigma": p.sigma, "n_ops": p.n_ops,
            "xi": list(p.xi[:m + 1]), "d": [complex(p.d_re[k], p.d_im[k]) for k in range(m + 1)]}


def expmv_plan(grid: Grid, tau: float, method="leja", m=0, s=0, eps_A=1e-12, rho=0.0,
               beta=0.0) -> dict:
    o = _opts(method, m, s, eps_A, rho, False, beta)
    p = abi.paraexp_plan_info()
    check(abi.lib.paraexp_expmv_plan(grid.handle, float(tau), C.byref(o), C.byref(p)),
          "paraexp_expmv_plan")
    return _plan_dict(p)


def plan_host(method, m, s, eps_A, tau, rho, dt=1.0) -> dict:
    p = abi.paraexp_plan_info()
    check(abi.lib.paraexp_plan_host(_METHOD[method], int(m), int(s), float(eps_A), float(tau),
                                    float(rho), float(dt), C.byref(p)), "paraexp_plan_host")
    return _plan_dict(p)


def theta(method, m, eps_A) -> float:
    return abi.lib.paraexp_theta(_METHOD[method], int(m), float(eps_A))


def leja_points(count: int) -> list:
    out = (C.c_double * count)()
    check(abi.lib.paraexp_leja_points(int(count), out), "paraexp_leja_points")
    return list(out)


def partition(nsteps: int, p: int) -> list:
    out = (C.c_int64 * (p + 1))()
    check(abi.lib.paraexp_partition(int(nsteps), int(p), out), "paraexp_partition")
    return list(out)


def schedule(p: int, world: int, rank: int, tail_ratio: float = 0.0, has_u0: bool = False) -> tuple:
    """paraexp_schedule: (first, last, root); tail_ratio <= 0 gives equal shares."""
    f, l, r = C.c_int32(), C.c_int32(), C.c_int32()
    check(abi.lib.paraexp_schedule(int(p), int(world), int(rank), float(tail_ratio), int(bool(has_u0)),
                                   C.byref(f), C.byref(l), C.byref(r)), "paraexp_schedule")
    return f.value, l.value, r.value


def schedule_lpt(p: int, world: int, tail_ratio: float = 1.0, has_u0: bool = False) -> tuple:
    """paraexp_schedule_lpt: (owner list [owner of u0 tail, owner of 1, ..., owner of p], root)."""
    o = (C.c_int32 * (p + 1))()
    r = C.c_int32()
    check(abi.lib.paraexp_schedule_lpt(int(p), int(world), float(tail_ratio), int(bool(has_u0)), o,
                                       C.byref(r)), "paraexp_schedule_lpt")
    return list(o), r.value


class Comm:
    """paraexp_comm_*: the library's own NCCL communicator.  The 128-byte id is created on
    rank 0 and broadcast with torch.distributed (plumbing only)."""

    def __init__(self, rank: int, world: int, device: int, id_bytes: Optional[bytes] = None):
        if id_bytes is None:
            id_bytes = Comm.unique_id_via_torch(rank)
        buf = (C.c_uint8 * 128).from_buffer_copy(id_bytes)
        h = C.c_void_p()
        check(abi.lib.paraexp_comm_create(buf, int(rank), int(world), int(device), C.byref(h)),
              "paraexp_comm_create")
        self._h = h
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(abi.lib.paraexp_comm_unique_id(buf), "paraexp_comm_unique_id")
        return bytes(buf)

    @staticmethod
    def unique_id_via_torch(rank: int) -> bytes:
        import torch
        import torch.distributed as dist
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t = torch.tensor(list(Comm.unique_id()), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0)
        return bytes(t.cpu().tolist())

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            abi.lib.paraexp_comm_destroy(self._h)
            self._h = None


def _tail_mode(tail_mode):
    return tail_mode if isinstance(tail_mode, int) else {"exp": TAIL_EXP, "leapfrog": TAIL_LEAPFROG,
                                                         "exp_lpt": TAIL_EXP_LPT}[tail_mode]


def solve(grid: Grid, nsteps: int, p: int, sources=None, t0: float = 0.0, method="leja", m=0,
          s=0, eps_A=1e-12, rho=0.0, tail_mode=TAIL_EXP, u0=None, e_out=None, h_out=None,
          comm: Optional[Comm] = None, broadcast_out=False, stream=None, early_term=False,
          beta=0.0, rho_check=0) -> dict:
    """paraexp_solve (Algorithm 1): returns the stats dict; output in e_out/h_out."""
    arr, n = make_sources(sources)
    o = _opts(method, m, s, eps_A, rho, early_term, beta, rho_check)
    st = abi.paraexp_stats()
    e0 = h0 = C.c_void_p(0)
    if u0 is not None:
        e0 = _field(u0[0], grid, "e0")
        h0 = _field(u0[1], grid, "h0")
    eo = _field(e_out, grid, "e_out") if e_out is not None else C.c_void_p(0)
    ho = _field(h_out, grid, "h_out") if h_out is not None else C.c_void_p(0)
    tm = _tail_mode(tail_mode)
    check(abi.lib.paraexp_solve(grid.handle, comm.handle if comm else C.c_void_p(0), arr, n,
                                float(t0), int(nsteps), int(p), C.byref(o), tm,
                                int(bool(broadcast_out)), e0, h0, eo, ho, _stream(stream, grid),
                                C.byref(st)), "paraexp_solve", st)
    return st.as_dict()


def solve_trace(grid: Grid, nsteps: int, p: int, sources=None, t0: float = 0.0, method="leja", m=0,
                s=0, eps_A=1e-12, rho=0.0, u0=None, e_out=None, h_out=None, probes=None,
                energy: bool = True, comm: Optional[Comm] = None, broadcast_out=False, stream=None,
                early_term=False, beta=0.0):
    """paraexp_solve_trace: solve plus the energy / probe rows at the sub-interval boundaries
    T_1..T_p (f1).  Returns (stats, energy[p] or None, probe[p, nprobe] or None)."""
    arr, n = make_sources(sources)
    o = _opts(method, m, s, eps_A, rho, early_term, beta)
    t, en, pr = _trace(grid, p, probes, energy)
    st = abi.paraexp_stats()
    e0 = h0 = C.c_void_p(0)
    if u0 is not None:
        e0 = _field(u0[0], grid, "e0")
        h0 = _field(u0[1], grid, "h0")
    eo = _field(e_out, grid, "e_out") if e_out is not None else C.c_void_p(0)
    ho = _field(h_out, grid, "h_out") if h_out is not None else C.c_void_p(0)
    check(abi.lib.paraexp_solve_trace(grid.handle, comm.handle if comm else C.c_void_p(0), arr, n,
                                      float(t0), int(nsteps), int(p), C.byref(o),
                                      int(bool(broadcast_out)), e0, h0, eo, ho, C.byref(t),
                                      _stream(stream, grid), C.byref(st)), "paraexp_solve_trace", st)
    if pr is not None:
        pr = pr[:p * len(probes)].view(p, len(probes))
    if en is not None:
        en = en[:p]
    return st.as_dict(), en, pr


def solve_block(grid: Grid, rank: int, world: int, nsteps: int, p: int, w, sources=None,
                t0: float = 0.0, method="leja", m=0, s=0, eps_A=1e-12, rho=0.0, tail_mode=TAIL_EXP,
                u0=None, v=None, stream=None, early_term=False, beta=0.0, rho_check=0) -> dict:
    """paraexp_solve_block: this rank's tails W (written into the tensor pair w = (w_e, w_h))
    and, on the root (stats['root'] == rank), its particular state into v = (v_e, v_h)."""
    arr, n = make_sources(sources)
    o = _opts(method, m, s, eps_A, rho, early_term, beta, rho_check)
    st = abi.paraexp_stats()
    e0 = h0 = C.c_void_p(0)
    if u0 is not None:
        e0, h0 = _field(u0[0], grid, "e0"), _field(u0[1], grid, "h0")
    ve = vh = C.c_void_p(0)
    if v is not None:
        ve, vh = _field(v[0], grid, "v_e"), _field(v[1], grid, "v_h")
    check(abi.lib.paraexp_solve_block(grid.handle, int(rank), int(world), arr, n, float(t0), int(nsteps),
                                      int(p), C.byref(o), _tail_mode(tail_mode), e0, h0,
                                      _field(w[0], grid, "w_e"), _field(w[1], grid, "w_h"), ve, vh,
                                      _stream(stream, grid), C.byref(st)), "paraexp_solve_block", st)
    return st.as_dict()


def solve_finish(grid: Grid, w, v, e_out, h_out, method="leja", eps_A=1e-12, rho=0.0,
                 tail_mode=TAIL_EXP, stream=None) -> dict:
    """paraexp_solve_finish: reconstruction on the root from the summed W and its v."""
    o = _opts(method, 0, 0, eps_A, rho)
    st = abi.paraexp_stats()
    check(abi.lib.paraexp_solve_finish(grid.handle, C.byref(o), _tail_mode(tail_mode),
                                       _field(w[0], grid, "w_e"), _field(w[1], grid, "w_h"),
                                       _field(v[0], grid, "v_e"), _field(v[1], grid, "v_h"),
                                       _field(e_out, grid, "e_out"), _field(h_out, grid, "h_out"),
                                       _stream(stream, grid), C.byref(st)), "paraexp_solve_finish", st)
    return st.as_dict()
