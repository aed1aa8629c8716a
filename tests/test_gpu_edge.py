"""GPU edge cases and error behaviour of the C ABI (degenerate grids, empty runs, invalid
arguments, divergence detection)."""
import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from gpu_util import inputs, lib_expmv, lib_leapfrog, lib_solve
from oracle import fit
from synth import Source, gauss_sine, random_fields

pytestmark = pytest.mark.gpu


def test_zero_steps_and_zero_tau_are_identity_on_live_dofs():
    n = (9, 7, 5)
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    lg = pe.Grid(*n, d0=1e-3, dt_frac=0.9)
    e_raw, h_raw = random_fields(*n, seed=1)
    e, h = inputs(og, e_raw, h_raw)
    ge, gh, _ = lib_leapfrog(lg, e_raw, h_raw, 0, [])
    assert np.array_equal(ge, e) and np.array_equal(gh, h)    # dead DOFs zeroed, rest kept
    ge, gh, _ = lib_expmv(lg, 0.0, e_raw, h_raw, rho=og.rho_cfl, m=8, s=1)
    assert np.array_equal(ge, e) and np.array_equal(gh, h)


@pytest.mark.parametrize("n", [(1, 1, 1), (1, 4, 3), (2, 1, 5), (5, 3, 1), (33, 2, 2)])
def test_degenerate_grids(n):
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    lg = pe.Grid(*n, d0=1e-3, dt_frac=0.9)
    e, h = inputs(og, *random_fields(*n, seed=2))
    ref = fit.leapfrog(og, e, h, 25)
    ge, gh, _ = lib_leapfrog(lg, e, h, 25, [])
    np.testing.assert_allclose(ge, ref[0], rtol=0, atol=1e-12 * max(1.0, np.abs(ref[0]).max()))
    np.testing.assert_allclose(gh, ref[1], rtol=0, atol=1e-12 * max(1e-3, np.abs(ref[1]).max()))


def test_invalid_arguments():
    with pytest.raises(pe.ParaexpError) as ei:
        pe.Grid(0, 4, 4, d0=1e-3, dt_frac=0.9)
    assert ei.value.code == pe.EINVAL
    with pytest.raises(pe.ParaexpError):
        pe.Grid(4, 4, 4, d0=1e-3, dt_frac=0.9, dt=1e-12)             # both dt and dt_frac
    with pytest.raises(pe.ParaexpError):
        pe.Grid(4, 4, 4, d0=1e-3, dt_frac=0.9, eps_r=-np.ones(64))
    lg = pe.Grid(6, 6, 6, d0=1e-3, dt_frac=0.9)
    og = fit.Grid(6, 6, 6, d0=1e-3, dt_frac=0.9)
    e, h = og.zeros()
    with pytest.raises(pe.ParaexpError) as ei:                       # source on a PEC wall edge
        lib_leapfrog(lg, e, h, 3, [Source(0, 2, 0, 3, "gauss_paper", 1.0, 1e-12)])
    assert ei.value.code == pe.EINVAL
    with pytest.raises(pe.ParaexpError) as ei:                       # nsteps < p
        lib_solve(lg, 3, 4, [])
    assert ei.value.code == pe.EINVAL
    with pytest.raises(pe.ParaexpError) as ei:                       # odd Leja degree > 1
        lib_expmv(lg, 1e-12, e, h, m=3, s=1, rho=og.rho_cfl)
    assert ei.value.code == pe.EINVAL


def test_cfl_warning_and_divergence_detection():
    lg = pe.Grid(8, 8, 8, d0=1e-3, dt_frac=1.5)
    assert lg.warnings == pe.abi.WCFL                                 # warn, do not forbid
    og = fit.Grid(8, 8, 8, d0=1e-3, dt_frac=1.5)
    e, h = inputs(og, *random_fields(8, 8, 8, seed=3))
    with pytest.raises(pe.ParaexpError) as ei:
        lib_leapfrog(lg, e, h, 3000, [], check_finite=True)
    assert ei.value.code == pe.EDIVERGED


def test_host_only_grid_refuses_compute():
    lg = pe.Grid(4, 4, 4, d0=1e-3, dt_frac=0.9, device=-1)
    import torch
    t = torch.zeros(3 * lg.npts, dtype=torch.float64, device="cuda:0")
    with pytest.raises(Exception):
        pe.leapfrog(lg, t, t.clone(), 1)


def test_rho_pow_bounds():
    """K5 Lanczos estimate: <= rho_CFL and close to the closed-form rho on a uniform grid;
    on random eps (C2-like) clearly below rho_CFL (SURVEY finding 8)."""
    import math
    from oracle import dense
    lg = pe.Grid(16, 16, 16, d0=1e-3, dt_frac=0.9)
    inf = lg.info(compute_rho_pow=True)
    c = 1 / math.sqrt(fit.EPS0 * fit.MU0)
    rho = dense.cavity_frequencies(16, 16, 16, 1e-3, c).max()
    assert rho * 0.97 <= inf["rho_pow"] <= rho * 1.0000001
    eps = np.random.default_rng(2).uniform(1, 4, 32 ** 3)
    lg2 = pe.Grid(32, 32, 32, d0=1e-3, eps_r=eps, dt_frac=0.95)
    inf2 = lg2.info(compute_rho_pow=True)
    assert 0.6 * inf2["rho_cfl"] < inf2["rho_pow"] < 0.85 * inf2["rho_cfl"]


@pytest.mark.parametrize("window", ["0", "1"])
def test_nccl_path_one_rank(monkeypatch, window):
    """a8 on one GPU: a one-rank NCCL communicator with the collectives forced on
    (PARAEXP_FORCE_COLLECTIVES: ncclReduce of W, ncclAllReduce of the trace rows,
    ncclBroadcast of the output) gives the same result as the communicator-free solve; with
    PARAEXP_NCCL_WINDOW=1 the reduce goes through the ncclMemAlloc'd buffer registered with
    ncclCommWindowRegister (symmetric)."""
    import torch
    monkeypatch.setenv("PARAEXP_FORCE_COLLECTIVES", "1")
    monkeypatch.setenv("PARAEXP_NCCL_WINDOW", window)
    n = (24, 16, 9)
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    lg = pe.Grid(*n, d0=1e-3, dt_frac=0.9)
    u0 = inputs(og, *random_fields(*n, seed=12))
    src = [gauss_sine(2, 5, 5, 4, f0=60e9, bw=60e9)]
    comm = pe.Comm(0, 1, 0, id_bytes=pe.Comm.unique_id())
    outs = []
    for c in (None, comm):
        eo = torch.zeros(3 * lg.npts, dtype=torch.float64, device="cuda:0")
        ho = torch.zeros_like(eo)
        u = (torch.tensor(u0[0], device="cuda:0"), torch.tensor(u0[1], device="cuda:0"))
        st, en, pr = pe.solve_trace(lg, 40, 4, src, u0=u, m=16, s=3, rho=og.rho_cfl, e_out=eo,
                                    h_out=ho, probes=[(2, 5, 5, 4)], comm=c, broadcast_out=True)
        torch.cuda.synchronize()
        outs.append((eo.cpu().numpy(), ho.cpu().numpy(), en.cpu().numpy(), pr.cpu().numpy(), st))
    for a, b in zip(outs[0][:2] + outs[0][3:4], outs[1][:2] + outs[1][3:4]):   # e, h, probes
        assert np.array_equal(a, b)
    # energy rows: block partial sums are combined with atomics (order not reproducible)
    np.testing.assert_allclose(outs[1][2], outs[0][2], rtol=1e-13, atol=0)
    assert outs[1][4]["ms_reduce"] > 0          # the collective ran
    # auto rho (K5) goes through ncclBroadcast(rho) when the collectives are on: same plan, same bits
    auto = []
    for c in (None, comm):
        eo = torch.zeros(3 * lg.npts, dtype=torch.float64, device="cuda:0")
        ho = torch.zeros_like(eo)
        st = pe.solve(lg, 40, 4, src, eps_A=1e-10, e_out=eo, h_out=ho, comm=c)
        torch.cuda.synchronize()
        auto.append((eo.cpu().numpy(), ho.cpu().numpy(), st))
    assert auto[0][2]["rho"] == auto[1][2]["rho"] and 0 < auto[1][2]["rho"] <= og.rho_cfl * (1 + 1e-12)
    assert (auto[0][2]["m"], auto[0][2]["s_first"]) == (auto[1][2]["m"], auto[1][2]["s_first"])
    assert np.array_equal(auto[0][0], auto[1][0]) and np.array_equal(auto[0][1], auto[1][1])
    comm.close()


@pytest.mark.parametrize("pinned", [True, False])
def test_host_pointer_fields(pinned):
    """Fields passed as HOST pointers (pinned or pageable) are staged by the library and give
    bit-identical results to device pointers (leapfrog, expmv, solve with u0)."""
    import torch
    n = (20, 12, 7)
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    lg = pe.Grid(*n, d0=1e-3, dt_frac=0.9)
    e_raw, h_raw = random_fields(*n, seed=31)
    src = [gauss_sine(2, 5, 5, 3, f0=60e9, bw=60e9)]

    def host(x):
        t = torch.tensor(x, dtype=torch.float64)
        return t.pin_memory() if pinned else t

    de, dh = torch.tensor(e_raw, device="cuda:0"), torch.tensor(h_raw, device="cuda:0")
    he, hh = host(e_raw), host(h_raw)
    pe.leapfrog(lg, de, dh, 30, src)
    pe.leapfrog(lg, he, hh, 30, src)
    torch.cuda.synchronize()
    assert torch.equal(de.cpu(), he) and torch.equal(dh.cpu(), hh)
    pe.expmv(lg, 5 * og.dt, de, dh, m=16, s=2, rho=og.rho_cfl)
    pe.expmv(lg, 5 * og.dt, he, hh, m=16, s=2, rho=og.rho_cfl)
    torch.cuda.synchronize()
    assert torch.equal(de.cpu(), he) and torch.equal(dh.cpu(), hh)
    eo_d, ho_d = torch.zeros_like(de), torch.zeros_like(dh)
    eo_h, ho_h = host(np.zeros_like(e_raw)), host(np.zeros_like(h_raw))
    pe.solve(lg, 24, 3, src, u0=(de, dh), m=12, s=2, rho=og.rho_cfl, e_out=eo_d, h_out=ho_d)
    pe.solve(lg, 24, 3, src, u0=(he, hh), m=12, s=2, rho=og.rho_cfl, e_out=eo_h, h_out=ho_h)
    torch.cuda.synchronize()
    assert torch.equal(eo_d.cpu(), eo_h) and torch.equal(ho_d.cpu(), ho_h)
    assert eo_h.abs().max() > 0


def test_host_alloc_pinned_fields():
    """paraexp_host_alloc: page-locked memory (cudaPointerGetAttributes says host-registered via
    torch's is_pinned), usable as e_out / h_out of a solve with the bits of the device-buffer
    solve, against the oracle too; free is idempotent."""
    import torch
    n = (20, 12, 7)
    og = fit.Grid(*n, d0=1e-3, dt_frac=0.9)
    lg = pe.Grid(*n, d0=1e-3, dt_frac=0.9)
    src = [gauss_sine(2, 5, 5, 3, f0=60e9, bw=60e9)]
    he, hh = pe.HostField(lg), pe.HostField(lg)
    assert he.nbytes == 3 * lg.npts * 8 and he.ptr % 256 == 0
    assert he.tensor.is_pinned() and hh.tensor.is_pinned()
    he.tensor.fill_(7.0)
    hh.tensor.fill_(7.0)
    de = torch.zeros(3 * lg.npts, dtype=torch.float64, device="cuda:0")
    dh = torch.zeros_like(de)
    pe.solve(lg, 24, 3, src, m=12, s=2, rho=og.rho_cfl, e_out=de, h_out=dh)
    pe.solve(lg, 24, 3, src, m=12, s=2, rho=og.rho_cfl, e_out=he.tensor, h_out=hh.tensor)
    torch.cuda.synchronize()
    assert torch.equal(de.cpu(), he.tensor) and torch.equal(dh.cpu(), hh.tensor)
    rho = og.rho_cfl
    ref = fit.paraexp(og, src, 0.0, 24, 3, lambda tau: fit.make_plan("leja", 12, 2, tau, rho))
    for got, want in ((he.tensor.numpy(), ref[0]), (hh.tensor.numpy(), ref[1])):
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    he.close()
    he.close()
    hh.close()
    with pytest.raises(pe.ParaexpError) as ei:
        import ctypes
        pe.check(pe.abi.lib.paraexp_host_alloc(0, ctypes.byref(ctypes.c_void_p())), "paraexp_host_alloc")
    assert ei.value.code == pe.EINVAL


def test_c_example_runs(tmp_path):
    """examples/cavity_solve.c through the C ABI from plain C with host buffers: runs and prints
    a finite, nonzero ParaExp (exact-exponential tails) vs serial leapfrog gap on C1 -- large
    there, since C1's 100 GHz source is 3 cells per wavelength at 0.9 CFL (leapfrog dispersion)."""
    import os
    import re
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1705_08019_b200")
    exe = tmp_path / "cavity_solve"
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "cavity_solve.c"), "-L", libdir,
                           "-l:libparaexp.so", f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    rel = float(re.search(r"= ([0-9.e+-]+)\s*$", out.stdout.strip()).group(1))
    assert 0 < rel < 2.0, out.stdout


@pytest.mark.parametrize("world", [1, 3, 8])
def test_c_ranks_example(tmp_path, world):
    """examples/ranks_solve.c: paraexp_solve_block per (simulated) rank into HOST buffers, a host
    sum, paraexp_solve_finish -- equals the one-call paraexp_solve to summation order."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1705_08019_b200")
    exe = tmp_path / "ranks_solve"
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "ranks_solve.c"), "-L", libdir,
                           "-l:libparaexp.so", f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)])
    out = subprocess.run([str(exe), str(world)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("rank ") == world
