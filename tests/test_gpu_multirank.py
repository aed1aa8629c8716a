"""The library's multi-rank ParaExp path (a8, Algorithm 1's parfor + sum) on
one GPU, against the oracle.

* Virtual ranks: every rank's paraexp_solve_block (its cost-balanced contiguous block, the
  particular sweeps, the Horner tails carried to T_p) runs on cuda:0, the W blocks are summed
  on the device, and paraexp_solve_finish reconstructs on the root -- world in {2, 3, 5, 8},
  p in {2, 5, 8, 64}, idle ranks included.  This is exactly what paraexp_solve does per rank
  around its one ncclReduce.
* Two processes (gloo): each calls the library on cuda:0 for its rank and dist.reduce's W.
  The ranks' kernels never wait on one another (the sum is on the host), so sharing one GPU
  is safe.
* The rho safety net (SURVEY finding 8), the debug NaN hook that names the failing
  sub-interval, and stream ordering across calls on one grid.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch

import paper_1705_08019_b200 as pe
from gpu_util import TOL, assert_parity, inputs, lib_expmv, lib_solve, rel_l2, to_dev, to_host
from oracle import fit
from synth import Source, gauss_sine, random_fields

pytestmark = pytest.mark.gpu

N = (24, 16, 12)          # 4608 cells: the fused TMA kernels in fp64 and fp32
NSTEPS = 128
M_FIX, S_FIX = 16, 2


def _setup(dtype, n=N):
    eps = np.random.default_rng(3).uniform(1, 4, int(np.prod(n)))
    og = fit.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.9, dtype=dtype)
    lg = pe.Grid(*n, d0=1e-3, eps_r=eps, dt_frac=0.9, dtype=dtype)
    src = [gauss_sine(2, 7, 6, 5, f0=60e9, bw=60e9), Source(0, 4, 5, 3, "gauss_paper", 0.5, 20e-12)]
    u0 = inputs(og, *random_fields(*n, seed=21))
    return og, lg, src, u0


def _virtual_solve(lg, world, p, src, u0, rho, tail_mode="exp"):
    """Every rank's block on cuda:0, W summed on the device, finish on the root."""
    td = lg.torch_dtype()
    z = lambda: torch.zeros(3 * lg.npts, dtype=td, device="cuda:0")   # noqa: E731
    We, Wh = z(), z()
    v = (z(), z())
    roots, owned = set(), []
    tu0 = (to_dev(u0[0], lg), to_dev(u0[1], lg))
    for r in range(world):
        w = (z(), z())
        st = pe.solve_block(lg, r, world, NSTEPS, p, w, src, m=M_FIX, s=S_FIX, rho=rho, u0=tu0,
                            v=v, tail_mode=tail_mode)
        roots.add(st["root"])
        if st["first_interval"] >= 1:
            owned += list(range(st["first_interval"], st["last_interval"] + 1))
        We += w[0]
        Wh += w[1]
    assert len(roots) == 1
    if tail_mode != "exp_lpt":                 # contiguous blocks cover 1..p exactly once
        assert sorted(owned) == list(range(1, p + 1))
    eo, ho = z(), z()
    pe.solve_finish(lg, (We, Wh), v, eo, ho, rho=rho, tail_mode=tail_mode)
    torch.cuda.synchronize()
    return to_host(eo), to_host(ho)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("p", [2, 5, 8, 64])
def test_virtual_ranks_match_oracle(dtype, p):
    og, lg, src, u0 = _setup(dtype)
    rho = og.rho_cfl
    ref = fit.paraexp(og, src, 0.0, NSTEPS, p, lambda tau: fit.make_plan("leja", M_FIX, S_FIX, tau, rho),
                      u0=u0, rho=rho, dtype=dtype)
    for world in (1, 2, 3, 5, 8):
        got = _virtual_solve(lg, world, p, src, u0, rho)
        assert_parity(got, ref, dtype, f"world={world} p={p}")
        ee, eh = (np.abs(g - r).max() / np.abs(r).max() for g, r in zip(got, ref))
        assert ee <= 10 * TOL[dtype] and eh <= 10 * TOL[dtype], (world, p, ee, eh)   # max-abs


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("p", [5, 8])
def test_lpt_independent_tails_match_oracle(dtype, p):
    """Schedule (B): independent tails assigned longest-processing-time-first (tail_mode
    EXP_LPT) -- virtual ranks and the single-GPU solve against the oracle's independent-tail
    sum (a different association from Horner's)."""
    og, lg, src, u0 = _setup(dtype)
    rho = og.rho_cfl
    ref = fit.paraexp(og, src, 0.0, NSTEPS, p, lambda tau: fit.make_plan("leja", M_FIX, S_FIX, tau, rho),
                      u0=u0, rho=rho, dtype=dtype, sum_mode="independent")
    for world in (1, 2, 3, 8):
        got = _virtual_solve(lg, world, p, src, u0, rho, tail_mode="exp_lpt")
        assert_parity(got, ref, dtype, f"LPT world={world} p={p}")
    got = lib_solve(lg, NSTEPS, p, src, u0=u0, m=M_FIX, s=S_FIX, rho=rho, tail_mode="exp_lpt")
    assert_parity(got[:2], ref, dtype, f"LPT solve p={p}")
    assert got[2]["a_applications"] >= (p - 1) * p // 2 * M_FIX * S_FIX   # sum_j (p - j) propagators


def test_virtual_ranks_leapfrog_tails_equal_serial_leapfrog():
    """tail_mode LEAPFROG through the block/finish path equals serial leapfrog."""
    og, lg, src, u0 = _setup("f64")
    rho = og.rho_cfl
    h_half = fit.half_step_start(og, *u0)                   # reading 11
    ref = fit.leapfrog(og, u0[0], h_half, NSTEPS, src)
    for world, p in ((3, 8), (8, 5)):
        got = _virtual_solve(lg, world, p, src, u0, rho, tail_mode="leapfrog")
        assert_parity(got, ref, "f64", f"leapfrog tails world={world} p={p}")


def test_solve_equals_virtual_ranks():
    """paraexp_solve (one GPU) and the block/finish decomposition give the same fields."""
    og, lg, src, u0 = _setup("f64")
    rho = og.rho_cfl
    a = lib_solve(lg, NSTEPS, 8, src, u0=u0, m=M_FIX, s=S_FIX, rho=rho)
    b = _virtual_solve(lg, 4, 8, src, u0, rho)
    assert rel_l2(a[0], b[0]) <= 1e-13 and rel_l2(a[1], b[1]) <= 1e-13


def test_cost_balanced_blocks_in_solve_stats():
    og, lg, src, u0 = _setup("f64")
    rho = og.rho_cfl
    ratio = M_FIX * S_FIX / (NSTEPS // 64)
    for world in (2, 8):
        for r in range(world):
            w = tuple(torch.zeros(3 * lg.npts, dtype=torch.float64, device="cuda:0") for _ in range(2))
            st = pe.solve_block(lg, r, world, NSTEPS, 64, w, src, m=M_FIX, s=S_FIX, rho=rho)
            assert (st["first_interval"], st["last_interval"], st["root"]) == \
                pe.schedule(64, world, r, ratio, False)


# ---- two processes, gloo -------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, p, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        og, lg, src, u0 = _setup("f64")
        rho = og.rho_cfl
        z = lambda: torch.zeros(3 * lg.npts, dtype=torch.float64, device="cuda:0")   # noqa: E731
        w, v = (z(), z()), (z(), z())
        st = pe.solve_block(lg, rank, world, NSTEPS, p, w, src, m=M_FIX, s=S_FIX, rho=rho,
                            u0=(to_dev(u0[0], lg), to_dev(u0[1], lg)), v=v)
        buf = torch.cat([w[0], w[1]]).cpu()
        dist.reduce(buf, dst=st["root"], op=dist.ReduceOp.SUM)
        if rank == st["root"]:
            n = 3 * lg.npts
            W = (buf[:n].cuda(), buf[n:].cuda())
            eo, ho = z(), z()
            pe.solve_finish(lg, W, v, eo, ho, rho=rho)
            np.save(os.path.join(outdir, "out.npy"), torch.cat([eo, ho]).cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [3, 8])
def test_two_process_gloo_library(p, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_gloo_worker, args=(2, _free_port(), p, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "out.npy")
    og, lg, src, u0 = _setup("f64")
    rho = og.rho_cfl
    ref = fit.paraexp(og, src, 0.0, NSTEPS, p, lambda tau: fit.make_plan("leja", M_FIX, S_FIX, tau, rho),
                      u0=u0, rho=rho)
    n = 3 * og.Np
    assert_parity((got[:n], got[n:]), ref, "f64", f"gloo p={p}")


# ---- rho safety net --------------------------------------------------------------------------
NS = (20, 18, 16)


def _rho_setup():
    eps = np.random.default_rng(7).uniform(1, 4, int(np.prod(NS)))
    og = fit.Grid(*NS, d0=1e-3, eps_r=eps, dt_frac=0.95)
    lg = pe.Grid(*NS, d0=1e-3, eps_r=eps, dt_frac=0.95)
    return og, lg, fit.norm_A(og)


def test_rho_safety_net_expmv():
    og, lg, rho_true = _rho_setup()
    assert rho_true < 0.9 * og.rho_cfl
    e, h = inputs(og, *random_fields(*NS, seed=5))
    tau = 200 * og.dt
    # a 10% underestimate of ||A||_2: the spectrum leaves the Leja interval
    ge, gh, st = lib_expmv(lg, tau, e, h, rho=0.9 * rho_true, eps_A=1e-10, rho_check=1)
    assert st["rho_fallback"] == 1 and st["rho"] == og.rho_cfl
    plan = fit.make_plan("leja", st["m"], st["s_first"], tau, st["rho"])
    ref = fit.expmv(og, plan, e, h)
    assert_parity((ge, gh), ref, "f64", "expmv after the rho fallback")
    # without the net the same request is wrong (or overflows)
    try:
        be, bh, st2 = lib_expmv(lg, tau, e, h, rho=0.9 * rho_true, eps_A=1e-10, rho_check=-1)
        assert st2["rho_fallback"] == 0
        assert rel_l2(be, ref[0]) > 1e-6 or rel_l2(bh, ref[1]) > 1e-6
    except pe.ParaexpError as err:
        assert err.code == pe.EOVERFLOW
    # the K5 estimate (auto rho) passes the check without a fallback
    _, _, st3 = lib_expmv(lg, tau, e, h, eps_A=1e-10)
    assert st3["rho_fallback"] == 0 and st3["norm_deviation"] < 1e-8


def test_rho_safety_net_solve():
    og, lg, rho_true = _rho_setup()
    src = [gauss_sine(2, 9, 8, 7, f0=40e9, bw=40e9)]
    u0 = inputs(og, *random_fields(*NS, seed=6))
    nsteps, p = 240, 4
    ge, gh, st = lib_solve(lg, nsteps, p, src, u0=u0, rho=0.9 * rho_true, eps_A=1e-10, rho_check=1)
    assert st["rho_fallback"] == 1 and st["rho"] == og.rho_cfl and st["s_first"] == st["s_last"]
    ref = fit.paraexp(og, src, 0.0, nsteps, p,
                      lambda tau: fit.make_plan("leja", st["m"], st["s_first"], tau, st["rho"]),
                      u0=u0, rho=st["rho"])
    assert_parity((ge, gh), ref, "f64", "solve after the rho fallback")


# ---- debug NaN hook: the failing sub-interval is named ---------------------------------------
@pytest.mark.parametrize("concurrent", ["0", "1"])
@pytest.mark.parametrize("where,code", [("particular:3", pe.EDIVERGED), ("tail:4", pe.EOVERFLOW)])
def test_nan_hook_names_interval(monkeypatch, concurrent, where, code):
    og, lg, src, u0 = _setup("f64")
    monkeypatch.setenv("PARAEXP_CONCURRENT", concurrent)
    monkeypatch.setenv("PARAEXP_DEBUG_NAN", where)
    with pytest.raises(pe.ParaexpError) as ei:
        lib_solve(lg, 60, 6, src, u0=u0, m=M_FIX, s=S_FIX, rho=og.rho_cfl)
    assert ei.value.code == code
    assert ei.value.stats["fail_interval"] == int(where.split(":")[1])
    monkeypatch.delenv("PARAEXP_DEBUG_NAN")
    got = lib_solve(lg, 60, 6, src, u0=u0, m=M_FIX, s=S_FIX, rho=og.rho_cfl)   # grid still usable
    assert np.isfinite(got[0]).all()


# ---- stream order across calls on one grid ---------------------------------------------------
def test_calls_on_different_streams_are_ordered():
    og, lg, src, u0 = _setup("f64")
    e, h = u0
    ref_e, ref_h = fit.leapfrog(og, e, h, 50, src)
    ref = fit.expmv(og, fit.make_plan("leja", M_FIX, 3, 30 * og.dt, og.rho_cfl), ref_e, ref_h)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    te, th = to_dev(e, lg), to_dev(h, lg)
    torch.cuda.synchronize()
    pe.leapfrog(lg, te, th, 50, src, stream=s1.cuda_stream)
    # the second call, on another stream, must wait for the first one's workspace use; the
    # tensors themselves are ordered by the caller (as torch requires)
    s2.wait_stream(s1)
    pe.expmv(lg, 30 * og.dt, te, th, m=M_FIX, s=3, rho=og.rho_cfl, stream=s2.cuda_stream)
    torch.cuda.synchronize()
    assert_parity((to_host(te), to_host(th)), ref, "f64", "two streams")


def test_failed_block_reported_through_the_status_allreduce(monkeypatch):
    """With a communicator, the ranks all-reduce their blocks' status before the W reduce (a
    failed rank would otherwise leave its peers waiting in ncclReduce): a one-rank NCCL
    communicator with the collectives forced on still reports the divergence and its
    sub-interval, and the communicator stays usable."""
    og, lg, src, u0 = _setup("f64")
    monkeypatch.setenv("PARAEXP_FORCE_COLLECTIVES", "1")
    comm = pe.Comm(0, 1, 0, id_bytes=pe.Comm.unique_id())
    try:
        monkeypatch.setenv("PARAEXP_DEBUG_NAN", "particular:2")
        with pytest.raises(pe.ParaexpError) as ei:
            lib_solve(lg, 60, 6, src, u0=u0, m=M_FIX, s=S_FIX, rho=og.rho_cfl, comm=comm)
        assert ei.value.code == pe.EDIVERGED and ei.value.stats["fail_interval"] == 2
        monkeypatch.delenv("PARAEXP_DEBUG_NAN")
        got = lib_solve(lg, 60, 6, src, u0=u0, m=M_FIX, s=S_FIX, rho=og.rho_cfl, comm=comm)
        ref = fit.paraexp(og, src, 0.0, 60, 6, lambda tau: fit.make_plan("leja", M_FIX, S_FIX, tau, og.rho_cfl),
                          u0=u0, rho=og.rho_cfl)
        assert_parity(got[:2], ref, "f64", "after a failed solve")
    finally:
        comm.close()
