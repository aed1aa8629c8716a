"""GPU parity of the cooperative, shared-memory-resident leapfrog for mid-size grids (csrc/mid.cu):
one launch per leapfrog sequence, the state resident in the shared memory of up to one CTA per
SM, neighbour-only face exchange through tagged lines in L2 (the expmv and ParaExp parts of each
case run the TMA pair kernels beside it).  Every material
mode (scalar eps, z-table, per-edge eps with interior PEC, non-uniform mesh = per-face cH), ragged
box partitions, 1-cell-thick grids, long x rows and C2 itself, against the oracle at the
north_star tolerances (rel-L2 per field plus max-abs); the launch counts prove the mid path ran,
and repeated runs must be bit-identical (a race in the face exchange would not be)."""
import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from oracle import fit
from synth import config_c2, gauss_sine, layered_eps, random_fields
from gpu_util import assert_parity, inputs, lib_expmv, lib_leapfrog, lib_solve

pytestmark = pytest.mark.gpu


def _grid_kw(mode, n, seed=3):
    rng = np.random.default_rng(seed)
    nx, ny, nz = n
    if mode == "scalar":
        return dict(d0=1e-3)
    if mode == "ztable":
        return dict(d0=1e-3, eps_r=layered_eps(nx, ny, nz, (1.0, 2.2, 4.4, 9.8)))
    if mode == "edge":
        pec = np.zeros(nx * ny * nz, np.uint8)
        pec[rng.choice(nx * ny * nz, size=max(1, nx * ny * nz // 20), replace=False)] = 1
        return dict(d0=1e-3, eps_r=rng.uniform(1.0, 5.0, nx * ny * nz), pec_cell=pec)
    if mode == "nonuniform":
        return dict(dx=rng.uniform(0.5e-3, 1.5e-3, nx), dy=rng.uniform(0.5e-3, 1.5e-3, ny),
                    dz=rng.uniform(0.5e-3, 1.5e-3, nz), mu_r=rng.uniform(1.0, 2.0, nx * ny * nz))
    raise ValueError(mode)


CASES = [("scalar", (24, 20, 18), "f64"),
         ("ztable", (33, 17, 13), "f64"),       # ragged boxes in y and z
         ("edge", (20, 21, 19), "f64"),
         ("nonuniform", (19, 14, 12), "f64"),
         ("scalar", (200, 30, 1), "f64"),       # one cell thick in z
         ("ztable", (1000, 3, 4), "f64"),       # long x rows (one row per box)
         ("scalar", (40, 30, 20), "f32"),
         ("edge", (23, 19, 17), "f32"),
         ("nonuniform", (18, 16, 15), "f32"),
         ("ztable", (48, 40, 36), "f32")]


def run_case(mode, n, dtype, expect_mid=True, nsteps=60):
    kw = _grid_kw(mode, n)
    og = fit.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
    lg = pe.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
    e, h = inputs(og, *random_fields(*n, seed=7))
    ci = (n[0] // 2, n[1] // 2, n[2] // 2)
    src = [gauss_sine(2, *ci, f0=40e9, bw=40e9),
           gauss_sine(0, max(0, ci[0] - 1), ci[1], ci[2], f0=30e9, bw=30e9, amp=0.5),
           gauss_sine(1, ci[0], 0, ci[2], f0=30e9, bw=30e9, amp=0.7)]     # on the j = 0 box face
    src = [s for s in src if og.cE[og.edge_dof(s.comp, s.i, s.j, s.k)] != 0]
    ref = fit.leapfrog(og, e, h, nsteps, src)
    ge, gh, st = lib_leapfrog(lg, e, h, nsteps, src)
    assert_parity((ge, gh), ref, dtype, f"{mode} {n} {dtype} leapfrog")
    assert (st["kernel_launches"] < 10) == expect_mid, st
    ge2, gh2, _ = lib_leapfrog(lg, e, h, nsteps, src)
    assert np.array_equal(ge, ge2) and np.array_equal(gh, gh2), "leapfrog not bit-reproducible"
    rho = og.rho_cfl
    for m, s in ((150, 1), (40, 2), (1, 3)):
        plan = fit.make_plan("leja", m, s, 20 * og.dt, rho)
        r2 = fit.expmv(og, plan, e, h, dtype=dtype)
        ge, gh, st = lib_expmv(lg, 20 * og.dt, e, h, m=m, s=s, rho=rho)
        assert_parity((ge, gh), r2, dtype, f"{mode} {n} {dtype} expmv m={m} s={s}")
    r3 = fit.paraexp(og, src, 0.0, 48, 4, lambda tau: fit.make_plan("leja", 16, 2, tau, rho), u0=(e, h),
                     rho=rho, dtype=dtype)
    assert_parity(lib_solve(lg, 48, 4, src, u0=(e, h), m=16, s=2, rho=rho)[:2], r3, dtype,
                  f"{mode} {n} {dtype} solve")
    lg.close()


@pytest.mark.parametrize("mode,n,dtype", CASES)
def test_mid_parity(mode, n, dtype):
    run_case(mode, n, dtype)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mid_c2(dtype):
    """C2 itself (64^3, per-cell random eps, three sources): 200 leapfrog steps through the mid
    kernel and the bench plan's degree-148 substep against the oracle"""
    w = config_c2()
    og = fit.Grid.from_workload(w, dtype=dtype)
    lg = pe.Grid.from_workload(w, dtype=dtype)
    e, h = inputs(og, *random_fields(w.nx, w.ny, w.nz, seed=11))
    ref = fit.leapfrog(og, e, h, 200, w.sources)
    ge, gh, st = lib_leapfrog(lg, e, h, 200, w.sources)
    assert_parity((ge, gh), ref, dtype, f"C2 {dtype} leapfrog")
    assert st["kernel_launches"] < 10, st
    rho = og.rho_cfl
    tau = 300 * og.dt
    plan = fit.make_plan("leja", 148, 2, tau, rho)
    ge, gh, st = lib_expmv(lg, tau, e, h, m=148, s=2, rho=rho)
    assert_parity((ge, gh), fit.expmv(og, plan, e, h, dtype=dtype), dtype, f"C2 {dtype} expmv")
    lg.close()


def test_mid_vs_tma_same_grid():
    """the mid kernel and the TMA z-marching kernels (kernels="tma") agree on the same grid"""
    n = (32, 24, 20)
    kw = _grid_kw("edge", n)
    lm = pe.Grid(*n, dt_frac=0.95, **kw)
    lt = pe.Grid(*n, dt_frac=0.95, kernels="tma", **kw)
    og = fit.Grid(*n, dt_frac=0.95, **kw)
    e, h = inputs(og, *random_fields(*n, seed=5))
    a = lib_leapfrog(lm, e, h, 100, [])
    b = lib_leapfrog(lt, e, h, 100, [])
    assert a[2]["kernel_launches"] < 10 and b[2]["kernel_launches"] >= 100
    assert_parity(a[:2], b[:2], "f64", "mid vs tma leapfrog")
    lm.close()
    lt.close()


def test_mid_two_grids_concurrently():
    """Two grids stepped at the same time from two host threads on their own streams (each grid
    owns its exchange lines and tag counter; two cooperative launches may share the GPU): the
    results are bit-identical to the same runs one after the other."""
    import threading
    import torch
    shapes = [((48, 40, 36), "ztable", "f64"), ((40, 30, 20), "edge", "f32")]
    grids, fields = [], []
    for n, mode, dtype in shapes:
        kw = _grid_kw(mode, n)
        og = fit.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
        grids.append(pe.Grid(*n, dt_frac=0.95, dtype=dtype, **kw))
        fields.append(inputs(og, *random_fields(*n, seed=21)))
    src = [[gauss_sine(2, n[0] // 2, n[1] // 2, n[2] // 2, f0=40e9, bw=40e9)] for n, _, _ in shapes]
    seq = [lib_leapfrog(g, e, h, 800, s)[:2] for g, (e, h), s in zip(grids, fields, src)]
    out = [None, None]

    def run(q):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            e, h = fields[q]
            te = torch.tensor(e, dtype=grids[q].torch_dtype(), device="cuda:0")
            th = torch.tensor(h, dtype=grids[q].torch_dtype(), device="cuda:0")
            for _ in range(3):   # several calls: the tag counter advances per launch
                te.copy_(torch.tensor(e, dtype=grids[q].torch_dtype()))
                th.copy_(torch.tensor(h, dtype=grids[q].torch_dtype()))
                pe.leapfrog(grids[q], te, th, 800, src[q], stream=s.cuda_stream)
            s.synchronize()
            out[q] = (te.double().cpu().numpy(), th.double().cpu().numpy())

    ts = [threading.Thread(target=run, args=(q,)) for q in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for q in range(2):
        assert np.array_equal(out[q][0], seq[q][0]) and np.array_equal(out[q][1], seq[q][1]), q
    for g in grids:
        g.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mid_concurrent_sweeps_solve(dtype):
    """ParaExp on a mid-size refined grid (C3r 32^3, k = 10): the particular sweeps run as
    resident mid-kernel launches on SM partitions (one launch per sweep, not one per step),
    against Algorithm 1 in the oracle, with random u0 beside the source."""
    from synth import config_c3r
    w = config_c3r(k=10.0, n=32, dtype=dtype)
    og = fit.Grid.from_workload(w, dtype=dtype)
    lg = pe.Grid.from_workload(w, dtype=dtype)
    nsteps, p, m, s = 1600, 8, 32, 4
    rho = og.rho_cfl
    u0 = og.clean(*random_fields(w.nx, w.ny, w.nz, seed=12))
    got = lib_solve(lg, nsteps, p, w.sources, u0=u0, m=m, s=s, rho=rho)
    st = got[2]
    # 8 sweeps of 200 steps: far fewer launches than the 1600 steps (+ the pair launches)
    assert st["kernel_launches"] < nsteps, st
    ref = fit.paraexp(og, w.sources, 0.0, nsteps, p, lambda tau: fit.make_plan("leja", m, s, tau, rho),
                      u0=u0, rho=rho, dtype=dtype)
    assert_parity(got[:2], ref, dtype, f"C3r 32^3 {dtype} concurrent resident sweeps")
    lg.close()


def test_leapfrog_path_reported():
    """paraexp_grid_info_t.leapfrog_path names the kernels a leapfrog call runs: single-CTA
    (<= 2048 cells fp64), the mid-size resident kernel, the TMA kernels (large grids or
    kernels="tma"), unfused"""
    cases = [((16, 16, 8), "auto", pe.abi.PATH_SMALL), ((24, 20, 18), "auto", pe.abi.PATH_MID),
             ((24, 20, 18), "tma", pe.abi.PATH_TMA), ((24, 20, 18), "unfused", pe.abi.PATH_UNFUSED),
             ((128, 128, 64), "auto", pe.abi.PATH_TMA)]
    for n, kern, path in cases:
        g = pe.Grid(*n, d0=1e-3, dt_frac=0.95, kernels=kern)
        assert g.info()["leapfrog_path"] == path, (n, kern)
        g.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mid_leapfrog_trace(dtype):
    """f1 on a mid-size grid: the resident kernel's per-step energy (block reductions + one atomic
    per CTA per step) and probe values (owner threads) against the oracle's step-by-step trace,
    in ONE launch (per-edge eps with PEC cells)."""
    import torch
    from gpu_util import TOL, rel_l2, to_dev, to_host
    n = (33, 27, 21)
    kw = _grid_kw("edge", n)
    og = fit.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
    lg = pe.Grid(*n, dt_frac=0.95, dtype=dtype, **kw)
    assert lg.info()["leapfrog_path"] == pe.abi.PATH_MID
    e, h = inputs(og, *random_fields(*n, seed=31))
    src = [gauss_sine(2, 16, 13, 10, f0=40e9, bw=40e9)]
    src = [s for s in src if og.cE[og.edge_dof(s.comp, s.i, s.j, s.k)] != 0]
    probes = [(2, 16, 13, 10), (0, 5, 7, 3), (1, 30, 0, 20), (2, 1, 26, 0)]
    probes = [q for q in probes if og.cE[og.edge_dof(*q)] != 0]
    ref_e, ref_h, ref_en, ref_pr = fit.leapfrog_trace(og, e, h, 150, src, t0=1e-12, probes=probes)
    te, th = to_dev(e, lg), to_dev(h, lg)
    st, en, pr = pe.leapfrog_trace(lg, te, th, 150, src, 1e-12, probes=probes)
    torch.cuda.synchronize()
    assert st["kernel_launches"] < 10, st
    assert_parity((to_host(te), to_host(th)), (ref_e, ref_h), dtype, "mid trace fields")
    assert rel_l2(en.cpu().numpy(), ref_en) <= TOL[dtype]
    assert rel_l2(pr.cpu().numpy(), ref_pr) <= TOL[dtype]
    lg.close()
