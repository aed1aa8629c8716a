"""CPU tests of the C-ABI library: it loads, exports every symbol include/paraexp.h declares,
and its host-side logic (partition, schedule, Leja nodes, Newton coefficients, theta_m,
coefficient assembly, CFL, material-mode detection, argument validation) agrees with the
oracle / the paper's worked examples.  No GPU compute is called."""
import json
import math
import os
import re

import numpy as np
import pytest

import paper_1705_08019_b200 as pe
from paper_1705_08019_b200 import abi
from oracle import fit
from synth import config_c1, config_c2, config_c3, layered_eps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_values.json")))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "paraexp.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|double|const char \*)\s*\**(paraexp_\w+)\s*\(",
                              hdr, flags=re.M))
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(abi.lib, name), name
    assert declared == set(abi.EXPORTED)


def test_host_alloc_argument_checks():
    """paraexp_host_alloc validates its arguments before touching the driver; without a GPU
    the allocation itself fails loudly (ECUDA / ENOMEM) and leaves *out NULL; free(NULL) is a
    no-op."""
    import ctypes as C
    h = C.c_void_p(1234)
    assert abi.lib.paraexp_host_alloc(0, C.byref(h)) == pe.EINVAL
    assert abi.lib.paraexp_host_alloc(64, None) == pe.EINVAL
    rc = abi.lib.paraexp_host_alloc(4096, C.byref(h))
    if rc == 0:                       # a driver is present
        assert h.value
        abi.lib.paraexp_host_free(h)
    else:
        assert rc in (abi.ECUDA, abi.ENOMEM) and not h.value
        assert b"paraexp_host_alloc" in abi.lib.paraexp_last_error()
    abi.lib.paraexp_host_free(None)


def test_partition_and_schedule():
    ex = GOLD["partition_example"]
    b = pe.partition(ex["nsteps"], ex["p"])
    assert [y - x for x, y in zip(b[:-1], b[1:])] == ex["steps"]
    with pytest.raises(pe.ParaexpError):
        pe.partition(3, 4)
    for p in [1, 2, 3, 8, 16, 64]:
        for world in [1, 2, 3, 4, 8]:
            owned = []
            roots = set()
            for r in range(world):
                f, l, root = pe.schedule(p, world, r)
                owned += list(range(f, l + 1)) if f >= 1 else []
                roots.add(root)
                if f >= 1 and l == p:
                    assert root == r
            assert sorted(owned) == list(range(1, p + 1))   # every sub-interval exactly once
            assert len(roots) == 1


def _makespan(blocks, p, ratio, u0):
    return max((l - f + 1) + (p - f) * ratio + (ratio if (f == 1 and u0) else 0.0)
               for f, l in blocks if f >= 1)


def _brute_optimum(p, world, ratio, u0):
    """min over every split of 1..p into at most `world` contiguous non-empty blocks."""
    import itertools
    best = math.inf
    for k in range(1, min(p, world) + 1):
        for cuts in itertools.combinations(range(2, p + 1), k - 1):
            starts = (1,) + cuts
            blocks = [(f, (starts[q + 1] - 1 if q + 1 < k else p)) for q, f in enumerate(starts)]
            best = min(best, _makespan(blocks, p, ratio, u0))
    return best


@pytest.mark.parametrize("ratio", [0.5, 1.0, 3.0, 7.25])
@pytest.mark.parametrize("u0", [False, True])
def test_cost_balanced_schedule_is_optimal(ratio, u0):
    """paraexp_schedule with a tail ratio: contiguous blocks in rank order that
    cover 1..p exactly once, the root owns p, and the largest rank cost equals the brute-force
    optimum over all contiguous splits (never above the equal-share split)."""
    for p in (1, 2, 3, 5, 8, 11):
        for world in (1, 2, 3, 4, 8):
            blocks, roots = [], set()
            for r in range(world):
                f, l, root = pe.schedule(p, world, r, ratio, u0)
                roots.add(root)
                if f >= 1:
                    blocks.append((f, l))
                    if l == p:
                        assert root == r
                else:
                    assert l == -1
            assert len(roots) == 1
            cover = [j for f, l in blocks for j in range(f, l + 1)]
            assert cover == list(range(1, p + 1))              # contiguous, in rank order
            ms = _makespan(blocks, p, ratio, u0)
            assert abs(ms - _brute_optimum(p, world, ratio, u0)) < 1e-9, (p, world, blocks)
            eq = [pe.schedule(p, world, r) for r in range(world)]
            assert ms <= _makespan([(f, l) for f, l, _ in eq if f >= 1], p, ratio, u0) + 1e-9


@pytest.mark.parametrize("ratio", [0.5, 2.6, 16.0])
@pytest.mark.parametrize("u0", [False, True])
def test_lpt_schedule(ratio, u0):
    """Schedule (B) (paraexp_schedule_lpt): every job exactly once, the root owns
    sub-interval p, and the makespan obeys Graham's LPT bound (4/3 - 1/(3 world)) x the lower
    bound max(total / world, largest job)."""
    for p in (1, 2, 5, 8, 17, 64):
        for world in (1, 2, 3, 8):
            owner, root = pe.schedule_lpt(p, world, ratio, u0)
            assert len(owner) == p + 1 and root == owner[p]
            assert (owner[0] == -1) != u0 and all(0 <= o < world for o in owner[1:])
            cost = {j: 1.0 + (p - j) * ratio for j in range(1, p + 1)}
            if u0:
                cost[0] = p * ratio
            load = [0.0] * world
            for j, c in cost.items():
                load[owner[j]] += c
            lb = max(sum(cost.values()) / world, max(cost.values()))
            assert max(load) <= (4.0 / 3.0 - 1.0 / (3 * world)) * lb + 1e-9, (p, world, load, lb)


def test_leja_points_match_oracle():
    assert pe.leja_points(101) == list(fit.leja_points(101))


@pytest.mark.parametrize("m,theta", [(8, 3.0), (40, 30.0), (64, 55.0), (100, 90.0)])
def test_newton_coefficients_match_oracle(m, theta):
    """d-hat_k by the bidiagonal exponential (library) == mpmath divided differences (oracle)."""
    p = pe.plan_host("leja", m, 1, 1e-12, theta, 1.0)
    o = fit.make_plan("leja", m, 1, theta, 1.0)
    assert p["gamma"] == o.gamma and p["a"] == o.a
    d = np.array(p["d"])
    do = np.array(o.d)
    assert np.abs(d - do).max() <= 1e-15 * max(1.0, np.abs(do).max())


def test_taylor_coefficients():
    p = pe.plan_host("taylor", 24, 2, 1e-12, 1.0, 1.0)
    assert all(abs(p["d"][k] - 1.0 / math.factorial(k)) <= 2.3e-16 / math.factorial(k) for k in range(25))
    assert p["gamma"] == 1.0


@pytest.mark.parametrize("method,m,tol", [("leja", 32, 1e-8), ("leja", 64, 1e-13), ("taylor", 24, 1e-10)])
def test_theta_matches_oracle(method, m, tol):
    assert abs(pe.theta(method, m, tol) - fit.theta_m(method, m, tol)) <= 1e-9 * fit.theta_m(method, m, tol)


def test_theta_reference_table():
    """Regression against the theta table of SURVEY 8(c) (~1%; the oracle's theta_m is pinned in
    tests/test_oracle_theta.py and compared with the library above)."""
    ref = {(16, 1e-2): 11.9, (64, 1e-8): 41.3, (100, 1e-13): 61.1, (48, 1e-8): 27.9}
    for (m, tol), v in ref.items():
        assert abs(pe.theta("leja", m, tol) / v - 1) < 0.01


@pytest.mark.parametrize("tr", [300.0, 121.6])
def test_auto_plan_minimises_cost(tr):
    """The auto plan (reading 16) satisfies the criterion (s theta_m >= tau rho), is minimal in
    m at its s, and costs no more A-applications than any degree of a coarse reference list."""
    tau, tol = 1.0, 1e-10
    p = pe.plan_host("leja", 0, 0, tol, tau, tr)
    m, s_ = p["m"], p["s"]
    assert m % 2 == 0 and 8 <= m <= 150
    assert s_ * pe.theta("leja", m, tol) >= tau * tr
    assert m == 8 or s_ * pe.theta("leja", m - 2, tol) < tau * tr
    best = min(mm * max(1, math.ceil(tau * tr / pe.theta("leja", mm, tol)))
               for mm in [8, 12, 16, 20, 24, 32, 40, 48, 56, 64, 72, 80, 88, 100, 120, 150])
    assert m * s_ <= best


@pytest.mark.parametrize("wl", ["c1", "c3small", "random", "pec"])
def test_host_grid_coefficients_match_oracle(wl):
    n = (8, 8, 8)
    eps = pec = None
    if wl == "c3small":
        n = (12, 10, 16)
        eps = layered_eps(*n)
    elif wl == "random":
        n = (9, 7, 6)
        eps = np.random.default_rng(1).uniform(1, 4, np.prod(n))
    elif wl == "pec":
        n = (9, 7, 6)
        pec = (np.random.default_rng(2).uniform(size=np.prod(n)) < 0.1).astype(np.uint8)
    lg = pe.Grid(*n, d0=1e-3, eps_r=eps, pec_cell=pec, dt_frac=0.95, device=-1)
    og = fit.Grid(*n, d0=1e-3, eps_r=eps, pec_cell=pec, dt_frac=0.95)
    cE, cH = lg.coefficients()
    assert np.array_equal(cE != 0, og.cE != 0) and np.array_equal(cH != 0, og.cH != 0)
    np.testing.assert_allclose(cE, og.cE, rtol=1e-14, atol=0)
    np.testing.assert_allclose(cH, og.cH, rtol=1e-14, atol=0)
    assert abs(lg.dt_cfl - og.dt_cfl) <= 1e-15 * og.dt_cfl
    mode = lg.info()["material_mode"]
    assert mode == {"c1": abi.MAT_SCALAR, "c3small": abi.MAT_ZTABLE, "random": abi.MAT_ARRAY,
                    "pec": abi.MAT_ARRAY}[wl]


def test_config_material_modes():
    for w, mode in [(config_c1(), abi.MAT_SCALAR), (config_c2(nsteps=10), abi.MAT_ARRAY),
                    (config_c3(n=32), abi.MAT_ZTABLE)]:
        lg = pe.Grid.from_workload(w, device=-1)
        assert lg.info()["material_mode"] == mode


def test_grid_validation_host():
    for kw in [dict(nx=0), dict(eps_r=np.zeros(64)), dict(dt=1e-12), dict(dt_frac=0.0)]:
        args = dict(nx=4, ny=4, nz=4, d0=1e-3, dt_frac=0.9, device=-1)
        args.update(kw)
        with pytest.raises(pe.ParaexpError) as ei:
            pe.Grid(**args)
        assert ei.value.code == pe.EINVAL
    g = pe.Grid(4, 4, 4, d0=1e-3, dt_frac=1.2, device=-1)
    assert g.warnings == abi.WCFL


def test_host_only_grid_has_no_compute():
    g = pe.Grid(4, 4, 4, d0=1e-3, dt_frac=0.9, device=-1)
    st = abi.paraexp_stats()
    rc = abi.lib.paraexp_leapfrog(g.handle, None, 0, 0.0, 1, abi.C.c_void_p(8), abi.C.c_void_p(8),
                                  0, None, abi.C.byref(st))
    assert rc == pe.ENOTSUP


def test_optimal_tolerance_spec_examples():
    """eq:tolerance_leja_2 through the library's host helper: SPEC's worked
    examples (beta = 1, dt = 1e-9, ||A|| = 1e9 -> 1e-27 clamped to the 1e-14 floor; quadrupling
    dt multiplies eps* by 16; halving ||A|| doubles it)."""
    import paper_1705_08019_b200 as pe
    v, cl = pe.optimal_tolerance(1e-9, 1.0, 1e9)
    assert v == 1e-14 and cl
    a, _ = pe.optimal_tolerance(1e-12, 1e30, 1e12)
    b, _ = pe.optimal_tolerance(4e-12, 1e30, 1e12)
    c, _ = pe.optimal_tolerance(1e-12, 1e30, 0.5e12)
    assert abs(a - 1e-6) < 1e-20 and abs(b / a - 16) < 1e-12 and abs(c / a - 2) < 1e-12


def test_c_example_compiles_and_links(tmp_path):
    """The ABI is plain C: examples/cavity_solve.c (no Python, no CUDA headers) compiles with
    gcc -std=c11 against include/paraexp.h and links against libparaexp.so."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1705_08019_b200")
    exe = tmp_path / "cavity_solve"
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "cavity_solve.c"), "-L", libdir,
                           "-l:libparaexp.so", f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)])
    assert exe.exists()


def test_leapfrog_path_host_only_grid():
    """paraexp_grid_info_t.leapfrog_path is -1 on a host-only grid (no device to decide on)"""
    g = pe.Grid(8, 8, 8, d0=1e-3, dt_frac=0.9, device=-1)
    info = g.info()
    assert info["leapfrog_path"] == -1 and info["kernels"] == pe.abi.KERNELS_FUSED
    g.close()
