"""Multi-rank ParaExp on CPU (world_size 2 and 3, torch.distributed gloo on 127.0.0.1).

Each rank takes its contiguous block from the library's host schedule (paraexp_schedule),
computes its share of Algorithm 1 with the oracle (particular sweeps + Horner tails carried
to T_p), the tails are summed with dist.reduce onto the root (the owner of sub-interval p,
as the library's ncclReduce does), and the root reconstructs.  The result must equal the
single-process ParaExp.  Also checks the 128-byte NCCL id broadcast used to create the
library's communicator (paraexp_comm_unique_id + torch.distributed)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1705_08019_b200 as pe
from oracle import fit
from synth import Source, gauss_sine, random_fields

N = (7, 6, 5)
NSTEPS = 37


def _setup():
    g = fit.Grid(*N, d0=1e-3, eps_r=np.random.default_rng(3).uniform(1, 4, np.prod(N)), dt_frac=0.9)
    src = [gauss_sine(2, 3, 3, 2, f0=80e9, bw=80e9), Source(0, 2, 2, 1, "gauss_paper", 0.5, 8e-12)]
    u0 = g.clean(*random_fields(*N, seed=11))
    rho = g.rho_cfl

    def plan_for(tau):
        return fit.make_plan("leja", 16, max(1, math.ceil(tau * rho / 8.0)), tau, rho)
    return g, src, u0, rho, plan_for


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, src, u0, rho, plan_for = _setup()
        first, last, root = pe.schedule(p, world, rank)
        W, P = fit.paraexp_block(g, src, 0.0, NSTEPS, p, plan_for, first, last, u0=u0)
        buf = torch.from_numpy(np.concatenate(W)).clone()
        dist.reduce(buf, dst=root, op=dist.ReduceOp.SUM)
        if rank == root:
            assert P is not None, "root must own sub-interval p"
            Wsum = buf.numpy()
            n = 3 * g.Np
            out = fit.paraexp_finish(g, P, (Wsum[:n], Wsum[n:]), rho)
            np.save(os.path.join(outdir, "out.npy"), np.concatenate(out))
        uid = pe.Comm.unique_id_via_torch(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(x == ids[0] for x in ids) and len(uid) == 128
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p", [(2, 2), (2, 5), (3, 4), (3, 2)])
def test_multirank_paraexp_equals_single_process(world, p, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), p, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "out.npy")
    g, src, u0, rho, plan_for = _setup()
    ref = np.concatenate(fit.paraexp(g, src, 0.0, NSTEPS, p, plan_for, u0=u0, rho=rho))
    n = 3 * g.Np
    for sl in (slice(0, n), slice(n, 2 * n)):
        assert np.linalg.norm(got[sl] - ref[sl]) <= 1e-12 * np.linalg.norm(ref[sl])


def test_block_partials_sum_to_full_w():
    """Sum over ranks of the block partial sums == W of the full Horner (any world size)."""
    g, src, u0, rho, plan_for = _setup()
    p = 5
    for world in (1, 2, 3, 5, 8):
        parts = []
        P = None
        for r in range(world):
            f, l, root = pe.schedule(p, world, r)
            W, Pr = fit.paraexp_block(g, src, 0.0, NSTEPS, p, plan_for, f, l, u0=u0)
            parts.append(W)
            if Pr is not None:
                P = Pr
        We = sum(w[0] for w in parts)
        Wh = sum(w[1] for w in parts)
        out = fit.paraexp_finish(g, P, (We, Wh), rho)
        ref = fit.paraexp(g, src, 0.0, NSTEPS, p, plan_for, u0=u0, rho=rho)
        for a, b in zip(out, ref):
            assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
