"""Host-side logic of the slab decomposition, on the CPU with 2-3 gloo ranks.

Each rank takes its slab from ``paper_2501_19013_b200.dist`` (partition,
owned DOF range, halo extents: p node rows above, one below), runs the
reference CDM loop (oracle arithmetic, CSR rows of the global operator) on its
owned rows only, and exchanges exactly the halo DOFs the device path
exchanges, over torch.distributed (gloo).  The result must be bitwise equal to
the serial oracle -- which proves the halo extents cover every stencil column
and the exchange pattern is right, independent of the GPU."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from dataclasses import replace


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm
    if kind == "2d":
        return build_scm(replace(CONFIGS["config2"], n_e=24, name="c2s"))
    return build_scm(replace(CONFIGS["config5"], p=2, n_e=8, n_random=3,
                             r_range=(0.05, 0.1), name="c5s"))


def _worker(rank, world, port, kind, n_t, out):
    import torch
    import torch.distributed as tdist
    from oracle import cpu
    from paper_2501_19013_b200.dist import SlabScm, partition
    from paper_2501_19013_b200.setup.configs import ricker
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    prob = _problem(kind)
    K = cpu.scm_csr(prob).tocsr()
    lo, hi = partition(prob, world)[rank]
    slab = SlabScm(prob, lo, hi)
    g = prob.grid
    p, n1, d = g.p, g.n_e * g.p + 1, g.dim
    per_row = n1 ** (d - 1)
    lex = g.dofmap.lex_of_compact
    top = (int(np.searchsorted(lex, max(lo * p - p, 0) * per_row)), slab.d_lo)
    bot = (slab.d_hi, int(np.searchsorted(lex, (hi * p + 1) * per_row)) if not slab.last
           else slab.d_hi)
    # every column of an owned row lies in owned + halo DOFs
    rows = K[slab.d_lo:slab.d_hi]
    cols = np.unique(rows.indices)
    assert cols.min() >= top[0] and cols.max() < bot[1]
    n = prob.n_dof
    dt = 2e-5
    psi = np.zeros(n)
    prev = np.zeros(n)
    f = lambda t: ricker(t, 10.0)
    own = slice(slab.d_lo, slab.d_hi)
    m, F = prob.m_diag, prob.F_s
    # bootstrap (src/timeint.py:175-176), psi0 = v0 = 0
    a0 = (f(0.0) * F[own] - rows @ psi) / m[own]
    prev[own] = psi[own] - dt * 0.0 + (0.5 * dt * dt) * a0

    def exchange(x):
        reqs = []
        if rank > 0:   # p rows above <- previous slab; our first node row -> it
            first_row_end = int(np.searchsorted(lex, (lo * p + 1) * per_row))
            buf = torch.from_numpy(x[top[0]:top[1]].copy())
            reqs.append(("recv", tdist.irecv(buf, src=rank - 1), buf, top))
            reqs.append(("send", tdist.isend(torch.from_numpy(x[slab.d_lo:first_row_end].copy()),
                                             dst=rank - 1), None, None))
        if not slab.last:  # last p rows -> next slab; its first row -> our bottom halo
            last_rows_lo = int(np.searchsorted(lex, (hi * p - p) * per_row))
            reqs.append(("send", tdist.isend(torch.from_numpy(x[last_rows_lo:slab.d_hi].copy()),
                                             dst=rank + 1), None, None))
            buf = torch.from_numpy(x[bot[0]:bot[1]].copy())
            reqs.append(("recv", tdist.irecv(buf, src=rank + 1), buf, bot))
        for kind_, req, buf, rng in reqs:
            req.wait()
            if kind_ == "recv":
                x[rng[0]:rng[1]] = buf.numpy()

    for k in range(n_t):
        rhs = f(k * dt) * F[own] - rows @ psi
        new = 2.0 * psi[own] - prev[own] + (dt * dt) * (rhs / m[own])
        prev[own] = psi[own]
        psi[own] = new
        exchange(psi)
    out[rank] = psi[own].copy()
    tdist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("2d", 2), ("2d", 3), ("3d", 2)])
def test_slab_halo_exchange_reproduces_serial_cdm(kind, world):
    import torch.multiprocessing as mp
    from oracle import cpu, timeint as O
    from paper_2501_19013_b200.setup.configs import ricker
    prob = _problem(kind)
    n_t = 40
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, kind, n_t, out), nprocs=world, join=True)
    psi = np.concatenate([out[r] for r in range(world)])
    K = cpu.scm_csr(prob)
    ref, _, _ = O.cdm_run(sp.diags(prob.m_diag).tocsr(), K, prob.F_s,
                          lambda t: ricker(t, 10.0), 2e-5, n_t)
    assert np.array_equal(psi, ref)


def test_imex_slab_host_sets():
    """Slab c/d sets and DOF maps of the plane-strain IMEX partition (host only)."""
    from paper_2501_19013_b200.dist import SlabElastic, partition_imex
    from paper_2501_19013_b200.setup.elastic import ElasticProblem, lame
    from paper_2501_19013_b200.setup.geometry import BallVoids
    from paper_2501_19013_b200.setup.grid import Grid
    lam, mu = lame(1.0, 0.3)
    geom = BallVoids(2, [[0.22, 0.5], [0.7, 0.3]], [0.08, 0.09])
    prob = ElasticProblem.build(Grid.build(geom, "lagrange", 2, 20), lam, mu, 1e-4, 2)
    prob.set_point_source([0.1, 0.9])
    parts = partition_imex(prob, 3)
    assert parts[0][0] == 0 and parts[-1][1] == 20
    slabs = [SlabElastic(prob, lo, hi) for lo, hi in parts]
    g = np.concatenate([s.gdofs for s in slabs])
    assert np.array_equal(np.sort(g), np.arange(prob.n_dof))
    c_all = np.sort(np.concatenate([s.gdofs[s.c_idx] for s in slabs]))
    assert np.array_equal(c_all, np.sort(prob.c_idx))
    for s in slabs:
        assert s.c_idx.shape[0] + s.d_idx.shape[0] == s.n
        assert s.M[s.d_idx][:, s.c_idx].nnz == 0
