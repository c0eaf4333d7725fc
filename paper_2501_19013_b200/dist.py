"""Slab decomposition of spectral-cell systems across GPUs.

The grid is cut into slabs of cell rows along x -- the slowest axis of the
reference's DOF numbering (src/assembly.py:85-89) -- so every slab owns a
contiguous range of the global compact DOF numbering.  Slab r owns cell rows
[lo, hi) and node rows [lo*p, hi*p) (the last slab also node row n_e*p).  Per
time step each slab needs, besides its own nodes, the p node rows above
(to recompute the cell row above its first row, whose bottom row it shares)
and the one node row below (the bottom row of its last cell row): p rows
travel to the next slab and one row to the previous slab.  Interface values
are therefore computed redundantly from identical data in a fixed order -- the
sharded run is bitwise identical to the single-GPU run.

* :func:`partition` -- balanced cell-row ranges (by owned DOFs);
* :class:`SlabScm` -- the local operator description of one slab;
* :func:`group_cdm_run` -- all slabs in one process on one GPU (emulated
  ranks, device-copy halos): the same kernels and halo layout;
* :func:`dist_cdm_run` -- one slab per process under torchrun, halos over
  NCCL (grouped send/recv on the library's stream).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _lib
from .timeint import DivergenceError, RunResult, StageTimings, force_table


def partition(prob, world: int):
    """Cell-row ranges [(lo, hi), ...] with about equal owned DOFs."""
    g = prob.grid
    p, n_e, d = g.p, g.n_e, g.dim
    n1 = n_e * p + 1
    per_row = n1 ** (d - 1)
    lex = g.dofmap.lex_of_compact
    node_row = lex // per_row
    counts = np.bincount(node_row, minlength=n1)            # DOFs per node row
    cell_counts = np.add.reduceat(counts[: n_e * p], np.arange(0, n_e * p, p))
    cell_counts[-1] += counts[n_e * p]
    cum = np.cumsum(cell_counts)
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(cum, total * r / world))
        cuts.append(max(cuts[-1] + 1, min(c, n_e - (world - r))))
    cuts.append(n_e)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


class SlabScm:
    """Slab [lo, hi) of an ScmProblem: owned DOF range and local arrays."""

    def __init__(self, prob, lo: int, hi: int):
        g = prob.grid
        self.prob, self.lo, self.hi = prob, int(lo), int(hi)
        p, n_e, d = g.p, g.n_e, g.dim
        n1 = n_e * p + 1
        self.last = self.hi == n_e
        per_row = n1 ** (d - 1)
        lex = g.dofmap.lex_of_compact
        row_end = self.hi * p + (1 if self.last else 0)
        self.d_lo = int(np.searchsorted(lex, self.lo * p * per_row))
        self.d_hi = int(np.searchsorted(lex, row_end * per_row))
        cells_row = n_e ** (d - 1)
        first = self.lo - 1 if self.lo > 0 else 0
        self.cell_class = np.ascontiguousarray(
            g.classes.reshape(n_e, cells_row)[first:self.hi].ravel(), dtype=np.int8)
        cut = g.cut_lex
        crow = cut // cells_row
        sel = np.flatnonzero((crow >= self.lo - 1) & (crow < self.hi))
        self.cut_cells = np.ascontiguousarray(cut[sel])
        self.cut_K = np.ascontiguousarray(prob.cut_K[sel])
        self.lex = np.ascontiguousarray(lex[self.d_lo:self.d_hi])
        self.m = np.ascontiguousarray(prob.m_diag[self.d_lo:self.d_hi])
        self.F = np.ascontiguousarray(prob.F_s[self.d_lo:self.d_hi]) if prob.F_s is not None \
            else np.zeros(self.d_hi - self.d_lo)
        self.obs = (sp.csr_matrix(prob.obs_mat)[:, self.d_lo:self.d_hi]
                    if prob.obs_mat is not None else None)

    @property
    def n(self) -> int:
        return self.d_hi - self.d_lo

    def device_operator(self, device=None):
        from .operators import ScmOperator
        g = self.prob.grid
        return ScmOperator(dim=g.dim, p=g.p, n_e=(g.n_e,) * g.dim, k1=self.prob.k1,
                           m1=self.prob.m1, sk=self.prob.sk, cell_class=self.cell_class,
                           lex_of_compact=self.lex, cut_cells=self.cut_cells, cut_K=self.cut_K,
                           device=device, slab=(self.lo, self.hi, self.last))

    def halo(self, op) -> tuple:
        out = np.zeros(8, dtype=np.int64)
        _lib.load().wcb_operator_halo(op.handle, _lib.i64ptr(out))
        return tuple(int(v) for v in out)


def group_cdm_run(prob, f_t, dt: float, n_t: int, world: int, device=None) -> RunResult:
    """CDM over `world` slabs emulated in one process on one GPU (the halo
    exchange is a device copy); returns the global field and observers."""
    from .timeint import CdmPlan
    parts = partition(prob, world)
    slabs = [SlabScm(prob, lo, hi) for lo, hi in parts]
    ops = [s.device_operator(device=device) for s in slabs]
    plans = [CdmPlan(sp.diags(s.m).tocsr(), op, s.F, obs_mat=s.obs, device=device)
             for s, op in zip(slabs, ops)]
    n_t = int(n_t)
    ft = force_table(f_t, float(dt), n_t)
    outs = [np.empty(max(s.n, 1)) for s in slabs]
    lib = _lib.load()
    parr = (_lib.C.c_void_p * world)(*[pl.handle.value for pl in plans])
    oarr = (_lib.C.POINTER(_lib.C.c_double) * world)(*[_lib.dptr(o) for o in outs])
    n_obs = plans[0].n_obs
    obs = np.empty((n_obs, n_t + 1)) if n_obs else None
    div = _lib.Divergence()
    tm = _lib.Timings()
    code = lib.wcb_cdm_group_run(world, parr, _lib.dptr(ft), float(dt), n_t, oarr,
                                 _lib.dptr(obs) if obs is not None else None,
                                 _lib.C.byref(div), _lib.C.byref(tm))
    if code == _lib.WCB_E_DIVERGED:
        raise DivergenceError(int(div.step), float(div.amplitude))
    _lib.check(code)
    psi = np.concatenate([o[:s.n] for o, s in zip(outs, slabs)])
    return RunResult(method="cdm", dt=float(dt), t=np.arange(n_t + 1) * float(dt), obs=obs,
                     psi=psi, psi_dot=None, timings=StageTimings(rhs=float(tm.rhs)), fact_dim=0)


def init_nccl(ctx, rank: int, world: int):
    """Create the library's NCCL communicator (unique id broadcast over the
    default torch.distributed group)."""
    import torch.distributed as tdist
    lib = _lib.load()
    buf = _lib.C.create_string_buffer(128)
    if rank == 0:
        _lib.check(lib.wcb_dist_unique_id(buf))
    obj = [bytes(buf.raw) if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0)
    _lib.check(lib.wcb_dist_init(ctx.handle, rank, world, obj[0]))


def dist_cdm_run(prob, f_t, dt: float, n_t: int, device=None, gather: bool = True):
    """One slab per torchrun rank; halos over NCCL.  Returns this rank's
    (slab, RunResult of owned DOFs) and, on rank 0 when gather=True, the
    global field."""
    import torch.distributed as tdist
    from .timeint import CdmPlan
    rank, world = tdist.get_rank(), tdist.get_world_size()
    ctx = _lib.context(device)
    if not getattr(ctx, "_nccl", False):
        init_nccl(ctx, rank, world)
        ctx._nccl = True
    lo, hi = partition(prob, world)[rank]
    slab = SlabScm(prob, lo, hi)
    op = slab.device_operator(device=device)
    plan = CdmPlan(sp.diags(slab.m).tocsr(), op, slab.F, obs_mat=slab.obs, device=device)
    res = plan.run(f_t, dt, n_t)
    full = None
    if gather:
        pieces = [None] * world if rank == 0 else None
        tdist.gather_object(res.psi, pieces, dst=0)
        if rank == 0:
            full = np.concatenate(pieces)
    return slab, res, full


# --------------------------------------------------------------------------
# Plane-strain IMEX (BASELINE config 4) over x slabs.  The c set is a union of
# independent patches (the nodes of the cut cells around each void); a slab
# cut at cell row c is admissible when cell rows c-2, c-1 and c hold no cut
# cell, so every patch, every cell touching a patch node, and hence every c
# row of K lie inside one slab's owned rows.  The explicit d step is the slab kernel of the CDM
# path (p halo rows above, one below, exchanged once per step after the
# corrector); the c predictor / solve / corrector are slab-local.  Each slab
# factorises its own S_cc and M_cc blocks with SuperLU in the reference
# configuration (a block of independent patches: the same matrices, a
# per-slab ordering), so sharded fields agree with the single-GPU run to
# rounding (tested at 1e-12), not bitwise.

def partition_imex(prob, world: int):
    """Balanced cell-row ranges whose cuts avoid cut cells (see above)."""
    g = prob.grid
    n_e = g.n_e
    cut_rows = np.zeros(n_e, dtype=bool)
    cut_rows[np.asarray(g.cut_lex, dtype=np.int64) // n_e] = True
    # cut c admissible: no cut cell in rows c-2, c-1 (the upper slab's c rows
    # then never reach its bottom halo row c*p) nor in row c (the lower
    # slab's c rows never reach the cell row it recomputes from its top halo)
    ok = np.zeros(n_e + 1, dtype=bool)
    for c in range(2, n_e):
        ok[c] = not (cut_rows[c - 2] or cut_rows[c - 1] or cut_rows[c])
    # admissible cuts are scarce (config 4: 120 of 1024 rows, none between rows
    # 651 and 980), so the cuts are chosen by dynamic programming: smallest
    # largest slab, then smallest sum of squared sizes
    cand = [0] + [int(c) for c in np.flatnonzero(ok)] + [n_e]
    m = len(cand)
    INF = (float("inf"), float("inf"))
    # best[k][i]: (max size, sum of squares) of rows cand[i]..n_e split into k slabs
    best = [[INF] * m for _ in range(world + 1)]
    nxt = [[-1] * m for _ in range(world + 1)]
    for i in range(m - 1):
        sz = cand[-1] - cand[i]
        best[1][i] = (sz, sz * sz)
    for k in range(2, world + 1):
        for i in range(m - k):
            for j in range(i + 1, m - k + 1):
                tail = best[k - 1][j]
                if tail == INF:
                    continue
                sz = cand[j] - cand[i]
                v = (max(sz, tail[0]), sz * sz + tail[1])
                if v < best[k][i]:
                    best[k][i] = v
                    nxt[k][i] = j
    if world > m - 1 or best[world][0] == INF:
        raise ValueError(f"cannot cut {n_e} cell rows into {world} admissible slabs")
    cuts, i = [0], 0
    for k in range(world, 1, -1):
        i = nxt[k][i]
        cuts.append(cand[i])
    cuts.append(n_e)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


class _SlabBlockK:
    """Stiffness blocks of a slab's DOFs from the global problem (ImexPlan's
    K_cc source when the global CSR does not fit host memory)."""

    def __init__(self, prob, gdofs):
        self.prob, self.gdofs = prob, gdofs

    def stiffness_block(self, idx):
        return self.prob.stiffness_block(self.gdofs[np.asarray(idx, dtype=np.int64)])


class SlabElastic:
    """Slab [lo, hi) of an ElasticProblem: local DOFs (component major), mass,
    load, observers, c/d sets and the slab operator."""

    def __init__(self, prob, lo: int, hi: int, M=None):
        g = prob.grid
        self.prob, self.lo, self.hi = prob, int(lo), int(hi)
        p, n_e = g.p, g.n_e
        n1 = n_e * p + 1
        self.last = self.hi == n_e
        lex = g.dofmap.lex_of_compact
        row_end = self.hi * p + (1 if self.last else 0)
        self.d_lo = int(np.searchsorted(lex, self.lo * p * n1))
        self.d_hi = int(np.searchsorted(lex, row_end * n1))
        nn = prob.n_node
        nodes = np.arange(self.d_lo, self.d_hi, dtype=np.int64)
        self.gdofs = np.concatenate([nodes, nodes + nn])         # local dof -> global dof
        self.n_node_local = nodes.shape[0]
        first = self.lo - 1 if self.lo > 0 else 0
        self.cell_class = np.ascontiguousarray(g.classes.reshape(n_e, n_e)[first:self.hi].ravel(),
                                               dtype=np.int8)
        cut = np.asarray(g.cut_lex, dtype=np.int64)
        crow = cut // n_e
        sel = np.flatnonzero((crow >= self.lo - 1) & (crow < self.hi))
        self.cut_cells = np.ascontiguousarray(cut[sel])
        self.cut_K = np.ascontiguousarray(prob.cut_K[sel])
        self.lex = np.ascontiguousarray(lex[self.d_lo:self.d_hi])
        M = prob.mass_matrix() if M is None else M
        self.M = sp.csr_matrix(M)[self.gdofs][:, self.gdofs]
        self.F = np.ascontiguousarray(prob.F_s[self.gdofs])
        self.obs = (sp.csr_matrix(prob.obs_mat)[:, self.gdofs] if prob.obs_mat is not None else None)
        loc = np.full(prob.n_dof, -1, dtype=np.int64)
        loc[self.gdofs] = np.arange(self.gdofs.shape[0])
        c = loc[prob.c_idx]
        self.c_idx = np.sort(c[c >= 0])
        d = loc[prob.d_idx]
        self.d_idx = np.sort(d[d >= 0])

    @property
    def n(self) -> int:
        return self.gdofs.shape[0]

    def device_operator(self, device=None):
        from .operators import ElasticOperator
        g, pr = self.prob.grid, self.prob
        op = ElasticOperator(p=g.p, n_e=g.n_e, lam=pr.lam, mu=pr.mu, m1=pr.m1, k1=pr.k1, g1=pr.g1,
                             cell_class=self.cell_class, lex_of_compact=self.lex,
                             cut_cells=self.cut_cells, cut_K=self.cut_K, device=device,
                             slab=(self.lo, self.hi, self.last))
        op.problem = _SlabBlockK(self.prob, self.gdofs)
        return op

    def plan(self, dt: float, beta: float = 0.25, device=None):
        from .imex import ImexPlan
        return ImexPlan(self.M, self.device_operator(device=device), self.F, dt, self.c_idx, self.d_idx,
                        obs_mat=self.obs, beta=beta, device=device)


def _imex_tables(f_t, dt: float, n_t: int):
    f0 = float(f_t(0.0))
    ft_k = np.array([float(f_t(k * dt)) for k in range(n_t)] or [0.0])
    ft_new = np.array([float(f_t(k * dt + dt)) for k in range(n_t)] or [0.0])
    return f0, ft_k, ft_new


def group_imex_run(prob, f_t, dt: float, n_t: int, world: int, beta: float = 0.25,
                   gamma: float = 0.5, device=None) -> RunResult:
    """imex_run over `world` slabs emulated in one process on one GPU (halo
    exchange by device copies); returns the global field and observers."""
    parts = partition_imex(prob, world)
    M = prob.mass_matrix()
    slabs = [SlabElastic(prob, lo, hi, M=M) for lo, hi in parts]
    plans = [s.plan(dt, beta=beta, device=device) for s in slabs]
    n_t = int(n_t)
    f0, ft_k, ft_new = _imex_tables(f_t, float(dt), n_t)
    outs = [np.empty(max(s.n, 1)) for s in slabs]
    n_obs = plans[0].n_obs
    obs_parts = [np.zeros((n_obs, n_t + 1)) for _ in slabs] if n_obs else None
    lib = _lib.load()
    parr = (_lib.C.c_void_p * world)(*[pl._h.value for pl in plans])
    oarr = (_lib.C.POINTER(_lib.C.c_double) * world)(*[_lib.dptr(o) for o in outs])
    barr = ((_lib.C.POINTER(_lib.C.c_double) * world)(*[_lib.dptr(o) for o in obs_parts])
            if obs_parts else None)
    div = _lib.Divergence()
    tm = _lib.Timings()
    code = lib.wcb_imex_group_run(world, parr, f0, _lib.dptr(ft_k), _lib.dptr(ft_new), float(dt), n_t,
                                  float(beta), float(gamma), oarr, None, barr,
                                  _lib.C.byref(div), _lib.C.byref(tm))
    if code == _lib.WCB_E_DIVERGED:
        raise DivergenceError(int(div.step), float(div.amplitude))
    _lib.check(code)
    psi = np.zeros(prob.n_dof)
    for s, o in zip(slabs, outs):
        psi[s.gdofs] = o[:s.n]
    obs = sum(obs_parts) if obs_parts else None
    return RunResult(method="imex", dt=float(dt), t=np.arange(n_t + 1) * float(dt), obs=obs,
                     psi=psi, psi_dot=None,
                     timings=StageTimings(factorization=sum(p.factorization for p in plans), rhs=float(tm.rhs)),
                     fact_dim=0)


def dist_imex_plan(prob, dt: float, beta: float = 0.25, device=None):
    """One slab per torchrun rank (NCCL halos on the library context): this
    rank's SlabElastic and ImexPlan; ImexPlan.run then exchanges halos and
    all-reduces the divergence amplitude and observer partials."""
    import torch.distributed as tdist
    rank, world = tdist.get_rank(), tdist.get_world_size()
    ctx = _lib.context(device)
    if not getattr(ctx, "_nccl", False):
        init_nccl(ctx, rank, world)
        ctx._nccl = True
    lo, hi = partition_imex(prob, world)[rank]
    slab = SlabElastic(prob, lo, hi)
    return slab, slab.plan(dt, beta=beta, device=device)
