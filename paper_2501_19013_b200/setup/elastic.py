"""Plane-strain elastodynamics on the spectral-cell grid (BASELINE config 4).

The reference has no vector-valued operator (parity for this
operator is unpinned; the integrators are pinned by running the reference
``imex_run`` on the CSR assembled here).  The discretisation follows the
scalar SCM of src/assembly.py:263-295 / 518-603 component-wise:

* two displacement components per GLL node, DOFs numbered **component
  major**: ``dof = comp * n_node + node`` (node = the scalar compact id);
* uncut cells: ``K = [[(l+2m) Kxx + m Kyy, l Kxy + m Kxy^T],
  [(l Kxy + m Kxy^T)^T, m Kxx + (l+2m) Kyy]]`` with the 1D factors
  ``Kxx = k1 (x) m1``, ``Kyy = m1 (x) k1``, ``Kxy = g1 (x) g1^T`` where
  ``g1[a][b] = int phi_a' phi_b`` (GL-exact); in 2D the derivative and
  Jacobian scalings cancel, so no ``sk`` factor appears;
* cut cells: the same combination of space-tree integrals, physical part
  plus ``alpha`` times the fictitious part (src/assembly.py:575-583);
* mass: GLL nodal on uncut cells, consistent ``rho (h/2)^2 (M_in + alpha
  M_out)`` on cut cells (the IMEX c-set mass, PAPER 2.4), per component.

``c`` = both components of every node touching a cut cell, ``d`` = the rest.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .basis import gll_rule, uncut_1d, uncut_g1
from .cutcell import ElasticCutIntegrator
from .geometry import INSIDE
from .grid import Grid
from .problem import _LightGrid, _kron_list, _under_profiler


def lame(E: float, nu: float):
    """Plane-strain Lame parameters."""
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def elastic_element(lam, mu, Kxx, Kyy, Kxy):
    """(2L, 2L) plane-strain element matrix in component-major local order."""
    Kuu = (lam + 2.0 * mu) * Kxx + mu * Kyy
    Kvv = mu * Kxx + (lam + 2.0 * mu) * Kyy
    Kuv = lam * Kxy + mu * Kxy.T
    return np.block([[Kuu, Kuv], [Kuv.T, Kvv]])


def _elastic_chunk(args):
    grid, depth, cells, alpha, lam, mu, sm = args
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except ImportError:
        lim = None
    n = grid.p + 1
    Ld = n * n
    integ = ElasticCutIntegrator(grid, depth)
    K = np.empty((cells.shape[0], 2 * Ld, 2 * Ld))
    M = np.empty((cells.shape[0], Ld, Ld))
    shape = (grid.n_e, grid.n_e)
    for j, cl in enumerate(cells):
        acc = integ.integrate_elastic(np.unravel_index(int(cl), shape))
        comb = {nm: acc[(nm, "in")] + alpha * acc[(nm, "out")] for nm in ("M", "Kxx", "Kyy", "Kxy")}
        K[j] = elastic_element(lam, mu, comb["Kxx"], comb["Kyy"], comb["Kxy"])
        M[j] = sm * comb["M"]
    if lim is not None:
        lim.unregister()
    return K, M


def integrate_elastic_cut_cells(grid, depth, cut, alpha, lam, mu, sm, n_jobs=None):
    import os
    n_jobs = n_jobs or int(os.environ.get("WAVECELL_B200_JOBS", 0)) or min(32, os.cpu_count() or 1)
    if _under_profiler():
        n_jobs = 1
    if cut.shape[0] < 64 or n_jobs <= 1:
        return _elastic_chunk((grid, depth, cut, alpha, lam, mu, sm))
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    chunks = np.array_split(cut, n_jobs * 4)
    light = _LightGrid(grid)
    with ProcessPoolExecutor(max_workers=n_jobs, mp_context=mp.get_context("fork")) as ex:
        parts = list(ex.map(_elastic_chunk, [(light, depth, c, alpha, lam, mu, sm)
                                             for c in chunks if c.shape[0]]))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


@dataclass
class ElasticProblem:
    grid: Grid
    lam: float
    mu: float
    rho: float
    alpha: float
    depth: int
    m1: np.ndarray
    k1: np.ndarray
    g1: np.ndarray
    cut_K: np.ndarray          # (n_cut, 2L, 2L) physical stiffness of cut cells
    cut_M: np.ndarray          # (n_cut, L, L) consistent mass per component
    m_node: np.ndarray         # (n_node,) GLL nodal mass of the uncut cells
    F_s: np.ndarray = field(default=None)
    obs_mat: sp.csr_matrix = field(default=None)
    source_point: np.ndarray = field(default=None)

    @classmethod
    def build(cls, grid: Grid, lam: float, mu: float, alpha: float, depth: int,
              rho: float = 1.0):
        if grid.dim != 2 or grid.basis.family != "lagrange":
            raise ValueError("ElasticProblem is 2D with the Lagrange (GLL) family")
        h = grid.h
        sm = rho * (h / 2.0) ** 2
        m1, k1 = uncut_1d(grid.basis, 0)
        g1 = uncut_g1(grid.basis, 0)
        cut_K, cut_M = integrate_elastic_cut_cells(grid, depth, grid.cut_lex, alpha, lam, mu, sm)
        prob = cls(grid=grid, lam=float(lam), mu=float(mu), rho=float(rho), alpha=float(alpha),
                   depth=int(depth), m1=m1, k1=k1, g1=g1, cut_K=cut_K, cut_M=cut_M,
                   m_node=np.zeros(0))
        prob.m_node = prob._uncut_mass()
        return prob

    # ---------------------------------------------------------- numbering --
    @property
    def n_node(self) -> int:
        return self.grid.n_dof

    @property
    def n_dof(self) -> int:
        return 2 * self.grid.n_dof

    @property
    def c_idx(self) -> np.ndarray:
        c = self.grid.dofmap.c_idx
        return np.concatenate([c, c + self.n_node]).astype(np.int64)

    @property
    def d_idx(self) -> np.ndarray:
        d = self.grid.dofmap.d_idx
        return np.concatenate([d, d + self.n_node]).astype(np.int64)

    @property
    def sm(self) -> float:
        return self.rho * (self.grid.h / 2.0) ** 2

    def _uncut_mass(self) -> np.ndarray:
        g = self.grid
        p, n_e = g.p, g.n_e
        n1 = g.basis.n_funcs
        w = gll_rule(p)[1]
        uncut = (g.classes == INSIDE).astype(float)
        node = np.zeros((n1, n1))
        for a in range(p + 1):
            for b in range(p + 1):
                node[a:a + p * (n_e - 1) + 1:p, b:b + p * (n_e - 1) + 1:p] += \
                    self.sm * w[a] * w[b] * uncut
        return node.ravel()[g.dofmap.lex_of_compact]

    def cell_nodes(self, cells) -> np.ndarray:
        """(len(cells), L) compact node ids of cells given by lex id."""
        g = self.grid
        cells = np.asarray(cells, dtype=np.int64)
        n = g.p + 1
        n1 = g.basis.n_funcs
        ex, ey = np.divmod(cells, g.n_e)
        a = np.arange(n)
        lex = ((ex[:, None, None] * g.p + a[None, :, None]) * n1 +
               (ey[:, None, None] * g.p + a[None, None, :])).reshape(cells.shape[0], n * n)
        return g.dofmap.compact_of_lex[lex]

    def cell_dofs(self, cells) -> np.ndarray:
        nodes = self.cell_nodes(cells)
        return np.concatenate([nodes, nodes + self.n_node], axis=1)

    def uncut_element(self) -> np.ndarray:
        return elastic_element(self.lam, self.mu, np.kron(self.k1, self.m1),
                               np.kron(self.m1, self.k1), np.kron(self.g1, self.g1.T))

    # ------------------------------------------------------------ matrices --
    def mass_matrix(self) -> sp.csr_matrix:
        n, nn = self.n_dof, self.n_node
        L = self.cut_M.shape[-1] if self.cut_M.size else (self.grid.p + 1) ** 2
        nodes = self.cell_nodes(self.grid.cut_lex)
        rr, cc = np.divmod(np.arange(L * L), L)
        rows = [np.arange(n)]
        cols = [np.arange(n)]
        vals = [np.concatenate([self.m_node, self.m_node])]
        for comp in (0, 1):
            off = comp * nn
            rows.append((nodes[:, rr] + off).ravel())
            cols.append((nodes[:, cc] + off).ravel())
            vals.append(self.cut_M.reshape(-1, L * L).ravel())
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(n, n)).tocsr()
        A.eliminate_zeros()
        return A

    def _assemble(self, cells_uncut, keep=None) -> sp.csr_matrix:
        n = self.n_dof
        Ke = self.uncut_element()
        L2 = Ke.shape[0]
        rr, cc = np.divmod(np.arange(L2 * L2), L2)
        rows, cols, vals = [], [], []
        chunk = 4096
        for s in range(0, cells_uncut.shape[0], chunk):
            dofs = self.cell_dofs(cells_uncut[s:s + chunk])
            rows.append(dofs[:, rr].ravel())
            cols.append(dofs[:, cc].ravel())
            vals.append(np.broadcast_to(Ke.ravel(), (dofs.shape[0], L2 * L2)).ravel())
        if self.grid.cut_lex.size:
            dofs = self.cell_dofs(self.grid.cut_lex)
            rows.append(dofs[:, rr].ravel())
            cols.append(dofs[:, cc].ravel())
            vals.append(self.cut_K.reshape(-1, L2 * L2).ravel())
        if not rows:
            return sp.csr_matrix((n, n))
        r = np.concatenate(rows)
        c = np.concatenate(cols)
        v = np.concatenate(vals)
        if keep is not None:
            m = keep[r] & keep[c]
            r, c, v = r[m], c[m], v[m]
        A = sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr()
        A.eliminate_zeros()
        return A

    def csr_stiffness(self) -> sp.csr_matrix:
        """Global stiffness as CSR (small problems; cross-checks and oracle runs)."""
        uncut = np.flatnonzero(self.grid.classes.ravel() == INSIDE)
        return self._assemble(uncut)

    def stiffness_block(self, idx) -> sp.csr_matrix:
        """K[idx][:, idx] assembled from the cells touching idx only (the IMEX
        c-c block at sizes where the global CSR does not fit host memory)."""
        idx = np.asarray(idx, dtype=np.int64)
        keep = np.zeros(self.n_dof, dtype=bool)
        keep[idx] = True
        g = self.grid
        uncut = np.flatnonzero(g.classes.ravel() == INSIDE)
        touch = np.zeros(uncut.shape[0], dtype=bool)
        for s in range(0, uncut.shape[0], 1 << 16):
            touch[s:s + (1 << 16)] = keep[self.cell_dofs(uncut[s:s + (1 << 16)])].any(axis=1)
        A = self._assemble(uncut[touch], keep)
        return A[idx][:, idx]

    # ------------------------------------------------------------- points --
    def point_row(self, x):
        g = self.grid
        x = np.asarray(x, dtype=float)
        idx = g.locate(x)
        lo, _ = g.cell_box(idx)
        xi = np.clip(2.0 * (x - lo) / g.h - 1.0, -1.0, 1.0)
        V = [g.basis.eval(int(idx[k]), np.array([xi[k]]))[0][0] for k in range(2)]
        vals = _kron_list([v.reshape(1, -1) for v in V]).ravel()
        nodes = g.dofmap.cell_dofs(g.basis, idx)
        if np.any(nodes < 0):
            raise ValueError("point lies in a discarded cell")
        return nodes, vals, idx

    def set_point_source(self, x_s, direction=(1.0, 0.0)):
        """Point force rho * alpha(x_s) * N(x_s) * direction."""
        nodes, vals, _ = self.point_row(x_s)
        a = 1.0 if bool(self.grid.geom.contains(np.asarray(x_s)[None])[0]) else self.alpha
        F = np.zeros(self.n_dof)
        for comp in (0, 1):
            if direction[comp] != 0.0:
                np.add.at(F, nodes + comp * self.n_node, self.rho * a * direction[comp] * vals)
        self.F_s = F
        self.source_point = np.asarray(x_s, dtype=float)
        return F

    def set_observers(self, points):
        """Two rows per point: displacement x then y."""
        rows, cols, vals = [], [], []
        for i, x in enumerate(points):
            nodes, v, _ = self.point_row(x)
            for comp in (0, 1):
                rows.extend([2 * i + comp] * nodes.shape[0])
                cols.extend((nodes + comp * self.n_node).tolist())
                vals.extend(v.tolist())
        self.obs_mat = sp.csr_matrix((vals, (rows, cols)), shape=(2 * len(points), self.n_dof))
        return self.obs_mat

    # ------------------------------------------------------------ device --
    def device_operator(self, device=None):
        from ..operators import ElasticOperator
        g = self.grid
        op = ElasticOperator(p=g.p, n_e=g.n_e, lam=self.lam, mu=self.mu, m1=self.m1, k1=self.k1,
                             g1=self.g1, cell_class=g.classes.ravel(),
                             lex_of_compact=g.dofmap.lex_of_compact, cut_cells=g.cut_lex,
                             cut_K=self.cut_K, device=device)
        op.problem = self
        return op
