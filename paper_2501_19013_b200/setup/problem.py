"""Spectral-cell (GLL Lagrange) systems in the form the device consumes.

``ScmProblem.build`` restates the reference assembly (src/assembly.py:518-603)
without ever forming the global CSR stiffness: it keeps the shared uncut 1D
factors ``m1, k1`` (src/assembly.py:263-295), the physical cut-cell
stiffness ``K_o = sk (K_in + alpha K_out)`` (src/assembly.py:582) and the
lumped diagonal mass (GLL nodal on uncut cells, src/assembly.py:289-291;
HRZ or row-sum on cut cells, src/assembly.py:586-592).  ``csr_stiffness``
assembles the same operator as a scipy CSR for cross-checks at small sizes.

Sources and observers are point evaluations of the basis
(src/harness.py:59-98): ``F_s = rho * alpha(x_s) * N(x_s)``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .basis import Basis1D, gll_rule, uncut_1d
from .cutcell import CutCellIntegrator, hrz_lump, row_sum_lump
from .geometry import CUT, INSIDE, OUTSIDE
from .grid import Grid


def _kron_list(mats):
    out = mats[0]
    for m in mats[1:]:
        out = np.kron(out, m)
    return out


def _cut_chunk(args):
    grid, depth, cells, alpha, sk, sm, lumping = args
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except ImportError:
        lim = None
    d = grid.dim
    L = (grid.p + 1) ** d
    integ = CutCellIntegrator(grid, depth)
    K = np.empty((cells.shape[0], L, L))
    M = np.empty((cells.shape[0], L) if lumping != "none" else (cells.shape[0], L, L))
    shape = (grid.n_e,) * d
    for j, cl in enumerate(cells):
        Mi, Mo, Ki, Ko = integ.integrate(np.unravel_index(int(cl), shape))
        K[j] = sk * (Ki + alpha * Ko)
        M_o = sm * (Mi + alpha * Mo)
        if lumping == "none":
            M[j] = M_o           # consistent cut mass (IMEX, src/assembly.py:591-592)
        else:
            M[j] = hrz_lump(M_o) if lumping == "hrz" else row_sum_lump(M_o)
    if lim is not None:
        lim.unregister()
    return K, M


def _under_profiler() -> bool:
    import os
    if any(k.startswith(("CUDA_INJECTION", "NV_TPS", "NV_NSIGHT")) for k in os.environ):
        return True
    return "TreeLauncher" in os.environ.get("LD_PRELOAD", "")


def integrate_cut_cells(grid, depth, cut, alpha, sk, sm, lumping, n_jobs=None):
    """Physical cut-cell stiffness and (lumped) mass for every cut cell;
    large sets are spread over host processes (each cell is independent)."""
    import os
    from . import native
    if native.enabled(grid.geom, grid.basis.family):   # C++ threads (setup/native.py)
        return native.cut_cells(grid, depth, cut, alpha, sk, sm, lumping)
    n_jobs = n_jobs or int(os.environ.get("WAVECELL_B200_JOBS", 0)) or min(32, os.cpu_count() or 1)
    if _under_profiler():
        n_jobs = 1   # under ncu: forked workers crash the injected tool
    if cut.shape[0] < 256 or n_jobs <= 1:
        return _cut_chunk((grid, depth, cut, alpha, sk, sm, lumping))
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    chunks = np.array_split(cut, n_jobs * 4)
    light = _LightGrid(grid)
    with ProcessPoolExecutor(max_workers=n_jobs, mp_context=mp.get_context("fork")) as ex:
        parts = list(ex.map(_cut_chunk, [(light, depth, c, alpha, sk, sm, lumping)
                                         for c in chunks if c.shape[0]]))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


class _LightGrid:
    """What the cut-cell integrator needs from a Grid (cheap to pickle)."""

    def __init__(self, g):
        self.geom, self.basis, self.dim, self.origin, self.h = g.geom, g.basis, g.dim, g.origin, g.h

    @property
    def p(self):
        return self.basis.p

    @property
    def n_e(self):
        return self.basis.n_e

    def cell_box(self, ijk):
        lo = self.origin + np.asarray(ijk, dtype=float) * self.h
        return lo, lo + self.h


@dataclass
class ScmProblem:
    grid: Grid
    rho: float
    c: float
    alpha: float
    depth: int
    lumping: str
    sk: float
    sm: float
    m1: np.ndarray
    k1: np.ndarray
    cut_K: np.ndarray          # (n_cut, L, L) physical stiffness of cut cells
    cut_M: np.ndarray          # (n_cut, L) lumped mass of cut cells
    m_diag: np.ndarray         # (n_dof,) assembled lumped mass
    F_s: np.ndarray = field(default=None)
    obs_mat: sp.csr_matrix = field(default=None)
    source_point: np.ndarray = field(default=None)

    # ------------------------------------------------------------ build --
    @classmethod
    def build(cls, grid: Grid, alpha: float, depth: int, rho: float = 1.0, c: float = 1.0,
              lumping: str = "hrz", epsilon: float = 0.0, f_lambda: float = 1e-2):
        """``epsilon > 0``: eigenvalue-stabilised cut-cell masses before the
        lumping (src/assembly.py:584-585, src/stabilization.py:73-102), the
        batched eigen-solves on the device (stabilization.evs_stabilize)."""
        if grid.basis.family != "lagrange":
            raise ValueError("ScmProblem needs the Lagrange (GLL) family")
        if lumping not in ("hrz", "row_sum", "none"):
            raise ValueError("lumping must be 'hrz', 'row_sum' or 'none'")
        d, p, h = grid.dim, grid.p, grid.h
        n = p + 1
        L = n ** d
        # src/assembly.py:504-505 for d = 3; (h/2)^(d-2) and (h/2)^d in general
        sk = rho * c * c * (h / 2.0) ** (d - 2)
        sm = rho * (h / 2.0) ** d
        m1, k1 = uncut_1d(grid.basis, 0)
        cut = grid.cut_lex
        if epsilon > 0.0 and cut.shape[0]:
            from ..stabilization import evs_stabilize
            cut_K, M_o = integrate_cut_cells(grid, depth, cut, alpha, sk, sm, "none")
            _, M_f = integrate_cut_cells(grid, depth, cut, 1.0, sk, sm, "none")
            M_o = evs_stabilize(M_o, M_f, epsilon, f_lambda)
            cut_M = M_o if lumping == "none" else (hrz_lump(M_o) if lumping == "hrz" else row_sum_lump(M_o))
        else:
            cut_K, cut_M = integrate_cut_cells(grid, depth, cut, alpha, sk, sm, lumping)
        prob = cls(grid=grid, rho=rho, c=c, alpha=alpha, depth=depth, lumping=lumping,
                   sk=sk, sm=sm, m1=m1, k1=k1, cut_K=cut_K, cut_M=cut_M,
                   m_diag=np.zeros(0))
        prob.m_diag = prob._assemble_mass()
        return prob

    @property
    def n_dof(self) -> int:
        return self.grid.n_dof

    def _assemble_mass(self) -> np.ndarray:
        """Diagonal mass: sm * (w (x) w [(x) w]) on uncut kept cells, the lumped
        cut-cell vectors elsewhere, summed per DOF."""
        g = self.grid
        d, p, n_e = g.dim, g.p, g.n_e
        n1 = g.basis.n_funcs
        w = gll_rule(p)[1]
        from . import native
        if native.lib_ok():
            return native.lumped_mass(g, w, self.sm, self.cut_M if self.lumping != "none" else
                                      np.zeros((0, (p + 1) ** d)))
        uncut = (g.classes == INSIDE).astype(float)
        node = np.zeros((n1,) * d)
        for local in np.ndindex(*([p + 1] * d)):
            wt = self.sm * np.prod([w[a] for a in local])
            sl = tuple(slice(a, a + p * (n_e - 1) + 1, p) for a in local)
            node[sl] += wt * uncut
        node = node.ravel()
        m = node[g.dofmap.lex_of_compact]
        cut = g.cut_lex
        if cut.shape[0] and self.lumping != "none":
            dofs = self.cut_dofs()
            np.add.at(m, dofs.ravel(), self.cut_M.ravel())
        return m

    def cut_dofs(self) -> np.ndarray:
        """(n_cut, L) compact DOF ids of every cut cell."""
        g = self.grid
        shape = (g.n_e,) * g.dim
        return np.stack([g.dofmap.cell_dofs(g.basis, np.unravel_index(int(c), shape))
                         for c in g.cut_lex]) if g.cut_lex.size else \
            np.zeros((0, (g.p + 1) ** g.dim), dtype=np.int64)

    # ------------------------------------------------------------ points --
    def point_row(self, x):
        """(dofs, values) of the basis functions at a grid-frame point."""
        g = self.grid
        x = np.asarray(x, dtype=float)
        idx = g.locate(x)
        lo, _ = g.cell_box(idx)
        xi = np.clip(2.0 * (x - lo) / g.h - 1.0, -1.0, 1.0)
        V = [g.basis.eval(int(idx[k]), np.array([xi[k]]))[0][0] for k in range(g.dim)]
        vals = _kron_list([v.reshape(1, -1) for v in V]).ravel()
        dofs = g.dofmap.cell_dofs(g.basis, idx)
        if np.any(dofs < 0):
            raise ValueError("point lies in a discarded cell")
        return dofs, vals, idx

    def set_point_source(self, x_s):
        """F_s = rho * alpha(x_s) * N(x_s): a Dirac load at x_s."""
        dofs, vals, idx = self.point_row(x_s)
        a = 1.0 if bool(self.grid.geom.contains(np.asarray(x_s)[None])[0]) else self.alpha
        F = np.zeros(self.n_dof)
        np.add.at(F, dofs, self.rho * a * vals)
        self.F_s = F
        self.source_point = np.asarray(x_s, dtype=float)
        return F

    def set_observers(self, points):
        rows, cols, vals = [], [], []
        for i, x in enumerate(points):
            dofs, v, _ = self.point_row(x)
            rows.extend([i] * dofs.shape[0])
            cols.extend(dofs.tolist())
            vals.extend(v.tolist())
        self.obs_mat = sp.csr_matrix((vals, (rows, cols)), shape=(len(points), self.n_dof))
        return self.obs_mat

    # ----------------------------------------------------------- device --
    def device_operator(self, device=None):
        from ..operators import ScmOperator
        g = self.grid
        op = ScmOperator(dim=g.dim, p=g.p, n_e=(g.n_e,) * g.dim, k1=self.k1, m1=self.m1,
                         sk=self.sk, cell_class=g.classes.ravel(),
                         lex_of_compact=g.dofmap.lex_of_compact, cut_cells=g.cut_lex,
                         cut_K=self.cut_K, device=device)
        op.problem = self
        return op

    def mass_matrix(self) -> sp.csr_matrix:
        """Global mass: diagonal when lumped; with lumping 'none' the cut cells
        keep their consistent blocks (the IMEX c-set mass)."""
        if self.lumping != "none":
            return sp.diags(self.m_diag).tocsr()
        L = self.cut_M.shape[-1]
        dofs = self.cut_dofs()
        rr, cc = np.divmod(np.arange(L * L), L)
        rows = np.concatenate([np.arange(self.n_dof)] + [d[rr] for d in dofs])
        cols = np.concatenate([np.arange(self.n_dof)] + [d[cc] for d in dofs])
        vals = np.concatenate([self.m_diag] + [Mj.ravel() for Mj in self.cut_M])
        A = sp.coo_matrix((vals, (rows, cols)), shape=(self.n_dof, self.n_dof)).tocsr()
        A.eliminate_zeros()
        return A

    # -------------------------------------------------------------- CSR --
    def csr_stiffness(self) -> sp.csr_matrix:
        """Global stiffness as CSR (small problems; cross-checks only)."""
        g = self.grid
        d, p = g.dim, g.p
        L = (p + 1) ** d
        mats = [self.m1] * d
        K_ref = np.zeros((L, L))
        for k in range(d):
            parts = list(mats)
            parts[k] = self.k1
            K_ref += _kron_list(parts)
        K_ref *= self.sk
        shape = (g.n_e,) * d
        uncut = np.flatnonzero(g.classes.ravel() == INSIDE)
        rows, cols, vals = [], [], []
        rr, cc = np.divmod(np.arange(L * L), L)
        for cl in uncut:
            dofs = g.dofmap.cell_dofs(g.basis, np.unravel_index(int(cl), shape))
            rows.append(dofs[rr]); cols.append(dofs[cc]); vals.append(K_ref.ravel())
        for j, dofs in enumerate(self.cut_dofs()):
            rows.append(dofs[rr]); cols.append(dofs[cc]); vals.append(self.cut_K[j].ravel())
        if not rows:
            return sp.csr_matrix((self.n_dof, self.n_dof))
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n_dof, self.n_dof)).tocsr()
        A.eliminate_zeros()
        return A
