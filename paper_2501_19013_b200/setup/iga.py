"""IGA-FCM (maximally smooth B-spline) systems: the CSR path (BASELINE config 3).

Restates the reference assembly for ``family="bspline"`` (src/assembly.py:
518-612) in d = 2, 3 dimensions:

* uncut cells: ``sk * sum_k (m1 (x) .. k1 .. (x) m1)`` with per-cell 1D tables
  that depend on the cell's boundary signature (src/assembly.py:256-272);
* cut cells: 2^d-tree quadrature integrals (``cutcell.CutCellIntegrator``),
  combined as ``sk (K_in + alpha K_out)``;
* mass: row-sum lumped on every cell (src/stabilization.py:105-114; for
  B-splines all entries are non-negative, so the lumped diagonal is positive).

The global CSR is built without a per-cell loop: for every stencil offset the
sum over incident kept uncut cells is a separable array expression over the
whole node grid, the cut cells are added as COO, and exact zeros are dropped
like ``_to_csr`` (src/assembly.py:606-612).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .basis import Basis1D, uncut_1d
from .cutcell import CutCellIntegrator, row_sum_lump
from .geometry import CUT, INSIDE, OUTSIDE, PolygonVoid
from .grid import Grid


def _kron_list(mats):
    out = mats[0]
    for m in mats[1:]:
        out = np.kron(out, m)
    return out


@dataclass
class IgaProblem:
    grid: Grid
    rho: float
    c: float
    alpha: float
    depth: int
    sk: float
    sm: float
    K: sp.csr_matrix
    m_diag: np.ndarray
    F_s: np.ndarray = field(default=None)
    obs_mat: sp.csr_matrix = field(default=None)
    source_point: np.ndarray = field(default=None)

    @classmethod
    def build(cls, grid: Grid, alpha: float, depth: int, rho: float = 1.0, c: float = 1.0):
        if grid.basis.family != "bspline":
            raise ValueError("IgaProblem needs the B-spline family")
        d, p, n_e, h = grid.dim, grid.p, grid.n_e, grid.h
        N = p + 1
        sk = rho * c * c * (h / 2.0) ** (d - 2)
        sm = rho * (h / 2.0) ** d
        b = grid.basis
        # per-cell 1D tables along one axis (same for every axis: cubic grid)
        m1 = np.empty((n_e, N, N))
        k1 = np.empty((n_e, N, N))
        cache = {}
        for e in range(n_e):
            key = b.signature(e)
            if key not in cache:
                cache[key] = uncut_1d(b, e)
            m1[e], k1[e] = cache[key]
        n1 = b.n_funcs
        classes = grid.classes
        uncut = (classes == INSIDE).astype(np.float64)
        kept = classes != OUTSIDE
        K = _stencil_csr(d, p, n_e, n1, uncut, kept, m1, k1, sk, grid.dofmap)
        # cut cells
        cut = grid.cut_lex
        integ = CutCellIntegrator(grid, depth)
        rows, cols, vals = [], [], []
        cut_M = np.empty((cut.shape[0], N ** d))
        L = N ** d
        rr, cc = np.divmod(np.arange(L * L), L)
        shape = (n_e,) * d
        for j, cl in enumerate(cut):
            ijk = np.unravel_index(int(cl), shape)
            Mi, Mo, Ki, Ko = integ.integrate(ijk)
            dofs = grid.dofmap.cell_dofs(b, ijk)
            rows.append(dofs[rr]); cols.append(dofs[cc])
            vals.append((sk * (Ki + alpha * Ko)).ravel())
            cut_M[j] = row_sum_lump(sm * (Mi + alpha * Mo))
        n = grid.n_dof
        if rows:
            Kc = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(n, n)).tocsr()
            K = (K + Kc).tocsr()
        K.eliminate_zeros()
        K.sort_indices()
        # row-sum lumped mass: uncut cells give (m1 1) (x) (m1 1) per cell
        rs = m1.sum(axis=2)                              # (n_e, N) row sums per cell
        node = np.zeros((n1,) * d)
        for local in np.ndindex(*([N] * d)):
            w = sm
            arr = uncut.copy()
            for ax in range(d):
                shp = [1] * d
                shp[ax] = n_e
                arr = arr * rs[:, local[ax]].reshape(shp)
            sl = tuple(slice(local[ax], local[ax] + n_e) for ax in range(d))
            node[sl] += w * arr
        m = node.ravel()[grid.dofmap.lex_of_compact]
        if cut.shape[0]:
            cdofs = np.stack([grid.dofmap.cell_dofs(b, np.unravel_index(int(cl), shape)) for cl in cut])
            np.add.at(m, cdofs.ravel(), cut_M.ravel())
        return cls(grid=grid, rho=rho, c=c, alpha=alpha, depth=depth, sk=sk, sm=sm, K=K,
                   m_diag=m)

    @property
    def n_dof(self) -> int:
        return self.grid.n_dof

    def mass_matrix(self) -> sp.csr_matrix:
        return sp.diags(self.m_diag).tocsr()

    def point_row(self, x):
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
        dofs, vals, _ = self.point_row(x_s)
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
            rows.extend([i] * dofs.shape[0]); cols.extend(dofs.tolist()); vals.extend(v.tolist())
        self.obs_mat = sp.csr_matrix((vals, (rows, cols)), shape=(len(points), self.n_dof))
        return self.obs_mat

    def device_operator(self, device=None):
        from ..operators import CsrOperator
        return CsrOperator(self.K, device=device)


def _stencil_csr(d, p, n_e, n1, uncut, kept, m1, k1, sk, dofmap):
    """Sum of uncut-cell Kronecker matrices as CSR, one stencil offset at a time.

    For offset o (per axis in -p..p) the value at node I is
    sum over local a with 0 <= a, a+o <= p of cell (I - a):
      chi(cell) * prod_ax T_ax[cell_ax][a_ax, a_ax + o_ax],
    with T = k1 on one axis and m1 on the others (summed over that axis).
    Structural entries come from every incident kept cell (uncut or cut) so
    the pattern matches the reference's COO -> CSR of all kept cells.
    """
    N = p + 1
    offsets = list(np.ndindex(*([2 * p + 1] * d)))
    lex = dofmap.compact_of_lex.reshape((n1,) * d)
    rows_all, cols_all, vals_all = [], [], []
    for off in offsets:
        o = [oo - p for oo in off]
        val = np.zeros((n1,) * d)
        struct = np.zeros((n1,) * d, dtype=bool)
        ranges = [range(max(0, -oa), min(N, N - oa)) for oa in o]
        for a in np.ndindex(*[len(r) for r in ranges]):
            loc = [ranges[ax][a[ax]] for ax in range(d)]
            # cells (I - loc) for node I: slice of the node grid shifted by loc
            sl = tuple(slice(loc[ax], loc[ax] + n_e) for ax in range(d))
            struct[sl] |= kept
            for kax in range(d):
                term = uncut.copy()
                for ax in range(d):
                    T = k1 if ax == kax else m1
                    coef = T[:, loc[ax], loc[ax] + o[ax]]        # per cell along ax
                    shp = [1] * d
                    shp[ax] = n_e
                    term = term * coef.reshape(shp)
                val[sl] += sk * term
        nz = struct & (lex >= 0)
        idx = np.flatnonzero(nz.ravel())
        if idx.size == 0:
            continue
        coords = np.unravel_index(idx, (n1,) * d)
        tgt = [coords[ax] + o[ax] for ax in range(d)]
        ok = np.ones(idx.shape[0], dtype=bool)
        for ax in range(d):
            ok &= (tgt[ax] >= 0) & (tgt[ax] < n1)
        idx = idx[ok]
        tgt = [t[ok] for t in tgt]
        tl = np.ravel_multi_index(tgt, (n1,) * d)
        r = lex.ravel()[idx]
        cc = lex.ravel()[tl]
        keep = cc >= 0
        rows_all.append(r[keep]); cols_all.append(cc[keep]); vals_all.append(val.ravel()[idx][keep])
    n = dofmap.n_dof
    K = sp.csr_matrix((np.concatenate(vals_all), (np.concatenate(rows_all), np.concatenate(cols_all))),
                      shape=(n, n))
    return K


def polygon_void(rng, n_vertices=12):
    """Config 3's seeded random polygon: sorted U(0, 2 pi) angles, radii
    U(0.1, 0.3) about a U(0.3, 0.7)^2 centre."""
    centre = rng.uniform(0.3, 0.7, size=2)
    ang = np.sort(rng.uniform(0.0, 2.0 * np.pi, size=n_vertices))
    rad = rng.uniform(0.1, 0.3, size=n_vertices)
    return centre + np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1)


def build_config3(n_e=1024, p=3, alpha=1e-5, depth=4, seed=0):
    """BASELINE config 3: 2D IGA-FCM, B-splines p=3 on n_e^2 spans, polygon void."""
    from .configs import pick_source
    rng = np.random.default_rng(seed)
    geom = PolygonVoid(polygon_void(rng))
    grid = Grid.build(geom, "bspline", p, n_e)
    prob = IgaProblem.build(grid, alpha, depth)
    x_s = pick_source(grid, rng)
    prob.set_point_source(x_s)
    centre = np.full(2, 0.5)
    if not bool(geom.contains(centre[None])[0]) or grid.classes[tuple(grid.locate(centre))] == 0:
        centre = pick_source(grid, rng)
    prob.set_observers([x_s, centre])
    return prob
