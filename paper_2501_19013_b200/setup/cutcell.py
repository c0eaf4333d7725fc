"""Alpha-independent cut-cell integrals by 2^d-tree quadrature (d = 2, 3).

Restates ``ElementIntegralCache._integrate_cut`` / ``_accumulate_pointwise``
(src/assembly.py:310-423) for any dimension:

* the cell is partitioned by recursive 2^d-section (src/geometry.py:316-346);
* settled (inside/outside) leaves keep the tensor structure: their mass and
  stiffness are Kronecker sums of per-interval 1D tables (the dyadic tables,
  src/assembly.py:310-330);
* leaves still cut at the maximum depth classify every GL point
  individually; their full-leaf integral is the same Kronecker sum and the
  physical part is summed point by point, the fictitious part is the
  difference (as src/assembly.py:410-422 does);
* physical/fictitious parts stay separate so alpha is applied afterwards.

Local DOF order: last axis fastest (src/assembly.py:85-89, _kron3 :426-429).
"""

from __future__ import annotations

import numpy as np

from .basis import Basis1D, dyadic_tables
from .geometry import CUT, INSIDE, OUTSIDE, tree_partition


def kron_sum(mats):
    """sum_l kron(mats[0][l], mats[1][l], ...) for batches of 1D matrices."""
    d = len(mats)
    n = mats[0].shape[-1]
    if d == 2:
        out = np.einsum("lac,lbd->abcd", mats[0], mats[1], optimize=True)
    else:
        out = np.einsum("lad,lbe,lcf->abcdef", mats[0], mats[1], mats[2], optimize=True)
    return out.reshape(n ** d, n ** d)


def _tensor_rows(parts):
    """Rows of tensor-product values at tensor points: parts[k] is (L, q, n)
    for direction k; result (L*q^d, n^d), point and function order last axis
    fastest."""
    d = len(parts)
    L, q, n = parts[0].shape
    if d == 2:
        G = np.einsum("lqa,lrb->lqrab", parts[0], parts[1])
    else:
        G = np.einsum("lqa,lrb,lsc->lqrsabc", parts[0], parts[1], parts[2])
    return G.reshape(L * q ** d, n ** d)


class CutCellIntegrator:
    """Builds ``(M_in, M_out, K_in, K_out)`` of cut cells of one grid."""

    def __init__(self, grid, depth: int, q: int | None = None):
        self.grid = grid
        self.depth = int(depth)
        self.q = grid.p + 1 if q is None else int(q)
        self._tabs = {}

    def tables(self, e: int):
        key = self.grid.basis.signature(int(e))
        if key not in self._tabs:
            self._tabs[key] = dyadic_tables(self.grid.basis, int(e), self.depth, self.q)
        return self._tabs[key]

    def integrate(self, ijk):
        grid = self.grid
        d = grid.dim
        n = grid.p + 1
        Ld = n ** d
        lo, hi = grid.cell_box(ijk)
        geom = grid.geom.restricted(lo, hi) if hasattr(grid.geom, "restricted") else grid.geom
        llo, lhi, lcls, ldep = tree_partition(geom, lo, hi, self.depth)
        tabs = [self.tables(e) for e in ijk]
        A = 2.0 * (llo - lo) / (hi - lo) - 1.0
        pos = np.rint((A + 1.0) / 2.0 * (2.0 ** ldep[:, None])).astype(np.int64)
        ids = tabs[0]["offsets"][ldep][:, None] + pos
        M_in = np.zeros((Ld, Ld))
        M_out = np.zeros((Ld, Ld))
        K_in = np.zeros((Ld, Ld))
        K_out = np.zeros((Ld, Ld))

        def settled(sel, M_acc, K_acc):
            m = [tabs[k]["m1"][ids[sel, k]] for k in range(d)]
            kk = [tabs[k]["k1"][ids[sel, k]] for k in range(d)]
            M_acc += kron_sum(m)
            for k in range(d):
                parts = list(m)
                parts[k] = kk[k]
                K_acc += kron_sum(parts)

        for klass, Ma, Ka in ((INSIDE, M_in, K_in), (OUTSIDE, M_out, K_out)):
            sel = np.flatnonzero(lcls == klass)
            if sel.shape[0]:
                settled(sel, Ma, Ka)
        sel = np.flatnonzero(lcls == CUT)
        if sel.shape[0]:
            M_all = np.zeros((Ld, Ld))
            K_all = np.zeros((Ld, Ld))
            settled(sel, M_all, K_all)
            Vd = [tabs[k]["V"][ids[sel, k]] for k in range(d)]
            Dd = [tabs[k]["D"][ids[sel, k]] for k in range(d)]
            xd = [tabs[k]["xi"][ids[sel, k]] for k in range(d)]
            wd = [tabs[k]["w"][ids[sel, k]] for k in range(d)]
            q = self.q
            Lc = sel.shape[0]
            # global coordinates of every tensor point, last axis fastest
            pts = np.empty((Lc,) + (q,) * d + (d,))
            for k in range(d):
                g = lo[k] + (xd[k] + 1.0) / 2.0 * (hi[k] - lo[k])      # (Lc, q)
                pts[..., k] = _broadcast_axis(g, k, d, q)
            inside = geom.contains(pts.reshape(-1, d))
            wt = _tensor_weights(wd)
            w_in = np.where(inside, wt, 0.0)
            V = _tensor_rows(Vd)
            m_in = (V * w_in[:, None]).T @ V
            M_in += m_in
            M_out += M_all - m_in
            for k in range(d):
                parts = list(Vd)
                parts[k] = Dd[k]
                G = _tensor_rows(parts)
                g_in = (G * w_in[:, None]).T @ G
                K_in += g_in
                K_all -= g_in
            K_out += K_all
        return M_in, M_out, K_in, K_out


class ElasticCutIntegrator(CutCellIntegrator):
    """2D cut-cell integrals for plane-strain elasticity: mass and the three
    derivative pairings, physical ("in") and fictitious ("out") parts
    separate.  Kxy[a][b] = int dN_a/dx dN_b/dy; Kyx = Kxy^T."""

    def integrate_elastic(self, ij):
        grid = self.grid
        if grid.dim != 2:
            raise ValueError("elastic cut integration is 2D")
        n = grid.p + 1
        Ld = n * n
        lo, hi = grid.cell_box(ij)
        geom = grid.geom.restricted(lo, hi) if hasattr(grid.geom, "restricted") else grid.geom
        llo, lhi, lcls, ldep = tree_partition(geom, lo, hi, self.depth)
        tabs = [self.tables(e) for e in ij]
        A = 2.0 * (llo - lo) / (hi - lo) - 1.0
        pos = np.rint((A + 1.0) / 2.0 * (2.0 ** ldep[:, None])).astype(np.int64)
        ids = tabs[0]["offsets"][ldep][:, None] + pos
        names = ("M", "Kxx", "Kyy", "Kxy")
        acc = {(nm, part): np.zeros((Ld, Ld)) for nm in names for part in ("in", "out")}

        def settled(sel):
            t = [{key: tabs[k][key][ids[sel, k]] for key in ("m1", "k1", "g1")} for k in range(2)]
            return {"M": kron_sum([t[0]["m1"], t[1]["m1"]]),
                    "Kxx": kron_sum([t[0]["k1"], t[1]["m1"]]),
                    "Kyy": kron_sum([t[0]["m1"], t[1]["k1"]]),
                    "Kxy": kron_sum([t[0]["g1"], np.swapaxes(t[1]["g1"], 1, 2)])}

        for klass, part in ((INSIDE, "in"), (OUTSIDE, "out")):
            sel = np.flatnonzero(lcls == klass)
            if sel.shape[0]:
                for nm, v in settled(sel).items():
                    acc[(nm, part)] += v
        sel = np.flatnonzero(lcls == CUT)
        if sel.shape[0]:
            full = settled(sel)
            Vd = [tabs[k]["V"][ids[sel, k]] for k in range(2)]
            Dd = [tabs[k]["D"][ids[sel, k]] for k in range(2)]
            xd = [tabs[k]["xi"][ids[sel, k]] for k in range(2)]
            wd = [tabs[k]["w"][ids[sel, k]] for k in range(2)]
            q = self.q
            Lc = sel.shape[0]
            pts = np.empty((Lc, q, q, 2))
            for k in range(2):
                g = lo[k] + (xd[k] + 1.0) / 2.0 * (hi[k] - lo[k])
                pts[..., k] = _broadcast_axis(g, k, 2, q)
            inside = geom.contains(pts.reshape(-1, 2))
            w_in = np.where(inside, _tensor_weights(wd), 0.0)
            V = _tensor_rows(Vd)
            DX = _tensor_rows([Dd[0], Vd[1]])
            DY = _tensor_rows([Vd[0], Dd[1]])
            ins = {"M": (V * w_in[:, None]).T @ V,
                   "Kxx": (DX * w_in[:, None]).T @ DX,
                   "Kyy": (DY * w_in[:, None]).T @ DY,
                   "Kxy": (DX * w_in[:, None]).T @ DY}
            for nm in names:
                acc[(nm, "in")] += ins[nm]
                acc[(nm, "out")] += full[nm] - ins[nm]
        return acc


def _broadcast_axis(g, k, d, q):
    """(Lc, q) per-axis coordinates broadcast to (Lc, q, ..., q) along axis k."""
    shape = [g.shape[0]] + [1] * d
    shape[1 + k] = q
    return np.broadcast_to(g.reshape(shape), (g.shape[0],) + (q,) * d)


def _tensor_weights(wd):
    d = len(wd)
    if d == 2:
        w = np.einsum("lq,lr->lqr", wd[0], wd[1])
    else:
        w = np.einsum("lq,lr,ls->lqrs", wd[0], wd[1], wd[2])
    return w.reshape(-1)


def hrz_lump(M):
    """HRZ lumped diagonal(s): diag scaled to the element mass (sum of all
    entries), src/stabilization.py:117-131."""
    M = np.asarray(M, dtype=float)
    diag = np.diagonal(M, axis1=-2, axis2=-1).copy()
    m_e = M.sum(axis=(-2, -1))
    scale = np.asarray(m_e) / diag.sum(axis=-1)
    return diag * scale[..., None] if diag.ndim > 1 else diag * scale


def row_sum_lump(M):
    """Row-sum lumped diagonal(s) computed as M @ 1 (src/stabilization.py:105-114)."""
    M = np.asarray(M, dtype=float)
    return M @ np.ones(M.shape[-1])
