"""The reference's benchmark geometry restated for the tests (TEST
INFRASTRUCTURE: imported only by tests/, never by the product package).

:class:`RotatedCube` -- cube of edge l_p rotated by Cardan angles inside
[0, l_e]^3 (src/geometry.py:128-272): separating-axis classification of
boxes, convex-hull volume of the box/cube intersection, and the sliver
certificate of src/assembly.py:187-211.  It lets the product's host set-up
(paper_2501_19013_b200/setup) be pinned to the reference's own grids, cut
cells and operators (tests/test_setup.py, tests/test_gpu_paper.py).
"""

from __future__ import annotations

import numpy as np

from paper_2501_19013_b200.setup.geometry import CUT, INSIDE, OUTSIDE, _corner_unit


class RotatedCube:
    """Cube of edge l_p rotated by Cardan angles inside [0, l_e]^3
    (src/geometry.py:128-272)."""

    dim = 3

    def __init__(self, l_p=0.3, l_e=0.5, angles_deg=(10.0, 10.0, 10.0), center=None):
        phi, theta, psi = np.radians(np.asarray(angles_deg, dtype=float))

        def rx(a):
            c, s = np.cos(a), np.sin(a)
            return np.array([[1.0, 0.0, 0.0], [0.0, c, -s], [0.0, s, c]])

        def ry(a):
            c, s = np.cos(a), np.sin(a)
            return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])

        def rz(a):
            c, s = np.cos(a), np.sin(a)
            return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])

        self.T = rz(psi) @ ry(theta) @ rx(phi)
        self.l_p, self.l_e = float(l_p), float(l_e)
        self.center = np.full(3, l_e / 2.0) if center is None else np.asarray(center, float)
        eye = np.eye(3)
        axes = [eye[i] for i in range(3)] + [self.T[:, i] for i in range(3)]
        axes += [np.cross(eye[i], self.T[:, j]) for i in range(3) for j in range(3)]
        self._axes = np.array(axes)
        self.domain_lo = np.zeros(3)
        self.domain_hi = np.full(3, self.l_e)

    def to_local(self, x):
        return (np.asarray(x, dtype=float) - self.center) @ self.T

    def to_global(self, x):
        return np.asarray(x, dtype=float) @ self.T.T + self.center

    def contains(self, x):
        return np.max(np.abs(self.to_local(x)), axis=-1) <= self.l_p / 2.0

    def classify_boxes(self, lo, hi):
        lo = np.atleast_2d(np.asarray(lo, dtype=float))
        hi = np.atleast_2d(np.asarray(hi, dtype=float))
        half = self.l_p / 2.0
        cu = _corner_unit(3)
        corners = lo[:, None, :] + cu[None] * (hi - lo)[:, None, :]
        inside = np.max(np.abs((corners - self.center) @ self.T), axis=(1, 2)) <= half
        d = 0.5 * (lo + hi) - self.center
        ew = 0.5 * (hi - lo)
        A = self._axes
        r_box = np.abs(A) @ ew.T
        r_cube = (np.abs(A @ self.T) @ np.full(3, half))[:, None]
        separated = np.any(np.abs(A @ d.T) > r_box + r_cube, axis=0)
        cls = np.full(lo.shape[0], CUT, dtype=np.int8)
        cls[separated] = OUTSIDE
        cls[inside] = INSIDE
        return cls

    def volume_fraction(self, lo, hi, stop_above=None):
        """Exact: convex hull of the box/cube intersection vertices
        (src/geometry.py:224-272)."""
        from scipy.spatial import ConvexHull, QhullError
        lo = np.asarray(lo, dtype=float)
        hi = np.asarray(hi, dtype=float)
        c = int(self.classify_boxes(lo[None], hi[None])[0])
        if c == INSIDE:
            return 1.0
        if c == OUTSIDE:
            return 0.0
        half = self.l_p / 2.0
        clo, chi = np.full(3, -half), np.full(3, half)
        cu = _corner_unit(3)
        box_c = lo + cu * (hi - lo)
        box_l = self.to_local(box_c)
        cube_l = clo + cu * (chi - clo)
        cube_g = self.to_global(cube_l)
        pts = [q for q in box_l if np.max(np.abs(q)) <= half + 1e-15]
        eps = 1e-15
        pts += [ql for qg, ql in zip(cube_g, cube_l)
                if np.all((qg >= lo - eps) & (qg <= hi + eps))]
        edges = [(0, 1), (2, 3), (4, 5), (6, 7), (0, 2), (1, 3), (4, 6), (5, 7),
                 (0, 4), (1, 5), (2, 6), (3, 7)]
        for a, b in edges:
            s = _clip(box_l[a], box_l[b], clo, chi)
            if s is not None:
                pts += list(s)
        for a, b in edges:
            s = _clip(cube_g[a], cube_g[b], lo, hi)
            if s is not None:
                pts += list(self.to_local(np.array(s)))
        if len(pts) < 4:
            return 0.0
        pts = np.unique(np.round(np.array(pts), 14), axis=0)
        if len(pts) < 4:
            return 0.0
        try:
            vol = ConvexHull(pts).volume
        except QhullError:
            try:
                vol = ConvexHull(pts, qhull_options="QJ").volume
            except QhullError:
                return 0.0
        return min(vol / float(np.prod(hi - lo)), 1.0)

    def sliver_candidates(self, lo, h):
        """Cut cells lacking an interior sample with margin 0.01 h
        (src/assembly.py:194-207)."""
        t = (2.0 * np.arange(4) + 1.0) / 8.0
        P = np.stack(np.meshgrid(t, t, t, indexing="ij"), axis=-1).reshape(-1, 3) * h
        pts = lo[:, None, :] + P[None]
        loc = self.to_local(pts.reshape(-1, 3)).reshape(lo.shape[0], -1, 3)
        margin = self.l_p / 2.0 - np.max(np.abs(loc), axis=-1)
        return np.flatnonzero(np.max(margin, axis=1) < 0.01 * h)


def _clip(p0, p1, lo, hi):
    """Liang-Barsky clip of segment p0-p1 to a box."""
    d = p1 - p0
    t0, t1 = 0.0, 1.0
    for i in range(p0.shape[0]):
        if d[i] == 0.0:
            if p0[i] < lo[i] or p0[i] > hi[i]:
                return None
        else:
            a = (lo[i] - p0[i]) / d[i]
            b = (hi[i] - p0[i]) / d[i]
            if a > b:
                a, b = b, a
            t0, t1 = max(t0, a), min(t1, b)
            if t0 > t1:
                return None
    return p0 + t0 * d, p0 + t1 * d
