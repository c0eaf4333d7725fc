"""Immersed geometries for the host-side set-up (cell classification,
point membership, volume fractions).

Every geometry exposes the interface the reference's ``ImmersedGeometry``
gives the mesh layer (src/geometry.py:128-272):

* ``dim``
* ``contains(x)`` -- points (..., d) in the closed physical domain;
* ``classify_boxes(lo, hi)`` -- exact ElementClass per axis-aligned box
  (0 outside, 1 inside, 2 cut; src/geometry.py:36-41);
* ``volume_fraction(lo, hi)`` -- physical fraction of one box;
* ``sliver_candidates(lo, h)`` -- the cheap interior-sample certificate of
  src/assembly.py:187-211 (cells not listed certainly exceed the threshold).

Plug-ins:

* :class:`BallVoids` -- unit square / cube minus a union of open disks /
  balls (BASELINE configs 1, 2, 4, 5).
* :class:`PolygonVoid` -- unit square minus one simple polygon (config 3).

The reference's own benchmark geometry (the rotated cube) is restated in
``oracle/geometry_cube.py``: it is test infrastructure (it pins this set-up
to the reference's grids), not part of the product.

Voids are open sets: points on a void boundary belong to the material, as
the reference's closed cube does (src/geometry.py:187-190).
"""

from __future__ import annotations

import numpy as np

OUTSIDE, INSIDE, CUT = 0, 1, 2
MIN_VOLUME_FRACTION = 2.0 ** -24   # src/geometry.py:33


def _corner_unit(d):
    """Corner offsets, last axis fastest (src/geometry.py:110-112)."""
    g = np.stack(np.meshgrid(*([np.array([0.0, 1.0])] * d), indexing="ij"), axis=-1)
    return g.reshape(-1, d)


def split_children(lo, hi):
    """2^d congruent children of each box (src/geometry.py:120-125)."""
    d = lo.shape[1]
    cu = _corner_unit(d)
    mid = 0.5 * (lo + hi)
    clo = np.where(cu[None] == 0, lo[:, None, :], mid[:, None, :])
    chi = np.where(cu[None] == 0, mid[:, None, :], hi[:, None, :])
    return clo.reshape(-1, d), chi.reshape(-1, d)


def tree_partition(geom, lo, hi, max_depth):
    """Leaves of the recursive 2^d-section of one cut box, deterministic order
    (src/geometry.py:316-346).  Returns (lo, hi, cls, depth)."""
    if max_depth < 0:
        raise ValueError("max_depth must be >= 0")
    lo = np.asarray(lo, dtype=float)[None, :].copy()
    hi = np.asarray(hi, dtype=float)[None, :].copy()
    outs = []
    for depth in range(max_depth + 1):
        cls = geom.classify_boxes(lo, hi)
        cut = cls == CUT
        settled = ~cut if depth < max_depth else np.ones(cls.shape[0], dtype=bool)
        if np.any(settled):
            outs.append((lo[settled], hi[settled], cls[settled],
                         np.full(int(settled.sum()), depth)))
        if depth == max_depth or not np.any(cut):
            break
        lo, hi = split_children(lo[cut], hi[cut])
    return tuple(np.concatenate([o[i] for o in outs]) for i in range(4))


def _fraction_by_subdivision(geom, lo, hi, depth, stop_above=None):
    """Physical fraction of one box by adaptive 2^d-section: settled leaves
    count exactly, cut leaves at ``depth`` by their centre point.  With
    ``stop_above`` the walk returns as soon as the certified inside volume
    exceeds that fraction (enough to decide the sliver rule)."""
    lo = np.asarray(lo, dtype=float)[None, :]
    hi = np.asarray(hi, dtype=float)[None, :]
    vol = float(np.prod(hi - lo))
    acc = 0.0
    for level in range(depth + 1):
        cls = geom.classify_boxes(lo, hi)
        w = np.prod(hi - lo, axis=1)
        acc += float(np.sum(w[cls == INSIDE]))
        if stop_above is not None and acc > stop_above * vol:
            return acc / vol
        cut = cls == CUT
        if level == depth:
            c = 0.5 * (lo[cut] + hi[cut])
            acc += float(np.sum(w[cut][geom.contains(c)]))
            break
        if not np.any(cut):
            break
        lo, hi = split_children(lo[cut], hi[cut])
    return acc / vol


class BallVoids:
    """Unit square (d=2) or cube (d=3) minus a union of open disks/balls."""

    def __init__(self, dim, centers, radii):
        self.dim = int(dim)
        self.centers = np.asarray(centers, dtype=float).reshape(-1, self.dim)
        self.radii = np.asarray(radii, dtype=float).reshape(-1)
        self.domain_lo = np.zeros(self.dim)
        self.domain_hi = np.ones(self.dim)

    def restricted(self, lo, hi):
        """Same geometry inside the box [lo, hi]: only the voids that reach it."""
        near = np.clip(self.centers, lo, hi) - self.centers
        sel = np.sum(near * near, axis=1) < self.radii ** 2
        out = BallVoids(self.dim, self.centers[sel], self.radii[sel])
        return out

    def contains(self, x):
        x = np.asarray(x, dtype=float)
        flat = x.reshape(-1, self.dim)
        ok = np.ones(flat.shape[0], dtype=bool)
        for c, r in zip(self.centers, self.radii):
            ok &= np.sum((flat - c) ** 2, axis=1) >= r * r
        ok &= np.all((flat >= self.domain_lo) & (flat <= self.domain_hi), axis=1)
        return ok.reshape(x.shape[:-1])

    def classify_boxes(self, lo, hi):
        """INSIDE: the closed box misses every open void; OUTSIDE: the box lies
        in one void (all corners strictly inside it -- balls are convex); CUT
        otherwise.  Boxes covered only by a union of several voids come out
        CUT and are demoted by the sliver rule."""
        lo = np.atleast_2d(np.asarray(lo, dtype=float))
        hi = np.atleast_2d(np.asarray(hi, dtype=float))
        n = lo.shape[0]
        touches = np.zeros(n, dtype=bool)
        covered = np.zeros(n, dtype=bool)
        for c, r in zip(self.centers, self.radii):
            near = np.clip(c, lo, hi) - c
            touches |= np.sum(near * near, axis=1) < r * r
            far = np.maximum(np.abs(lo - c), np.abs(hi - c))
            covered |= np.sum(far * far, axis=1) < r * r
        cls = np.full(n, INSIDE, dtype=np.int8)
        cls[touches] = CUT
        cls[covered] = OUTSIDE
        return cls

    def volume_fraction(self, lo, hi, depth=None, stop_above=None):
        depth = (26 // self.dim + 1) if depth is None else depth
        return _fraction_by_subdivision(self, lo, hi, depth, stop_above)

    def sliver_candidates(self, lo, h):
        """Cut cells without an interior sample point whose distance to every
        void boundary is >= 0.01 h (the material then holds a ball of radius
        0.01 h, far above the 2^-24 threshold)."""
        d = self.dim
        t = (2.0 * np.arange(4) + 1.0) / 8.0
        P = np.stack(np.meshgrid(*([t] * d), indexing="ij"), axis=-1).reshape(-1, d) * h
        pts = lo[:, None, :] + P[None]
        flat = pts.reshape(-1, d)
        margin = np.full(flat.shape[0], np.inf)
        for c, r in zip(self.centers, self.radii):
            margin = np.minimum(margin, np.sqrt(np.sum((flat - c) ** 2, axis=1)) - r)
        margin = margin.reshape(lo.shape[0], -1)
        return np.flatnonzero(np.max(margin, axis=1) < 0.01 * h)


class PolygonVoid:
    """Unit square minus the interior of one simple polygon (2D)."""

    dim = 2

    def __init__(self, vertices):
        self.v = np.asarray(vertices, dtype=float).reshape(-1, 2)
        self.domain_lo = np.zeros(2)
        self.domain_hi = np.ones(2)

    def _inside_polygon(self, pts):
        """Even-odd ray casting (strict interior, boundary -> material)."""
        x, y = pts[:, 0], pts[:, 1]
        inside = np.zeros(pts.shape[0], dtype=bool)
        v = self.v
        for i in range(v.shape[0]):
            (x0, y0), (x1, y1) = v[i], v[(i + 1) % v.shape[0]]
            cond = (y0 > y) != (y1 > y)
            with np.errstate(divide="ignore", invalid="ignore"):
                xc = x0 + (y - y0) * (x1 - x0) / (y1 - y0)
            inside ^= cond & (x < xc)
        return inside

    def contains(self, x):
        x = np.asarray(x, dtype=float)
        flat = x.reshape(-1, 2)
        ok = ~self._inside_polygon(flat)
        ok &= np.all((flat >= 0.0) & (flat <= 1.0), axis=1)
        return ok.reshape(x.shape[:-1])

    def _edges_hit_boxes(self, lo, hi):
        """Whether any polygon edge meets each closed box (slab clipping)."""
        n = lo.shape[0]
        hit = np.zeros(n, dtype=bool)
        v = self.v
        for i in range(v.shape[0]):
            p0, p1 = v[i], v[(i + 1) % v.shape[0]]
            d = p1 - p0
            t0 = np.zeros(n)
            t1 = np.ones(n)
            ok = np.ones(n, dtype=bool)
            for a in range(2):
                if d[a] == 0.0:
                    ok &= (p0[a] >= lo[:, a]) & (p0[a] <= hi[:, a])
                else:
                    ta = (lo[:, a] - p0[a]) / d[a]
                    tb = (hi[:, a] - p0[a]) / d[a]
                    t0 = np.maximum(t0, np.minimum(ta, tb))
                    t1 = np.minimum(t1, np.maximum(ta, tb))
            hit |= ok & (t0 <= t1)
        return hit

    def classify_boxes(self, lo, hi):
        lo = np.atleast_2d(np.asarray(lo, dtype=float))
        hi = np.atleast_2d(np.asarray(hi, dtype=float))
        edge = self._edges_hit_boxes(lo, hi)
        centre_in = self._inside_polygon(0.5 * (lo + hi))
        cls = np.full(lo.shape[0], INSIDE, dtype=np.int8)
        cls[~edge & centre_in] = OUTSIDE
        cls[edge] = CUT
        return cls

    def volume_fraction(self, lo, hi, depth=14, stop_above=None):
        return _fraction_by_subdivision(self, lo, hi, depth, stop_above)

    def sliver_candidates(self, lo, h):
        return np.arange(lo.shape[0])
