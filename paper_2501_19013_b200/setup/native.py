"""Native (C++, multi-threaded) host set-up for ball-void geometries
(SURVEY 8(f)-2): the grid classification and the cut-cell integrals of
``setup/grid.py`` / ``setup/cutcell.py`` for ``BallVoids``, through
``wcb_setup_ball_classify`` / ``wcb_setup_ball_cut_cells`` of the C ABI.

The Python restatement stays the specification (tests compare the two to
rounding); ``WAVECELL_B200_PY_SETUP=1`` selects it.
"""

from __future__ import annotations

import os

import numpy as np

from .basis import dyadic_tables
from .geometry import BallVoids


def enabled(geom, family: str = "lagrange") -> bool:
    if os.environ.get("WAVECELL_B200_PY_SETUP", "0") == "1":
        return False
    if not isinstance(geom, BallVoids) or family != "lagrange":
        return False
    if not np.array_equal(geom.domain_lo, np.zeros(geom.dim)) or \
            not np.array_equal(geom.domain_hi, np.ones(geom.dim)):
        return False
    try:
        from .. import _lib
        _lib.load()
    except ImportError:
        return False
    return True


def lib_ok() -> bool:
    """The native library is there (geometry-independent set-up steps)."""
    if os.environ.get("WAVECELL_B200_PY_SETUP", "0") == "1":
        return False
    try:
        from .. import _lib
        _lib.load()
    except ImportError:
        return False
    return True


def dofmap(classes: np.ndarray, p: int):
    """(lex_of_compact, c_idx, d_idx, compact_of_lex) of a classified Lagrange
    grid (Grid.dofmap), all from one threaded pass."""
    from .. import _lib
    d, n_e = classes.ndim, classes.shape[0]
    cls = np.ascontiguousarray(classes, dtype=np.int8).reshape(-1)
    lib = _lib.load()
    nc = _lib.C.c_int64(0)
    n = lib.wcb_setup_dofmap(d, int(p), int(n_e), _lib.i8ptr(cls), None, None, _lib.C.byref(nc), None, None)
    if n < 0:
        _lib.check(int(-n))
    lex = np.empty(n, dtype=np.int64)
    c = np.empty(max(nc.value, 1), dtype=np.int64)
    dd = np.empty(max(n - nc.value, 1), dtype=np.int64)
    compact = np.empty((int(n_e) * int(p) + 1) ** d, dtype=np.int64)
    lib.wcb_setup_dofmap(d, int(p), int(n_e), _lib.i8ptr(cls), _lib.i64ptr(lex), _lib.i64ptr(c),
                         _lib.C.byref(nc), _lib.i64ptr(dd), _lib.i64ptr(compact))
    return lex, c[: nc.value], dd[: n - nc.value], compact


def lumped_mass(grid, w, sm: float, cut_M) -> np.ndarray:
    """ScmProblem._assemble_mass (same sums, same order)."""
    from .. import _lib
    cls = np.ascontiguousarray(grid.classes, dtype=np.int8).reshape(-1)
    dm = grid.dofmap
    m = np.empty(dm.n_dof)
    cm = np.ascontiguousarray(cut_M, dtype=np.float64).reshape(-1)
    cut = np.ascontiguousarray(grid.cut_lex if cm.size else np.zeros(0), dtype=np.int64)
    _lib.check(_lib.load().wcb_setup_lumped_mass(
        grid.dim, grid.p, grid.n_e, _lib.i8ptr(cls), _lib.dptr(np.ascontiguousarray(w, dtype=np.float64)),
        float(sm), dm.n_dof, _lib.i64ptr(np.ascontiguousarray(dm.lex_of_compact)), cut.shape[0],
        _lib.i64ptr(cut) if cut.size else None, _lib.dptr(cm) if cm.size else None,
        _lib.i64ptr(np.ascontiguousarray(dm.compact_of_lex)), _lib.dptr(m)))
    return m


def classify(geom: BallVoids, n_e: int) -> np.ndarray:
    """Cell classes (0 outside, 1 inside, 2 cut) of the n_e^d grid on [0,1]^d."""
    from .. import _lib
    d = geom.dim
    cls = np.empty((n_e,) * d, dtype=np.int8)
    c = np.ascontiguousarray(geom.centers, dtype=np.float64)
    r = np.ascontiguousarray(geom.radii, dtype=np.float64)
    _lib.check(_lib.load().wcb_setup_ball_classify(d, int(n_e), r.shape[0], _lib.dptr(c.reshape(-1)),
                                                   _lib.dptr(r), _lib.i8ptr(cls.reshape(-1))))
    return cls


def slivers(geom: BallVoids, n_e: int, cut_lex, min_fraction: float) -> np.ndarray:
    """Mask of the cut cells the sliver rule demotes (setup/grid.py _discard_slivers)."""
    import ctypes as C
    from .. import _lib
    d = geom.dim
    cut = np.ascontiguousarray(cut_lex, dtype=np.int64)
    out = np.zeros(cut.shape[0], dtype=np.uint8)
    c = np.ascontiguousarray(geom.centers, dtype=np.float64).reshape(-1)
    r = np.ascontiguousarray(geom.radii, dtype=np.float64)
    if cut.shape[0]:
        _lib.check(_lib.load().wcb_setup_ball_slivers(
            d, int(n_e), r.shape[0], _lib.dptr(c), _lib.dptr(r), cut.shape[0], _lib.i64ptr(cut),
            float(min_fraction), 26 // d + 1, out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out.astype(bool)


def cut_cells(grid, depth: int, cells, alpha: float, sk: float, sm: float, lumping: str,
              q: int | None = None, nthreads: int = 0):
    """(K_o (n, L, L), M (n, L) lumped or (n, L, L) consistent) of the cut cells."""
    from .. import _lib
    geom = grid.geom
    d, p = grid.dim, grid.p
    N = p + 1
    L = N ** d
    q = p + 1 if q is None else int(q)
    t = dyadic_tables(grid.basis, 0, int(depth), q)
    arr = {k: np.ascontiguousarray(t[k], dtype=np.float64).reshape(-1)
           for k in ("xi", "w", "V", "D", "m1", "k1")}
    offs = np.ascontiguousarray(t["offsets"], dtype=np.int64)
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    n = cells.shape[0]
    K = np.empty((n, L, L))
    lump = {"none": 0, "hrz": 1, "row_sum": 2}[lumping]
    M = np.empty((n, L, L)) if lump == 0 else np.empty((n, L))
    c = np.ascontiguousarray(geom.centers, dtype=np.float64).reshape(-1)
    r = np.ascontiguousarray(geom.radii, dtype=np.float64)
    if n:
        _lib.check(_lib.load().wcb_setup_ball_cut_cells(
            d, p, int(grid.n_e), r.shape[0], _lib.dptr(c), _lib.dptr(r), int(depth), q, _lib.i64ptr(offs),
            _lib.dptr(arr["xi"]), _lib.dptr(arr["w"]), _lib.dptr(arr["V"]), _lib.dptr(arr["D"]),
            _lib.dptr(arr["m1"]), _lib.dptr(arr["k1"]), n, _lib.i64ptr(cells), float(alpha), float(sk),
            float(sm), lump, int(nthreads), _lib.dptr(K.reshape(-1)), _lib.dptr(M.reshape(-1))))
    return K, M
