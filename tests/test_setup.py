"""Host-side set-up restatement pinned to the reference (CPU only).

The product's set-up (paper_2501_19013_b200/setup) restates the reference's
basis, grid, DOF map, cut-cell integration and assembly for d = 2, 3.  On the
reference's own geometry (the rotated cube) it must reproduce the reference's
outputs, recorded as golden vectors by tests/golden/make_golden.py."""

import numpy as np
import pytest

from conftest import csr_from, load_golden
from paper_2501_19013_b200.setup import basis as B
from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm
from oracle.geometry_cube import RotatedCube
from paper_2501_19013_b200.setup.geometry import BallVoids, PolygonVoid
from paper_2501_19013_b200.setup.grid import Grid
from paper_2501_19013_b200.setup.problem import ScmProblem


def test_basis_matches_reference():
    g = load_golden("basis")
    x = np.linspace(-1.0, 1.0, 13)
    for p in range(1, 8):
        nodes, w = B.gll_rule(p)
        assert np.array_equal(nodes, g[f"gll{p}_x"]) and np.array_equal(w, g[f"gll{p}_w"])
        V, D = B.lagrange_eval(nodes, x)
        assert np.abs(V - g[f"lag{p}_V"]).max() <= 1e-14
        assert np.abs(D - g[f"lag{p}_D"]).max() <= 1e-12
    for p in (2, 3):
        span, V, D = B.bspline_eval(B.open_uniform_knots(7, p), p, np.linspace(0, 1, 29))
        assert np.array_equal(span, g[f"bs{p}_span"])
        assert np.abs(V - g[f"bs{p}_V"]).max() <= 1e-14
        assert np.abs(D - g[f"bs{p}_D"]).max() <= 1e-13
    for p in range(1, 6):
        b = B.Basis1D("lagrange", p, 2)
        m1, k1 = B.uncut_1d(b, 0)
        assert np.abs(m1 - g[f"m1_{p}"]).max() <= 1e-15
        assert np.abs(k1 - g[f"k1_{p}"]).max() <= 1e-13


@pytest.mark.parametrize("family,p,n_e,expected", [
    ("lagrange", 2, 28, 52353), ("lagrange", 3, 13, 22816), ("lagrange", 4, 9, 21109),
    ("lagrange", 5, 7, 22706), ("bspline", 2, 34, 14122), ("bspline", 3, 32, 14073)])
def test_dof_counts_match_reference(family, p, n_e, expected):
    # lagrange: PAPER table (exact); bspline: the reference's own counts
    assert Grid.build(RotatedCube(), family, p, n_e).n_dof == expected


@pytest.mark.parametrize("name,p,n_e,alpha,depth", [
    ("cube_p2n4", 2, 4, 1e-6, 2), ("cube_p3n6", 3, 6, 1e-8, 3)])
def test_cube_system_matches_reference(name, p, n_e, alpha, depth):
    g = load_golden(name)
    grid = Grid.build(RotatedCube(), "lagrange", p, n_e)
    assert np.array_equal(grid.classes.ravel(), g["cell_class"])
    assert np.array_equal(grid.dofmap.lex_of_compact, g["lex_of_compact"])
    assert np.array_equal(grid.cut_lex, g["cut_cells"])
    assert np.array_equal(grid.dofmap.c_idx, g["c_idx"])
    prob = ScmProblem.build(grid, alpha, depth)
    assert np.abs(prob.m_diag - g["M"]).max() <= 1e-14 * g["M"].max()
    assert np.abs(prob.cut_K - g["cut_K"]).max() <= 1e-14 * np.abs(g["cut_K"]).max()
    assert np.abs(prob.k1 - g["k1"]).max() == 0.0
    K = prob.csr_stiffness()
    assert np.abs(K @ g["X"] - g["KX"]).max() <= 1e-14 * np.abs(g["KX"]).max()
    if "K_data" in g:
        Kr = csr_from(g, "K")
        assert K.nnz == Kr.nnz
        assert abs(K - Kr).max() <= 1e-14 * abs(Kr).max()


def test_scm_invariants_2d_voids():
    """K 1 = 0, symmetry, alpha-affinity and total mass on a 2D void grid
    (the reference's tests/test_assembly.py:57-100 invariants)."""
    geom = BallVoids(2, [[0.5, 0.5], [0.2, 0.3]], [0.25, 0.07])
    grid = Grid.build(geom, "lagrange", 3, 12)
    pa = ScmProblem.build(grid, 1e-2, 3)
    pb = ScmProblem.build(grid, 1e-6, 3)
    pm = ScmProblem.build(grid, 0.5 * (1e-2 + 1e-6), 3)
    K = pa.csr_stiffness()
    assert np.abs(K @ np.ones(K.shape[0])).max() <= 1e-12 * np.abs(K.data).max()
    assert abs(K - K.T).max() <= 1e-13 * np.abs(K.data).max()
    Km = pm.csr_stiffness()
    d = 0.5 * (K + pb.csr_stiffness()) - Km
    assert abs(d).max() <= 1e-14 * np.abs(Km.data).max()
    area = 1.0 - np.pi * 0.25 ** 2 - np.pi * 0.07 ** 2
    assert abs(pb.m_diag.sum() - area) <= 2e-3 * area
    assert (pa.m_diag > 0).all()


def test_polygon_and_ball_classification_consistent():
    poly = PolygonVoid([[0.3, 0.3], [0.7, 0.35], [0.6, 0.7], [0.35, 0.6]])
    balls = BallVoids(3, [[0.5, 0.5, 0.5]], [0.3])
    for geom in (poly, balls):
        d = geom.dim
        rng = np.random.default_rng(0)
        lo = rng.uniform(0, 0.9, (400, d))
        hi = lo + rng.uniform(0.01, 0.1, (400, d))
        cls = geom.classify_boxes(lo, hi)
        pts = lo[:, None, :] + rng.uniform(0, 1, (400, 64, d)) * (hi - lo)[:, None, :]
        inside = geom.contains(pts.reshape(-1, d)).reshape(400, 64)
        assert inside[cls == 1].all()          # inside boxes: every sample is material
        assert not inside[cls == 0].any()      # outside boxes: no sample is material


def test_config1_sizes():
    prob = build_scm(CONFIGS["config1"])
    assert prob.n_dof == 14128
    assert prob.grid.cut_lex.shape[0] == 60
    assert (prob.m_diag > 0).all()
    assert prob.F_s.sum() == pytest.approx(1.0)   # partition of unity at the source


def test_bspline_cube_system_matches_reference():
    """IGA-FCM assembly (stencil CSR + cut cells + row-sum lumping) vs the
    reference's own assemble() on its rotated cube (golden)."""
    from paper_2501_19013_b200.setup.iga import IgaProblem
    g = load_golden("bspline_cube_p2n5")
    grid = Grid.build(RotatedCube(), "bspline", 2, 5)
    assert np.array_equal(grid.dofmap.lex_of_compact, g["lex_of_compact"])
    prob = IgaProblem.build(grid, 1e-6, 2)
    Kr = csr_from(g, "K")
    assert prob.K.nnz == Kr.nnz
    assert abs(prob.K - Kr).max() <= 1e-14 * abs(Kr).max()
    assert np.abs(prob.m_diag - g["M"]).max() <= 1e-14 * g["M"].max()
