"""Device IMEX (src/timeint.py:196-292) against the reference's own IMEX
tests (tests/test_timeint.py:109-174,229-243 of the reference), its golden
outputs, and the CPU oracle on a 2D void problem with consistent cut mass."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import IMEX_A12_TOL_P2N4, csr_from, load_golden
from oracle import timeint as O

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import cdm_run, imex_run, newmark_run  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def bar():
    g = load_golden("bar")
    return sp.csr_matrix(g["M"]), sp.csr_matrix(g["K"]), g


def test_imex_empty_c_equals_cdm():
    M, K, g = bar()
    F = np.array([0.0, 1.0, 0.5, 0.2])
    obs = sp.identity(4, format="csr")
    f = lambda t: np.sin(6.0 * t)
    r_imex = imex_run(M, K, F, f, 5e-3, 200, np.array([], dtype=int), np.arange(4), obs_mat=obs)
    r_cdm = cdm_run(M, K, F, f, 5e-3, 200, obs_mat=obs)
    assert np.abs(r_imex.obs - r_cdm.obs).max() <= 1e-12
    assert r_imex.fact_dim == 0


def test_imex_empty_d_equals_newmark_golden():
    M, K, g = bar()
    Mc = sp.csr_matrix(g["Mc"])
    f = lambda t: np.sin(6.0 * t)
    r = imex_run(Mc, K, g["F"], f, float(g["dt"]), int(g["n_t"]), np.arange(4),
                 np.array([], dtype=int), obs_mat=sp.identity(4, format="csr"))
    assert np.abs(r.obs - g["imexc_obs"]).max() <= 1e-12 * max(np.abs(g["imexc_obs"]).max(), 1.0)
    assert np.abs(r.psi_dot - g["imexc_vdot"]).max() <= 1e-12 * max(np.abs(g["imexc_vdot"]).max(), 1.0)
    assert r.fact_dim == 4


def test_imex_split_bar_matches_reference():
    M, K, g = bar()
    f = lambda t: np.sin(6.0 * t)
    r = imex_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]), np.array([1, 2]),
                 np.array([0, 3]), obs_mat=sp.identity(4, format="csr"))
    assert np.abs(r.obs - g["imex_obs"]).max() <= 1e-13 * np.abs(g["imex_obs"]).max()
    assert r.psi_dot is None and r.fact_dim == 2


def test_imex_second_order_on_split_bar():
    M, K, _ = bar()
    F = np.array([0.0, 1.0, 0.5, 0.2])
    obs = sp.identity(4, format="csr")
    f = lambda t: np.sin(6.0 * t)
    _, _, ref = O.newmark_run(M, K, F, f, 1.0 / 25600, 25600, obs_mat=obs)
    errs = []
    for n_t in (50, 100, 200):
        r = imex_run(M, K, F, f, 1.0 / n_t, n_t, np.array([1, 2]), np.array([0, 3]), obs_mat=obs)
        errs.append(np.linalg.norm(r.obs[:, ::n_t // 50] - ref[:, ::512]))
    assert 3.0 <= errs[0] / errs[1] <= 5.0
    assert 3.0 <= errs[1] / errs[2] <= 5.0


def test_imex_rejects_bad_partitions():
    M, K, _ = bar()
    F = np.zeros(4)
    z = lambda t: 0.0
    with pytest.raises(ValueError, match="partition"):
        imex_run(M, K, F, z, 1e-3, 3, np.array([1]), np.array([0, 3]))
    M_cons = sp.csr_matrix(np.array([[2.0, 1.0, 0.0, 0.0], [1.0, 4.0, 1.0, 0.0],
                                     [0.0, 1.0, 4.0, 1.0], [0.0, 0.0, 1.0, 2.0]]) / 18.0)
    with pytest.raises(ValueError, match="couple"):
        imex_run(M_cons, K, F, z, 1e-3, 3, np.array([1, 2]), np.array([0, 3]))
    with pytest.raises(ValueError, match="not diagonal"):
        imex_run(M_cons, K, F, z, 1e-3, 3, np.array([], dtype=int), np.arange(4))


@pytest.mark.parametrize("name,tol", [
    # alpha = 1e-4: a 2e-16 relative perturbation of K moves the reference's
    # own 150-step field by 4e-13 -> the north-star bar 1e-10 applies.
    ("cube_imex_p2n4_a4", 1e-10),
    # alpha = 1e-12 (the paper's IMEX case): cond(S_cc) ~ 5e13 and a 1-ulp
    # perturbation of K alone moves the reference's field by ~3e-8
    # (tests/test_paper_setup.py measures it); conftest.IMEX_A12_TOL_P2N4.
    ("cube_imex_p2n4", IMEX_A12_TOL_P2N4)])
def test_imex_cube_matches_reference_golden(name, tol):
    """Reference rotated cube, consistent cut mass: 150 IMEX steps at 0.9 x the
    d-subsystem critical step (reference output pinned)."""
    g = load_golden(name)
    M, K = csr_from(g, "M"), csr_from(g, "K")
    f = lambda t: O.ricker(t, 10.0)
    r = imex_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]), g["c_idx"], g["d_idx"],
                 obs_mat=csr_from(g, "obs"))
    assert rel(r.psi, g["psi"]) <= tol
    assert rel(r.obs, g["obs"]) <= tol
    assert r.fact_dim == g["c_idx"].shape[0]


def test_imex_scm_operator_2d_voids():
    """Matrix-free SCM K with consistent cut mass: device IMEX vs the oracle."""
    from paper_2501_19013_b200.setup.configs import ricker
    from paper_2501_19013_b200.setup.geometry import BallVoids
    from paper_2501_19013_b200.setup.grid import Grid
    from paper_2501_19013_b200.setup.problem import ScmProblem
    from paper_2501_19013_b200 import imex_critical_time_step
    geom = BallVoids(2, [[0.5, 0.5], [0.2, 0.75]], [0.23, 0.09])
    prob = ScmProblem.build(Grid.build(geom, "lagrange", 4, 24), 1e-6, 3, lumping="none")
    prob.set_point_source([0.15, 0.2])
    M = prob.mass_matrix()
    K = prob.csr_stiffness()
    op = prob.device_operator()
    dm = prob.grid.dofmap
    dtd = imex_critical_time_step(op, M, dm.d_idx, tol=1e-7)
    dtd_ref = 2.0 / np.sqrt(O.max_gen_eig(K[dm.d_idx][:, dm.d_idx], M[dm.d_idx][:, dm.d_idx],
                                          tol=1e-7)[0])
    assert abs(dtd - dtd_ref) <= 1e-10 * dtd_ref
    f = lambda t: ricker(t, 10.0)
    dt = 0.9 * dtd_ref
    psi_ref, _, _ = O.imex_run(M, K, prob.F_s, f, dt, 200, dm.c_idx, dm.d_idx)
    r = imex_run(M, op, prob.F_s, f, dt, 200, dm.c_idx, dm.d_idx)
    assert rel(r.psi, psi_ref) <= 1e-10
    r2 = imex_run(M, K, prob.F_s, f, dt, 200, dm.c_idx, dm.d_idx)
    assert rel(r2.psi, psi_ref) <= 1e-10


def test_newmark_run_matches_reference_golden():
    """newmark_run drop-in (src/timeint.py:109-156) vs the reference's own output."""
    M, K, g = bar()
    f = lambda t: np.sin(6.0 * t)
    r = newmark_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]),
                    obs_mat=sp.identity(4, format="csr"))
    assert np.abs(r.obs - g["nm_obs"]).max() <= 1e-12 * np.abs(g["nm_obs"]).max()
    assert r.method == "newmark" and r.fact_dim == 4 and r.psi_dot.shape == (4,)
    r0 = newmark_run(M, K, g["F"], f, float(g["dt"]), 50, beta=0.0)
    psi_ref, v_ref, _ = O.newmark_run(M, K, g["F"], f, float(g["dt"]), 50, beta=0.0)
    assert rel(r0.psi, psi_ref) <= 1e-12 and rel(r0.psi_dot, v_ref) <= 1e-12
    with pytest.raises(TypeError):
        newmark_run(M, K, g["F"], f, 1e-3, 3, s_factory=lambda: None)   # no .solve


def test_newmark_scm_operator_matches_oracle():
    """Whole-system Newmark with the matrix-free SCM K on a 2D void problem."""
    from paper_2501_19013_b200.setup.configs import ricker
    from paper_2501_19013_b200.setup.geometry import BallVoids
    from paper_2501_19013_b200.setup.grid import Grid
    from paper_2501_19013_b200.setup.problem import ScmProblem
    geom = BallVoids(2, [[0.5, 0.5]], [0.21])
    prob = ScmProblem.build(Grid.build(geom, "lagrange", 3, 12), 1e-3, 2)
    prob.set_point_source([0.15, 0.2])
    M = prob.mass_matrix()
    K = prob.csr_stiffness()
    op = prob.device_operator()
    f = lambda t: ricker(t, 10.0)
    dt = 2e-3
    psi_ref, v_ref, _ = O.newmark_run(M, K, prob.F_s, f, dt, 120)
    r = newmark_run(M, op, prob.F_s, f, dt, 120)
    assert rel(r.psi, psi_ref) <= 1e-10 and rel(r.psi_dot, v_ref) <= 1e-10
