"""CPU checks behind tests/test_gpu_paper.py and the alpha = 1e-12 IMEX
tolerances (conftest.IMEX_A12_TOL_*):

* the host set-up restatement rebuilds the reference's benchmark systems
  (rotated cube, SCM p=3, n_e 13 and 10, octree depth 4, consistent cut
  mass) -- K X and M X agree with the reference's to rounding;
* the reference arithmetic (oracle) on the alpha = 1e-12 IMEX systems moves
  by the measured spread under a symmetric 1-ulp perturbation of K, which
  bounds how closely any other summation order (the device's) can match.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import IMEX_A12_TOL_N13, IMEX_A12_TOL_P2N4, NEAR_CRITICAL_TOL, csr_from, load_golden
from oracle import timeint as O
from oracle.geometry_cube import RotatedCube
from paper_2501_19013_b200.setup.configs import ricker
from paper_2501_19013_b200.setup.grid import Grid
from paper_2501_19013_b200.setup.problem import ScmProblem


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def f(t):
    return ricker(t, 10.0)


def perturbed(K, seed):
    """K with every stored value moved by +-1 ulp (kept symmetric)."""
    rng = np.random.default_rng(seed)
    Kp = sp.csr_matrix(K, copy=True)
    Kp.data = Kp.data * (1.0 + rng.choice([-1.0, 1.0], Kp.data.shape) * 2.0 ** -52)
    return ((Kp + Kp.T) * 0.5).tocsr()


@pytest.fixture(scope="module")
def n13():
    grid = Grid.build(RotatedCube(), "lagrange", 3, 13)
    return grid, ScmProblem.build(grid, 1e-8, 4, lumping="none"), \
        ScmProblem.build(grid, 1e-12, 4, lumping="none")


def test_paper_systems_match_reference(n13):
    g = load_golden("paper_n13")
    grid, p8, p12 = n13
    assert grid.n_dof == 22816 and grid.n_dof == g["X"].shape[0]
    for tag, p in (("8", p8), ("12", p12)):
        K, M = p.csr_stiffness(), p.mass_matrix()
        assert rel(K @ g["X"], g["KX" + tag]) <= 1e-15
        assert rel(M @ g["X"], g["MX" + tag]) <= 1e-15
        assert M.nnz > M.shape[0]                   # consistent cut-cell blocks
    assert p8.mass_matrix().nnz == int(g["Mnnz8"])
    g10 = load_golden("paper_n10")
    grid10 = Grid.build(RotatedCube(), "lagrange", 3, 10)
    p10 = ScmProblem.build(grid10, 1e-8, 4, lumping="none")
    assert rel(p10.csr_stiffness() @ g10["X"], g10["KX"]) <= 1e-15
    assert rel(p10.mass_matrix() @ g10["X"], g10["MX"]) <= 1e-15


def test_imex_alpha12_sensitivity_cube_p2n4():
    """150 IMEX steps of the reference cube (p=2, n_e=4, alpha 1e-12): the
    reference's own field under 1-ulp perturbations of K."""
    g = load_golden("cube_imex_p2n4")
    M, K = csr_from(g, "M"), csr_from(g, "K")
    args = (g["F"], f, float(g["dt"]), int(g["n_t"]), g["c_idx"], g["d_idx"])
    base, _, _ = O.imex_run(M, K, *args)
    assert np.array_equal(base, g["psi"])            # the oracle is the reference here
    spread = max(rel(O.imex_run(M, perturbed(K, s), *args)[0], base) for s in range(4))
    # the device tolerance is a small multiple of the reference's own spread
    assert 1e-9 <= spread <= IMEX_A12_TOL_P2N4 <= 10.0 * spread, spread


def test_imex_alpha12_sensitivity_paper_n13(n13):
    """2000 IMEX steps of the paper's alpha = 1e-12 case (n_e 13): the
    restated set-up (K within 1e-16 of the reference's) and a 1-ulp
    perturbation both move the reference-arithmetic field by ~1e-6."""
    g = load_golden("paper_n13")
    grid, _, p12 = n13
    K, M = p12.csr_stiffness(), p12.mass_matrix()
    dm = grid.dofmap
    args = (g["F12"], f, 0.9 * float(g["dtd12"]), 2000, dm.c_idx, dm.d_idx)
    base, _, _ = O.imex_run(M, K, *args)
    setup_dev = rel(base, g["psi12"])
    spread = rel(O.imex_run(M, perturbed(K, 5), *args)[0], base)
    assert setup_dev <= IMEX_A12_TOL_N13 and 1e-7 <= spread <= IMEX_A12_TOL_N13 <= 10.0 * spread, \
        (setup_dev, spread)


def test_near_critical_cdm_sensitivity_paper_n10():
    """2000 consistent-mass CDM steps at 0.99 dt_crit (criterion 3, n_e 10):
    the reference arithmetic moves by ~2e-10 under a 1-ulp perturbation of
    K, which is why the device check of this case uses NEAR_CRITICAL_TOL."""
    g = load_golden("paper_n10")
    grid = Grid.build(RotatedCube(), "lagrange", 3, 10)
    p = ScmProblem.build(grid, 1e-8, 4, lumping="none")
    K, M = p.csr_stiffness(), p.mass_matrix()
    args = (g["F"], f, 0.99 * float(g["dtc"]), 2000)
    base, _, _ = O.cdm_run(M, K, *args)
    assert rel(base, g["psi"]) <= NEAR_CRITICAL_TOL
    spread = rel(O.cdm_run(M, perturbed(K, 1), *args)[0], base)
    assert 1e-11 <= spread <= NEAR_CRITICAL_TOL <= 10.0 * spread, spread
