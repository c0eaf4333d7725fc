"""Eigenvalue stabilisation on the device: the batched Jacobi
eigensolver and evs_stabilize against the reference's own outputs
(tests/golden/make_golden.py gen_evs: src/linalg.py:133-212,
src/stabilization.py:73-102), and an EVS-stabilised cut-cell problem run
through the device integrator."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200.stabilization import evs_stabilize, jacobi_eig  # noqa: E402


def test_jacobi_eig_matches_reference():
    g = load_golden("evs")
    lam, V = jacobi_eig(g["A"])
    scale = np.abs(g["lam"]).max(axis=1, keepdims=True)
    assert np.abs(lam - g["lam"]).max() <= 1e-13 * scale.max()
    # eigenvectors: orthonormal and reproducing A (columns up to sign)
    rec = np.einsum("bik,bk,bjk->bij", V, lam, V)
    assert np.abs(rec - g["A"]).max() <= 1e-13 * np.abs(g["A"]).max()
    dots = np.abs(np.einsum("bik,bik->bk", V, g["V"]))
    assert np.all(np.abs(dots - 1.0) <= 1e-8)
    lam1, V1 = jacobi_eig(g["A"][3])
    assert lam1.shape == (27,) and np.abs(lam1 - g["lam"][3]).max() <= 1e-13 * scale[3, 0]


def test_evs_stabilize_matches_reference():
    g = load_golden("evs")
    out = evs_stabilize(g["A"], g["Mf"], 0.1, 1e-2)
    assert np.abs(out - g["evs"]).max() <= 1e-12 * np.abs(g["evs"]).max()
    out_c = evs_stabilize(g["Mo_c"], g["Mf_c"], 0.01, 1e-2)
    assert np.abs(out_c - g["evs_c"]).max() <= 1e-12 * np.abs(g["evs_c"]).max()
    assert np.array_equal(evs_stabilize(g["Mo_c"], g["Mf_c"], 0.0), g["Mo_c"])


def test_evs_stabilised_problem_runs():
    """alpha = 1e-8 cut cells with EVS (epsilon 0.01): larger critical step
    than without, device CDM vs the oracle on the same system."""
    from oracle import timeint as O
    from paper_2501_19013_b200 import cdm_run, max_gen_eig
    from paper_2501_19013_b200.setup.configs import ricker
    from paper_2501_19013_b200.setup.geometry import BallVoids
    from paper_2501_19013_b200.setup.grid import Grid
    from paper_2501_19013_b200.setup.problem import ScmProblem
    geom = BallVoids(2, [[0.5, 0.5], [0.23, 0.71]], [0.26, 0.11])
    grid = Grid.build(geom, "lagrange", 3, 16)
    plain = ScmProblem.build(grid, 1e-8, 3)
    stab = ScmProblem.build(grid, 1e-8, 3, epsilon=0.01)
    lam_p = max_gen_eig(plain.device_operator(), plain.mass_matrix(), tol=1e-7)[0]
    lam_s = max_gen_eig(stab.device_operator(), stab.mass_matrix(), tol=1e-7)[0]
    assert lam_s < lam_p            # stabilised masses raise the critical step
    stab.set_point_source([0.1, 0.15])
    M, K = stab.mass_matrix(), stab.csr_stiffness()
    dt = 0.9 * 2.0 / np.sqrt(lam_s)
    f = lambda t: ricker(t, 10.0)  # noqa: E731
    psi, _, _ = O.cdm_run(M, K, stab.F_s, f, dt, 200)
    r = cdm_run(M, stab.device_operator(), stab.F_s, f, dt, 200)
    assert np.linalg.norm(r.psi - psi) <= 1e-10 * np.linalg.norm(psi)
