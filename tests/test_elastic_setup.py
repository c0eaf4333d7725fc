"""Plane-strain elastic set-up (config 4) invariants on the host.

The reference has no vector-valued operator, so the operator
is pinned by its defining properties: symmetry, exactly three zero-energy
modes (two translations and the infinitesimal rotation, sampled at the GLL
nodes), positive semi-definiteness, the alpha-weighted mass total, and the
restricted c-c block equal to the slice of the global CSR."""

import numpy as np

from paper_2501_19013_b200.setup.basis import gll_rule
from paper_2501_19013_b200.setup.elastic import ElasticProblem, lame
from paper_2501_19013_b200.setup.geometry import BallVoids
from paper_2501_19013_b200.setup.grid import Grid


def _problem(p=3, n_e=12, alpha=1e-3):
    lam, mu = lame(1.0, 0.3)
    geom = BallVoids(2, np.array([[0.5, 0.5], [0.23, 0.31]]), np.array([0.2, 0.07]))
    return ElasticProblem.build(Grid.build(geom, "lagrange", p, n_e), lam, mu, alpha, 3)


def _coords(grid):
    n1 = grid.basis.n_funcs
    I, J = np.divmod(grid.dofmap.lex_of_compact, n1)
    xi = gll_rule(grid.p)[0]

    def c(k):
        e = np.minimum(k // grid.p, grid.n_e - 1)
        return e * grid.h + (xi[k - e * grid.p] + 1.0) / 2.0 * grid.h
    return grid.origin[0] + c(I), grid.origin[1] + c(J)


def test_lame_plane_strain():
    lam, mu = lame(1.0, 0.3)
    assert abs(lam - 0.3 / (1.3 * 0.4)) < 1e-15 and abs(mu - 1.0 / 2.6) < 1e-15


def test_elastic_operator_invariants():
    prob = _problem()
    K = prob.csr_stiffness()
    assert abs(K - K.T).max() <= 1e-14 * abs(K).max()
    x, y = _coords(prob.grid)
    nn = prob.n_node
    for u, v in ((np.ones(nn), np.zeros(nn)), (np.zeros(nn), np.ones(nn)), (-y, x)):
        r = np.concatenate([u, v])
        assert np.abs(K @ r).max() <= 1e-13 * np.abs(K).max()
    ev = np.linalg.eigvalsh(K.toarray())
    assert ev[0] > -1e-12 * ev[-1]
    assert np.sum(np.abs(ev) <= 1e-12 * ev[-1]) == 3
    # linear displacement u = x: uniform strain e_xx = 1, energy (l+2m)/2 * area
    r = np.concatenate([x, np.zeros(nn)])
    area = 1.0 - np.pi * (0.2 ** 2 + 0.07 ** 2)
    energy = 0.5 * r @ (K @ r)
    assert abs(energy - 0.5 * (prob.lam + 2 * prob.mu) * area) <= 5e-3 * energy


def test_elastic_mass_and_blocks():
    prob = _problem(alpha=1e-4)
    M = prob.mass_matrix()
    nn = prob.n_node
    assert abs(M - M.T).max() <= 1e-15 * abs(M).max()
    area = 1.0 - np.pi * (0.2 ** 2 + 0.07 ** 2)
    assert abs(M[:nn][:, :nn].sum() - area) <= 2e-3
    assert abs(M[nn:][:, nn:].sum() - M[:nn][:, :nn].sum()) <= 1e-14
    d = prob.d_idx
    Mdd = M[d][:, d]
    assert Mdd.nnz == d.shape[0] and M[d][:, prob.c_idx].nnz == 0
    K = prob.csr_stiffness()
    c = prob.c_idx
    assert abs(prob.stiffness_block(c) - K[c][:, c]).max() <= 1e-15 * abs(K).max()


def test_elastic_point_source_and_observers():
    prob = _problem()
    F = prob.set_point_source([0.1, 0.9], direction=(0.6, 0.8))
    nn = prob.n_node
    assert abs(F[:nn].sum() - 0.6) <= 1e-12 and abs(F[nn:].sum() - 0.8) <= 1e-12
    O = prob.set_observers([[0.1, 0.9], [0.8, 0.2]])
    assert O.shape == (4, prob.n_dof)
    assert np.allclose(np.asarray(O.sum(axis=1)).ravel(), 1.0)
