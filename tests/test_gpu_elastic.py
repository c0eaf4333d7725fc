"""Plane-strain elastic operator (config 4) on the device: matrix-free
apply vs the CSR assembly of the same system, the fused CDM step and the
IMEX split vs the CPU oracle (reference integrator arithmetic) on that CSR.
Bar: rel L2 <= 1e-10 of the fp64 field; applies agree to rounding."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import timeint as O

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import cdm_run, imex_run, imex_critical_time_step  # noqa: E402
from paper_2501_19013_b200.setup.configs import ricker  # noqa: E402
from paper_2501_19013_b200.setup.elastic import ElasticProblem, lame  # noqa: E402
from paper_2501_19013_b200.setup.geometry import BallVoids  # noqa: E402
from paper_2501_19013_b200.setup.grid import Grid  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _problem(p, n_e, alpha=1e-3, voids=(([0.5, 0.5], 0.27), ([0.15, 0.8], 0.1))):
    lam, mu = lame(1.0, 0.3)
    geom = BallVoids(2, [c for c, _ in voids], [r for _, r in voids])
    return ElasticProblem.build(Grid.build(geom, "lagrange", p, n_e), lam, mu, alpha, 3)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_elastic_apply_matches_csr(p):
    for n_e in (5, 23):
        prob = _problem(p, n_e)
        K = prob.csr_stiffness()
        op = prob.device_operator()
        rng = np.random.default_rng(p)
        for _ in range(2):
            x = rng.standard_normal(prob.n_dof)
            assert rel(op @ x, K @ x) <= 1e-13, (p, n_e)


def test_elastic_cdm_step_parity():
    """Fused step kernel with a diagonal mass (the consistent cut blocks'
    diagonal) vs the oracle's CDM loop on the CSR."""
    prob = _problem(5, 12)
    prob.set_point_source([0.12, 0.15], direction=(0.6, 0.8))
    prob.set_observers([[0.12, 0.15], [0.85, 0.2]])
    K = prob.csr_stiffness()
    M = sp.diags(prob.mass_matrix().diagonal()).tocsr()
    op = prob.device_operator()
    lam, _ = O.max_gen_eig(K, M, tol=1e-7, seed=0)
    dt = 0.9 * 2.0 / np.sqrt(lam)
    f = lambda t: ricker(t, 10.0)
    psi_ref, obs_ref, _ = O.cdm_run(M, K, prob.F_s, f, dt, 300, obs_mat=prob.obs_mat)
    r = cdm_run(M, op, prob.F_s, f, dt, 300, obs_mat=prob.obs_mat)
    assert rel(r.psi, psi_ref) <= 1e-10
    assert rel(r.obs, obs_ref) <= 1e-10
    r2 = cdm_run(M, op, prob.F_s, f, dt, 300, obs_mat=prob.obs_mat)
    assert np.array_equal(r.psi, r2.psi)


def test_elastic_imex_parity():
    """Config-4 scheme at reduced scale: explicit CDM on d, Newmark on c with
    the consistent cut mass; dt from the d subsystem."""
    prob = _problem(5, 16, alpha=1e-4,
                    voids=(([0.5, 0.5], 0.13), ([0.2, 0.3], 0.05), ([0.77, 0.71], 0.08)))
    prob.set_point_source([0.1, 0.9])
    M = prob.mass_matrix()
    K = prob.csr_stiffness()
    op = prob.device_operator()
    c, d = prob.c_idx, prob.d_idx
    dtd = imex_critical_time_step(op, M, d, tol=1e-7)
    dtd_ref = 2.0 / np.sqrt(O.max_gen_eig(K[d][:, d], M[d][:, d], tol=1e-7)[0])
    assert abs(dtd - dtd_ref) <= 1e-9 * dtd_ref
    dt = 0.9 * dtd_ref
    f = lambda t: ricker(t, 10.0)
    psi_ref, _, _ = O.imex_run(M, K, prob.F_s, f, dt, 150, c, d)
    r = imex_run(M, op, prob.F_s, f, dt, 150, c, d)
    assert rel(r.psi, psi_ref) <= 1e-10
    assert r.fact_dim == c.shape[0]


def test_imex_grouped_solves_match_level_solves(monkeypatch):
    """k_trsv_ring solves runs of narrow levels as groups (outside entries at
    once, then the host-inverted triangular block).  Same linear solve, other
    rounding: the IMEX field agrees with the one-piece-per-level solve far
    inside the 1e-10 parity bar, and with the oracle at the bar."""
    prob = _problem(5, 24, alpha=1e-4,
                    voids=(([0.5, 0.5], 0.2), ([0.2, 0.3], 0.07), ([0.77, 0.71], 0.1)))
    prob.set_point_source([0.1, 0.9])
    M = prob.mass_matrix()
    op = prob.device_operator()
    c, d = prob.c_idx, prob.d_idx
    dt = 0.9 * imex_critical_time_step(op, M, d, tol=1e-7)
    f = lambda t: ricker(t, 10.0)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("WAVECELL_B200_TRSV_GROUPS", flag)
        out[flag] = imex_run(M, op, prob.F_s, f, dt, 200, c, d).psi
    assert np.isfinite(out["1"]).all()
    assert rel(out["1"], out["0"]) <= 1e-12
    K = prob.csr_stiffness()
    psi_ref, _, _ = O.imex_run(M, K, prob.F_s, f, dt, 200, c, d)
    assert rel(out["1"], psi_ref) <= 1e-10
