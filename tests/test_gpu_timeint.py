"""Device integrators against the reference's own timeint tests
(tests/test_timeint.py of the reference, re-run through the drop-in) and the
golden vectors of the reference (tests/golden/*.npz).

Tolerances: fields are fp64; the device sums K psi in a different order than
SciPy's CSR matvec, so agreement is to rounding (rel. L2 <= 1e-10 is the
north-star bar; the small systems here agree to ~1e-14)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import csr_from, load_golden
from oracle import timeint as O

pytestmark = pytest.mark.gpu

wc = pytest.importorskip("paper_2501_19013_b200")
from paper_2501_19013_b200 import (DIVERGENCE_LIMIT, DivergenceError, cdm_run,  # noqa: E402
                                   dt_crit, max_gen_eig, select_dt)
from paper_2501_19013_b200.operators import CsrOperator  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def scalar_system(omega):
    M = sp.csr_matrix(np.array([[1.0]]))
    K = sp.csr_matrix(np.array([[omega * omega]]))
    return M, K, np.zeros(1), sp.identity(1, format="csr")


def bar_system():
    g = load_golden("bar")
    return sp.csr_matrix(g["M"]), sp.csr_matrix(g["K"])


def zero_f(t):
    return 0.0


def test_cdm_conserves_zero():
    M, K = bar_system()
    r = cdm_run(M, K, np.zeros(4), zero_f, 1e-2, 50, obs_mat=sp.identity(4, format="csr"))
    assert np.all(r.psi == 0.0) and np.all(r.obs == 0.0)
    assert r.t.shape == (51,) and r.t[-1] == pytest.approx(0.5)


def test_cdm_stability_dichotomy():
    M, K, F, obs = scalar_system(1.0)
    r = cdm_run(M, K, F, zero_f, 1.99, 10000, obs_mat=obs, psi0=[1.0])
    assert np.abs(r.obs).max() <= 50.0
    g = load_golden("scalar")
    assert np.abs(r.obs - g["stable_obs"]).max() <= 1e-12
    with pytest.raises(DivergenceError) as exc:
        cdm_run(M, K, F, zero_f, 2.01, 10000, obs_mat=obs, psi0=[1.0])
    assert exc.value.step == int(g["div_step"])
    assert exc.value.amplitude > DIVERGENCE_LIMIT


def test_second_order_convergence_scalar():
    omega, T = 5.0, 2.0
    M, K, F, obs = scalar_system(omega)
    errs = []
    for n_t in (100, 200):
        r = cdm_run(M, K, F, zero_f, T / n_t, n_t, obs_mat=obs, psi0=[1.0])
        stride = n_t // 100
        errs.append(np.linalg.norm(r.obs[0, ::stride] - np.cos(omega * r.t[::stride])))
    assert 3.6 <= errs[0] / errs[1] <= 4.4


def test_bar_cdm_matches_reference_golden():
    g = load_golden("bar")
    M, K = sp.csr_matrix(g["M"]), sp.csr_matrix(g["K"])
    r = cdm_run(M, K, g["F"], lambda t: np.sin(6.0 * t), float(g["dt"]), int(g["n_t"]),
                obs_mat=sp.identity(4, format="csr"))
    assert np.abs(r.obs - g["cdm_obs"]).max() <= 1e-13 * np.abs(g["cdm_obs"]).max()
    r = cdm_run(M, K, g["F"], np.cos, 1e-2, 100, obs_mat=sp.identity(4, format="csr"),
                psi0=g["psi0"], v0=g["v0"])
    assert np.abs(r.obs - g["init_obs"]).max() <= 1e-13 * np.abs(g["init_obs"]).max()


def test_linearity_of_runs():
    M, K = bar_system()
    F = np.array([0.2, -0.4, 1.0, 0.3])
    obs = sp.identity(4, format="csr")
    f = lambda t: np.cos(2.0 * t)
    psi0 = np.array([0.1, 0.0, -0.2, 0.05])
    v0 = np.array([0.0, 0.3, 0.1, -0.1])
    r_f = cdm_run(M, K, F, f, 1e-2, 100, obs_mat=obs)
    r_h = cdm_run(M, K, np.zeros(4), zero_f, 1e-2, 100, obs_mat=obs, psi0=psi0, v0=v0)
    r_b = cdm_run(M, K, F, f, 1e-2, 100, obs_mat=obs, psi0=psi0, v0=v0)
    assert np.abs(r_f.obs + r_h.obs - r_b.obs).max() <= 1e-12 * np.abs(r_b.obs).max()


def test_timings_and_fact_dims_reported():
    M, K = bar_system()
    r = cdm_run(M, K, np.array([0.0, 1.0, 0.5, 0.2]), lambda t: np.sin(6.0 * t), 1e-3, 50)
    assert r.fact_dim == 0 and r.timings.factorization == 0.0 and r.timings.rhs > 0.0
    assert r.obs is None and r.psi_dot is None


def test_rand10_power_iteration_and_cdm_golden():
    g = load_golden("rand10")
    M = sp.diags(g["M"]).tocsr()
    K = sp.csr_matrix(g["K"])
    lam, it = max_gen_eig(K, M)
    assert abs(lam - float(g["lam"])) <= 1e-13 * float(g["lam"])
    assert it == int(g["iters"])   # same stopping iteration as the reference
    assert dt_crit(K, M) == pytest.approx(2.0 / np.sqrt(float(g["lam"])), rel=1e-12)
    r = cdm_run(M, K, g["F"], lambda t: np.sin(3.0 * t), float(g["dt"]), 200,
                obs_mat=sp.identity(10, format="csr"), psi0=g["psi0"])
    assert rel(r.obs, g["obs"]) <= 1e-13


def test_max_gen_eig_closed_forms():
    K = sp.diags([1.0, 2.0, 3.0]).tocsr()
    lam, n_iter = max_gen_eig(K, sp.identity(3, format="csr"), tol=1e-12)
    assert lam == pytest.approx(3.0, rel=1e-10) and n_iter >= 1
    h, c = 0.2, 2.0
    K = sp.csr_matrix(c * c / h * np.array([[1.0, -1.0], [-1.0, 1.0]]))
    Ml = sp.diags([h / 2.0, h / 2.0]).tocsr()
    assert max_gen_eig(K, Ml, tol=1e-12)[0] == pytest.approx(4.0 * c * c / h**2, rel=1e-9)
    assert dt_crit(K, Ml, tol=1e-12) == pytest.approx(h / c, rel=1e-9)
    assert max_gen_eig(sp.csr_matrix((2, 2)), sp.identity(2, format="csr"))[0] == 0.0


def test_cube_p2n4_csr_matches_reference():
    """Immersed rotated cube (reference assemble, HRZ): device CSR loop vs the
    reference's field after 300 steps and its critical step."""
    g = load_golden("cube_p2n4")
    K = csr_from(g, "K")
    M = sp.diags(g["M"]).tocsr()
    lam, it = max_gen_eig(K, M, tol=1e-7, seed=0)
    assert abs(lam - float(g["lam"])) <= 1e-12 * float(g["lam"])
    assert it == int(g["iters"])   # same stopping iteration as the reference
    f = lambda t: O.ricker(t, 10.0)
    r = cdm_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]), obs_mat=csr_from(g, "obs"))
    assert rel(r.psi, g["psi"]) <= 1e-10
    assert rel(r.obs, g["obs"]) <= 1e-10
    # bit-identical repetitions (src/harness.py:462-485 contract)
    r2 = cdm_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]), obs_mat=csr_from(g, "obs"))
    assert np.array_equal(r.psi, r2.psi) and np.array_equal(r.obs, r2.obs)


def test_operator_matmul_and_reuse():
    g = load_golden("cube_p2n4")
    K = csr_from(g, "K")
    op = CsrOperator(K)
    x = np.random.default_rng(0).standard_normal(K.shape[0])
    assert rel(op @ x, K @ x) <= 1e-14
    M = sp.diags(g["M"]).tocsr()
    f = lambda t: O.ricker(t, 10.0)
    r1 = cdm_run(M, op, g["F"], f, float(g["dt"]), 50)
    r2 = cdm_run(M, K, g["F"], f, float(g["dt"]), 50)
    assert np.array_equal(r1.psi, r2.psi)


def test_rejects_indefinite_and_nondiagonal_mass():
    M, K = bar_system()
    from paper_2501_19013_b200 import IndefiniteMatrixError
    with pytest.raises(IndefiniteMatrixError):
        cdm_run(sp.diags([1.0, -1.0, 1.0, 1.0]).tocsr(), K, np.zeros(4), zero_f, 1e-3, 3)
    # a consistent (non-diagonal) mass runs through the device M solves
    Mc = sp.csr_matrix(M.toarray() + 0.05)
    F = np.array([0.0, 1.0, 0.5, 0.2])
    f = lambda t: np.sin(6.0 * t)  # noqa: E731
    r = cdm_run(Mc, K, F, f, 5e-3, 200)
    psi_ref, _, _ = O.cdm_run(Mc, K, F, f, 5e-3, 200)
    assert rel(r.psi, psi_ref) <= 1e-12 and r.fact_dim == 4
    with pytest.raises(IndefiniteMatrixError):
        cdm_run(sp.csr_matrix(M.toarray() - 0.5), K, np.zeros(4), zero_f, 1e-3, 3)


def test_select_dt_rules():
    assert select_dt(4.17564e-3, 6.8966e-3) == pytest.approx(3.758076e-3, rel=1e-9)
    assert select_dt(1.0) == pytest.approx(0.9)
    assert select_dt(1.0, 0.5) == 0.5
