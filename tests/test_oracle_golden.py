"""Pin the CPU oracle (oracle/timeint.py) to the reference's own outputs.

The golden vectors come from running the reference package in this container
(tests/golden/make_golden.py).  Bitwise equality is expected: the oracle
restates the same arithmetic on the same SciPy kernels."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import csr_from, load_golden
from oracle import timeint as O


def test_bar_cdm_newmark_imex_bitwise():
    g = load_golden("bar")
    M, K, F = sp.csr_matrix(g["M"]), sp.csr_matrix(g["K"]), g["F"]
    obs = sp.identity(4, format="csr")
    f = lambda t: np.sin(6.0 * t)
    dt, n_t = float(g["dt"]), int(g["n_t"])
    psi, o, _ = O.cdm_run(M, K, F, f, dt, n_t, obs_mat=obs)
    assert np.array_equal(o, g["cdm_obs"]) and np.array_equal(psi, g["cdm_psi"])
    _, _, o = O.newmark_run(M, K, F, f, dt, n_t, obs_mat=obs)
    assert np.array_equal(o, g["nm_obs"])
    psi, _, o = O.imex_run(M, K, F, f, dt, n_t, [1, 2], [0, 3], obs_mat=obs)
    assert np.array_equal(o, g["imex_obs"]) and np.array_equal(psi, g["imex_psi"])
    psi, o, _ = O.cdm_run(M, K, F, np.cos, 1e-2, 100, obs_mat=obs, psi0=g["psi0"], v0=g["v0"])
    assert np.array_equal(o, g["init_obs"])
    _, vdot, o = O.imex_run(sp.csr_matrix(g["Mc"]), K, F, f, dt, n_t, np.arange(4),
                            np.array([], dtype=int), obs_mat=obs)
    assert np.array_equal(o, g["imexc_obs"]) and np.array_equal(vdot, g["imexc_vdot"])


def test_scalar_stability_dichotomy_matches_reference():
    g = load_golden("scalar")
    M = sp.csr_matrix(np.array([[1.0]]))
    psi, o, _ = O.cdm_run(M, M, np.zeros(1), lambda t: 0.0, 1.99, 10000,
                          obs_mat=sp.identity(1, format="csr"), psi0=[1.0])
    assert np.array_equal(o, g["stable_obs"])
    with pytest.raises(O.OracleDivergence) as e:
        O.cdm_run(M, M, np.zeros(1), lambda t: 0.0, 2.01, 10000, psi0=[1.0])
    assert e.value.step == int(g["div_step"])
    assert e.value.amplitude == float(g["div_amp"])


def test_rand10_power_iteration_and_cdm():
    g = load_golden("rand10")
    M = sp.diags(g["M"]).tocsr()
    K = sp.csr_matrix(g["K"])
    lam, it = O.max_gen_eig(K, M)
    assert lam == float(g["lam"]) and it == int(g["iters"])
    psi, o, _ = O.cdm_run(M, K, g["F"], lambda t: np.sin(3.0 * t), float(g["dt"]), 200,
                          obs_mat=sp.identity(10, format="csr"), psi0=g["psi0"])
    assert np.array_equal(o, g["obs"])


def test_cube_p2n4_oracle_reproduces_reference():
    g = load_golden("cube_p2n4")
    K = csr_from(g, "K")
    M = sp.diags(g["M"]).tocsr()
    lam, it = O.max_gen_eig(K, M, tol=1e-7, seed=0)
    assert lam == float(g["lam"]) and it == int(g["iters"])
    f = lambda t: O.ricker(t, 10.0)
    psi, o, _ = O.cdm_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]),
                          obs_mat=csr_from(g, "obs"))
    assert np.array_equal(psi, g["psi"])
    assert np.array_equal(o, g["obs"])


def test_cube_imex_oracle_reproduces_reference():
    g = load_golden("cube_imex_p2n4")
    M, K = csr_from(g, "M"), csr_from(g, "K")
    f = lambda t: O.ricker(t, 10.0)
    psi, _, o = O.imex_run(M, K, g["F"], f, float(g["dt"]), int(g["n_t"]), g["c_idx"],
                           g["d_idx"], obs_mat=csr_from(g, "obs"))
    assert np.array_equal(psi, g["psi"])
    assert np.array_equal(o, g["obs"])


# ---- the C/OpenMP port (oracle/wc_oracle.c): the bench's reference arm ----
# It must reproduce the reference bitwise too: same row-sum order as SciPy's
# csr_matvec, no FMA contraction (-ffp-contract=off), rhs / m division.

def _c_cdm(K, m, F, f, dt, n_t, psi0=None, threads=4):
    from oracle import cpu
    from paper_2501_19013_b200.timeint import force_table
    return cpu.cdm_run(K, m, F, force_table(f, dt, n_t), dt, n_t, psi0=psi0, threads=threads)


def test_c_port_cube_p2n4_bitwise():
    g = load_golden("cube_p2n4")
    psi, div = _c_cdm(csr_from(g, "K"), g["M"], g["F"], lambda t: O.ricker(t, 10.0),
                      float(g["dt"]), int(g["n_t"]))
    assert div == 0
    assert np.array_equal(psi, g["psi"])


def test_c_port_rand10_bitwise_any_thread_count():
    g = load_golden("rand10")
    for threads in (1, 3):
        psi, div = _c_cdm(sp.csr_matrix(g["K"]), g["M"], g["F"], lambda t: np.sin(3.0 * t),
                          float(g["dt"]), 200, psi0=g["psi0"], threads=threads)
        assert div == 0 and np.array_equal(psi, g["psi"])


def test_c_port_divergence_step_matches_reference():
    g = load_golden("scalar")
    one = sp.csr_matrix(np.array([[1.0]]))
    psi, div = _c_cdm(one, np.ones(1), np.zeros(1), lambda t: 0.0, 1.99, 10000, psi0=np.ones(1))
    assert div == 0 and np.array_equal(psi, g["stable_psi"])
    _, div = _c_cdm(one, np.ones(1), np.zeros(1), lambda t: 0.0, 2.01, 10000, psi0=np.ones(1))
    assert div == int(g["div_step"])


def test_c_port_observers_bitwise():
    g = load_golden("cube_p2n4")
    from oracle import cpu
    from paper_2501_19013_b200.timeint import force_table
    f = lambda t: O.ricker(t, 10.0)  # noqa: E731
    dt, n_t = float(g["dt"]), int(g["n_t"])
    psi, obs, div = cpu.cdm_run(csr_from(g, "K"), g["M"], g["F"], force_table(f, dt, n_t), dt, n_t,
                                threads=2, obs_mat=csr_from(g, "obs"))
    assert div == 0 and np.array_equal(psi, g["psi"]) and np.array_equal(obs, g["obs"])
