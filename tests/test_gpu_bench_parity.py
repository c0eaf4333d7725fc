"""Parity at the benchmarked sizes: the fields bench.py times, checked
against the reference arithmetic on the same inputs.

* config 2 (512^2 cells, p = 4, 4.0M DOFs, 2000 CDM steps) and config 3
  (1024^2 B-spline spans, 1.0M DOFs, 1000 steps): the device loop vs the C
  port of src/timeint.py:159-193 (pinned bitwise to the reference goldens in
  tests/test_oracle_golden.py) on the CSR of the same system, same dt, at
  relative L2 <= 1e-10 for psi and the observers;
* the critical step of both: the device power iteration stops at the
  reference-arithmetic iteration (oracle/timeint.py max_gen_eig) with
  |d lambda| / lambda <= 1e-13 (bitwise equality would need SciPy/OpenBLAS's
  CPU-specific reduction order);
* configs 4 and 5 at the largest reduced grids whose CSR fits host RAM
  comfortably (config 5: 48^3 cells, 3.0M DOFs; config 4: 128^2 cells).
"""

from dataclasses import replace

import numpy as np
import pytest

from oracle import cpu
from oracle import timeint as O

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import cdm_run, imex_critical_time_step, imex_run, max_gen_eig  # noqa: E402
from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm, ricker  # noqa: E402
from paper_2501_19013_b200.timeint import force_table  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def f(t):
    return ricker(t, 10.0)


def _check_cdm(prob, K, op, n_t):
    M = prob.mass_matrix()
    lam, it = max_gen_eig(op, M, tol=1e-7, seed=0)
    lam_ref, it_ref = O.max_gen_eig(K, M, tol=1e-7, seed=0)
    assert it == it_ref
    assert abs(lam - lam_ref) <= 1e-13 * lam_ref, abs(lam - lam_ref) / lam_ref
    dt = 0.9 * 2.0 / np.sqrt(lam_ref)
    psi_ref, obs_ref, div = cpu.cdm_run(K, prob.m_diag, prob.F_s, force_table(f, dt, n_t), dt, n_t,
                                        obs_mat=prob.obs_mat)
    assert div == 0
    r = cdm_run(M, op, prob.F_s, f, dt, n_t, obs_mat=prob.obs_mat)
    assert rel(r.psi, psi_ref) <= 1e-10
    assert rel(r.obs, obs_ref) <= 1e-10
    return rel(r.psi, psi_ref)


@pytest.mark.timeout(1800)
def test_config2_full_size_parity():
    prob = build_scm(CONFIGS["config2"])
    assert prob.n_dof == 4013112
    _check_cdm(prob, cpu.scm_csr(prob), prob.device_operator(), CONFIGS["config2"].n_t)


@pytest.mark.timeout(1800)
def test_config3_full_size_parity():
    from paper_2501_19013_b200.setup.iga import build_config3
    prob = build_config3(seed=0)
    assert prob.grid.n_e == 1024
    _check_cdm(prob, prob.K, prob.device_operator(), 1000)


@pytest.mark.timeout(1800)
def test_config5_reduced_parity():
    prob = build_scm(replace(CONFIGS["config5"], n_e=48, name="config5@48"))
    _check_cdm(prob, cpu.scm_csr(prob), prob.device_operator(), 200)


@pytest.mark.timeout(1800)
def test_config4_reduced_imex_parity():
    from paper_2501_19013_b200.setup.configs import ElasticConfig, build_elastic
    cfg = ElasticConfig().scaled(128)
    prob = build_elastic(cfg)
    K, M = prob.csr_stiffness(), prob.mass_matrix()
    c, d = prob.c_idx, prob.d_idx
    op = prob.device_operator()
    dtd = imex_critical_time_step(op, M, d, tol=1e-7, seed=cfg.seed)
    lam_ref, _ = O.max_gen_eig(K[d][:, d], M[d][:, d], tol=1e-7, seed=cfg.seed)
    assert abs(dtd - 2.0 / np.sqrt(lam_ref)) <= 1e-12 * dtd
    dt = cfg.safety * 2.0 / np.sqrt(lam_ref)
    psi_ref, _, obs_ref = O.imex_run(M, K, prob.F_s, f, dt, 200, c, d, obs_mat=prob.obs_mat)
    r = imex_run(M, op, prob.F_s, f, dt, 200, c, d, obs_mat=prob.obs_mat)
    assert rel(r.psi, psi_ref) <= 1e-10
    assert rel(r.obs, obs_ref) <= 1e-10
