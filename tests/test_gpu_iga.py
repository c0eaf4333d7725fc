"""IGA-FCM (B-spline) CSR path: the reference's own B-spline system on the
rotated cube (golden) and BASELINE config 3's geometry at reduced size."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import csr_from, load_golden
from oracle import timeint as O

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import cdm_run, max_gen_eig  # noqa: E402
from paper_2501_19013_b200.setup.configs import ricker  # noqa: E402
from paper_2501_19013_b200.setup.iga import build_config3  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_bspline_cube_matches_reference():
    g = load_golden("bspline_cube_p2n5")
    K = csr_from(g, "K")
    M = sp.diags(g["M"]).tocsr()
    lam, it = max_gen_eig(K, M, tol=1e-7, seed=0)
    assert abs(lam - float(g["lam"])) <= 1e-12 * float(g["lam"])
    r = cdm_run(M, K, g["F"], lambda t: ricker(t, 10.0), float(g["dt"]), 200)
    assert rel(r.psi, g["psi"]) <= 1e-10


def test_config3_reduced_cdm_parity():
    prob = build_config3(n_e=96)
    M = prob.mass_matrix()
    op = prob.device_operator()
    x = np.random.default_rng(0).standard_normal(prob.n_dof)
    assert rel(op @ x, prob.K @ x) <= 1e-14
    lam, _ = max_gen_eig(op, M, tol=1e-7, seed=0)
    lam_ref, _ = O.max_gen_eig(prob.K, M, tol=1e-7, seed=0)
    assert abs(lam - lam_ref) <= 1e-10 * lam_ref
    dt = 0.9 * 2.0 / np.sqrt(lam_ref)
    f = lambda t: ricker(t, 10.0)
    psi_ref, obs_ref, _ = O.cdm_run(M, prob.K, prob.F_s, f, dt, 400, obs_mat=prob.obs_mat)
    r = cdm_run(M, op, prob.F_s, f, dt, 400, obs_mat=prob.obs_mat)
    assert rel(r.psi, psi_ref) <= 1e-10
    assert rel(r.obs, obs_ref) <= 1e-10


def test_shared_stencil_slices_bitwise(monkeypatch):
    """SELL slices with translation-invariant rows keep one offset/value
    vector; the field equals the plain SELL layout's bitwise (same stored
    order of every row sum)."""
    from paper_2501_19013_b200.operators import CsrOperator
    prob = build_config3(n_e=96)
    M = prob.mass_matrix()
    f = lambda t: ricker(t, 10.0)  # noqa: E731
    x = np.random.default_rng(3).standard_normal(prob.n_dof)
    outs = []
    # plain SELL; shared-stencil slices without and with the kernel-parameter
    # stencil (slice types 3 / 4)
    for flags in ({"WAVECELL_B200_NO_SHARED_STENCIL": "1"}, {"WAVECELL_B200_NO_SELL_GP": "1"}, {}):
        for k in ("WAVECELL_B200_NO_SHARED_STENCIL", "WAVECELL_B200_NO_SELL_GP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in flags.items():
            monkeypatch.setenv(k, v)
        op = CsrOperator(prob.K)
        outs.append((op @ x, cdm_run(M, op, prob.F_s, f, 1e-4, 200).psi))
    for y, psi in outs[1:]:
        assert np.array_equal(outs[0][0], y)
        assert np.array_equal(outs[0][1], psi)
