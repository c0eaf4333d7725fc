"""Slab decomposition on one GPU (emulated ranks sharing a context; halos by
device copies): the same kernels and halo layout as the NCCL path, which must
give a field bitwise identical to the single-slab run."""

import numpy as np
import pytest
from dataclasses import replace

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import cdm_run, max_gen_eig  # noqa: E402
from paper_2501_19013_b200.dist import SlabScm, group_cdm_run, partition  # noqa: E402
from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm, ricker  # noqa: E402


@pytest.mark.parametrize("cfg", [
    replace(CONFIGS["config2"], n_e=48, name="c2s"),
    replace(CONFIGS["config5"], p=3, n_e=14, n_random=5, r_range=(0.03, 0.08), name="c5s"),
    replace(CONFIGS["config5"], p=2, n_e=11, n_random=4, r_range=(0.04, 0.09), name="c5s2"),
])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_group_slabs_bitwise_equal_single(cfg, world):
    prob = build_scm(cfg)
    op = prob.device_operator()
    M = prob.mass_matrix()
    lam, _ = max_gen_eig(op, M, tol=1e-7, seed=0)
    dt = 0.9 * 2.0 / np.sqrt(lam)
    f = lambda t: ricker(t, 10.0)
    ref = cdm_run(M, op, prob.F_s, f, dt, 120, obs_mat=prob.obs_mat)
    got = group_cdm_run(prob, f, dt, 120, world)
    assert np.array_equal(got.psi, ref.psi)
    # observers are summed from per-slab partials: equal to rounding
    assert np.abs(got.obs - ref.obs).max() <= 1e-13 * np.abs(ref.obs).max()


@pytest.mark.parametrize("cfg", [
    replace(CONFIGS["config2"], n_e=64, name="c2o"),
    replace(CONFIGS["config5"], p=3, n_e=24, n_random=5, r_range=(0.03, 0.08), name="c5o"),
])
@pytest.mark.parametrize("world", [2, 3])
def test_group_slabs_halo_overlap_bitwise(cfg, world, monkeypatch):
    """Slab steps split around the halo exchange (rows the neighbours need
    first, exchange on a second stream, interior rows meanwhile): bitwise the
    field of the unsplit group run and of the single-slab run."""
    monkeypatch.setenv("WAVECELL_B200_XCHUNKS", "3")   # 3D: first / interior / last x chunk
    prob = build_scm(cfg)
    op = prob.device_operator()
    M = prob.mass_matrix()
    lam, _ = max_gen_eig(op, M, tol=1e-7, seed=0)
    dt = 0.9 * 2.0 / np.sqrt(lam)
    f = lambda t: ricker(t, 10.0)
    ref = cdm_run(M, op, prob.F_s, f, dt, 80, obs_mat=prob.obs_mat)
    outs = []
    for ov in ("1", "0"):
        monkeypatch.setenv("WAVECELL_B200_HALO_OVERLAP", ov)
        outs.append(group_cdm_run(prob, f, dt, 80, world))
    for got in outs:
        assert np.array_equal(got.psi, ref.psi)
        assert np.abs(got.obs - ref.obs).max() <= 1e-13 * np.abs(ref.obs).max()
