"""Plane-strain IMEX over x slabs emulated on one GPU:
slabs share one context, halos move by device copies after every step --
the same kernels and halo layout as the NCCL path.  Each slab factorises its
own S_cc / M_cc blocks, so the sharded field equals the single-GPU field to
rounding."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import imex_critical_time_step  # noqa: E402
from paper_2501_19013_b200.dist import group_imex_run, partition_imex  # noqa: E402
from paper_2501_19013_b200.imex import ImexPlan  # noqa: E402
from paper_2501_19013_b200.setup.configs import ricker  # noqa: E402
from paper_2501_19013_b200.setup.elastic import ElasticProblem, lame  # noqa: E402
from paper_2501_19013_b200.setup.geometry import BallVoids  # noqa: E402
from paper_2501_19013_b200.setup.grid import Grid  # noqa: E402

VOIDS = (([0.22, 0.5], 0.08), ([0.7, 0.3], 0.09), ([0.74, 0.8], 0.05))


def _problem(p, n_e):
    lam, mu = lame(1.0, 0.3)
    geom = BallVoids(2, [c for c, _ in VOIDS], [r for _, r in VOIDS])
    prob = ElasticProblem.build(Grid.build(geom, "lagrange", p, n_e), lam, mu, 1e-4, 3)
    prob.set_point_source([0.1, 0.9])
    prob.set_observers([[0.1, 0.9], [0.5, 0.5]])
    return prob


@pytest.mark.parametrize("p,n_e,world", [(3, 24, 2), (3, 24, 3), (5, 16, 2)])
def test_imex_slabs_match_single(p, n_e, world):
    prob = _problem(p, n_e)
    M = prob.mass_matrix()
    op = prob.device_operator()
    dt = 0.9 * imex_critical_time_step(op, M, prob.d_idx, tol=1e-7)
    f = lambda t: ricker(t, 10.0)  # noqa: E731
    ref = ImexPlan(M, op, prob.F_s, dt, prob.c_idx, prob.d_idx, obs_mat=prob.obs_mat).run(f, 120)
    got = group_imex_run(prob, f, dt, 120, world)
    scale = np.linalg.norm(ref.psi)
    assert scale > 0
    assert np.linalg.norm(got.psi - ref.psi) <= 1e-12 * scale
    assert np.abs(got.obs - ref.obs).max() <= 1e-12 * np.abs(ref.obs).max()
    # the cuts avoid cut cells: rows lo-2, lo-1, lo
    cut_rows = set((np.asarray(prob.grid.cut_lex) // n_e).tolist())
    for lo, _ in partition_imex(prob, world)[1:]:
        assert not {lo - 2, lo - 1, lo} & cut_rows
