"""Tiny runs of every device kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): the 2D TMA tile step (k_scm2d), the 3D
x-streaming step (k_scm3d + k_cut_pre), the plane-strain tile step (k_ela2d),
the SELL CSR step (k_sell), the power iteration, and the IMEX c chain
(k_trsv_comp).  Each case is checked against the CPU oracle so a sanitizer
run also shows the results stayed correct.

  compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""

import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle import cpu, timeint as O  # noqa: E402
from paper_2501_19013_b200 import cdm_run, imex_run, max_gen_eig  # noqa: E402
from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm, ricker  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f(t):
    return ricker(t, 10.0)


def scm2d():
    prob = build_scm(CONFIGS["config1"].scaled(12))
    K, M, op = prob.csr_stiffness(), prob.mass_matrix(), prob.device_operator()
    lam, _ = max_gen_eig(op, M, tol=1e-7)
    dt = 0.9 * 2 / np.sqrt(lam)
    psi, _, _ = O.cdm_run(M, K, prob.F_s, f, dt, 20)
    return rel(cdm_run(M, op, prob.F_s, f, dt, 20).psi, psi)


def scm3d():
    prob = build_scm(replace(CONFIGS["config5"], p=3, n_e=6, n_random=3,
                             r_range=(0.05, 0.1), name="san3d"))
    K, M, op = cpu.scm_csr(prob), prob.mass_matrix(), prob.device_operator()
    dt = 1e-3
    psi, _, _ = O.cdm_run(M, K, prob.F_s, f, dt, 10)
    return rel(cdm_run(M, op, prob.F_s, f, dt, 10).psi, psi)


def sell():
    from paper_2501_19013_b200.setup.iga import build_config3
    prob = build_config3(n_e=24)
    M, op = prob.mass_matrix(), prob.device_operator()
    dt = 1e-4
    psi, _, _ = O.cdm_run(M, prob.K, prob.F_s, f, dt, 10)
    return rel(cdm_run(M, op, prob.F_s, f, dt, 10).psi, psi)


def imex_scm():
    from paper_2501_19013_b200.setup.geometry import BallVoids
    from paper_2501_19013_b200.setup.grid import Grid
    from paper_2501_19013_b200.setup.problem import ScmProblem
    geom = BallVoids(2, [[0.5, 0.5], [0.2, 0.75]], [0.23, 0.09])
    prob = ScmProblem.build(Grid.build(geom, "lagrange", 4, 10), 1e-6, 3, lumping="none")
    prob.set_point_source([0.15, 0.2])
    M, K, op = prob.mass_matrix(), prob.csr_stiffness(), prob.device_operator()
    dm = prob.grid.dofmap
    dt = 1e-3
    psi, _, _ = O.imex_run(M, K, prob.F_s, f, dt, 10, dm.c_idx, dm.d_idx)
    return rel(imex_run(M, op, prob.F_s, f, dt, 10, dm.c_idx, dm.d_idx).psi, psi)


def elastic():
    from paper_2501_19013_b200.setup.configs import ElasticConfig, build_elastic
    cfg = replace(ElasticConfig().scaled(8), p=3, n_random=4, r_range=(0.05, 0.1))
    prob = build_elastic(cfg)
    K, M, op = prob.csr_stiffness(), prob.mass_matrix(), prob.device_operator()
    c, d = prob.c_idx, prob.d_idx
    dt = 1e-3
    psi, _, _ = O.imex_run(M, K, prob.F_s, f, dt, 10, c, d)
    return rel(imex_run(M, op, prob.F_s, f, dt, 10, c, d).psi, psi)


if __name__ == "__main__":
    cases = [scm2d, scm3d, sell, imex_scm, elastic]
    want = set(sys.argv[1:])
    worst = 0.0
    for case in cases:
        if want and case.__name__ not in want:
            continue
        e = case()
        worst = max(worst, e)
        print(f"{case.__name__}: rel L2 vs oracle {e:.2e}", flush=True)
    assert worst <= 1e-10, worst
    print("sanitize_probe OK")
