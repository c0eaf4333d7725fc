"""Config-4 (elastic IMEX) timing helper: set-up stages and the device loop
at a chosen resolution.  python tools/imex_bench.py [n_e] [n_t]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2501_19013_b200 import imex_critical_time_step
from paper_2501_19013_b200.imex import ImexPlan
from paper_2501_19013_b200.setup.configs import ElasticConfig, build_elastic, ricker

n_e = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = ElasticConfig().scaled(n_e, n_t)
T = {}
t0 = time.perf_counter()
prob = build_elastic(cfg)
T["build"] = time.perf_counter() - t0
t0 = time.perf_counter()
op = prob.device_operator()
M = prob.mass_matrix()
T["op+mass"] = time.perf_counter() - t0
c, d = prob.c_idx, prob.d_idx
t0 = time.perf_counter()
dtd = imex_critical_time_step(op, M, d, tol=1e-7)
T["dt_crit(d)"] = time.perf_counter() - t0
dt = cfg.safety * dtd
t0 = time.perf_counter()
plan = ImexPlan(M, op, prob.F_s, dt, c, d, obs_mat=prob.obs_mat, beta=cfg.beta)
T["plan(factor)"] = time.perf_counter() - t0
f = lambda t: ricker(t, cfg.f_e)
for rep in range(2):
    t0 = time.perf_counter()
    r = plan.run(f, n_t, gamma=cfg.gamma)
    T[f"run{rep}"] = time.perf_counter() - t0
    T[f"loop{rep}"] = r.timings.rhs
print(f"n_e={n_e} n_dof={prob.n_dof} n_c={c.shape[0]} n_cut={prob.grid.cut_lex.shape[0]} "
      f"fact_nnz={plan.fact_nnz} dt={dt:.4e} factor_s={plan.factorization:.2f}")
print({k: round(v, 3) for k, v in T.items()})
print(f"loop per step {1e6 * T['loop1'] / n_t:.1f} us; DOF-updates/s {prob.n_dof * n_t / T['loop1']:.3e}; "
      f"max|psi| {np.abs(r.psi).max():.3e}")
