"""Host-side breakdown of one public ``cdm_run`` call (tuning helper):
    python tools/e2e_profile.py [config] [n_t]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2501_19013_b200 import _lib
from paper_2501_19013_b200.linalg import diagonal_mass
from paper_2501_19013_b200.timeint import CdmPlan, force_table, _observer
from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm, ricker

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
prob = build_scm(CONFIGS[name])
op = prob.device_operator()
M = prob.mass_matrix()
F = prob.F_s
obs = prob.obs_mat
dt = 1e-7
f = lambda t: ricker(t, 10.0)
torch.cuda.synchronize()
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    T = {}
    t0 = time.perf_counter()
    m = diagonal_mass(M); T["diagonal_mass"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    o, keep = _observer(obs, op.n); T["observer"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    plan = CdmPlan(M, op, F, obs_mat=obs); T["plan_total"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    ft = force_table(f, dt, n_t); T["force_table"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    r = plan.run(f, dt, n_t); T["run_total"] = time.perf_counter() - t1
    T["run_loop(device)"] = r.timings.rhs
    t1 = time.perf_counter()
    plan.close(); T["close"] = time.perf_counter() - t1
    print(rep, {k: round(v * 1e3, 2) for k, v in T.items()}, flush=True)
