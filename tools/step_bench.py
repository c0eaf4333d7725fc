"""Kernel tuning helper: time the fused step loop of a config at a fixed dt
(no power iteration).  python tools/step_bench.py [config] [n_t] [reps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2501_19013_b200 import _lib
from paper_2501_19013_b200.timeint import CdmPlan, force_table
from paper_2501_19013_b200.setup.configs import CONFIGS, build_scm, ricker

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 500
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
base, _, scale = name.partition("@")
cfg = CONFIGS[base] if not scale else CONFIGS[base].scaled(int(scale))
prob = build_scm(cfg)
op = prob.device_operator()
plan = CdmPlan(prob.mass_matrix(), op, prob.F_s)
dt = 1e-7
ft = torch.from_numpy(force_table(lambda t: ricker(t, 10.0), dt, n_t)).cuda()
out = torch.empty(prob.n_dof, dtype=torch.float64, device="cuda")
lib = _lib.load()
best = 1e9
for r in range(reps + 1):
    div, tm = _lib.Divergence(), _lib.Timings()
    _lib.check(lib.wcb_cdm_plan_run_device(plan.handle, ft.data_ptr(), dt, n_t, None, None,
                                           out.data_ptr(), None, _lib.C.byref(div), _lib.C.byref(tm)))
    if r:
        best = min(best, tm.rhs / n_t)
print(f"{name}: {best * 1e6:.2f} us/step  {prob.n_dof * 32 / best / 1e9:.0f} GB/s (32 B/DOF)")
