"""Host<->device copy throughput of the public API (tuning helper): a diagonal
CSR K of n DOFs, CdmPlan (H2D of M) and a one-step run (D2H of psi).
    python tools/copy_probe.py [n_millions] [reps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import scipy.sparse as sp
from paper_2501_19013_b200.timeint import CdmPlan

n = int(float(sys.argv[1] if len(sys.argv) > 1 else 64) * 1e6)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K = sp.identity(n, format="csr")
M = sp.diags(np.full(n, 2.0)).tocsr()
F = np.zeros(n); F[n // 2] = 1.0
for r in range(reps):
    t0 = time.perf_counter()
    plan = CdmPlan(M, K, F)
    t1 = time.perf_counter()
    res = plan.run(lambda t: 0.0, 1e-3, 1)
    t2 = time.perf_counter()
    plan.close()
    gb = n * 8 / 1e9
    print(f"n={n} plan {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms (loop {1e3*res.timings.rhs:.1f})  "
          f"D2H-ish {gb/(t2-t1-res.timings.rhs):.1f} GB/s", flush=True)
