"""Host<->device copies of the public API: large pageable arrays go through
the pinned staging ring (csrc/wcb_core.cu copy_h2d / copy_d2h) and CDM outputs
are pre-faulted during the device loop.  Exact round trips at sizes that are
not multiples of the ring chunk, with the ring wrapping (1 MiB chunks, three
buffers), and the same values as the driver's pageable path."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

PROBE = r"""
import sys
import numpy as np
import scipy.sparse as sp
sys.path.insert(0, sys.argv[1])
from paper_2501_19013_b200.operators import CsrOperator
from paper_2501_19013_b200 import cdm_run
n = int(sys.argv[2])
rng = np.random.default_rng(7)
d = rng.uniform(0.5, 2.0, n)
x = rng.standard_normal(n)
K = sp.diags(d).tocsr()
y = CsrOperator(K) @ x
assert np.array_equal(y, d * x), "K @ x through the staged copies"
# CDM with K = diag(d), M = I and no force: psi_1 = psi_0 + dt v_0 - dt^2/2 d psi_0 ...
M = sp.identity(n, format="csr")
psi0 = rng.standard_normal(n)
r = cdm_run(M, K, np.zeros(n), lambda t: 0.0, 1e-3, 2, psi0=psi0, v0=np.zeros(n))
dt = 1e-3
prev = psi0 - dt * 0.0 + (0.5 * dt * dt) * ((0.0 - d * psi0) / 1.0)
cur = psi0
for _ in range(2):
    nxt = (2.0 * cur - prev) + (dt * dt) * ((0.0 - d * cur) * 1.0)
    prev, cur = cur, nxt
rel = np.linalg.norm(r.psi - cur) / np.linalg.norm(cur)
assert rel < 1e-14, rel
print("OK", n)
"""


def _run(n, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", PROBE, str(ROOT), str(n)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout


@pytest.mark.parametrize("n", [262_144 + 3, 5_000_011])
@pytest.mark.parametrize("env", [{}, {"WAVECELL_B200_STAGE_MB": "1", "WAVECELL_B200_STAGE_THREADS": "3"},
                                 {"WAVECELL_B200_NO_STAGE": "1"}],
                         ids=["default", "1MiB-ring", "pageable"])
def test_staged_round_trip(n, env):
    _run(n, env)
