"""Shared fixtures.  Tests that need a B200 are marked ``@pytest.mark.gpu``;
everything else runs on the CPU box (``pytest -m "not gpu"``)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libwavecell_b200.so)")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def csr_from(g, prefix):
    import scipy.sparse as sp
    return sp.csr_matrix((g[f"{prefix}_data"], g[f"{prefix}_indices"], g[f"{prefix}_indptr"]),
                         shape=tuple(g[f"{prefix}_shape"]))


@pytest.fixture(scope="session")
def golden():
    return load_golden
