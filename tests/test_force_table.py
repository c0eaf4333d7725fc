"""Force tables (src/timeint.py:180-182: f_t is called once per step with a
Python float).  The drop-in may evaluate f_t in one array call, but only keeps
that table when it equals the scalar calls bit for bit."""

import numpy as np
import pytest

from paper_2501_19013_b200.setup.configs import ricker
from paper_2501_19013_b200.timeint import eval_force, eval_force_deferred


def _bumped(t):
    """sin, except that the array form is off by one ulp-ish at entry 777."""
    if np.ndim(t):
        r = np.sin(t)
        r[777] += 1e-16
        return r
    return np.sin(t)


def test_vectorised_table_is_verified_everywhere():
    t = np.arange(2000) * 1e-4
    ref = np.array([float(np.sin(float(x))) for x in t])
    assert np.array_equal(eval_force(_bumped, t), ref)          # falls back to the scalar loop
    v, check = eval_force_deferred(_bumped, t)
    assert check is not None and check() is False               # the probes pass, the full check does not


def test_exact_vectorised_table_is_kept():
    f = lambda x: ricker(x, 10.0)  # noqa: E731
    t = np.arange(3000) * 2e-4
    ref = np.array([float(f(float(x))) for x in t])
    assert np.array_equal(eval_force(f, t), ref)
    v, check = eval_force_deferred(f, t)
    assert np.array_equal(v, ref) and (check is None or check() is True)


def test_scalar_only_callable():
    def f(x):
        if np.ndim(x):
            raise TypeError("scalar only")
        return float(x) ** 2
    t = np.arange(100) * 0.5
    v, check = eval_force_deferred(f, t)
    assert check is None and np.array_equal(v, t ** 2)


@pytest.mark.gpu
def test_cdm_run_repeats_with_the_scalar_table_on_a_mismatch():
    """A callable whose array form differs from its scalar form in one entry:
    the run must be the scalar table's (the verification runs beside the
    device loop and the loop is repeated)."""
    import scipy.sparse as sp
    from paper_2501_19013_b200 import cdm_run
    n = 200
    K = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n)).tocsr()
    M = sp.identity(n, format="csr")
    F = np.zeros(n)
    F[n // 2] = 1.0
    calls = {"n": 0}

    def f_bad(t):
        if np.ndim(t):
            r = np.sin(40.0 * t)
            r[500] += 1e-3
            return r
        calls["n"] += 1
        return np.sin(40.0 * t)

    f_ref = lambda t: float(np.sin(40.0 * float(t)))  # noqa: E731
    a = cdm_run(M, K, F, f_bad, 0.05, 1500)
    b = cdm_run(M, K, F, f_ref, 0.05, 1500)
    assert np.array_equal(a.psi, b.psi)
