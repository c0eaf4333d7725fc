"""Device time integration: drop-in for ``wavecell.timeint``.

Same names, signatures, return type and error behaviour as the reference
(src/timeint.py:1-303):

* :func:`cdm_run` -- central differences, src/timeint.py:159-193.  The whole
  step loop runs on the B200; one fused kernel per step computes
  ``psi_{k+1} = 2 psi_k - psi_{k-1} + dt^2 M^-1 (f_t(k dt) F_s - K psi_k)``,
  the divergence amplitude and (optionally) the observer samples.
* :func:`imex_run` -- Algorithm 2, src/timeint.py:196-292 (device IMEX plan).
* :func:`select_dt`, :func:`imex_critical_time_step` -- src/timeint.py:71-88.

The force ``f_t`` is evaluated on the host at exactly the reference's float
times (``k * dt``; ``t_k + dt`` for IMEX) and shipped as a table, so the device
sees bit-identical force values.  Stage timings come from CUDA events; the K
apply and the update are one kernel, so the loop time is reported under
``rhs`` and ``backward_insertion`` stays 0 for CDM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .linalg import (IndefiniteMatrixError, diagonal_mass, dt_crit as _dt_crit,
                     is_structurally_diagonal)
from .operators import DeviceOperator, as_device_operator

DIVERGENCE_LIMIT = 1.0e12


class DivergenceError(RuntimeError):
    """The solution amplitude exploded (unstable time step), src/timeint.py:36-43."""

    def __init__(self, step: int, amplitude: float):
        super().__init__(
            f"solution diverged at step {step}: max |psi| = {amplitude:.3e}")
        self.step = step
        self.amplitude = amplitude


@dataclass
class StageTimings:
    """Accumulated seconds per solver stage (src/timeint.py:46-56)."""

    factorization: float = 0.0
    rhs: float = 0.0
    backward_insertion: float = 0.0

    @property
    def total(self) -> float:
        return self.factorization + self.rhs + self.backward_insertion


@dataclass
class RunResult:
    """Integrator output (src/timeint.py:59-68)."""

    method: str
    dt: float
    t: np.ndarray
    obs: np.ndarray | None
    psi: np.ndarray
    psi_dot: np.ndarray | None
    timings: StageTimings
    fact_dim: int = 0


def select_dt(dt_c: float, dt_max: float | None = None, safety: float = 0.9) -> float:
    """Working step: safety factor times the critical step, capped
    (src/timeint.py:71-77)."""
    dt = safety * dt_c
    if dt_max is not None:
        dt = min(dt, dt_max)
    return dt


def _restrict(K, idx):
    """Principal submatrix K[idx][:, idx] on the host (scipy slicing)."""
    return sp.csr_matrix(K)[idx][:, idx]


def imex_critical_time_step(K, M, d_idx, tol: float = 1e-9, seed: int = 0,
                            device: int | None = None) -> float:
    """Critical step of the explicit (d) subsystem (src/timeint.py:80-88)."""
    d_idx = np.asarray(d_idx)
    if d_idx.shape[0] == 0:
        raise ValueError("explicit subsystem is empty")
    if isinstance(K, DeviceOperator):
        # power iteration on the d block inside the operator's own apply
        from .linalg import max_gen_eig_sub
        M_dd = _restrict(M, d_idx)
        if not is_structurally_diagonal(M_dd):
            raise NotImplementedError("the d mass block must be diagonal")
        m = np.ones(K.n)
        m[np.asarray(d_idx, dtype=np.int64)] = sp.csr_matrix(M_dd).diagonal()
        lam, _ = max_gen_eig_sub(K, m, d_idx, tol=tol, seed=seed)
        if lam <= 0.0:
            raise ValueError("largest generalized eigenvalue must be positive")
        return 2.0 / np.sqrt(lam)
    K_dd = _restrict(K, d_idx)
    M_dd = _restrict(M, d_idx)
    return _dt_crit(K_dd, M_dd, tol=tol, seed=seed, device=device)


def eval_force(f_t, t) -> np.ndarray:
    """``[float(f_t(float(x))) for x in t]`` bit for bit.  A NumPy ufunc
    expression is evaluated in one array call and kept only if it reproduces
    the scalar calls exactly -- at every point for tables up to 20000 entries,
    else at 4096 evenly strided points plus both ends (SIMD and scalar
    transcendentals can differ in the last bit, so the check is not a
    formality); anything else runs the reference's scalar loop."""
    t = np.asarray(t, dtype=np.float64)
    n = t.shape[0]
    if n > 64:
        try:
            with np.errstate(all="ignore"):
                v = np.array(f_t(t), dtype=np.float64)
            if v.shape == (n,):
                probe = np.arange(n) if n <= 20000 else np.unique(
                    np.concatenate([np.linspace(0, n - 1, 4096).astype(np.int64), [0, 1, n - 2, n - 1]]))
                if all(v[k] == float(f_t(float(t[k]))) for k in probe):
                    return v
        except Exception:
            pass
    return np.array([float(f_t(float(x))) for x in t], dtype=np.float64).reshape(n)


def eval_force_deferred(f_t, t):
    """``(table, check)``: like :func:`eval_force`, but when the one-call array
    evaluation passes a few probe points its point-by-point verification is
    returned as ``check`` (a callable giving True when the table equals the
    scalar calls bit for bit) instead of being run.  ``check`` is ``None`` when
    the table already is the scalar loop's.  :meth:`CdmPlan.run` verifies on a
    second thread while the device loop runs and repeats the run with the
    scalar table in the (so far unseen) case of a mismatch, so the result
    always belongs to the bit-exact table."""
    t = np.asarray(t, dtype=np.float64)
    n = t.shape[0]
    if n > 64:
        try:
            with np.errstate(all="ignore"):
                v = np.array(f_t(t), dtype=np.float64)
            if v.shape == (n,):
                quick = sorted({0, 1, n // 3, n // 2, (2 * n) // 3, n - 2, n - 1})
                if all(v[k] == float(f_t(float(t[k]))) for k in quick):
                    probe = np.arange(n) if n <= 20000 else np.unique(
                        np.concatenate([np.linspace(0, n - 1, 4096).astype(np.int64), [0, 1, n - 2, n - 1]]))

                    def check():
                        try:
                            return all(v[k] == float(f_t(float(t[k]))) for k in probe)
                        except Exception:
                            return False
                    return v, check
        except Exception:
            pass
    return np.array([float(f_t(float(x))) for x in t], dtype=np.float64).reshape(n), None


def force_table(f_t, dt: float, n_t: int) -> np.ndarray:
    """``[f_t(k * dt) for k in range(n_t)]`` at the reference's float times
    (src/timeint.py:180-182); entry 0 is ``f_t(0.0)`` (the bootstrap force,
    src/timeint.py:175) and is always present."""
    n = max(int(n_t), 1)
    return eval_force(f_t, np.arange(n, dtype=np.float64) * dt)


def _observer(obs_mat, n):
    if obs_mat is None:
        return None, None
    A = sp.csr_matrix(obs_mat, dtype=np.float64)
    if A.shape[1] != n:
        raise ValueError("observer matrix has the wrong number of columns")
    keep = (np.ascontiguousarray(A.indptr, dtype=np.int64),
            np.ascontiguousarray(A.indices, dtype=np.int64),
            np.ascontiguousarray(A.data, dtype=np.float64))
    o = _lib.Observer()
    o.n_obs = A.shape[0]
    o.indptr = _lib.i64ptr(keep[0])
    o.indices = _lib.i64ptr(keep[1])
    o.data = _lib.dptr(keep[2])
    return o, keep


class CdmPlan:
    """Device-resident ``(K, M, F_s, obs_mat)`` for repeated CDM runs."""

    def __init__(self, M, K, F_s, obs_mat=None, device: int | None = None):
        self.op = as_device_operator(K, device=device)
        n = self.op.n
        self.m = diagonal_mass(M)
        if self.m.shape[0] != n:
            raise ValueError("K and M sizes differ")
        self.F_s = np.ascontiguousarray(np.asarray(F_s, dtype=np.float64).reshape(-1))
        if self.F_s.shape[0] != n:
            raise ValueError("F_s has the wrong length")
        obs, self._obs_keep = _observer(obs_mat, n)
        self.n_obs = 0 if obs is None else int(obs.n_obs)
        h = _lib.C.c_void_p()
        _lib.check(_lib.load().wcb_cdm_plan_create(
            self.op.handle, _lib.dptr(self.m), _lib.dptr(self.F_s),
            _lib.C.byref(obs) if obs is not None else None, _lib.C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def step_bytes(self) -> float:
        """Algorithmic HBM bytes of one fused time step of this plan (32 B per
        DOF, 24 B where 1/m comes from the interior-cell table, plus the
        operator's cut-cell / CSR data)."""
        out = _lib.C.c_double()
        _lib.check(_lib.load().wcb_cdm_plan_step_bytes(self._h, _lib.C.byref(out)))
        return float(out.value)

    def run(self, f_t, dt: float, n_t: int, psi0=None, v0=None,
            record: bool = True, record_every: int = 1) -> RunResult:
        """``record_every = s`` keeps the observers at steps 0, s, 2s, ...
        only (``RunResult.t`` / ``obs`` hold those columns): the exact-hit
        samples of ``sample_observers`` (src/harness.py:101-131) without the
        full history."""
        n = self.op.n
        dt = float(dt)
        n_t = int(n_t)
        rec = int(record_every)
        if rec < 1:
            raise ValueError("record_every must be >= 1")
        times = np.arange(max(n_t, 1), dtype=np.float64) * dt
        ft, check = eval_force_deferred(f_t, times)
        psi0_a = None if psi0 is None else np.ascontiguousarray(
            np.array(psi0, dtype=float).reshape(-1))
        v0_a = None if v0 is None else np.ascontiguousarray(np.array(v0, dtype=float).reshape(-1))
        for a in (psi0_a, v0_a):
            if a is not None and a.shape[0] != n:
                raise ValueError("initial state has the wrong length")
        while True:
            psi = np.empty(n)
            obs = np.empty((self.n_obs, n_t // rec + 1)) if (self.n_obs and record) else None
            div = _lib.Divergence()
            tm = _lib.Timings()
            verdict = []
            th = None
            if check is not None:   # verify the array-evaluated table while the device loop runs
                import threading
                th = threading.Thread(target=lambda: verdict.append(check()))
                th.start()
            code = _lib.load().wcb_cdm_plan_run_sampled(
                self._h, _lib.dptr(ft), dt, n_t, rec, _lib.dptr(psi0_a), _lib.dptr(v0_a),
                _lib.dptr(psi), _lib.dptr(obs) if obs is not None else None,
                _lib.C.byref(div), _lib.C.byref(tm))
            if th is not None:
                th.join()
                if not (verdict and verdict[0]):   # not bit-identical: the scalar table decides
                    ft = np.array([float(f_t(float(x))) for x in times], dtype=np.float64)
                    check = None
                    continue
            break
        if code == _lib.WCB_E_DIVERGED:
            raise DivergenceError(int(div.step), float(div.amplitude))
        _lib.check(code)
        t = np.arange(0, n_t + 1, rec) * dt
        timings = StageTimings(factorization=0.0, rhs=float(tm.rhs),
                               backward_insertion=float(tm.backward_insertion))
        return RunResult(method="cdm", dt=dt, t=t, obs=obs, psi=psi, psi_dot=None,
                         timings=timings, fact_dim=0)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().wcb_cdm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cdm_run(M, K, F_s, f_t, dt: float, n_t: int, obs_mat=None, psi0=None,
            v0=None, device: int | None = None) -> RunResult:
    """Central difference method in two-step displacement form, on the device
    (src/timeint.py:159-193).  A diagonal ``M`` takes the fused one-kernel
    step (``factorize``'s fast path, ``fact_dim = 0``); any other SPD ``M``
    the consistent-mass plan (SuperLU factors of its coupled block, device
    triangular solves every step, ``fact_dim = n``).  ``K`` is any
    sparse/dense matrix, a ``TensorSystem`` stiffness operator or a
    :class:`DeviceOperator`."""
    try:
        plan = CdmPlan(M, K, F_s, obs_mat=obs_mat, device=device)
    except NotImplementedError:
        from .imex import MassPlan
        mplan = MassPlan(M, K, F_s, obs_mat=obs_mat, device=device)
        try:
            return mplan.run_cdm(f_t, dt, n_t, psi0=psi0, v0=v0)
        finally:
            mplan.close()
    try:
        return plan.run(f_t, dt, n_t, psi0=psi0, v0=v0)
    finally:
        plan.close()


def imex_run(M, K, F_s, f_t, dt: float, n_t: int, c_idx, d_idx, obs_mat=None,
             beta: float = 0.25, gamma: float = 0.5, psi0=None, v0=None,
             device: int | None = None) -> RunResult:
    """Implicit-explicit split integration on the device (src/timeint.py:196-292)."""
    from .imex import imex_run as _imex_run
    return _imex_run(M, K, F_s, f_t, dt, n_t, c_idx, d_idx, obs_mat=obs_mat, beta=beta,
                     gamma=gamma, psi0=psi0, v0=v0, device=device)


def sample_history(result: RunResult, times) -> np.ndarray:
    """Observer history linearly interpolated onto the given times
    (src/timeint.py:295-303)."""
    if result.obs is None:
        raise ValueError("run was made without an observer matrix")
    times = np.asarray(times, dtype=float)
    out = np.empty((result.obs.shape[0], times.shape[0]))
    for i in range(result.obs.shape[0]):
        out[i] = np.interp(times, result.t, result.obs[i])
    return out


__all__ = ["DIVERGENCE_LIMIT", "DivergenceError", "StageTimings", "RunResult",
           "select_dt", "imex_critical_time_step", "force_table", "eval_force_deferred", "CdmPlan", "cdm_run",
           "imex_run", "sample_history", "IndefiniteMatrixError", "is_structurally_diagonal"]
