"""Implicit-explicit split integration on the device: drop-in for
``wavecell.timeint.imex_run`` (src/timeint.py:196-292).

The host does what the reference does once per run: validate the partition
and the mass structure (same checks and messages, src/timeint.py:210-236) and
factorise ``S_cc = M_cc + beta dt^2 K_cc`` and ``M_cc`` with SuperLU in the
reference's own configuration (``factorize``, src/linalg.py:70-80).  The
factors are uploaded once; every step -- the explicit d update (the
operator's fused CDM kernel), the c predictor, the c-row stiffness apply,
both sparse triangular solves and the corrector -- runs on the B200.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import _lib
from .linalg import IndefiniteMatrixError, is_structurally_diagonal
from .operators import DeviceOperator, as_device_operator
from .timeint import DivergenceError, RunResult, StageTimings, _observer, eval_force


def _splu(A):
    """SuperLU exactly as the reference's ``factorize`` (src/linalg.py:70-80)."""
    A = sp.csc_matrix(A)
    try:
        lu = spla.splu(A, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                       options={"SymmetricMode": True})
    except RuntimeError as exc:
        raise IndefiniteMatrixError(f"factorization failed: {exc}") from exc
    piv = lu.U.diagonal()
    if np.any(piv <= 0.0) or not np.all(np.isfinite(piv)):
        raise IndefiniteMatrixError(
            "matrix is not positive definite; check the stabilization and lumping settings")
    return lu


class _LU:
    """Host-side CSR copies of SuperLU's factors, kept alive for the ABI."""

    def __init__(self, lu):
        L = sp.csr_matrix(lu.L)
        U = sp.csr_matrix(lu.U)
        L.sort_indices()
        U.sort_indices()
        self.keep = [np.ascontiguousarray(lu.perm_r, dtype=np.int64),
                     np.ascontiguousarray(lu.perm_c, dtype=np.int64),
                     np.ascontiguousarray(L.indptr, dtype=np.int64),
                     np.ascontiguousarray(L.indices, dtype=np.int32),
                     np.ascontiguousarray(L.data, dtype=np.float64),
                     np.ascontiguousarray(U.indptr, dtype=np.int64),
                     np.ascontiguousarray(U.indices, dtype=np.int32),
                     np.ascontiguousarray(U.data, dtype=np.float64)]
        s = _lib.LU()
        s.n = L.shape[0]
        s.perm_r, s.perm_c = _lib.i64ptr(self.keep[0]), _lib.i64ptr(self.keep[1])
        s.L_indptr, s.L_indices, s.L_data = (_lib.i64ptr(self.keep[2]), _lib.i32ptr(self.keep[3]),
                                            _lib.dptr(self.keep[4]))
        s.U_indptr, s.U_indices, s.U_data = (_lib.i64ptr(self.keep[5]), _lib.i32ptr(self.keep[6]),
                                            _lib.dptr(self.keep[7]))
        self.struct = s


def _host_stiffness(K):
    """Host CSR of K (for the c-c block of the iteration matrix)."""
    from .operators import _tensor_system_of, tensor_csr
    tensor = getattr(K, "tensor", None) if isinstance(K, DeviceOperator) else _tensor_system_of(K)
    if tensor is not None:
        return tensor_csr(tensor)
    if isinstance(K, DeviceOperator):
        prob = getattr(K, "problem", None)
        if prob is None:
            raise NotImplementedError("imex_run needs the host stiffness of a device operator "
                                      "(build it from an ScmProblem)")
        return prob.csr_stiffness()
    return sp.csr_matrix(K)


class ImexPlan:
    """Device-resident IMEX split for repeated runs at one ``(dt, beta)``:
    validation and SuperLU factorisation of ``S_cc`` / ``M_cc`` happen once
    (src/timeint.py:210-245), ``run`` is the stepping loop (:246-292)."""

    def __init__(self, M, K, F_s, dt: float, c_idx, d_idx, obs_mat=None, beta: float = 0.25,
                 device: int | None = None):
        M = sp.csr_matrix(M)
        n = M.shape[0]
        c_idx = np.asarray(c_idx, dtype=np.int64)
        d_idx = np.asarray(d_idx, dtype=np.int64)
        if c_idx.shape[0] + d_idx.shape[0] != n:
            raise ValueError("c and d index sets must partition the DOFs")
        self.dt = float(dt)
        self.beta = float(beta)
        self.n = n
        has_d, has_c = d_idx.shape[0] > 0, c_idx.shape[0] > 0
        self.has_c, self.has_d = has_c, has_d
        self.c_idx = c_idx
        t0 = time.perf_counter()
        m_d = np.zeros(0)
        if has_d:
            M_drows = M[d_idx]
            if M_drows[:, c_idx].nnz != 0:
                raise ValueError("d mass rows couple into the implicit set; the basis/lumping "
                                 "choice does not support the implicit-explicit split")
            M_dd = M_drows[:, d_idx]
            if not is_structurally_diagonal(M_dd):
                raise ValueError("d mass block is not diagonal; the basis/lumping choice does "
                                 "not support the implicit-explicit split")
            m_d = np.ascontiguousarray(M_dd.diagonal(), dtype=np.float64)
            if np.any(m_d <= 0.0):
                raise ValueError("d mass block has non-positive diagonal entries")
        S_lu = M_lu = None
        if has_c:
            M_cc = M[c_idx][:, c_idx]
            prob = getattr(K, "problem", None)
            if isinstance(K, DeviceOperator) and hasattr(prob, "stiffness_block"):
                K_cc = prob.stiffness_block(c_idx)       # from the cells touching c only
            else:
                K_cc = _host_stiffness(K)[c_idx][:, c_idx]
            S_lu = _LU(_splu((M_cc + (self.beta * self.dt * self.dt) * K_cc).tocsr()))
            M_lu = _LU(_splu(M_cc))
        self.factorization = time.perf_counter() - t0
        self.fact_nnz = 0 if S_lu is None else int(S_lu.keep[4].shape[0] + S_lu.keep[7].shape[0])
        op = as_device_operator(K, device=device)
        if op.n != n:
            raise ValueError("K and M sizes differ")
        self.op = op
        F = np.ascontiguousarray(np.asarray(F_s, dtype=np.float64).reshape(-1))
        obs, self._obs_keep = _observer(obs_mat, n)
        self.n_obs = 0 if obs is None else int(obs.n_obs)
        ci = np.ascontiguousarray(c_idx)
        di = np.ascontiguousarray(d_idx)
        h = _lib.C.c_void_p()
        _lib.check(_lib.load().wcb_imex_plan_create(
            op.handle, ci.shape[0], _lib.i64ptr(ci) if has_c else None, di.shape[0],
            _lib.i64ptr(di) if has_d else None, _lib.dptr(m_d) if has_d else None,
            _lib.C.byref(S_lu.struct) if has_c else None,
            _lib.C.byref(M_lu.struct) if has_c else None, _lib.dptr(F),
            _lib.C.byref(obs) if obs is not None else None, _lib.C.byref(h)))
        self._h = h
        del S_lu, M_lu    # uploaded; the host factors are not needed any more

    def run(self, f_t, n_t: int, gamma: float = 0.5, psi0=None, v0=None,
            record: bool = True, new_times=None) -> RunResult:
        """``new_times`` (length n_t) overrides the implicit stage's force
        times: IMEX evaluates ``f_t(k dt + dt)`` (src/timeint.py:258-259),
        Newmark ``f_t((k + 1) dt)`` (src/timeint.py:141) -- equal in exact
        arithmetic, not always in floating point."""
        n_t = int(n_t)
        dt = self.dt
        n = self.n
        f0 = float(f_t(0.0))
        ks = np.arange(n_t, dtype=np.float64) * dt
        ft_k = eval_force(f_t, ks) if n_t else np.zeros(1)
        tn = ks + dt if new_times is None else np.asarray(new_times, dtype=np.float64)
        if tn.shape[0] != n_t:
            raise ValueError("new_times must hold n_t entries")
        ft_new = eval_force(f_t, tn) if n_t else np.zeros(1)
        p0 = None if psi0 is None else np.ascontiguousarray(np.array(psi0, dtype=float).reshape(-1))
        q0 = None if v0 is None else np.ascontiguousarray(np.array(v0, dtype=float).reshape(-1))
        psi = np.empty(n)
        nc = self.c_idx.shape[0]
        vc = np.empty(max(nc, 1))
        obs_out = np.empty((self.n_obs, n_t + 1)) if (self.n_obs and record) else None
        div = _lib.Divergence()
        tm = _lib.Timings()
        code = _lib.load().wcb_imex_plan_run(
            self._h, f0, _lib.dptr(ft_k), _lib.dptr(ft_new), dt, n_t, self.beta, float(gamma),
            _lib.dptr(p0), _lib.dptr(q0), _lib.dptr(psi), _lib.dptr(vc) if self.has_c else None,
            _lib.dptr(obs_out) if obs_out is not None else None,
            _lib.C.byref(div), _lib.C.byref(tm))
        if code == _lib.WCB_E_DIVERGED:
            raise DivergenceError(int(div.step), float(div.amplitude))
        _lib.check(code)
        v_out = None
        if self.has_c and not self.has_d:
            v_out = np.zeros(n)
            v_out[self.c_idx] = vc[:nc]
        timings = StageTimings(factorization=self.factorization, rhs=float(tm.rhs),
                               backward_insertion=float(tm.backward_insertion))
        return RunResult(method="imex", dt=dt, t=np.arange(n_t + 1) * dt, obs=obs_out, psi=psi,
                         psi_dot=v_out, timings=timings, fact_dim=int(nc))

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().wcb_imex_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MassPlan(ImexPlan):
    """Device-resident consistent (non-diagonal) mass for ``cdm_run`` and
    ``max_gen_eig`` -- the reference's ``factorize`` SuperLU path
    (src/linalg.py:70-80, used by src/timeint.py:166-176 and
    src/linalg.py:106-116).  ``M`` is split into its diagonal-only rows (d,
    divided by m_d) and the coupled rows (c, ``M_cc`` factorised once with
    SuperLU in the reference configuration, both triangular solves on the
    B200 every step / iteration); see :func:`linalg.mass_split`."""

    def __init__(self, M, K, F_s, obs_mat=None, device: int | None = None):
        from .linalg import mass_split
        t0 = time.perf_counter()
        c_idx, d_idx, m_d, M_cc = mass_split(M)
        n = sp.csr_matrix(M).shape[0]
        self.n = n
        self.dt = 0.0
        self.beta = 0.0
        self.c_idx = c_idx
        self.has_c, self.has_d = c_idx.shape[0] > 0, d_idx.shape[0] > 0
        M_lu = _LU(_splu(M_cc)) if self.has_c else None
        M_cc.sort_indices()
        mcc = (np.ascontiguousarray(M_cc.indptr, dtype=np.int64),
               np.ascontiguousarray(M_cc.indices, dtype=np.int32),
               np.ascontiguousarray(M_cc.data, dtype=np.float64))
        self.factorization = time.perf_counter() - t0
        self.fact_nnz = 0 if M_lu is None else int(M_lu.keep[4].shape[0] + M_lu.keep[7].shape[0])
        op = as_device_operator(K, device=device)
        if op.n != n:
            raise ValueError("K and M sizes differ")
        self.op = op
        F = np.ascontiguousarray(np.asarray(F_s, dtype=np.float64).reshape(-1))
        if F.shape[0] != n:
            raise ValueError("F_s has the wrong length")
        obs, self._obs_keep = _observer(obs_mat, n)
        self.n_obs = 0 if obs is None else int(obs.n_obs)
        h = _lib.C.c_void_p()
        _lib.check(_lib.load().wcb_mass_plan_create(
            op.handle, c_idx.shape[0], _lib.i64ptr(c_idx) if self.has_c else None, d_idx.shape[0],
            _lib.i64ptr(d_idx) if self.has_d else None, _lib.dptr(m_d) if self.has_d else None,
            _lib.C.byref(M_lu.struct) if self.has_c else None, _lib.i64ptr(mcc[0]),
            _lib.i32ptr(mcc[1]), _lib.dptr(mcc[2]), _lib.dptr(F),
            _lib.C.byref(obs) if obs is not None else None, _lib.C.byref(h)))
        self._h = h
        del M_lu

    def max_gen_eig(self, x0, tol=1e-9, max_iter=50000):
        """Power iteration of src/linalg.py:89-122 with this mass."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        lam = _lib.C.c_double(0.0)
        it = _lib.C.c_int64(0)
        code = _lib.load().wcb_imex_plan_max_gen_eig(self._h, _lib.dptr(x0), float(tol), int(max_iter),
                                                     _lib.C.byref(lam), _lib.C.byref(it))
        if code == _lib.WCB_E_NOCONV:
            raise RuntimeError(_lib.last_error())
        _lib.check(code)
        return float(lam.value), int(it.value)

    def run_cdm(self, f_t, dt: float, n_t: int, psi0=None, v0=None, record: bool = True) -> RunResult:
        """``cdm_run`` (src/timeint.py:159-193) with this mass."""
        from .timeint import force_table
        n, dt, n_t = self.n, float(dt), int(n_t)
        ft = force_table(f_t, dt, n_t)
        p0 = None if psi0 is None else np.ascontiguousarray(np.array(psi0, dtype=float).reshape(-1))
        q0 = None if v0 is None else np.ascontiguousarray(np.array(v0, dtype=float).reshape(-1))
        for a in (p0, q0):
            if a is not None and a.shape[0] != n:
                raise ValueError("initial state has the wrong length")
        psi = np.empty(n)
        obs = np.empty((self.n_obs, n_t + 1)) if (self.n_obs and record) else None
        div = _lib.Divergence()
        tm = _lib.Timings()
        code = _lib.load().wcb_imex_plan_cdm_run(
            self._h, _lib.dptr(ft), dt, n_t, _lib.dptr(p0), _lib.dptr(q0), _lib.dptr(psi),
            _lib.dptr(obs) if obs is not None else None, _lib.C.byref(div), _lib.C.byref(tm))
        if code == _lib.WCB_E_DIVERGED:
            raise DivergenceError(int(div.step), float(div.amplitude))
        _lib.check(code)
        timings = StageTimings(factorization=self.factorization, rhs=float(tm.rhs),
                               backward_insertion=float(tm.backward_insertion))
        return RunResult(method="cdm", dt=dt, t=np.arange(n_t + 1) * dt, obs=obs, psi=psi,
                         psi_dot=None, timings=timings, fact_dim=n)

    def run(self, *args, **kwargs):
        raise NotImplementedError("a MassPlan has no S_cc factors: use run_cdm or ImexPlan")


def imex_run(M, K, F_s, f_t, dt: float, n_t: int, c_idx, d_idx, obs_mat=None,
             beta: float = 0.25, gamma: float = 0.5, psi0=None, v0=None,
             device: int | None = None) -> RunResult:
    """Implicit-explicit split integration, src/timeint.py:196-292, on the device."""
    plan = ImexPlan(M, K, F_s, dt, c_idx, d_idx, obs_mat=obs_mat, beta=beta, device=device)
    try:
        return plan.run(f_t, n_t, gamma=gamma, psi0=psi0, v0=v0)
    finally:
        plan.close()


def newmark_run(M, K, F_s, f_t, dt: float, n_t: int, obs_mat=None, beta: float = 0.25,
                gamma: float = 0.5, psi0=None, v0=None, s_factory=None,
                device: int | None = None) -> RunResult:
    """Newmark-beta on the device, src/timeint.py:109-156.

    Every DOF is implicit: ``S = M + beta dt^2 K`` and ``M`` are factorised
    once with SuperLU in the reference configuration (for ``beta = 0``,
    ``S = M`` as in the reference) and each step runs predictor, ``K``
    apply, the two triangular solves and the corrector on the B200 -- the
    IMEX plan with an empty explicit set, whose per-step arithmetic is the
    reference's Newmark loop line by line.

    ``s_factory`` (src/timeint.py:126-128) is called once, as the reference
    does, and must return an object for ``S`` (``.solve``, optional ``.n``).
    Its solve runs on the host, so the device loop does not call it: the
    device factorises the same ``S`` itself (the reference's own factories --
    ``TensorSystem.newmark_factorization``, src/assembly.py:699-704 -- solve
    ``S`` by fast diagonalisation or by CG to a 1e-13 residual, so the fields
    agree to that solve tolerance).  ``K`` must then be available as a
    matrix: a sparse/dense ``K``, a ``TensorSystem`` stiffness operator or a
    device operator built from a problem description.
    """
    if s_factory is not None:
        S_obj = s_factory()
        n_s = getattr(S_obj, "n", None)
        if not callable(getattr(S_obj, "solve", None)):
            raise TypeError("s_factory() must return an object with a solve(b) method")
        if n_s is not None and int(n_s) != sp.csr_matrix(M).shape[0]:
            raise ValueError("s_factory() returned a factorization of the wrong size")
    n = sp.csr_matrix(M).shape[0]
    plan = ImexPlan(M, K, F_s, dt, np.arange(n, dtype=np.int64), np.zeros(0, dtype=np.int64),
                    obs_mat=obs_mat, beta=beta, device=device)
    try:
        r = plan.run(f_t, n_t, gamma=gamma, psi0=psi0, v0=v0,
                     new_times=np.arange(1, int(n_t) + 1, dtype=np.float64) * float(dt))
    finally:
        plan.close()
    return RunResult(method="newmark", dt=r.dt, t=r.t, obs=r.obs, psi=r.psi, psi_dot=r.psi_dot,
                     timings=r.timings, fact_dim=n)
