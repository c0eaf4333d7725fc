"""CPU restatement of the reference integrators (TEST INFRASTRUCTURE ONLY).

Each function follows the cited reference lines operation for operation so
that, on the same inputs, it reproduces the reference bit for bit (checked
against golden vectors in tests/test_oracle_golden.py).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DIVERGENCE_LIMIT = 1.0e12   # src/timeint.py:33


class OracleDivergence(RuntimeError):
    def __init__(self, step, amplitude):
        super().__init__(f"diverged at step {step}: {amplitude:.3e}")
        self.step = step
        self.amplitude = amplitude


class Fact:
    """Diagonal or SuperLU factorisation, src/linalg.py:27-81."""

    def __init__(self, A):
        A = sp.csr_matrix(A)
        self.n = A.shape[0]
        coo = A.tocoo()
        nz = coo.data != 0.0
        if np.all(coo.row[nz] == coo.col[nz]):
            self.kind = "diagonal"
            self.d = A.diagonal().copy()
            if np.any(self.d <= 0.0) or not np.all(np.isfinite(self.d)):
                raise ValueError("indefinite diagonal")
            self.lu = None
        else:
            self.kind = "sparse_lu"
            self.lu = spla.splu(A.tocsc(), permc_spec="MMD_AT_PLUS_A",
                                diag_pivot_thresh=0.0, options={"SymmetricMode": True})
            piv = self.lu.U.diagonal()
            if np.any(piv <= 0.0) or not np.all(np.isfinite(piv)):
                raise ValueError("indefinite matrix")

    def solve(self, b):
        b = np.asarray(b, dtype=float)
        if self.kind == "diagonal":
            return b / self.d if b.ndim == 1 else b / self.d[:, None]
        return self.lu.solve(b)


def _check(psi, step):
    # src/timeint.py:91-94
    amp = float(np.max(np.abs(psi))) if psi.size else 0.0
    if not np.isfinite(amp) or amp > DIVERGENCE_LIMIT:
        raise OracleDivergence(step, amp)


def _obs_init(obs_mat, n_t):
    if obs_mat is None:
        return None
    return np.empty((obs_mat.shape[0], n_t + 1))


def cdm_run(M, K, F_s, f_t, dt, n_t, obs_mat=None, psi0=None, v0=None):
    """src/timeint.py:159-193.  Returns (psi, obs, t)."""
    n = M.shape[0]
    psi = np.zeros(n) if psi0 is None else np.array(psi0, dtype=float)
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=float)
    fac = Fact(M)
    obs = _obs_init(obs_mat, n_t)
    a = fac.solve(f_t(0.0) * F_s - K @ psi)            # :175
    prev = psi - dt * v + (0.5 * dt * dt) * a           # :176
    if obs is not None:
        obs[:, 0] = obs_mat @ psi
    for k in range(n_t):                                # :179-190
        rhs = f_t(k * dt) * F_s - K @ psi
        new = 2.0 * psi - prev + (dt * dt) * fac.solve(rhs)
        prev, psi = psi, new
        if obs is not None:
            obs[:, k + 1] = obs_mat @ psi
        _check(psi, k + 1)
    return psi, obs, np.arange(n_t + 1) * dt


def newmark_run(M, K, F_s, f_t, dt, n_t, obs_mat=None, beta=0.25, gamma=0.5,
                psi0=None, v0=None):
    """src/timeint.py:109-156.  Returns (psi, v, obs)."""
    n = M.shape[0]
    psi = np.zeros(n) if psi0 is None else np.array(psi0, dtype=float)
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=float)
    if beta != 0.0:
        S = Fact((M + (beta * dt * dt) * K).tocsr())
        Mf = Fact(M)
    else:
        S = Fact(M)
        Mf = S
    obs = _obs_init(obs_mat, n_t)
    a = Mf.solve(f_t(0.0) * F_s - K @ psi)
    if obs is not None:
        obs[:, 0] = obs_mat @ psi
    for k in range(n_t):
        t_new = (k + 1) * dt
        pp = psi + dt * v + (0.5 * dt * dt * (1.0 - 2.0 * beta)) * a
        vp = v + (dt * (1.0 - gamma)) * a
        a = S.solve(f_t(t_new) * F_s - K @ pp)
        psi = pp + (beta * dt * dt) * a
        v = vp + (gamma * dt) * a
        if obs is not None:
            obs[:, k + 1] = obs_mat @ psi
        _check(psi, k + 1)
    return psi, v, obs


def imex_run(M, K, F_s, f_t, dt, n_t, c_idx, d_idx, obs_mat=None, beta=0.25,
             gamma=0.5, psi0=None, v0=None):
    """src/timeint.py:196-292.  Returns (psi, v_out, obs)."""
    n = M.shape[0]
    c_idx = np.asarray(c_idx, dtype=np.int64)
    d_idx = np.asarray(d_idx, dtype=np.int64)
    psi = np.zeros(n) if psi0 is None else np.array(psi0, dtype=float)
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=float)
    M = sp.csr_matrix(M)
    K = sp.csr_matrix(K)
    has_d, has_c = d_idx.size > 0, c_idx.size > 0
    if has_d:
        m_d = M[d_idx][:, d_idx].diagonal()
        K_d = K[d_idx]
    if has_c:
        M_cc = M[c_idx][:, c_idx]
        K_c = K[c_idx]
        K_cc = K_c[:, c_idx]
        S = Fact((M_cc + (beta * dt * dt) * K_cc).tocsr())
        Mcc = Fact(M_cc)
    obs = _obs_init(obs_mat, n_t)
    r0 = f_t(0.0) * F_s - K @ psi
    a_c = Mcc.solve(r0[c_idx]) if has_c else None
    if has_d:
        a_d = r0[d_idx] / m_d
        prev_d = psi[d_idx] - dt * v[d_idx] + (0.5 * dt * dt) * a_d
    if has_c:
        psi_c = psi[c_idx].copy()
        v_c = v[c_idx].copy()
    if obs is not None:
        obs[:, 0] = obs_mat @ psi
    for k in range(n_t):
        t_k = k * dt
        t_new = t_k + dt
        if has_d:
            rhs_d = f_t(t_k) * F_s[d_idx] - K_d @ psi
            new_d = 2.0 * psi[d_idx] - prev_d + (dt * dt) * (rhs_d / m_d)
            prev_d = psi[d_idx].copy()
            psi[d_idx] = new_d
        if has_c:
            pc = psi_c + dt * v_c + (0.5 * dt * dt * (1.0 - 2.0 * beta)) * a_c
            vp = v_c + (dt * (1.0 - gamma)) * a_c
            psi[c_idx] = pc
            rhs_c = f_t(t_new) * F_s[c_idx] - K_c @ psi
            a_c = S.solve(rhs_c)
            psi_c = pc + (beta * dt * dt) * a_c
            v_c = vp + (gamma * dt) * a_c
            psi[c_idx] = psi_c
        if obs is not None:
            obs[:, k + 1] = obs_mat @ psi
        _check(psi, k + 1)
    v_out = None
    if has_c and not has_d:
        v_out = np.zeros(n)
        v_out[c_idx] = v_c
    return psi, v_out, obs


def max_gen_eig(K, M, tol=1e-9, max_iter=50000, seed=0):
    """src/linalg.py:89-122.  Returns (lam, n_iter)."""
    n = K.shape[0]
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    x /= np.linalg.norm(x)
    fac = Fact(M)
    lam_old = np.inf
    for it in range(1, max_iter + 1):
        y = fac.solve(K @ x)
        ny = np.linalg.norm(y)
        if ny == 0.0:
            return 0.0, it
        x = y / ny
        lam = float(x @ (K @ x)) / float(x @ (M @ x))
        if abs(lam - lam_old) <= tol * abs(lam):
            return lam, it
        lam_old = lam
    raise RuntimeError("power iteration did not converge")


def dt_crit(K, M, tol=1e-9, seed=0):
    """src/linalg.py:125-130."""
    lam, _ = max_gen_eig(K, M, tol=tol, seed=seed)
    return 2.0 / np.sqrt(lam)


def ricker(t, f_e):
    """src/assembly.py:43-49."""
    t = np.asarray(t, dtype=float)
    t_s = 2.0 * np.sqrt(6.0) / (np.pi * f_e)
    q = np.pi * f_e * (t - t_s)
    return (1.0 - 2.0 * q * q) * np.exp(-q * q)
