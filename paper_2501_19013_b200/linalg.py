"""Critical time step on the device: drop-in for ``wavecell.linalg``
``max_gen_eig`` / ``dt_crit`` (src/linalg.py:89-130).

Same signature, same seeded start vector (``default_rng(seed)``, normalised,
compact DOF order, src/linalg.py:103-105), same Rayleigh-quotient estimate and
stopping rule ``|lam - lam_old| <= tol |lam|`` (src/linalg.py:116-117).  The
iteration runs in HBM through the operator's own apply kernel; only the
converged estimate comes back.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _lib
from .operators import DeviceOperator, as_device_operator


class IndefiniteMatrixError(RuntimeError):
    """The matrix handed to ``factorize`` is not positive definite
    (src/linalg.py:23-24)."""


def is_structurally_diagonal(A) -> bool:
    """True if all stored nonzero entries of A lie on the diagonal
    (src/linalg.py:45-49)."""
    coo = sp.csr_matrix(A).tocoo()
    mask = coo.data != 0.0
    return bool(np.all(coo.row[mask] == coo.col[mask]))


def _csr_identity_pattern(M) -> bool:
    """Fast path: a CSR matrix storing exactly its diagonal, in order."""
    if not sp.issparse(M) or M.format != "csr" or M.shape[0] != M.shape[1]:
        return False
    n = M.shape[0]
    if M.nnz != n:
        return False
    ar = np.arange(n + 1, dtype=M.indptr.dtype)
    return bool(np.array_equal(M.indptr, ar) and np.array_equal(M.indices, ar[:n]))


def _native_diag(M):
    """Threaded native check of a CSR diagonal (wcb_csr_diagonal_check): the
    diagonal, or None when the pattern is not the identity; raises like
    factorize when a value is not positive/finite."""
    if not (sp.issparse(M) and M.format == "csr" and M.shape[0] == M.shape[1] and M.nnz == M.shape[0]):
        return None
    ip, ix = M.indptr, M.indices
    if ip.dtype != ix.dtype or ip.dtype not in (np.int32, np.int64) or M.data.dtype != np.float64:
        return None
    from . import _lib
    try:
        lib = _lib.load()
    except ImportError:
        return None
    d = np.ascontiguousarray(M.data)
    r = lib.wcb_csr_diagonal_check(M.shape[0], ip.ctypes.data, ix.ctypes.data, ip.dtype.itemsize,
                                   _lib.dptr(d))
    if r < 0:
        return None
    if r == 0:
        raise IndefiniteMatrixError("diagonal matrix has non-positive entries; "
                                    "check the stabilization and lumping settings")
    return d


def diagonal_mass(M) -> np.ndarray:
    """The diagonal of a structurally diagonal SPD mass, with the checks of
    ``factorize``'s fast path (src/linalg.py:63-69)."""
    if isinstance(M, np.ndarray) and M.ndim == 1:
        d = np.ascontiguousarray(M, dtype=np.float64)
    elif (d := _native_diag(M)) is not None:
        return d
    elif _csr_identity_pattern(M):
        d = np.ascontiguousarray(M.data, dtype=np.float64)
    else:
        A = sp.csr_matrix(M)
        if A.shape[0] != A.shape[1]:
            raise ValueError("matrix must be square")
        if not is_structurally_diagonal(A):
            raise NotImplementedError(
                "the device integrators need a diagonal (lumped / nodal) mass matrix; "
                "use imex_run for a consistent cut-cell mass block")
        d = np.ascontiguousarray(A.diagonal(), dtype=np.float64)
    if np.any(d <= 0.0) or not np.all(np.isfinite(d)):
        raise IndefiniteMatrixError(
            "diagonal matrix has non-positive entries; "
            "check the stabilization and lumping settings")
    return d


def mass_split(M):
    """Split a non-diagonal symmetric mass for the device: ``(c_idx, d_idx,
    m_d, M_cc)`` with c = the rows storing an off-diagonal nonzero and d the
    rows storing only their diagonal, so ``M = blockdiag(diag(m_d), M_cc)``
    after permutation (the factorize() SuperLU path, src/linalg.py:70-80, on
    the blocks).  Raises like factorize for a non-positive diagonal entry."""
    A = sp.csr_matrix(M, dtype=np.float64)
    if A.shape[0] != A.shape[1]:
        raise ValueError("matrix must be square")
    coo = A.tocoo()
    off = (coo.row != coo.col) & (coo.data != 0.0)
    is_c = np.zeros(A.shape[0], dtype=bool)
    is_c[coo.row[off]] = True
    is_c[coo.col[off]] = True
    c_idx = np.flatnonzero(is_c).astype(np.int64)
    d_idx = np.flatnonzero(~is_c).astype(np.int64)
    m_d = np.ascontiguousarray(A.diagonal()[d_idx], dtype=np.float64)
    if np.any(m_d <= 0.0) or not np.all(np.isfinite(m_d)):
        raise IndefiniteMatrixError("matrix is not positive definite; "
                                    "check the stabilization and lumping settings")
    return c_idx, d_idx, m_d, A[c_idx][:, c_idx].tocsr()


def start_vector(n: int, seed: int) -> np.ndarray:
    """Seeded normalised start vector of src/linalg.py:103-105."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    x /= np.linalg.norm(x)
    return x


def max_gen_eig(K, M, tol=1e-9, max_iter=50000, seed=0, device: int | None = None):
    """Largest eigenvalue of ``K x = lam M x`` by power iteration on the device.

    Returns ``(lam, n_iter)`` like src/linalg.py:89-122.
    """
    op = as_device_operator(K, device=device)
    n = op.n
    try:
        m = diagonal_mass(M)
    except NotImplementedError:
        # consistent mass: M^-1 through the device triangular solves of M_cc
        from .imex import MassPlan
        if sp.csr_matrix(M).shape[0] != n:
            raise ValueError("K and M sizes differ")
        plan = MassPlan(M, op, np.zeros(n), device=device)
        try:
            return plan.max_gen_eig(start_vector(n, seed), tol=tol, max_iter=max_iter)
        finally:
            plan.close()
    if m.shape[0] != n:
        raise ValueError("K and M sizes differ")
    x0 = start_vector(n, seed)
    lam = _lib.C.c_double(0.0)
    it = _lib.C.c_int64(0)
    code = _lib.load().wcb_max_gen_eig(op.handle, _lib.dptr(m), _lib.dptr(x0), float(tol),
                                       int(max_iter), _lib.C.byref(lam), _lib.C.byref(it))
    if code == _lib.WCB_E_NOCONV:
        raise RuntimeError(_lib.last_error())
    _lib.check(code)
    return float(lam.value), int(it.value)


def max_gen_eig_sub(op, m_diag, sub_idx, tol=1e-9, max_iter=50000, seed=0):
    """``max_gen_eig(K[s][:, s], diag(m)[s])`` on the device without forming
    the sub-matrix: the other DOFs are frozen at zero inside the operator's
    own apply.  The start vector is the reference's for size ``len(s)``."""
    sub = np.ascontiguousarray(sub_idx, dtype=np.int64)
    m = np.ascontiguousarray(m_diag, dtype=np.float64)
    if m.shape[0] != op.n:
        raise ValueError("K and M sizes differ")
    ms = m[sub]
    if np.any(ms <= 0.0) or not np.all(np.isfinite(ms)):
        raise IndefiniteMatrixError("diagonal matrix has non-positive entries; "
                                    "check the stabilization and lumping settings")
    x0 = start_vector(sub.shape[0], seed)
    lam = _lib.C.c_double(0.0)
    it = _lib.C.c_int64(0)
    code = _lib.load().wcb_max_gen_eig_sub(op.handle, _lib.dptr(m), sub.shape[0],
                                           _lib.i64ptr(sub), _lib.dptr(x0), float(tol),
                                           int(max_iter), _lib.C.byref(lam), _lib.C.byref(it))
    if code == _lib.WCB_E_NOCONV:
        raise RuntimeError(_lib.last_error())
    _lib.check(code)
    return float(lam.value), int(it.value)


def dt_crit(K, M, tol=1e-9, seed=0, device: int | None = None) -> float:
    """Critical time step of central differences, ``2 / sqrt(lam_max(K, M))``
    (src/linalg.py:125-130)."""
    lam, _ = max_gen_eig(K, M, tol=tol, seed=seed, device=device)
    if lam <= 0.0:
        raise ValueError("largest generalized eigenvalue must be positive")
    return 2.0 / np.sqrt(lam)


__all__ = ["IndefiniteMatrixError", "is_structurally_diagonal", "diagonal_mass", "mass_split",
           "start_vector", "max_gen_eig", "max_gen_eig_sub", "dt_crit", "DeviceOperator"]
