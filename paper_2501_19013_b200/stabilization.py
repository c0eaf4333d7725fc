"""Eigenvalue stabilisation of cut-cell mass matrices on the device: drop-in
for ``wavecell.linalg.jacobi_eig`` (src/linalg.py:133-212) and
``wavecell.stabilization.evs_stabilize`` (src/stabilization.py:73-102)
(SURVEY 8(f)-4).

Both run the reference's algorithm -- row-cyclic Jacobi sweeps with the same
rotation formula and stopping rule, then the scaled projector onto the small
eigenspace -- as one CTA per matrix (``wcb_jacobi_eig`` /
``wcb_evs_stabilize``); batches of cut cells are solved in one launch.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def jacobi_eig(A, max_sweeps: int = 100, tol: float = 1e-12, device: int | None = None):
    """Eigen-decomposition of symmetric matrices (single (n, n) or batch
    (..., n, n)); returns ascending ``lam`` and eigenvector columns ``V``."""
    A = np.asarray(A, dtype=np.float64)
    single = A.ndim == 2
    if single:
        A = A[None]
    batch, n = A.shape[:-2], A.shape[-1]
    flat = np.ascontiguousarray(A.reshape(-1, n, n))
    m = flat.shape[0]
    lam = np.empty((m, n))
    V = np.empty((m, n, n))
    code = _lib.load().wcb_jacobi_eig(_lib.context(device).handle, m, n, _lib.dptr(flat.reshape(-1)),
                                      int(max_sweeps), float(tol), _lib.dptr(lam.reshape(-1)),
                                      _lib.dptr(V.reshape(-1)))
    if code == _lib.WCB_E_NOCONV:
        raise RuntimeError(_lib.last_error())
    _lib.check(code)
    lam = lam.reshape(*batch, n)
    V = V.reshape(*batch, n, n)
    return (lam[0], V[0]) if single else (lam, V)


def evs_stabilize(M_o, M_f, epsilon: float, f_lambda: float = 1e-2, device: int | None = None):
    """``M_o + epsilon * scale * Phi_s Phi_s^T`` with ``Phi_s`` the
    eigenvectors of ``M_o`` below ``f_lambda * lambda_max`` and ``scale`` =
    max|M_f| / max|Phi_s Phi_s^T| (src/stabilization.py:73-102)."""
    M_o = np.asarray(M_o, dtype=np.float64)
    M_f = np.asarray(M_f, dtype=np.float64)
    if epsilon == 0.0:
        return M_o.copy()
    single = M_o.ndim == 2
    Mb = M_o[None] if single else M_o
    Mf = M_f[None] if M_f.ndim == 2 else M_f
    Mf = np.broadcast_to(Mf, Mb.shape)
    n = Mb.shape[-1]
    out = np.ascontiguousarray(Mb.reshape(-1, n, n)).copy()
    num = np.ascontiguousarray(np.max(np.abs(Mf.reshape(-1, n, n)), axis=(1, 2)))
    _lib.check(_lib.load().wcb_evs_stabilize(_lib.context(device).handle, out.shape[0], n,
                                             _lib.dptr(out.reshape(-1)), _lib.dptr(num), float(epsilon),
                                             float(f_lambda)))
    out = out.reshape(Mb.shape)
    return out[0] if single else out


__all__ = ["jacobi_eig", "evs_stabilize"]
