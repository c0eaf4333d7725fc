"""ctypes wrapper of oracle/_build/libwc_oracle.so (TEST INFRASTRUCTURE /
CPU BASELINE ONLY).  Builds the reference-style CSR of a spectral-cell system
and runs the reference CDM loop on the host cores."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np
import scipy.sparse as sp

LIB = Path(__file__).resolve().parent / "_build" / "libwc_oracle.so"
_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise ImportError(f"{LIB} missing; run `make -C oracle`")
        lib = C.CDLL(str(LIB))
        P = C.c_void_p
        lib.wco_scm_csr.restype = C.c_int64
        lib.wco_scm_csr.argtypes = [C.c_int, C.c_int, C.c_int64, P, P, C.c_double, P, P, P,
                                    C.c_int64, P, P, P, P, P]
        lib.wco_cdm_run.restype = C.c_int64
        lib.wco_cdm_run.argtypes = [C.c_int64, P, P, P, P, P, P, C.c_double, C.c_int64, P, P,
                                    P, C.c_int]
        lib.wco_cdm_run_obs.restype = C.c_int64
        lib.wco_cdm_run_obs.argtypes = [C.c_int64, P, P, P, P, P, P, C.c_double, C.c_int64, P, P,
                                        P, C.c_int, C.c_int64, P, P, P, P]
        lib.wco_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def scm_csr(prob) -> sp.csr_matrix:
    """CSR stiffness of an ``ScmProblem`` (reference assembly semantics)."""
    lib = load()
    g = prob.grid
    d, p, n_e = g.dim, g.p, g.n_e
    cls = np.ascontiguousarray(g.classes.ravel(), dtype=np.int8)
    compact = np.ascontiguousarray(g.dofmap.compact_of_lex, dtype=np.int64)
    lex = np.ascontiguousarray(g.dofmap.lex_of_compact, dtype=np.int64)
    cut_index = np.full(cls.shape[0], -1, dtype=np.int64)
    cut_index[g.cut_lex] = np.arange(g.cut_lex.shape[0])
    cutK = np.ascontiguousarray(prob.cut_K, dtype=np.float64)
    k1 = np.ascontiguousarray(prob.k1)
    m1 = np.ascontiguousarray(prob.m1)
    n = lex.shape[0]
    indptr = np.zeros(n + 1, dtype=np.int64)
    lib.wco_scm_csr(d, p, n_e, _p(k1), _p(m1), prob.sk, _p(cls), _p(compact), _p(lex), n,
                    _p(cut_index), _p(cutK), _p(indptr), None, None)
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int64)
    data = np.empty(nnz)
    lib.wco_scm_csr(d, p, n_e, _p(k1), _p(m1), prob.sk, _p(cls), _p(compact), _p(lex), n,
                    _p(cut_index), _p(cutK), _p(indptr), _p(indices), _p(data))
    return sp.csr_matrix((data, indices, indptr), shape=(n, n))


def cdm_run(K, m, F, ft, dt, n_t, psi0=None, v0=None, threads=0, obs_mat=None):
    """Reference CDM loop (src/timeint.py:159-193) on the host.
    Returns (psi, diverged_step), or (psi, obs, diverged_step) with obs_mat."""
    lib = load()
    K = sp.csr_matrix(K)
    indptr = np.ascontiguousarray(K.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(K.indices, dtype=np.int64)
    data = np.ascontiguousarray(K.data, dtype=np.float64)
    m = np.ascontiguousarray(m, dtype=np.float64)
    F = np.ascontiguousarray(F, dtype=np.float64)
    ft = np.ascontiguousarray(ft, dtype=np.float64)
    n = K.shape[0]
    out = np.empty(n)
    p0 = None if psi0 is None else np.ascontiguousarray(psi0, dtype=np.float64)
    q0 = None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
    if obs_mat is not None:
        A = sp.csr_matrix(obs_mat)
        op_ = np.ascontiguousarray(A.indptr, dtype=np.int64)
        oi = np.ascontiguousarray(A.indices, dtype=np.int64)
        ov = np.ascontiguousarray(A.data, dtype=np.float64)
        obs = np.zeros((A.shape[0], int(n_t) + 1))
        div = lib.wco_cdm_run_obs(n, _p(indptr), _p(indices), _p(data), _p(m), _p(F), _p(ft), float(dt),
                                  int(n_t), _p(p0), _p(q0), _p(out), int(threads), A.shape[0], _p(op_),
                                  _p(oi), _p(ov), _p(obs))
        return out, obs, int(div)
    div = lib.wco_cdm_run(n, _p(indptr), _p(indices), _p(data), _p(m), _p(F), _p(ft), float(dt),
                          int(n_t), _p(p0), _p(q0), _p(out), int(threads))
    return out, int(div)


def max_threads() -> int:
    return int(load().wco_max_threads())


def host_cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    return os.cpu_count() or 1
