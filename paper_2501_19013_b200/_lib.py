"""ctypes binding of ``libwavecell_b200.so`` (the C ABI in include/wavecell_b200.h).

This is the only module that touches the native library.  There is no CPU
fallback: if the shared object is missing, or no B200 is visible, the calls
raise instead of silently computing something else.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_NAME = "libwavecell_b200.so"
LIB_PATH = Path(__file__).resolve().parent / os.environ.get("WAVECELL_B200_LIB", LIB_NAME)

WCB_OK = 0
WCB_E_ARG = 1
WCB_E_CUDA = 2
WCB_E_DIVERGED = 3
WCB_E_NOCONV = 4
WCB_E_UNSUPPORTED = 5

# Every entry point declared in include/wavecell_b200.h (checked by tests).
EXPORTS = (
    "wcb_abi_version", "wcb_last_error", "wcb_device_count",
    "wcb_context_create", "wcb_context_destroy", "wcb_context_stream",
    "wcb_context_launches", "wcb_operator_csr_create", "wcb_operator_scm_create",
    "wcb_operator_elastic_create",
    "wcb_operator_destroy", "wcb_operator_n", "wcb_operator_apply", "wcb_operator_halo",
    "wcb_max_gen_eig", "wcb_max_gen_eig_sub", "wcb_cdm_plan_create", "wcb_cdm_plan_destroy",
    "wcb_cdm_plan_run", "wcb_cdm_plan_run_device", "wcb_imex_plan_create",
    "wcb_imex_plan_destroy", "wcb_imex_plan_run", "wcb_dist_unique_id", "wcb_dist_init",
    "wcb_dist_finalize", "wcb_cdm_group_run", "wcb_cdm_plan_step_bytes", "wcb_imex_group_run",
    "wcb_csr_diagonal_check", "wcb_mass_plan_create", "wcb_imex_plan_cdm_run",
    "wcb_imex_plan_max_gen_eig", "wcb_operator_step_kernel", "wcb_setup_ball_classify",
    "wcb_setup_ball_cut_cells", "wcb_setup_ball_slivers", "wcb_jacobi_eig", "wcb_evs_stabilize",
    "wcb_cdm_plan_run_sampled", "wcb_setup_dofmap", "wcb_setup_lumped_mass",
)

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)


class Timings(C.Structure):
    _fields_ = [("factorization", _d), ("rhs", _d), ("backward_insertion", _d)]


class Divergence(C.Structure):
    _fields_ = [("step", _i64), ("amplitude", _d)]


class Observer(C.Structure):
    _fields_ = [("n_obs", _i64), ("indptr", _i64p), ("indices", _i64p), ("data", _dp)]


class ScmDesc(C.Structure):
    _fields_ = [("dim", _i32), ("p", _i32), ("n_e", _i64 * 3), ("k1", _dp), ("m1", _dp),
                ("sk", _d), ("cell_class", _i8p), ("n_dof", _i64),
                ("lex_of_compact", _i64p), ("n_cut", _i64), ("cut_cells", _i64p),
                ("cut_K", _dp), ("x_cell_lo", _i64), ("x_cell_hi", _i64),
                ("x_owns_last", _i32)]


class ElasticDesc(C.Structure):
    _fields_ = [("p", _i32), ("n_e", _i64 * 2), ("lam", _d), ("mu", _d), ("m1", _dp),
                ("k1", _dp), ("g1", _dp), ("cell_class", _i8p), ("n_node", _i64),
                ("lex_of_compact", _i64p), ("n_cut", _i64), ("cut_cells", _i64p),
                ("cut_K", _dp), ("x_cell_lo", _i64), ("x_cell_hi", _i64),
                ("x_owns_last", _i32)]


class LU(C.Structure):
    _fields_ = [("n", _i64), ("perm_r", _i64p), ("perm_c", _i64p),
                ("L_indptr", _i64p), ("L_indices", _i32p), ("L_data", _dp),
                ("U_indptr", _i64p), ("U_indices", _i32p), ("U_data", _dp)]


_SIGS = {
    "wcb_abi_version": (C.c_int, []),
    "wcb_last_error": (C.c_char_p, []),
    "wcb_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "wcb_context_create": (C.c_int, [C.c_int, C.POINTER(_p)]),
    "wcb_context_destroy": (C.c_int, [_p]),
    "wcb_context_stream": (_p, [_p]),
    "wcb_context_launches": (_i64, [_p]),
    "wcb_operator_csr_create": (C.c_int, [_p, _i64, _i64p, _i32p, _dp, C.POINTER(_p)]),
    "wcb_operator_scm_create": (C.c_int, [_p, C.POINTER(ScmDesc), C.POINTER(_p)]),
    "wcb_operator_elastic_create": (C.c_int, [_p, C.POINTER(ElasticDesc), C.POINTER(_p)]),
    "wcb_operator_destroy": (C.c_int, [_p]),
    "wcb_operator_n": (_i64, [_p]),
    "wcb_operator_apply": (C.c_int, [_p, _dp, _dp]),
    "wcb_operator_halo": (C.c_int, [_p, _i64p]),
    "wcb_operator_step_kernel": (C.c_int, [_p, C.c_char_p, _i64]),
    "wcb_setup_ball_classify": (C.c_int, [C.c_int, _i64, _i64, _dp, _dp, _i8p]),
    "wcb_setup_dofmap": (_i64, [C.c_int, C.c_int, _i64, _i8p, _i64p, _i64p, _i64p, _i64p, _i64p]),
    "wcb_setup_lumped_mass": (C.c_int, [C.c_int, C.c_int, _i64, _i8p, _dp, _d, _i64, _i64p, _i64, _i64p, _dp,
                                        _i64p, _dp]),
    "wcb_jacobi_eig": (C.c_int, [_p, _i64, C.c_int, _dp, C.c_int, _d, _dp, _dp]),
    "wcb_evs_stabilize": (C.c_int, [_p, _i64, C.c_int, _dp, _dp, _d, _d]),
    "wcb_setup_ball_slivers": (C.c_int, [C.c_int, _i64, _i64, _dp, _dp, _i64, _i64p, _d, C.c_int,
                                         C.POINTER(C.c_uint8)]),
    "wcb_setup_ball_cut_cells": (C.c_int, [C.c_int, C.c_int, _i64, _i64, _dp, _dp, C.c_int, C.c_int, _i64p,
                                           _dp, _dp, _dp, _dp, _dp, _dp, _i64, _i64p, _d, _d, _d, C.c_int,
                                           C.c_int, _dp, _dp]),
    "wcb_max_gen_eig": (C.c_int, [_p, _dp, _dp, _d, _i64, _dp, _i64p]),
    "wcb_max_gen_eig_sub": (C.c_int, [_p, _dp, _i64, _i64p, _dp, _d, _i64, _dp, _i64p]),
    "wcb_cdm_plan_create": (C.c_int, [_p, _dp, _dp, C.POINTER(Observer), C.POINTER(_p)]),
    "wcb_cdm_plan_destroy": (C.c_int, [_p]),
    "wcb_csr_diagonal_check": (C.c_int, [_i64, _p, _p, C.c_int, _dp]),
    "wcb_cdm_plan_step_bytes": (C.c_int, [_p, _dp]),
    "wcb_cdm_plan_run": (C.c_int, [_p, _dp, _d, _i64, _dp, _dp, _dp, _dp,
                                   C.POINTER(Divergence), C.POINTER(Timings)]),
    "wcb_cdm_plan_run_sampled": (C.c_int, [_p, _dp, _d, _i64, _i64, _dp, _dp, _dp, _dp,
                                           C.POINTER(Divergence), C.POINTER(Timings)]),
    "wcb_cdm_plan_run_device": (C.c_int, [_p, _p, _d, _i64, _p, _p, _p, _p,
                                          C.POINTER(Divergence), C.POINTER(Timings)]),
    "wcb_imex_plan_create": (C.c_int, [_p, _i64, _i64p, _i64, _i64p, _dp, C.POINTER(LU),
                                       C.POINTER(LU), _dp, C.POINTER(Observer),
                                       C.POINTER(_p)]),
    "wcb_imex_plan_destroy": (C.c_int, [_p]),
    "wcb_mass_plan_create": (C.c_int, [_p, _i64, _i64p, _i64, _i64p, _dp, C.POINTER(LU), _i64p, _i32p,
                                       _dp, _dp, C.POINTER(Observer), C.POINTER(_p)]),
    "wcb_imex_plan_cdm_run": (C.c_int, [_p, _dp, _d, _i64, _dp, _dp, _dp, _dp,
                                        C.POINTER(Divergence), C.POINTER(Timings)]),
    "wcb_imex_plan_max_gen_eig": (C.c_int, [_p, _dp, _d, _i64, _dp, _i64p]),
    "wcb_dist_unique_id": (C.c_int, [C.c_char_p]),
    "wcb_dist_init": (C.c_int, [_p, C.c_int, C.c_int, C.c_char_p]),
    "wcb_dist_finalize": (C.c_int, [_p]),
    "wcb_cdm_group_run": (C.c_int, [C.c_int, C.POINTER(_p), _dp, _d, _i64, C.POINTER(_dp), _dp,
                                    C.POINTER(Divergence), C.POINTER(Timings)]),
    "wcb_imex_plan_run": (C.c_int, [_p, _d, _dp, _dp, _d, _i64, _d, _d, _dp, _dp, _dp,
                                    _dp, _dp, C.POINTER(Divergence), C.POINTER(Timings)]),
    "wcb_imex_group_run": (C.c_int, [C.c_int, C.POINTER(_p), _d, _dp, _dp, _d, _i64, _d, _d,
                                     C.POINTER(_dp), C.POINTER(_dp), C.POINTER(_dp),
                                     C.POINTER(Divergence), C.POINTER(Timings)]),
}

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    """A call into libwavecell_b200 failed."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def load() -> C.CDLL:
    """Load the shared library (build it with ``__graft_entry__.build()``)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: the CUDA extension has not been built "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                    "there is no CPU fallback")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return load().wcb_last_error().decode(errors="replace")


def check(code: int):
    if code != WCB_OK:
        msg = last_error()
        if code == WCB_E_ARG:
            raise ValueError(msg)
        if code == WCB_E_UNSUPPORTED:
            raise NotImplementedError(msg)
        raise NativeError(code, msg)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def i32ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_i32p)


def i8ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int8 and a.flags.c_contiguous
    return a.ctypes.data_as(_i8p)


class Context:
    """One CUDA device + stream owned by the native library."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _p()
        check(lib.wcb_context_create(int(device), C.byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return int(load().wcb_context_stream(self._h) or 0)

    @property
    def launches(self) -> int:
        return int(load().wcb_context_launches(self._h))

    def close(self):
        if getattr(self, "_h", None):
            load().wcb_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def default_device() -> int:
    env = os.environ.get("WAVECELL_B200_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0")) if "LOCAL_RANK" in os.environ else 0


def context(device: int | None = None) -> Context:
    """Process-wide context for ``device`` (created on first use)."""
    dev = default_device() if device is None else int(device)
    with _lock:
        ctx = _contexts.get(dev)
    if ctx is None:
        ctx = Context(dev)
        with _lock:
            _contexts[dev] = ctx
    return ctx


def device_count() -> int:
    n = C.c_int(0)
    check(load().wcb_device_count(C.byref(n)))
    return int(n.value)
