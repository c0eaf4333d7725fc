"""B200-native (sm_100a) explicit wave-stepping hot path of arXiv 2501.19013.

Drop-in for the integrator / critical-step API of the reference package
``wavecell`` (src/__init__.py:5-20): ``cdm_run``, ``imex_run``,
``newmark_run``, ``max_gen_eig``, ``dt_crit``, ``imex_critical_time_step``, ``select_dt``,
``RunResult``, ``StageTimings``, ``DivergenceError``.  Every step runs in HBM
through hand-written CUDA kernels in ``libwavecell_b200.so`` (C ABI:
include/wavecell_b200.h); there is no CPU fallback.
"""

from .linalg import IndefiniteMatrixError, dt_crit, max_gen_eig
from .imex import ImexPlan, newmark_run
from .operators import (CsrOperator, DeviceOperator, ElasticOperator, ScmOperator,
                        as_device_operator)
from .timeint import (DIVERGENCE_LIMIT, CdmPlan, DivergenceError, RunResult,
                      StageTimings, cdm_run, imex_critical_time_step, imex_run,
                      sample_history, select_dt)

__version__ = "0.1.0"

__all__ = [
    "CdmPlan", "CsrOperator", "DIVERGENCE_LIMIT", "DeviceOperator", "DivergenceError",
    "ElasticOperator", "ImexPlan", "IndefiniteMatrixError", "RunResult", "ScmOperator",
    "StageTimings",
    "as_device_operator", "cdm_run", "dt_crit", "imex_critical_time_step", "imex_run",
    "max_gen_eig", "newmark_run", "sample_history", "select_dt",
]
