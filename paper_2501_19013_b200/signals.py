"""Observer signals and the accuracy metric of the reference's studies
(src/harness.py:96-141, writers :488-511), for runs made on the device.

``sample_observers`` takes the exact step hits of a recorded history when
the step count is a multiple of the sample count (else linear interpolation,
as the reference); a run made with ``CdmPlan.run(record_every=s)`` records
only those columns on the device, so long runs do not move the full history
back.  ``relative_error`` is the mean over observers of the relative L2
signal error (the e_ts / e_ss metric).
"""

from __future__ import annotations

import csv

import numpy as np

STUDY_COLUMNS = ("method", "p", "n_e", "n_dof", "dt_crit", "dt", "error",
                 "t_fact", "t_rhs", "t_binsert")


def sample_times(T: float, n_s: int) -> np.ndarray:
    """n_s equidistant sampling times j T / n_s, j = 1..n_s (src/harness.py:101-103)."""
    return np.arange(1, n_s + 1) * (T / n_s)


def sample_observers(result, n_s: int, T: float | None = None) -> np.ndarray:
    """Observer signals at n_s equidistant times (src/harness.py:106-131)."""
    if result.obs is None:
        raise ValueError("run was made without an observer matrix")
    n_t = result.t.shape[0] - 1
    T_run = float(result.t[-1])
    if T is None:
        T = T_run
    exact = (n_t % n_s == 0 if n_t >= n_s else False)
    if exact and abs(T - T_run) <= 1e-12 * max(T_run, 1.0):
        stride = n_t // n_s
        return result.obs[:, stride::stride].copy()
    times = sample_times(T, n_s)
    if times[-1] > T_run * (1.0 + 1e-12):
        raise ValueError("sampling window extends past the end of the run")
    out = np.empty((result.obs.shape[0], n_s))
    for i in range(result.obs.shape[0]):
        out[i] = np.interp(times, result.t, result.obs[i])
    return out


def relative_error(sig, ref) -> float:
    """Mean over observers of ||sig_i - ref_i||_2 / ||ref_i||_2 (src/harness.py:134-141)."""
    sig = np.asarray(sig, dtype=float)
    ref = np.asarray(ref, dtype=float)
    if sig.shape != ref.shape:
        raise ValueError("signal matrices must have the same shape")
    norms = np.linalg.norm(ref, axis=1)
    if np.any(norms == 0.0):
        raise ValueError("reference signal with zero norm")
    return float(np.mean(np.linalg.norm(sig - ref, axis=1) / norms))


def write_signals_csv(path, times, samples):
    """Header t, psi_1..psi_k; one row per sampling time (src/harness.py:488-496)."""
    samples = np.asarray(samples)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["t"] + [f"psi_{i + 1}" for i in range(samples.shape[0])])
        for j, t in enumerate(np.asarray(times)):
            w.writerow([repr(float(t))] + [repr(float(v)) for v in samples[:, j]])


def write_study_csv(path, reports):
    """Study table, one row per report (src/harness.py:499-511); reports are
    objects or dicts with the STUDY_COLUMNS fields."""
    def get(r, k):
        return r[k] if isinstance(r, dict) else getattr(r, k)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(STUDY_COLUMNS)
        for r in reports:
            dtc, err = get(r, "dt_crit"), get(r, "error")
            w.writerow([get(r, "method"), get(r, "p"), get(r, "n_e"), get(r, "n_dof"),
                        "" if dtc is None else repr(float(dtc)), repr(float(get(r, "dt"))),
                        "" if err is None else repr(float(err)), repr(float(get(r, "t_fact"))),
                        repr(float(get(r, "t_rhs"))), repr(float(get(r, "t_binsert")))])


__all__ = ["STUDY_COLUMNS", "sample_times", "sample_observers", "relative_error", "write_signals_csv",
           "write_study_csv"]
