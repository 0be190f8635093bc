"""Host-side error metrics over device results (the reference's metrics.hpp /
metrics.cpp error part): the analytic LCO propagator, the one-step error
against it, the normalised final error and the per-run error report. They run
on the host over vectors the device returned; sums are taken in index order
(the reference's sequential loops) via cumulative sums."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .solver import SolveResult


def _seq_sum(v: np.ndarray) -> float:
    """Left-to-right sum (cumsum is sequential), the order of a plain loop."""
    return float(np.cumsum(v)[-1]) if v.size else 0.0


def lco_analytic(x0, t: float) -> np.ndarray:
    """systems.cpp:270-306: the agent mean rotates, deviations decay through
    exp(tA) with A = [[-1, 1], [-1, 0]]."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    if x0.size % 2 != 0:
        raise ValueError("lco_analytic: state length must be 2N")
    n = x0.size // 2
    xm0 = _seq_sum(x0[0::2]) / n
    vm0 = _seq_sum(x0[1::2]) / n
    ct, st = math.cos(t), math.sin(t)
    xm = xm0 * ct + vm0 * st
    vm = -xm0 * st + vm0 * ct
    w = math.sqrt(3.0) / 2.0
    decay = math.exp(-0.5 * t)
    cw, sw = math.cos(w * t), math.sin(w * t) / w
    p00, p01 = decay * (cw - 0.5 * sw), decay * sw
    p10, p11 = decay * -sw, decay * (cw + 0.5 * sw)
    du, dv = x0[0::2] - xm0, x0[1::2] - vm0
    out = np.empty_like(x0)
    out[0::2] = (xm + p00 * du) + p01 * dv
    out[1::2] = (vm + p10 * du) + p11 * dv
    return out


def normalized_final_error(x_ref, x, n_agents: int) -> float:
    """metrics.cpp:10-17: ||x_ref - x||_2 / sqrt(N)."""
    a, b = np.asarray(x_ref, dtype=np.float64), np.asarray(x, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("normalized_final_error: length mismatch")
    if n_agents < 1:
        raise ValueError("normalized_final_error: N must be >= 1")
    d = a - b
    return math.sqrt(_seq_sum(d * d)) / math.sqrt(float(n_agents))


def real_local_error(x_n, x_next, h_n: float, ab: float, rel: float) -> float:
    """metrics.cpp:42-52: max_k |x_next,k - x_ex,k| / max(|x_ex,k|, ab/rel),
    x_ex the analytic propagator re-anchored at x_n."""
    x_ex = lco_analytic(x_n, h_n)
    w = np.maximum(np.abs(x_ex), ab / rel)
    return float(np.max(np.abs(np.asarray(x_next) - x_ex) / w)) if x_ex.size else 0.0


@dataclass
class ErrorReport:  # metrics.hpp:31-35
    normalized_final_error: float = 0.0
    mean_e_bs: float = 0.0
    mean_e_analytic: float | None = None


def error_report(run: SolveResult, x_ref_final, n_agents: int, ab: float, rel: float) -> ErrorReport:
    """metrics.cpp:19-40: final error against a reference run, the mean
    estimated local error over accepted steps and, with snapshots, the mean
    analytic local error (linear-oscillator runs)."""
    er = ErrorReport(normalized_final_error(x_ref_final, run.final_state, n_agents))
    acc = np.array([r.err for r in run.step_log if r.accepted], dtype=np.float64)
    er.mean_e_bs = _seq_sum(acc) / acc.size if acc.size else 0.0
    if run.snapshots:
        errs = np.array([real_local_error(s.x_before, s.x_after, s.h, ab, rel) for s in run.snapshots])
        er.mean_e_analytic = _seq_sum(errs) / errs.size
    return er
