"""BS3(2) solver API on the B200 — mirror of proj/include/mixedstep/solver.hpp
(SolverConfig :39-61, SolveStatus :63-71, StepOutcome :75-86, StepRecord :88-93,
FlopTally :104-113, SolveResult :115-126, and the entry points :128-163).

Config errors raise ``ValueError`` where the reference throws
``std::invalid_argument`` (solver.cpp:217-224); numerical failure is reported
in ``SolveResult.status`` and never raised (solver.hpp:151-153).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field, fields

import numpy as np

from . import _abi
from .precision import PrecisionPolicy
from .systems import DeviceSystem

kSchemeFlopsBs32 = 30  # solver.hpp:37


class SolveStatus(enum.IntEnum):  # solver.hpp:63-71
    Completed = _abi.MS_COMPLETED
    MaxIterations = _abi.MS_MAX_ITERATIONS
    MaxFailedSteps = _abi.MS_MAX_FAILED_STEPS
    WallClock = _abi.MS_WALL_CLOCK
    SlowSolver = _abi.MS_SLOW_SOLVER
    StepTooSmall = _abi.MS_STEP_TOO_SMALL
    NonFinite = _abi.MS_NON_FINITE


def status_name(s: SolveStatus) -> str:
    return SolveStatus(s).name


@dataclass
class SolverConfig:  # solver.hpp:39-61
    rel_tol: float = 1e-6
    abs_tol: float = 1e-8
    h_min_factor: float = 100.0
    max_iterations: int = 100000
    max_failed_steps: int = 85000
    time_limits_enabled: bool = True
    wall_clock_limit: float = 5400.0
    slow_solver_elapsed: float = 2700.0
    slow_solver_progress: float = 0.10
    safety: float = 0.9
    fac_min: float = 0.2
    fac_max: float = 5.0
    controller_exponent: float = 1.0 / 3.0
    record_step_log: bool = True
    record_snapshots: bool = False

    def c(self) -> _abi.SolverConfigC:
        c = _abi.SolverConfigC()
        for f in fields(self):
            v = getattr(self, f.name)
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


@dataclass
class StepRecord:  # solver.hpp:88-93
    t: float
    h: float
    err: float
    accepted: bool


@dataclass
class StepSnapshot:  # solver.hpp:96-100: the state pair of one accepted step
    x_before: np.ndarray
    x_after: np.ndarray
    h: float


@dataclass
class FlopTally:  # solver.hpp:104-113
    low: int = 0
    high: int = 0
    rhs_evals: int = 0

    def low_fraction(self) -> float:
        tot = float(self.low) + float(self.high)
        return float(self.low) / tot if tot > 0 else 0.0


@dataclass
class SolveResult:  # solver.hpp:115-126
    status: SolveStatus
    final_state: np.ndarray
    t_reached: float
    n_accepted: int
    n_failed: int
    step_log: list
    flops: FlopTally
    device_ms: float = 0.0
    step_log_count: int = 0
    snapshots: list = field(default_factory=list)
    snapshot_count: int = 0
    y_eval: np.ndarray | None = None  # dense output rows (D6 extension), one per t_eval

    def total_steps(self) -> int:
        return self.n_accepted + self.n_failed


@dataclass
class StepOutcome:  # solver.hpp:75-86
    x_next: np.ndarray
    x_tilde: np.ndarray
    err: float
    accepted: bool
    k4: np.ndarray
    x_store: np.ndarray
    h_used: float
    h_next: float
    flops: FlopTally = field(default_factory=FlopTally)


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def estimate_error(x_n, x_next, x_tilde, ab: float, rel: float) -> float:
    """solver.cpp:399-411 (device reduction)."""
    a, b, c = _f64(x_n), _f64(x_next), _f64(x_tilde)
    if not (a.shape == b.shape == c.shape):
        raise ValueError("estimate_error: length mismatch")
    out = C.c_double()
    _abi.check(_abi.lib().ms_estimate_error(a.size, _abi.dptr(a), _abi.dptr(b), _abi.dptr(c), ab, rel,
                                            C.byref(out)), "ms_estimate_error")
    return out.value


def adjust_step(h: float, err: float, rel_tol: float, cfg: SolverConfig) -> float:
    """solver.cpp:413-418 (device arithmetic)."""
    out = C.c_double()
    cc = cfg.c()
    _abi.check(_abi.lib().ms_adjust_step(h, err, rel_tol, C.byref(cc), C.byref(out)), "ms_adjust_step")
    return out.value


def initial_step(sys: DeviceSystem, t0: float, t_final: float, x0, cfg: SolverConfig, order: int = 3,
                 tally: FlopTally | None = None) -> float:
    """solver.cpp:420-451: two binary64 evaluations on the device."""
    x0 = _f64(x0)
    h0 = C.c_double()
    ev = C.c_int64()
    cc = cfg.c()
    _abi.check(_abi.lib().ms_initial_step(sys.handle, t0, t_final, _abi.dptr(x0), C.byref(cc), order,
                                          C.byref(h0), C.byref(ev)), "ms_initial_step")
    if tally is not None:
        tally.rhs_evals += ev.value
    return h0.value


def bs32_step(sys: DeviceSystem, t: float, x_n, h: float, k1, policy: PrecisionPolicy,
              cfg: SolverConfig) -> StepOutcome:
    """One BS3(2) attempt with supplied k1 (solver.cpp:453-460)."""
    x_n, k1 = _f64(x_n), _f64(k1)
    n = x_n.size
    bufs = [np.empty(n) for _ in range(4)]
    o = _abi.StepOutcomeC()
    o.x_next, o.x_tilde, o.k4, o.x_store = (_abi.dptr(b) for b in bufs)
    pol, cc = policy.c(), cfg.c()
    _abi.check(_abi.lib().ms_bs32_step(sys.handle, t, _abi.dptr(x_n), h, _abi.dptr(k1), C.byref(pol),
                                       C.byref(cc), C.byref(o)), "ms_bs32_step")
    return StepOutcome(bufs[0], bufs[1], o.err, bool(o.accepted), bufs[2], bufs[3], o.h_used, o.h_next,
                       FlopTally(o.flops_low, o.flops_high, o.rhs_evals))


def _result(r: _abi.SolveResultC, final: np.ndarray, log: np.ndarray | None, snaps=None) -> SolveResult:
    steps = []
    if log is not None:
        m = min(len(log), r.step_log_count)
        steps = [StepRecord(float(e.t), float(e.h), float(e.err), bool(e.accepted)) for e in log[:m]]
    shots = []
    if snaps is not None:
        rows, hs = snaps
        m = min(len(hs), r.snapshot_count)
        shots = [StepSnapshot(rows[k], rows[k + 1], float(hs[k])) for k in range(m)]
    return SolveResult(SolveStatus(r.status), final, r.t_reached, r.n_accepted, r.n_failed, steps,
                       FlopTally(r.flops_low, r.flops_high, r.rhs_evals), r.device_ms, r.step_log_count,
                       shots, r.snapshot_count if snaps is not None else 0)


def _snapshot_buffers(cfg: SolverConfig, dn: int, capacity: int | None):
    """Host rows for StepSnapshots: by default as many accepted steps as fit
    in 256 MiB (the count reported says whether the run had more)."""
    if not cfg.record_snapshots:
        return None
    if capacity is None:
        capacity = min(cfg.max_iterations, max(1, (256 << 20) // (8 * max(dn, 1)) - 1))
    cap = max(int(capacity), 1)
    return np.empty((cap + 1, dn)), np.empty(cap)


def _log_buffer(cfg: SolverConfig, capacity: int | None):
    if not cfg.record_step_log:
        return None, None
    cap = int(capacity if capacity is not None else min(cfg.max_iterations, 1 << 20))
    arr = (_abi.StepRecordC * max(cap, 1))()
    return arr, cap


def solve(sys: DeviceSystem, x0, t0: float, t_final: float, policy: PrecisionPolicy, cfg: SolverConfig,
          log_capacity: int | None = None, snapshot_capacity: int | None = None, t_eval=None) -> SolveResult:
    """Adaptive BS3(2) solve (solver.cpp:462-470); the step loop runs on the device.
    With ``cfg.record_snapshots`` the device copies the state after every
    accepted step (solver.cpp:324-327) into ``result.snapshots``. ``t_eval``
    (sorted, within [t0, t_final]) asks for dense output: the cubic Hermite
    interpolant of the accepted steps at those times, ``result.y_eval``
    (rows beyond a premature stop are NaN)."""
    x0 = _f64(x0)
    final = np.empty_like(x0)
    log, cap = _log_buffer(cfg, log_capacity)
    snaps = _snapshot_buffers(cfg, x0.size, snapshot_capacity)
    te = ye = None
    if t_eval is not None:
        te = _f64(t_eval).ravel()
        ye = np.full((te.size, x0.size), np.nan)
    r = _abi.SolveResultC()
    if te is not None and te.size:
        r.t_eval, r.n_eval, r.y_eval = _abi.dptr(te), te.size, _abi.dptr(ye)
    r.final_state = _abi.dptr(final)
    if log is not None:
        r.step_log = C.cast(log, C.POINTER(_abi.StepRecordC))
        r.step_log_capacity = cap
    if snaps is not None:
        r.snapshots, r.snapshot_h = _abi.dptr(snaps[0]), _abi.dptr(snaps[1])
        r.snapshot_capacity = len(snaps[1])
    pol, cc = policy.c(), cfg.c()
    _abi.check(_abi.lib().ms_solve(sys.handle, _abi.dptr(x0), t0, t_final, C.byref(pol), C.byref(cc),
                                   C.byref(r)), "ms_solve")
    out = _result(r, final, log, snaps)
    out.y_eval = ye
    return out


class DeviceVariants:
    """Concurrent solves of one system under up to four policies (the
    harness's variant set, harness.cpp:113-121) in lock-step on the device:
    each stage of all variants is one K sweep when the model allows it, and
    each variant's result is bit-identical to its own ``solve``."""

    def __init__(self, sys: DeviceSystem, count: int):
        self.sys, self.count = sys, int(count)
        h = C.c_void_p()
        _abi.check(_abi.lib().ms_variants_create(sys.handle, self.count, C.byref(h)), "ms_variants_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None:
            _abi.lib().ms_variants_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, x0, t0: float, t_final: float, policies, cfg: SolverConfig,
              log_capacity: int | None = None) -> list:
        if len(policies) != self.count:
            raise ValueError(f"expected {self.count} policies")
        x0 = _f64(x0)
        finals = [np.empty_like(x0) for _ in policies]
        logs = [_log_buffer(cfg, log_capacity) for _ in policies]
        res = (_abi.SolveResultC * self.count)()
        for r, fin, (log, cap) in zip(res, finals, logs):
            r.final_state = _abi.dptr(fin)
            if log is not None:
                r.step_log = C.cast(log, C.POINTER(_abi.StepRecordC))
                r.step_log_capacity = cap
        pols = (_abi.Policy * self.count)(*[p.c() for p in policies])
        cc = cfg.c()
        _abi.check(_abi.lib().ms_variants_solve(self._h, _abi.dptr(x0), t0, t_final, pols, C.byref(cc), res),
                   "ms_variants_solve")
        return [_result(r, fin, log) for r, fin, (log, _) in zip(res, finals, logs)]


def solve_variants(sys: DeviceSystem, x0, t0: float, t_final: float, policies, cfg: SolverConfig,
                   log_capacity: int | None = None) -> list:
    """One-shot DeviceVariants.solve."""
    v = DeviceVariants(sys, len(policies))
    try:
        return v.solve(x0, t0, t_final, policies, cfg, log_capacity)
    finally:
        v.close()


def solve_device(sys: DeviceSystem, x0_dev_ptr: int, final_dev_ptr: int, t0: float, t_final: float,
                 policy: PrecisionPolicy, cfg: SolverConfig, stream: int = 0,
                 log_capacity: int | None = 0) -> SolveResult:
    """solve() on device-resident buffers (raw CUDA pointers, e.g. torch
    ``tensor.data_ptr()``); ``stream`` is a cudaStream_t handle or 0."""
    log, cap = _log_buffer(cfg, log_capacity) if log_capacity else (None, None)
    r = _abi.SolveResultC()
    r.final_state = C.cast(C.c_void_p(final_dev_ptr), _abi._DP)
    if log is not None:
        r.step_log = C.cast(log, C.POINTER(_abi.StepRecordC))
        r.step_log_capacity = cap
    pol, cc = policy.c(), cfg.c()
    _abi.check(_abi.lib().ms_solve_device(sys.handle, C.c_void_p(x0_dev_ptr), t0, t_final, C.byref(pol),
                                          C.byref(cc), C.byref(r), C.c_void_p(stream)), "ms_solve_device")
    return _result(r, np.empty(0), log)


def dp54_reference(sys: DeviceSystem, x0, t0: float, t_final: float, cfg: SolverConfig | None = None,
                   log_capacity: int | None = None) -> SolveResult:
    """All-binary64 DP5(4) at rel = abs = 1e-9 (solver.cpp:472-483), on the device."""
    cfg = cfg or SolverConfig()
    x0 = _f64(x0)
    final = np.empty_like(x0)
    log, cap = _log_buffer(cfg, log_capacity)
    r = _abi.SolveResultC()
    r.final_state = _abi.dptr(final)
    if log is not None:
        r.step_log = C.cast(log, C.POINTER(_abi.StepRecordC))
        r.step_log_capacity = cap
    cc = cfg.c()
    _abi.check(_abi.lib().ms_dp54_reference(sys.handle, _abi.dptr(x0), t0, t_final, C.byref(cc), C.byref(r)),
               "ms_dp54_reference")
    return _result(r, final, log)
