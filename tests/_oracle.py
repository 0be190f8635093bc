"""ctypes binding of the CPU oracle ``oracle/liborc.so`` (TEST INFRASTRUCTURE).

The oracle is the checker of the device path; only tests/, smoke() and
bench.py's CPU legs load it. It shares the struct layouts of the product ABI.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200.precision import PrecisionPolicy, StagePrecision
from paper_2605_23727_b200.solver import (FlopTally, SolveResult, SolverConfig, SolveStatus, StepOutcome, StepRecord,
                                          StepSnapshot)
from paper_2605_23727_b200.systems import SystemSpec

ROOT = Path(__file__).resolve().parent.parent
ORC_PATH = ROOT / "oracle" / "liborc.so"
_DP = C.POINTER(C.c_double)
_VP = C.c_void_p

_SIGS = [
    ("orc_last_error", C.c_char_p, []),
    ("orc_set_threads", None, [C.c_int]),
    ("orc_get_threads", C.c_int, []),
    ("orc_round_to", C.c_double, [C.c_double, C.c_int]),
    ("orc_machine_epsilon", C.c_double, [C.c_int]),
    ("orc_round_k", C.c_double, [C.c_double, C.c_int]),
    ("orc_policy_for", C.c_int, [C.c_int, C.POINTER(_abi.Policy)]),
    ("orc_policy_lowest_format", C.c_int, [C.POINTER(_abi.Policy)]),
    ("orc_rng_next", C.c_uint64, [C.c_uint64, C.c_uint64, C.c_int64]),
    ("orc_rng_uniform", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_double, _DP]),
    ("orc_rng_normal", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, _DP]),
    ("orc_system_create", C.c_int, [C.POINTER(_abi.SystemDesc), C.POINTER(_VP)]),
    ("orc_system_destroy", C.c_int, [_VP]),
    ("orc_system_fill_k_uniform", C.c_int, [_VP, C.c_uint64, C.c_uint64, C.c_double, C.c_double]),
    ("orc_system_get_k", C.c_int, [_VP, _DP]),
    ("orc_system_set_op_round", C.c_int, [_VP, C.c_int]),
    ("orc_system_set_omega", C.c_int, [_VP, _DP]),
    ("orc_make_lco", C.c_int, [C.c_int, C.c_uint64, C.POINTER(_VP)]),
    ("orc_make_kuramoto", C.c_int, [C.c_int, C.c_double, C.c_double, C.c_uint64, C.POINTER(_VP)]),
    ("orc_make_cc", C.c_int, [C.c_int, C.c_double, C.c_double, C.c_uint64, C.POINTER(_VP)]),
    ("orc_system_get_param", C.c_int, [_VP, C.c_int, _DP]),
    ("orc_system_dim", C.c_int, [_VP]),
    ("orc_system_agents", C.c_int, [_VP]),
    ("orc_system_flop_profile", C.c_int, [_VP, C.POINTER(C.c_int64)]),
    ("orc_eval_rhs", C.c_int, [_VP, C.c_double, _DP, _abi.StagePrec, _DP]),
    ("orc_estimate_error", C.c_int, [C.c_int64, _DP, _DP, _DP, C.c_double, C.c_double, _DP]),
    ("orc_adjust_step", C.c_int, [C.c_double, C.c_double, C.c_double, C.POINTER(_abi.SolverConfigC), _DP]),
    ("orc_initial_step", C.c_int, [_VP, C.c_double, C.c_double, _DP, C.POINTER(_abi.SolverConfigC), C.c_int, _DP,
                                   C.POINTER(C.c_int64)]),
    ("orc_bs32_step", C.c_int, [_VP, C.c_double, _DP, C.c_double, _DP, C.POINTER(_abi.Policy),
                                C.POINTER(_abi.SolverConfigC), C.POINTER(_abi.StepOutcomeC)]),
    ("orc_solve", C.c_int, [_VP, _DP, C.c_double, C.c_double, C.POINTER(_abi.Policy),
                            C.POINTER(_abi.SolverConfigC), C.POINTER(_abi.SolveResultC)]),
    ("orc_dp54_reference", C.c_int, [_VP, _DP, C.c_double, C.c_double, C.POINTER(_abi.SolverConfigC),
                                     C.POINTER(_abi.SolveResultC)]),
    ("orc_lco_analytic", C.c_int, [C.c_int64, _DP, C.c_double, _DP]),
    ("orc_scheme_flops_bs32", C.c_int, []),
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORC_PATH.exists():
            from paper_2605_23727_b200.build import build_oracle
            build_oracle()
        L = C.CDLL(str(ORC_PATH))
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = (lib().orc_last_error() or b"").decode()
    if rc == 1:
        raise ValueError(f"{what}: {msg}")
    raise OracleError(f"{what}: {msg}")


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


class OracleSystem:
    """The CPU restatement of CoupledSystem for a SystemSpec (same inputs as the device)."""

    def __init__(self, spec: SystemSpec | None = None, handle=None):
        self.spec = spec
        if handle is not None:
            self._h = handle
            return
        desc, keep = spec.desc()
        h = C.c_void_p()
        check(lib().orc_system_create(C.byref(desc), C.byref(h)), "orc_system_create")
        self._h = h
        del keep
        if spec.k_uniform is not None:
            seed, stream, lo, hi = spec.k_uniform
            check(lib().orc_system_fill_k_uniform(self._h, seed, stream, lo, hi), "fill_k")

    @classmethod
    def make_lco(cls, n, seed=0):
        h = C.c_void_p()
        check(lib().orc_make_lco(n, seed, C.byref(h)), "make_lco")
        return cls(handle=h)

    @classmethod
    def make_kuramoto(cls, n, sigma, k, seed):
        h = C.c_void_p()
        check(lib().orc_make_kuramoto(n, sigma, k, seed, C.byref(h)), "make_kuramoto")
        return cls(handle=h)

    @classmethod
    def make_cc(cls, n, k, i0, seed):
        h = C.c_void_p()
        check(lib().orc_make_cc(n, k, i0, seed, C.byref(h)), "make_cc")
        return cls(handle=h)

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            lib().orc_system_destroy(self._h)
            self._h = None

    def dim(self):
        return lib().orc_system_dim(self._h)

    def agents(self):
        return lib().orc_system_agents(self._h)

    def size(self):
        return self.dim() * self.agents()

    def param(self, which: int) -> np.ndarray:
        buf = np.empty(max(self.agents(), 4))
        n = lib().orc_system_get_param(self._h, which, buf.ctypes.data_as(_DP))
        return buf[:n].copy()

    def flop_profile(self):
        out = (C.c_int64 * 4)()
        lib().orc_system_flop_profile(self._h, out)
        return tuple(out)

    def set_op_round(self, ks: int) -> None:
        check(lib().orc_system_set_op_round(self._h, ks), "set_op_round")

    def set_omega(self, omega) -> None:
        om = f64(omega)
        check(lib().orc_system_set_omega(self._h, om.ctypes.data_as(_DP)), "set_omega")

    def get_k(self) -> np.ndarray:
        n = self.agents()
        out = np.empty((n, n))
        check(lib().orc_system_get_k(self._h, out.ctypes.data_as(_DP)), "get_k")
        return out

    def eval_rhs(self, t, x, sp: StagePrecision) -> np.ndarray:
        x = f64(x)
        out = np.empty_like(x)
        check(lib().orc_eval_rhs(self._h, t, x.ctypes.data_as(_DP), sp.c(), out.ctypes.data_as(_DP)), "eval_rhs")
        return out


def estimate_error(a, b, c, ab, rel) -> float:
    a, b, c = f64(a), f64(b), f64(c)
    if not (a.shape == b.shape == c.shape):
        raise ValueError("estimate_error: length mismatch")
    out = C.c_double()
    check(lib().orc_estimate_error(a.size, a.ctypes.data_as(_DP), b.ctypes.data_as(_DP), c.ctypes.data_as(_DP),
                                   ab, rel, C.byref(out)), "estimate_error")
    return out.value


def adjust_step(h, err, rel, cfg: SolverConfig) -> float:
    out = C.c_double()
    cc = cfg.c()
    check(lib().orc_adjust_step(h, err, rel, C.byref(cc), C.byref(out)), "adjust_step")
    return out.value


def initial_step(sys: OracleSystem, t0, tf, x0, cfg: SolverConfig, order=3):
    x0 = f64(x0)
    h0 = C.c_double()
    ev = C.c_int64()
    cc = cfg.c()
    check(lib().orc_initial_step(sys._h, t0, tf, x0.ctypes.data_as(_DP), C.byref(cc), order, C.byref(h0),
                                 C.byref(ev)), "initial_step")
    return h0.value


def bs32_step(sys: OracleSystem, t, x_n, h, k1, policy: PrecisionPolicy, cfg: SolverConfig) -> StepOutcome:
    x_n, k1 = f64(x_n), f64(k1)
    bufs = [np.empty(x_n.size) for _ in range(4)]
    o = _abi.StepOutcomeC()
    o.x_next, o.x_tilde, o.k4, o.x_store = (b.ctypes.data_as(_DP) for b in bufs)
    pol, cc = policy.c(), cfg.c()
    check(lib().orc_bs32_step(sys._h, t, x_n.ctypes.data_as(_DP), h, k1.ctypes.data_as(_DP), C.byref(pol),
                              C.byref(cc), C.byref(o)), "bs32_step")
    return StepOutcome(bufs[0], bufs[1], o.err, bool(o.accepted), bufs[2], bufs[3], o.h_used, o.h_next,
                       FlopTally(o.flops_low, o.flops_high, o.rhs_evals))


def _run(fn, sys, x0, cap, snap_cap=0, t_eval=None):
    x0 = f64(x0)
    final = np.empty_like(x0)
    log = (_abi.StepRecordC * cap)()
    r = _abi.SolveResultC()
    r.final_state = final.ctypes.data_as(_DP)
    r.step_log = C.cast(log, C.POINTER(_abi.StepRecordC))
    r.step_log_capacity = cap
    rows = hs = None
    if snap_cap:
        rows, hs = np.empty((snap_cap + 1, x0.size)), np.empty(snap_cap)
        r.snapshots, r.snapshot_h = rows.ctypes.data_as(_DP), hs.ctypes.data_as(_DP)
        r.snapshot_capacity = snap_cap
    te = ye = None
    if t_eval is not None:
        te = f64(t_eval).ravel()
        ye = np.full((te.size, x0.size), np.nan)
        r.t_eval, r.n_eval, r.y_eval = te.ctypes.data_as(_DP), te.size, ye.ctypes.data_as(_DP)
    check(fn(sys._h, x0.ctypes.data_as(_DP), r), "oracle solve")
    m = min(cap, r.step_log_count)
    steps = [StepRecord(e.t, e.h, e.err, bool(e.accepted)) for e in log[:m]]
    shots = []
    if snap_cap:
        shots = [StepSnapshot(rows[k], rows[k + 1], float(hs[k])) for k in range(min(snap_cap, r.snapshot_count))]
    out = SolveResult(SolveStatus(r.status), final, r.t_reached, r.n_accepted, r.n_failed, steps,
                      FlopTally(r.flops_low, r.flops_high, r.rhs_evals), 0.0, r.step_log_count,
                      shots, r.snapshot_count)
    out.y_eval = ye
    return out


def solve(sys: OracleSystem, x0, t0, tf, policy: PrecisionPolicy, cfg: SolverConfig, cap: int = 200000,
          snapshot_capacity: int = 4096, t_eval=None):
    pol, cc = policy.c(), cfg.c()
    return _run(lambda h, x, r: lib().orc_solve(h, x, t0, tf, C.byref(pol), C.byref(cc), C.byref(r)),
                sys, x0, cap, snapshot_capacity if cfg.record_snapshots else 0, t_eval)


def dp54_reference(sys: OracleSystem, x0, t0, tf, cfg: SolverConfig | None = None, cap: int = 200000):
    cc = (cfg or SolverConfig()).c()
    return _run(lambda h, x, r: lib().orc_dp54_reference(h, x, t0, tf, C.byref(cc), C.byref(r)), sys, x0, cap)


def lco_analytic(x0, t) -> np.ndarray:
    x0 = f64(x0)
    out = np.empty_like(x0)
    check(lib().orc_lco_analytic(x0.size, x0.ctypes.data_as(_DP), t, out.ctypes.data_as(_DP)), "lco_analytic")
    return out


def rng_uniform(seed, stream, n, lo, hi):
    out = np.empty(n)
    lib().orc_rng_uniform(seed, stream, n, lo, hi, out.ctypes.data_as(_DP))
    return out


def rng_normal(seed, stream, n):
    out = np.empty(n)
    lib().orc_rng_normal(seed, stream, n, out.ctypes.data_as(_DP))
    return out
