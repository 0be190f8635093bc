"""The reference's test runner (harness.cpp:97-195 run_one, :305-343 inputs,
:518-553 persistence) over the device C-ABI: one test case = the tight DP5(4)
reference plus every requested precision variant on the same system and
initial state, reported as rows of the reference's results.csv schema
(harness.cpp:199-201) and, optionally, steps.csv (harness.cpp:394) — so a
device campaign and an oracle/reference campaign can be diffed line by line.

The solver calls go through an ``engine`` (default: the device), which makes
the same runner usable with the CPU oracle in the tests. The reference's Sobol
campaign generator and its thread pool are not part of the hot path (SURVEY.md
section 2) and are not rebuilt: callers pass the TestCases."""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from decimal import Decimal
from pathlib import Path

import numpy as np

from . import metrics as M
from . import solver as S
from .configs import reference_ic
from .precision import PolicyVariant, policy_for
from .solver import SolverConfig, SolveStatus

RESULTS_CSV_HEADER = ("test_id,benchmark,N,rel_tol,abs_tol,variant,status,n_accepted,n_failed,"
                      "final_error,mean_ebs,mean_eanalytic,beta,rho,gamma,capital_gamma,t_final")
STEPS_CSV_HEADER = "test_id,variant,t,h,e_bs,accepted"
VARIANT_NAMES = {PolicyVariant.Single: "Single", PolicyVariant.Mixed1: "Mixed1",
                 PolicyVariant.Mixed2: "Mixed2", PolicyVariant.Double: "Double"}  # precision.cpp:44-52
STATUS_NAMES = ["Completed", "MaxIterations", "MaxFailedSteps", "WallClock", "SlowSolver", "StepTooSmall",
                "NonFinite"]  # solver.cpp:386-397
BENCHMARKS = ("lco", "kuramoto", "cc")  # systems.cpp:193-200


def format_double(v: float) -> str:
    """std::to_chars(double) (harness.cpp:199-203): the precision of the
    shortest round-trip representation, printed as %f or %e, whichever is
    shorter (%f on a tie). Checked against libstdc++ on 20 000 values
    (tests/golden/to_chars.txt)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign, digits, exp = Decimal(repr(v)).as_tuple()
    ds = "".join(map(str, digits)).rstrip("0")
    exp += len(digits) - len(ds)  # value = int(ds) * 10**exp
    n = len(ds)
    e10 = exp + n - 1
    sci = ds[0] + ("." + ds[1:] if n > 1 else "") + "e" + ("-" if e10 < 0 else "+") + f"{abs(e10):02d}"
    if exp >= 0:  # an integer: %.0f prints its exact digits (same length)
        fixed = str(abs(int(v)))
    elif n + exp > 0:
        fixed = ds[:n + exp] + "." + ds[n + exp:]
    else:
        fixed = "0." + "0" * (-(n + exp)) + ds
    s = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + s


@dataclass
class TestCase:  # harness.hpp:18-30 (the test id seeds every draw of the test)
    test_id: int = 0
    benchmark: str = "lco"
    agents: int = 0
    rel_tol: float = 1e-6
    abs_tol: float = 1e-8
    t_final: float = 0.0
    sigma: float = 0.0
    coupling_k: float = 0.0
    stimulus_i0: float = 0.0


@dataclass
class ResultRow:  # harness.hpp:62-81
    test_id: int = 0
    benchmark: str = "lco"
    agents: int = 0
    rel_tol: float = 0.0
    abs_tol: float = 0.0
    variant: str = ""
    status: SolveStatus = SolveStatus.Completed
    n_accepted: int = 0
    n_failed: int = 0
    final_error: float | None = None
    mean_ebs: float | None = None
    mean_eanalytic: float | None = None
    beta: float | None = None
    rho: float | None = None
    gamma: float | None = None
    capital_gamma: float | None = None
    t_final: float = 0.0


@dataclass
class RunOptions:  # harness.hpp:52-60 (jobs: one device, cases run in order)
    time_limits: bool = True
    wall_clock_limit: float = 5400.0
    slow_solver_elapsed: float = 2700.0
    slow_solver_progress: float = 0.10
    output_dir: str = ""
    step_log_csv: bool = False
    rhs_mode: str = "fast"
    # run the variants of a case concurrently (DeviceVariants: one K sweep per
    # stage for all of them; results bit-identical to one solve each)
    concurrent_variants: bool = True


@dataclass
class CampaignSpec:  # harness.hpp:32-50 (the run_one-relevant fields)
    variants: list = field(default_factory=lambda: [PolicyVariant.Single, PolicyVariant.Mixed1,
                                                    PolicyVariant.Mixed2, PolicyVariant.Double])
    snapshots: bool = False
    speedup_r: float = 0.5


def initial_conditions(tc: TestCase) -> np.ndarray:
    """harness.cpp:305-330: stream 1 of the test id."""
    if tc.benchmark not in BENCHMARKS:
        raise ValueError(f"initial_conditions: unknown benchmark {tc.benchmark!r}")
    return reference_ic(tc.benchmark, tc.agents, tc.test_id)


class DeviceEngine:
    """Systems and solves on the B200 through the C-ABI."""

    def __init__(self, rhs_mode: str = "fast"):
        self.rhs_mode = rhs_mode

    def build_system(self, tc: TestCase):  # harness.cpp:332-343
        from .systems import make_cc, make_kuramoto, make_lco
        if tc.benchmark == "lco":
            return make_lco(tc.agents, tc.test_id, rhs_mode=self.rhs_mode)
        if tc.benchmark == "kuramoto":
            return make_kuramoto(tc.agents, tc.sigma, tc.coupling_k, tc.test_id, rhs_mode=self.rhs_mode)
        if tc.benchmark == "cc":
            return make_cc(tc.agents, tc.coupling_k, tc.stimulus_i0, tc.test_id, rhs_mode=self.rhs_mode)
        raise ValueError(f"build_system: unknown benchmark {tc.benchmark!r}")

    def solve(self, sys, x0, tf, policy, cfg):
        return S.solve(sys, x0, 0.0, tf, policy, cfg)

    def dp54_reference(self, sys, x0, tf, cfg):
        return S.dp54_reference(sys, x0, 0.0, tf, cfg)

    def solve_variants(self, sys, x0, tf, policies, cfg):
        return S.solve_variants(sys, x0, 0.0, tf, policies, cfg)

    def release(self, sys):
        sys.close()


def _mean_ebs(r) -> float | None:  # harness.cpp:123-134
    acc = np.array([e.err for e in r.step_log if e.accepted], dtype=np.float64)
    if acc.size == 0:
        return None
    return float(np.cumsum(acc)[-1]) / acc.size


def _low_fraction(r) -> float:  # solver.hpp:109-112
    tot = float(r.flops.low) + float(r.flops.high)
    return float(r.flops.low) / tot if tot > 0.0 else 0.0


def gamma_of(rho: float, r: float) -> float:  # metrics.cpp:95-101
    if not 0.0 <= rho <= 1.0:
        raise ValueError("gamma_of: rho must lie in [0, 1]")
    if not 0.0 < r < 1.0:
        raise ValueError("gamma_of: r must lie in (0, 1)")
    return rho * r + (1.0 - rho)


def beta_of(n_steps_high: int, n_steps_mixed: int) -> float:  # metrics.cpp:103-107
    if n_steps_high < 1 or n_steps_mixed < 1:
        raise ValueError("beta_of: step counts must be >= 1")
    return float(n_steps_high) / float(n_steps_mixed)


def capital_gamma_of(gamma: float, beta: float) -> float:  # metrics.cpp:109-113
    if beta <= 0.0:
        raise ValueError("capital_gamma_of: beta must be positive")
    return gamma / beta


def _step_rows(test_id: int, variant: str, log) -> str:  # harness.cpp:75-95
    return "".join(f"{test_id},{variant},{format_double(e.t)},{format_double(e.h)},{format_double(e.err)},"
                   f"{1 if e.accepted else 0}\n" for e in log)


def run_one(tc: TestCase, spec: CampaignSpec | None = None, opt: RunOptions | None = None, engine=None):
    """harness.cpp:97-195: the DP5(4) reference and every variant on one case.
    Returns (rows, steps_csv_text); the Reference row comes last."""
    spec = spec or CampaignSpec()
    opt = opt or RunOptions()
    engine = engine or DeviceEngine(opt.rhs_mode)
    sys = engine.build_system(tc)
    try:
        x0 = initial_conditions(tc)
        base = SolverConfig(rel_tol=tc.rel_tol, abs_tol=tc.abs_tol, time_limits_enabled=opt.time_limits,
                            wall_clock_limit=opt.wall_clock_limit, slow_solver_elapsed=opt.slow_solver_elapsed,
                            slow_solver_progress=opt.slow_solver_progress)
        ref = engine.dp54_reference(sys, x0, tc.t_final, base)
        snaps = spec.snapshots and tc.benchmark == "lco"
        cfg = SolverConfig(**{**base.__dict__, "record_snapshots": snaps})
        if (opt.concurrent_variants and not snaps and hasattr(engine, "solve_variants")
                and 1 <= len(spec.variants) <= 4):
            runs = engine.solve_variants(sys, x0, tc.t_final, [policy_for(v) for v in spec.variants], cfg)
        else:
            runs = [engine.solve(sys, x0, tc.t_final, policy_for(v), cfg) for v in spec.variants]
        double_steps = None
        for v, r in zip(spec.variants, runs):
            if v == PolicyVariant.Double and r.total_steps() > 0:
                double_steps = r.total_steps()
    finally:
        engine.release(sys)
    rows, steps = [], ""
    for v, r in zip(spec.variants, runs):
        row = ResultRow(tc.test_id, tc.benchmark, tc.agents, tc.rel_tol, tc.abs_tol, VARIANT_NAMES[v], r.status,
                        r.n_accepted, r.n_failed, t_final=tc.t_final)
        if r.status == SolveStatus.Completed and ref.status == SolveStatus.Completed:
            er = M.error_report(r, ref.final_state, tc.agents, tc.abs_tol, tc.rel_tol)
            row.final_error, row.mean_ebs, row.mean_eanalytic = er.normalized_final_error, er.mean_e_bs, \
                er.mean_e_analytic
        else:  # failed runs still report what they measured
            row.mean_ebs = _mean_ebs(r)
            if r.snapshots:
                e = np.array([M.real_local_error(s.x_before, s.x_after, s.h, tc.abs_tol, tc.rel_tol)
                              for s in r.snapshots])
                row.mean_eanalytic = float(np.cumsum(e)[-1]) / e.size
        row.rho = _low_fraction(r)
        row.gamma = gamma_of(row.rho, spec.speedup_r)
        if double_steps and r.total_steps() > 0:
            row.beta = beta_of(double_steps, r.total_steps())
        if row.beta is not None:
            row.capital_gamma = capital_gamma_of(row.gamma, row.beta)
        rows.append(row)
        if opt.step_log_csv:
            steps += _step_rows(tc.test_id, VARIANT_NAMES[v], r.step_log)
    rows.append(ResultRow(tc.test_id, tc.benchmark, tc.agents, tc.rel_tol, tc.abs_tol, "Reference", ref.status,
                          ref.n_accepted, ref.n_failed, mean_ebs=_mean_ebs(ref), t_final=tc.t_final))
    if opt.step_log_csv:
        steps += _step_rows(tc.test_id, "Reference", ref.step_log)
    return rows, steps


def _opt(v: float | None) -> str:
    return "" if v is None else format_double(v)


def result_row_to_csv(r: ResultRow) -> str:  # harness.cpp:518-553
    return ",".join([str(r.test_id), r.benchmark, str(r.agents), format_double(r.rel_tol), format_double(r.abs_tol),
                     r.variant, STATUS_NAMES[int(r.status)], str(r.n_accepted), str(r.n_failed),
                     _opt(r.final_error), _opt(r.mean_ebs), _opt(r.mean_eanalytic), _opt(r.beta), _opt(r.rho),
                     _opt(r.gamma), _opt(r.capital_gamma), format_double(r.t_final)])


def write_results_csv(path, rows) -> None:
    Path(path).write_text(RESULTS_CSV_HEADER + "\n" + "".join(result_row_to_csv(r) + "\n" for r in rows))


def read_results_csv(path, lenient: bool = False) -> list:
    """Strict mode raises on any malformed row; lenient mode skips torn lines."""
    lines = Path(path).read_text().splitlines()
    if not lines or lines[0] != RESULTS_CSV_HEADER:
        raise ValueError(f"{path}: not a results.csv (header mismatch)")
    out = []
    for ln in lines[1:]:
        f = ln.split(",")
        try:
            if len(f) != 17 or f[1] not in BENCHMARKS:
                raise ValueError(ln)
            opt = [None if s == "" else float(s) for s in f[9:16]]
            out.append(ResultRow(int(f[0]), f[1], int(f[2]), float(f[3]), float(f[4]), f[5],
                                 SolveStatus(STATUS_NAMES.index(f[6])), int(f[7]), int(f[8]), *opt, float(f[16])))
        except ValueError:
            if not lenient:
                raise ValueError(f"{path}: malformed row {ln!r}") from None
    return out


def run_cases(cases, spec: CampaignSpec | None = None, opt: RunOptions | None = None, engine=None) -> list:
    """run_campaign (harness.cpp:345-470) on one device, cases in order: with
    an output directory the rows of each finished case are appended to
    results.csv (and steps.csv) at once, and a rerun keeps the cases whose
    rows are all there (resume)."""
    spec = spec or CampaignSpec()
    opt = opt or RunOptions()
    if not cases:
        raise ValueError("run_campaign: empty case list")
    if not spec.variants:
        raise ValueError("run_campaign: empty variant list")
    if not 0.0 < spec.speedup_r < 1.0:
        raise ValueError("run_campaign: speedup_r must lie in (0, 1)")
    kept, kept_steps = {}, {}
    res_f = steps_f = None
    if opt.output_dir:
        d = Path(opt.output_dir)
        d.mkdir(parents=True, exist_ok=True)
        rp, sp = d / "results.csv", d / "steps.csv"
        if rp.exists():
            groups = {}
            for r in read_results_csv(rp, lenient=True):
                groups.setdefault(r.test_id, []).append(r)
            kept = {k: v for k, v in groups.items() if len(v) == len(spec.variants) + 1}
        if opt.step_log_csv and sp.exists():
            for ln in sp.read_text().splitlines()[1:]:
                tid = int(ln.split(",", 1)[0])
                if tid in kept:
                    kept_steps[tid] = kept_steps.get(tid, "") + ln + "\n"
        res_f = open(rp, "w")
        res_f.write(RESULTS_CSV_HEADER + "\n")
        if opt.step_log_csv:
            steps_f = open(sp, "w")
            steps_f.write(STEPS_CSV_HEADER + "\n")
    out = []
    try:
        for tc in cases:
            if tc.test_id in kept:
                rows, steps = kept[tc.test_id], kept_steps.get(tc.test_id, "")
            else:
                rows, steps = run_one(tc, spec, opt, engine)
            if steps_f:
                steps_f.write(steps)
                steps_f.flush()
            if res_f:
                res_f.write("".join(result_row_to_csv(r) + "\n" for r in rows))
                res_f.flush()
                os.fsync(res_f.fileno())
            out.extend(rows)
    finally:
        if res_f:
            res_f.close()
        if steps_f:
            steps_f.close()
    return out
