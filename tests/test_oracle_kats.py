"""Pin the CPU oracle to the reference's own known-answer tests.

The reference cannot be built here (Eigen3/doctest absent),
so its KATs are restated against the oracle; each test cites the reference
test it restates. Golden values are in tests/golden/reference_kats.json.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200.precision import (B32, B64, DDD, DDS, SSS, PolicyVariant, StagePrecision, custom_policy,
                                             kAllBinary32, kAllBinary64, policy_for)
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import SystemSpec

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_kats.json").read_text())
PI = 3.14159265358979323846


def fixture(kind):
    return O.OracleSystem(SystemSpec("scalar_" + kind, 1))


# ---- precision (test_precision.cpp) -------------------------------------------------
def test_machine_epsilon():  # test_precision.cpp:26-32
    L = O.lib()
    assert L.orc_machine_epsilon(0) == 1.1920928955078125e-7
    assert L.orc_machine_epsilon(1) == 2.220446049250313e-16


def test_round_to_basics():  # test_precision.cpp:34-49
    r = O.lib().orc_round_to
    assert r(1.0, 0) == 1.0
    assert r(1.0 + 2.0 ** -24, 0) == 1.0
    assert r(0.1, 0) == 0.100000001490116119384765625
    assert r(0.1, 1) == 0.1
    assert r(math.inf, 0) == math.inf and r(-math.inf, 0) == -math.inf
    assert math.isnan(r(math.nan, 0))
    assert r(1e39, 0) == math.inf and r(-1e39, 0) == -math.inf


def _round32_oracle(x):  # test_precision.cpp:13-22 (frexp/ldexp mantissa rounding)
    if not math.isfinite(x) or x == 0.0:
        return x
    m, e = math.frexp(x)
    m = np.rint(m * 16777216.0) / 16777216.0
    return math.ldexp(m, e)


def test_round_to_property():  # test_precision.cpp:51-59 (20000 draws, SplitMix64(7))
    L = O.lib()
    u = O.rng_uniform(7, 0, 40000, 0.0, 1.0)
    for i in range(20000):
        mag = math.exp(-40.0 + 80.0 * u[2 * i])
        x = (-1.0 if u[2 * i + 1] < 0.5 else 1.0) * mag
        assert L.orc_round_to(x, 0) == _round32_oracle(x)


def test_policy_table():  # test_precision.cpp:82-124
    import ctypes as C
    from paper_2605_23727_b200 import _abi
    for v in (0, 1, 2, 3):
        p = _abi.Policy()
        assert O.lib().orc_policy_for(v, C.byref(p)) == 0
        ref = policy_for(PolicyVariant(v))
        got = [(r.f_prec, r.sum_prec, r.g_prec) for r in p.per_stage]
        assert got == [(int(s.f_prec), int(s.sum_prec), int(s.g_prec)) for s in ref.per_stage]
        k1 = p.first_step_k1
        assert (k1.f_prec, k1.sum_prec, k1.g_prec) == got[2]
        assert p.storage == (0 if v == 0 else 1)
        assert O.lib().orc_policy_lowest_format(C.byref(p)) == (1 if v == 3 else 0)
    assert policy_for(PolicyVariant.Mixed1).per_stage == (SSS, SSS, DDS)
    assert policy_for(PolicyVariant.Mixed2).per_stage == (DDS, DDS, DDS)


# ---- rng (rng.hpp:13-52) ----------------------------------------------------------
def test_splitmix_known_answers():
    # splitmix64 with seed 0 / stream 0: the published splitmix64 reference stream
    L = O.lib()
    for k, v in enumerate(GOLD["splitmix64_seed0"]):
        assert L.orc_rng_next(0, 0, k) == int(v, 16)
    # stream offset: state = seed + stream * 0xD1342543DE82EF95
    s = (5 + 3 * 0xD1342543DE82EF95) & (2 ** 64 - 1)
    z = (s + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
    z ^= z >> 31
    assert L.orc_rng_next(5, 3, 0) == z


def test_normal_pairs_cos_first():  # rng.hpp:33-46
    L = O.lib()
    u1 = (L.orc_rng_next(9, 0, 0) >> 11) * 2.0 ** -53
    u2 = (L.orc_rng_next(9, 0, 1) >> 11) * 2.0 ** -53
    r = math.sqrt(-2.0 * math.log(u1))
    a = 6.283185307179586476925286766559 * u2
    z = O.rng_normal(9, 0, 2)
    assert z[0] == r * math.cos(a) and z[1] == r * math.sin(a)


# ---- systems (test_systems.cpp) ------------------------------------------------------
def test_lco_identical_agents():  # test_systems.cpp:99-110
    sys = O.OracleSystem.make_lco(2, 1)
    x = np.array([1.0, 0.0, 1.0, 0.0])
    for sp in (kAllBinary64, kAllBinary32):
        assert list(sys.eval_rhs(0.0, x, sp)) == [0.0, -1.0, 0.0, -1.0]


def test_kuramoto_hand_values():  # test_systems.cpp:112-127
    sys = O.OracleSystem.make_kuramoto(2, 0.0, 1.0, 3)
    assert list(sys.param(0)) == [0.0, 0.0]
    out = sys.eval_rhs(0.0, [0.0, PI], kAllBinary64)
    assert abs(out[0]) <= 1e-15 and abs(out[1]) <= 1e-15
    out = sys.eval_rhs(0.0, [0.0, PI / 2.0], kAllBinary64)
    assert out[0] == pytest.approx(0.5, rel=1e-14) and out[1] == pytest.approx(-0.5, rel=1e-14)


def _lco_rhs_float(x, n):  # test_systems.cpp:24-43 (plain single-precision loops)
    f = np.float32
    xf = x.astype(np.float32)
    m0 = f(1.0 / n)
    out = np.empty(2 * n)
    for i in range(n):
        acc0 = f(0.0)
        acc1 = f(0.0)
        for j in range(n):
            acc0 = f(acc0 + f(m0 * f(xf[2 * j] - xf[2 * i])))
            acc1 = f(acc1 + f(f(0.0) * f(0.0)))
        out[2 * i] = float(f(xf[2 * i + 1] + acc0))
        out[2 * i + 1] = float(f(-xf[2 * i] + acc1))
    return out


def _lco_rhs_double(x, n):  # test_systems.cpp:45-60
    m0 = 1.0 / n
    out = np.empty(2 * n)
    for i in range(n):
        acc0 = 0.0
        acc1 = 0.0
        for j in range(n):
            acc0 = acc0 + m0 * (x[2 * j] - x[2 * i])
            acc1 = acc1 + 0.0 * 0.0
        out[2 * i] = x[2 * i + 1] + acc0
        out[2 * i + 1] = -x[2 * i] + acc1
    return out


def _kuramoto_rhs_double(x, omega, k, n):  # test_systems.cpp:62-71
    m = 1.0 / n
    out = np.empty(n)
    for i in range(n):
        acc = 0.0
        for j in range(n):
            acc = acc + m * (k * math.sin(x[j] - x[i]))
        out[i] = omega[i] + acc
    return out


def test_bitwise_vs_plain_loops():  # test_systems.cpp:129-140
    n = 17
    x = O.rng_uniform(99, 0, 2 * n, -2.0, 2.0)
    sys = O.OracleSystem.make_lco(n, 1)
    assert np.array_equal(sys.eval_rhs(0.0, x, kAllBinary64), _lco_rhs_double(x, n))
    assert np.array_equal(sys.eval_rhs(0.0, x, kAllBinary32), _lco_rhs_float(x, n))
    kur = O.OracleSystem.make_kuramoto(n, 0.7, 1.3, 5)
    xp = O.rng_uniform(100, 0, n, 0.0, 2.0 * PI)
    assert np.array_equal(kur.eval_rhs(0.0, xp, kAllBinary64), _kuramoto_rhs_double(xp, kur.param(0), 1.3, n))


def test_kuramoto_mean_cancellation():  # test_systems.cpp:142-155
    n, k = 64, 2.0
    sys = O.OracleSystem.make_kuramoto(n, 0.5, k, 21)
    x = O.rng_uniform(22, 0, n, 0.0, 2.0 * PI)
    for sp in (kAllBinary64, kAllBinary32, DDS):
        out = sys.eval_rhs(0.0, x, sp)
        drift = out.mean() - sys.param(0).mean()
        eps = 2.0 ** -23 if sp.sum_prec == B32 else 2.0 ** -52
        assert abs(drift) <= 10.0 * n * eps * k


def test_lco_rhs_analytic_derivative():  # test_systems.cpp:157-193
    n = 6
    sys = O.OracleSystem.make_lco(n, 1)
    x0 = O.rng_uniform(31, 0, 2 * n, 0.0, 2.0)
    f = sys.eval_rhs(0.0, x0, kAllBinary64)
    xm, vm = x0[0::2].mean(), x0[1::2].mean()
    du, dv = x0[0::2] - xm, x0[1::2] - vm
    deriv = np.empty(2 * n)
    deriv[0::2] = vm + (-du + dv)
    deriv[1::2] = -xm + (-du)
    assert np.allclose(f, deriv, rtol=1e-12, atol=0)
    d = 1e-4
    fs = [O.lco_analytic(x0, k * d) for k in (1, 2, 3, 4)]
    fd = (-25.0 * x0 + 48.0 * fs[0] - 36.0 * fs[1] + 16.0 * fs[2] - 3.0 * fs[3]) / (12.0 * d)
    assert np.allclose(f, fd, rtol=1e-9, atol=1e-12)


def test_lco_analytic_solution():  # test_systems.cpp:195-226
    x0 = np.tile([1.0, 0.0], 3)
    for t in (0.0, 0.4, 2.0, 7.5):
        xt = O.lco_analytic(x0, t)
        assert np.allclose(xt[0::2], math.cos(t), rtol=1e-14, atol=1e-15)
        assert np.allclose(xt[1::2], -math.sin(t), rtol=1e-14, atol=1e-15)
    xr = O.rng_uniform(77, 0, 10, -1.0, 1.0)
    assert np.array_equal(O.lco_analytic(xr, 0.0), xr)
    # series expm of the deviation block A = [[-1, 1], [-1, 0]] at t = 1
    a = np.array([[-1.0, 1.0], [-1.0, 0.0]])
    term, p = np.eye(2), np.eye(2)
    for k in range(1, 200):
        term = term @ a / k
        p = p + term
    got = O.lco_analytic([1.0, 0.0, -1.0, 0.0], 1.0)
    assert got[0] == pytest.approx(p[0, 0], rel=1e-13) and got[1] == pytest.approx(p[1, 0], rel=1e-13)


def test_factories():  # test_systems.cpp:228-257
    with pytest.raises(ValueError):
        O.OracleSystem.make_lco(0, 1)
    with pytest.raises(ValueError):
        O.OracleSystem.make_kuramoto(0, 0.1, 1.0, 1)
    with pytest.raises(ValueError):
        O.OracleSystem.make_kuramoto(4, -0.1, 1.0, 1)
    lco = O.OracleSystem.make_lco(8, 1)
    assert list(lco.param(3)[:2]) == [1.0 / 8.0, 0.0] and lco.dim() == 2 and lco.size() == 16
    k1 = O.OracleSystem.make_kuramoto(32, 0.4, 1.0, 9).param(0)
    assert np.array_equal(k1, O.OracleSystem.make_kuramoto(32, 0.4, 1.0, 9).param(0))
    assert not np.array_equal(k1, O.OracleSystem.make_kuramoto(32, 0.4, 1.0, 10).param(0))
    for seed in (1, 2, 17, 400):
        cc = O.OracleSystem.make_cc(64, 1.0, 1.5, seed)
        k1v, th = cc.param(1), cc.param(2)
        assert np.all(k1v > 0.05) and np.all(k1v < 1.95) and np.all(th > 0)
        assert np.allclose(th, k1v / (2.0 - k1v), rtol=1e-15)


def test_flop_profiles():  # test_systems.cpp:259-320 (values of the instrumented count)
    assert O.OracleSystem.make_lco(4, 1).flop_profile() == (1, 1, 4, 2)
    assert O.OracleSystem.make_kuramoto(4, 0.3, 1.2, 1).flop_profile() == (1, 3, 2, 1)
    assert O.OracleSystem.make_cc(4, 1.0, 1.5, 1).flop_profile() == (28, 10, 8, 4)


def test_cc_finite():  # test_systems.cpp:322-340
    for k in (0.001, 10.0):
        for i0 in (0.228249, 10.0):
            sys = O.OracleSystem.make_cc(6, k, i0, 12)
            x = np.tile([1.0, 1.0, -1.19, -0.62], 6)
            for _ in range(2000):
                x = x + 0.01 * sys.eval_rhs(0.0, x, kAllBinary64)
            assert np.all(np.isfinite(x))


# ---- solver (test_solver.cpp) ----------------------------------------------------------
def test_scheme_flops():  # test_solver.cpp:31-53
    assert O.lib().orc_scheme_flops_bs32() == 30


def test_estimate_error_kats():  # test_solver.cpp:55-75
    assert O.estimate_error([0.0], [0.0], [0.0], 1e-2, 1.0) == 0.0
    assert O.estimate_error([0.0], [0.0], [1e-6], 1e-2, 1.0) == pytest.approx(1e-4, rel=1e-12)
    xn, xnext, xt = np.array([2.0, -3.0]), np.array([2.1, -3.1]), np.array([2.1000004, -3.0999996])
    e1 = O.estimate_error(xn, xnext, xt, 1e-8, 1e-2)
    e2 = O.estimate_error(10 * xn, 10 * xnext, 10 * xt, 1e-8, 1e-2)
    assert e1 == pytest.approx(e2, rel=1e-9)
    with pytest.raises(ValueError):
        O.estimate_error([0.0], [0.0], [0.0, 1.0], 1e-2, 1.0)


def test_adjust_step_kats():  # test_solver.cpp:77-87
    cfg = SolverConfig()
    tol = cfg.rel_tol
    assert O.adjust_step(1.0, tol, tol, cfg) == pytest.approx(0.9, rel=1e-15)
    assert O.adjust_step(2.0, 8.0 * tol, tol, cfg) == pytest.approx(0.9, rel=1e-14)
    assert O.adjust_step(1.0, 0.0, tol, cfg) == 5.0
    assert O.adjust_step(1.0, 1e9 * tol, tol, cfg) == 0.2
    assert O.adjust_step(1.0, 1e-12 * tol, tol, cfg) == 5.0


def test_initial_step_kats():  # test_solver.cpp:89-109
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
    assert O.initial_step(fixture("zero"), 0.0, 5.0, [1.0], cfg) == 0.5
    h0 = O.initial_step(fixture("exp"), 0.0, 1.0, [1.0], cfg)
    assert 0.0 < h0 <= 0.1
    h0 = O.initial_step(fixture("exp"), 0.0, 50.0, [1.0], cfg)
    assert 0.0 < h0 <= 0.1
    assert math.isnan(O.initial_step(fixture("nan"), 0.0, 1.0, [1.0], cfg))


def test_bs32_step_exp_kat():  # test_solver.cpp:111-133
    g = GOLD["bs32_exp_step"]
    cfg = SolverConfig(rel_tol=1e-2, abs_tol=1e-2)
    o = O.bs32_step(fixture("exp"), 0.0, [1.0], 0.1, [1.0], policy_for(PolicyVariant.Double), cfg)
    assert o.x_next[0] == pytest.approx(g["x_next"], rel=1e-15)
    assert o.x_tilde[0] == pytest.approx(g["x_tilde"], rel=1e-15)
    assert o.err == pytest.approx(g["err"], rel=1e-12)
    assert o.k4[0] == o.x_next[0] and o.accepted
    cfg = SolverConfig(rel_tol=1e-2, abs_tol=1e-1)
    o = O.bs32_step(fixture("exp"), 0.0, [1.0], 0.1, [1.0], policy_for(PolicyVariant.Double), cfg)
    assert o.err == pytest.approx(g["err_floor10"], rel=1e-12)


def test_bs32_step_zero_kat():  # test_solver.cpp:135-148
    o = O.bs32_step(fixture("zero"), 0.0, [1.0], 1.0, [0.0], policy_for(PolicyVariant.Single), SolverConfig())
    assert o.x_next[0] == 1.0 and o.x_tilde[0] == 1.0 and o.err == 0.0 and o.accepted and o.h_next == 5.0


def test_solve_to_e():  # test_solver.cpp:150-168
    cfg = SolverConfig(rel_tol=1e-8, abs_tol=1e-10)
    r = O.solve(fixture("exp"), [1.0], 0.0, 1.0, policy_for(PolicyVariant.Double), cfg)
    assert r.status == SolveStatus.Completed and r.t_reached == 1.0
    assert abs(r.final_state[0] - math.e) / math.e <= 1e-6
    for rec in r.step_log:
        assert (rec.err <= cfg.rel_tol) if rec.accepted else (rec.err > cfg.rel_tol or not math.isfinite(rec.err))


def test_lco_periodic_return():  # test_solver.cpp:170-181
    sys = O.OracleSystem.make_lco(4, 1)
    x0 = np.tile([1.0, 0.0], 4)
    r = O.solve(sys, x0, 0.0, 2.0 * PI, policy_for(PolicyVariant.Double), SolverConfig(rel_tol=1e-6, abs_tol=1e-8))
    assert r.status == SolveStatus.Completed
    assert np.all(np.abs(r.final_state - x0) <= 1e-4)


def test_step_too_small_single():  # test_solver.cpp:183-195
    sys = O.OracleSystem.make_lco(8, 3)
    x0 = O.rng_uniform(5, 0, 16, 0.0, 2.0)
    r = O.solve(sys, x0, 0.0, 10.0, policy_for(PolicyVariant.Single), SolverConfig(rel_tol=1e-12, abs_tol=1e-14))
    assert r.status == SolveStatus.StepTooSmall and r.t_reached < 10.0


def test_dp54_quality():  # test_solver.cpp:197-211
    r = O.dp54_reference(fixture("exp"), [1.0], 0.0, 1.0)
    assert r.status == SolveStatus.Completed and abs(r.final_state[0] - math.e) / math.e <= 1e-8
    lco = O.OracleSystem.make_lco(4, 1)
    y0 = np.tile([1.0, 0.0], 4)
    p = O.dp54_reference(lco, y0, 0.0, 2.0 * PI)
    assert p.status == SolveStatus.Completed and np.all(np.abs(p.final_state - y0) <= 1e-7)


def test_fsal_budget_and_bitwise_k4():  # test_solver.cpp:213-237
    cfg = SolverConfig(rel_tol=1e-5, abs_tol=1e-7)
    r = O.solve(fixture("exp"), [1.0], 0.0, 1.0, policy_for(PolicyVariant.Double), cfg)
    assert r.status == SolveStatus.Completed and r.n_failed == 0
    assert r.flops.rhs_evals == 3 + 3 * r.n_accepted
    lco = O.OracleSystem.make_lco(3, 1)
    y = np.array([0.3, 1.1, -0.4, 0.2, 1.7, 0.9])
    pol = policy_for(PolicyVariant.Mixed1)
    k1 = lco.eval_rhs(0.0, y, pol.first_step_k1)
    o = O.bs32_step(lco, 0.0, y, 0.005, k1, pol, cfg)
    assert o.accepted
    assert np.array_equal(o.k4, lco.eval_rhs(0.005, o.x_next, pol.stage(4)))


def test_all_d_policy_equals_double():  # test_solver.cpp:239-265
    sys = O.OracleSystem.make_kuramoto(12, 0.6, 0.9, 8)
    x0 = O.rng_uniform(9, 0, 12, 0.0, 2 * PI)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
    a = O.solve(sys, x0, 0.0, 20.0, policy_for(PolicyVariant.Double), cfg)
    all_d = custom_policy((DDD, DDD, DDD), DDD, B64)
    b = O.solve(sys, x0, 0.0, 20.0, all_d, cfg)
    assert a.status == b.status and np.array_equal(a.final_state, b.final_state)
    assert [(s.t, s.h, s.err, s.accepted) for s in a.step_log] == [(s.t, s.h, s.err, s.accepted) for s in b.step_log]


def test_determinism():  # test_solver.cpp:267-291
    sys = O.OracleSystem.make_cc(5, 1.0, 1.5, 4)
    u = O.rng_uniform(14, 0, 5, 0.0, 1.0)
    x0 = np.array([[1.0 + 0.1 * u[i], 1.0, -1.19, -0.62] for i in range(5)]).reshape(-1)
    cfg = SolverConfig(rel_tol=1e-5, abs_tol=1e-7, time_limits_enabled=False)
    pol = policy_for(PolicyVariant.Mixed2)
    a = O.solve(sys, x0, 0.0, 30.0, pol, cfg)
    b = O.solve(sys, x0, 0.0, 30.0, pol, cfg)
    assert (a.status, a.n_accepted, a.n_failed) == (b.status, b.n_accepted, b.n_failed)
    assert np.array_equal(a.final_state, b.final_state)
    assert [s.err for s in a.step_log] == [s.err for s in b.step_log]


def test_one_step_order():  # test_solver.cpp:293-318
    sys = O.OracleSystem.make_lco(4, 1)
    x0 = O.rng_uniform(3, 0, 8, 0.0, 2.0)
    cfg = SolverConfig(rel_tol=0.5, abs_tol=0.5)
    k1 = sys.eval_rhs(0.0, x0, kAllBinary64)
    prev, h = 0.0, 0.1
    for level in range(4):
        o = O.bs32_step(sys, 0.0, x0, h, k1, policy_for(PolicyVariant.Double), cfg)
        err = np.max(np.abs(o.x_next - O.lco_analytic(x0, h)))
        if level > 0:
            assert 12.0 <= prev / err <= 20.0
        prev, h = err, h * 0.5


def test_failure_statuses():  # test_solver.cpp:320-359
    sys = O.OracleSystem.make_lco(4, 2)
    x0 = O.rng_uniform(6, 0, 8, 0.0, 2.0)
    D = policy_for(PolicyVariant.Double)
    r = O.solve(sys, x0, 0.0, 1e4, D, SolverConfig(rel_tol=1e-8, abs_tol=1e-10, max_iterations=5))
    assert r.status == SolveStatus.MaxIterations and r.total_steps() <= 5
    r = O.solve(sys, x0, 0.0, 1e4, D, SolverConfig(rel_tol=1e-8, abs_tol=1e-10, wall_clock_limit=0.0))
    assert r.status == SolveStatus.WallClock
    r = O.solve(sys, x0, 0.0, 1e4, D, SolverConfig(rel_tol=1e-8, abs_tol=1e-10, slow_solver_elapsed=0.0))
    assert r.status == SolveStatus.SlowSolver
    r = O.solve(fixture("nan"), [1.0], 0.0, 1.0, D, SolverConfig(rel_tol=1e-8, abs_tol=1e-10))
    assert r.status == SolveStatus.NonFinite
    with pytest.raises(ValueError):
        O.solve(sys, x0, 0.0, 1.0, D, SolverConfig(rel_tol=1e-8, abs_tol=1.0))
    with pytest.raises(ValueError):
        O.solve(sys, x0, 1.0, 1.0, D, SolverConfig())


def test_single_binary32_storage():  # test_solver.cpp:361-406
    sys = O.OracleSystem.make_lco(6, 2)
    x0 = O.rng_uniform(20, 0, 12, 0.0, 2.0)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
    S = policy_for(PolicyVariant.Single)
    r = O.solve(sys, x0, 0.0, 5.0, S, cfg)
    assert r.status == SolveStatus.Completed
    f = r.final_state
    assert np.array_equal(f.astype(np.float32).astype(np.float64), f)
    xf = x0.astype(np.float32).astype(np.float64)
    k1 = sys.eval_rhs(0.0, xf, S.first_step_k1)
    o = O.bs32_step(sys, 0.0, xf, 0.002, k1, S, cfg)
    assert o.accepted
    assert np.array_equal(o.x_store.astype(np.float32).astype(np.float64), o.x_store)
    assert np.all(np.abs(o.x_store - o.x_next) <= 4.0 * 2.0 ** -23 * (np.abs(o.x_next) + 1.0))
    assert np.array_equal(o.k4, sys.eval_rhs(0.002, o.x_store, S.stage(4)))
    rd = O.solve(sys, x0, 0.0, 5.0, policy_for(PolicyVariant.Double), cfg)
    assert np.any(rd.final_state.astype(np.float32).astype(np.float64) != rd.final_state)


# ---- acceptance criteria touching the hot path (acceptance.cpp) ------------------------
def test_acceptance_c1_order_exp():  # acceptance.cpp:91-115
    cfg = SolverConfig(rel_tol=0.5, abs_tol=0.5)
    prev = 0.0
    for i in range(4):
        h = 0.1 / 2.0 ** i
        o = O.bs32_step(fixture("exp"), 0.0, [1.0], h, [1.0], policy_for(PolicyVariant.Double), cfg)
        err = abs(o.x_next[0] - math.exp(h))
        if i > 0:
            assert 12.0 <= prev / err <= 20.0
        prev = err


def test_acceptance_c11_mean_phase_drift():  # acceptance.cpp:382-411 (one test case, N=100)
    from paper_2605_23727_b200.configs import TWO_PI
    sys = O.OracleSystem.make_kuramoto(100, 0.5, 0.7, 1)
    x0 = O.rng_uniform(1, 1, 100, 0.0, TWO_PI)
    cfg = SolverConfig(rel_tol=1e-8, abs_tol=1e-10)
    r = O.solve(sys, x0, 0.0, 10.0, policy_for(PolicyVariant.Double), cfg)
    assert r.status == SolveStatus.Completed
    drift = abs(r.final_state.mean() - x0.mean() - sys.param(0).mean() * 10.0)
    assert drift <= 1e-5 * 10.0
