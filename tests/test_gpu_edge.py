"""Edge sizes through every device path: N = 1, 2, 3 and a prime N, tiny and
single-trajectory ensembles, concurrent variants and dense output on them —
each against the oracle (bitwise where the path is transcendental-free)."""
import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.batch import DeviceBatch
from paper_2605_23727_b200.configs import TWO_PI, rng_normal, rng_uniform
from paper_2605_23727_b200.precision import B32, B64, DDD, DDS, SSS, PolicyVariant, StagePrecision, policy_for
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec, cc_parameters

pytestmark = pytest.mark.gpu
ROWS = [SSS, DDS, DDD]


def _spec(model, n, ks, mode):
    kw = dict(k_storage=ks, rhs_mode=mode, coupling_k=0.7)
    if ks != "scalar":
        kw["k_uniform"] = (3, 2, 0.0, 2.0)
    if model == "kuramoto":
        return SystemSpec("kuramoto", n, omega=rng_normal(2, 0, n), **kw)
    if model == "cc":
        k1, th = cc_parameters(n, 2)
        return SystemSpec("cc", n, cc_k1=k1, cc_theta_h=th, stimulus_i0=0.2, **kw)
    return SystemSpec("lco", n, **kw)


def _x(model, n):
    if model == "cc":
        u = rng_uniform(5, 1, 4 * n, 0.0, 1.0).reshape(n, 4)
        return (np.array([1.0, 1.0, -1.19, -0.62]) + 0.2 * (u - 0.5)).reshape(-1)
    d = 2 if model == "lco" else 1
    return rng_uniform(5, 1, d * n, 0.0, TWO_PI if model == "kuramoto" else 1.0)


@pytest.mark.parametrize("n", [1, 2, 3, 37])
@pytest.mark.parametrize("model", ["lco", "kuramoto", "cc"])
@pytest.mark.parametrize("ks", ["scalar", "f32", "f16"])
@pytest.mark.parametrize("mode", ["fast", "faithful"])
def test_tiny_systems_rhs_and_solve(gpu, n, model, ks, mode):
    spec = _spec(model, n, ks, mode)
    dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
    x = _x(model, n)
    for sp in ROWS:
        a, b = dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp)
        scale = np.maximum(np.abs(b), 1.0)
        eps = 2.0 ** -23 if sp.sum_prec == B32 or sp.g_prec == B32 else 2.0 ** -52
        assert np.all(np.abs(a - b) <= 64 * eps * scale), (sp, float(np.max(np.abs(a - b) / scale)))
        if model == "lco" and mode == "faithful":
            assert np.array_equal(a, b)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    tf = 1.0 if model != "cc" else 3.0
    r = S.solve(dev, x, 0.0, tf, policy_for(PolicyVariant.Double), cfg, t_eval=[0.0, 0.5 * tf, tf])
    o = O.solve(orc, x, 0.0, tf, policy_for(PolicyVariant.Double), cfg)
    assert r.status == o.status == SolveStatus.Completed
    assert abs(r.n_accepted - o.n_accepted) <= 1
    assert np.allclose(r.final_state, o.final_state, rtol=1e-6, atol=1e-8)
    assert np.array_equal(r.y_eval[-1], r.final_state) and np.array_equal(r.y_eval[0], x)
    # the four named variants concurrently equal their own solves
    pols = [policy_for(v) for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2,
                                    PolicyVariant.Double)]
    for p, c in zip(pols, S.solve_variants(dev, x, 0.0, tf, pols, cfg)):
        s_ = S.solve(dev, x, 0.0, tf, p, cfg)
        assert np.array_equal(c.final_state, s_.final_state) and c.n_accepted == s_.n_accepted


@pytest.mark.parametrize("shape", [(1, 1), (1, 8), (2, 3), (1, 300), (3, 129)])
@pytest.mark.parametrize("tc", [False, True])
def test_tiny_ensembles(gpu, shape, tc):
    B, n = shape
    spec = SystemSpec("kuramoto", n, k_storage="bf16", omega=np.zeros(n), k_uniform=(4, 2, 0.0, 2.0))
    omega = rng_normal(4, 0, B * n).reshape(B, n)
    x = rng_uniform(4, 1, B * n, 0.0, TWO_PI).reshape(B, n)
    dev = DeviceSystem(spec)
    bat = DeviceBatch(dev, omega, tensor_cores=tc)
    got = bat.eval_rhs(x, SSS)
    orc = O.OracleSystem(spec)
    if tc:
        orc.set_op_round(_abi.MS_K_BF16)
    for b in range(B):
        orc.set_omega(omega[b])
        ref = orc.eval_rhs(0.0, x[b], SSS)
        assert np.all(np.abs(got[b] - ref) <= 1e-4 * (1.0 + np.abs(ref))), b
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    res = bat.solve(x, 0.0, 0.5, policy_for(PolicyVariant.Single), cfg)
    assert all(s == SolveStatus.Completed for s in res.status)
    assert np.all(np.isfinite(res.final_state))


@pytest.mark.parametrize("model", ["lco", "kuramoto", "cc"])
def test_non_finite_inputs_end_as_nonfinite(gpu, model):
    """A NaN in x0 (initial_step returns NaN, solver.cpp:426) and an infinite
    K entry (the first stage goes non-finite) end the solve with NonFinite,
    as in the oracle."""
    n = 16
    spec = _spec(model, n, "f32", "fast")
    dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
    x = _x(model, n)
    x[3] = np.nan
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    pol = policy_for(PolicyVariant.Mixed2)
    r = S.solve(dev, x, 0.0, 1.0, pol, cfg)
    o = O.solve(orc, x, 0.0, 1.0, pol, cfg)
    assert r.status == o.status == SolveStatus.NonFinite
    k = np.full((n, n), 0.5)
    k[2, 5] = np.inf
    spec_k = SystemSpec(**{**spec.__dict__, "k_uniform": None, "K": k})
    devk, orck = DeviceSystem(spec_k), O.OracleSystem(spec_k)
    xk = _x(model, n)
    r = S.solve(devk, xk, 0.0, 1.0, pol, cfg)
    o = O.solve(orck, xk, 0.0, 1.0, pol, cfg)
    assert r.status == o.status == SolveStatus.NonFinite
    assert r.n_accepted == o.n_accepted


def test_batch_trajectories_fail_independently(gpu):
    """One trajectory with a NaN start ends NonFinite; the others complete
    exactly as a clean ensemble of the same trajectories does."""
    B, n = 4, 64
    spec = SystemSpec("kuramoto", n, k_storage="f32", omega=np.zeros(n), k_uniform=(4, 2, 0.0, 2.0))
    omega = rng_normal(4, 0, B * n).reshape(B, n)
    x = rng_uniform(4, 1, B * n, 0.0, TWO_PI).reshape(B, n)
    dev = DeviceSystem(spec)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    clean = DeviceBatch(dev, omega, tensor_cores=False).solve(x, 0.0, 1.0, policy_for(PolicyVariant.Mixed2), cfg)
    bad = x.copy()
    bad[2, 7] = np.nan
    res = DeviceBatch(dev, omega, tensor_cores=False).solve(bad, 0.0, 1.0, policy_for(PolicyVariant.Mixed2), cfg)
    assert res.status[2] == SolveStatus.NonFinite
    for b in (0, 1, 3):
        assert res.status[b] == SolveStatus.Completed
        assert res.n_accepted[b] == clean.n_accepted[b] and np.array_equal(res.final_state[b], clean.final_state[b])


def test_interleaved_api_use_leaves_no_state_behind(gpu):
    """One handle driven through every entry point in turn (eval_rhs, bs32_step,
    solves under different policies with and without logs/snapshots/dense
    output, concurrent variants, DP5(4)) gives the same answers as fresh
    handles: no workspace, graph or control-block state leaks between calls."""
    from paper_2605_23727_b200.configs import config2_kuramoto
    w = config2_kuramoto(n=300, rtol=1e-6)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    pols = [policy_for(v) for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2,
                                    PolicyVariant.Double)]

    def fresh(fn):
        d = DeviceSystem(w.spec)
        out = fn(d)
        d.close()
        return out

    shared = DeviceSystem(w.spec)
    calls = [
        lambda d: d.eval_rhs(0.0, w.x0, DDS),
        lambda d: S.solve(d, w.x0, 0.0, 2.0, pols[0], cfg).final_state,
        lambda d: S.bs32_step(d, 0.0, w.x0, 1e-3, d.eval_rhs(0.0, w.x0, SSS), pols[0], cfg).x_next,
        lambda d: S.solve(d, w.x0, 0.0, 2.0, pols[3], SolverConfig(**{**cfg.__dict__, "record_snapshots": True}),
                          t_eval=[0.5, 1.5]).y_eval,
        lambda d: np.stack([r.final_state for r in S.solve_variants(d, w.x0, 0.0, 1.0, pols, cfg)]),
        lambda d: S.solve(d, w.x0, 0.0, 2.0, pols[2], cfg, log_capacity=3).final_state,
        lambda d: S.dp54_reference(d, w.x0, 0.0, 0.5, cfg).final_state,
        lambda d: S.solve(d, w.x0, 0.0, 2.0, pols[0], cfg).final_state,
    ]
    for k, fn in enumerate(calls):
        assert np.array_equal(fn(shared), fresh(fn)), k
