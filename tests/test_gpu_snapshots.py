"""StepSnapshots recorded by the device loop (solver.cpp:324-327) and the host
error metrics over them, against the reference's tests (test_solver.cpp:361-422,
test_metrics.cpp:150-172) and bitwise against the oracle."""
import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200 import metrics as M
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import rng_uniform
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import make_lco

pytestmark = pytest.mark.gpu


def identical_lco_state(n, x, v):  # test_solver.cpp:20-27
    s = np.empty(2 * n)
    s[0::2], s[1::2] = x, v
    return s


def test_snapshots_capture_accepted_steps(gpu):  # test_solver.cpp:408-422
    sys = make_lco(3)
    x0 = identical_lco_state(3, 1.0, 0.5)
    cfg = SolverConfig(rel_tol=1e-4, abs_tol=1e-6, record_snapshots=True)
    r = S.solve(sys, x0, 0.0, 3.0, policy_for(PolicyVariant.Double), cfg)
    assert r.status == SolveStatus.Completed
    assert len(r.snapshots) == r.snapshot_count == r.n_accepted
    assert np.array_equal(r.snapshots[0].x_before, x0)
    assert np.array_equal(r.snapshots[-1].x_after, r.final_state)
    assert sum(s.h for s in r.snapshots) == pytest.approx(3.0, rel=1e-12)
    for a, b in zip(r.snapshots, r.snapshots[1:]):
        assert np.array_equal(a.x_after, b.x_before)
    # accepted records of the step log carry the same h
    acc = [e.h for e in r.step_log if e.accepted]
    assert acc == [s.h for s in r.snapshots]


def test_single_policy_snapshots_are_binary32(gpu):  # test_solver.cpp:361-380
    sys = make_lco(6)
    x0 = rng_uniform(20, 0, 12, 0.0, 2.0)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-8, record_snapshots=True)
    r = S.solve(sys, x0, 0.0, 5.0, policy_for(PolicyVariant.Single), cfg)
    assert r.status == SolveStatus.Completed
    assert len(r.snapshots) == r.n_accepted
    # the first x_before is x0 rounded to binary32 (solver.cpp:263)
    assert np.array_equal(r.snapshots[0].x_before, x0.astype(np.float32).astype(np.float64))
    for s in r.snapshots:
        assert np.array_equal(s.x_after.astype(np.float32).astype(np.float64), s.x_after)


@pytest.mark.parametrize("variant", [PolicyVariant.Double, PolicyVariant.Mixed2, PolicyVariant.Single])
def test_snapshots_bitwise_vs_oracle(gpu, variant):
    """The faithful LCO sweep is transcendental-free: the device run is the
    oracle's run bit for bit, snapshots included."""
    from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec
    spec = SystemSpec("lco", 16, coupling_k=1.0, rhs_mode="faithful")
    dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
    x0 = rng_uniform(31, 1, 32, -1.0, 1.0)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, record_snapshots=True, time_limits_enabled=False)
    pol = policy_for(variant)
    r = S.solve(dev, x0, 0.0, 4.0, pol, cfg)
    o = O.solve(orc, x0, 0.0, 4.0, pol, cfg)
    assert r.status == o.status == SolveStatus.Completed
    assert len(r.snapshots) == r.n_accepted and len(o.snapshots) == o.n_accepted
    # bitwise until the controller's pow (device: correctly rounded; glibc:
    # ~0.1 % of calls 1 ulp off) first picks a different h, then stop
    for a, b in zip(r.snapshots, o.snapshots):
        assert np.array_equal(a.x_before, b.x_before)
        if a.h != b.h:
            assert abs(a.h - b.h) <= 4 * np.spacing(b.h)
            break
        assert np.array_equal(a.x_after, b.x_after)
    else:
        assert r.n_accepted == o.n_accepted


def test_snapshot_capacity_truncates(gpu):
    sys = make_lco(3)
    x0 = identical_lco_state(3, 1.0, 0.5)
    cfg = SolverConfig(rel_tol=1e-4, abs_tol=1e-6, record_snapshots=True)
    full = S.solve(sys, x0, 0.0, 3.0, policy_for(PolicyVariant.Double), cfg)
    r = S.solve(sys, x0, 0.0, 3.0, policy_for(PolicyVariant.Double), cfg, snapshot_capacity=3)
    assert r.snapshot_count == r.n_accepted > 3
    assert len(r.snapshots) == 3
    for a, b in zip(r.snapshots, full.snapshots):
        assert np.array_equal(a.x_after, b.x_after) and a.h == b.h
    # no snapshots when not asked for, and the loop is unchanged
    off = S.solve(sys, x0, 0.0, 3.0, policy_for(PolicyVariant.Double), SolverConfig(rel_tol=1e-4, abs_tol=1e-6))
    assert off.snapshots == [] and off.snapshot_count == 0
    assert np.array_equal(off.final_state, full.final_state) and off.n_accepted == full.n_accepted


def test_error_report_aggregation(gpu):  # test_metrics.cpp:150-172
    sys = make_lco(4)
    x0 = rng_uniform(50, 0, 8, 0.0, 2.0)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-8, record_snapshots=True)
    run = S.solve(sys, x0, 0.0, 4.0, policy_for(PolicyVariant.Double), cfg)
    ref = S.dp54_reference(sys, x0, 0.0, 4.0, cfg)
    assert run.status == ref.status == SolveStatus.Completed
    er = M.error_report(run, ref.final_state, 4, cfg.abs_tol, cfg.rel_tol)
    assert er.normalized_final_error == M.normalized_final_error(ref.final_state, run.final_state, 4)
    assert 0.0 < er.mean_e_bs <= cfg.rel_tol
    assert er.mean_e_analytic is not None and er.mean_e_analytic < cfg.rel_tol


def test_batch_rejects_snapshots(gpu):
    from paper_2605_23727_b200.batch import DeviceBatch
    from paper_2605_23727_b200.configs import config5_batch
    from paper_2605_23727_b200.systems import DeviceSystem
    w = config5_batch(batch=2, n=64)
    b = DeviceBatch(DeviceSystem(w.spec), w.omega, tensor_cores=False)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, record_snapshots=True)
    with pytest.raises(ValueError):
        b.solve(w.x0, 0.0, 0.1, w.policy, cfg)
