"""Dense output on the device (D6 extension; k_dense after each accepted
attempt) against the oracle's restatement of the same interpolant."""
import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config2_kuramoto, rng_uniform
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [PolicyVariant.Double, PolicyVariant.Mixed2, PolicyVariant.Single])
def test_dense_output_bitwise_vs_oracle(gpu, variant):
    spec = SystemSpec("lco", 16, coupling_k=1.0, rhs_mode="faithful")
    dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
    x0 = rng_uniform(31, 1, 32, -1.0, 1.0)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    t_eval = np.concatenate([[0.0, 0.0], np.linspace(0.01, 4.0, 97)])
    pol = policy_for(variant)
    r = S.solve(dev, x0, 0.0, 4.0, pol, cfg, t_eval=t_eval)
    o = O.solve(orc, x0, 0.0, 4.0, pol, cfg, t_eval=t_eval)
    assert r.status == o.status == SolveStatus.Completed
    assert np.array_equal(r.y_eval[-1], r.final_state)
    # bitwise up to the first step where the controller's pow splits the runs
    split = next((k for k, (a, b) in enumerate(zip(r.step_log, o.step_log)) if a.h != b.h), None)
    t_split = r.step_log[split].t if split is not None else np.inf
    for t, a, b in zip(t_eval, r.y_eval, o.y_eval):
        if t > t_split:
            break
        assert np.array_equal(a, b), t


def test_dense_output_kuramoto_and_limits(gpu):
    w = config2_kuramoto(n=512, rtol=1e-6)
    dev = DeviceSystem(w.spec)
    t_eval = np.linspace(0.0, 3.0, 31)
    r = S.solve(dev, w.x0, 0.0, 3.0, w.policy, w.cfg, t_eval=t_eval)
    full = S.solve(dev, w.x0, 0.0, 3.0, w.policy, w.cfg)
    assert np.array_equal(r.final_state, full.final_state) and r.n_accepted == full.n_accepted
    assert np.array_equal(r.y_eval[0], w.x0) and np.array_equal(r.y_eval[-1], r.final_state)
    # interpolated states track a tight solve to the solve's own accuracy
    tight = S.solve(dev, w.x0, 0.0, 3.0, policy_for(PolicyVariant.Double),
                    SolverConfig(rel_tol=1e-10, abs_tol=1e-13, time_limits_enabled=False), t_eval=t_eval)
    assert np.max(np.abs(r.y_eval - tight.y_eval)) < 1e-3
    # a stopped solve fills only the times it reached
    cut = S.solve(dev, w.x0, 0.0, 3.0, w.policy, SolverConfig(rel_tol=1e-6, abs_tol=1e-9, max_iterations=8),
                  t_eval=t_eval)
    done = int(np.sum(t_eval <= cut.t_reached))
    assert np.all(np.isfinite(cut.y_eval[:done])) and np.all(np.isnan(cut.y_eval[done:]))
    with pytest.raises(ValueError):
        S.solve(dev, w.x0, 0.0, 3.0, w.policy, w.cfg, t_eval=[1.0, 0.5])
    with pytest.raises(ValueError):
        S.solve(dev, w.x0, 0.0, 3.0, w.policy, w.cfg, t_eval=[4.0])
