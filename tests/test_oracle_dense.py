"""Dense output (D6 extension, not in the reference: SPEC.md:278 lists it as a
non-goal) in the oracle: the cubic Hermite interpolant of accepted steps.
Checked by its defining properties and against the LCO's analytic solution
(systems.cpp:270-306)."""
import numpy as np

import _oracle as O
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus


def test_dense_output_oracle_properties():
    orc = O.OracleSystem.make_lco(8, 0)
    x0 = O.rng_uniform(3, 1, 16, 0.0, 2.0)
    cfg = SolverConfig(rel_tol=1e-9, abs_tol=1e-11, record_snapshots=True)
    t_eval = np.concatenate([[0.0], np.linspace(0.05, 3.0, 60)])
    r = O.solve(orc, x0, 0.0, 3.0, policy_for(PolicyVariant.Double), cfg, t_eval=t_eval)
    assert r.status == SolveStatus.Completed
    assert np.array_equal(r.y_eval[0], x0)                # t0: the starting state
    assert np.array_equal(r.y_eval[-1], r.final_state)    # t_final: the last step's end, exactly
    # a step boundary is reproduced exactly (theta = 1 of the step ending there)
    tb = np.cumsum([s.h for s in r.snapshots])[3]
    rb = O.solve(orc, x0, 0.0, 3.0, policy_for(PolicyVariant.Double), cfg, t_eval=[tb])
    assert np.array_equal(rb.y_eval[0], r.snapshots[3].x_after)
    # third-order interpolant of a 1e-9-tolerance solve vs the analytic LCO
    for t, y in zip(t_eval, r.y_eval):
        assert np.max(np.abs(y - O.lco_analytic(x0, t))) < 5e-7, t


def test_dense_output_stops_with_the_solve():
    orc = O.OracleSystem.make_lco(4, 0)
    x0 = O.rng_uniform(4, 1, 8, 0.0, 2.0)
    cfg = SolverConfig(rel_tol=1e-8, abs_tol=1e-10, max_iterations=10)
    t_eval = np.linspace(0.0, 5.0, 11)
    r = O.solve(orc, x0, 0.0, 5.0, policy_for(PolicyVariant.Double), cfg, t_eval=t_eval)
    assert r.status == SolveStatus.MaxIterations
    done = int(np.sum(t_eval <= r.t_reached))
    assert np.all(np.isfinite(r.y_eval[:done])) and np.all(np.isnan(r.y_eval[done:]))
