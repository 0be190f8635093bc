"""Seeded workload builders (BASELINE.json configs)."""
import numpy as np

import _oracle as O
from paper_2605_23727_b200.configs import (TWO_PI, config1_lco, config2_kuramoto, config3_cc, config4_kuramoto,
                                           reference_ic, rng_normal, rng_uniform)
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import SystemSpec


def test_config1_shapes_and_distributions():
    w = config1_lco(n=128)
    K = w.spec.K
    assert K.shape == (128, 128) and np.array_equal(K, K.T) and np.all(np.diag(K) == 0)
    assert abs(K[np.triu_indices(128, 1)].std() - 1.0) < 0.05
    assert np.all((w.spec.w2 >= 0.25) & (w.spec.w2 < 2.25))
    assert w.x0.size == 256 and np.all(np.abs(w.x0) <= 1.0)
    assert w.spec.coupled_slot == 1 and w.tf == 10.0


def test_kuramoto_configs():
    w = config2_kuramoto(n=4096)
    assert w.tf == 50.0 and w.cfg.abs_tol == w.cfg.rel_tol * 1e-3
    assert np.all((w.x0 >= 0) & (w.x0 < TWO_PI))
    assert abs(w.spec.omega.std() - 1.0) < 0.05
    assert w.spec.k_uniform == (1, 2, 0.0, 2.0)
    w4 = config4_kuramoto(n=32)
    assert w4.tf == 20.0 and w4.cfg.rel_tol == 1e-6 and w4.cfg.abs_tol == 1e-9
    # omega is make_kuramoto's draw (systems.cpp:230-231): sigma * normal(), stream 0
    assert np.array_equal(w4.spec.omega, O.OracleSystem.make_kuramoto(32, 1.0, 1.0, 3).param(0))


def test_reference_ic_matches_harness():  # harness.cpp:305-330
    x = reference_ic("lco", 5, 9)
    assert np.array_equal(x, 2.0 * O.rng_uniform(9, 1, 10, 0.0, 1.0))
    c = reference_ic("cc", 3, 4).reshape(3, 4)
    u = O.rng_uniform(4, 1, 12, 0.0, 1.0).reshape(3, 4)
    assert np.array_equal(c, np.array([1.0, 1.0, -1.19, -0.62]) + 0.2 * (u - 0.5))


def test_cc_baseline_ic_blows_up_in_the_reference_model():
    """Why C3 uses the reference IC: from x0 ~ U(0,1) (BASELINE.json) the
    reference CC model's Goodwin variable explodes (oracle, all-binary64)."""
    w = config3_cc(n=128)
    orc = O.OracleSystem(w.spec)
    x0 = rng_uniform(2, 1, 4 * 128, 0.0, 1.0)
    r = O.solve(orc, x0, 0.0, 2.0, policy_for(PolicyVariant.Double), w.cfg)
    assert np.max(np.abs(r.final_state)) > 1e6 or r.status != SolveStatus.Completed
    r2 = O.solve(orc, w.x0, 0.0, 2.0, policy_for(PolicyVariant.Double), w.cfg)
    assert r2.status == SolveStatus.Completed and np.max(np.abs(r2.final_state)) < 1e3
