"""The committed whole-solve fixtures (tests/golden/solves/, made by
tools/make_golden_solves.py with the oracle) are what the -m gpu parity tests
compare the device against. Here, without a GPU: every fixture exists, was made
from exactly the inputs the configs build today, is internally consistent with
the reference loop's evaluation budget (solver.cpp:255-306), and the cheapest
one reproduces bit for bit when the oracle is re-run."""
import os

import numpy as np
import pytest

import _oracle as O
import golden_cases as G
from paper_2605_23727_b200.solver import SolveStatus


@pytest.mark.parametrize("name", list(G.CASES))
def test_fixture_matches_inputs_and_budget(name):
    p = G.OUT / f"{name}.npz"
    assert p.exists(), f"run tools/make_golden_solves.py {name}"
    d = G.load(name)
    w = G.CASES[name]["build"]()
    assert d["meta"]["inputs"] == G.input_hash(w)
    acc, rej, ev = (np.atleast_1d(d[k]).astype(np.int64) for k in ("n_accepted", "n_failed", "rhs_evals"))
    assert np.all(np.atleast_1d(d["status"]) == int(SolveStatus.Completed))
    assert np.all(ev == 3 + 3 * acc + 4 * rej)
    assert np.all(np.atleast_1d(d["t_reached"]) == w.tf)
    if "final_state" in d:
        assert d["final_state"].shape == w.x0.shape and np.all(np.isfinite(d["final_state"]))
    else:
        assert d["final_states"].shape == (len(d["sample"]), w.x0.shape[1])


def test_fixture_reproduces_bitwise():
    name = "c2_rtol1e-6_f32"
    d = G.load(name)
    w = G.CASES[name]["build"]()
    O.set_threads(os.cpu_count() or 1)
    o = O.solve(O.OracleSystem(w.spec), w.x0, w.t0, w.tf, w.policy, w.cfg)
    assert (o.n_accepted, o.n_failed, o.flops.rhs_evals) == (int(d["n_accepted"]), int(d["n_failed"]),
                                                            int(d["rhs_evals"]))
    assert np.array_equal(o.final_state, d["final_state"])
    assert np.array_equal(np.array([s.h for s in o.step_log]), d["log_h"])
