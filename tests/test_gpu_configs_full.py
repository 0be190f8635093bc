"""BASELINE.json configs 1-3 at their full sizes, device vs the oracle under the
same policy on the same seeded inputs (slow: the oracle runs with OpenMP over
rows, bitwise its sequential order). Gate: accepted and
rejected counts within 1 % (rejected relative to attempts), final state within
1e-5 of the oracle (weighted like Eq. 7, floor ab/rel).

Two runs that differ in summation order take different step sequences, so
their final states are two solutions of the same problem, each accurate to its
tolerance. Where they differ by more than 1e-5 (loose rtol, oscillators over
long spans), the test checks the property the gate stands for: against a tight
binary64 DP5(4) run (rel = abs = 1e-9, the reference's dp54_reference) the
device's global error is no larger than the oracle's (x1.5 + 1e-7)."""
import os

import numpy as np
import pytest

import _oracle as O
from _gates import gate as _gate
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config1_lco, config2_kuramoto, config3_cc
from paper_2605_23727_b200.systems import DeviceSystem

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(w):
    O.set_threads(os.cpu_count() or 1)
    dev, orc = DeviceSystem(w.spec), O.OracleSystem(w.spec)
    r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
    o = O.solve(orc, w.x0, w.t0, w.tf, w.policy, w.cfg)
    return r, o, dev


@pytest.mark.parametrize("mode", ["fast", "faithful"])
def test_config1_full(gpu, mode):
    w = config1_lco(rhs_mode=mode)
    r, o, dev = _run(w)
    assert o.status == S.SolveStatus.Completed
    _gate(r, o, w.cfg, dev, w)


@pytest.mark.parametrize("rtol", [1e-3, 1e-4])
@pytest.mark.parametrize("ks", ["f32", "f16"])
def test_config2_full(gpu, rtol, ks):
    w = config2_kuramoto(rtol=rtol, k_storage=ks)
    r, o, dev = _run(w)
    assert o.status == S.SolveStatus.Completed
    _gate(r, o, w.cfg, dev, w)

# C3 over its whole span, C2 at rtol 1e-6 / 1e-8 (f32 and f16 K): against the oracle's
# committed whole solves, tests/test_gpu_golden_solves.py.
