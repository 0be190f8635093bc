"""Concurrent policy variants: the harness's four variants
of one case in lock-step, one K sweep per stage for all of them (split
Kuramoto) or back-to-back sweeps (other models). Each variant must equal its
own device solve bit for bit — state, counts, evaluation tallies, step log."""
import os

import numpy as np
import pytest

from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config2_kuramoto, reference_ic
from paper_2605_23727_b200.precision import (B32, B64, DDD, DDS, SSS, PolicyVariant, StagePrecision, custom_policy,
                                             policy_for)
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec, make_cc, make_lco

pytestmark = pytest.mark.gpu
NAMED = [policy_for(v) for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2,
                                 PolicyVariant.Double)]


def _same(a, b):
    assert a.status == b.status
    assert (a.n_accepted, a.n_failed) == (b.n_accepted, b.n_failed)
    assert a.t_reached == b.t_reached
    assert np.array_equal(a.final_state, b.final_state)
    assert (a.flops.rhs_evals, a.flops.low, a.flops.high) == (b.flops.rhs_evals, b.flops.low, b.flops.high)
    assert len(a.step_log) == len(b.step_log)
    for x, y in zip(a.step_log, b.step_log):
        assert (x.t, x.h, x.err, x.accepted) == (y.t, y.h, y.err, y.accepted)


def _check(sys, x0, tf, pols, cfg):
    conc = S.solve_variants(sys, x0, 0.0, tf, pols, cfg)
    for p, r in zip(pols, conc):
        _same(r, S.solve(sys, x0, 0.0, tf, p, cfg))
    return conc


@pytest.mark.parametrize("ks", ["f32", "f16", "bf16"])
def test_kuramoto_fused_sweep_is_bitwise(gpu, ks):
    w = config2_kuramoto(n=512, rtol=1e-5, k_storage=ks)
    sys = DeviceSystem(w.spec)
    r = _check(sys, w.x0, 5.0, NAMED, w.cfg)
    assert all(x.status == SolveStatus.Completed for x in r)


def test_kuramoto_ragged_rows_and_custom_lanes(gpu):
    """N not a multiple of the chunk, and a lane with binary64 G under a
    binary32 sum (the one (SS, GS) pair no named policy uses)."""
    w = config2_kuramoto(n=1000, rtol=1e-5)
    sys = DeviceSystem(w.spec)
    sgd = StagePrecision(B32, B32, B64)
    pols = [custom_policy((sgd, sgd, sgd), sgd, B64), policy_for(PolicyVariant.Double),
            custom_policy((SSS, DDS, DDD), DDD, B32)]
    _check(sys, w.x0, 3.0, pols, w.cfg)


def test_fused_equals_unfused(gpu, monkeypatch):
    w = config2_kuramoto(n=512, rtol=1e-5)
    sys = DeviceSystem(w.spec)
    fused = S.solve_variants(sys, w.x0, 0.0, 4.0, NAMED, w.cfg)
    monkeypatch.setenv("MS_MULTI", "off")
    plain = S.solve_variants(sys, w.x0, 0.0, 4.0, NAMED, w.cfg)
    for a, b in zip(fused, plain):
        _same(a, b)


@pytest.mark.parametrize("model", ["lco", "lco_faithful", "cc"])
def test_other_models_lockstep_is_bitwise(gpu, model):
    if model == "cc":
        sys = make_cc(16, 0.1, 0.228249, 3)
        x0 = reference_ic("cc", 16, 3)
        tf, cfg = 6.0, SolverConfig(rel_tol=1e-5, abs_tol=1e-7)
    else:
        sys = make_lco(12, 0, rhs_mode="faithful" if model == "lco_faithful" else "fast")
        x0 = reference_ic("lco", 12, 5)
        tf, cfg = 4.0, SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
    _check(sys, x0, tf, NAMED, cfg)


def test_subsets_and_limits(gpu):
    w = config2_kuramoto(n=256, rtol=1e-4)
    sys = DeviceSystem(w.spec)
    _check(sys, w.x0, 3.0, NAMED[3:], w.cfg)
    _check(sys, w.x0, 3.0, [NAMED[0], NAMED[0]], w.cfg)
    with pytest.raises(ValueError):
        S.DeviceVariants(sys, 5)
    with pytest.raises(ValueError):
        S.DeviceVariants(sys, 0)
    with pytest.raises(ValueError):
        S.solve_variants(sys, w.x0, 0.0, 1.0, NAMED, SolverConfig(record_snapshots=True))


def test_c2_full_size_four_variants(gpu):
    w = config2_kuramoto()  # N = 4096, K f32
    sys = DeviceSystem(w.spec)
    r = _check(sys, w.x0, w.tf, NAMED, w.cfg)
    assert all(x.status == SolveStatus.Completed for x in r)
