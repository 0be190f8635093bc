"""Batched ensembles sharing one K (config C5) against per-trajectory oracle
systems (same K, own omega_b), through the ms_batch_* C-ABI.

CUDA-core rows sum each (i, b) in ascending j — the oracle's split order — so
they agree up to the libm ulp of sin/cos. Tensor-core rows (binary32, K in
f16/bf16) use operands rounded to K's format with exact products and the
tensor core's fp32 accumulation: the oracle applies the same operand rounding
(op_round) and the reordering bound TOL = 2 N eps32 mw sum_j |K_ij| is used."""
import itertools

import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200.batch import DeviceBatch
from paper_2605_23727_b200.configs import TWO_PI, config5_batch, rng_normal, rng_uniform
from paper_2605_23727_b200.precision import B32, B64, DDD, DDS, SSS, StagePrecision
from paper_2605_23727_b200.solver import SolveStatus
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec

pytestmark = pytest.mark.gpu
ROWS = [StagePrecision(f, s, g) for f, s, g in itertools.product((B32, B64), repeat=3)]
OPR = {"bf16": _abi.MS_K_BF16, "f16": _abi.MS_K_F16}


def _ensemble(B, n, ks, seed=5):
    spec = SystemSpec("kuramoto", n, k_storage=ks, omega=np.zeros(n), k_uniform=(seed, 2, 0.0, 2.0))
    omega = rng_normal(seed, 0, B * n).reshape(B, n)
    x = rng_uniform(seed, 1, B * n, 0.0, TWO_PI).reshape(B, n)
    return spec, omega, x


def _tol(sp, n, out, kabs_rowsum):
    eps = lambda f: 2.0 ** -23 if f == B32 else 2.0 ** -52
    ws = B32 if (sp.f_prec == B32 and sp.sum_prec == B32) else B64
    return 2.0 * n * eps(sp.sum_prec) * kabs_rowsum / n * 2.0 + 4.0 * eps(B32) * kabs_rowsum / n \
        + 4.0 * eps(ws) * np.abs(out) + 1e-300


@pytest.mark.parametrize("sp", ROWS, ids=str)
def test_batch_rhs_cuda_core(gpu, sp):
    spec, omega, x = _ensemble(5, 203, "f32")
    dev = DeviceSystem(spec)
    bat = DeviceBatch(dev, omega, tensor_cores=False)
    got = bat.eval_rhs(x, sp)
    orc = O.OracleSystem(spec)
    ks = np.abs(orc.get_k()).sum(axis=1)
    for b in range(5):
        orc.set_omega(omega[b])
        ref = orc.eval_rhs(0.0, x[b], sp)
        assert np.all(np.abs(got[b] - ref) <= _tol(sp, 203, ref, ks)), b


@pytest.mark.parametrize("ks", ["bf16", "f16"])
@pytest.mark.parametrize("shape", [(160, 300), (64, 128), (7, 1000)])
def test_batch_rhs_tensor_cores(gpu, ks, shape):
    B, n = shape
    spec, omega, x = _ensemble(B, n, ks)
    dev = DeviceSystem(spec)
    bat = DeviceBatch(dev, omega, tensor_cores=True)
    orc = O.OracleSystem(spec)
    kabs = np.abs(orc.get_k()).sum(axis=1)
    got = bat.eval_rhs(x, SSS)
    orc.set_op_round(OPR[ks])
    picks = sorted({0, 1, B // 2, B - 1})
    for b in picks:
        orc.set_omega(omega[b])
        ref = orc.eval_rhs(0.0, x[b], SSS)
        err = np.abs(got[b] - ref)
        tol = _tol(SSS, n, ref, kabs)
        assert np.all(err <= tol), (b, float(np.max(err / tol)))
    # binary64 rows of the same ensemble stay exact on CUDA cores
    got64 = bat.eval_rhs(x, DDD)
    orc.set_op_round(0)
    for b in picks[:2]:
        orc.set_omega(omega[b])
        ref = orc.eval_rhs(0.0, x[b], DDD)
        assert np.all(np.abs(got64[b] - ref) <= _tol(DDD, n, ref, kabs))


def test_batch_tensor_cores_full_c5_shape(gpu):
    """The C5 shape (B = 1024, N = 2048): whole GEMM tiles, spot-checked rows."""
    w = config5_batch()
    dev = DeviceSystem(w.spec)
    bat = DeviceBatch(dev, w.omega, tensor_cores=True)
    got = bat.eval_rhs(w.x0, SSS)
    assert np.all(np.isfinite(got))
    orc = O.OracleSystem(w.spec)
    orc.set_op_round(_abi.MS_K_BF16)
    kabs = np.abs(orc.get_k()).sum(axis=1)
    for b in (0, 511, 1023):
        orc.set_omega(w.omega[b])
        ref = orc.eval_rhs(0.0, w.x0[b], SSS)
        assert np.all(np.abs(got[b] - ref) <= _tol(SSS, 2048, ref, kabs)), b


@pytest.mark.parametrize("tc", [False, True])
def test_batch_solve_vs_oracle(gpu, tc):
    B, n = 6, 128
    spec, omega, x0 = _ensemble(B, n, "bf16", seed=9)
    from paper_2605_23727_b200.configs import SSS_D
    from paper_2605_23727_b200.solver import SolverConfig
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    dev = DeviceSystem(spec)
    bat = DeviceBatch(dev, omega, tensor_cores=tc)
    res = bat.solve(x0, 0.0, 4.0, SSS_D, cfg)
    orc = O.OracleSystem(spec)
    if tc:
        orc.set_op_round(_abi.MS_K_BF16)
    O.set_threads(4)
    tot = {"dev_rej": 0, "orc_rej": 0, "att": 0}
    for b in range(B):
        orc.set_omega(omega[b])
        o = O.solve(orc, x0[b], 0.0, 4.0, SSS_D, cfg)
        assert res.status[b] == o.status == SolveStatus.Completed
        att = o.n_accepted + o.n_failed
        # near-threshold accept/reject decisions flip on ulp-level differences;
        # per trajectory within 3 % of the attempts, over the ensemble within 1 %
        assert abs(res.n_accepted[b] - o.n_accepted) <= max(2, 0.03 * o.n_accepted), b
        assert abs(res.n_failed[b] - o.n_failed) <= max(4, 0.05 * att), b
        tot["dev_acc"] = tot.get("dev_acc", 0) + int(res.n_accepted[b])
        tot["orc_acc"] = tot.get("orc_acc", 0) + o.n_accepted
        tot["dev_rej"] += int(res.n_failed[b])
        tot["orc_rej"] += o.n_failed
        tot["att"] += att
        assert res.t_reached[b] == o.t_reached
        scale = np.maximum(np.abs(o.final_state), 1e-3)
        # the tensor core sums each window of the contraction in its own order
        # (ms_gemm_tc.cuh, MS_T2_DRAIN), not the oracle's sequential one; the
        # full-size ensemble's accuracy is gated against DP5(4) in
        # tests/test_gpu_golden_solves.py
        tol = 3e-5 if tc else 1e-5
        assert np.all(np.abs(res.final_state[b] - o.final_state) <= tol * scale), b
        # evaluation budget of the reference loop: 2 (initial_step) + 1 (cold k1)
        # + 3 per accepted + 4 per rejected attempt (solver.cpp:255-306)
        assert res.rhs_evals[b] == 3 + 3 * res.n_accepted[b] + 4 * res.n_failed[b]
        assert o.flops.rhs_evals == 3 + 3 * o.n_accepted + 4 * o.n_failed
    print("ensemble counts dev/oracle:", tot)
    assert abs(tot["dev_rej"] - tot["orc_rej"]) <= max(2, 0.02 * tot["att"])
    assert abs(tot["dev_acc"] - tot["orc_acc"]) <= max(2, 0.01 * tot["orc_acc"])
    assert res.attempts >= int(max(res.n_accepted + res.n_failed))


@pytest.mark.parametrize("ks", ["bf16", "f16"])
@pytest.mark.parametrize("pol", ["SSS_D", "Single", "Mixed1"])
def test_batch_tc_specialised_prep_is_bitwise(gpu, monkeypatch, ks, pol):
    """The tensor-core path's specialised stage prep (kb_prep_tc) against the
    generic kb_prep (MS_PREP_TC=0): identical ensembles, bit for bit."""
    from paper_2605_23727_b200.configs import SSS_D
    from paper_2605_23727_b200.precision import PolicyVariant, policy_for
    from paper_2605_23727_b200.solver import SolverConfig
    B, n = 40, 256
    spec, omega, x0 = _ensemble(B, n, ks, seed=11)
    policy = SSS_D if pol == "SSS_D" else policy_for(getattr(PolicyVariant, pol))
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    dev = DeviceSystem(spec)
    runs = []
    for mode in ("generic", "specialised"):
        if mode == "generic":
            monkeypatch.setenv("MS_PREP_TC", "0")
        else:
            monkeypatch.delenv("MS_PREP_TC", raising=False)
        runs.append(DeviceBatch(dev, omega, tensor_cores=True).solve(x0, 0.0, 3.0, policy, cfg))
    a, b = runs
    assert list(a.status) == list(b.status)
    assert np.array_equal(a.n_accepted, b.n_accepted) and np.array_equal(a.n_failed, b.n_failed)
    assert np.array_equal(a.rhs_evals, b.rhs_evals)
    assert np.array_equal(a.final_state, b.final_state)
    assert np.array_equal(a.t_reached, b.t_reached)


@pytest.mark.parametrize("tc", [True, False])
@pytest.mark.parametrize("pol", ["SSS_D", "Single", "Mixed2"])
def test_batch_finalize_partial_sum_is_bitwise(gpu, monkeypatch, tc, pol):
    """The last stage prep hands the finalize P = b~1 k1 + b~2 k2 + b~3 k3 (the
    first three terms of x_tilde's sum, same order): ensembles with and without
    it (MS_BFIN_P=off) must agree bit for bit, on the tensor-core and the
    CUDA-core paths."""
    from paper_2605_23727_b200.configs import SSS_D
    from paper_2605_23727_b200.precision import PolicyVariant, policy_for
    from paper_2605_23727_b200.solver import SolverConfig
    B, n = 40, 256
    spec, omega, x0 = _ensemble(B, n, "bf16", seed=12)
    policy = SSS_D if pol == "SSS_D" else policy_for(getattr(PolicyVariant, pol))
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    dev = DeviceSystem(spec)
    runs = []
    for mode in ("on", "off"):
        monkeypatch.setenv("MS_BFIN_P", mode)
        runs.append(DeviceBatch(dev, omega, tensor_cores=tc).solve(x0, 0.0, 3.0, policy, cfg))
    a, b = runs
    assert list(a.status) == list(b.status)
    assert np.array_equal(a.n_accepted, b.n_accepted) and np.array_equal(a.n_failed, b.n_failed)
    assert np.array_equal(a.final_state, b.final_state)
    assert np.array_equal(a.t_reached, b.t_reached)


@pytest.mark.parametrize("tc", [True, False])
def test_batch_controller_on_shared_copy_is_bitwise(gpu, monkeypatch, tc):
    """kb_finalize runs each trajectory's controller on a shared-memory copy of
    Ctl[b] (MS_CTL_SMEM): ensembles with the controller in place must agree
    bit for bit (statuses, counts, final states, t_reached)."""
    from paper_2605_23727_b200.configs import SSS_D
    from paper_2605_23727_b200.solver import SolverConfig
    B, n = 37, 256
    spec, omega, x0 = _ensemble(B, n, "bf16", seed=13)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    dev = DeviceSystem(spec)
    runs = []
    for mode in ("on", "off"):
        monkeypatch.setenv("MS_CTL_SMEM", mode)
        runs.append(DeviceBatch(dev, omega, tensor_cores=tc).solve(x0, 0.0, 3.0, SSS_D, cfg))
    a, b = runs
    assert list(a.status) == list(b.status)
    assert np.array_equal(a.n_accepted, b.n_accepted) and np.array_equal(a.n_failed, b.n_failed)
    assert np.array_equal(a.rhs_evals, b.rhs_evals)
    assert np.array_equal(a.final_state, b.final_state)
    assert np.array_equal(a.t_reached, b.t_reached)


@pytest.mark.parametrize("tc", [True, False])
@pytest.mark.parametrize("pol", ["SSS_D", "Single", "Mixed2"])
def test_batch_finalize_max_without_division_is_bitwise(gpu, monkeypatch, tc, pol):
    """kb_finalize's weighted max-norm (solver.cpp:403-408) as RN of the largest
    exact quotient (ms_kernels.cuh QuotMax: candidates compared as product +
    FMA remainder, one division per thread) against a division per element
    (MS_BFIN_QUOT=off): identical ensembles, bit for bit."""
    from paper_2605_23727_b200.configs import SSS_D
    from paper_2605_23727_b200.precision import PolicyVariant, policy_for
    from paper_2605_23727_b200.solver import SolverConfig
    B, n = 48, 320
    spec, omega, x0 = _ensemble(B, n, "bf16", seed=15)
    policy = SSS_D if pol == "SSS_D" else policy_for(getattr(PolicyVariant, pol))
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    dev = DeviceSystem(spec)
    runs = []
    for mode in ("on", "off"):
        monkeypatch.setenv("MS_BFIN_QUOT", mode)
        runs.append(DeviceBatch(dev, omega, tensor_cores=tc).solve(x0, 0.0, 3.0, policy, cfg))
    a, b = runs
    assert list(a.status) == list(b.status)
    assert np.array_equal(a.n_accepted, b.n_accepted) and np.array_equal(a.n_failed, b.n_failed)
    assert np.array_equal(a.final_state, b.final_state)
    assert np.array_equal(a.t_reached, b.t_reached)
