"""The f16-K tensor-core sweep (MS_SWEEP=tc16, csrc/ms_gemv_tc.cuh) against the
CPU oracle and against itself.

It evaluates the split Kuramoto coupling (systems.cpp:141-143) with the
column values as f16 hi + lo (~22 bits; products with f16 K are exact), each
16-column dot product formed by one MMA from a zero accumulator and the dot
products summed in binary32 in ascending column order. That is not the oracle's
order, so the RHS is held to the reordering bound of tests/test_gpu_rhs.py
(plus the operand split's 2^-22 relative error per term) and whole solves to
the gate of the other fp16 runs (tests/_gates.py). Its order depends only on
N: a row-range handle reproduces the whole handle's rows bit for bit."""
from types import SimpleNamespace

import numpy as np
import pytest

import golden_cases as G
import _oracle as O
from _gates import gate
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import TWO_PI, rng_uniform
from paper_2605_23727_b200.precision import B32, StagePrecision
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec

pytestmark = pytest.mark.gpu

SSS = StagePrecision(B32, B32, B32)


def kur_spec(n, seed=11, coupling_k=1.0):
    om = rng_uniform(seed, 0, n, -1.0, 1.0)
    return SystemSpec("kuramoto", n, k_storage="f16", omega=om, coupling_k=coupling_k, k_uniform=(seed, 2, 0.0, 2.0))


@pytest.mark.parametrize("n", [256, 512, 4096, 4352, 8960])
def test_tc16_rhs_vs_oracle(gpu, n, monkeypatch):
    monkeypatch.setenv("MS_SWEEP", "tc16")
    spec = kur_spec(n)
    dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
    x = rng_uniform(6, 1, n, 0.0, 50.0)
    a, b = dev.eval_rhs(0.0, x, SSS), orc.eval_rhs(0.0, x, SSS)
    gsum = np.abs(orc.get_k()).sum(axis=1)
    eps = 2.0 ** -23
    # reordering a binary32 sum + binary32 products (test_gpu_rhs.reorder_tol) + the operand split
    tol = (2.0 * n * eps + 8.0 * eps) * gsum / n + 4.0 * eps * np.abs(b) + 1e-300
    r = np.abs(a - b) / tol
    print(f"n={n}: max |dev - oracle| / tol = {float(r.max()):.3f}, max abs {float(np.max(np.abs(a - b))):.3e}")
    assert np.all(r <= 1.0)
    # and it is a different evaluation from the CUDA-core sweep (the switch is live)
    monkeypatch.setenv("MS_SWEEP", "ldg")
    c = dev.eval_rhs(0.0, x, SSS)
    assert not np.array_equal(a, c)
    dev.close()


def test_tc16_row_shards_bitwise(gpu, monkeypatch):
    """Row-range handles (ranks of a row-sharded K, tiles not aligned to the
    128-row MMA tile) give the whole handle's rows bit for bit."""
    monkeypatch.setenv("MS_SWEEP", "tc16")
    n = 4352
    full = DeviceSystem(kur_spec(n))
    x = rng_uniform(8, 1, n, 0.0, TWO_PI)
    ref = full.eval_rhs(0.0, x, SSS)
    for r0, r1 in ((0, 1000), (1000, 1001), (1001, 4352)):
        spec = kur_spec(n)
        spec.row_begin, spec.row_end = r0, r1
        part = DeviceSystem(spec)
        got = part.eval_rhs(0.0, x, SSS)
        assert np.array_equal(got[r0:r1], ref[r0:r1]), (r0, r1)
        part.close()
    full.close()


def test_tc16_repeatable(gpu, monkeypatch):
    """The chunk tickets reset themselves: repeated evaluations (and a solve's
    thousands of launches) are bitwise identical."""
    monkeypatch.setenv("MS_SWEEP", "tc16")
    n = 4096
    dev = DeviceSystem(kur_spec(n))
    x = rng_uniform(9, 1, n, 0.0, TWO_PI)
    first = dev.eval_rhs(0.0, x, SSS)
    for _ in range(5):
        assert np.array_equal(dev.eval_rhs(0.0, x, SSS), first)
    dev.close()


@pytest.mark.slow
def test_tc16_c4_whole_solve_vs_oracle(gpu, monkeypatch):
    """C4 (Kuramoto N=32768, K f16, SSS rows, rtol 1e-6) through the tensor-core
    sweep against the oracle's whole solve with the same f16 K (fixture c4_f16):
    the gate of every other fp16 run."""
    monkeypatch.setenv("MS_SWEEP", "tc16")
    name = "c4_f16"
    w = G.CASES[name]["build"]()
    d = G.load(name)
    assert G.input_hash(w) == d["meta"]["inputs"]
    o = SimpleNamespace(status=S.SolveStatus(int(d["status"])), n_accepted=int(d["n_accepted"]),
                        n_failed=int(d["n_failed"]), final_state=d["final_state"], t_reached=float(d["t_reached"]))
    dev = DeviceSystem(w.spec)
    r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg, log_capacity=1)
    print(f"C4 f16 tc16: device {r.n_accepted}/{r.n_failed}, oracle {o.n_accepted}/{o.n_failed}")
    assert r.flops.rhs_evals == 3 + 3 * r.n_accepted + 4 * r.n_failed
    gate(r, o, w.cfg, dev, w)
    dev.close()


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_tc16_non_finite_column_poisons_every_row_like_the_cuda_core_sweep(gpu, monkeypatch, bad):
    """A non-finite state element (eval_core would produce non-finite rows:
    systems.cpp:30-64; the solver then takes the non-finite branch,
    solver.cpp:150-162): the tensor-core sweep's rows are non-finite exactly
    where the CUDA-core sweep's are."""
    n = 4096
    dev = DeviceSystem(kur_spec(n))
    x = rng_uniform(10, 1, n, 0.0, TWO_PI)
    x[1234] = bad
    monkeypatch.setenv("MS_SWEEP", "tc16")
    a = dev.eval_rhs(0.0, x, SSS)
    monkeypatch.setenv("MS_SWEEP", "ldg")
    b = dev.eval_rhs(0.0, x, SSS)
    assert np.array_equal(np.isfinite(a), np.isfinite(b))
    assert not np.isfinite(a).any()
    dev.close()


@pytest.mark.parametrize("n", [1024, 4352])
@pytest.mark.parametrize("storage32", [False, True])
def test_tc16_folded_next_prep_is_bitwise_the_separate_prep(gpu, n, storage32, monkeypatch):
    """The tensor-core sweep runs the next stage's prep for the rows of every
    tile it completes (k_rhs_tc16<NEXT>, launch_stage in ms_api.cu; column data
    and operand image into the other buffers): the whole solve -- final state,
    counts, evaluation tallies and every step record -- must equal the solve
    with k_prep launched for every stage (MS_FUSE_NEXT=off)."""
    from paper_2605_23727_b200.configs import config2_kuramoto
    from paper_2605_23727_b200.precision import PolicyVariant, policy_for
    from paper_2605_23727_b200.solver import SolveStatus
    monkeypatch.setenv("MS_SWEEP", "tc16")
    w = config2_kuramoto(n=n, rtol=1e-6, k_storage="f16")
    w.tf = 5.0
    pol = policy_for(PolicyVariant.Single) if storage32 else w.policy
    res, launches = [], []
    from paper_2605_23727_b200 import _abi
    for f in ("on", "off"):
        monkeypatch.setenv("MS_FUSE_NEXT", f)
        dev = DeviceSystem(w.spec)  # its own graph cache: the env is read while capturing
        monkeypatch.setenv("MS_LOOP", "host")  # plain launches, so the launch counter sees the fold
        l0 = _abi.lib().ms_launch_count()
        res.append(S.solve(dev, w.x0, w.t0, w.tf, pol, w.cfg))
        launches.append(_abi.lib().ms_launch_count() - l0)
        monkeypatch.delenv("MS_LOOP")
        dev.close()
    a, b = res
    assert a.status == b.status == SolveStatus.Completed
    assert (a.n_accepted, a.n_failed) == (b.n_accepted, b.n_failed)
    assert a.flops.rhs_evals == b.flops.rhs_evals
    assert np.array_equal(a.final_state, b.final_state)
    assert [(r.t, r.h, r.err, r.accepted) for r in a.step_log] == [(r.t, r.h, r.err, r.accepted) for r in b.step_log]
    # the fold is live: two k_prep launches fewer per attempt
    attempts = a.n_accepted + a.n_failed
    print(f"n={n}: launches folded {launches[0]} vs separate {launches[1]} over {attempts} attempts")
    assert launches[1] - launches[0] >= 2 * attempts - 2
