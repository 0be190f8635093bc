"""The row-sharded loop on the device (ms_loop_* segments + NCCL), run as one
rank on one GPU: with the attempt captured into a CUDA graph (kernels + NCCL
all-gather) or launched segment by segment, it must reproduce ms_solve's
result bit for bit (same kernels, same order of every row's sum)."""
import os
import socket

import numpy as np
import pytest

from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config2_kuramoto, reference_ic
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.sharded import DeviceEngine, ShardedSolver, TorchComm
from paper_2605_23727_b200.solver import SolverConfig, SolveStatus
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg(gpu):
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _same(a, b):
    assert (a.status, a.n_accepted, a.n_failed, a.t_reached) == (b.status, b.n_accepted, b.n_failed, b.t_reached)
    assert np.array_equal(a.final_state, b.final_state, equal_nan=True)
    key = lambda r: [(s.t, s.h, repr(s.err), s.accepted) for s in r.step_log]  # noqa: E731  (NaN err)
    assert key(a) == key(b)
    assert a.flops.rhs_evals == b.flops.rhs_evals


@pytest.mark.parametrize("use_graph", [False, True])
@pytest.mark.parametrize("case", ["kuramoto", "kuramoto_f16", "lco_single", "lco_mixed1"])
def test_sharded_loop_one_rank_equals_solve(pg, use_graph, case):
    if case.startswith("kuramoto"):
        w = config2_kuramoto(n=512, rtol=1e-6, k_storage="f16" if case.endswith("f16") else "f32")
        spec, x0, tf, pol, cfg = w.spec, w.x0, 5.0, w.policy, w.cfg
    else:
        spec = SystemSpec("lco", 64, rhs_mode="faithful")
        x0 = reference_ic("lco", 64, 5)
        tf, cfg = 6.0, SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
        pol = policy_for(PolicyVariant.Single if case == "lco_single" else PolicyVariant.Mixed1)
    dev = DeviceSystem(spec)
    ref = S.solve(dev, x0, 0.0, tf, pol, cfg)
    got = ShardedSolver(DeviceEngine(dev), TorchComm(), check_every=4, use_graph=use_graph).solve(x0, 0.0, tf, pol, cfg)
    _same(got, ref)


@pytest.mark.parametrize("bad", ["x0_nan", "k_inf"])
def test_sharded_loop_non_finite_equals_solve(pg, bad):
    """Non-finite stages through the loop: the scan of each gathered stage is
    folded into the next prep and the sweep counts the evaluation, which must
    give ms_solve's status, counts and step log."""
    n = 64
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    pol = policy_for(PolicyVariant.Mixed2)
    k = np.full((n, n), 0.5)
    if bad == "k_inf":
        k[2, 5] = np.inf
    spec = SystemSpec("kuramoto", n, k_storage="f32", omega=np.linspace(-1.0, 1.0, n), K=k)
    x0 = np.linspace(0.0, 6.0, n)
    if bad == "x0_nan":
        x0[3] = np.nan
    dev = DeviceSystem(spec)
    ref = S.solve(dev, x0, 0.0, 1.0, pol, cfg)
    for use_graph in (False, True):
        got = ShardedSolver(DeviceEngine(dev), TorchComm(), check_every=4, use_graph=use_graph).solve(
            x0, 0.0, 1.0, pol, cfg)
        _same(got, ref)


class _PoisonComm(TorchComm):
    """All-gather that writes a NaN into the gathered vector after call
    number `at` -- a non-finite row arriving from another rank."""

    def __init__(self, at: int, elem: int):
        super().__init__()
        self.calls, self.at, self.elem = 0, at, elem

    def gather(self, ex):
        super().gather(ex)
        if self.calls == self.at:
            ex.buf[self.elem] = float("nan")
        self.calls += 1


@pytest.mark.parametrize("variant", [PolicyVariant.Mixed2, PolicyVariant.Single, PolicyVariant.Double])
@pytest.mark.parametrize("at", [3, 4, 5, 6, 9, 13])
def test_sharded_loop_gathered_nan_matches_separate_scan(pg, monkeypatch, variant, at):
    """A NaN arriving in a gathered stage vector rejects the attempt (err NaN,
    h * fac_min / 2), skips and does not count the attempt's later stages: the
    folded scan (inside the next prep / the finalize) against the separate
    scan launch of MS_LOOP_SCAN=separate, bit for bit."""
    w = config2_kuramoto(n=256, rtol=1e-6)
    dev = DeviceSystem(w.spec)
    pol = policy_for(variant)
    runs = []
    for mode in ("folded", "separate"):
        if mode == "separate":
            monkeypatch.setenv("MS_LOOP_SCAN", "separate")
        else:
            monkeypatch.delenv("MS_LOOP_SCAN", raising=False)
        comm = _PoisonComm(at, 37)
        runs.append(ShardedSolver(DeviceEngine(dev), comm, check_every=1, use_graph=False).solve(
            w.x0, 0.0, 2.0, pol, w.cfg))
    got, ref = runs
    _same(got, ref)
    if got.status == SolveStatus.NonFinite:  # a NaN in a recomputed k1 ends the solve
        return
    bad = [s for s in got.step_log if np.isnan(s.err)]
    assert len(bad) == 1 and not bad[0].accepted
    i = next(k for k, s in enumerate(got.step_log) if np.isnan(s.err))
    assert got.step_log[i + 1].h == got.step_log[i].h * w.cfg.fac_min * 0.5
