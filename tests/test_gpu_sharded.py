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
from paper_2605_23727_b200.solver import SolverConfig
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
    assert np.array_equal(a.final_state, b.final_state)
    assert [(s.t, s.h, s.err, s.accepted) for s in a.step_log] == [(s.t, s.h, s.err, s.accepted) for s in b.step_log]
    assert a.flops.rhs_evals == b.flops.rhs_evals


@pytest.mark.parametrize("use_graph", [False, True])
@pytest.mark.parametrize("case", ["kuramoto", "lco_single", "lco_mixed1"])
def test_sharded_loop_one_rank_equals_solve(pg, use_graph, case):
    if case == "kuramoto":
        w = config2_kuramoto(n=512, rtol=1e-6)
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
