"""The multi-GPU row-sharded driver (paper_2605_23727_b200.sharded), run with
world_size 2 over gloo on CPU: each rank evaluates only its rows of the RHS and
the all-gather makes the state whole; the sharded solve must equal the
single-process oracle solve bit for bit (the controller is replicated)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle as O
from paper_2605_23727_b200.configs import config2_kuramoto, reference_ic
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.sharded import ShardedSolver, TorchComm, row_range
from paper_2605_23727_b200.solver import SolverConfig
from paper_2605_23727_b200.systems import SystemSpec


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    if name == "lco":
        spec = SystemSpec("lco", 24, rhs_mode="faithful")
        return spec, reference_ic("lco", 24, 7), 0.0, 8.0, policy_for(PolicyVariant.Double), \
            SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
    if name == "lco_single":
        spec = SystemSpec("lco", 24, rhs_mode="faithful")
        return spec, reference_ic("lco", 24, 3), 0.0, 5.0, policy_for(PolicyVariant.Single), \
            SolverConfig(rel_tol=1e-5, abs_tol=1e-7)
    w = config2_kuramoto(n=64, rtol=1e-5)
    return w.spec, w.x0, 0.0, 3.0, w.policy, w.cfg


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from _shard_engine import ShardCpuEngine
    spec, x0, t0, tf, pol, cfg = _case(name)
    orc = O.OracleSystem(spec)
    r0, r1 = row_range(spec.n_agents, rank, world)
    eng = ShardCpuEngine(orc, r0, r1, spec.dim)
    res = ShardedSolver(eng, TorchComm(), check_every=3, use_graph=False).solve(x0, t0, tf, pol, cfg)
    q.put((rank, res.status, res.n_accepted, res.n_failed, res.final_state,
           [(s.t, s.h, s.err, s.accepted) for s in res.step_log], res.flops.rhs_evals))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["lco", "lco_single", "kuramoto"])
def test_sharded_driver_world2_equals_oracle(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((v[0], v[1:]) for v in (q.get(timeout=240) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec, x0, t0, tf, pol, cfg = _case(name)
    ref = O.solve(O.OracleSystem(spec), x0, t0, tf, pol, cfg)
    for rank in (0, 1):
        status, acc, fail, final, log, evals = out[rank]
        assert (status, acc, fail) == (ref.status, ref.n_accepted, ref.n_failed)
        assert np.array_equal(final, ref.final_state)
        assert log == [(s.t, s.h, s.err, s.accepted) for s in ref.step_log]
        assert evals == ref.flops.rhs_evals


def test_row_range_partition():
    assert [row_range(32768, r, 8) for r in (0, 7)] == [(0, 4096), (28672, 32768)]
    with pytest.raises(ValueError):
        row_range(10, 0, 3)
