"""C5's multi-GPU path — trajectories sharded over ranks, K replicated, one
all-gather of the per-trajectory results at the end — run with world_size 2
over gloo on CPU. Each rank's engine solves its trajectories with the oracle
(test infrastructure); the merged result must equal the single-process solve
of every trajectory bit for bit, whatever the split."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_23727_b200.batch import BatchResult, ShardedBatch, trajectory_range
from paper_2605_23727_b200.configs import config5_batch


def test_trajectory_range_partitions():
    for B in (1, 5, 6, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            spans = [trajectory_range(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        trajectory_range(4, 2, 2)


class OracleBatch:
    """Per-trajectory oracle solves with the DeviceBatch.solve signature."""

    def __init__(self, spec, omega):
        import _oracle as O
        self.O, self.spec, self.omega = O, spec, omega

    def solve(self, x0, t0, tf, pol, cfg):
        from paper_2605_23727_b200.systems import SystemSpec
        st, tr, na, nf, ev, fin = [], [], [], [], [], []
        for b in range(self.omega.shape[0]):
            spec = SystemSpec(**{**self.spec.__dict__, "omega": self.omega[b]})
            r = self.O.solve(self.O.OracleSystem(spec), x0[b], t0, tf, pol, cfg)
            st.append(r.status); tr.append(r.t_reached); na.append(r.n_accepted); nf.append(r.n_failed)
            ev.append(r.flops.rhs_evals); fin.append(r.final_state)
        return BatchResult(np.array(st), np.array(tr), np.array(na, dtype=np.int64), np.array(nf, dtype=np.int64),
                           np.array(ev, dtype=np.int64), np.array(fin), int(max(na) + max(nf)), 0.0)


def _case():
    w = config5_batch(batch=5, n=12, tf=0.5, rtol=1e-5, atol=1e-8, k_storage="f32")
    return w


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    w = _case()
    sb = ShardedBatch(lambda om: OracleBatch(w.spec, om), w.omega)
    r = sb.solve(w.x0, w.t0, w.tf, w.policy, w.cfg)
    q.put((rank, [int(s) for s in r.status], r.t_reached, r.n_accepted, r.n_failed, r.rhs_evals, r.final_state))
    dist.destroy_process_group()


def test_sharded_batch_matches_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = _case()
    ref = OracleBatch(w.spec, w.omega).solve(w.x0, w.t0, w.tf, w.policy, w.cfg)
    for rank, st, tr, na, nf, ev, fin in got:
        assert st == [int(s) for s in ref.status]
        assert np.array_equal(tr, ref.t_reached) and np.array_equal(na, ref.n_accepted)
        assert np.array_equal(nf, ref.n_failed) and np.array_equal(ev, ref.rhs_evals)
        assert np.array_equal(fin, ref.final_state)
