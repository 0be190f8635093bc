"""Host logic of the push exchange (sharded.PushComm + ShardedSolver), world 2
over gloo on CPU. The CUDA pieces are replaced by fakes: the IPC export of a
"device pointer" is its bytes, the import decodes them, and the engine records
what the library would be told. Checked: every rank hands ms_loop_push_setup
the full, rank-ordered table of workspace and mailbox pointers (its own entry
its own, the peers' the imported ones); a rank whose workspace moved between
solves makes every rank re-import (the exchange is collective on every
solve); the segments run ms_loop_push_wait after each one and never gather."""
import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class FakeEngine:
    def __init__(self, rank):
        self.rank = rank
        self.ws = 0x1000_0000 * (rank + 1)
        self.mb = 0x2000_0000 * (rank + 1)
        self.setups = []
        self.calls = []

    def push_info(self):
        return self.ws, 4096, self.mb

    def push_setup(self, world, rank, peer_ws, peer_mb):
        self.setups.append((world, rank, list(peer_ws), list(peer_mb)))

    def segment_count(self, lst):
        return 3 if lst == 0 else 2

    def run_segment(self, lst, i):
        from paper_2605_23727_b200.sharded import Exchange
        self.calls.append(("seg", lst, i))
        return Exchange(False, None, 0, 0, 0)

    def push_wait(self):
        self.calls.append(("wait",))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_23727_b200 import sharded
    sharded._ipc_export = lambda ptr: int(ptr).to_bytes(8, "little") + bytes(56)
    sharded._ipc_import = lambda h: int.from_bytes(h[:8], "little") + 0x5  # a "mapping" of the peer's pointer
    eng = FakeEngine(rank)
    comm = sharded.PushComm()
    comm.setup(eng)
    if rank == 1:
        eng.ws += 0x100  # this rank's workspace moved (a larger step log)
    comm.setup(eng)
    solver = sharded.ShardedSolver(eng, comm, use_graph=False)
    solver._segments(0)
    solver._segments(1)
    q.put((rank, eng.setups, eng.calls))
    dist.barrier()
    dist.destroy_process_group()


def test_push_comm_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict((r, (s, c)) for r, s, c in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    ws = {0: 0x1000_0000, 1: 0x2000_0000}
    mb = {0: 0x2000_0000, 1: 0x4000_0000}
    for r in (0, 1):
        setups, calls = out[r]
        assert len(setups) == 2
        q_ = 1 - r
        for k, (world, rank, pws, pmb) in enumerate(setups):
            peer_ws = ws[q_] + (0x100 if (q_ == 1 and k == 1) else 0)
            own_ws = ws[r] + (0x100 if (r == 1 and k == 1) else 0)
            assert (world, rank) == (2, r)
            assert pws[r] == own_ws and pmb[r] == mb[r]
            assert pws[q_] == peer_ws + 0x5 and pmb[q_] == mb[q_] + 0x5
        # every segment is followed by the mailbox wait, and nothing is gathered
        assert calls == [x for i in range(3) for x in (("seg", 0, i), ("wait",))] + \
                        [x for i in range(2) for x in (("seg", 1, i), ("wait",))]
