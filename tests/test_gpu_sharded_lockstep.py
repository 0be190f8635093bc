"""The row-sharded device loop at world size > 1 on ONE GPU: G row-range
handles of the same system (rows [r N/G, (r+1) N/G), each with its own
stream and its own copy of the O(N) state) run the ms_loop_* segments in
lock-step, and every exchange is a device-to-device copy of each handle's
owned block into the others' vectors (what the NCCL all-gather does across
GPUs). The result must equal ms_solve on the whole-K handle BIT FOR BIT: a
row's sum order depends only on N (the sweep's lane/column order), never on
the row partition (the reference's reduction sites are
systems.cpp:41-63 and solver.cpp:399-411).

The ranks' kernels never wait on one another (no cross-stream spin): each
segment is issued on every rank's stream, then the copies are issued after
an event wait, so this is a faithful single-GPU stand-in for the exchange."""
import numpy as np
import pytest

from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config2_kuramoto, config4_kuramoto
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.sharded import DeviceEngine, row_range
from paper_2605_23727_b200.systems import DeviceSystem

pytestmark = pytest.mark.gpu


class Lockstep:
    """Drives G DeviceEngines of one system like G ranks of ShardedSolver."""

    def __init__(self, engines):
        import torch
        self.torch = torch
        self.E = engines
        self.copies = 0

    def _segments(self, lst):
        torch = self.torch
        n = self.E[0].segment_count(lst)
        assert all(e.segment_count(lst) == n for e in self.E)
        for i in range(n):
            exs = []
            for e in self.E:
                with e.context():
                    exs.append(e.run_segment(lst, i))
            if not exs[0].needed:
                assert not any(x.needed for x in exs)
                continue
            done = []
            for e in self.E:
                ev = torch.cuda.Event()
                ev.record(e.s)
                done.append(ev)
            for d, (e, dx) in enumerate(zip(self.E, exs)):
                for s, sx in enumerate(exs):
                    if s == d:
                        continue
                    assert (sx.offset, sx.count, sx.total) == (s * sx.count, dx.count, dx.total)
                    e.s.wait_event(done[s])
                    with torch.cuda.stream(e.s):
                        dx.buf[sx.offset:sx.offset + sx.count].copy_(sx.buf[sx.offset:sx.offset + sx.count])
                    self.copies += 1
            # no rank may overwrite a block before every peer has copied it
            after = []
            for e in self.E:
                ev = torch.cuda.Event()
                ev.record(e.s)
                after.append(ev)
            for e in self.E:
                for ev in after:
                    e.s.wait_event(ev)

    def solve(self, x0, t0, tf, policy, cfg, cap=1 << 16):
        for e in self.E:
            with e.context():
                e.begin(x0, t0, tf, policy, cfg, cap)
        self._segments(0)
        while True:
            for _ in range(4):
                self._segments(1)
            flags = []
            for e in self.E:
                with e.context():
                    flags.append(e.done())
            assert len(set(flags)) == 1, flags
            if flags[0]:
                break
        outs = []
        for e in self.E:
            with e.context():
                outs.append(e.end())
        return outs


class LockstepPush(Lockstep):
    """The push exchange (ms_loop_push_*) at world G on one GPU: every rank's
    sweeps store their rows straight into the other handles' workspaces (the
    same-device stand-in for NVLink peer memory) and each segment ends with the
    epoch release into the peers' mailboxes. The ranks never wait on one another
    inside a kernel here: each rank's mailbox wait is issued only after its
    stream has waited (host-side events) for every peer's segment, so the wait
    kernel finds the epochs already released -- it checks the protocol (a wrong
    epoch would trap after 20 s) without a cross-rank spin."""

    def setup(self):
        infos = []
        for e in self.E:
            with e.context():
                infos.append(e.push_info())
        ws, mb = [i[0] for i in infos], [i[2] for i in infos]
        assert len(set(i[1] for i in infos)) == 1  # identical workspace layouts
        for r, e in enumerate(self.E):
            with e.context():
                e.push_setup(len(self.E), r, ws, mb)

    def _segments(self, lst):
        torch = self.torch
        n = self.E[0].segment_count(lst)
        for i in range(n):
            for e in self.E:
                with e.context():
                    ex = e.run_segment(lst, i)
                assert not ex.needed  # the sweeps already pushed their rows
            done = []
            for e in self.E:
                ev = torch.cuda.Event()
                ev.record(e.s)
                done.append(ev)
            for r, e in enumerate(self.E):
                for q, ev in enumerate(done):
                    if q != r:
                        e.s.wait_event(ev)
                with e.context():
                    e.push_wait()

    def solve(self, x0, t0, tf, policy, cfg, cap=1 << 16):
        for e in self.E:
            with e.context():
                e.begin(x0, t0, tf, policy, cfg, cap)
        self.setup()
        self._segments(0)
        while True:
            for _ in range(4):
                self._segments(1)
            flags = []
            for e in self.E:
                with e.context():
                    flags.append(e.done())
            assert len(set(flags)) == 1, flags
            if flags[0]:
                break
        outs = []
        for e in self.E:
            with e.context():
                outs.append(e.end())
        return outs


def _same(a, b):
    assert (a.status, a.n_accepted, a.n_failed, a.t_reached) == (b.status, b.n_accepted, b.n_failed, b.t_reached)
    assert np.array_equal(a.final_state, b.final_state)
    assert [(s.t, s.h, s.err, s.accepted) for s in a.step_log] == [(s.t, s.h, s.err, s.accepted) for s in b.step_log]
    assert a.flops.rhs_evals == b.flops.rhs_evals


def _run(w, world, policy=None, tf=None, push=False):
    pol = policy or w.policy
    tf = w.tf if tf is None else tf
    full = DeviceSystem(w.spec)
    ref = S.solve(full, w.x0, w.t0, tf, pol, w.cfg, log_capacity=1 << 16)
    full.close()
    handles = []
    for r in range(world):
        w.spec.row_begin, w.spec.row_end = row_range(w.spec.n_agents, r, world)
        handles.append(DeviceSystem(w.spec))
    w.spec.row_begin = w.spec.row_end = 0
    ls = (LockstepPush if push else Lockstep)([DeviceEngine(h) for h in handles])
    outs = ls.solve(w.x0, w.t0, tf, pol, w.cfg)
    for o in outs:
        _same(o, ref)
    assert (ls.copies == 0) if push else (ls.copies > 0)
    for h in handles:
        h.close()
    return ref


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("ks", ["f32", "f16"])
def test_c2_row_shards_bitwise_equal_solve(gpu, world, ks):
    w = config2_kuramoto(rtol=1e-6, k_storage=ks)
    ref = _run(w, world, tf=10.0)
    assert ref.n_accepted > 100


def test_c2_mixed2_row_shards_bitwise(gpu):
    w = config2_kuramoto(rtol=1e-6)
    _run(w, 2, policy=policy_for(PolicyVariant.Mixed2), tf=5.0)


@pytest.mark.slow
def test_c4_row_shards_bitwise_equal_solve(gpu):
    """C4 at its full size, K split in two row blocks of 2 GiB (f32): the
    whole benchmark solve, bit for bit."""
    w = config4_kuramoto()
    ref = _run(w, 2)
    assert ref.status == S.SolveStatus.Completed and ref.n_accepted > 1000


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 4])
def test_c4_f16_tensor_core_sweep_row_shards_bitwise(gpu, world):
    """C4 with K f16 (the tensor-core sweep k_rhs_tc16, the default at this N):
    the row-sharded loop gives the whole-K solve bit for bit -- each row's
    dot-product order depends only on N (rows that do not align
    with the 128-row MMA tiles: tests/test_gpu_tc16.py). A shortened span keeps
    the test quick."""
    w = config4_kuramoto(k_storage="f16")
    ref = _run(w, world, tf=2.0)
    assert ref.status == S.SolveStatus.Completed and ref.n_accepted > 50


# ---- push exchange: the sweeps store their rows into the peers (no gather) ----

@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("ks", ["f32", "f16"])
def test_c2_push_exchange_bitwise_equal_solve(gpu, world, ks):
    """C2 through the push exchange (f32 K: the TMA row-copy sweep; f16 K: the
    2D-tile sweep): bitwise ms_solve."""
    w = config2_kuramoto(rtol=1e-6, k_storage=ks)
    ref = _run(w, world, tf=10.0, push=True)
    assert ref.n_accepted > 100


def test_c2_mixed2_push_exchange_bitwise(gpu):
    """binary64 sums (the register sweep's DDS rows) through the push exchange"""
    w = config2_kuramoto(rtol=1e-6)
    _run(w, 2, policy=policy_for(PolicyVariant.Mixed2), tf=5.0, push=True)


@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_lco_cc_push_exchange_bitwise(gpu, cfg):
    """per-pair models (LCO, CC: the register sweep, d > 1 with only the
    coupled slot exchanged) through the push exchange"""
    from paper_2605_23727_b200.configs import config1_lco, config3_cc
    w = config1_lco() if cfg == "c1" else config3_cc()
    _run(w, 2, tf=2.0 if cfg == "c1" else 10.0, push=True)


@pytest.mark.slow
def test_c4_f16_push_exchange_bitwise(gpu):
    """C4 f16 (the tensor-core sweep k_rhs_tc16 pushes its rows) at world 2"""
    w = config4_kuramoto(k_storage="f16")
    ref = _run(w, 2, tf=2.0, push=True)
    assert ref.n_accepted > 50

