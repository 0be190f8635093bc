"""Row-sharded solve over several GPUs.

Rank r owns rows [r N/G, (r+1) N/G) of K (a row-range DeviceSystem). Every rank
holds the full O(N) state and runs the same stage combination and controller;
after each coupling sweep the stage-derivative rows are all-gathered, so every
rank sees identical vectors and takes identical accept/reject decisions (no
error-norm collective is needed). Each row's reduction order depends only on N,
so the result is bit-identical for any G.

The loop is host-driven over the segments of ``ms_loop_*`` (one attempt =
[k1 recompute] + 3 x (prep, sweep, all-gather) + finalize). On GPUs the attempt
(kernels + NCCL collectives) is captured once into a CUDA graph and replayed;
the done flag is read every ``check_every`` replays (kernels of a finished
solve no-op, so overshooting is harmless).

``ShardedSolver`` is written against two small interfaces, an *engine*
(the C-ABI segments) and a *communicator* (torch.distributed), so the same
driver is exercised on CPU with gloo and a reference engine (tests/).
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .precision import PrecisionPolicy
from .solver import SolverConfig, SolveResult, _result


def row_range(n: int, rank: int, world: int):
    """Equal row blocks (NCCL in-place all-gather needs equal counts)."""
    if n % world:
        raise ValueError(f"row sharding needs N divisible by the world size ({n} % {world})")
    b = n // world
    return rank * b, (rank + 1) * b


@dataclass
class Exchange:
    needed: bool
    buf: object     # engine-specific full vector (torch CUDA tensor or numpy array)
    offset: int
    count: int
    total: int


class _CAI:
    """Zero-copy view of a device pointer for torch.as_tensor."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


class DeviceEngine:
    """The ms_loop_* segments of one row-sharded DeviceSystem."""

    def __init__(self, sys):
        import torch
        self.torch = torch
        self.sys = sys
        self.L = _abi.lib()
        self._views = {}
        # a real (non-legacy) stream: the library's kernels and torch's NCCL
        # collectives are ordered on it; a capture stream replaces it while capturing
        self.s = torch.cuda.Stream()

    def context(self):
        return self.torch.cuda.stream(self.s)

    def stream(self) -> int:
        return self.torch.cuda.current_stream().cuda_stream

    def begin(self, x0, t0, tf, policy: PrecisionPolicy, cfg: SolverConfig, log_capacity: int):
        self.x0 = np.ascontiguousarray(x0, dtype=np.float64)
        self.cfg = cfg
        self.cap = log_capacity
        pol, cc = policy.c(), cfg.c()
        _abi.check(self.L.ms_loop_begin(self.sys.handle, self.x0.ctypes.data_as(C.c_void_p), 0, t0, tf,
                                        C.byref(pol), C.byref(cc), log_capacity, C.c_void_p(self.stream())),
                   "ms_loop_begin")

    def segment_count(self, lst: int) -> int:
        n = C.c_int()
        _abi.check(self.L.ms_loop_segment_count(self.sys.handle, lst, C.byref(n)), "segment_count")
        return n.value

    def run_segment(self, lst: int, idx: int) -> Exchange:
        ex = _abi.ExchangeC()
        _abi.check(self.L.ms_loop_run_segment(self.sys.handle, lst, idx, C.c_void_p(self.stream()), C.byref(ex)),
                   "ms_loop_run_segment")
        if not ex.needed:
            return Exchange(False, None, 0, 0, 0)
        key = (ex.buf, ex.total)
        if key not in self._views:
            self._views[key] = self.torch.as_tensor(_CAI(ex.buf, ex.total), device="cuda")
        return Exchange(True, self._views[key], ex.offset, ex.count, ex.total)

    # push exchange (ms_loop_push_*): the sweeps store their rows into every
    # peer's workspace; each segment ends with an epoch release into the peers'
    # mailboxes and the next one starts after push_wait
    def push_info(self):
        ws, nb, mb = C.c_void_p(), C.c_size_t(), C.c_void_p()
        _abi.check(self.L.ms_loop_push_info(self.sys.handle, C.byref(ws), C.byref(nb), C.byref(mb)), "push_info")
        return ws.value, nb.value, mb.value

    def push_setup(self, world: int, rank: int, peer_ws, peer_mbox) -> None:
        pw = (C.c_void_p * world)(*[C.c_void_p(p) for p in peer_ws])
        pm = (C.c_void_p * world)(*[C.c_void_p(p) for p in peer_mbox])
        _abi.check(self.L.ms_loop_push_setup(self.sys.handle, world, rank, pw, pm), "push_setup")

    def push_wait(self) -> None:
        _abi.check(self.L.ms_loop_push_wait(self.sys.handle, C.c_void_p(self.stream())), "push_wait")

    def done(self) -> bool:
        d = C.c_int()
        _abi.check(self.L.ms_loop_done(self.sys.handle, C.c_void_p(self.stream()), C.byref(d)), "ms_loop_done")
        return bool(d.value)

    def end(self) -> SolveResult:
        final = np.empty_like(self.x0)
        r = _abi.SolveResultC()
        r.final_state = _abi.dptr(final)
        log = None
        if self.cfg.record_step_log and self.cap > 0:
            log = (_abi.StepRecordC * self.cap)()
            r.step_log = C.cast(log, C.POINTER(_abi.StepRecordC))
            r.step_log_capacity = self.cap
        _abi.check(self.L.ms_loop_end(self.sys.handle, C.byref(r), 0, C.c_void_p(self.stream())), "ms_loop_end")
        return _result(r, final, log)


class TorchComm:
    """All-gather of owned row blocks over a torch.distributed group (NCCL on
    GPUs — in place, so no staging copy; gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def gather(self, ex: Exchange) -> None:
        import torch
        buf = ex.buf if isinstance(ex.buf, torch.Tensor) else torch.from_numpy(ex.buf)
        own = buf[ex.offset:ex.offset + ex.count]
        if self.world == 1 and not buf.is_cuda:
            return
        if ex.count * self.world != ex.total or ex.offset != self.rank * ex.count:
            raise ValueError("all-gather needs equal, rank-ordered blocks")
        if buf.is_cuda:
            self.dist.all_gather_into_tensor(buf, own, group=self.group)
        else:
            parts = list(buf.view(self.world, ex.count).unbind(0))
            tmp = [torch.empty_like(own) for _ in range(self.world)]
            self.dist.all_gather(tmp, own.clone(), group=self.group)
            for p, t in zip(parts, tmp):
                p.copy_(t)


def _ipc_export(ptr: int) -> bytes:
    h = (C.c_ubyte * 64)()
    _abi.check(_abi.lib().ms_ipc_export(C.c_void_p(ptr), h), "ms_ipc_export")
    return bytes(h)


def _ipc_import(handle: bytes) -> int:
    h = (C.c_ubyte * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _abi.check(_abi.lib().ms_ipc_import(h, C.byref(p)), "ms_ipc_import")
    return p.value


class PushComm:
    """The push exchange across processes (one GPU each): every rank exports
    its workspace and mailbox with CUDA IPC, imports the peers' (NVLink peer
    mappings), and hands them to ms_loop_push_setup; the sweeps then store
    their rows straight into the peers' memory and the segments synchronize
    through the mailboxes (ms_loop_push_wait) -- no all-gather. Setup runs
    after every ms_loop_begin (cheap when the workspace did not move)."""

    push = True

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._opened = {}

    def setup(self, engine) -> None:
        if self.world <= 1:
            return
        ws, _, mb = engine.push_info()
        # collective on every solve (a rank whose workspace moved needs the
        # others to import its new handle); handles already open are reused
        mine = (_ipc_export(ws), _ipc_export(mb))
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        peer_ws, peer_mb = [], []
        for q, (hw, hm) in enumerate(allh):
            if q == self.rank:
                peer_ws.append(ws)
                peer_mb.append(mb)
                continue
            for h in (hw, hm):
                if h not in self._opened:
                    self._opened[h] = _ipc_import(h)
            peer_ws.append(self._opened[hw])
            peer_mb.append(self._opened[hm])
        engine.push_setup(self.world, self.rank, peer_ws, peer_mb)
        self.dist.barrier(group=self.group)  # every mailbox reset before any epoch is released

    def gather(self, ex: Exchange) -> None:
        raise RuntimeError("push exchange: the segments need no gather")


class ShardedSolver:
    def __init__(self, engine, comm, check_every: int = 8, use_graph: bool = True):
        self.engine = engine
        self.comm = comm
        self.check_every = max(1, int(check_every))
        self.use_graph = use_graph

    def _segments(self, lst: int) -> None:
        push = getattr(self.comm, "push", False) and getattr(self.comm, "world", 1) > 1
        for i in range(self.engine.segment_count(lst)):
            ex = self.engine.run_segment(lst, i)
            if push:
                self.engine.push_wait()
            elif ex.needed:
                self.comm.gather(ex)

    def solve(self, x0, t0: float, t_final: float, policy: PrecisionPolicy, cfg: SolverConfig,
              log_capacity: int | None = None) -> SolveResult:
        cap = int(log_capacity if log_capacity is not None else (min(cfg.max_iterations, 1 << 20)
                                                                if cfg.record_step_log else 0))
        ctx = self.engine.context() if hasattr(self.engine, "context") else contextlib.nullcontext()
        with ctx:
            self.engine.begin(x0, t0, t_final, policy, cfg, cap)
            if getattr(self.comm, "push", False):
                self.comm.setup(self.engine)
            self._segments(0)
            graph = self._capture() if self.use_graph else None
            while True:
                for _ in range(self.check_every):
                    if graph is not None:
                        graph.replay()
                    else:
                        self._segments(1)
                if self.engine.done():
                    break
            return self.engine.end()

    def _capture(self):
        import torch
        if not torch.cuda.is_available() or not isinstance(self.engine, DeviceEngine):
            return None
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            # capture one attempt; replays run it with the current device flags
            with torch.cuda.graph(g, stream=s):
                self._segments(1)
        torch.cuda.current_stream().wait_stream(s)
        return g
