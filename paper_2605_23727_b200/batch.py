"""Batched Kuramoto ensembles sharing one K (BASELINE.json configs[4]) — the
ms_batch_* C-ABI. Every trajectory is an independent reference solve
(solver.cpp:226-347) with its own omega_b, theta0_b, h, t and status; the
device advances them in lock-step attempts so that a stage is one dense
contraction K·[S|C] (a tcgen05 GEMM for binary32 rows when K is f16/bf16)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .precision import PrecisionPolicy, StagePrecision
from .solver import SolverConfig, SolveStatus
from .systems import DeviceSystem


@dataclass
class BatchResult:
    status: np.ndarray
    t_reached: np.ndarray
    n_accepted: np.ndarray
    n_failed: np.ndarray
    rhs_evals: np.ndarray
    final_state: np.ndarray
    attempts: int
    device_ms: float


class DeviceBatch:
    def __init__(self, sys: DeviceSystem, omega, tensor_cores: bool = True):
        self.sys = sys  # keeps K alive
        self.omega = np.ascontiguousarray(omega, dtype=np.float64)
        self.B, self.n = self.omega.shape
        if self.n != sys.agents():
            raise ValueError("omega must be [B][N]")
        h = C.c_void_p()
        _abi.check(_abi.lib().ms_batch_create(sys.handle, self.B, _abi.dptr(self.omega), int(tensor_cores),
                                              C.byref(h)), "ms_batch_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None:
            _abi.lib().ms_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def eval_rhs(self, x, sp: StagePrecision) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.B, self.n):
            raise ValueError("x must be [B][N]")
        out = np.empty_like(x)
        _abi.check(_abi.lib().ms_batch_eval_rhs(self._h, _abi.dptr(x), sp.c(), _abi.dptr(out)), "ms_batch_eval_rhs")
        return out

    def solve(self, x0, t0: float, t_final: float, policy: PrecisionPolicy, cfg: SolverConfig) -> BatchResult:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        if x0.shape != (self.B, self.n):
            raise ValueError("x0 must be [B][N]")
        st = np.zeros(self.B, dtype=np.int32)
        tr = np.zeros(self.B)
        na = np.zeros(self.B, dtype=np.int64)
        nf = np.zeros(self.B, dtype=np.int64)
        ev = np.zeros(self.B, dtype=np.int64)
        fin = np.empty_like(x0)
        r = _abi.BatchResultC()
        r.status = st.ctypes.data_as(C.POINTER(C.c_int32))
        r.t_reached = _abi.dptr(tr)
        r.n_accepted = na.ctypes.data_as(C.POINTER(C.c_int64))
        r.n_failed = nf.ctypes.data_as(C.POINTER(C.c_int64))
        r.rhs_evals = ev.ctypes.data_as(C.POINTER(C.c_int64))
        r.final_state = _abi.dptr(fin)
        pol, cc = policy.c(), cfg.c()
        _abi.check(_abi.lib().ms_batch_solve(self._h, _abi.dptr(x0), t0, t_final, C.byref(pol), C.byref(cc),
                                             C.byref(r)), "ms_batch_solve")
        return BatchResult(np.array([SolveStatus(s) for s in st]), tr, na, nf, ev, fin, r.attempts, r.device_ms)


# ---- multi-GPU: trajectories sharded across ranks ---------------

def trajectory_range(batch: int, rank: int, world: int):
    """Contiguous, balanced trajectory blocks: rank r owns [b0, b1)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(batch, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


class ShardedBatch:
    """An ensemble split by trajectory over a torch.distributed group: K is
    replicated (each rank holds its own DeviceSystem), every rank advances only
    its trajectories, and nothing is exchanged while they run — trajectories
    are independent solves (harness.cpp:113-121). The per-trajectory results
    are all-gathered once at the end, so every rank returns the whole
    BatchResult; attempts and device time are the maxima over ranks.

    ``make_local(omega_slice)`` builds the rank's engine (a DeviceBatch on the
    GPU); anything with the DeviceBatch.solve signature works."""

    def __init__(self, make_local, omega, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        omega = np.ascontiguousarray(omega, dtype=np.float64)
        self.B, self.n = omega.shape
        self.b0, self.b1 = trajectory_range(self.B, self.rank, self.world)
        self.local = make_local(omega[self.b0:self.b1])
        self._dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def _gather(self, arr: np.ndarray) -> np.ndarray:
        """Concatenate the ranks' leading-axis blocks (sizes may differ by one)."""
        import torch
        rows = (self.B + self.world - 1) // self.world
        pad = np.zeros((rows,) + arr.shape[1:], dtype=arr.dtype)
        pad[:arr.shape[0]] = arr
        t = torch.from_numpy(pad).to(self._dev)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        out = []
        for r, p in enumerate(parts):
            b0, b1 = trajectory_range(self.B, r, self.world)
            out.append(p.cpu().numpy()[:b1 - b0])
        return np.concatenate(out, axis=0)

    def _max(self, v: float) -> float:
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64, device=self._dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def solve(self, x0, t0: float, t_final: float, policy: PrecisionPolicy, cfg: SolverConfig) -> BatchResult:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        if x0.shape != (self.B, self.n):
            raise ValueError("x0 must be [B][N]")
        r = self.local.solve(x0[self.b0:self.b1], t0, t_final, policy, cfg)
        status = self._gather(np.array([int(s) for s in r.status], dtype=np.int32))
        return BatchResult(np.array([SolveStatus(int(s)) for s in status]), self._gather(r.t_reached),
                           self._gather(r.n_accepted), self._gather(r.n_failed), self._gather(r.rhs_evals),
                           self._gather(r.final_state), int(self._max(r.attempts)), self._max(r.device_ms))
