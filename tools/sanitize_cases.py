"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck).

Each case exercises one pipeline of the library at a size the sanitizer
finishes in a minute: the f32 TMA sweep with the folded next-stage prep and its
mbarrier ring, the 16-bit register sweep, the fused small-system kernel, the
batched tensor-core GEMM (CTA pairs, TMEM), the CUDA-core batch path, the
concurrent-variant sweep, dense output / snapshots, and the host-driven loop.

  python tools/sanitize_cases.py <case>      (case in CASES, or "all")
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import (SSS_D, TWO_PI, config1_lco, config2_kuramoto, config3_cc,  # noqa: E402
                                           rng_normal, rng_uniform)
from paper_2605_23727_b200.precision import PolicyVariant, policy_for  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec  # noqa: E402


def _cfg(**kw):
    return S.SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False, **kw)


def c2_f32():
    w = config2_kuramoto(n=1000, rtol=1e-5)
    r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 0.5, w.policy, w.cfg)
    return r.status, r.n_accepted


def c2_f16():
    w = config2_kuramoto(n=1000, rtol=1e-5, k_storage="f16")
    r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 0.5, w.policy, w.cfg)
    return r.status, r.n_accepted


def c2_policies():
    w = config2_kuramoto(n=520, rtol=1e-5)
    dev = DeviceSystem(w.spec)
    out = []
    for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2, PolicyVariant.Double):
        r = S.solve(dev, w.x0, 0.0, 0.3, policy_for(v), w.cfg)
        out.append((r.status, r.n_accepted))
    return out


def c4_f16_tc16():
    """the f16-K tensor-core sweep (k_rhs_tc16: tile images, op16 image, chunk tickets)"""
    os.environ["MS_SWEEP"] = "tc16"
    try:
        w = config2_kuramoto(n=4352, rtol=1e-5, k_storage="f16")
        r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 0.3, w.policy, w.cfg)
    finally:
        del os.environ["MS_SWEEP"]
    return r.status, r.n_accepted


def c1_fused():
    w = config1_lco(n=256)
    r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 0.5, w.policy, w.cfg)
    return r.status, r.n_accepted


def c3_fused():
    w = config3_cc(n=256)
    r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 1.0, w.policy, w.cfg)
    return r.status, r.n_accepted


def faithful():
    w = config2_kuramoto(n=300, rtol=1e-5, rhs_mode="faithful")
    r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 0.2, w.policy, w.cfg)
    return r.status, r.n_accepted


def dense_snapshots():
    w = config2_kuramoto(n=256, rtol=1e-5)
    cfg = _cfg(record_snapshots=True)
    r = S.solve(DeviceSystem(w.spec), w.x0, 0.0, 0.3, w.policy, cfg, t_eval=np.linspace(0.0, 0.3, 7))
    return r.status, r.n_accepted


def variants():
    w = config2_kuramoto(n=640, rtol=1e-5)
    dev = DeviceSystem(w.spec)
    pols = [policy_for(v) for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2,
                                    PolicyVariant.Double)]
    rs = S.solve_variants(dev, w.x0, 0.0, 0.3, pols, w.cfg)
    return [(r.status, r.n_accepted) for r in rs]


def _batch(tc, ks="bf16", B=256, n=256, tf=0.3):
    from paper_2605_23727_b200.batch import DeviceBatch
    spec = SystemSpec("kuramoto", n, k_storage=ks, omega=np.zeros(n), k_uniform=(4, 2, 0.0, 2.0))
    omega = rng_normal(4, 0, B * n).reshape(B, n)
    x0 = rng_uniform(4, 1, B * n, 0.0, TWO_PI).reshape(B, n)
    res = DeviceBatch(DeviceSystem(spec), omega, tensor_cores=tc).solve(x0, 0.0, tf, SSS_D, _cfg())
    return list(res.status[:4]), int(res.n_accepted.sum())


def batch_tc():
    return _batch(True)


def batch_cuda_cores():
    return _batch(False, ks="f32", B=16)


def dp54():
    w = config2_kuramoto(n=256, rtol=1e-5)
    r = S.dp54_reference(DeviceSystem(w.spec), w.x0, 0.0, 0.2, S.SolverConfig(time_limits_enabled=False))
    return r.status, r.n_accepted


def sharded_one_rank():
    import torch
    import torch.distributed as dist
    from paper_2605_23727_b200.sharded import DeviceEngine, ShardedSolver, TorchComm
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    w = config2_kuramoto(n=768, rtol=1e-5)
    r = ShardedSolver(DeviceEngine(DeviceSystem(w.spec)), TorchComm(), use_graph=False).solve(
        w.x0, 0.0, 0.3, w.policy, w.cfg)
    dist.destroy_process_group()
    return r.status, r.n_accepted


CASES = {f.__name__: f for f in (c2_f32, c2_f16, c4_f16_tc16, c2_policies, c1_fused, c3_fused, faithful, dense_snapshots,
                                 variants, batch_tc, batch_cuda_cores, dp54, sharded_one_rank)}

if __name__ == "__main__":
    names = list(CASES) if sys.argv[1:] in ([], ["all"]) else sys.argv[1:]
    for nm in names:
        print(nm, CASES[nm](), flush=True)
