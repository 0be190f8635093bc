"""C5: batched Kuramoto ensemble (B=1024 x N=2048, shared bf16 K) on the B200.
Prints one JSON line: trajectory-steps/s of the full lock-step solve, and the
tensor-core roofline of the tcgen05 contraction (FLOPs / CUDA-event time).
Under torchrun the batch is sharded by trajectory (batch.ShardedBatch): the
global batch stays fixed, each rank solves its block, the value is all the
ranks' accepted trajectory-steps over the slowest rank's device time."""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import _abi  # noqa: E402
from paper_2605_23727_b200.batch import DeviceBatch  # noqa: E402
from paper_2605_23727_b200.configs import config5_batch  # noqa: E402
from paper_2605_23727_b200.precision import SSS  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--tf", type=float, default=20.0)
ap.add_argument("--tc", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--kdtype", default="bf16", choices=["bf16", "f16"])
a = ap.parse_args()
ws, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))
w = config5_batch(batch=a.batch, n=a.n, tf=a.tf, k_storage=a.kdtype)
w.spec.device = local
dev = DeviceSystem(w.spec)
if ws > 1:
    import torch
    import torch.distributed as dist
    from paper_2605_23727_b200.batch import ShardedBatch
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bat = ShardedBatch(lambda om: DeviceBatch(dev, om, tensor_cores=bool(a.tc)), w.omega)
    prof_h, b_local = bat.local._h, bat.b1 - bat.b0
    xl = np.ascontiguousarray(w.x0[bat.b0:bat.b1])
else:
    bat = DeviceBatch(dev, w.omega, tensor_cores=bool(a.tc))
    prof_h, b_local = bat._h, a.batch
    xl = np.ascontiguousarray(w.x0)
rhs, prep = C.c_double(), C.c_double()
_abi.check(_abi.lib().ms_batch_profile_rhs(prof_h, _abi.dptr(xl), SSS.c(), 20, C.byref(rhs), C.byref(prep)), "prof")
flops = 2.0 * a.n * a.n * 2 * b_local
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
peak = peaks.get("bf16_tflops", 1590.0)
bat.solve(w.x0, w.t0, w.tf, w.policy, w.cfg)  # warm-up (graph instantiation)
res = [bat.solve(w.x0, w.t0, w.tf, w.policy, w.cfg) for _ in range(a.steps)]
ms = sum(r.device_ms for r in res)
acc = sum(int(r.n_accepted.sum()) for r in res)
r0 = res[0]
line = {
    "workload": f"C5 batched Kuramoto B={a.batch} N={a.n} K {a.kdtype}, t in [0,{a.tf}], rtol 1e-6 atol 1e-9",
    "n_gpus": ws, "scaling": "strong" if ws > 1 else "weak",
    "parallelism": f"trajectory shards x{ws} (no per-step exchange)" if ws > 1 else "single GPU",
    "tensor_cores": bool(a.tc),
    "value": acc / (ms / 1e3), "unit": "trajectory_accepted_steps/s",
    "ms_per_solve": ms / a.steps, "lockstep_attempts": r0.attempts,
    "accepted_per_traj_mean": float(r0.n_accepted.mean()), "rejected_per_traj_mean": float(r0.n_failed.mean()),
    "completed": int((r0.status == 0).sum()),
    "contraction": {"kernel": ("k_tc_gemm2 (tcgen05.mma.cta_group::2 kind::f16, 256 x 512 pair tiles)"
                               if os.environ.get("MS_TC") != "1cta" else "k_tc_gemm (tcgen05 kind::f16 M128 N256)")
                    if a.tc else "kb_rhs_cc",
                    "ms": rhs.value, "prep_ms": prep.value, "TFLOPs": flops / (rhs.value * 1e-3) / 1e12,
                    "peak_bf16_TFLOPs": peak, "frac": flops / (rhs.value * 1e-3) / 1e12 / peak},
}
if rank == 0:
    print(json.dumps(line), flush=True)
if ws > 1:
    dist.destroy_process_group()
