"""Short C4 workload for ncu: builds the N=32768 Kuramoto system, runs the RHS
(prep + K sweep) a few times outside any CUDA graph, then a few attempts of the
solve with the host-driven loop (MS_LOOP=host) so every kernel launch is
visible to ncu (kernels inside a conditional-node graph are not)."""
import argparse
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_23727_b200 import _abi, solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config4_kuramoto  # noqa: E402
from paper_2605_23727_b200.precision import SSS  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--kdtype", default="f32")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--attempts", type=int, default=4)
a = ap.parse_args()
w = config4_kuramoto(n=a.n, k_storage=a.kdtype)
dev = DeviceSystem(w.spec)
rhs, prep = C.c_double(), C.c_double()
x = np.ascontiguousarray(w.x0)
_abi.check(_abi.lib().ms_profile_rhs(dev.handle, _abi.dptr(x), SSS.c(), a.iters, C.byref(rhs), C.byref(prep)), "prof")
ks = {"f32": 4, "f16": 2, "bf16": 2}[a.kdtype]
print(f"rhs {rhs.value:.4f} ms  prep {prep.value:.4f} ms  -> {a.n * a.n * ks / rhs.value / 1e6:.1f} GB/s")
os.environ["MS_LOOP"] = "host"
w.cfg.max_iterations = a.attempts
r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
print(r.status, r.n_accepted, r.n_failed)
