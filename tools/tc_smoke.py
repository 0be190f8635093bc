"""Small tcgen05 ensemble GEMM check (run under `timeout` before the full tests)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import _oracle as O  # noqa: E402
from paper_2605_23727_b200 import _abi  # noqa: E402
from paper_2605_23727_b200.batch import DeviceBatch  # noqa: E402
from paper_2605_23727_b200.configs import TWO_PI, rng_normal, rng_uniform  # noqa: E402
from paper_2605_23727_b200.precision import SSS  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec  # noqa: E402

for B, n in ((128, 128), (160, 300), (1024, 2048)):
    spec = SystemSpec("kuramoto", n, k_storage="bf16", omega=np.zeros(n), k_uniform=(5, 2, 0.0, 2.0))
    omega = rng_normal(5, 0, B * n).reshape(B, n)
    x = rng_uniform(5, 1, B * n, 0.0, TWO_PI).reshape(B, n)
    dev = DeviceSystem(spec)
    got_tc = DeviceBatch(dev, omega, tensor_cores=True).eval_rhs(x, SSS)
    got_cc = DeviceBatch(dev, omega, tensor_cores=False).eval_rhs(x, SSS)
    orc = O.OracleSystem(spec)
    orc.set_op_round(_abi.MS_K_BF16)
    errs = []
    for b in (0, B - 1):
        orc.set_omega(omega[b])
        ref = orc.eval_rhs(0.0, x[b], SSS)
        errs.append(float(np.max(np.abs(got_tc[b] - ref))))
    print(f"B={B} N={n}: max|tc - oracle(op-rounded)| = {max(errs):.3e}; "
          f"max|tc - cuda-core(unrounded)| = {float(np.max(np.abs(got_tc - got_cc))):.3e}", flush=True)
