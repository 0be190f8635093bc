"""C4 first attempts: device vs oracle step logs (diagnostic)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import _oracle as O  # noqa: E402
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config4_kuramoto  # noqa: E402
from paper_2605_23727_b200.precision import DDD  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

w = config4_kuramoto()
O.set_threads(os.cpu_count() or 1)
dev, orc = DeviceSystem(w.spec), O.OracleSystem(w.spec)
print("h0 dev/orc", S.initial_step(dev, w.t0, w.tf, w.x0, w.cfg), O.initial_step(orc, w.t0, w.tf, w.x0, w.cfg))
cfg = S.SolverConfig(rel_tol=w.cfg.rel_tol, abs_tol=w.cfg.abs_tol, time_limits_enabled=False, max_iterations=6)
for sweep in ("ldg", "tma"):
    os.environ["MS_SWEEP"] = sweep
    r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, cfg)
    print(sweep, [(s.t, s.h, s.err, s.accepted) for s in r.step_log])
o = O.solve(orc, w.x0, w.t0, w.tf, w.policy, cfg)
print("orc", [(s.t, s.h, s.err, s.accepted) for s in o.step_log])
f0d, f0o = dev.eval_rhs(0.0, w.x0, DDD), orc.eval_rhs(0.0, w.x0, DDD)
print("DDD eval max|diff|", float(np.max(np.abs(f0d - f0o))))
