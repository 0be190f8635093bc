import os, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config4_kuramoto
from paper_2605_23727_b200.precision import DDD, DDS, SSS, PolicyVariant, policy_for
from paper_2605_23727_b200.systems import DeviceSystem
w = config4_kuramoto()
dev = DeviceSystem(w.spec)
cfg = S.SolverConfig(rel_tol=w.cfg.rel_tol, abs_tol=w.cfg.abs_tol, time_limits_enabled=False, max_iterations=5)
for sweep in ("ldg", "tma", "tma", "tma"):
    os.environ["MS_SWEEP"] = sweep
    outs = {nm: dev.eval_rhs(0.0, w.x0, sp) for nm, sp in (("SSS", SSS), ("DDS", DDS), ("DDD", DDD))}
    print(sweep, {k: (bool(np.all(np.isfinite(v))), float(np.sum(v))) for k, v in outs.items()})
    for pol in ("Mixed2", "Double", "Single"):
        r = S.solve(dev, w.x0, w.t0, w.tf, policy_for(PolicyVariant[pol]), cfg)
        print("  ", pol, S.status_name(r.status), r.n_accepted, r.n_failed, [(s.h, s.err) for s in r.step_log[:2]])
