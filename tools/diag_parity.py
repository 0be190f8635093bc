"""Where device and oracle step logs part (diagnostic)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import _oracle as O  # noqa: E402
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import reference_ic, rng_uniform  # noqa: E402
from paper_2605_23727_b200.precision import PolicyVariant, policy_for  # noqa: E402
from paper_2605_23727_b200.solver import SolverConfig  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec  # noqa: E402

cfg = SolverConfig()
errs = rng_uniform(4, 0, 3000, 1e-9, 1e-5)
mism = sum(S.adjust_step(0.01, e, 1e-6, cfg) != O.adjust_step(0.01, e, 1e-6, cfg) for e in errs)
print("adjust_step bitwise mismatches:", mism, "of", len(errs))
n = 20
spec = SystemSpec("lco", n, rhs_mode="faithful")
dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
x0 = reference_ic("lco", n, 7)
print("h0 dev/orc:", S.initial_step(dev, 0.0, 31.4, x0, SolverConfig(rel_tol=1e-6, abs_tol=1e-8)),
      O.initial_step(orc, 0.0, 31.4, x0, SolverConfig(rel_tol=1e-6, abs_tol=1e-8)))
for v in (PolicyVariant.Double, PolicyVariant.Mixed1):
    c = SolverConfig(rel_tol=1e-6, abs_tol=1e-8)
    r = S.solve(dev, x0, 0.0, 31.4, policy_for(v), c)
    o = O.solve(orc, x0, 0.0, 31.4, policy_for(v), c)
    a = [(s.t, s.h, s.err, s.accepted) for s in r.step_log]
    b = [(s.t, s.h, s.err, s.accepted) for s in o.step_log]
    i = next((i for i, (u, w) in enumerate(zip(a, b)) if u != w), None)
    print(v.name, "first diff at", i)
    if i is not None:
        for j in range(max(0, i - 2), min(i + 2, len(a))):
            print("  dev", a[j]); print("  orc", b[j])
        # recompute the controller for record i-1 on both sides
        t, h, e, acc = b[i - 1]
        print("  adjust(dev, orc):", S.adjust_step(h, e, c.rel_tol, c).hex(), O.adjust_step(h, e, c.rel_tol, c).hex())
