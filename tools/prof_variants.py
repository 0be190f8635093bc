"""A short concurrent-variants solve (C2 or C4 shape) for ncu captures of k_rhs_multi."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config2_kuramoto, config4_kuramoto  # noqa: E402
from paper_2605_23727_b200.precision import PolicyVariant, policy_for  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

w = config4_kuramoto() if "c4" in sys.argv else config2_kuramoto(rtol=1e-6)
dev = DeviceSystem(w.spec)
pols = [policy_for(v) for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2, PolicyVariant.Double)]
r = S.solve_variants(dev, w.x0, w.t0, 0.05, pols, w.cfg, log_capacity=1)
print([x.n_accepted for x in r], r[0].device_ms)
