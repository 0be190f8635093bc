"""C2 with K in f16: device us per attempt (graph), for sweep comparisons."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config2_kuramoto  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

w = config2_kuramoto(rtol=1e-6, k_storage=sys.argv[1] if len(sys.argv) > 1 else "f16")
dev = DeviceSystem(w.spec)
S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
print("c2", w.spec.k_storage, r.n_accepted, r.n_failed, r.device_ms, "ms", r.device_ms * 1e3 / (r.n_accepted + r.n_failed), "us/attempt")
