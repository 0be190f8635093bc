"""A few attempts of C1/C2/C3 with the host-driven loop, for ncu launch lists."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config1_lco, config2_kuramoto, config3_cc  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = {"c1": config1_lco, "c2": lambda: config2_kuramoto(rtol=1e-6), "c3": config3_cc}[which]()
dev = DeviceSystem(w.spec)
r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)  # graph run: device time per attempt
print(which, "graph", r.n_accepted, r.n_failed, r.device_ms, "ms", r.device_ms * 1e3 / (r.n_accepted + r.n_failed), "us/attempt")
os.environ["MS_LOOP"] = "host"
w.cfg.max_iterations = 20
r = S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
print(which, "host", r.n_accepted, r.n_failed)
