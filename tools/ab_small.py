"""Device time per attempt of whole C1/C2/C3 solves (no CPU oracle): one line
per config, for A/B runs of build or runtime switches (e.g. MS_CTL_SMEM)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config1_lco, config2_kuramoto, config3_cc  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
for name, w in (("C1", config1_lco()), ("C2", config2_kuramoto(rtol=1e-6)), ("C3", config3_cc())):
    dev = DeviceSystem(w.spec)
    S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
    rs = [S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg) for _ in range(3)]
    ms = min(r.device_ms for r in rs)
    r = rs[0]
    att = r.n_accepted + r.n_failed
    print(json.dumps({"tag": tag, "config": name, "accepted": r.n_accepted, "rejected": r.n_failed,
                      "ms": round(ms, 3), "us_per_attempt": round(1e3 * ms / att, 2),
                      "steps_per_s": round(r.n_accepted / (ms / 1e3), 1)}), flush=True)
    dev.close()
