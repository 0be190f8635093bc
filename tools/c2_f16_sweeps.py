import json, os, sys
sys.path.insert(0, "/root/repo")
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config2_kuramoto
from paper_2605_23727_b200.systems import DeviceSystem
for sw in ("", "tc16", "tile", "ldg"):
    if sw: os.environ["MS_SWEEP"] = sw
    else: os.environ.pop("MS_SWEEP", None)
    w = config2_kuramoto(rtol=1e-6, k_storage="f16")
    dev = DeviceSystem(w.spec)
    S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
    rs = [S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg) for _ in range(3)]
    ms = min(r.device_ms for r in rs); r = rs[0]; att = r.n_accepted + r.n_failed
    print(json.dumps({"sweep": sw or "default", "acc": r.n_accepted, "rej": r.n_failed, "us_per_attempt": round(1e3*ms/att, 2), "steps_per_s": round(r.n_accepted/(ms/1e3), 1)}), flush=True)
    dev.close()
