import sys, json
sys.path.insert(0, ".")
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config2_kuramoto
from paper_2605_23727_b200.systems import DeviceSystem
for ks in ("f32", "f16"):
    w = config2_kuramoto(rtol=1e-6, k_storage=ks)
    dev = DeviceSystem(w.spec)
    S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)
    rs = [S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg) for _ in range(3)]
    ms = min(r.device_ms for r in rs)
    print("C2", ks, rs[0].n_accepted, rs[0].n_failed, ms, 1e3 * ms / (rs[0].n_accepted + rs[0].n_failed), "us/attempt")
    dev.close()
