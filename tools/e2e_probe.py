"""Wall time of one C4 solve through the public host-buffer call (ms_solve) vs
the device-resident call (ms_solve_device), alternating, per K storage: where
bench.py's e2e and value differ."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config4_kuramoto  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

ks = sys.argv[1] if len(sys.argv) > 1 else "f16"
w = config4_kuramoto(k_storage=ks)
dev = DeviceSystem(w.spec)
x0_d = torch.from_numpy(w.x0).cuda()
xf_d = torch.empty_like(x0_d)
st = torch.cuda.Stream()
paths = {
    "device_nolog": lambda: S.solve_device(dev, x0_d.data_ptr(), xf_d.data_ptr(), w.t0, w.tf, w.policy, w.cfg,
                                           stream=st.cuda_stream, log_capacity=0),
    "host_log": lambda: S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg),
    "host_nolog": lambda: S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg, log_capacity=0),
}
for f in paths.values():
    f()
torch.cuda.synchronize()
for it in range(3):
    for name, f in paths.items():
        t = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
        print(ks, it, name, f"wall {wall * 1e3:.1f} ms device {r.device_ms:.1f} ms acc {r.n_accepted}", flush=True)
