"""Time the concurrent-variant sweep geometries (tools/build_variants.py multi_*)
on C4 (four named variants, t in [0, 1]) and check each against the base."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
VAR = ROOT / "paper_2605_23727_b200" / "_variants"
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, "%s")
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config4_kuramoto
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.systems import DeviceSystem
w = config4_kuramoto()
dev = DeviceSystem(w.spec)
pols = [policy_for(v) for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2, PolicyVariant.Double)]
v = S.DeviceVariants(dev, 4)
v.solve(w.x0, 0.0, 0.2, pols, w.cfg, log_capacity=1)
r = v.solve(w.x0, 0.0, 1.0, pols, w.cfg, log_capacity=1)
print("JSON" + json.dumps({"ms": r[0].device_ms, "attempts": [x.n_accepted + x.n_failed for x in r],
                            "digest": [float(np.sum(x.final_state)) for x in r]}))
''' % ROOT
for lib in sorted(VAR.glob(sys.argv[1] if len(sys.argv) > 1 else "lib_multi_*.so")):
    name = lib.stem[4:]
    r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, MS_LIB_PATH=str(lib)),
                       capture_output=True, text=True, timeout=600)
    line = [l for l in r.stdout.splitlines() if l.startswith("JSON")]
    print(name, line[0][4:] if line else r.stderr[-600:], flush=True)
