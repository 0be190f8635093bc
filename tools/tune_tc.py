"""Time the tcgen05 ensemble contraction variants (tools/build_variants.py tc_*)
on the C5 shape and check each against the base variant."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
VAR = ROOT / "paper_2605_23727_b200" / "_variants"
CHILD = r'''
import ctypes as C, sys, json, numpy as np
sys.path.insert(0, "%s")
from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200.batch import DeviceBatch
from paper_2605_23727_b200.configs import config5_batch
from paper_2605_23727_b200.precision import SSS
from paper_2605_23727_b200.systems import DeviceSystem
w = config5_batch()
dev = DeviceSystem(w.spec)
bat = DeviceBatch(dev, w.omega, tensor_cores=True)
x = np.ascontiguousarray(w.x0)
rhs, prep = C.c_double(), C.c_double()
_abi.check(_abi.lib().ms_batch_profile_rhs(bat._h, _abi.dptr(x), SSS.c(), 30, C.byref(rhs), C.byref(prep)), "p")
out = bat.eval_rhs(x, SSS)
print("JSON" + json.dumps({"gemm_ms": rhs.value, "prep_ms": prep.value, "digest": float(np.sum(out[:, :64]))}))
''' % ROOT
res = {}
for lib in sorted(VAR.glob(sys.argv[1] if len(sys.argv) > 1 else "lib_tc*.so")):
    name = lib.stem[4:]
    r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, MS_LIB_PATH=str(lib)),
                       capture_output=True, text=True, timeout=600)
    line = [l for l in r.stdout.splitlines() if l.startswith("JSON")]
    res[name] = json.loads(line[0][4:]) if line else {"error": r.stderr[-600:]}
    print(name, json.dumps(res[name]), flush=True)
