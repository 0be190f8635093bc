"""Time every K-sweep variant of tools/build_variants.py on C4 (f32 and f16 K)
and check that each reproduces the base variant bit for bit."""
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
from paper_2605_23727_b200.configs import config4_kuramoto
from paper_2605_23727_b200.precision import SSS, DDS, DDD
from paper_2605_23727_b200.systems import DeviceSystem
res = {}
import os
for ks in ("f32", "f16"):
    w = config4_kuramoto(n=32768, k_storage=ks)
    dev = DeviceSystem(w.spec)
    x = np.ascontiguousarray(w.x0)
    for name, sp in (("SSS", SSS), ("DDS", DDS), ("DDD", DDD)):
        if ks == "f16" and name != "SSS":
            continue
        rhs, prep = C.c_double(), C.c_double()
        _abi.check(_abi.lib().ms_profile_rhs(dev.handle, _abi.dptr(x), sp.c(), 30, C.byref(rhs), C.byref(prep)), "p")
        out = dev.eval_rhs(0.0, x, sp)
        res[ks + "_" + name] = {"ms": rhs.value, "GBps": 32768 * 32768 * (4 if ks == "f32" else 2) / rhs.value / 1e6,
                                "digest": float(np.sum(out * np.arange(out.size)))}
    dev.close()
print("JSON" + json.dumps(res))
''' % ROOT


def main():
    out = {}
    for lib in sorted(VAR.glob("lib_*.so")):
        name = lib.stem[4:]
        env = dict(os.environ, MS_LIB_PATH=str(lib), MS_SWEEP=os.environ.get("MS_SWEEP", "tma"))
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("JSON")]
        out[name] = json.loads(line[0][4:]) if line else {"error": r.stderr[-800:]}
        print(name, json.dumps(out[name]), flush=True)
    base = out.get("base", {})
    for name, v in out.items():
        if "error" in v or not base:
            continue
        same = all(v[k]["digest"] == base[k]["digest"] for k in base if k in v)
        print(f"{name:14s} bitwise-equal-to-base={same} " +
              " ".join(f"{k}={v[k]['GBps']:.0f}GB/s" for k in v))


if __name__ == "__main__":
    main()
