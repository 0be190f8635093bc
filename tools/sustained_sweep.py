"""C4 K sweep (N = 32768) in burst (30 sweeps, ~20 ms) and sustained (~3 s of
back-to-back sweeps, the regime of a whole solve, where the board runs into its
power cap) for each sweep kernel / build variant, with nvidia-smi clocks and
power sampled during the sustained run.
usage: python tools/sustained_sweep.py [mode[:lib] ...]   (mode = tma|ldg|tile)"""
import ctypes as C
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import ctypes as C, sys, json, numpy as np
sys.path.insert(0, "%s")
from bench import ClockSampler
from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200.configs import config4_kuramoto
from paper_2605_23727_b200.precision import SSS
from paper_2605_23727_b200.systems import DeviceSystem
ks = sys.argv[1]
w = config4_kuramoto(n=32768, k_storage=ks)
dev = DeviceSystem(w.spec)
x = np.ascontiguousarray(w.x0)
nbytes = 32768 * 32768 * (4 if ks == "f32" else 2)
def prof(iters):
    rhs, prep = C.c_double(), C.c_double()
    _abi.check(_abi.lib().ms_profile_rhs(dev.handle, _abi.dptr(x), SSS.c(), iters, C.byref(rhs), C.byref(prep)), "p")
    return rhs.value, prep.value
b, _ = prof(30)
with ClockSampler() as cs:
    s, p = prof(int(3000.0 / b))
print("JSON" + json.dumps({"burst_GBps": nbytes / b / 1e6, "sustained_GBps": nbytes / s / 1e6, "prep_us": p * 1e3,
                          "clocks": cs.summary()}))
''' % ROOT


def main(specs):
    for spec in specs or ["tma", "ldg", "tile"]:
        mode, _, lib = spec.partition(":")
        kss = os.environ.get("SW_KS", "f32" if mode == "tma" else "f32,f16")
        for ks in kss.split(","):
            env = dict(os.environ, MS_SWEEP=mode)
            if lib:
                env["MS_LIB_PATH"] = str(ROOT / "paper_2605_23727_b200" / "_variants" / f"lib_{lib}.so")
            r = subprocess.run([sys.executable, "-c", CHILD, ks], env=env, capture_output=True, text=True, timeout=900)
            line = [l for l in r.stdout.splitlines() if l.startswith("JSON")]
            print(spec, ks, line[0][4:] if line else r.stderr[-600:], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
