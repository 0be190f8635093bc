"""Whole C4 solves (device-resident, ms_solve_device) with alternative builds of
the library, alternating on one box: accepted steps/s per build.
usage: python tools/ab_solve.py <kdtype> <lib-name|cur> ...   (libs under paper_2605_23727_b200/_variants)"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, json
sys.path.insert(0, "%s")
import torch
from paper_2605_23727_b200 import solver as S
from paper_2605_23727_b200.configs import config4_kuramoto
from paper_2605_23727_b200.systems import DeviceSystem
w = config4_kuramoto(k_storage=sys.argv[1])
dev = DeviceSystem(w.spec)
x0 = torch.from_numpy(w.x0).cuda(); xf = torch.empty_like(x0)
one = lambda: S.solve_device(dev, x0.data_ptr(), xf.data_ptr(), w.t0, w.tf, w.policy, w.cfg, log_capacity=0)
one(); one()
rs = [one() for _ in range(3)]
ms = sum(r.device_ms for r in rs); acc = sum(r.n_accepted for r in rs)
print("JSON" + json.dumps({"steps_per_s": acc / ms * 1e3, "ms_per_solve": ms / 3, "acc": rs[0].n_accepted, "rej": rs[0].n_failed}))
''' % ROOT

ks, libs = sys.argv[1], sys.argv[2:]
for rnd in range(2):
    for lib in libs:
        env = dict(os.environ)
        if lib != "cur":
            env["MS_LIB_PATH"] = str(ROOT / "paper_2605_23727_b200" / "_variants" / f"lib_{lib}.so")
        r = subprocess.run([sys.executable, "-c", CHILD, ks], env=env, capture_output=True, text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("JSON")]
        print(ks, lib, line[0][4:] if line else r.stderr[-500:], flush=True)
