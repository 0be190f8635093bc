"""C5 experiment: the ensemble split into G independent trajectory groups, each
its own ms_batch handle (own stream, own lock-step loop graph) over the one
shared K, solved concurrently from G host threads. One group's memory-bound
preps/finalize can then overlap another group's tensor-core contraction.
Prints one JSON line per G (wall-clock over the concurrent solves)."""
import argparse
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200.batch import DeviceBatch  # noqa: E402
from paper_2605_23727_b200.configs import config5_batch  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--groups", default="1,2,4")
ap.add_argument("--tf", type=float, default=20.0)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
w = config5_batch(tf=a.tf)
dev = DeviceSystem(w.spec)
B = w.omega.shape[0]
ref = None
for G in [int(g) for g in a.groups.split(",")]:
    cuts = [B * k // G for k in range(G + 1)]
    bats = [DeviceBatch(dev, w.omega[cuts[k]:cuts[k + 1]]) for k in range(G)]
    xs = [np.ascontiguousarray(w.x0[cuts[k]:cuts[k + 1]]) for k in range(G)]
    out = [None] * G

    def run(k):
        out[k] = bats[k].solve(xs[k], w.t0, w.tf, w.policy, w.cfg)

    def once():
        th = [threading.Thread(target=run, args=(k,)) for k in range(G)]
        t = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        return time.perf_counter() - t

    once()  # warm-up: graph instantiation
    walls = [once() for _ in range(a.reps)]
    acc = sum(int(r.n_accepted.sum()) for r in out)
    fin = np.concatenate([r.final_state for r in out])
    na = np.concatenate([r.n_accepted for r in out])
    same = None
    if ref is None:
        ref = (fin, na)
    else:
        same = bool(np.array_equal(fin, ref[0]) and np.array_equal(na, ref[1]))
    wall = min(walls)
    print(json.dumps({"groups": G, "wall_ms": wall * 1e3, "walls_ms": [x * 1e3 for x in walls],
                      "device_ms": [r.device_ms for r in out], "attempts": [r.attempts for r in out],
                      "value": acc / wall, "unit": "trajectory_accepted_steps/s", "bitwise_vs_G1": same}),
          flush=True)
    for b in bats:
        b.close()
