"""C5 accuracy: the sampled trajectories' global error (weighted like Eq. 7,
floor ab/rel) against each trajectory's tight binary64 DP5(4) run (rel = abs =
1e-9), for the tensor-core ensemble, the CUDA-core ensemble (binary32 split on
CUDA cores, no operand rounding) and the oracle's solves with the tensor-core
operand rounding (fixture c5_bf16). Prints one JSON line per trajectory."""
import copy
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import golden_cases as G  # noqa: E402
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.batch import DeviceBatch  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

w = G.CASES["c5_bf16"]["build"]()
d = G.load("c5_bf16")
dev = DeviceSystem(w.spec)
out = {}
for tc in (True, False):
    bat = DeviceBatch(dev, w.omega, tensor_cores=tc)
    r = bat.solve(w.x0, w.t0, w.tf, w.policy, w.cfg)
    out[tc] = r
    print(json.dumps({"tensor_cores": tc, "accepted": int(r.n_accepted.sum()), "rejected": int(r.n_failed.sum()),
                      "ms": r.device_ms}), flush=True)
    bat.close()
floor = w.cfg.abs_tol / w.cfg.rel_tol
wrel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))  # noqa: E731
rows = []
for k, b in enumerate(d["sample"]):
    spec = copy.copy(w.spec)
    spec.omega = np.ascontiguousarray(w.omega[b])
    one = DeviceSystem(spec)
    ref = S.dp54_reference(one, w.x0[b], w.t0, w.tf, S.SolverConfig(time_limits_enabled=False), log_capacity=1)
    one.close()
    row = {"traj": int(b), "tc": wrel(out[True].final_state[b], ref.final_state),
           "cuda_core": wrel(out[False].final_state[b], ref.final_state),
           "oracle": wrel(d["final_states"][k], ref.final_state),
           "tc_vs_oracle": wrel(out[True].final_state[b], d["final_states"][k])}
    rows.append(row)
    print(json.dumps(row), flush=True)
for key in ("tc", "cuda_core", "oracle"):
    v = np.array([r[key] for r in rows])
    print(json.dumps({"summary": key, "median": float(np.median(v)), "max": float(v.max())}))
# the single-solve gate (tests/_gates.py): device global error <= 1.5 x the oracle's + 1e-7
g = [r["tc"] / (1.5 * r["oracle"] + 1e-7) for r in rows]
print(json.dumps({"summary": "gate_ratio_tc", "max": float(max(g)), "worst_traj": rows[int(np.argmax(g))]["traj"]}))
