"""Concurrent policy variants against the harness's sequential
runs (harness.cpp:113-121): the four named variants of one case solved one
after another vs in lock-step with one K sweep per stage. Device time from the
library's CUDA events. One JSON line per workload."""
import argparse
import json
import sys

import numpy as np
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config2_kuramoto, config4_kuramoto  # noqa: E402
from paper_2605_23727_b200.precision import PolicyVariant, policy_for  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="c2,c4")
ap.add_argument("--c4-tf", type=float, default=2.0)
a = ap.parse_args()
NAMES = ("Single", "Mixed1", "Mixed2", "Double")
POLS = [policy_for(getattr(PolicyVariant, n)) for n in NAMES]
for wl in a.workloads.split(","):
    if wl == "c2":
        w, tf = config2_kuramoto(rtol=1e-6), 50.0
    else:
        w, tf = config4_kuramoto(), a.c4_tf
    dev = DeviceSystem(w.spec)
    cfg = w.cfg
    seq = [S.solve(dev, w.x0, w.t0, tf, p, cfg, log_capacity=1) for p in POLS]  # warm-up (graphs)
    seq = [S.solve(dev, w.x0, w.t0, tf, p, cfg, log_capacity=1) for p in POLS]
    v = S.DeviceVariants(dev, 4)
    v.solve(w.x0, w.t0, tf, POLS, cfg, log_capacity=1)
    conc = v.solve(w.x0, w.t0, tf, POLS, cfg, log_capacity=1)
    same = all((c.n_accepted, c.n_failed) == (s.n_accepted, s.n_failed) and (c.final_state == s.final_state).all()
               for c, s in zip(conc, seq))
    seq_ms = sum(r.device_ms for r in seq)
    # accuracy of every variant against the tight binary64 DP5(4) run
    # (solver.cpp:472-483; metrics.cpp:10-17 for the l2/sqrt(N) column)
    ref = S.dp54_reference(dev, w.x0, w.t0, tf, S.SolverConfig(time_limits_enabled=False), log_capacity=1)
    floor = cfg.abs_tol / cfg.rel_tol
    acc = {}
    for n_, r in zip(NAMES, conc):
        d = np.abs(r.final_state - ref.final_state)
        acc[n_] = {"max_abs": float(d.max()),
                   "max_rel_weighted": float(np.max(d / np.maximum(np.abs(ref.final_state), floor))),
                   "l2_over_sqrtN": float(np.linalg.norm(d) / np.sqrt(w.spec.n_agents))}
    line = {"workload": f"{wl.upper()} Kuramoto N={w.spec.n_agents} K {w.spec.k_storage}, t in [0,{tf}], "
                        f"rtol {cfg.rel_tol:g}, variants {'/'.join(NAMES)}",
            "sequential_ms": seq_ms, "per_variant_ms": {n: r.device_ms for n, r in zip(NAMES, seq)},
            "concurrent_ms": conc[0].device_ms, "speedup": seq_ms / conc[0].device_ms,
            "accepted": {n: r.n_accepted for n, r in zip(NAMES, conc)},
            "rejected": {n: r.n_failed for n, r in zip(NAMES, conc)},
            "bitwise_equal_to_sequential": bool(same),
            "error_vs_dp54_1e-9": acc, "dp54_steps": [ref.n_accepted, ref.n_failed]}
    print(json.dumps(line), flush=True)
    v.close()
    dev.close()
