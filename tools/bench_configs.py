"""Device solves of BASELINE.json configs 1-3 (+ C4 f16 and C5 summaries come
from bench.py / tools/bench_c5.py) with a CPU-oracle sample beside each.
Writes one JSON object per line (profiles/r1_configs.jsonl)."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import _oracle as O  # noqa: E402
from paper_2605_23727_b200 import solver as S  # noqa: E402
from paper_2605_23727_b200.configs import config1_lco, config2_kuramoto, config3_cc  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402


def cpu_attempt_s(w, attempts=2):
    O.set_threads(os.cpu_count() or 1)
    orc = O.OracleSystem(w.spec)
    h0 = O.initial_step(orc, w.t0, w.tf, w.x0, w.cfg)
    k1 = orc.eval_rhs(0.0, w.x0, w.policy.first_step_k1)
    t = time.perf_counter()
    for _ in range(attempts):
        O.bs32_step(orc, 0.0, w.x0, h0, k1, w.policy, w.cfg)
    return (time.perf_counter() - t) / attempts


FINALS = {}


def run(name, w, reps=2, compare_to=None):
    dev = DeviceSystem(w.spec)
    S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)  # warm-up (graph instantiation)
    rs = [S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg) for _ in range(reps)]
    FINALS[name] = rs[0].final_state
    ms = sum(r.device_ms for r in rs) / reps
    r = rs[0]
    cpu = cpu_attempt_s(w)
    att_per_acc = (r.n_accepted + r.n_failed) / max(r.n_accepted, 1)
    line = {"config": name, "n": w.spec.n_agents, "k": w.spec.k_storage, "rtol": w.cfg.rel_tol,
            "status": S.status_name(r.status), "accepted": r.n_accepted, "rejected": r.n_failed,
            "device_ms_per_solve": ms, "accepted_steps_per_s": r.n_accepted / (ms / 1e3),
            "cpu_oracle_s_per_attempt": cpu, "cpu_cores": os.cpu_count(),
            "cpu_oracle_accepted_steps_per_s_est": 1.0 / (cpu * att_per_acc),
            "speedup_vs_cpu_est": (r.n_accepted / (ms / 1e3)) * cpu * att_per_acc}
    if compare_to in FINALS:
        # K storage effect: the same solve with K rounded to f16 vs K in f32
        # (weighted like Eq. 7, floor atol/rtol)
        ref = FINALS[compare_to]
        d = np.abs(r.final_state - ref) / np.maximum(np.abs(ref), w.cfg.abs_tol / w.cfg.rel_tol)
        line["final_state_vs"] = {"run": compare_to, "max_rel_weighted": float(d.max())}
    print(json.dumps(line), flush=True)
    dev.close()


if __name__ == "__main__":
    run("C1 LCO N=1024 K f32", config1_lco())
    for ks in ("f32", "f16"):
        for rtol in (1e-3, 1e-4, 1e-6, 1e-8):
            run(f"C2 Kuramoto N=4096 K {ks} rtol {rtol:g}", config2_kuramoto(rtol=rtol, k_storage=ks), reps=1,
                compare_to=f"C2 Kuramoto N=4096 K f32 rtol {rtol:g}" if ks == "f16" else None)
    run("C3 CC N=2048 K f32 t in [0,240]", config3_cc(), reps=1)
