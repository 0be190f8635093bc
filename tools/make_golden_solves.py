"""Generate the whole-solve golden fixtures under tests/golden/solves/ with the
CPU oracle (TEST INFRASTRUCTURE: this script runs in the build container, not on
the GPU box; the -m gpu tests compare device solves against its outputs).

The oracle (oracle/mixedstep_oracle.cpp) restates proj/src/solver.cpp:226-347
and systems.cpp:30-189; its rows are summed sequentially in ascending j, so its
results do not depend on the thread count. Each fixture records the oracle
source hash and a hash of the inputs, so a stale fixture is detected
(tests/test_golden_solves.py).

  python tools/make_golden_solves.py [case ...]     (default: every case)
"""
from __future__ import annotations

import hashlib
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
from golden_cases import CASES, OUT, input_hash, oracle_source_hash  # noqa: E402


def _log_arrays(res):
    return (np.array([s.t for s in res.step_log]), np.array([s.h for s in res.step_log]),
            np.array([s.err for s in res.step_log]), np.array([s.accepted for s in res.step_log], dtype=np.int8))


def run_single(name, case):
    w = case["build"]()
    orc = O.OracleSystem(w.spec)
    t = time.perf_counter()
    o = O.solve(orc, w.x0, w.t0, w.tf, w.policy, w.cfg, cap=400000, snapshot_capacity=0)
    dt = time.perf_counter() - t
    lt, lh, le, la = _log_arrays(o) if case.get("log", True) else (np.zeros(0),) * 3 + (np.zeros(0, np.int8),)
    meta = {"case": name, "what": case["what"], "oracle_src": oracle_source_hash(), "inputs": input_hash(w),
            "oracle_s": dt, "threads": O.lib().orc_get_threads(), "t0": w.t0, "tf": w.tf}
    np.savez_compressed(OUT / f"{name}.npz", final_state=o.final_state, status=int(o.status),
                        n_accepted=o.n_accepted, n_failed=o.n_failed, t_reached=o.t_reached,
                        rhs_evals=o.flops.rhs_evals, flops_low=o.flops.low, flops_high=o.flops.high,
                        log_t=lt, log_h=lh, log_err=le, log_acc=la, meta=json.dumps(meta))
    print(f"{name}: {o.status.name} {o.n_accepted}/{o.n_failed} evals {o.flops.rhs_evals} in {dt:.1f} s", flush=True)


def _batch_worker(args):
    """One process, one oracle thread: a contiguous block of trajectories."""
    name, b0, b1 = args
    case = CASES[name]
    O.set_threads(1)
    w = case["build"]()
    orc = O.OracleSystem(w.spec)
    orc.set_op_round(case["op_round"])
    out = []
    for b in range(b0, b1):
        orc.set_omega(w.omega[b])
        o = O.solve(orc, w.x0[b], w.t0, w.tf, w.policy, w.cfg, cap=1, snapshot_capacity=0)
        fs = o.final_state if b in case["sample"] else None
        out.append((b, o.n_accepted, o.n_failed, o.flops.rhs_evals, int(o.status), o.t_reached, fs))
    return out


def run_batch(name, case):
    """Every trajectory of the ensemble through the oracle (per-trajectory
    omega, shared K, the tensor-core operand rounding); counts for all of them,
    final states for the sampled ones. Trajectories are independent solves
    (the reference's campaign model, harness.cpp:449-456): one single-threaded
    oracle process per core."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    w = case["build"]()
    B = w.omega.shape[0]
    sample = np.array(case["sample"], dtype=np.int64)
    acc, rej, evals, status, tr = (np.zeros(B, np.int64), np.zeros(B, np.int64), np.zeros(B, np.int64),
                                   np.zeros(B, np.int32), np.zeros(B))
    finals = np.zeros((sample.size, w.x0.shape[1]))
    t = time.perf_counter()
    nproc = os.cpu_count() or 1
    blocks = [(name, B * k // (4 * nproc), B * (k + 1) // (4 * nproc)) for k in range(4 * nproc)]
    done = 0
    with ProcessPoolExecutor(nproc, mp_context=mp.get_context("spawn")) as ex:
        for part in ex.map(_batch_worker, blocks):
            for b, a_, r_, e_, s_, t_, fs in part:
                acc[b], rej[b], evals[b], status[b], tr[b] = a_, r_, e_, s_, t_
                if fs is not None:
                    finals[int(np.nonzero(sample == b)[0][0])] = fs
            done += len(part)
            print(f"  {name}: {done}/{B} trajectories, {time.perf_counter() - t:.0f} s", flush=True)
    dt = time.perf_counter() - t
    meta = {"case": name, "what": case["what"], "oracle_src": oracle_source_hash(), "inputs": input_hash(w),
            "oracle_s": dt, "threads": nproc, "t0": w.t0, "tf": w.tf}
    np.savez_compressed(OUT / f"{name}.npz", sample=sample, final_states=finals, n_accepted=acc, n_failed=rej,
                        rhs_evals=evals, status=status, t_reached=tr, meta=json.dumps(meta))
    print(f"{name}: {int(acc.sum())}/{int(rej.sum())} over {B} trajectories in {dt:.1f} s", flush=True)


if __name__ == "__main__":
    O.set_threads(os.cpu_count() or 1)
    OUT.mkdir(parents=True, exist_ok=True)
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        c = CASES[nm]
        (run_batch if c.get("batch") else run_single)(nm, c)
