#!/usr/bin/env python
"""Benchmark of the hot path: Kuramoto N=32768 BS3(2) (BASELINE.json configs[3],
the metric's workload) on B200.

One bench "step" = one full adaptive solve of C4 (t in [0,20], rtol 1e-6,
atol 1e-9, policy {SSS x3, binary64 storage}, K f32 row-major 4 GiB resident in
HBM). ``value`` = accepted BS3(2) steps/s over the timed solves with inputs
resident on the device (ms_solve_device); ``e2e`` = the same through the
reference-facing call ms_solve with host x0 / host final state (H2D + D2H
inside the timed region). K (4 GiB) is larger than L2 (126 MB), so no flush is
needed between iterations.

``--impl reference`` times the reference algorithm on the host cores: the CPU
oracle (a line-by-line restatement of proj/src/{systems,solver}.cpp, compiled
-O3 -ffp-contract=off, OpenMP over rows — bitwise the sequential reference) on
a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Kuramoto N=32768 BS3(2) accepted steps/s"
UNIT = "accepted_steps/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.rows = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].strip().lower() == "active"})
        pw = [float(r[3]) for r in self.rows if len(r) > 3 and r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w": statistics.median(pw) if pw else None}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def bytes_per_eval(n, rows, ks_bytes):
    # N^2 s_K + (dN s_G + 2 dN 8 + p N 8); here the K rows of
    # this rank, the sin/cos vectors (f32), x in / k out (f64) and omega
    return rows * n * ks_bytes + n * 2 * 4 + 2 * n * 8 + n * 8


def ncu_traffic(kernel_prefix):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed `ncu --set full` capture (profiles/), or None."""
    import csv
    p = ROOT / "profiles" / "r1_k_rhs_tma_f32_raw.csv"
    if not p.exists():
        return None
    rows = list(csv.reader(p.open()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if kernel_prefix in r[hdr.index("Kernel Name")]:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(k)
                tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
            return tot
    return None


def cpu_sample(n, seed, threads, attempts=2, ks="f32"):
    """The oracle on a bounded sample of C4: `attempts` BS3(2) attempts from
    theta0 at the initial step (3 RHS evaluations each), OpenMP over rows."""
    sys.path.insert(0, str(ROOT / "tests"))
    import _oracle as O
    from paper_2605_23727_b200.configs import config4_kuramoto
    w = config4_kuramoto(n=n, seed=seed, k_storage=ks)
    O.set_threads(threads)
    t0 = time.perf_counter()
    orc = O.OracleSystem(w.spec)
    t_gen = time.perf_counter() - t0
    h0 = O.initial_step(orc, w.t0, w.tf, w.x0, w.cfg)
    k1 = orc.eval_rhs(0.0, w.x0, w.policy.first_step_k1)
    times = []
    acc = 0
    for _ in range(attempts):
        t0 = time.perf_counter()
        o = O.bs32_step(orc, 0.0, w.x0, h0, k1, w.policy, w.cfg)
        times.append(time.perf_counter() - t0)
        acc += int(o.accepted)
    return {"per_attempt_s": float(np.mean(times)), "attempts": attempts, "accepted": acc,
            "k_gen_s": t_gen, "h0": h0}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = args.n
    res = []
    sample = cpu_sample(n, args.seed, threads, attempts=args.warmup + args.steps, ks=args.kdtype)
    per = sample["per_attempt_s"]
    value = 1.0 / per  # every sampled attempt is accepted at h0 (checked below)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (RHS) / f64 (stages)", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": f"C4 Kuramoto N={n} K {args.kdtype}", "n_agents": n, "t_final": 20.0,
                   "rtol": 1e-6, "atol": 1e-9, "policy": "SSS x3, binary64 storage"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample['attempts']} BS3(2) attempts (3 RHS evals each) of C4 from theta0 at h0; "
                                   f"oracle restatement, OpenMP rows over {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "accepted_in_sample": sample["accepted"],
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    ws, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_23727_b200 import solver as S
    from paper_2605_23727_b200.configs import config4_kuramoto
    from paper_2605_23727_b200.precision import DDD, B64, custom_policy
    from paper_2605_23727_b200.systems import DeviceSystem

    n = args.n
    shard = ws > 1 or args.shard
    w = config4_kuramoto(n=n, seed=args.seed, k_storage=args.kdtype)
    w.spec.device = local
    rows = n
    if shard:
        from paper_2605_23727_b200.sharded import DeviceEngine, ShardedSolver, TorchComm, row_range
        if ws == 1 and not torch.distributed.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            torch.distributed.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        r0, r1 = row_range(n, rank, ws)
        w.spec.row_begin, w.spec.row_end = r0, r1
        rows = r1 - r0
    dev = DeviceSystem(w.spec)  # K (this rank's rows) generated on the device, resident
    stream = torch.cuda.Stream()

    if shard:
        solver = ShardedSolver(DeviceEngine(dev), TorchComm(), check_every=args.check_every)

        def one():
            return solver.solve(w.x0, w.t0, w.tf, w.policy, w.cfg, log_capacity=0)
    else:
        x0_d = torch.from_numpy(w.x0).to(f"cuda:{local}")
        xf_d = torch.empty_like(x0_d)

        def one():
            return S.solve_device(dev, x0_d.data_ptr(), xf_d.data_ptr(), w.t0, w.tf, w.policy, w.cfg,
                                  stream=stream.cuda_stream, log_capacity=0)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        results = []
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            for _ in range(args.steps):
                results.append(one())
            torch.cuda.synchronize()
    # device time of each solve: CUDA events recorded by the library on its stream
    # around the whole adaptive loop (initial step included)
    ms = float(sum(r.device_ms for r in results))
    if ws > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    acc = sum(r.n_accepted for r in results)
    att = sum(r.n_accepted + r.n_failed for r in results)
    evals = sum(r.flops.rhs_evals for r in results)
    launched_evals = evals - sum(r.n_failed for r in results)  # elided k1 recomputes are counted, not run
    # sharded: all ranks cooperate on one solve (strong scaling); replicas would multiply
    value = acc / (ms / 1e3)
    ms_per_step = ms / args.steps

    # e2e: the public call with host buffers (H2D x0, D2H final state (+ log on 1 GPU));
    # one untimed call first (its own graph instantiation and log buffers)
    def e2e_one():
        if shard:
            return solver.solve(w.x0, w.t0, w.tf, w.policy, w.cfg, log_capacity=None)
        return S.solve(dev, w.x0, w.t0, w.tf, w.policy, w.cfg)

    e2e_one()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_res = [e2e_one() for _ in range(args.steps)]
    e2e_s = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = sum(r.n_accepted for r in e2e_res) / e2e_s
    log_bytes = max(r.step_log_count for r in e2e_res) * 32

    # roofline of the dominant kernel (this rank's K sweep), CUDA events on its stream
    from paper_2605_23727_b200.precision import SSS
    import ctypes as C
    from paper_2605_23727_b200 import _abi
    rhs_ms, prep_ms = C.c_double(), C.c_double()
    x0c = np.ascontiguousarray(w.x0)
    _abi.check(_abi.lib().ms_profile_rhs(dev.handle, _abi.dptr(x0c), SSS.c(), 20, C.byref(rhs_ms), C.byref(prep_ms)),
               "profile_rhs")
    ks_bytes = {"f32": 4, "f16": 2, "bf16": 2}[args.kdtype]
    bpe = bytes_per_eval(n, rows, ks_bytes)
    peak, peak_kind = peaks()
    achieved = bpe / (rhs_ms.value * 1e-3) / 1e9
    solve_gbs = launched_evals / args.steps * bpe / (ms_per_step * 1e-3) / 1e9

    # accuracy: device SSS solve vs the same-tolerance all-binary64 device solve
    err = {}
    if not args.no_accuracy:
        D = custom_policy((DDD, DDD, DDD), DDD, B64)
        rd = solver.solve(w.x0, w.t0, w.tf, D, w.cfg) if shard else S.solve(dev, w.x0, w.t0, w.tf, D, w.cfg)
        r0_ = e2e_res[0]
        diff = np.abs(r0_.final_state - rd.final_state)
        err = {"vs": "device all-binary64 BS3(2), same rtol/atol",
               "max_abs": float(diff.max()),
               "max_rel_weighted": float(np.max(diff / np.maximum(np.abs(rd.final_state), w.cfg.abs_tol / w.cfg.rel_tol))),
               "l2_over_sqrtN": float(np.linalg.norm(r0_.final_state - rd.final_state) / np.sqrt(n)),
               "double_steps": [rd.n_accepted, rd.n_failed]}

    # launches per attempt: (prep + sweep [+ scan]) x 3 + finalize [+ fsal copy]; the f32
    # TMA sweep of stages 1 and 2 also runs the next stage's prep (MS_FUSE_NEXT), 5 then
    sweep_env = os.environ.get("MS_SWEEP", "tma")
    folded = (not shard and args.kdtype == "f32" and os.environ.get("MS_FUSE_NEXT", "on") != "off"
              and sweep_env not in ("ldg", "tile", "small"))
    per_attempt = 11 if shard else (5 if folded else 7)
    gpu_launches = sum(10 + per_attempt * (r.n_accepted + r.n_failed) for r in results)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "f32 (RHS, K) / f64 (stages, error control)",
        "data": "synthetic (seeded SplitMix64: omega~N(0,1), K~U(0,2), theta0~U(0,2pi))",
        "config": {"workload": f"C4 Kuramoto N={n} K {args.kdtype} (BASELINE configs[3])", "n_agents": n,
                   "t_final": 20.0, "rtol": 1e-6, "atol": 1e-9, "policy": "SSS x3 rows, binary64 storage",
                   "step": "one full adaptive solve", "l2": "K (4 GiB) > L2: no flush needed",
                   "parallelism": f"row-shard x{ws} (NCCL all-gather per stage)" if shard else "single GPU"},
        "accepted_steps_per_solve": results[0].n_accepted, "rejected_per_solve": results[0].n_failed,
        "rhs_evals_per_solve": results[0].flops.rhs_evals,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "frac_nominal_8TBps": achieved / 8000.0,  # both denominators
                     "traffic": (ncu_traffic("k_rhs_tma<float, float, 1>")
                                 if args.kdtype == "f32" and rows == n and os.environ.get("MS_SWEEP", "tma") != "ldg"
                                 else None),
                     "traffic_source": "profiles/r1_k_rhs_tma_f32_raw.csv (ncu --set full, one launch)",
                     "peak_kind": peak_kind,
                     "kernel": ("k_rhs_tma<f32, f32, K f32> (cp.async.bulk-fed K sweep)" if args.kdtype == "f32"
                                and os.environ.get("MS_SWEEP", "tma") != "ldg"
                                else f"k_rhs_fast<Kuramoto split, f32, f32, K {args.kdtype}>"),
                     "bytes_per_launch": bpe, "launch_ms": rhs_ms.value, "prep_ms": prep_ms.value,
                     "solve_effective_GBps": solve_gbs},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * 8,
                "d2h_bytes_per_step": n * 8 + log_bytes},
        "gpu_launches": gpu_launches,
        "accuracy": err,
    }
    if rank == 0 and not args.no_cpu_baseline and ws == 1:
        cs = cpu_sample(args.cpu_n or n, args.seed, os.cpu_count() or 1, attempts=1, ks=args.kdtype)
        line["cpu_baseline"] = {"value": 1.0 / cs["per_attempt_s"], "unit": UNIT, "cores": os.cpu_count() or 1,
                                "kind": "port",
                                "sample": f"1 BS3(2) attempt (3 RHS evals) of C4 N={args.cpu_n or n} from theta0 at h0, "
                                          "oracle restatement, OpenMP rows"}
    line["clocks"] = clk.summary()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    dev.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--kdtype", default="f32", choices=["f32", "f16", "bf16"])
    ap.add_argument("--cpu-n", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--shard", action="store_true", help="use the row-sharded loop even on 1 GPU")
    ap.add_argument("--check-every", type=int, default=8)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
