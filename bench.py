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
DATA = "synthetic (seeded SplitMix64: omega~N(0,1), K~U(0,2), theta0~U(0,2pi))"


def peaks(key="hbm_gbs", fallback=6650.0):
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        if key in d:
            return float(d[key]), "measured"
    return fallback, "fallback"


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


# ncu --set full of the K sweeps of one host-loop C4 attempt (tools/gpu_ncu_c4.sh <kdtype>)
TRAFFIC_CSV = "profiles/r2_c4_sweeps_{ks}_raw.csv"


def ncu_traffic(kernel_prefix, path):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the first
    launch whose name starts with `kernel_prefix` in the committed
    `ncu --set full` capture, or None."""
    import csv
    p = ROOT / path
    if not p.exists():
        return None
    rows = list(csv.reader(p.open()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if r[hdr.index("Kernel Name")].startswith(kernel_prefix):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(k)
                tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
            return tot
    return None


def sweep_kernel(kdtype, whole):
    """The dominant kernel of the benchmark solve (the K sweep that runs 2 of
    the 3 stage evaluations of an attempt) and its ncu DRAM traffic."""
    if kdtype == "f32" and os.environ.get("MS_SWEEP", "tma") == "tma":
        nxt = 1 if whole and os.environ.get("MS_FUSE_NEXT", "on") != "off" else 0
        name = f"void k_rhs_tma<float, float, 1, {nxt}>"
        label = f"k_rhs_tma<f32 sum, f32 G, K f32, NEXT={nxt}> (cp.async.bulk-fed K sweep" + \
                (", folds the next stage's prep)" if nxt else ")")
    elif kdtype == "f16" and os.environ.get("MS_SWEEP", "tc16") == "tc16":
        nxt = 1 if whole and os.environ.get("MS_FUSE_NEXT", "on") != "off" else 0
        name = f"void k_rhs_tc16<2, {nxt}>"
        label = (f"k_rhs_tc16<K f16, NEXT={nxt}> (tcgen05 M128 N16 sweep over 16 KB K tile images, f16 hi+lo "
                 "operands, binary32 sums of the 16-column dot products" +
                 (", folds the next stage's prep)" if nxt else ")"))
        kdtype = "f16tc"
    else:
        ks = {"f32": 1, "f16": 2, "bf16": 3}[kdtype]
        name = f"void k_rhs_fast<1, 1, float, float, {ks}>"
        label = f"k_rhs_fast<Kuramoto split, f32 sum, f32 G, K {kdtype}> (register-fed K sweep)"
    path = TRAFFIC_CSV.format(ks=kdtype)
    tr = ncu_traffic(name, path) if whole else None
    return label, tr, (f"{path} ({name}, ncu --set full, one launch)" if tr else None)


def mapped_repo_libs():
    """Shared objects under this repo mapped into the process (evidence that
    the reference arm runs only oracle/ code)."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return None
    return sorted({ln.split()[-1].replace(str(ROOT) + "/", "") for ln in maps
                   if ln.endswith(".so") and str(ROOT) in ln})


def workload_config(n, kdtype, ws):
    """The `config` dict of BOTH arms (identical, so the driver can pair them)."""
    return {"workload": f"C4 Kuramoto N={n} K {kdtype} (BASELINE configs[3])", "n_agents": n, "t_final": 20.0,
            "rtol": 1e-6, "atol": 1e-9, "policy": "SSS x3 rows, binary64 storage", "k_storage": kdtype,
            "l2": "K (4 GiB f32 / 2 GiB f16) > L2 (126 MB): no flush needed",
            "parallelism": (f"row-shard x{ws} (each stage's rows pushed into the peers' memory by the sweep, "
                            "NCCL all-gather if the peer mappings fail)") if ws > 1 else "single GPU"}


def dtype_label(kdtype):
    return f"{kdtype} (K storage), f32 (RHS rows) / f64 (stages, error control)"


def oracle_c4_inputs(n, seed, kdtype, rhs_mode):
    """C4's seeded inputs drawn with the ORACLE's SplitMix64 (rng.hpp:13-52) so
    the reference arm never maps this repo's library: omega ~ N(0,1) (stream 0),
    theta0 ~ U(0, 2 pi) (stream 1), K ~ U(0,2) (stream 2, filled by the oracle)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import _oracle as O
    from paper_2605_23727_b200.configs import SSS_D, TWO_PI
    from paper_2605_23727_b200.solver import SolverConfig
    from paper_2605_23727_b200.systems import SystemSpec
    omega = O.rng_normal(seed, 0, n)
    theta0 = O.rng_uniform(seed, 1, n, 0.0, TWO_PI)
    spec = SystemSpec("kuramoto", n, k_storage=kdtype, rhs_mode=rhs_mode, omega=omega, k_uniform=(seed, 2, 0.0, 2.0))
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    return O, spec, theta0, cfg, SSS_D


def cpu_prefix(n, seed, kdtype, threads, warm, timed, rhs_mode="faithful"):
    """The reference algorithm on the host cores over a bounded PREFIX of the
    real C4 solve: initial_step + cold k1 (untimed setup), then `warm` untimed
    and `timed` timed attempts of solve_core's loop (solver.cpp:255-347: the
    attempt is bs32_step = rk_step, solver.cpp:110-215; an accepted attempt
    moves t/x/k1 (FSAL), a rejected one recomputes k1 at the next attempt,
    :298-306), so rejections are timed where the solve takes them.
    rhs_mode "faithful" = the reference's eval_core order, one sinf per pair
    (systems.cpp:30-64, 141-143); "fast" = the oracle's split GEMV-2 form.
    OpenMP over rows keeps every row's j-sum sequential (bitwise the
    single-thread reference)."""
    O, spec, x0, cfg, policy = oracle_c4_inputs(n, seed, kdtype, rhs_mode)
    O.set_threads(threads)
    t0 = time.perf_counter()
    orc = O.OracleSystem(spec)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    h = O.initial_step(orc, 0.0, 20.0, x0, cfg)
    k1 = orc.eval_rhs(0.0, x0, policy.first_step_k1)
    t_setup = time.perf_counter() - t0
    t, x, need_k1, tf = 0.0, x0, False, 20.0
    rec = []
    for a in range(warm + timed):
        s0 = time.perf_counter()
        ev = 3
        if need_k1:
            k1 = orc.eval_rhs(t, x, policy.first_step_k1)
            need_k1, ev = False, 4
        h_att = tf - t if t + 1.01 * h >= tf else h
        o = O.bs32_step(orc, t, x, h_att, k1, policy, cfg)
        dt = time.perf_counter() - s0
        if o.accepted:
            x, t, k1 = o.x_store, t + h_att, o.k4
        else:
            need_k1 = True
        h = o.h_next
        rec.append((dt, bool(o.accepted), ev))
    tim = rec[warm:]
    secs = sum(r[0] for r in tim)
    acc = sum(r[1] for r in tim)
    evals = sum(r[2] for r in tim)
    return {"seconds": secs, "accepted": acc, "attempts": len(tim), "rejected": len(tim) - acc, "evals": evals,
            "per_attempt_s": [r[0] for r in tim], "k_gen_s": t_gen, "setup_s": t_setup, "t_reached": t,
            "threads": threads, "value": acc / secs if secs > 0 else 0.0,
            "per_eval_s": secs / max(evals, 1)}


def cpu_single_eval(n, seed, kdtype, threads, rhs_mode):
    """Seconds of ONE SSS-row RHS evaluation of C4 on `threads` host threads."""
    O, spec, x0, cfg, policy = oracle_c4_inputs(n, seed, kdtype, rhs_mode)
    O.set_threads(threads)
    orc = O.OracleSystem(spec)
    from paper_2605_23727_b200.precision import SSS
    t0 = time.perf_counter()
    orc.eval_rhs(0.0, x0, SSS)
    return time.perf_counter() - t0


def oracle_counts(kdtype):
    """The oracle's own whole-solve counts for C4 (tests/golden/solves, made by
    tools/make_golden_solves.py; the tests check them against live runs)."""
    p = ROOT / "tests" / "golden" / "solves" / f"c4_{kdtype}.npz"
    if not p.exists():
        return None
    d = np.load(p)
    return {"n_accepted": int(d["n_accepted"]), "n_failed": int(d["n_failed"]), "rhs_evals": int(d["rhs_evals"]),
            "final_state": d["final_state"]}


def project(per_eval_s, counts):
    """Accepted steps/s of the whole solve at a measured per-evaluation time,
    with the oracle's own evaluation count (3 + 3 accepted + 4 rejected)."""
    if not counts:
        return None
    return counts["n_accepted"] / (per_eval_s * counts["rhs_evals"])


def _c5_cpu_worker(item):
    """One host process, one oracle thread: trajectories [b0, b1) of the C5
    ensemble solved one after another (the reference's campaign model: B
    independent single-threaded solves over a pool, harness.cpp:424-456),
    inputs from the oracle's own SplitMix64 (rng.hpp:13-52)."""
    b0, b1, n, tf = item
    sys.path.insert(0, str(ROOT / "tests"))
    import _oracle as O
    from paper_2605_23727_b200.configs import SSS_D, TWO_PI
    from paper_2605_23727_b200.solver import SolverConfig
    from paper_2605_23727_b200.systems import SystemSpec
    O.set_threads(1)
    seed = 4
    spec = SystemSpec("kuramoto", n, k_storage="bf16", omega=np.zeros(n), k_uniform=(seed, 2, 0.0, 2.0))
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    orc = O.OracleSystem(spec)
    orc.set_op_round(3)  # MS_K_BF16: the tensor-core operand rounding (hi + lo bf16)
    omega = O.rng_normal(seed, 0, b1 * n).reshape(b1, n)
    x0 = O.rng_uniform(seed, 1, b1 * n, 0.0, TWO_PI).reshape(b1, n)
    acc = 0
    t = time.perf_counter()
    for b in range(b0, b1):
        orc.set_omega(omega[b])
        acc += O.solve(orc, x0[b], 0.0, tf, SSS_D, cfg, cap=1, snapshot_capacity=0).n_accepted
    return acc, time.perf_counter() - t


def c5_line(steps, cpu):
    """BASELINE.json configs[4] (C5) on this GPU: B=1024 trajectories x N=2048
    sharing a bf16 K, t in [0,20], rtol 1e-6: trajectory accepted steps/s of
    the whole lock-step solve (device time), the contraction's tensor-pipe
    rate, and the reference model on the host cores (one single-threaded
    oracle solve per core over a sample of trajectories)."""
    import ctypes as C
    from paper_2605_23727_b200 import _abi
    from paper_2605_23727_b200.batch import DeviceBatch
    from paper_2605_23727_b200.configs import config5_batch
    from paper_2605_23727_b200.precision import SSS
    from paper_2605_23727_b200.systems import DeviceSystem
    w = config5_batch()
    dev = DeviceSystem(w.spec)
    bat = DeviceBatch(dev, w.omega, tensor_cores=True)
    B, n = w.omega.shape
    rhs, prep = C.c_double(), C.c_double()
    x = np.ascontiguousarray(w.x0)
    _abi.check(_abi.lib().ms_batch_profile_rhs(bat._h, _abi.dptr(x), SSS.c(), 20, C.byref(rhs), C.byref(prep)), "prof")
    bat.solve(w.x0, w.t0, w.tf, w.policy, w.cfg)  # graph instantiation
    res = [bat.solve(w.x0, w.t0, w.tf, w.policy, w.cfg) for _ in range(steps)]
    ms = sum(r.device_ms for r in res)
    acc = sum(int(r.n_accepted.sum()) for r in res)
    flops = 2.0 * n * n * 2 * B
    peak, _ = peaks("bf16_tflops", 1682.1)
    tf = flops / (rhs.value * 1e-3) / 1e12
    out = {"workload": "C5 batched Kuramoto B=1024 N=2048 K bf16 (BASELINE configs[4]), t in [0,20], rtol 1e-6",
           "value": acc / (ms / 1e3), "unit": "trajectory_accepted_steps/s", "ms_per_solve": ms / steps,
           "lockstep_attempts": res[0].attempts, "accepted_per_traj_mean": float(res[0].n_accepted.mean()),
           "contraction": {"kernel": ("k_tc_gemm2 (tcgen05.mma.cta_group::2 kind::f16, 256-row x 128-trajectory pair "
                                      "tiles, hi+lo bf16 operands, sums in windows of "
                                      f"{os.environ.get('MS_TC_WINDOW', '2')} k-blocks added in binary32)"),
                           "ms": rhs.value, "TFLOPs_algorithmic": tf, "peak_bf16_TFLOPs": peak, "frac": tf / peak,
                           # the tensor pipe executes both operand terms (hi and lo): twice the algorithmic flops,
                           # on the 128 SMs the 64 pair tiles occupy
                           "TFLOPs_mma_issued": 2.0 * tf, "frac_mma_issued": 2.0 * tf / peak}}
    bat.close()
    dev.close()
    if cpu:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        cores = os.cpu_count() or 1
        k = min(cores, 16)
        t = time.perf_counter()
        with ProcessPoolExecutor(k, mp_context=mp.get_context("spawn")) as ex:
            parts = list(ex.map(_c5_cpu_worker, [(b, b + 1, n, w.tf) for b in range(k)]))
        wall = time.perf_counter() - t
        cacc = sum(p[0] for p in parts)
        out["cpu_baseline"] = {"value": cacc / wall, "unit": "trajectory_accepted_steps/s", "cores": k, "kind": "port",
                               "sample": f"trajectories 0..{k - 1} of the ensemble, whole t in [0,20] each, one "
                                         f"single-threaded oracle solve per process ({cacc} accepted steps in "
                                         f"{wall:.1f} s wall incl. process start and K generation)"}
    return out


def c4_f16_line(steps, seed):
    """C4 with K stored f16 (BASELINE.json configs[3] names fp32 and fp16 K):
    accepted steps/s over whole device-resident solves with the default f16
    sweep (the tensor-core k_rhs_tc16 at this N)."""
    import torch
    from paper_2605_23727_b200 import solver as S
    from paper_2605_23727_b200.configs import config4_kuramoto
    from paper_2605_23727_b200.systems import DeviceSystem
    w = config4_kuramoto(seed=seed, k_storage="f16")
    dev = DeviceSystem(w.spec)
    x0_d = torch.from_numpy(w.x0).to("cuda")
    xf_d = torch.empty_like(x0_d)
    st = torch.cuda.Stream()
    one = lambda: S.solve_device(dev, x0_d.data_ptr(), xf_d.data_ptr(), w.t0, w.tf, w.policy, w.cfg,  # noqa: E731
                                 stream=st.cuda_stream, log_capacity=0)
    one()
    res = [one() for _ in range(steps)]
    ms = sum(r.device_ms for r in res)
    dev.close()
    return {"workload": "C4 Kuramoto N=32768 K f16", "value": sum(r.n_accepted for r in res) / (ms / 1e3),
            "unit": UNIT, "ms_per_solve": ms / steps, "accepted_steps_per_solve": res[0].n_accepted,
            "rejected_per_solve": res[0].n_failed,
            "sweep": "k_rhs_tc16" if os.environ.get("MS_SWEEP", "tc16") == "tc16" else os.environ.get("MS_SWEEP")}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = args.n
    pre = cpu_prefix(n, args.seed, args.kdtype, threads, args.warmup, args.steps)
    value = pre["value"]
    counts = oracle_counts(args.kdtype) if n == 32768 else None
    extras = {}
    if not args.no_cpu_extras:
        t1 = cpu_single_eval(n, args.seed, args.kdtype, 1, "faithful")
        ts = cpu_single_eval(n, args.seed, args.kdtype, threads, "fast")
        extras = {
            "single_thread_faithful": {"eval_s": t1, "projected_value": project(t1, counts),
                                       "what": "one SSS eval_core evaluation (per-pair sinf) on 1 thread; value "
                                               "projected with the oracle's whole-solve evaluation count"},
            "all_cores_faithful_projected": project(pre["per_eval_s"], counts),
            "split_form_all_cores": {"eval_s": ts, "projected_value": project(ts, counts),
                                     "what": "the oracle's split GEMV-2 form (not the reference's order), "
                                             f"{threads} threads, one evaluation"},
        }
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": pre["seconds"] / max(pre["attempts"], 1) * 1e3,
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None,
        "dtype": dtype_label(args.kdtype), "data": DATA,
        "config": workload_config(n, args.kdtype, ws),
        "step_def": "one BS3(2) attempt of the real C4 solve prefix (after W untimed attempts)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"attempts {args.warmup + 1}..{args.warmup + args.steps} of the C4 solve "
                                   f"({pre['accepted']} accepted, {pre['rejected']} rejected, {pre['evals']} RHS "
                                   f"evals, t reached {pre['t_reached']:.4g}); reference eval_core order "
                                   f"(per-pair sinf, systems.cpp:30-64) restated in oracle/, OpenMP rows over "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "prefix": {k: pre[k] for k in ("seconds", "accepted", "rejected", "evals", "per_eval_s", "k_gen_s",
                                       "setup_s")},
        "oracle_whole_solve_counts": ({k: counts[k] for k in ("n_accepted", "n_failed", "rhs_evals")}
                                      if counts else None),
        **extras,
        "native_libs": mapped_repo_libs(),
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

    exchange = None
    if shard:
        from paper_2605_23727_b200.sharded import PushComm
        engine = DeviceEngine(dev)
        exchange = "push" if (ws > 1 and args.exchange == "push") else "nccl"
        solver = ShardedSolver(engine, PushComm() if exchange == "push" else TorchComm(), check_every=args.check_every)
        if exchange == "push":
            # the peer mappings are made on the first solve; any rank failing
            # there sends every rank to the NCCL all-gather
            ok = 1
            try:
                solver.solve(w.x0, w.t0, min(w.tf, 0.05), w.policy, w.cfg, log_capacity=0)
            except Exception as e:  # noqa: BLE001
                print(f"push exchange unavailable ({type(e).__name__}: {e}); NCCL all-gather", file=sys.stderr)
                ok = 0
            t = torch.tensor([ok], device=f"cuda:{local}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
            if int(t.item()) == 0:
                exchange = "nccl (push setup failed)"
                solver = ShardedSolver(engine, TorchComm(), check_every=args.check_every)

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
        from paper_2605_23727_b200 import _abi as _A
        launches0 = _A.lib().ms_launch_count()
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            for _ in range(args.steps):
                results.append(one())
            torch.cuda.synchronize()
        gpu_launches = _A.lib().ms_launch_count() - launches0
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
    replicas = None
    if ws > 1:
        # every rank holds the whole (replicated) final state and counts: they
        # must agree bit for bit across ranks, whichever exchange ran
        fs = np.ascontiguousarray(e2e_res[0].final_state)
        sig = float(np.frombuffer(fs.tobytes(), dtype=np.uint64).astype(np.float64).sum() % 1e15)
        v = torch.tensor([sig, float(e2e_res[0].n_accepted), float(e2e_res[0].n_failed)], device=f"cuda:{local}",
                         dtype=torch.float64)
        lo, hi = v.clone(), v.clone()
        torch.distributed.all_reduce(lo, op=torch.distributed.ReduceOp.MIN)
        torch.distributed.all_reduce(hi, op=torch.distributed.ReduceOp.MAX)
        replicas = bool(torch.equal(lo, hi))

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
    kname, traffic, traffic_src = sweep_kernel(args.kdtype, rows == n)

    # accuracy, outside the timed region: the benchmark solve
    # vs (1) the same-tolerance all-binary64 device BS3(2) run, (2) the tight
    # binary64 DP5(4) run at rel = abs = 1e-9 (dp54_reference, solver.cpp:472-483)
    # on the device, and (3) the oracle's own whole solve (counts and final
    # state from tests/golden/solves; its global error vs the same DP5(4) run)
    err = {}
    if not args.no_accuracy:
        r0_ = e2e_res[0]
        floor = w.cfg.abs_tol / w.cfg.rel_tol

        def dev_err(ref, x=None):
            x = r0_.final_state if x is None else x
            d = np.abs(x - ref)
            return {"max_abs": float(d.max()),
                    "max_rel_weighted": float(np.max(d / np.maximum(np.abs(ref), floor))),
                    "l2_over_sqrtN": float(np.linalg.norm(x - ref) / np.sqrt(n))}

        D = custom_policy((DDD, DDD, DDD), DDD, B64)
        rd = solver.solve(w.x0, w.t0, w.tf, D, w.cfg) if shard else S.solve(dev, w.x0, w.t0, w.tf, D, w.cfg)
        err["vs_binary64_bs32_same_tol"] = {**dev_err(rd.final_state), "steps": [rd.n_accepted, rd.n_failed]}
        if rows == n:
            t_dp = time.perf_counter()
            rdp = S.dp54_reference(dev, w.x0, w.t0, w.tf, S.SolverConfig(time_limits_enabled=False), log_capacity=1)
            err["vs_dp54_1e-9"] = {**dev_err(rdp.final_state), "status": int(rdp.status),
                                   "steps": [rdp.n_accepted, rdp.n_failed],
                                   "wall_s": round(time.perf_counter() - t_dp, 2),
                                   "what": "global error vs the tight binary64 DP5(4) device run (rel=abs=1e-9)"}
            oc = oracle_counts(args.kdtype) if n == 32768 else None
            if oc:
                of = oc["final_state"]
                err["oracle_vs_dp54_1e-9"] = dev_err(rdp.final_state, of)
                err["vs_oracle"] = {
                    "oracle_counts": [oc["n_accepted"], oc["n_failed"]],
                    "device_counts": [r0_.n_accepted, r0_.n_failed],
                    "accepted_within_1pct": bool(abs(r0_.n_accepted - oc["n_accepted"])
                                                 <= max(1, 0.01 * oc["n_accepted"])),
                    "rejected_within_1pct_of_attempts": bool(abs(r0_.n_failed - oc["n_failed"])
                                                             <= max(1, 0.01 * (oc["n_accepted"] + oc["n_failed"]))),
                    "final_state": dev_err(of),
                    "source": f"tests/golden/solves/c4_{args.kdtype}.npz (the oracle's whole solve)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": dtype_label(args.kdtype), "data": DATA,
        "config": workload_config(n, args.kdtype, ws),
        "step_def": "one full adaptive solve (t in [0,20], initial_step included)",
        "accepted_steps_per_solve": results[0].n_accepted, "rejected_per_solve": results[0].n_failed,
        "rhs_evals_per_solve": results[0].flops.rhs_evals,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "frac_nominal_8TBps": achieved / 8000.0,  # both denominators
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind, "kernel": kname,
                     "bytes_per_launch": bpe, "launch_ms": rhs_ms.value, "prep_ms": prep_ms.value,
                     "solve_effective_GBps": solve_gbs},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * 8,
                "d2h_bytes_per_step": n * 8 + log_bytes},
        "gpu_launches": gpu_launches,
        "exchange": exchange,
        "replicas_agree": replicas,
        "accuracy": err,
    }
    if rank == 0 and not args.no_cpu_baseline and ws == 1:
        thr = os.cpu_count() or 1
        cs = cpu_prefix(args.cpu_n or n, args.seed, args.kdtype, thr, 0, args.cpu_attempts)
        line["cpu_baseline"] = {"value": cs["value"], "unit": UNIT, "cores": thr, "kind": "port",
                                "sample": f"the first {cs['attempts']} attempts of the C4 solve (N={args.cpu_n or n}: "
                                          f"{cs['accepted']} accepted, {cs['evals']} RHS evals, {cs['seconds']:.1f} s) "
                                          "in the reference eval_core order (per-pair sinf, systems.cpp:30-64) "
                                          f"restated in oracle/, OpenMP rows over {thr} threads"}
    line["clocks"] = clk.summary()
    if rank == 0 and ws == 1 and not args.no_also and args.n == 32768:
        # the other stated configurations this GPU runs, measured after the
        # headline (informative; not part of the timed region above)
        also = {}
        # an extra that fails is reported, never allowed to cost the headline line
        try:
            if args.kdtype == "f32":
                also["c4_f16"] = c4_f16_line(2, args.seed)
        except Exception as e:  # noqa: BLE001
            also["c4_f16"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        try:
            also["c5"] = c5_line(2, not args.no_cpu_baseline)
        except Exception as e:  # noqa: BLE001
            also["c5"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        line["also"] = also
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
    ap.add_argument("--cpu-attempts", type=int, default=3, help="attempts timed by the GPU arm's cpu_baseline leg")
    ap.add_argument("--no-cpu-extras", action="store_true", help="reference arm: skip the 1-thread/split extras")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--shard", action="store_true", help="use the row-sharded loop even on 1 GPU")
    ap.add_argument("--check-every", type=int, default=8)
    ap.add_argument("--no-also", action="store_true", help="skip the C4-f16 and C5 lines after the headline")
    ap.add_argument("--exchange", default="push", choices=["push", "nccl"],
                    help="row-sharded runs (N>1): rows pushed into peer memory by the sweeps, or NCCL all-gather")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
